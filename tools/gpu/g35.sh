#!/bin/bash
# tile interleave A/B (TD_TILE_INTERLEAVE) on configs 3 and 2
mkdir -p gpurun_out
for pass in 1 2 3; do
for cfg in cfg3 cfg2; do
for b in 0 1; do
  echo "pass $pass $cfg interleave $b" >> gpurun_out/g35.txt
  TD_TILE_INTERLEAVE=$b timeout 600 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python tools/_bench_brief.py >> gpurun_out/g35.txt
done
done
done
TD_TILE_INTERLEAVE=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_gpu.py -x -q -m gpu 2>&1 | tail -2 >> gpurun_out/g35.txt
cat gpurun_out/g35.txt
