#!/bin/bash
# td_segnorm CTAs/SM A/B (TD_BLOCKS_PER_SM) across configs
mkdir -p gpurun_out
for pass in 1 2; do
for cfg in cfg3 cfg2 cfg5:1024 cfg5:4096; do
for b in 3 4; do
  echo "pass $pass $cfg bps $b" >> gpurun_out/g34.txt
  TD_BLOCKS_PER_SM=$b timeout 600 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python tools/_bench_brief.py >> gpurun_out/g34.txt
done
done
done
cat gpurun_out/g34.txt
