#!/bin/bash
# grid balance A/B on config-5 sizes (small_probe) and the config-3 bench
set -x
mkdir -p gpurun_out
for gb in 0 1; do
  TD_GRID_BALANCE=$gb timeout 600 python tools/small_probe.py --sizes 16,64,256,1024,4096 --targets 1184,2368 --bps 2,3,4 --reps 20 > gpurun_out/g33_gb$gb.jsonl 2>&1
done
for gb in 0 1 0 1; do
  TD_GRID_BALANCE=$gb timeout 600 python bench.py --steps 20 --warmup 3 2>/dev/null | tail -1 | python tools/_bench_brief.py >> gpurun_out/g33_bench.txt
done
cat gpurun_out/g33_bench.txt
