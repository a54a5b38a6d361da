#!/bin/bash
# small-tensor probe under ncu: per-launch kernel durations (cold caches)
set -x
mkdir -p gpurun_out
timeout 600 python tools/small_probe.py --sizes 1,16,64 --targets 1184 --bps 4 --reps 5 > gpurun_out/g31_small.jsonl 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_active.avg --clock-control none --csv \
  --log-file gpurun_out/g31_ncu.csv python tools/small_probe.py --sizes 1,16,64 --targets 1184 --bps 4 --reps 3 > gpurun_out/g31_ncu_stdout.txt 2>&1
tail -3 gpurun_out/g31_ncu.csv
