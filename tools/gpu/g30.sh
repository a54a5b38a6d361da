#!/bin/bash
# small-tensor probe: flush style x tile target x CTAs/SM
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv
timeout 600 python tools/small_probe.py --sizes 16,64,256,1024 --targets 1184,2368,4736,9472 --bps 3,4 > gpurun_out/g30_small.jsonl 2>&1
tail -3 gpurun_out/g30_small.jsonl
