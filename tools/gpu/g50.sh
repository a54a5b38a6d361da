#!/bin/bash
# aux-stream pool: soak (RSS / device memory over 200 iterations per phase) + the GPU suite
mkdir -p gpurun_out
timeout 1100 python tools/soak.py --iters 200 > gpurun_out/g50_soak.txt 2>&1; echo "soak rc=$?"; tail -c 600 gpurun_out/g50_soak.txt
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/g50_gputest.txt 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/g50_gputest.txt
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 | python tools/_bench_brief.py
