#!/bin/bash
# round-end state: smoke, the full GPU suite, the default bench line
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g41_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/g41_smoke.log
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/g41_gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/g41_gputest.log
timeout 900 python bench.py > gpurun_out/g41_bench.json 2> gpurun_out/g41_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/g41_bench.json | python tools/_bench_brief.py
timeout 900 python bench.py --impl reference > gpurun_out/g41_ref.json 2> gpurun_out/g41_ref.err; echo "ref rc=$?"; tail -1 gpurun_out/g41_ref.json | cut -c1-300
