mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g37_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/g37_smoke.log
timeout 1300 python -m pytest tests -m gpu -q > gpurun_out/g37_gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/g37_gputest.log
timeout 1200 python tools/fuzz_distributed.py --cases 1000 --seed 3030 > gpurun_out/g37_fuzz_dist.txt 2>&1; echo "dist rc=$?"; tail -1 gpurun_out/g37_fuzz_dist.txt
