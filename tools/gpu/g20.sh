mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g20_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/g20_smoke.log
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/g20_gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/g20_gputest.log
