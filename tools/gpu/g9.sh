mkdir -p gpurun_out
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/g9_gputest.log 2>&1; echo "gputest rc=$?"; tail -3 gpurun_out/g9_gputest.log
grep -E "passed|failed" gpurun_out/g9_gputest.log | tail -2
