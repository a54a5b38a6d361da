mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/g7_gputest.log 2>&1; echo "gputest rc=$?"; tail -3 gpurun_out/g7_gputest.log
timeout 900 python bench.py > gpurun_out/g7_cfg3.json 2>gpurun_out/g7_cfg3.err; echo "cfg3 rc=$?"
