mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_tp_capture.py tests/test_fullsize_gpu.py tests/test_runner.py -m gpu -q > gpurun_out/g8_gputest.log 2>&1; echo "gputest rc=$?"; tail -3 gpurun_out/g8_gputest.log
python tools/plan_profile.py cfg2 > gpurun_out/g8_plan.txt 2>&1; python tools/plan_profile.py cfg3 >> gpurun_out/g8_plan.txt 2>&1; cat gpurun_out/g8_plan.txt
