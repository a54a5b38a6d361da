mkdir -p gpurun_out
free -g > gpurun_out/g10_free.txt; nproc >> gpurun_out/g10_free.txt
timeout 900 python -m pytest tests/test_tp_capture.py -m gpu -q -k config1 > gpurun_out/g10_cfg1.log 2>&1; echo "rc=$?"
grep -n "AssertionError" -A3 gpurun_out/g10_cfg1.log | head -20
