mkdir -p gpurun_out
for pass in 1 2; do for m in 0 1; do echo "staged=$m $(TD_GATHER_STAGED=$m python tools/bench_gather.py)"; done; done > gpurun_out/g29_gather_ab.txt 2>&1
cat gpurun_out/g29_gather_ab.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "gather or read_trace or write_trace or device_reader or cli" > gpurun_out/g29_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g29_tests.log
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -q -k "gather_bytes_any" > gpurun_out/g29_memcheck.log 2>&1; echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/g29_memcheck.log | tail -3
timeout 900 compute-sanitizer --tool racecheck python -m pytest tests/test_gpu_parity.py -m gpu -q -k "gather_bytes_any" > gpurun_out/g29_racecheck.log 2>&1; echo "racecheck rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|passed|failed" gpurun_out/g29_racecheck.log | tail -3
