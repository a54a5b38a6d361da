mkdir -p gpurun_out
for pass in 1 2; do for l in v1 v2; do echo "$l $(TD_LIB=$PWD/tools/libtd_g_$l.so python tools/bench_gather.py)"; done; done > gpurun_out/g18_gather_ab.txt 2>&1
cat gpurun_out/g18_gather_ab.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "gather or read_trace or write_trace or device_reader" > gpurun_out/g18_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g18_tests.log
timeout 900 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -q -k "gather_bytes_any" > gpurun_out/g18_memcheck.log 2>&1; echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/g18_memcheck.log | tail -3
