mkdir -p gpurun_out
timeout 900 python tools/bench_cli.py > gpurun_out/g33_cli.txt 2>&1; echo "cli rc=$?"; tail -3 gpurun_out/g33_cli.txt
timeout 900 python tools/bench_write_trace.py > gpurun_out/g33_write.txt 2>&1; echo "write rc=$?"; tail -3 gpurun_out/g33_write.txt
