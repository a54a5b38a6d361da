mkdir -p gpurun_out
timeout 1500 python tools/fuzz_distributed.py --cases 300 --seed 202 > gpurun_out/g14_fuzz_dist.txt 2>&1; echo "fuzz_dist rc=$?"; tail -3 gpurun_out/g14_fuzz_dist.txt
timeout 1500 python tools/fuzz_parity.py --cases 600 --seed 202 > gpurun_out/g14_fuzz_parity.txt 2>&1; echo "fuzz_parity rc=$?"; tail -3 gpurun_out/g14_fuzz_parity.txt
