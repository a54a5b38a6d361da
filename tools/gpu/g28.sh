mkdir -p gpurun_out
timeout 2400 python tools/fuzz_parity.py --cases 3000 --seed 2026 > gpurun_out/g28_fuzz_parity.txt 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/g28_fuzz_parity.txt
timeout 2400 python tools/fuzz_distributed.py --cases 1000 --seed 2026 > gpurun_out/g28_fuzz_dist.txt 2>&1; echo "dist rc=$?"; tail -1 gpurun_out/g28_fuzz_dist.txt
timeout 1200 python tools/fuzz_perturb.py --cases 10000 --seed 2026 > gpurun_out/g28_fuzz_perturb.txt 2>&1; echo "perturb rc=$?"; tail -1 gpurun_out/g28_fuzz_perturb.txt
