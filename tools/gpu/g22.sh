mkdir -p gpurun_out
for c in cfg2 cfg3 cfg4; do python tools/plan_profile.py $c; done > gpurun_out/g22_plan.txt 2>&1; cat gpurun_out/g22_plan.txt
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/g22_gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/g22_gputest.log
timeout 900 python tools/fuzz_parity.py --cases 300 --seed 303 > gpurun_out/g22_fuzz_parity.txt 2>&1; echo "fuzz rc=$?"; tail -1 gpurun_out/g22_fuzz_parity.txt
