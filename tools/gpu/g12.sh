mkdir -p gpurun_out
bash tools/tune_perturb.sh > gpurun_out/g12_perturb_ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "perturb or quantize or uniform" > gpurun_out/g12_perturb_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g12_perturb_tests.log
python tools/fuzz_perturb.py --cases 3000 > gpurun_out/g12_fuzz_perturb.txt 2>&1; echo "fuzz rc=$?"; tail -3 gpurun_out/g12_fuzz_perturb.txt
timeout 600 ncu --set full --clock-control none -k regex:k_perturb_bf16 -c 1 -f -o gpurun_out/g12_perturb python tools/bench_perturb.py > /dev/null 2>&1
ncu -i gpurun_out/g12_perturb.ncu-rep --page raw --csv > gpurun_out/g12_perturb_raw.csv 2>/dev/null
cat gpurun_out/g12_perturb_ab.txt
