mkdir -p gpurun_out
bash tools/tune_perturb.sh > gpurun_out/g13_perturb_ab.txt 2>&1
cat gpurun_out/g13_perturb_ab.txt
