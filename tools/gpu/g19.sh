mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none -k regex:"k_segnorm|k_finalize" -s 10 -c 4 -f -o gpurun_out/g19_small python tools/sweep_cfg5.py --sizes 1 --maps identity:1 --reps 3 > /dev/null 2>&1
ncu -i gpurun_out/g19_small.ncu-rep --page raw --csv > gpurun_out/g19_small_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/g19_small_raw.csv
