mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none -k regex:"k_segnorm|k_fingerprint" -s 0 -c 3 -f -o gpurun_out/g27_cfg4 python bench.py --config cfg4 --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
ncu -i gpurun_out/g27_cfg4.ncu-rep --page raw --csv > gpurun_out/g27_cfg4_raw.csv 2>/dev/null
python tools/ncu_summary.py gpurun_out/g27_cfg4_raw.csv
