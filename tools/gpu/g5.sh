mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g5_gputest.log 2>&1; echo "gputest rc=$?"; tail -3 gpurun_out/g5_gputest.log
timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/g5_cfg4.json 2>/dev/null; echo "cfg4 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_segnorm_bulk -s 0 -c 1 -f -o gpurun_out/g5_cfg4_bulk python bench.py --config cfg4 --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
ncu -i gpurun_out/g5_cfg4_bulk.ncu-rep --page raw --csv > gpurun_out/g5_cfg4_bulk_raw.csv 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_segnorm|k_finalize|k_reduce|k_verdict|k_fingerprint|k_combine" --log-file gpurun_out/g5_cfg4_launches.csv python bench.py --config cfg4 --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
