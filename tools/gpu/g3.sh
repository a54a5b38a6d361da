# A/B of the bulk (TMA-engine) digest walker variants on the config-4 share
mkdir -p gpurun_out
bash tools/tune_bulk.sh cfg4 "1" > gpurun_out/g3_tune_bulk.txt 2>&1
TD_LIB=$PWD/tools/libtd_base.so TD_BULK=0 timeout 600 python bench.py --config cfg4 --steps 20 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 > gpurun_out/g3_bulk0.json
for lib in base m2s3 m3s2; do
  TD_LIB=$PWD/tools/libtd_$lib.so timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:"k_segnorm" \
      --log-file gpurun_out/g3_launches_$lib.csv python bench.py --config cfg4 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
done
