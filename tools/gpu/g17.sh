mkdir -p gpurun_out
run() { echo "== $* $(env "$@" timeout 900 python bench.py --config $CFG --steps 20 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python3 -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')"; }
for pass in 1 2; do
for CFG in cfg3 cfg2; do
  run TD_BULK=1
  run TD_BULK=3
done
done > gpurun_out/g17_bulk_plain.txt 2>&1
cat gpurun_out/g17_bulk_plain.txt
TD_BULK=3 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:"k_segnorm" --log-file gpurun_out/g17_launches_bulk3.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
grep k_segnorm gpurun_out/g17_launches_bulk3.csv | awk -F'","' '{print $5, $NF}' | head -8
