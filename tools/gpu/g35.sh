mkdir -p gpurun_out
run() { echo "== $* $(env "$@" timeout 900 python bench.py --config $CFG --steps 30 --warmup 5 --no-e2e --no-cpu 2>&1 | tail -1 | python3 -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"], d["verdict_counts"])')"; }
for pass in 1 2; do
CFG=cfg3
for l in ic00 ic11 ic81 ic55; do run TD_LIB=$PWD/tools/libtd_$l.so; done
CFG=cfg2
for l in ic00 ic55; do run TD_LIB=$PWD/tools/libtd_$l.so; done
done > gpurun_out/g35_iconv.txt 2>&1
cat gpurun_out/g35_iconv.txt
for l in ic00 ic55; do TD_LIB=$PWD/tools/libtd_$l.so timeout 900 ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active --clock-control none --csv -k regex:"k_segnorm_vec<1, 0" -c 2 --log-file gpurun_out/g35_ncu_$l.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; grep -o '"[a-z_]*__[a-z_.]*","[a-z%]*","[0-9.,]*"' gpurun_out/g35_ncu_$l.csv | head -4; done
