# overlap A/B: concurrent vs serial classes / fingerprint, bulk variants (config 4), classes (config 3)
mkdir -p gpurun_out
run() { echo "== $* $(env "$@" timeout 600 python bench.py --config $CFG --steps 20 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python3 -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],3), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')"; }
for pass in 1 2; do
CFG=cfg4
for lib in base m2s3; do
  run TD_LIB=$PWD/tools/libtd_$lib.so TD_SERIAL_CLASSES=0 TD_SERIAL_FP=0
  run TD_LIB=$PWD/tools/libtd_$lib.so TD_SERIAL_CLASSES=1 TD_SERIAL_FP=0
  run TD_LIB=$PWD/tools/libtd_$lib.so TD_SERIAL_CLASSES=1 TD_SERIAL_FP=1
done
CFG=cfg3
run TD_LIB=$PWD/tools/libtd_base.so TD_SERIAL_CLASSES=0
run TD_LIB=$PWD/tools/libtd_base.so TD_SERIAL_CLASSES=1
done > gpurun_out/g4_overlap.txt 2>&1
nvidia-smi -q -d POWER,CLOCK > gpurun_out/g4_smi.txt 2>&1
