#!/bin/bash
# A/B the bulk-copy walker: library variants (build_variants.sh) x TD_BULK modes
# on the config-4 share (digest classes) and config 3 (plain compare classes)
cfg=${1:-cfg4}
modes=${2:-"0 1"}
for pass in 1 2; do
for lib in tools/libtd_*.so; do
for m in $modes; do
  echo "== pass $pass $lib TD_BULK=$m $(TD_BULK=$m TD_LIB=$PWD/$lib timeout 600 python bench.py --config $cfg --steps 20 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python3 -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],3), round(d["roofline"]["achieved"]), d.get("verdict_counts", d.get("verdict_counts_partial")), d["clocks"]["sm_mhz"], d["clocks"]["reasons"])')"
done
done
done
