#!/bin/bash
# A/B the config-4 share step across library variants in tools/ (build_variants.sh)
for pass in 1 2; do
for lib in tools/libtd_*.so; do
  echo "== pass $pass $lib $(TD_LIB=$PWD/$lib timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 2>&1 | tail -1 | python3 -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],2), round(d["roofline"]["achieved"]))')"
done
done
