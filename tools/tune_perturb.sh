#!/bin/bash
# A/B td_perturb across library variants in tools/ (see build_variants.sh), two passes.
for pass in 1 2; do
for lib in tools/libtd_*.so; do
  echo "== pass $pass $lib $(TD_LIB=$PWD/$lib timeout 300 python tools/bench_perturb.py 2>&1 | grep splitmix | head -2 | python3 -c 'import sys,json; print([round(json.loads(l)["gbs"]) for l in sys.stdin])')"
done
done
