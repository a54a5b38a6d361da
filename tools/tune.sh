#!/bin/bash
# run the cfg2 bench (device path only) against each library variant in tools/
for lib in tools/libtd_*.so; do
  echo "== $lib"
  TD_LIB=$PWD/$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu 2>&1 | python3 -c '
import json,sys
for l in sys.stdin:
    if l.startswith("{"):
        d=json.loads(l); r=d["roofline"]; print(f"value {d[\"value\"]:.0f} GB/s  segnorm {r[\"achieved\"]:.0f} GB/s frac {r[\"frac\"]:.3f}  ms/step {d[\"ms_per_step\"]:.4f}")
    elif "Error" in l: print(l.strip())'
done
