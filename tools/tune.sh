#!/bin/bash
# run the cfg2 bench (device path only) against each library variant in tools/
for lib in tools/libtd_*.so; do
  echo "== $lib"
  TD_LIB=$PWD/$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu 2>&1 | python3 tools/summarize_bench.py
done
echo "== default lib, classes serialised"
TD_SERIAL_CLASSES=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu 2>&1 | python3 tools/summarize_bench.py
