#!/bin/bash
for pass in 1 2; do
for lib in tools/libtd_*.so; do
  echo "== pass $pass $lib"
  TD_LIB=$PWD/$lib timeout 900 python bench.py --config cfg3 --steps 10 --warmup 3 --no-e2e --no-cpu 2>&1 | python3 tools/summarize_bench.py
done
done
