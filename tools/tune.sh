#!/bin/bash
# A/B the cfg2 bench (device path only) across library variants in tools/,
# twice in alternating order to expose box drift.  A variant named *tileNk*
# needs the matching host tile size (TD_TILE_UNITS).
for pass in 1 2; do
for lib in tools/libtd_*.so; do
  tu=8192
  case $lib in *tile16k*) tu=16384;; *tile4k*) tu=4096;; esac
  echo "== pass $pass $lib"
  TD_TILE_UNITS=$tu TD_LIB=$PWD/$lib timeout 600 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu 2>&1 | python3 tools/summarize_bench.py
done
done
