#!/bin/bash
# Build libtdb200 variants with extra -D flags into tools/libtd_<name>.so for A/B runs
# (TD_LIB=... selects one at run time).  Usage: tools/build_variants.sh name:"-DX=1" ...
cd "$(dirname "$0")/.."
for spec in "$@"; do
  name=${spec%%:*}; flags=${spec#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
       -I include $flags -o tools/libtd_$name.so paper_2506_09280_b200/csrc/td_kernels.cu &
done
wait
