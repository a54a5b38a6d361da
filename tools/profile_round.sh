#!/bin/bash
# Round profile pass (run on the GPU box through gpurun, one GPU):
#   launch lists (per-launch gpu__time_duration, cold/serialised) and one
#   `ncu --set full` capture of the td_segnorm class launches, per config.
# Output: gpurun_out/prof_<cfg>_launches.csv, gpurun_out/prof_<cfg>_full.ncu-rep
# and its raw CSV page.
set -u
mkdir -p gpurun_out
for cfg in ${CONFIGS:-cfg2 cfg3}; do
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/prof_${cfg}_launches.csv \
      python bench.py --config $cfg --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof_${cfg}_launches.log 2>&1
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_segnorm -s 0 -c ${NCLASS:-4} \
      -f -o gpurun_out/prof_${cfg}_full \
      python bench.py --config $cfg --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/prof_${cfg}_full.log 2>&1
  ncu -i gpurun_out/prof_${cfg}_full.ncu-rep --page raw --csv > gpurun_out/prof_${cfg}_full_raw.csv 2>/dev/null
done
