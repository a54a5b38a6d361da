#!/bin/bash
# Round profile pass (run on the GPU box through gpurun, one GPU):
#   launch lists (per-launch gpu__time_duration, cold/serialised) and one
#   `ncu --set full` capture of the td_segnorm class launches, per config;
#   then full captures of td_perturb, td_fingerprint and td_rel_err.
# Output under gpurun_out/: prof_<cfg>_launches.csv, prof_<cfg>_full.ncu-rep
# (+ raw CSV pages), prof_{perturb,fingerprint,relerr}_full_raw.csv.
set -u
mkdir -p gpurun_out
for cfg in ${CONFIGS:-cfg2 cfg3}; do
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      -k regex:"k_segnorm|k_finalize|k_reduce|k_verdict|k_fingerprint" \
      --log-file gpurun_out/prof_${cfg}_launches.csv \
      python bench.py --config $cfg --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof_${cfg}_launches.log 2>&1
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_segnorm -s 0 -c ${NCLASS:-4} \
      -f -o gpurun_out/prof_${cfg}_full \
      python bench.py --config $cfg --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/prof_${cfg}_full.log 2>&1
  ncu -i gpurun_out/prof_${cfg}_full.ncu-rep --page raw --csv > gpurun_out/prof_${cfg}_full_raw.csv 2>/dev/null
done
if [ "${KERNELS:-1}" = "1" ]; then
  timeout 600 ncu --set full --clock-control none -k regex:k_perturb_bf16 -c 1 -f -o gpurun_out/prof_perturb \
      python tools/bench_perturb.py > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none -k regex:k_fingerprint -s 3 -c 1 -f -o gpurun_out/prof_fingerprint \
      python tools/bench_digest.py > /dev/null 2>&1
  # the 1 GiB pair of tools/bench_relerr.py (after 53 + 53 + 13 + 3 launches)
  timeout 600 ncu --set full --clock-control none -k regex:k_rel_err -s 122 -c 1 -f -o gpurun_out/prof_relerr \
      python tools/bench_relerr.py > /dev/null 2>&1
  for k in perturb fingerprint relerr; do
    ncu -i gpurun_out/prof_$k.ncu-rep --page raw --csv > gpurun_out/prof_${k}_full_raw.csv 2>/dev/null
  done
fi
