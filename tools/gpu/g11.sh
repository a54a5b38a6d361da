# round-2 closing bench lines (one per config) + reference arms + the default run's launch list
mkdir -p gpurun_out
for c in cfg1 cfg2 cfg4 cfg5:64 cfg5:1024; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/g11_bench_${c/:/_}.json 2> gpurun_out/g11_bench_${c/:/_}.err; echo "$c rc=$?"
done
timeout 900 python bench.py > gpurun_out/g11_bench_default.json 2> gpurun_out/g11_bench_default.err; echo "default rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/g11_ref_default.json 2>&1; echo "ref rc=$?"
timeout 600 python bench.py --impl reference --config cfg2 --steps 3 --warmup 3 > gpurun_out/g11_ref_cfg2.json 2>&1; echo "ref2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_" -c 400 --log-file gpurun_out/g11_launches_default.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo "ncu rc=$?"
