mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g31_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/g31_smoke.log
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/g31_gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/g31_gputest.log
for c in cfg1 cfg2 cfg4 cfg5:64 cfg5:1024; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 5 > gpurun_out/g31_bench_${c/:/_}.json 2> gpurun_out/g31_bench_${c/:/_}.err; echo "$c rc=$?"
done
timeout 1200 python bench.py > gpurun_out/g31_bench_default.json 2> gpurun_out/g31_bench_default.err; echo "default rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/g31_ref_default.json 2>&1; echo "ref rc=$?"
timeout 600 python bench.py --impl reference --config cfg2 --steps 3 --warmup 3 > gpurun_out/g31_ref_cfg2.json 2>&1; echo "ref2 rc=$?"
