mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/g1_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g1_gputest.log 2>&1; echo "gputest rc=$?"
tail -3 gpurun_out/g1_gputest.log
timeout 900 python bench.py > gpurun_out/g1_bench_cfg3.json 2> gpurun_out/g1_bench_cfg3.err; echo "bench rc=$?"
timeout 900 python bench.py --config cfg4 --steps 20 --warmup 3 > gpurun_out/g1_bench_cfg4.json 2> gpurun_out/g1_bench_cfg4.err; echo "cfg4 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/g1_bench_ref.json 2> gpurun_out/g1_bench_ref.err; echo "ref rc=$?"
