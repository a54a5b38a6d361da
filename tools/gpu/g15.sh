mkdir -p gpurun_out
timeout 900 python bench.py --config cfg2 --steps 10 --warmup 3 --no-cpu > gpurun_out/g15_cfg2.json 2> gpurun_out/g15_cfg2.err; echo "cfg2 rc=$?"
timeout 1200 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/g15_cfg3.json 2> gpurun_out/g15_cfg3.err; echo "cfg3 rc=$?"
free -g
