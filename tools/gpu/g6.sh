mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/g6_gputest.log 2>&1; echo "gputest rc=$?"; tail -3 gpurun_out/g6_gputest.log
timeout 600 python bench.py --config cfg2 --steps 20 --warmup 5 > gpurun_out/g6_cfg2.json 2>/dev/null; echo "cfg2 rc=$?"
timeout 900 python tools/sweep_cfg5.py --maps identity:1,columns:8 > gpurun_out/g6_sweep_cfg5.jsonl 2>&1; echo "sweep rc=$?"
