mkdir -p gpurun_out
for t in 0 1; do echo "templates=$t $(TD_PLAN_TEMPLATES=$t python tools/dplan_profile.py | tail -1)"; done
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/g24_gputest.log 2>&1; echo "gputest rc=$?"; tail -2 gpurun_out/g24_gputest.log
timeout 1200 python tools/fuzz_distributed.py --cases 200 --seed 404 > gpurun_out/g24_fuzz_dist.txt 2>&1; echo "fuzz rc=$?"; tail -1 gpurun_out/g24_fuzz_dist.txt
timeout 900 python bench.py --config cfg4 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/g24_cfg4.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/g24_cfg4.json').read().strip().splitlines()[-1]); print('cfg4', d['value'], 'plan_s', d['plan_seconds'])"
