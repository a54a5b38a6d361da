#!/bin/bash
# graphed distributed step: tests, cfg4 share bench (graph vs eager), 2-rank same-device gloo bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_share.py -m gpu -q -x -k "graph" > gpurun_out/g48_tests.txt 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g48_tests.txt
for g in 1 0 1; do
  TD_BENCH_GRAPH=$g timeout 900 python bench.py --config cfg4 --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1 > gpurun_out/g48_cfg4_$g.json
  python -c "import json; d=json.loads(open('gpurun_out/g48_cfg4_$g.json').read()); print('graph=$g', round(d['value'],1), round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4), d['exchange']['step_launch'], d.get('verdict_counts_partial'), d['clocks']['sm_mhz'])"
done
TD_BENCH_BACKEND=gloo TD_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config cfg3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/g48_n2.json 2> gpurun_out/g48_n2.err; echo "n2 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/g48_n2.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d.get('verdict_counts'), d['exchange'])"
