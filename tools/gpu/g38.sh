mkdir -p gpurun_out
for c in cfg4 cfg5:64 cfg2; do
TD_BENCH_BACKEND=gloo TD_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 --config $c --steps 3 --warmup 3 > gpurun_out/g38_$c.json 2> gpurun_out/g38_$c.err; echo "$c rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/g38_$c.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d.get('verdict_counts') or d.get('verdict_counts_partial'), d['scaling'], (d.get('e2e') or {}).get('value'))"
done
