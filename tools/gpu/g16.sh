mkdir -p gpurun_out
for t in 8 16; do
  TD_STAGE_THREADS=$t timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/g16_t$t.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/g16_t$t.json').read().strip().splitlines()[-1]); print('threads $t', d['e2e']['value'], d['e2e']['pageable'])"
done
