#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "batch or cache or reproduces" > gpurun_out/g60_tests.txt 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/g60_tests.txt
for i in 1 2; do
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 > gpurun_out/g60_bench$i.json
python -c "import json; d=json.loads(open('gpurun_out/g60_bench$i.json').read()); e=d['e2e']; print('value', round(d['value'],1), 'e2e', round(e['value'],2), 'cold', round(e['cold']['value'],2), 'pageable', round(e['pageable']['value'],2), 'clk', d['clocks']['sm_mhz'])"
done
