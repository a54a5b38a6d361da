#!/bin/bash
# A/B the config-4 share step across environment settings: tools/tune_cfg4_env.sh "A=1" "A=0"
for pass in 1 2; do
for env in "$@"; do
  echo "== pass $pass $env $(env $env timeout 600 python bench.py --config cfg4 --steps 10 --warmup 3 2>&1 | tail -1 | python3 -c 'import sys,json; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],2), round(d["roofline"]["achieved"]))')"
done
done
