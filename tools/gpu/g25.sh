mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_distributed.py tests/test_share.py tests/test_tp_capture.py -m gpu -q > gpurun_out/g25_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/g25_tests.log
timeout 600 python tools/fuzz_distributed.py --cases 200 --seed 505 > gpurun_out/g25_fuzz.txt 2>&1; echo "fuzz rc=$?"; tail -1 gpurun_out/g25_fuzz.txt
TD_BENCH_BACKEND=gloo TD_BENCH_SAME_DEVICE=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > gpurun_out/g25_n2.json 2> gpurun_out/g25_n2.err; echo "n2 rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/g25_n2.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['verdict_counts'], d['exchange']['steps_on_bug_path'])"
