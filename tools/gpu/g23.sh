mkdir -p gpurun_out
TD_BENCH_BACKEND=gloo TD_BENCH_SAME_DEVICE=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/g23_n2.json 2> gpurun_out/g23_n2.err; echo "n2 rc=$?"
tail -c 1500 gpurun_out/g23_n2.json; tail -5 gpurun_out/g23_n2.err
