"""One config-3 check split over W logical ranks as threads on ONE GPU
(ThreadComm: exchanges are device copies, so NVLink-like rather than gloo's
host staging).  Times a step the way bench.py --gpus W does — digests +
compares, the one exchange + td_combine + verdicts, the bug path when a
cross-rank replica group differs (config 3's missing all-reduce does) — to
see what the multi-GPU control path costs per step beyond the kernels.

    python tools/bench_threads_split.py [--world 2] [--steps 5] [--config cfg3]
"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--config", default="cfg3")
    args = ap.parse_args()
    import torch
    from paper_2506_09280_b200 import _native as N
    from paper_2506_09280_b200 import synthetic
    from paper_2506_09280_b200.checker import ToleranceMap
    from paper_2506_09280_b200.distributed import DistributedCheckPlan, ThreadComm
    import bench
    desc, spec = bench.describe(args.config)
    fmt, tp, world = spec["fmt"], spec["pcfg"].tp, args.world
    lay = synthetic.ShareLayout(spec["model"], spec["pcfg"], world, owner=lambda s, w=world, t=tp: s.rank[1] * w // t)
    shares = [lay.build(r, seed=0, eps=fmt.eps, bugs=spec.get("bugs")) for r in range(world)]
    tol = ToleranceMap({i: 2 * fmt.eps for i in lay.ids}, n_samples=1, eps_p=fmt.eps)
    hub = ThreadComm.hub(world)
    out, errors = [None] * world, []

    def worker(rank):
        try:
            torch.cuda.set_device(0)
            comm = ThreadComm(hub, rank)
            dcp = DistributedCheckPlan(*shares[rank], tol, 3.0, fmt=fmt, comm=comm)
            b = dcp.bind()
            stream = b.prep.stream
            times, kern, bug = [], [], 0
            for k in range(args.steps + 2):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                sh = N.stream_handle(stream)
                b.digest_pass(sh)
                b.exchange(sh)
                res = b.fetch()
                t1 = time.perf_counter()
                if res[3]:
                    bug += 1
                    res = dcp._bug_path(b)
                torch.cuda.synchronize()
                t2 = time.perf_counter()
                if k >= 2:
                    times.append((t1 - t0, t2 - t1))
            counts = {int(v): int((res[0]["verdict"] == v).sum()) for v in (0, 1, 2, 3)}
            out[rank] = {"clean_path_ms": 1e3 * sum(a for a, _ in times) / len(times),
                         "bug_path_ms": 1e3 * sum(c for _, c in times) / len(times),
                         "bug_steps": bug, "verdicts": counts}
        except Exception as exc:  # pragma: no cover
            import traceback
            errors.append(traceback.format_exc())
            hub.barrier.abort()
    threads = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise SystemExit(errors[0])
    print(json.dumps({"config": args.config, "world": world, "ranks": out}))


if __name__ == "__main__":
    main()
