"""Soak test: repeated public-API checks must not leak device memory, pinned
host memory or process RSS.  Loops over a few layouts (single-GPU check()
with device and host payloads, check_streaming, the distributed check on
thread-ranks), fresh payloads every iteration, and prints the memory
high-water marks per phase as one JSON line.

    python tools/soak.py [--iters 200]      (GPU)
"""
import argparse
import gc
import json
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rss_mb() -> float:
    import psutil
    return psutil.Process().memory_info().rss / 2 ** 20


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=200)
    args = ap.parse_args()
    import torch
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200 import layout as L
    from paper_2506_09280_b200 import synthetic
    from paper_2506_09280_b200.distributed import DistributedCheckPlan, ThreadComm
    model = L.ModelShape(layers=2, d_model=128, n_heads=4, d_ff=256, seq_len=256, vocab=512)
    layouts = [L.ParallelConfig(tp=2, microbatches=2), L.ParallelConfig(tp=4, dp=2, microbatches=2),
               L.ParallelConfig(tp=2, cp=2, sp=True, microbatches=2)]
    eps = td.FloatFormat.BF16.eps
    out = {}

    def phase(name, fn):
        marks = []
        for k in range(args.iters):
            fn(k)
            if k in (args.iters // 4, args.iters - 1):
                gc.collect()
                torch.cuda.synchronize()
                marks.append((torch.cuda.memory_allocated() / 2 ** 20, torch.cuda.memory_reserved() / 2 ** 20,
                              rss_mb()))
        (a0, r0, h0), (a1, r1, h1) = marks
        out[name] = {"alloc_mib": [round(a0, 1), round(a1, 1)], "reserved_mib": [round(r0, 1), round(r1, 1)],
                     "rss_mib": [round(h0, 1), round(h1, 1)]}

    def single(k, host=False):
        p = layouts[k % len(layouts)]
        ref, cand = synthetic.build(model, p, seed=k, eps=eps, bugs={})
        if host:
            for t in (ref, cand):
                for r in t.records:
                    r.payload = r.payload.cpu()
        tol = td.ToleranceMap({r.id.encode(): 2 * eps for r in ref.records}, n_samples=1, eps_p=eps)
        rep = td.check(ref, cand, tol, fmt=td.FloatFormat.BF16)
        assert rep.counts["pass"] == len(rep.entries) - rep.counts["missing"], rep.counts

    phase("check_device", lambda k: single(k))
    phase("check_host", lambda k: single(k, host=True))

    lay = synthetic.ShareLayout(model, L.ParallelConfig(tp=2, dp=2, microbatches=2), 4)
    tol = td.ToleranceMap({i: 2 * eps for i in lay.ids}, n_samples=1, eps_p=eps)

    def distributed(k):
        shares = [lay.build(r, seed=k) for r in range(4)]
        hub = ThreadComm.hub(4)
        errors = []

        def worker(rank):
            try:
                ref, cand = shares[rank]
                DistributedCheckPlan(ref, cand, tol, fmt=td.FloatFormat.BF16, comm=ThreadComm(hub, rank)).run()
            except Exception:     # pragma: no cover
                import traceback
                errors.append(traceback.format_exc())
                hub.barrier.abort()
        ts = [threading.Thread(target=worker, args=(r,)) for r in range(4)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not errors, errors[0]

    phase("distributed_threads", distributed)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
