"""Concurrency stress: T host threads call the public check() at the same
time on traces of a few shared layouts (so they hit the same cached plans,
the same pinned staging ring and the native library concurrently), with
device or host payloads, and every report must equal the one a serial
check of the same traces gave.  Prints one JSON line.

    python tools/stress_threads.py [--threads 8] [--iters 20]      (GPU)
"""
import argparse
import json
import os
import random
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--threads", type=int, default=8)
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    import torch
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200 import layout as L
    from paper_2506_09280_b200 import synthetic
    # host payloads large enough (> 64 MiB per check) to go through the pinned staging ring
    model = L.ModelShape(layers=2, d_model=512, n_heads=8, d_ff=1024, seq_len=2048, vocab=4096)
    layouts = [L.ParallelConfig(tp=2, microbatches=1), L.ParallelConfig(tp=4, microbatches=1)]
    eps = td.FloatFormat.BF16.eps
    cases = []
    for k in range(2 * len(layouts)):
        p = layouts[k % len(layouts)]
        bugs = {}
        ref, cand = synthetic.build(model, p, seed=k, eps=eps, bugs=bugs)
        ids = sorted({r.id.encode() for r in cand.records})
        rnd = random.Random(k)
        for ident in rnd.sample(ids, 2):                 # value bugs that differ per case
            for r in cand.records:
                if r.id.encode() == ident:
                    r.payload.mul_(1.5)
        tol = td.ToleranceMap({r.id.encode(): 2 * eps for r in ref.records}, n_samples=1, eps_p=eps)
        host = (k // len(layouts)) % 2 == 1
        if host:
            for t in (ref, cand):
                for r in t.records:
                    r.payload = r.payload.cpu()
        want = td.render_report(td.check(ref, cand, tol, fmt=td.FloatFormat.BF16), "json")
        cases.append((ref, cand, tol, want, host))
    torch.cuda.synchronize()
    errors, done = [], [0]
    lock = threading.Lock()

    def worker(t):
        rnd = random.Random(1000 + t)
        try:
            for _ in range(args.iters):
                ref, cand, tol, want, _ = cases[rnd.randrange(len(cases))]
                got = td.render_report(td.check(ref, cand, tol, fmt=td.FloatFormat.BF16), "json")
                if got != want:
                    raise AssertionError("report differs from the serial check's")
                with lock:
                    done[0] += 1
        except Exception:                  # noqa: BLE001
            import traceback
            errors.append(traceback.format_exc())
    t0 = time.time()
    threads = [threading.Thread(target=worker, args=(t,)) for t in range(args.threads)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    out = {"threads": args.threads, "checks": done[0], "errors": len(errors),
           "host_cases": sum(c[4] for c in cases), "device_cases": sum(not c[4] for c in cases),
           "bytes_per_check": [int(sum(r.nbytes for r in c[0].records) + sum(r.nbytes for r in c[1].records))
                               for c in cases],
           "seconds": round(time.time() - t0, 1)}
    print(json.dumps(out))
    if errors:
        print(errors[0])
        sys.exit(1)


if __name__ == "__main__":
    main()
