"""Differential fuzzing of the multi-GPU algorithm: random small
models x random layouts, split into per-GPU shares (synthetic.ShareLayout:
balanced compares, digests, reference slices), the shares run as threads on
one GPU (ThreadComm, real kernels, digest exchange, copy-0 handover), with
random corruptions of random records (replica bugs, value bugs).  Every
rank's report must equal a single-GPU check() of the union of the shares.

    python tools/fuzz_distributed.py [--cases 50] [--seed 0]     (GPU)
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
sys.path.insert(0, os.path.join(ROOT, "tools"))


def run_case(rnd, k):
    import torch
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200 import synthetic
    from paper_2506_09280_b200.checker import check
    from paper_2506_09280_b200.distributed import DistributedCheckPlan, ThreadComm
    from paper_2506_09280_b200.tracestore import Trace
    import fuzz_parity
    m, p, _ = fuzz_parity.random_case(rnd)
    world = rnd.choice([2, 3, 4])
    lay = synthetic.ShareLayout(m, p, world)
    shares = [lay.build(r, seed=k) for r in range(world)]
    for _ in range(rnd.choice([0, 1, 2])):           # corrupt a random candidate record
        r = rnd.randrange(world)
        if shares[r][1].records:
            rec = rnd.choice(shares[r][1].records)
            if rec.payload.numel():
                rec.payload.mul_(rnd.choice([2.0, -1.0, 1.5]))
    eps = td.FloatFormat.BF16.eps
    tol = td.ToleranceMap({i: 2 * eps for i in lay.ids}, n_samples=1, eps_p=eps)
    hub = ThreadComm.hub(world)
    reports, errors = [None] * world, []

    def worker(rank):
        try:
            ref, cand = shares[rank]
            plan = DistributedCheckPlan(ref, cand, tol, fmt=td.FloatFormat.BF16, comm=ThreadComm(hub, rank))
            reports[rank] = json.loads(td.render_report(plan.run(), "json"))
        except Exception:
            import traceback
            errors.append(traceback.format_exc())
            hub.barrier.abort()
    threads = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    if errors:
        raise RuntimeError(errors[0])
    ref_all, cand_all = Trace(header=dict(shares[0][0].header)), Trace(header=dict(shares[0][0].header))
    for r, c in shares:
        ref_all.records.extend(r.records)
        cand_all.records.extend(c.records)
    # the single-process traces the shares split: global execution order
    from paper_2506_09280_b200.distributed import execution_sorted
    ref_all.records, cand_all.records = execution_sorted(ref_all.records), execution_sorted(cand_all.records)
    want = json.loads(td.render_report(check(ref_all, cand_all, tol, fmt=td.FloatFormat.BF16), "json"))
    from tests.test_gpu_parity import assert_reports_match
    for rep in reports:
        assert_reports_match(rep, want, f"case {k}")
    return (m, p, world, want["summary"], len(lay.ids))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=50)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    rnd = random.Random(args.seed)
    t0 = time.time()
    stats = {"cases": 0, "ids": 0, "flag": 0, "replica-mismatch": 0, "layouts": set(), "worlds": {}}
    for k in range(args.cases):
        try:
            m, p, world, summary, n = run_case(rnd, k)
        except Exception as exc:
            print(json.dumps({"failed_case": k, "error": str(exc)[-800:]}))
            sys.exit(1)
        stats["cases"] += 1
        stats["ids"] += n
        stats["flag"] += summary["flag"]
        stats["replica-mismatch"] += summary["replica-mismatch"]
        stats["layouts"].add((p.tp, p.dp, p.pp, p.vp, p.cp, p.sp, p.microbatches))
        stats["worlds"][world] = stats["worlds"].get(world, 0) + 1
    stats["layouts"] = len(stats["layouts"])
    stats["seconds"] = round(time.time() - t0, 1)
    print(json.dumps(stats))


if __name__ == "__main__":
    main()
