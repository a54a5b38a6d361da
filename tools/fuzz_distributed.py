"""Differential fuzzing of the multi-GPU algorithm: random small
models x random layouts, split into per-GPU shares (synthetic.ShareLayout:
balanced compares, digests, reference slices), the shares run as threads on
one GPU (ThreadComm, real kernels, digest exchange, copy-0 handover), with
random corruptions of random records (replica bugs, value bugs).  Every
rank's report must equal a single-GPU check() of the union of the shares.
--faults adds 1-3 of tools/fuzz_faults.py's structural / numeric faults to
random shares (dropped / duplicated / re-declared copies, missing and extra
ids, moved boxes, rank changes, NaN/inf, zero payloads): the distributed
error paths must give the single-GPU report too (or both raise).

    python tools/fuzz_distributed.py [--cases 50] [--seed 0] [--faults]     (GPU)
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


def run_case(rnd, k, faults=False):
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
    if faults:
        # candidate faults first, then the reference re-split for the faulted
        # candidate's global metadata (distributed.split_reference: what a
        # job does, every rank holding the reference slices of its boxes),
        # then value / declaration faults on the reference slices
        import fuzz_faults
        from paper_2506_09280_b200.distributed import (StaticComm, _metas, execution_sorted, global_trace,
                                                       split_reference)
        for _ in range(rnd.choice([1, 1, 2, 3])):
            fuzz_faults.inject(rnd, shares[rnd.randrange(world)][1], rnd.choice(fuzz_faults.FAULTS))
        metas = [_metas(c, r, None) for r, (_, c) in enumerate(shares)]
        gcand = global_trace(shares[0][1], StaticComm(0, world, [metas]))
        ref_union = Trace(header=dict(shares[0][0].header))
        ref_union.records = execution_sorted([rec for r, _ in shares for rec in r.records])
        refs = split_reference(ref_union, gcand, world)
        shares = [(refs[r], shares[r][1]) for r in range(world)]
        for _ in range(rnd.choice([0, 0, 1])):
            fuzz_faults.inject(rnd, shares[rnd.randrange(world)][0], rnd.choice(("special", "zero", "declared")))
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
    ref_all, cand_all = Trace(header=dict(shares[0][0].header)), Trace(header=dict(shares[0][0].header))
    for r, c in shares:
        ref_all.records.extend(r.records)
        cand_all.records.extend(c.records)
    # the single-process traces the shares split: global execution order
    from paper_2506_09280_b200.distributed import execution_sorted
    ref_all.records, cand_all.records = execution_sorted(ref_all.records), execution_sorted(cand_all.records)
    try:
        want = json.loads(td.render_report(check(ref_all, cand_all, tol, fmt=td.FloatFormat.BF16), "json"))
    except Exception as exc:              # noqa: BLE001 — the distributed check must raise too
        if faults and errors:
            return (m, p, world, {"flag": 0, "replica-mismatch": 0, "raised": type(exc).__name__}, len(lay.ids))
        raise
    if errors:
        raise RuntimeError(errors[0])
    from tests.test_gpu_parity import assert_reports_match
    for rep in reports:
        assert_reports_match(rep, want, f"case {k}")
    return (m, p, world, want["summary"], len(lay.ids))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=50)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--faults", action="store_true")
    args = ap.parse_args()
    rnd = random.Random(args.seed)
    t0 = time.time()
    stats = {"cases": 0, "ids": 0, "flag": 0, "replica-mismatch": 0, "merge-error": 0, "missing": 0,
             "raised": 0, "layouts": set(), "worlds": {}}
    for k in range(args.cases):
        try:
            m, p, world, summary, n = run_case(rnd, k, args.faults)
        except Exception as exc:
            print(json.dumps({"failed_case": k, "error": str(exc)[-800:]}))
            sys.exit(1)
        stats["cases"] += 1
        stats["ids"] += n
        stats["flag"] += summary["flag"]
        stats["replica-mismatch"] += summary["replica-mismatch"]
        stats["merge-error"] += summary.get("merge-error", 0)
        stats["missing"] += summary.get("missing", 0)
        stats["raised"] += 1 if "raised" in summary else 0
        stats["layouts"].add((p.tp, p.dp, p.pp, p.vp, p.cp, p.sp, p.microbatches))
        stats["worlds"][world] = stats["worlds"].get(world, 0) + 1
    stats["layouts"] = len(stats["layouts"])
    stats["seconds"] = round(time.time() - t0, 1)
    print(json.dumps(stats))


if __name__ == "__main__":
    main()
