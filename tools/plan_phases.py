"""Where a cold CheckPlan spends its time (host only, no GPU needed):
by_id + merge_view per side, PlanEntry list, and Plan's phases, best of N
runs with memo caches cleared.

    python tools/plan_phases.py [cfg2|cfg3|cfg4] [runs]
"""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import plan_profile as PP  # noqa: E402

from paper_2506_09280_b200 import layout as L  # noqa: E402
from paper_2506_09280_b200 import plan as PL  # noqa: E402
from paper_2506_09280_b200.checker import ToleranceMap  # noqa: E402

PHASES = ("_plan_entry", "_record_entry", "_replay_entry", "_fill_replayed_rows", "_columns", "_retile",
          "_freeze_segments", "_chunk_slots")


def main(name="cfg2", runs=15):
    model, pcfg = PP.CFGS[name]
    hdr = {"digest": "plan-phases", "mode": "cascade"}
    ref = PP.meta_trace(L.emit_records(model, L.ParallelConfig(microbatches=pcfg.microbatches)), hdr)
    cand = PP.meta_trace(L.emit_records(model, pcfg), hdr)
    tol = ToleranceMap({}, n_samples=1, eps_p=2.0 ** -8)
    acc: dict = {}

    def wrap(obj, fname):
        f = getattr(obj, fname)

        def g(*a, **k):
            t = time.perf_counter()
            r = f(*a, **k)
            acc[fname] = acc.get(fname, 0.0) + time.perf_counter() - t
            return r
        setattr(obj, fname, g)
    for fname in PHASES:
        wrap(PL.Plan, fname)
    wrap(PL, "_shared_entries")
    best: dict = {}
    for _ in range(runs):
        PL._MERGE_DETAIL.clear()
        PL._RUN_BLOCKS.clear()
        PL._run_blocks.cache_clear()
        acc.clear()
        gc.disable()
        t0 = time.perf_counter()
        rv = PL.merge_view(ref)
        t1 = time.perf_counter()
        cv = PL.merge_view(cand)
        t2 = time.perf_counter()
        ents = [PL.PlanEntry(i, x=rv[i], y=cv[i], x_rep=True, y_rep=True, tolerance=tol.get(i))
                for i in cv if i in rv]
        t3 = time.perf_counter()
        PL.Plan(ents, disjoint=set(map(id, ref.records)).isdisjoint(map(id, cand.records)))
        t4 = time.perf_counter()
        gc.enable()
        acc.update(merge_view_ref=t1 - t0, merge_view_cand=t2 - t1, plan_entries=t3 - t2, plan=t4 - t3,
                   total=t4 - t0)
        if not best or acc["total"] < best["total"]:
            best = dict(acc)
    print(name, {k: round(v * 1e3, 2) for k, v in best.items()})


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "cfg2", int(sys.argv[2]) if len(sys.argv) > 2 else 15)
