"""The public check() on device-resident traces (the torchtap -> check flow):
first call plans (host), repeated calls of one layout hit the plan cache.
Config-2 traces, two 'steps' with different values and the same layout.
Prints JSON: seconds per call (miss / hit), and that the hit's report equals
a fresh plan's."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200 import checker
    _, ref0, cand0, tol, fmt = bench.workload("cfg2", rank=0)
    _, ref1, cand1, _, _ = bench.workload("cfg2", rank=1)
    torch.cuda.synchronize()
    out = {}
    checker._PLAN_CACHE.clear()
    t0 = time.perf_counter()
    td.check(ref0, cand0, tol, fmt=fmt)
    out["miss_s"] = time.perf_counter() - t0
    times = []
    for _ in range(5):
        t0 = time.perf_counter()
        rep = td.check(ref1, cand1, tol, fmt=fmt)
        times.append(time.perf_counter() - t0)
    out["hit_s"] = min(times)
    checker._PLAN_CACHE.clear()
    fresh = td.check(ref1, cand1, tol, fmt=fmt)
    out["hit_report_equals_fresh"] = td.render_report(rep, "json") == td.render_report(fresh, "json")
    t0 = time.perf_counter()
    key = checker._check_key(ref1, cand1, tol, 3.0, fmt)
    out["layout_key_s"] = time.perf_counter() - t0
    out["bytes"] = ref1.nbytes + cand1.nbytes
    out["hit_gbs"] = out["bytes"] / out["hit_s"] / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
