"""cProfile of warm check() calls on device-resident config-2 traces (host overhead per call)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import bench
import paper_2506_09280_b200 as td
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
_, ref, cand, tol, fmt = bench.workload(cfg, rank=0)
torch.cuda.synchronize()
td.check(ref, cand, tol, fmt=fmt)
ts = []
for _ in range(10):
    t0 = time.perf_counter(); td.check(ref, cand, tol, fmt=fmt); ts.append(time.perf_counter() - t0)
print(cfg, "hit ms", sorted(ts)[:3])
pr = cProfile.Profile(); pr.enable()
for _ in range(5):
    td.check(ref, cand, tol, fmt=fmt)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
