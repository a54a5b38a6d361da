"""Where the time of the public check() goes with pinned host payloads
(config 2): host stage issue, planning (overlaps the DMA), DMA end, kernels,
fetch, report assembly.  Prints one JSON line (ms)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_2506_09280_b200.checker import CheckPlan, check
    from paper_2506_09280_b200.device import resolve_operands, stage_host_payloads
    from paper_2506_09280_b200.tracestore import pack_pinned
    desc, ref, cand, tol, fmt = bench.workload(os.environ.get("CFG", "cfg2"))
    href, hcand = pack_pinned(ref), pack_pinned(cand)
    del ref, cand
    torch.cuda.empty_cache()
    check(href, hcand, tol, 3.0, fmt=fmt)
    rows = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        staged = stage_host_payloads([href, hcand])
        dma = torch.cuda.Event()
        dma.record()
        t1 = time.perf_counter()
        cp = CheckPlan(href, hcand, tol, 3.0, fmt=fmt)
        t2 = time.perf_counter()
        dma.synchronize()
        t3 = time.perf_counter()
        ptrs, keep = resolve_operands(cp.plan.operands, cp.plan.operand_dtypes, staged)
        prep = cp.plan.prepare(ptrs, kappa=3.0, eps=fmt.eps, replica_eps=fmt.eps)
        t4 = time.perf_counter()
        prep.launch()
        torch.cuda.synchronize()
        t5 = time.perf_counter()
        idres, gres, ties = prep.fetch()
        t6 = time.perf_counter()
        rep = cp.report(idres, gres, ties)
        t7 = time.perf_counter()
        rows.append([t1 - t0, t2 - t1, t3 - t0, t4 - t3, t5 - t4, t6 - t5, t7 - t6, t7 - t0])
        del keep, prep, staged
    names = ["stage_issue", "plan", "dma_done_from_start", "resolve_prepare", "kernels", "fetch",
             "report", "total"]
    best = min(rows, key=lambda r: r[-1])
    print(json.dumps({n: round(v * 1e3, 3) for n, v in zip(names, best)}))


if __name__ == "__main__":
    main()
