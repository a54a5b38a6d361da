"""Config 5: raw compare sweep, one id per size, 1 MiB - 8 GiB of bf16 per
tensor, shape (N/4096, 4096); candidate identity / G-way column shards /
CP-style 2-stripe.  L2 is flushed (256 MiB memset) before every timed rep;
td_segnorm timed alone with CUDA events.  Prints one JSON line per point.

    python tools/sweep_cfg5.py [--sizes 1,4,...] [--reps 20]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1,4,16,64,256,1024,2048,4096,8192")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--maps", default="identity:1,columns:4,columns:8,stripes:2")
    args = ap.parse_args()
    import torch
    from paper_2506_09280_b200 import _native as N
    from paper_2506_09280_b200 import synthetic
    from paper_2506_09280_b200.checker import CheckPlan, ToleranceMap
    from paper_2506_09280_b200.device import resolve_operands
    from paper_2506_09280_b200.tensor import FloatFormat
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for mib in [int(s) for s in args.sizes.split(",")]:
        for spec in args.maps.split(","):
            maps, g = spec.split(":")
            ref, cand = synthetic.sweep_pair(mib << 20, maps=maps, g=int(g))
            tol = ToleranceMap({}, n_samples=1, eps_p=0.0)
            cp = CheckPlan(ref, cand, tol, fmt=FloatFormat.BF16)
            ptrs, keep = resolve_operands(cp.plan.operands, cp.plan.operand_dtypes)
            prep = cp.plan.prepare(ptrs, kappa=3.0, eps=FloatFormat.BF16.eps,
                                   replica_eps=FloatFormat.BF16.eps)
            seg_ms, step_ms = [], []
            for rep in range(args.reps + 3):
                flush.zero_()
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
                ev[0].record()
                prep.segnorm(N.stream_handle())
                ev[1].record()
                prep.finalize(N.stream_handle())
                ev[2].record()
                torch.cuda.synchronize()
                if rep >= 3:
                    seg_ms.append(ev[0].elapsed_time(ev[1]))
                    step_ms.append(ev[0].elapsed_time(ev[2]))
            seg = sorted(seg_ms)[len(seg_ms) // 2]
            step = sorted(step_ms)[len(step_ms) // 2]
            # the same check as one CUDA-graph replay (launch latency folded)
            graph = prep.capture()
            gms = []
            for rep in range(args.reps + 3):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                graph.replay()
                e1.record()
                torch.cuda.synchronize()
                if rep >= 3:
                    gms.append(e0.elapsed_time(e1))
            gstep = sorted(gms)[len(gms) // 2]
            b = cp.algorithmic_bytes
            print(json.dumps({"mib": mib, "maps": maps, "shards": int(g), "bytes": b,
                              "segnorm_ms": seg, "segnorm_gbs": b / seg / 1e6, "frac": b / seg / 1e6 / peak,
                              "check_ms": step, "check_gbs": b / step / 1e6,
                              "checks_per_s": 1e3 / step, "graph_check_ms": gstep,
                              "graph_checks_per_s": 1e3 / gstep}), flush=True)
            del keep, prep, cp, ref, cand
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
