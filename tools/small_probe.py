"""Config 5 small-tensor probe: one identity id per size, td_segnorm timed
alone with CUDA events, median of --reps, under
  * flush "write"      : 256 MiB memset before each rep (L2 left full of
                         dirty lines that drain during the timed kernel)
  * flush "write+read" : the memset, then a read of a second 256 MiB buffer
                         (L2 left clean, holding none of the inputs)
and several planner tile targets (Plan.TARGET_TILES) / CTAs per SM.

    python tools/small_probe.py [--sizes 16,64,256] [--targets 1184,2368,4736]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="16,64,256,1024")
    ap.add_argument("--targets", default="1184,2368,4736,9472")
    ap.add_argument("--bps", default="4")
    ap.add_argument("--reps", type=int, default=30)
    args = ap.parse_args()
    import torch
    from paper_2506_09280_b200 import _native as N
    from paper_2506_09280_b200 import plan as PL
    from paper_2506_09280_b200 import synthetic
    from paper_2506_09280_b200.checker import CheckPlan, ToleranceMap
    from paper_2506_09280_b200.device import resolve_operands
    from paper_2506_09280_b200.tensor import FloatFormat
    fa = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    fb = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
    sink = torch.empty((), dtype=torch.int64, device="cuda")

    def flush(mode):
        fa.zero_()
        if mode == "write+read":
            sink.copy_(fb.view(torch.int64).sum())

    for mib in [int(s) for s in args.sizes.split(",")]:
        ref, cand = synthetic.sweep_pair(mib << 20)
        for target in [int(t) for t in args.targets.split(",")]:
            PL.Plan.TARGET_TILES = target
            cp = CheckPlan(ref, cand, ToleranceMap({}, n_samples=1, eps_p=0.0), fmt=FloatFormat.BF16)
            ptrs, keep = resolve_operands(cp.plan.operands, cp.plan.operand_dtypes)
            prep = cp.plan.prepare(ptrs, kappa=3.0, eps=FloatFormat.BF16.eps, replica_eps=FloatFormat.BF16.eps)
            b = cp.algorithmic_bytes
            for bps in [int(x) for x in args.bps.split(",")]:
                for mode in ("write", "write+read"):
                    ms = []
                    for rep in range(args.reps + 3):
                        flush(mode)
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        sh = N.stream_handle()
                        e0.record()
                        N.call("td_segnorm", prep.seg_ptr, prep.classes.ctypes.data, len(prep.classes),
                               prep.part_ptr, bps, sh)
                        e1.record()
                        torch.cuda.synchronize()
                        if rep >= 3:
                            ms.append(e0.elapsed_time(e1))
                    med = sorted(ms)[len(ms) // 2]
                    print(json.dumps({"mib": mib, "target": target, "tiles": cp.plan.n_tiles,
                                      "tile_units": cp.plan.tile_units, "bps": bps, "flush": mode,
                                      "ms": round(med, 5), "gbs": round(b / med / 1e6, 1)}), flush=True)
            del keep, prep, cp
        # comparator: torch's own int64 sum over the same number of bytes
        rd = torch.ones(2 * (mib << 20) // 8, dtype=torch.int64, device="cuda")
        for mode in ("write", "write+read"):
            ms = []
            for rep in range(args.reps + 3):
                flush(mode)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                rd.sum()
                e1.record()
                torch.cuda.synchronize()
                if rep >= 3:
                    ms.append(e0.elapsed_time(e1))
            med = sorted(ms)[len(ms) // 2]
            print(json.dumps({"mib": mib, "target": "torch.sum", "tiles": 0, "tile_units": 0, "bps": 0,
                              "flush": mode, "ms": round(med, 5), "gbs": round(rd.numel() * 8 / med / 1e6, 1)}),
                  flush=True)
        del rd, ref, cand
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
