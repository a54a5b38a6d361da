"""Cold-plan cost of check() on CPU (no GPU needed): the named configs'
layouts with meta-device payloads (shapes and dtypes only), timed through
CheckPlan's host planner (merge views + Plan construction).

    python tools/plan_profile.py [cfg2|cfg3] [--profile]
"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2506_09280_b200 import layout as L  # noqa: E402
from paper_2506_09280_b200.canonical import parse_canonical  # noqa: E402
from paper_2506_09280_b200.checker import CheckPlan, ToleranceMap  # noqa: E402
from paper_2506_09280_b200.tensor import FloatFormat  # noqa: E402
from paper_2506_09280_b200.tracestore import RankMeta, Trace, TraceRecord  # noqa: E402

CFGS = {"cfg2": (L.GPT2_MEDIUM, L.ParallelConfig(tp=4)),
        "cfg3": (L.LLAMA3_1B, L.ParallelConfig(tp=8)),
        "cfg4": (L.LLAMA3_8B, L.ParallelConfig(tp=2, dp=4, microbatches=4))}


def meta_trace(specs, hdr):
    t = Trace(header=dict(hdr))
    for s in specs:
        payload = torch.empty(s.mapping.local_shape, dtype=torch.bfloat16, device="meta")
        t.records.append(TraceRecord(parse_canonical(s.ident), RankMeta(*s.rank), s.mapping, s.replica,
                                     payload, s.module_class))
    return t


def main(name="cfg2", profile=False):
    model, pcfg = CFGS[name]
    hdr = {"digest": "plan-profile", "mode": "cascade"}
    ref = meta_trace(L.emit_records(model, L.ParallelConfig(microbatches=pcfg.microbatches)), hdr)
    cand = meta_trace(L.emit_records(model, pcfg), hdr)
    tol = ToleranceMap({}, n_samples=1, eps_p=2.0 ** -8)
    from paper_2506_09280_b200 import plan as PL
    times = []
    for _ in range(int(os.environ.get("PP_RUNS", "7"))):
        PL._MERGE_DETAIL.clear()          # cold: no memoised merge witnesses
        PL._RUN_BLOCKS.clear()
        PL._run_blocks.cache_clear()
        t0 = time.perf_counter()
        CheckPlan(ref, cand, tol, fmt=FloatFormat.BF16)
        times.append(time.perf_counter() - t0)
    times.sort()
    print(f"{name}: {len(ref.records)} ref + {len(cand.records)} cand records, cold plan "
          f"min {times[0] * 1e3:.1f} ms, median {times[len(times) // 2] * 1e3:.1f} ms")
    if profile:
        pr = cProfile.Profile()
        pr.enable()
        CheckPlan(ref, cand, tol, fmt=FloatFormat.BF16)
        pr.disable()
        pstats.Stats(pr).sort_stats("cumulative").print_stats(30)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "cfg2", "--profile" in sys.argv)
