"""Cold DistributedCheckPlan construction of one config-4 share (rank 0 of the
8-GPU TP=2 x DP=4 job) from metadata alone (meta-device payloads, StaticComm).

    python tools/dplan_profile.py [prof]
"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_09280_b200 import layout as L, synthetic
from paper_2506_09280_b200.canonical import parse_canonical
from paper_2506_09280_b200.tracestore import Trace, TraceRecord, RankMeta
from paper_2506_09280_b200.distributed import DistributedCheckPlan, StaticComm
from paper_2506_09280_b200.checker import ToleranceMap
from paper_2506_09280_b200.tensor import FloatFormat
lay = synthetic.ShareLayout(L.LLAMA3_8B, L.ParallelConfig(tp=2, dp=4, microbatches=4), 8)
hdr={"digest":"x","mode":"cascade"}
def traces(rank):
    ref, cand = Trace(header=dict(hdr)), Trace(header=dict(hdr))
    for ident, s in lay.cand[rank]:
        cand.records.append(TraceRecord(parse_canonical(ident), RankMeta(*s.rank), s.mapping, s.replica, torch.empty(s.mapping.local_shape, dtype=torch.bfloat16, device="meta"), s.module_class))
    for ident, k, m, mc in lay.ref[rank]:
        ref.records.append(TraceRecord(parse_canonical(ident), RankMeta(0, k, 0, 0, 0, 0), m, 1, torch.empty(m.local_shape, dtype=torch.bfloat16, device="meta"), mc))
    return ref, cand
ref, cand = traces(0)
rm, cm = lay.metas()
tol = ToleranceMap({i: 2**-7 for i in lay.ids}, n_samples=1, eps_p=2**-8)
for rep in range(3):
    t0=time.perf_counter()
    dcp = DistributedCheckPlan(ref, cand, tol, 3.0, fmt=FloatFormat.BF16, comm=StaticComm(0, 8, [rm, cm]))
    print("dplan", round((time.perf_counter()-t0)*1e3,1), "ms")
if len(sys.argv) > 1:
    pr=cProfile.Profile(); pr.enable()
    DistributedCheckPlan(ref, cand, tol, 3.0, fmt=FloatFormat.BF16, comm=StaticComm(0, 8, [rm, cm]))
    pr.disable(); pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
