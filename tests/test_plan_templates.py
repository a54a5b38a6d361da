"""The planner's per-entry templates (plan.py: record the first id of each
structure, replay it for the others) produce exactly the plan of the
general per-entry path: every device table, every operand, every group
slot — over the golden traces of the reference (all check scenarios, bugs
included), randomised shardings, and the BASELINE configs' layouts built
from metadata alone (meta-device payloads)."""

import os

import numpy as np
import pytest
import torch

from paper_2506_09280_b200 import layout as L
from paper_2506_09280_b200 import plan as PL
from paper_2506_09280_b200.canonical import parse_canonical
from paper_2506_09280_b200.tracestore import RankMeta, Trace, TraceRecord, trace_from_bytes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _plan(ref, cand, templates, monkeypatch, x_rep=True):
    monkeypatch.setattr(PL, "_TEMPLATES", templates)
    rv, cv = PL.merge_view(ref), PL.merge_view(cand)
    common = [i for i in cv if i in rv]
    return PL.Plan([PL.PlanEntry(i, x=rv[i], y=cv[i], x_rep=x_rep, y_rep=True, tolerance=0.01 * k)
                    for k, i in enumerate(common)])


def _same(a, b, opkey=id):
    assert a.segs.tobytes() == b.segs.tobytes()
    assert a.ids.tobytes() == b.ids.tobytes() and a.groups.tobytes() == b.groups.tobytes()
    for f in ("tile_seg", "seg_xslot", "seg_xoff", "seg_yslot", "seg_yoff", "seg_zslot"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert a.class_keys == b.class_keys and a.class_segs == b.class_segs
    assert all(np.array_equal(x, y) for x, y in zip(a.class_lists, b.class_lists))
    assert [opkey(o) for o in a.operands] == [opkey(o) for o in b.operands]
    assert a.operand_dtypes == b.operand_dtypes
    assert a.group_owner == b.group_owner and a.group_offset == b.group_offset and a.subslots == b.subslots
    assert a.algorithmic_bytes == b.algorithmic_bytes and a.n_tiles == b.n_tiles


def _same_view(trace, monkeypatch):
    monkeypatch.setattr(PL, "_TEMPLATES", True)
    a = PL.merge_view(trace)
    monkeypatch.setattr(PL, "_TEMPLATES", False)
    b = PL.merge_view(trace)
    assert list(a) == list(b)
    for ident in a:
        x, y = a[ident], b[ident]
        assert (x.exec_index, x.global_shape, x.rank_problem, x.merge_detail) == \
            (y.exec_index, y.global_shape, y.rank_problem, y.merge_detail), ident
        assert [([id(r) for r in g.records], g.declared_detail, g.numeric) for g in x.groups] == \
            [([id(r) for r in g.records], g.declared_detail, g.numeric) for g in y.groups], ident


def _meta_trace(specs):
    t = Trace(header={"digest": "t", "mode": "cascade"})
    for s in specs:
        t.records.append(TraceRecord(parse_canonical(s.ident), RankMeta(*s.rank), s.mapping, s.replica,
                                     torch.empty(s.mapping.local_shape, dtype=torch.bfloat16, device="meta"),
                                     s.module_class))
    return t


def test_templates_equal_general_path_on_golden_scenarios(cases, golden_trace_bytes, monkeypatch):
    for case in cases["checks"]:
        ref = trace_from_bytes(golden_trace_bytes(case["ref"]))
        cand = trace_from_bytes(golden_trace_bytes(case["cand"]))
        _same(_plan(ref, cand, True, monkeypatch), _plan(ref, cand, False, monkeypatch))
        _same_view(ref, monkeypatch)
        _same_view(cand, monkeypatch)
        # a trace against itself: sides share record objects (no templates)
        _same(_plan(cand, cand, True, monkeypatch), _plan(cand, cand, False, monkeypatch))


@pytest.mark.parametrize("model,pcfg", [
    (L.GPT2_MEDIUM, L.ParallelConfig(tp=4)),
    (L.LLAMA3_1B, L.ParallelConfig(tp=8)),
    (L.LLAMA3_8B, L.ParallelConfig(tp=2, dp=4, microbatches=4)),
    (L.ModelShape(layers=4, d_model=64, n_heads=4, d_ff=128, seq_len=32, vocab=96),
     L.ParallelConfig(tp=2, cp=2, pp=2, microbatches=2)),
    (L.ModelShape(layers=4, d_model=64, n_heads=4, d_ff=128, seq_len=32, vocab=96),
     L.ParallelConfig(tp=2, sp=True, dp=2, microbatches=2)),
], ids=["cfg2", "cfg3", "cfg4", "tp2cp2pp2", "tp2sp_dp2"])
def test_templates_equal_general_path_on_layouts(model, pcfg, monkeypatch):
    ref = _meta_trace(L.emit_records(model, L.ParallelConfig(microbatches=pcfg.microbatches)))
    cand = _meta_trace(L.emit_records(model, pcfg))
    _same(_plan(ref, cand, True, monkeypatch), _plan(ref, cand, False, monkeypatch))
    _same_view(cand, monkeypatch)
    _same(_plan(ref, cand, True, monkeypatch, x_rep=False), _plan(ref, cand, False, monkeypatch, x_rep=False))


def _share_traces(lay, rank):
    from paper_2506_09280_b200.canonical import parse_canonical as pc
    hdr = {"digest": "t", "mode": "cascade"}
    ref, cand = Trace(header=dict(hdr)), Trace(header=dict(hdr))
    for ident, s in lay.cand[rank]:
        cand.records.append(TraceRecord(pc(ident), RankMeta(*s.rank), s.mapping, s.replica,
                                        torch.empty(s.mapping.local_shape, dtype=torch.bfloat16, device="meta"),
                                        s.module_class))
    for ident, k, m, mc in lay.ref[rank]:
        ref.records.append(TraceRecord(pc(ident), RankMeta(0, k, 0, 0, 0, 0), m, 1,
                                       torch.empty(m.local_shape, dtype=torch.bfloat16, device="meta"), mc))
    return ref, cand


@pytest.mark.parametrize("model,pcfg,world,ranks", [
    (L.ModelShape(layers=8, d_model=256, n_heads=8, d_ff=512, seq_len=64, vocab=320, n_kv_heads=2,
                  gated_mlp=True, norm_bias=False, position_table=False),
     L.ParallelConfig(tp=2, dp=4, microbatches=4), 8, range(8)),
    (L.ModelShape(layers=4, d_model=64, n_heads=4, d_ff=128, seq_len=32, vocab=96),
     L.ParallelConfig(tp=4, microbatches=1), 3, range(3)),
    (L.LLAMA3_8B, L.ParallelConfig(tp=2, dp=4, microbatches=4), 8, (0, 5)),
], ids=["tp2dp4", "tp4_on_3", "cfg4"])
def test_templates_equal_general_path_on_distributed_plans(model, pcfg, world, ranks, monkeypatch):
    """Owner-aware plans (every rank of a multi-GPU job planned from the
    global metadata, compares balanced over replica holders, digests fused
    in the compare pass): templated == general path, including the
    cross-rank group lists and fused digest slots."""
    from paper_2506_09280_b200 import synthetic
    from paper_2506_09280_b200.checker import ToleranceMap
    from paper_2506_09280_b200.distributed import DistributedCheckPlan, StaticComm
    from paper_2506_09280_b200.tensor import FloatFormat
    lay = synthetic.ShareLayout(model, pcfg, world)
    rm, cm = lay.metas()
    tol = ToleranceMap({i: 2.0 ** -7 for i in lay.ids}, n_samples=1, eps_p=2.0 ** -8)
    for rank in ranks:
        ref, cand = _share_traces(lay, rank)
        plans = []
        for flag in (True, False):
            monkeypatch.setattr(PL, "_TEMPLATES", flag)
            plans.append(DistributedCheckPlan(ref, cand, tol, 3.0, fmt=FloatFormat.BF16,
                                              comm=StaticComm(rank, world, [rm, cm])))
        a, b = plans[0].plan, plans[1].plan
        # operands are this rank's RecordMeta objects, rebuilt per plan
        _same(a, b, opkey=lambda m: (m.id.encode(), m.rank_meta.as_tuple(), m.owner))
        assert a.remote_groups == b.remote_groups and a.compare_reads == b.compare_reads
        assert a.fused_digests == b.fused_digests
        assert plans[0].where == plans[1].where and np.array_equal(plans[0].copy_off, plans[1].copy_off)
