"""The planner's per-entry templates (plan.py: record the first id of each
structure, replay it for the others) produce exactly the plan of the
general per-entry path: every device table, every operand, every group
slot — over the golden traces of the reference (all check scenarios, bugs
included), randomised shardings, and the BASELINE configs' layouts built
from metadata alone (meta-device payloads)."""

import gzip
import json
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


def _same(a, b):
    assert a.segs.tobytes() == b.segs.tobytes()
    assert a.ids.tobytes() == b.ids.tobytes() and a.groups.tobytes() == b.groups.tobytes()
    for f in ("tile_seg", "seg_xslot", "seg_xoff", "seg_yslot", "seg_yoff", "seg_zslot"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert a.class_keys == b.class_keys and a.class_segs == b.class_segs
    assert all(np.array_equal(x, y) for x, y in zip(a.class_lists, b.class_lists))
    assert [id(o) for o in a.operands] == [id(o) for o in b.operands]
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
