"""The warm-check record walks in C++ (csrc/td_host.cpp) against their
Python twins: checker._layout_key / _host_bytes and
device._resolve_resident must return the same values (the layout key is a
plan-cache key, so equal AND equally hashed), including the cases the C
side hands back to Python."""
import gzip
import glob
import os

import numpy as np
import pytest
import torch

from paper_2506_09280_b200 import _native as N
from paper_2506_09280_b200 import checker as C
from paper_2506_09280_b200 import device as D
from paper_2506_09280_b200.canonical import CanonicalId, TensorKind, identity_mapping
from paper_2506_09280_b200.tracestore import RankMeta, Trace, TraceRecord, trace_from_bytes

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "traces")


def _ext():
    ext = N.host_ext()
    if ext is None:
        pytest.skip("_td_host not built")
    return ext


def _trace(payloads):
    t = Trace(header={"digest": "x", "mode": "cascade"})
    for k, p in enumerate(payloads):
        ident = CanonicalId(0, k % 2, TensorKind.ACTIVATION_OUT, f"model.layers.{k}.mlp")
        t.records.append(TraceRecord(ident, RankMeta(tp=k % 3, dp=k % 2), identity_mapping(tuple(p.shape)),
                                     1 + k % 2, p, "MLP"))
    return t


def test_module_is_built_and_loaded():
    from paper_2506_09280_b200 import build
    if os.path.exists(build.host_output()):
        assert N.host_ext() is not None


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "*.ttrc.gz")))[:8])
def test_layout_key_numpy_payloads(path):
    _ext()
    t = trace_from_bytes(gzip.open(path).read())
    a, b = C._layout_key(t), C._layout_key_py(t)
    assert a == b and hash(a) == hash(b)
    assert C._host_bytes(t) == C._host_bytes_py(t)


def test_layout_key_and_host_bytes_torch_payloads():
    _ext()
    g = torch.Generator().manual_seed(3)
    pays = [torch.randn((4, 8), generator=g).to(dt) for dt in (torch.float32, torch.bfloat16, torch.float16,
                                                             torch.float64)]
    pays += [torch.randn((), generator=g), torch.zeros((0, 5)), torch.randn((3, 1, 2), generator=g)]
    t = _trace(pays)
    a, b = C._layout_key(t), C._layout_key_py(t)
    assert a == b and hash(a) == hash(b)
    assert C._host_bytes(t) == C._host_bytes_py(t) == sum(p.numel() * p.element_size() for p in pays)


def test_layout_key_unsupported_dtype_raises_like_python():
    _ext()
    t = _trace([torch.zeros((2, 2), dtype=torch.float8_e4m3fn)])
    with pytest.raises(TypeError):
        C._layout_key_py(t)
    with pytest.raises(TypeError):
        C._layout_key(t)


@pytest.mark.gpu
def test_resident_pointers_match_python():
    _ext()
    D.resolve_operands([], [])          # initialises the dtype table the Python twin reads
    g = torch.Generator(device="cuda").manual_seed(5)
    base = torch.randn((64, 32), generator=g, device="cuda")
    pays = [base.to(torch.bfloat16), base[:16].clone(), base.double(), base.half()[8:24]]
    t = _trace(pays)
    ops, dts = t.records, [N.dtype_code(p) for p in pays]
    got, want = D._resolve_resident(ops, dts, None), D._resolve_resident_py(ops, dts)
    assert got is not None and want is not None
    assert np.array_equal(got[0], want[0]) and all(x is y for x, y in zip(got[1], want[1]))
    assert C._host_bytes(t) == C._host_bytes_py(t) == 0
    # every case the fast path declines, declined by both
    odd = torch.zeros(17, dtype=torch.bfloat16, device="cuda")[1:]           # 2-byte aligned
    strided = _trace([base.t().contiguous()])
    strided.records[0].payload = base.t()       # records normalise payloads; a later assignment does not
    cases = [
        (_trace([odd]).records, [N.BF16]),
        (strided.records, [N.F32]),                                            # not contiguous
        (_trace([base]).records, [N.BF16]),                                    # needs a widening cast
        (_trace([base.cpu()]).records, [N.F32]),                               # host payload
        ([D._Raw(base.reshape(-1))], [N.F32]),                                 # not a record
    ]
    for recs, d in cases:
        assert D._resolve_resident(recs, d, None) is None
        assert D._resolve_resident_py(recs, d) is None
    mixed = _trace([base, base.cpu()])
    assert C._host_bytes(mixed) == C._host_bytes_py(mixed) == base.numel() * 4


@pytest.mark.gpu
def test_check_reports_equal_with_and_without_the_extension(cases, golden_trace_bytes):
    import paper_2506_09280_b200 as td
    _ext()
    for case in cases["checks"][:6]:
        ref = trace_from_bytes(golden_trace_bytes(case["ref"]), device="cuda")
        cand = trace_from_bytes(golden_trace_bytes(case["cand"]), device="cuda")
        tol = td.ToleranceMap.from_json(cases["tols"][case["tol"]])
        fmt = td.FloatFormat(case["fmt"])
        runs = []
        for on in (True, False, True):           # cold, then Python walks on the cached plan, then C again
            saved = N._HOST_EXT
            N._HOST_EXT = saved if on else False
            try:
                runs.append(td.render_report(td.check(ref, cand, tol, case["kappa"], fmt=fmt), "json"))
            finally:
                N._HOST_EXT = saved
        assert runs[0] == runs[1] == runs[2], case["name"]


def _view_signature(view):
    return [(ident, m.exec_index, m.global_shape, m.rank_problem, m.merge_detail, m.struct_key,
             [([id(r) for r in g.records], g.declared_detail, g.numeric) for g in m.groups])
            for ident, m in view.items()]


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "*.ttrc.gz"))))
def test_grouped_merge_view_equals_python(path):
    """merge_view over _td_host.group_by_id == merge_view's Python walk
    (every golden trace: TP/SP/CP/PP/DP layouts, replica groups, shard maps)."""
    from paper_2506_09280_b200 import plan as P
    _ext()
    t = trace_from_bytes(gzip.open(path).read())
    grouped = P.merge_view(t)
    saved = N._HOST_EXT
    N._HOST_EXT = False
    try:
        plain = P.merge_view(t)
    finally:
        N._HOST_EXT = saved
    assert _view_signature(grouped) == _view_signature(plain)
    ids, pos, keys = N.host_ext().group_by_id(t.records)
    assert ids == list(t.by_id()) and pos == [[k for k, _ in e] for e in t.by_id().values()]
