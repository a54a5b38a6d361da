"""The BASELINE configs' trace shapes at reduced size, with the config-3 bug
injections, checked end to end on the GPU against the CPU oracle on the
very same traces (host copies): identical verdicts and details, norms
within 1e-12."""

import json

import pytest
import torch

from oracle import traindiff_oracle as O

pytestmark = pytest.mark.gpu


def _oracle_recs(trace):
    return [O.Rec(r.id.encode(), r.rank_meta.as_tuple(), r.mapping.local_shape, r.mapping.global_shape,
                  [(l.bounds, g.bounds) for l, g in r.mapping.pairs], r.replica_group_size,
                  r.payload.float().cpu().numpy()) for r in trace.records]


def _compare(ref, cand, tol, fmt):
    import paper_2506_09280_b200 as td
    from tests.test_gpu_parity import assert_reports_match
    rep = td.check(ref, cand, tol, fmt=fmt)
    want = O.check(_oracle_recs(ref), _oracle_recs(cand), ref.header, cand.header, tol.responses,
                   3.0, fmt.value)
    assert_reports_match(json.loads(td.render_report(rep, "json")), want)
    return rep


@pytest.fixture(autouse=True, scope="module")
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def test_config3_llama_tp8_injected_bugs():
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200 import layout as L, synthetic
    m = L.ModelShape(layers=2, d_model=256, n_heads=8, d_ff=512, seq_len=128, vocab=1024,
                     n_kv_heads=2, gated_mlp=True, norm_bias=False, position_table=False)
    p = L.ParallelConfig(tp=8)
    bugs = {"iter=0|mb=0|kind=ActivationOut|mod=model.lm_head": "order",          # wrong shard order
            "iter=0|mb=0|kind=ActivationOut|mod=model.layers.1.attn": "partial",    # missing allreduce
            "iter=0|mb=0|kind=ActivationOut|mod=model.embedding": "scale"}          # scale error
    ref, cand = synthetic.build(m, p, bugs=bugs, seed=3)
    eps = td.FloatFormat.BF16.eps
    tol = td.ToleranceMap({r.id.encode(): 2 * eps for r in ref.records}, n_samples=1, eps_p=eps)
    rep = _compare(ref, cand, tol, td.FloatFormat.BF16)
    verdicts = {e.ident: e.verdict for e in rep.entries}
    assert verdicts["iter=0|mb=0|kind=ActivationOut|mod=model.lm_head"] == "flag"
    assert verdicts["iter=0|mb=0|kind=ActivationOut|mod=model.layers.1.attn"] == "replica-mismatch"
    assert verdicts["iter=0|mb=0|kind=ActivationOut|mod=model.embedding"] == "flag"
    assert rep.earliest_divergence == "iter=0|mb=0|kind=ActivationOut|mod=model.embedding"
    assert rep.counts["flag"] == 2 and rep.counts["replica-mismatch"] == 1
    assert rep.exit_code() == 3


def test_config1_fp32_tp2_and_config2_bf16_tp4_clean():
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200 import layout as L, synthetic
    m1 = L.ModelShape(layers=2, d_model=96, n_heads=12, d_ff=384, seq_len=64, vocab=512)
    ref, cand = synthetic.build(m1, L.ParallelConfig(tp=2), dtype=torch.float32, eps=2.0 ** -24)
    tol = td.ToleranceMap({r.id.encode(): 2.0 ** -23 for r in ref.records}, n_samples=1, eps_p=2.0 ** -24)
    rep = _compare(ref, cand, tol, td.FloatFormat.FP32)
    assert rep.exit_code() == 0
    m2 = L.ModelShape(layers=3, d_model=128, n_heads=16, d_ff=512, seq_len=64, vocab=1024)
    ref, cand = synthetic.build(m2, L.ParallelConfig(tp=4, dp=2, microbatches=2))
    eps = td.FloatFormat.BF16.eps
    tol = td.ToleranceMap({r.id.encode(): 2 * eps for r in ref.records}, n_samples=1, eps_p=eps)
    rep = _compare(ref, cand, tol, td.FloatFormat.BF16)
    assert rep.exit_code() == 0 and rep.counts["missing"] == 0


def test_config4_shape_tp2_dp2_sp_cp_layout():
    """Llama-8B-shaped id grammar (GQA, w3, RMSNorm) under TP2 x DP2 with SP
    and CP=2 zigzag stripes — multi-pair shard maps, sub-sliced rows."""
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200 import layout as L, synthetic
    m = L.ModelShape(layers=2, d_model=128, n_heads=8, d_ff=448, seq_len=64, vocab=512,
                     n_kv_heads=2, gated_mlp=True, norm_bias=False, position_table=False)
    p = L.ParallelConfig(tp=2, dp=2, cp=2, sp=True, microbatches=2)
    ref, cand = synthetic.build(m, p, seed=5)
    eps = td.FloatFormat.BF16.eps
    tol = td.ToleranceMap({r.id.encode(): 2 * eps for r in ref.records}, n_samples=1, eps_p=eps)
    rep = _compare(ref, cand, tol, td.FloatFormat.BF16)
    assert rep.exit_code() == 0


def test_fuzzed_layouts_and_bugs_match_oracle():
    """A slice of tools/fuzz_parity.py: random small models x random valid
    parallel layouts (tp/dp/pp/vp/cp/sp/microbatches) x random storage dtype,
    kappa and injected bugs — device check == CPU oracle on every case."""
    import random
    import sys
    import os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import fuzz_parity
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200 import synthetic
    rnd = random.Random(1234)
    for k in range(40):
        m, p, bugs = fuzz_parity.random_case(rnd)
        dtype = rnd.choice([torch.bfloat16, torch.float32, torch.float16])
        fmt = td.FloatFormat.BF16 if dtype != torch.float32 else td.FloatFormat.FP32
        ref, cand = synthetic.build(m, p, dtype=dtype, seed=k, eps=fmt.eps, bugs=bugs)
        fuzz_parity.scramble_dtypes(rnd, ref, cand)
        tol = td.ToleranceMap({r.id.encode(): 2 * fmt.eps for r in ref.records}, n_samples=1, eps_p=fmt.eps)
        _compare(ref, cand, tol, fmt)
