"""BASELINE configs at full size.  Configs 1 and 2 (2.8 GB, 8.2 GB) run the CPU
oracle on the whole trace: identical reports.  Config 3 (Llama-3-1B shape, S=8192, TP=8, 69 GB
of bf16 traces in HBM) with the three injected bugs.  Too big for the CPU
oracle as a whole, so: the verdicts are exactly the injections; the CPU
oracle re-checks a sample of ids (every 16th id under 256 MB of reference
payload, plus the replica and scale bugs — each id's report entry is
independent of the others') and its entries equal ours; and the observed
rel_err of the bug ids (the 2.1 GB logits included) equals an independent
torch fp64 computation over the materialised merges (copy 0 of every shard
group, reference semantics) within 1e-12."""

import pytest
import torch

pytestmark = pytest.mark.gpu

BUGS = {"iter=0|mb=0|kind=ActivationOut|mod=model.lm_head": "order",
        "iter=0|mb=0|kind=ActivationOut|mod=model.layers.7.attn": "partial",
        "iter=0|mb=0|kind=ActivationOut|mod=model.embedding": "scale"}


def _merged_f64(trace, ident):
    """merge() of copy 0 of each shard group, in fp64, with torch indexing."""
    recs = [r for r in trace.records if r.id.encode() == ident]
    seen, out = set(), None
    for r in recs:
        key = (tuple(r.mapping.local_shape), tuple((l.bounds, g.bounds) for l, g in r.mapping.pairs))
        if key in seen:
            continue
        seen.add(key)
        if out is None:
            out = torch.zeros(r.mapping.global_shape, dtype=torch.float64, device="cuda")
        for loc, glob in r.mapping.pairs:
            out[glob.as_slices()] = r.payload[loc.as_slices()].double()
    return out


def _rel_err_fp64(a, b):
    d = torch.linalg.vector_norm((a - b).reshape(-1), dtype=torch.float64)
    r = torch.linalg.vector_norm(a.reshape(-1), dtype=torch.float64)
    return float(d / r)


def test_config3_full_size_injections_and_fp64_norms():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if torch.cuda.get_device_properties(0).total_memory < 150e9:
        pytest.skip("needs a 180 GB B200")
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200 import layout as L, synthetic
    ref, cand = synthetic.build(L.LLAMA3_1B, L.ParallelConfig(tp=8), bugs=BUGS, seed=0)
    eps = td.FloatFormat.BF16.eps
    tol = td.ToleranceMap({r.id.encode(): 2 * eps for r in ref.records}, n_samples=1, eps_p=eps)
    rep = td.check(ref, cand, tol, fmt=td.FloatFormat.BF16)
    verdicts = {e.ident: e for e in rep.entries}
    assert rep.counts["flag"] == 2 and rep.counts["replica-mismatch"] == 1
    assert rep.counts["pass"] == len(rep.entries) - 3 and rep.near_ties == 0
    assert verdicts[[k for k, v in BUGS.items() if v == "order"][0]].verdict == "flag"
    assert verdicts[[k for k, v in BUGS.items() if v == "scale"][0]].verdict == "flag"
    partial = verdicts[[k for k, v in BUGS.items() if v == "partial"][0]]
    assert partial.verdict == "replica-mismatch" and partial.detail.startswith("replicas diverge")
    sample = list(BUGS) + ["iter=0|mb=0|kind=ActivationIn|mod=model.layers.15.mlp",
                           "iter=0|mb=0|kind=ParamGrad|mod=model.layers.3.mlp.w1",
                           "iter=0|mb=0|kind=ActivationOut|mod=model.layers.0.attn"]
    for ident in sample:
        if ident not in verdicts:
            continue
        want = _rel_err_fp64(_merged_f64(ref, ident), _merged_f64(cand, ident))
        got = verdicts[ident].observed
        assert abs(got - want) <= 1e-12 * want, (ident, got, want)
        torch.cuda.empty_cache()
    # the scale bug multiplies by tp = 8 exactly: rel_err of 8x vs x is 7 up
    # to the simulated round-off
    assert abs(verdicts[[k for k, v in BUGS.items() if v == "scale"][0]].observed - 7.0) < 0.1
    # the CPU oracle on a sample of ids
    from oracle import traindiff_oracle as O
    from tests.test_gpu_parity import _close
    ref_bytes = {}
    for r in ref.records:
        ref_bytes[r.id.encode()] = ref_bytes.get(r.id.encode(), 0) + r.nbytes
    ids = [e.ident for e in rep.entries]
    sample = {i for i in ids[::16] if ref_bytes.get(i, 0) < (256 << 20)}
    sample |= {k for k, v in BUGS.items() if v != "order"}
    assert len(sample) >= 30

    def host(trace):
        return [O.Rec(r.id.encode(), r.rank_meta.as_tuple(), r.mapping.local_shape, r.mapping.global_shape,
                      [(lb.bounds, gb.bounds) for lb, gb in r.mapping.pairs], r.replica_group_size,
                      r.payload.float().cpu().numpy()) for r in trace.records if r.id.encode() in sample]
    doc = O.check(host(ref), host(cand), ref.header, cand.header, tol.responses, 3.0, "BF16")
    assert {e["id"] for e in doc["entries"]} == sample
    for w in doc["entries"]:
        g = verdicts[w["id"]]
        assert (g.verdict, g.detail) == (w["verdict"], w["detail"]), (w["id"], g, w)
        assert _close(g.observed, w["observed"]), (w["id"], g.observed, w["observed"])
        assert _close(g.threshold, w["threshold"])


def test_config1_full_size_against_cpu_oracle():
    """Config 1 at its full size (GPT-2-small shape, L=2, S=1024, V=50304,
    fp32, TP=2 candidate: 123 ids, 2.8 GB) — small enough for the CPU
    oracle on the whole trace: identical report (verdicts, details,
    thresholds; observed within 1e-12)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import json

    import paper_2506_09280_b200 as td
    from oracle import traindiff_oracle as O
    from paper_2506_09280_b200 import layout as L, synthetic
    from tests.test_configs_gpu import _oracle_recs
    from tests.test_gpu_parity import assert_reports_match
    eps = td.FloatFormat.FP32.eps
    ref, cand = synthetic.build(L.GPT2_SMALL_L2, L.ParallelConfig(tp=2), dtype=torch.float32, eps=eps, seed=1)
    tol = td.ToleranceMap({r.id.encode(): 2 * eps for r in ref.records}, n_samples=1, eps_p=eps)
    rep = td.check(ref, cand, tol, fmt=td.FloatFormat.FP32)
    assert len(rep.entries) == 123
    want = O.check(_oracle_recs(ref), _oracle_recs(cand), ref.header, cand.header, tol.responses, 3.0, "FP32")
    assert_reports_match(json.loads(td.render_report(rep, "json")), want, "config1 full size")


def test_config2_full_size_against_cpu_oracle():
    """Config 2, the bench workload, at its full size (GPT-2-medium shape,
    bf16, TP=4 candidate: 1179 ids, 8.2 GB) against the CPU oracle on the
    whole trace (~40 s of numpy): identical report."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import json

    import paper_2506_09280_b200 as td
    from oracle import traindiff_oracle as O
    from paper_2506_09280_b200 import layout as L, synthetic
    from tests.test_configs_gpu import _oracle_recs
    from tests.test_gpu_parity import assert_reports_match
    eps = td.FloatFormat.BF16.eps
    ref, cand = synthetic.build(L.GPT2_MEDIUM, L.ParallelConfig(tp=4), eps=eps, seed=2)
    tol = td.ToleranceMap({r.id.encode(): 2 * eps for r in ref.records}, n_samples=1, eps_p=eps)
    rep = td.check(ref, cand, tol, fmt=td.FloatFormat.BF16)
    assert len(rep.entries) == 1179 and rep.near_ties == 0
    got = json.loads(td.render_report(rep, "json"))
    rrecs, crecs, rh, ch = _oracle_recs(ref), _oracle_recs(cand), ref.header, cand.header
    del ref, cand
    torch.cuda.empty_cache()
    want = O.check(rrecs, crecs, rh, ch, tol.responses, 3.0, "BF16")
    assert_reports_match(got, want, "config2 full size")
