"""estimate_tolerance on a real bf16 PyTorch model (GPU): the perturbation
proxy through td_perturb in a forward hook, traces captured in HBM by the
device-resident torchtap, responses reduced by td_segnorm."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu


class Block(torch.nn.Module):
    def __init__(self, d, h):
        super().__init__()
        self.norm = torch.nn.LayerNorm(d)
        self.qkv = torch.nn.Linear(d, 3 * d, bias=False)
        self.wo = torch.nn.Linear(d, d, bias=False)
        self.h = h

    def forward(self, x):
        s, d = x.shape
        q, k, v = self.qkv(self.norm(x)).view(s, 3, self.h, d // self.h).unbind(1)
        o = torch.nn.functional.scaled_dot_product_attention(
            q.transpose(0, 1), k.transpose(0, 1), v.transpose(0, 1), is_causal=True)
        return x + self.wo(o.transpose(0, 1).reshape(s, d))


class Mlp(torch.nn.Module):
    def __init__(self, d, ff):
        super().__init__()
        self.norm = torch.nn.LayerNorm(d)
        self.w1 = torch.nn.Linear(d, ff, bias=False)
        self.w2 = torch.nn.Linear(ff, d, bias=False)

    def forward(self, x):
        return x + self.w2(torch.nn.functional.gelu(self.w1(self.norm(x))))


class Tiny(torch.nn.Module):
    def __init__(self, vocab=256, d=64, h=4, ff=256, layers=4, seq=64):
        super().__init__()
        self.embedding = torch.nn.Embedding(vocab, d)
        self.pos = torch.nn.Parameter(torch.randn(seq, d) * 0.02)
        self.layers = torch.nn.ModuleList()
        for _ in range(layers):
            self.layers.append(Block(d, h))
            self.layers.append(Mlp(d, ff))
        self.final_norm = torch.nn.LayerNorm(d)
        self.head = torch.nn.Linear(d, vocab, bias=False)

    def forward(self, ids):
        x = self.embedding(ids) + self.pos
        for layer in self.layers:
            x = layer(x)
        return self.head(self.final_norm(x))


@pytest.fixture(scope="module")
def setup():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.manual_seed(0)
    model = Tiny().cuda().bfloat16()
    ids = torch.randint(0, 256, (64,), device="cuda")
    labels = torch.roll(ids, -1)

    def step(m):
        logits = m(ids)
        torch.nn.functional.cross_entropy(logits.float(), labels).backward()
    return model, step


def _runner(model, step, **kw):
    from paper_2506_09280_b200.runner import torch_runner
    from paper_2506_09280_b200.torchtap import TapConfig
    return torch_runner(model, step, embedding="embedding",
                        tap=TapConfig(patterns=("embedding", "layers.*", "final_norm", "head"),
                                      precision="bf16"), **kw)


def test_tolerance_estimate_on_torch_model(setup):
    import paper_2506_09280_b200 as td
    model, step = setup
    eps = td.FloatFormat.BF16.eps
    runner = _runner(model, step)
    tol = td.estimate_tolerance(runner, n_samples=3, eps_p=eps)
    again = td.estimate_tolerance(runner, n_samples=3, eps_p=eps)
    assert tol == again                                   # deterministic
    token_in = "iter=0|mb=0|kind=ActivationIn|mod=model.embedding"
    assert tol.responses[token_in] == 0.0                 # upstream of the perturbation
    acts = [v for k, v in tol.responses.items() if "kind=ActivationOut|mod=model.layers" in k]
    assert acts and all(0.01 * eps <= v <= 100 * eps for v in acts), acts
    assert all(v >= 0 and math.isfinite(v) for v in tol.responses.values())


def test_clean_rerun_passes_and_bug_is_flagged(setup):
    import paper_2506_09280_b200 as td
    model, step = setup
    eps = td.FloatFormat.BF16.eps
    runner = _runner(model, step)
    tol = td.estimate_tolerance(runner, n_samples=3, eps_p=eps)
    ref = runner(None)
    cand = runner(None)
    rep = td.check(ref, cand, tol, fmt=td.FloatFormat.BF16)
    assert rep.exit_code() == 0, rep.counts
    # silent bug: layer 3 (an Mlp) output scaled by 1.1
    hook = model.layers[3].register_forward_hook(lambda m, a, o: o * 1.1)
    try:
        bad = runner(None)
    finally:
        hook.remove()
    rep = td.check(ref, bad, tol, fmt=td.FloatFormat.BF16)
    assert rep.exit_code() == 2
    assert rep.earliest_flag == "iter=0|mb=0|kind=ActivationOut|mod=model.layers.3"


def test_module_wise_perturbation_hits_every_listed_input(setup):
    import paper_2506_09280_b200 as td
    model, step = setup
    names = tuple(f"layers.{i}" for i in range(8))
    runner = _runner(model, step, module_inputs=names)
    base, pert = runner(None), runner(td.PerturbSpec(0, td.FloatFormat.BF16.eps))
    assert pert.header["mode"] == "module-wise"
    moved = {r.id.encode() for r, s in zip(base.records, pert.records)
             if not torch.equal(r.payload, s.payload)}
    for i in range(8):
        assert f"iter=0|mb=0|kind=ActivationIn|mod=model.layers.{i}" in moved


def test_rewrite_mode_regenerates_inputs_and_localises_a_bug(setup):
    """Module-wise mode (engine.py:363-377): every listed module's input is
    regenerated from its id on the GPU, so a corrupted block flags at its own
    output while downstream blocks stay clean (test_checker.py:358-372)."""
    import paper_2506_09280_b200 as td
    model, step = setup
    names = tuple(f"layers.{i}" for i in range(8))
    runner = _runner(model, step, module_inputs=names, rewrite=True)
    eps = td.FloatFormat.BF16.eps
    tol = td.estimate_tolerance(runner, n_samples=3, eps_p=eps)
    ref = runner(None)
    again = runner(None)
    assert td.check(ref, again, tol, fmt=td.FloatFormat.BF16).exit_code() == 0
    hook = model.layers[2].register_forward_hook(lambda m, a, o: o * 1.1)
    try:
        bad = runner(None)
    finally:
        hook.remove()
    rep = td.check(ref, bad, tol, fmt=td.FloatFormat.BF16)
    flagged_fwd = {e.ident for e in rep.entries if e.verdict == "flag" and "kind=Activation" in e.ident
                   and "Grad" not in e.ident}
    assert flagged_fwd == {"iter=0|mb=0|kind=ActivationOut|mod=model.layers.2"}


@pytest.mark.parametrize("module_wise", [False, True])
def test_streaming_estimate_equals_materialised(setup, module_wise):
    """estimate_tolerance_streaming (captures compared as they are produced,
    nothing kept) gives the responses estimate_tolerance gives on the
    materialised traces."""
    import paper_2506_09280_b200 as td
    model, step = setup
    kw = {}
    if module_wise:
        kw = dict(module_inputs=tuple(f"layers.{i}" for i in range(8)), rewrite=True)
    runner = _runner(model, step, **kw)
    eps = td.FloatFormat.BF16.eps
    want = td.estimate_tolerance(runner, n_samples=3, eps_p=eps)
    got = td.estimate_tolerance_streaming(runner, n_samples=3, eps_p=eps)
    assert sorted(got.responses) == sorted(want.responses)
    assert any(v > 0 for v in want.responses.values())
    for k, v in want.responses.items():
        g = got.responses[k]
        assert (g == v) or abs(g - v) <= 1e-12 * max(abs(v), abs(g)), (k, g, v)
    mean = td.estimate_tolerance_streaming(runner, n_samples=2, eps_p=eps, aggregation="mean")
    assert mean.aggregation == "mean" and len(mean.responses) == len(want.responses)


def test_check_streaming_equals_check_of_the_materialised_trace(setup):
    """check_streaming (a live candidate step compared against the resident
    reference as its captures are produced) reports exactly what check()
    reports for the materialised candidate trace — with a silent bug in the
    candidate (one MLP's output scaled by 1.25) so flags appear."""
    import json

    import paper_2506_09280_b200 as td
    model, step = setup
    runner = _runner(model, step)
    ref = runner(None)
    eps = td.FloatFormat.BF16.eps
    tol = td.estimate_tolerance(runner, n_samples=2, eps_p=eps)
    bug = model.layers[3].register_forward_hook(lambda m, a, out: out * 1.25)
    try:
        cand = runner(None)
        want = td.check(ref, cand, tol, fmt=td.FloatFormat.BF16)
        got = td.check_streaming(ref, lambda sink: runner(None, sink=sink), tol, fmt=td.FloatFormat.BF16)
    finally:
        bug.remove()
    w, g = json.loads(td.render_report(want, "json")), json.loads(td.render_report(got, "json"))
    assert w["summary"]["flag"] > 0
    from tests.test_gpu_parity import assert_reports_match
    assert_reports_match(g, w, "check_streaming")


def test_check_streaming_missing_extra_and_shape_mismatch():
    """Ids on one side only are 'missing' (candidate order, then reference
    only), a capture whose shape differs from its reference record is a
    merge error with the reference's detail, NaN passes, +inf flags — the
    same report check() gives for the materialised candidate trace."""
    import json

    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200.canonical import identity_mapping, parse_canonical
    from paper_2506_09280_b200.tracestore import RankMeta, Trace, TraceRecord
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    g = torch.Generator(device="cuda").manual_seed(9)
    hdr = {"digest": "d", "mode": "cascade"}

    def ident(name):
        return f"iter=0|mb=0|kind=ActivationOut|mod=model.{name}"
    base = {n: torch.randn(shape, device="cuda", generator=g).to(torch.bfloat16)
            for n, shape in (("a", (64, 32)), ("b", (16,)), ("c", (8, 8)), ("only_ref", (4,)), ("nan", (5,)),
                             ("inf", (6,)))}
    base["inf"][0] = 0.0
    ref = Trace(header=dict(hdr))
    for n, t in base.items():
        ref.records.append(TraceRecord(parse_canonical(ident(n)), RankMeta(), identity_mapping(tuple(t.shape)), 1,
                                       t, "Linear"))
    cand_t = {"a": base["a"] * 1.001, "only_cand": torch.ones(3, device="cuda", dtype=torch.bfloat16),
              "b": base["b"] * 2, "c": torch.zeros(4, 16, device="cuda", dtype=torch.bfloat16),
              "nan": base["nan"].clone(), "inf": base["inf"].clone()}
    cand_t["nan"][1] = float("nan")
    cand_t["inf"][0] = float("inf")
    cand = Trace(header=dict(hdr))
    for n, t in cand_t.items():
        cand.records.append(TraceRecord(parse_canonical(ident(n)), RankMeta(), identity_mapping(tuple(t.shape)), 1,
                                        t, "Linear"))
    tol = td.ToleranceMap({ident("a"): 0.01}, n_samples=1, eps_p=2.0 ** -8)

    def run(sink):
        for n, t in cand_t.items():
            sink(ident(n), t, "Linear")
    got = json.loads(td.render_report(td.check_streaming(ref, run, tol, fmt=td.FloatFormat.BF16), "json"))
    want = json.loads(td.render_report(td.check(ref, cand, tol, fmt=td.FloatFormat.BF16), "json"))
    from tests.test_gpu_parity import assert_reports_match
    assert_reports_match(got, want, "streaming edge cases")
    verdicts = {e["id"].split("mod=model.")[1]: e["verdict"] for e in got["entries"]}
    assert verdicts == {"a": "pass", "only_cand": "missing", "b": "flag", "c": "merge-error", "nan": "pass",
                        "inf": "flag", "only_ref": "missing"}
