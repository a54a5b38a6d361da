"""The reference's acceptance criterion for the per-layer gradient trend
(test_acceptance.py:258-276: module-wise rewrite, n=5, Spearman(layer,
response) <= -0.5) on a real bf16 Llama-shaped PyTorch model run on the GPU,
with the materialised and the streaming estimator."""

import math
import os
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _spearman(ys):
    xs = list(range(len(ys)))

    def ranks(v):
        order = sorted(range(len(v)), key=lambda i: v[i])
        r = [0.0] * len(v)
        for k, i in enumerate(order):
            r[i] = float(k)
        return r
    rx, ry = ranks(xs), ranks(ys)
    mx, my = sum(rx) / len(rx), sum(ry) / len(ry)
    num = sum((a - mx) * (b - my) for a, b in zip(rx, ry))
    return num / math.sqrt(sum((a - mx) ** 2 for a in rx) * sum((b - my) ** 2 for b in ry))


@pytest.mark.parametrize("streaming", [False, True])
def test_gradient_response_decreases_with_layer(streaming):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import depth_sweep
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200.runner import torch_runner
    from paper_2506_09280_b200.torchtap import TapConfig
    layers, d, seq, vocab = 16, 128, 128, 512
    torch.manual_seed(0)
    torch.set_default_dtype(torch.bfloat16)
    with torch.device("cuda"):
        model = depth_sweep.build(layers, d, seq, vocab, kv=2, heads=4)
    torch.set_default_dtype(torch.float32)
    for name, p in model.named_parameters():
        if p.dim() > 1:   # the reference's init (model.py:82-106)
            torch.nn.init.normal_(p, 0.0, 0.02 / math.sqrt(2 * layers) if name.endswith(("wo.weight", "w2.weight"))
                                  else 0.02)
    ids = torch.randint(0, vocab, (seq,), device="cuda")
    labels = torch.roll(ids, -1)

    def step(m):
        torch.nn.functional.cross_entropy(m(ids).float(), labels).backward()
    runner = torch_runner(model, step, embedding="embedding",
                          tap=TapConfig(patterns=("layers.*",), precision="bf16"),
                          module_inputs=tuple(f"layers.{i}" for i in range(2 * layers)), rewrite=True)
    eps = td.FloatFormat.BF16.eps
    estimate = td.estimate_tolerance_streaming if streaming else td.estimate_tolerance
    tol = estimate(runner, n_samples=5, eps_p=eps)
    per_layer = []
    for layer in range(layers):
        tags = (f"|kind=ParamGrad|mod=model.layers.{2 * layer}.", f"|kind=ParamGrad|mod=model.layers.{2 * layer + 1}.")
        vals = [r for ident, r in tol.responses.items() if any(t in ident for t in tags)]
        per_layer.append(sum(vals) / len(vals))
    assert all(0.02 * eps <= r <= 100 * eps for r in per_layer), [r / eps for r in per_layer]
    assert _spearman(per_layer) <= -0.5, [r / eps for r in per_layer]


def test_static_thresholds_fail_where_calibrated_check_holds(cases, golden_trace_bytes):
    """The reference's Table-4 ablation criterion (test_acceptance.py:281-294)
    on the golden traces, with the B200 kernels: a tight fixed threshold
    cries wolf on a correct run, a loose one sleeps through a real bug
    (MC_SP_NORM_GRAD), the calibrated check does neither."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200.tracestore import trace_from_bytes

    def load(name):
        case = next(c for c in cases["checks"] if c["name"] == name)
        ref = trace_from_bytes(golden_trace_bytes(case["ref"]), device="cuda")
        cand = trace_from_bytes(golden_trace_bytes(case["cand"]), device="cuda")
        tol = td.ToleranceMap.from_json(cases["tols"][case["tol"]])
        return ref, cand, td.check(ref, cand, tol, case["kappa"], fmt=td.FloatFormat(case["fmt"]))
    ref, clean, clean_report = load("clean_tp2_cp2_k3")
    _, buggy, bug_report = load("bug_sp_norm_grad_k3")
    tight = td.compare_static(ref, clean, atol=0.0, rtol=1e-5)
    loose = td.compare_static(ref, buggy, atol=1e-2, rtol=1e-1)
    assert tight.counts["flag"] > 0
    assert loose.counts["flag"] == 0
    assert clean_report.exit_code() == 0 and bug_report.exit_code() != 0


def test_every_bug_flagged_with_separation_margin(cases, golden_trace_bytes):
    """The reference's criteria (test_acceptance.py:208-236) over the golden
    catalog runs, with the B200 kernels: every injected bug gates the check
    (exit code != 0), and the earliest divergence's observed rel_err is at
    least 10x its tolerance."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200.tracestore import trace_from_bytes
    bugs = [c for c in cases["checks"] if c["name"].startswith("bug_") and c["name"].endswith("_k3")]
    assert len(bugs) == 9
    ratios = {}
    for case in bugs:
        ref = trace_from_bytes(golden_trace_bytes(case["ref"]), device="cuda")
        cand = trace_from_bytes(golden_trace_bytes(case["cand"]), device="cuda")
        tol = td.ToleranceMap.from_json(cases["tols"][case["tol"]])
        fmt = td.FloatFormat(case["fmt"])
        rep = td.check(ref, cand, tol, case["kappa"], fmt=fmt)
        assert rep.exit_code() != 0, case["name"]
        entry = next(e for e in rep.entries if e.ident == rep.earliest_divergence)
        ratios[case["name"]] = entry.observed / max(entry.tolerance, fmt.eps)
    assert all(r >= 10.0 for r in ratios.values()), ratios
