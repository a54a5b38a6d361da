"""torchtap drop-in: byte-identical flushes against the reference adapter's
own output (golden), the reference adapter's behavioural contract, and (GPU)
device-resident captures feeding check() with no host round trip."""

import numpy as np
import pytest
import torch

from paper_2506_09280_b200 import torchtap
from paper_2506_09280_b200.torchtap import PatternUnmatched, TapConfig, TapError


def two_linear():
    torch.manual_seed(7)
    net = torch.nn.Sequential(torch.nn.Linear(8, 16, bias=False), torch.nn.Linear(16, 4, bias=False))
    return net, torch.randn(5, 8)


def run_step(net, x):
    net(x).square().sum().backward()


def test_flush_bytes_match_reference_adapter(torchtap_golden):
    net, x = two_linear()
    h = torchtap.attach(net, TapConfig(patterns=("*",)))
    run_step(net, x)
    assert [r.ident for r in h.records] == torchtap_golden["two_linear"]["idents"]
    assert torchtap.to_bytes(h).hex() == torchtap_golden["two_linear"]["bytes_hex"]
    torch.manual_seed(3)
    mlp = torch.nn.Sequential(torch.nn.LayerNorm(16), torch.nn.Linear(16, 32), torch.nn.GELU(),
                              torch.nn.Linear(32, 16))
    xb = torch.randn(4, 16)
    h = torchtap.attach(mlp, TapConfig(patterns=("*",), iteration=2, microbatch=1, precision="bf16"))
    mlp(xb).sum().backward()
    assert torchtap.to_bytes(h).hex() == torchtap_golden["layernorm_mlp"]["bytes_hex"]


def test_capture_order_and_values():
    net, x = two_linear()
    h = torchtap.attach(net, TapConfig(patterns=("*",)))
    run_step(net, x)
    assert [r.ident for r in h.records] == [
        "iter=0|mb=0|kind=ActivationIn|mod=model.0", "iter=0|mb=0|kind=ActivationOut|mod=model.0",
        "iter=0|mb=0|kind=ActivationIn|mod=model.1", "iter=0|mb=0|kind=ActivationOut|mod=model.1",
        "iter=0|mb=0|kind=ParamGrad|mod=model.1.weight", "iter=0|mb=0|kind=ParamGrad|mod=model.0.weight"]
    for r in h.records:
        if "ParamGrad" in r.ident:
            p = dict(net.named_parameters())[r.ident.split("|mod=model.")[1]]
            assert np.array_equal(r.host(), p.grad.float().numpy())


def test_contract_errors_detach_rename(tmp_path):
    net, x = two_linear()
    with pytest.raises(PatternUnmatched):
        torchtap.attach(net, TapConfig(patterns=()))
    with pytest.raises(PatternUnmatched, match="decoder"):
        torchtap.attach(net, TapConfig(patterns=("0", "decoder.*")))
    h = torchtap.attach(net, TapConfig(patterns=("*",)))
    run_step(net, x)
    with pytest.raises(TapError, match="second"):
        net(x)
    h.clear()
    run_step(net, x)
    assert torchtap.flush(h, tmp_path / "a") == 6
    assert (tmp_path / "a").read_bytes() == torchtap.to_bytes(h)
    torchtap.detach(h)
    n = len(h.records)
    run_step(net, x)
    assert len(h.records) == n
    h2 = torchtap.attach(net, TapConfig(patterns=("0",), rename=lambda n: f"model.layers.{n}.mlp"))
    with torch.no_grad():
        net(x)
    assert h2.records[0].ident.endswith("|mod=model.layers.0.mlp")


def test_trace_reads_back_through_the_drop_in_reader(tmp_path):
    from paper_2506_09280_b200.tracestore import read_trace
    net, x = two_linear()
    h = torchtap.attach(net, TapConfig(patterns=("*",)))
    run_step(net, x)
    torchtap.flush(h, tmp_path / "t")
    trace = read_trace(tmp_path / "t")
    assert [r.id.encode() for r in trace.records] == [r.ident for r in h.records]
    for ours, theirs in zip(h.records, trace.records):
        assert np.array_equal(theirs.payload, ours.host())


@pytest.mark.gpu
def test_device_resident_capture_feeds_check():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2506_09280_b200 as td
    torch.manual_seed(0)
    net = torch.nn.Sequential(torch.nn.Linear(64, 128), torch.nn.GELU(), torch.nn.Linear(128, 64)).cuda().bfloat16()
    x = torch.randn(32, 64, device="cuda", dtype=torch.bfloat16)
    ref_h = torchtap.attach(net, TapConfig(patterns=("*",), precision="bf16"))
    net(x).float().square().sum().backward()
    assert all(r.payload.is_cuda and r.payload.dtype == torch.bfloat16 for r in ref_h.records)
    ref = ref_h.trace()
    torchtap.detach(ref_h)
    net.zero_grad()
    cand_h = torchtap.attach(net, TapConfig(patterns=("*",), precision="bf16"))
    net(x).float().square().sum().backward()
    cand = cand_h.trace()
    tol = td.ToleranceMap({}, n_samples=1, eps_p=td.FloatFormat.BF16.eps)
    rep = td.check(ref, cand, tol, fmt=td.FloatFormat.BF16)
    assert rep.exit_code() == 0 and rep.counts["pass"] == len(ref.records)
    # a corrupted activation is flagged at its id
    bad = cand_h.trace()
    bad.records[2].payload.mul_(1.5)
    rep = td.check(ref, bad, tol, fmt=td.FloatFormat.BF16)
    assert rep.earliest_flag == bad.records[2].id.encode()
