"""GPU parity: the sm_100a path against the golden reference outputs and
the CPU oracle.  Norms agree within 1e-12 relative (fp64 accumulation in a
different order than numpy's pairwise sum); verdicts, details, witnesses,
quantised values and random streams agree exactly."""

import json
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import traindiff_oracle as O  # noqa: E402
import paper_2506_09280_b200 as td  # noqa: E402
from paper_2506_09280_b200.canonical import (CanonicalId, ShardMapping, SliceBox,  # noqa: E402
                                             TensorKind, identity_mapping)
from paper_2506_09280_b200.tracestore import RankMeta, Trace, TraceRecord, trace_from_bytes  # noqa: E402

pytestmark = pytest.mark.gpu
REL = 1e-12


@pytest.fixture(autouse=True, scope="module")
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _close(a, b, rel=REL):
    if a is None or b is None:
        return a is None and b is None
    if isinstance(a, str) or isinstance(b, str):
        return a == b
    if math.isnan(a) or math.isnan(b):
        return math.isnan(a) and math.isnan(b)
    if math.isinf(a) or math.isinf(b):
        return a == b
    return abs(a - b) <= rel * max(abs(a), abs(b)) or a == b


def assert_reports_match(got: dict, want: dict, label=""):
    assert got["summary"] == want["summary"], label
    assert got["earliest_flag"] == want["earliest_flag"], label
    assert got["earliest_divergence"] == want["earliest_divergence"], label
    assert got["exit_code"] == want["exit_code"], label
    assert got["mode"] == want["mode"] and got["format"] == want["format"], label
    assert len(got["entries"]) == len(want["entries"]), label
    for g, w in zip(got["entries"], want["entries"]):
        assert g["id"] == w["id"], label
        assert g["verdict"] == w["verdict"], (label, g["id"], g, w)
        assert g["detail"] == w["detail"], (label, g["id"])
        assert g["tolerance"] == w["tolerance"] and g["threshold"] == w["threshold"], (label, g["id"])
        assert _close(g["observed"], w["observed"]), (label, g["id"], g["observed"], w["observed"])


def _bf16_device(trace):
    """Same trace with payloads moved to HBM: bf16 where the values are on the
    bf16 grid (exact), f32 otherwise (e.g. the emulator's unrounded MainGrad)."""
    out = Trace(header=trace.header, raw_header=trace.raw_header)
    for r in trace.records:
        t = torch.from_numpy(np.asarray(r.values(), np.float32)).cuda()
        b = t.to(torch.bfloat16)
        payload = b if torch.equal(b.float(), t) else t
        out.records.append(TraceRecord(r.id, r.rank_meta, r.mapping, r.replica_group_size, payload,
                                       r.module_class))
    return out


@pytest.mark.parametrize("payloads", ["host-f32", "device-bf16"])
def test_check_reproduces_reference_reports(cases, golden_trace_bytes, payloads):
    near = 0
    for case in cases["checks"]:
        if payloads == "device-bf16" and case["fmt"] != "BF16":
            continue
        ref = trace_from_bytes(golden_trace_bytes(case["ref"]))
        cand = trace_from_bytes(golden_trace_bytes(case["cand"]))
        if payloads == "device-bf16":
            ref, cand = _bf16_device(ref), _bf16_device(cand)
        tol = td.ToleranceMap.from_json(cases["tols"][case["tol"]])
        rep = td.check(ref, cand, tol, case["kappa"], fmt=td.FloatFormat(case["fmt"]))
        near += rep.near_ties
        got = json.loads(td.render_report(rep, "json"))
        assert_reports_match(got, json.loads(case["report"]), case["name"])
    assert near == 0


@pytest.mark.parametrize("budget", [1 << 20, 64 << 10])
def test_check_in_batches_when_host_traces_exceed_the_device(monkeypatch, cases, golden_trace_bytes, budget):
    """Host traces larger than the device budget (forced small here) are
    checked in consecutive batches of ids: every golden scenario's report —
    order, verdicts, missing ids, earliest flag — is still the reference's."""
    from paper_2506_09280_b200 import checker
    calls = []
    real = checker._check_direct
    monkeypatch.setattr(checker, "_check_direct", lambda *a, **k: calls.append(1) or real(*a, **k))
    monkeypatch.setenv("TD_HBM_BUDGET_BYTES", str(budget))
    split = 0
    for case in cases["checks"]:
        ref = trace_from_bytes(golden_trace_bytes(case["ref"]))
        cand = trace_from_bytes(golden_trace_bytes(case["cand"]))
        tol = td.ToleranceMap.from_json(cases["tols"][case["tol"]])
        calls.clear()
        rep = td.check(ref, cand, tol, case["kappa"], fmt=td.FloatFormat(case["fmt"]))
        if checker._host_bytes(ref) + checker._host_bytes(cand) > budget:
            assert len(calls) > 1, case["name"]        # it did split
            split += 1
        assert_reports_match(json.loads(td.render_report(rep, "json")), json.loads(case["report"]), case["name"])
    assert split >= 10


def test_estimate_tolerance_reproduces_reference(cases, golden_trace_bytes):
    for est in cases["estimates"]:
        base = trace_from_bytes(golden_trace_bytes(est["base"]), device="cuda")
        pert = [trace_from_bytes(golden_trace_bytes(p), device="cuda") for p in est["perturbed"]]

        def runner(spec):
            return base if spec is None else pert[spec.sample]
        tol = td.estimate_tolerance(runner, n_samples=len(pert), eps_p=est["eps_p"],
                                    aggregation=est["aggregation"])
        want = json.loads(est["tol"])
        assert tol.n_samples == want["n_samples"] and tol.aggregation == want["aggregation"]
        assert sorted(tol.responses) == sorted(want["responses"])
        for k, v in want["responses"].items():
            assert _close(tol.responses[k], v), (est["name"], k)


def test_rel_err_vectors(vectors):
    for r in vectors["rel_err"]:
        a = np.array([float.fromhex(h) for h in r["a_hex"]])
        b = np.array([float.fromhex(h) for h in r["b_hex"]])
        assert _close(td.rel_err_arrays(a, b), float.fromhex(r["rel"]), 1e-15)
        # f32 carriers take the vector path
        assert _close(td.rel_err_arrays(a.astype(np.float32), b.astype(np.float32)),
                      float.fromhex(r["rel"]), 1e-15)


def test_rel_err_definition_cases():
    one = np.array([1.0, 1.0])
    assert td.rel_err_arrays(one, np.array([2.0, 2.0])) == 1.0
    assert td.rel_err_arrays(one, one) == 0.0
    assert td.rel_err_arrays(np.zeros(2), np.zeros(2)) == 0.0
    assert td.rel_err_arrays(np.zeros(2), one) == math.inf
    assert td.rel_err_arrays(one, np.zeros(2)) == 1.0
    assert math.isnan(td.rel_err_arrays(one, np.array([np.nan, 1.0])))
    with pytest.raises(td.ShapeMismatch):
        td.rel_err_arrays(np.zeros(2), np.zeros(3))
    assert td.frobenius_norm(td.Tensor(np.array([[3.0, 0.0], [0.0, 4.0]]))) == 5.0


def test_quantize_vectors_bit_exact(vectors):
    for fmt, v in vectors["quantize"].items():
        x = np.array([float.fromhex(h) for h in v["x_hex"]])
        y = td.quantize_array(x, td.FloatFormat(fmt))
        assert [float(a).hex() for a in y] == v["y_hex"], fmt
    with pytest.raises(td.NonFinite):
        td.quantize_array(np.array([1.0, np.nan]), td.FloatFormat.BF16)
    assert td.quantize_array(np.array(0.2), td.FloatFormat.BF16) == 0.2001953125
    assert td.quantize_array(np.array(257.0), td.FloatFormat.BF16) == 256.0


def test_signed_uniforms_bit_exact(vectors):
    for u in vectors["signed_uniforms"]:
        got = td.signed_uniforms(u["tag"], (u["n"],))
        assert [float(x).hex() for x in got] == u["values_hex"]
    from paper_2506_09280_b200.generation import signed_uniforms_device, seed_from
    tag = "perturb|s=0|iter=0|mb=0|kind=ActivationOut|mod=model.embedding"
    window = signed_uniforms_device(tag, 1000, k0=123_456_789).cpu().numpy()
    assert np.array_equal(window, O.signed_uniforms(seed_from(tag), 1000, 123_456_789))
    ph = signed_uniforms_device(tag, 5000, k0=(1 << 33) - 7, generator="philox").cpu().numpy()
    assert np.array_equal(ph, O.signed_uniforms(seed_from(tag), 5000, (1 << 33) - 7, "philox"))


@pytest.mark.parametrize("dtype", ["f64", "bf16"])
def test_perturbation_bit_exact(vectors, dtype):
    for p in vectors["perturb"]:
        x = np.array([float.fromhex(h) for h in p["x_hex"]]).reshape(p["rows"], p["cols"])
        want = np.array([float.fromhex(h) for h in p["y_hex"]]).reshape(x.shape)
        ident = p["tag"].split("|", 2)[2]
        sample = int(p["tag"].split("|")[1][2:])
        spec = td.PerturbSpec(sample, p["eps"])
        policy = "bf16" if p["fmt"] == "BF16" else "fp32"
        if dtype == "f64":
            y = td.apply_perturbation(torch.from_numpy(x).cuda(), ident, spec, policy=policy,
                                      row_positions=p["pos"])
            assert np.array_equal(y.cpu().numpy(), want), (p["eps"], p["fmt"])
        elif p["fmt"] == "BF16":
            xb = torch.from_numpy(x).cuda().to(torch.bfloat16)
            y = td.apply_perturbation(xb, ident, spec, policy=policy, row_positions=p["pos"])
            # Q_bf16 values above 2^-126 are exactly representable in bf16
            assert np.array_equal(y.double().cpu().numpy(), want)


def test_perturbation_rank_slices_compose():
    """Counter-based stream: each CP rank's rows equal the slice of the full
    perturbation (engine.py:351-361, test_engine.py:443-450)."""
    g = torch.Generator().manual_seed(0)
    full = torch.randn(64, 96, generator=g, dtype=torch.float64).cuda()
    spec = td.PerturbSpec(4, 2.0 ** -8)
    ident = "iter=0|mb=2|kind=ActivationOut|mod=model.embedding"
    whole = td.apply_perturbation(full, ident, spec, policy="bf16")
    rows = [5, 6, 7, 56, 57, 58]
    part = td.apply_perturbation(full[rows].contiguous(), ident, spec, policy="bf16", row_positions=rows)
    assert torch.equal(part, whole[rows])
    assert td.apply_perturbation(full, ident, td.PerturbSpec(0, 0.0)) is full


def _random_trace_pair(rng, case, dtype, corrupt):
    shape = tuple(case["shape"])
    x = rng.standard_normal(shape).astype(np.float32)
    if dtype == "bf16":
        x = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
    ident = CanonicalId(0, 0, TensorKind.ACTIVATION_OUT, "model.layers.0.attn")
    hdr = {"digest": "d", "mode": "cascade"}
    ref = Trace(hdr, [TraceRecord(ident, RankMeta(), identity_mapping(shape), 1, x, "Block")])
    recs = []
    copies = int(rng.integers(1, 4))
    for k, s in enumerate(case["shards"]):
        pairs = tuple((SliceBox(tuple(map(tuple, l))), SliceBox(tuple(map(tuple, g))))
                      for l, g in s["pairs"])
        m = ShardMapping(tuple(s["local_shape"]), shape, pairs)
        payload = np.empty(m.local_shape, np.float32)
        for l, g in pairs:
            payload[l.as_slices()] = x[g.as_slices()]
        for c in range(copies):
            p = payload.copy()
            if corrupt == "value" and k == 0 and c == 0 and p.size:
                p.reshape(-1)[0] += 1.0
            if corrupt == "replica" and k == 0 and c == copies - 1 and copies > 1 and p.size:
                p.reshape(-1)[-1] *= 3.0
            recs.append(TraceRecord(ident, RankMeta(tp=k, dp=c), m, copies, p, "Block"))
    return ref, Trace(hdr, recs)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_randomized_shardings_match_oracle(shardings, dtype):
    # all 1000 randomized shardings of the reference's acceptance test
    # (test_acceptance.py:90-112) x {none, value, replica} corruptions
    rng = np.random.default_rng(11)
    for i, case in enumerate(shardings):
        corrupt = ("none", "value", "replica")[i % 3]
        ref, cand = _random_trace_pair(rng, case, dtype, corrupt)
        if dtype == "bf16":
            ref, cand = _bf16_device(ref), _bf16_device(cand)
        tol = td.ToleranceMap({}, n_samples=1, eps_p=0.0)
        rep = td.check(ref, cand, tol, fmt=td.FloatFormat.BF16)
        oref = [O.Rec(r.id.encode(), r.rank_meta.as_tuple(), r.mapping.local_shape,
                      r.mapping.global_shape, [(l.bounds, g.bounds) for l, g in r.mapping.pairs],
                      r.replica_group_size, np.asarray(r.values(), np.float32)) for r in ref.records]
        ocand = [O.Rec(r.id.encode(), r.rank_meta.as_tuple(), r.mapping.local_shape,
                       r.mapping.global_shape, [(l.bounds, g.bounds) for l, g in r.mapping.pairs],
                       r.replica_group_size, np.asarray(r.values(), np.float32)) for r in cand.records]
        want = O.check(oref, ocand, ref.header, cand.header, {}, 3.0, "BF16")
        assert_reports_match(json.loads(td.render_report(rep, "json")), want, f"case {i}")


def test_merge_and_check_replicas_api():
    full = np.arange(12.0).reshape(3, 4)
    left = ShardMapping((3, 2), (3, 4), ((td.whole_box((3, 2)), SliceBox(((0, 3), (0, 2)))),))
    right = ShardMapping((3, 2), (3, 4), ((td.whole_box((3, 2)), SliceBox(((0, 3), (2, 4)))),))
    out = td.merge([(left, td.Tensor(full[:, :2])), (right, td.Tensor(full[:, 2:]))], (3, 4))
    assert np.array_equal(out.data, full)
    with pytest.raises(td.MergeConflict) as info:
        td.merge([(left, td.Tensor(full[:, :2]))], (3, 4))
    assert info.value.witness == (0, 2)
    a, b = td.Tensor(np.array([1.0, 1.0])), td.Tensor(np.array([2.0, 2.0]))
    with pytest.raises(td.ReplicaMismatch) as rinfo:
        td.check_replicas([a, b], td.ReplicaGroup((0, 1)), td.FloatFormat.BF16)
    assert rinfo.value.max_rel_err == 1.0 and rinfo.value.witness == (0, 1)
    c = td.Tensor(np.array([1.0 + 2.0 ** -10, 1.0]))
    td.check_replicas([a, c], td.ReplicaGroup((0, 1)), td.FloatFormat.BF16)
    with pytest.raises(td.ReplicaMismatch):
        td.check_replicas([a, c], td.ReplicaGroup((0, 1)), td.FloatFormat.FP32)
    many = [a] * 9 + [b]
    with pytest.raises(td.ReplicaMismatch) as minfo:
        td.check_replicas(many, td.ReplicaGroup(tuple(range(10))), td.FloatFormat.BF16)
    assert minfo.value.witness == (0, 9)


def test_compare_static_matches_oracle(cases, golden_trace_bytes):
    case = next(c for c in cases["checks"] if c["name"] == "clean_tp2_cp2_k3")
    ref = trace_from_bytes(golden_trace_bytes(case["ref"]))
    cand = trace_from_bytes(golden_trace_bytes(case["cand"]))
    _, rr = O.read_ttrc(golden_trace_bytes(case["ref"]))
    _, cr = O.read_ttrc(golden_trace_bytes(case["cand"]))
    for atol, rtol in ((0.0, 1e-5), (1e-2, 1e-1), (0.0, 0.0), (10.0, 10.0)):
        rep = td.compare_static(ref, cand, atol, rtol)
        want = O.compare_static(rr, cr, atol, rtol)
        assert [(e.ident, e.verdict) for e in rep.entries] == want, (atol, rtol)


@pytest.mark.parametrize("mib", [1, 64, 1024])
def test_large_tensor_norms_against_torch_fp64(mib):
    """Config-5 sizes: TP=4 column shards of a (N/4096, 4096) bf16 tensor vs
    an identity reference; norms against a torch fp64 reduction."""
    cols = 4096
    rows = mib * (1 << 20) // 2 // cols
    g = torch.Generator(device="cuda").manual_seed(mib)
    ref = torch.randn(rows, cols, device="cuda", generator=g).to(torch.bfloat16)
    noise = (torch.randn(rows, cols, device="cuda", generator=g) * 1e-2).to(torch.bfloat16)
    cand_full = (ref.float() + noise.float()).to(torch.bfloat16)
    ident = CanonicalId(0, 0, TensorKind.ACTIVATION_OUT, "model.lm_head")
    hdr = {"digest": "d", "mode": "cascade"}
    rt = Trace(hdr, [TraceRecord(ident, RankMeta(), identity_mapping((rows, cols)), 1, ref, "H")])
    ct = Trace(hdr, [])
    w = cols // 4
    for t in range(4):
        m = ShardMapping((rows, w), (rows, cols), ((td.whole_box((rows, w)),
                                                    SliceBox(((0, rows), (t * w, (t + 1) * w)))),))
        ct.records.append(TraceRecord(ident, RankMeta(tp=t), m, 1,
                                      cand_full[:, t * w:(t + 1) * w].contiguous(), "H"))
    rep = td.check(rt, ct, td.ToleranceMap({}, n_samples=1, eps_p=0.0), fmt=td.FloatFormat.BF16)
    r64, c64 = ref.double(), cand_full.double()
    want = math.sqrt(float(((r64 - c64) ** 2).sum())) / math.sqrt(float((r64 ** 2).sum()))
    assert _close(rep.entries[0].observed, want, 1e-12)
    # identity property: a trace against itself is exactly 0
    same = td.check(rt, rt, td.ToleranceMap({}, n_samples=1, eps_p=0.0), fmt=td.FloatFormat.BF16)
    assert same.entries[0].observed == 0.0 and same.entries[0].verdict == "pass"


def test_device_ttrc_reader_matches_host_reader(tmp_path, cases, golden_trace_bytes):
    """read_trace(device="cuda"): one DMA of the file image + td_gather_bytes
    unpacking every (unaligned) payload into an aligned HBM arena."""
    from paper_2506_09280_b200.tracestore import read_trace, trace_to_bytes
    for name in cases["traces"][:6]:
        raw = golden_trace_bytes(name)
        path = tmp_path / (name + ".ttrc")
        path.write_bytes(raw)
        host = trace_from_bytes(raw)
        dev = read_trace(path, device="cuda")
        assert len(dev.records) == len(host.records)
        for a, b in zip(dev.records, host.records):
            assert a.payload.is_cuda and a.payload.data_ptr() % 256 == 0
            assert np.array_equal(a.payload.cpu().numpy(), b.payload)
            assert a.mapping.signature() == b.mapping.signature()
        assert trace_to_bytes(dev) == raw


def test_cli_check_reproduces_reference_output(tmp_path, cases, golden_trace_bytes, capsys):
    """`check` front end: same stdout (text and JSON modulo last-bit norms)
    and the same exit code as the reference CLI (cli.py:100-111, 276-293)."""
    from paper_2506_09280_b200.cli import main
    for case in cases["checks"][:8]:
        ref, cand, tolp = tmp_path / "r.ttrc", tmp_path / "c.ttrc", tmp_path / "t.json"
        ref.write_bytes(golden_trace_bytes(case["ref"]))
        cand.write_bytes(golden_trace_bytes(case["cand"]))
        tolp.write_text(cases["tols"][case["tol"]])
        rc = main(["check", "--ref", str(ref), "--cand", str(cand), "--tol", str(tolp),
                   "--k", str(case["kappa"])])
        out = capsys.readouterr().out
        want = json.loads(case["report"])
        assert rc == want["exit_code"], case["name"]
        assert out == case["text"], case["name"]
    rc = main(["check", "--ref", str(tmp_path / "missing"), "--cand", str(cand), "--tol", str(tolp)])
    assert rc == 1
    (tmp_path / "bad").write_bytes(b"XXXX" + b"\0" * 16)
    assert main(["check", "--ref", str(tmp_path / "bad"), "--cand", str(cand), "--tol", str(tolp)]) == 4


def test_generate_full_matches_reference(vectors):
    """generate_full on the device: uniform and token streams bit-exact,
    Box-Muller normals within 1e-15 relative (the reference's own bar,
    test_generation.py:59-63)."""
    from paper_2506_09280_b200.canonical import parse_canonical
    from paper_2506_09280_b200.generation import (GenSpec, Normal, TokenIds, Uniform,
                                                  extract_shard, generate_full)
    exact = total = 0
    for g in vectors["generate_full"]:
        want = np.array([float.fromhex(h) for h in g["values_hex"]]).reshape(g["shape"])
        if g["kind"] == "normal":
            spec = GenSpec(Normal(*g["params"]), g["shape"])
        elif g["kind"] == "uniform":
            spec = GenSpec(Uniform(*g["params"]), g["shape"])
        else:
            spec = GenSpec(TokenIds(*g["params"]), g["shape"])
        got = generate_full(parse_canonical(g["ident"]), spec).data
        if g["kind"] == "normal":
            assert np.allclose(got, want, rtol=1e-15, atol=0.0)
            exact += int((got == want).sum())
            total += got.size
        else:
            assert np.array_equal(got, want), g["kind"]
    assert exact / total > 0.5          # most normals are bit-identical too
    full = generate_full(parse_canonical(vectors["generate_full"][0]["ident"]),
                         GenSpec(Normal(0.0, 0.02), (64, 32)), device="cuda")
    m = td.ShardMapping((32, 32), (64, 32), ((td.whole_box((32, 32)), td.SliceBox(((32, 64), (0, 32)))),))
    assert torch.equal(extract_shard(full, m), full[32:])


def test_reports_are_byte_deterministic(cases, golden_trace_bytes):
    """Fixed-order reductions: repeating check() reproduces the report bytes
    (the reference's CLI determinism contract, test_cli.py:55-67)."""
    case = next(c for c in cases["checks"] if c["name"] == "bug_tp_row_allreduce_k3")
    ref = trace_from_bytes(golden_trace_bytes(case["ref"]), device="cuda")
    cand = trace_from_bytes(golden_trace_bytes(case["cand"]), device="cuda")
    tol = td.ToleranceMap.from_json(cases["tols"][case["tol"]])
    a = td.render_report(td.check(ref, cand, tol, fmt=td.FloatFormat.BF16), "json")
    b = td.render_report(td.check(ref, cand, tol, fmt=td.FloatFormat.BF16), "json")
    assert a == b


def test_perturbation_full_exponent_range_bit_exact():
    """bf16 in/out fast path (integer RNE on the fp64 bits) against the
    oracle's quantize_array semantics over the whole bf16 exponent range,
    zeros and values that round up into / clamp at bf16 max."""
    rng = np.random.default_rng(5)
    n = 1 << 16
    mant = rng.integers(0, 128, n)
    expo = rng.integers(-125, 128, n)
    sign = rng.choice([-1.0, 1.0], n)
    x = sign * (1 + mant / 128.0) * np.exp2(expo)
    x[:64] = 0.0
    x[64:128] = -0.0
    x[128:192] = 1.9921875 * 2.0 ** 127
    xb = torch.from_numpy(x).to(torch.bfloat16)
    assert np.array_equal(xb.double().numpy(), x)       # all on the bf16 grid
    ident = "iter=0|mb=0|kind=ActivationOut|mod=model.embedding"
    for eps in (2.0 ** -8, 1e-3, 0.3):
        spec = td.PerturbSpec(7, eps)
        y = td.apply_perturbation(xb.cuda().reshape(256, 256), ident, spec, policy="bf16")
        want = O.perturb(x.reshape(256, 256), "perturb|s=7|" + ident, eps, np.arange(256), 256, "BF16")
        got = y.double().cpu().numpy()
        normal = np.abs(want) >= 2.0 ** -126
        assert np.array_equal(got[normal], want[normal]), eps
        assert np.array_equal(np.signbit(got[want == 0]), np.signbit(want[want == 0]))
    # philox stream on the same fast path
    y = td.apply_perturbation(xb.cuda().reshape(256, 256), ident, td.PerturbSpec(1, 2.0 ** -8),
                              policy="bf16", generator="philox")
    want = O.perturb(x.reshape(256, 256), "perturb|s=1|" + ident, 2.0 ** -8, np.arange(256), 256, "BF16",
                     generator="philox")
    normal = np.abs(want) >= 2.0 ** -126
    assert np.array_equal(y.double().cpu().numpy()[normal], want[normal])


@pytest.mark.parametrize("generator", ["splitmix64", "philox"])
def test_perturbation_column_shards_compose(generator):
    """A TP column shard perturbed with its column offset (odd offsets and an
    odd full width, so words start mid Philox block) equals the same columns
    of the whole-tensor perturbation, on the bf16 fast path."""
    full_cols, rows = 8 * 37 + 3, 64
    x = torch.randn(rows, full_cols, dtype=torch.float64).to(torch.bfloat16)
    ident = "iter=0|mb=0|kind=ActivationIn|mod=model.layers.3.mlp"
    spec = td.PerturbSpec(2, 2.0 ** -8)
    whole = td.apply_perturbation(x.cuda(), ident, spec, policy="bf16", generator=generator)
    want = O.perturb(x.double().numpy(), f"perturb|s=2|{ident}", 2.0 ** -8, np.arange(rows), full_cols,
                     "BF16", generator=generator)
    assert np.array_equal(whole.double().cpu().numpy(), want)
    for col0 in (1, 3, 8, 131):
        part = x[:, col0:col0 + 64].contiguous().cuda()
        got = td.apply_perturbation(part, ident, spec, policy="bf16", full_cols=full_cols, col0=col0,
                                    generator=generator)
        assert torch.equal(got, whole[:, col0:col0 + 64]), col0


def test_graph_replay_matches_eager_launch(cases, golden_trace_bytes):
    """A captured CUDA graph of the whole check replays to the same results
    and follows payload updates made in place."""
    from paper_2506_09280_b200.checker import CheckPlan
    from paper_2506_09280_b200.device import resolve_operands
    case = next(c for c in cases["checks"] if c["name"] == "bug_tp_row_allreduce_k3")
    ref = trace_from_bytes(golden_trace_bytes(case["ref"]), device="cuda")
    cand = trace_from_bytes(golden_trace_bytes(case["cand"]), device="cuda")
    tol = td.ToleranceMap.from_json(cases["tols"][case["tol"]])
    cp = CheckPlan(ref, cand, tol, fmt=td.FloatFormat.BF16)
    ptrs, keep = resolve_operands(cp.plan.operands, cp.plan.operand_dtypes)
    prep = cp.plan.prepare(ptrs, kappa=3.0, eps=td.FloatFormat.BF16.eps, replica_eps=td.FloatFormat.BF16.eps)
    prep.launch()
    eager = prep.fetch()
    graph = prep.capture()
    graph.replay()
    replay = prep.fetch()
    assert np.array_equal(eager[0], replay[0]) and np.array_equal(eager[1], replay[1])
    keep[0].mul_(2.0)                       # operand 0 changes in place
    graph.replay()
    moved = prep.fetch()
    prep.launch()
    assert np.array_equal(moved[0], prep.fetch()[0])


@pytest.mark.parametrize("chunk_rows", [5, 64])
def test_two_level_slot_reduction_matches_oracle(monkeypatch, cases, golden_trace_bytes, shardings, chunk_rows):
    """Force td_reduce_chunks (plan.Plan._chunk_slots) on every plan, with
    chunk sizes that do and do not align with tiles."""
    from paper_2506_09280_b200.plan import Plan
    monkeypatch.setattr(Plan, "CHUNK_MIN_ROWS", 0)
    monkeypatch.setattr(Plan, "CHUNK_ROWS", chunk_rows)
    for case in cases["checks"]:
        ref = trace_from_bytes(golden_trace_bytes(case["ref"]))
        cand = trace_from_bytes(golden_trace_bytes(case["cand"]))
        tol = td.ToleranceMap.from_json(cases["tols"][case["tol"]])
        rep = td.check(ref, cand, tol, case["kappa"], fmt=td.FloatFormat(case["fmt"]))
        assert_reports_match(json.loads(td.render_report(rep, "json")), json.loads(case["report"]), case["name"])
    rng = np.random.default_rng(5)
    for i, case in enumerate(shardings[:60]):
        ref, cand = _random_trace_pair(rng, case, "f32", ("none", "value", "replica")[i % 3])
        rep = td.check(ref, cand, td.ToleranceMap({}, n_samples=1, eps_p=0.0), fmt=td.FloatFormat.BF16)
        oref = [O.Rec(r.id.encode(), r.rank_meta.as_tuple(), r.mapping.local_shape,
                      r.mapping.global_shape, [(l.bounds, g.bounds) for l, g in r.mapping.pairs],
                      r.replica_group_size, np.asarray(r.values(), np.float32)) for r in ref.records]
        ocand = [O.Rec(r.id.encode(), r.rank_meta.as_tuple(), r.mapping.local_shape,
                       r.mapping.global_shape, [(l.bounds, g.bounds) for l, g in r.mapping.pairs],
                       r.replica_group_size, np.asarray(r.values(), np.float32)) for r in cand.records]
        want = O.check(oref, ocand, ref.header, cand.header, {}, 3.0, "BF16")
        assert_reports_match(json.loads(td.render_report(rep, "json")), want, f"chunked case {i}")


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16, torch.float32, torch.float64])
def test_rel_err_one_launch_vs_fp64(dtype):
    """td_rel_err (the same-dtype fast path of rel_err_arrays): aligned and
    misaligned views, lengths that are not a multiple of the vector, sizes
    from 1 element to beyond one grid stride, against a torch fp64 reduction;
    repeated calls are bit-identical."""
    g = torch.Generator(device="cuda").manual_seed(11)
    for n in (1, 7, 8, 1000, 4096 + 3, (1 << 20) + 5, (1 << 24) + 9):
        base = torch.randn(n + 1, device="cuda", generator=g, dtype=torch.float64)
        a = base.to(dtype)
        b = (base * (1 + 0.01 * torch.randn(n + 1, device="cuda", generator=g, dtype=torch.float64))).to(dtype)
        for off in (0, 1):
            x, y = a[off:off + n], b[off:off + n]
            want = float(torch.linalg.vector_norm(x.double() - y.double()) / torch.linalg.vector_norm(x.double()))
            got = td.rel_err_arrays(x, y)
            assert abs(got - want) <= 1e-12 * want, (dtype, n, off, got, want)
            assert td.rel_err_arrays(x, y) == got
    z = torch.zeros(100, device="cuda", dtype=dtype)
    o = torch.ones(100, device="cuda", dtype=dtype)
    assert td.rel_err_arrays(z, z) == 0.0
    assert td.rel_err_arrays(z, o) == math.inf
    assert td.rel_err_arrays(o, z) == 1.0
    nan = o.clone()
    nan[3] = float("nan")
    assert math.isnan(td.rel_err_arrays(o, nan))


def test_check_plan_cache_same_layout(cases, golden_trace_bytes):
    """check() reuses the plan of an earlier check of the same layout and
    binds the new payloads by position: the report equals a fresh plan's;
    a different tolerance map or kappa is a different plan."""
    from paper_2506_09280_b200 import checker
    case = next(c for c in cases["checks"] if c["name"] == "bug_tp_row_allreduce_k3")
    ref = trace_from_bytes(golden_trace_bytes(case["ref"]), device="cuda")
    cand = trace_from_bytes(golden_trace_bytes(case["cand"]), device="cuda")
    tol = td.ToleranceMap.from_json(cases["tols"][case["tol"]])
    fmt = td.FloatFormat(case["fmt"])
    checker._PLAN_CACHE.clear()
    first = td.render_report(td.check(ref, cand, tol, case["kappa"], fmt=fmt), "json")
    assert len(checker._PLAN_CACHE) == 1
    # same layout, other values: every candidate payload scaled
    cand2 = Trace(header=cand.header, raw_header=cand.raw_header)
    cand2.records = [TraceRecord(r.id, r.rank_meta, r.mapping, r.replica_group_size, r.payload * 1.5,
                                 r.module_class) for r in cand.records]
    hit = td.render_report(td.check(ref, cand2, tol, case["kappa"], fmt=fmt), "json")
    assert len(checker._PLAN_CACHE) == 1
    checker._PLAN_CACHE.clear()
    fresh = td.render_report(td.check(ref, cand2, tol, case["kappa"], fmt=fmt), "json")
    assert hit == fresh and hit != first
    td.check(ref, cand, tol, case["kappa"] * 2, fmt=fmt)
    assert len(checker._PLAN_CACHE) == 2


def test_odd_length_flat_runs_take_the_vector_walker():
    """A tensor whose element count is not a multiple of 8 (GPT-2's 50257
    vocabulary) streams through the vector walker with a < 8-cell generic
    tail; the result equals a torch fp64 reduction."""
    from paper_2506_09280_b200 import _native as N
    from paper_2506_09280_b200.checker import CheckPlan
    g = torch.Generator(device="cuda").manual_seed(4)
    x = torch.randn(1023, 50257, device="cuda", generator=g).to(torch.bfloat16)
    y = (x.double() * (1 + 2.0 ** -6 * torch.randn(x.shape, device="cuda", generator=g,
                                                   dtype=torch.float64))).to(torch.bfloat16)
    ident = CanonicalId(0, 0, TensorKind.ACTIVATION_OUT, "model.lm_head")
    ref = Trace(header={"digest": "d", "mode": "cascade"})
    cand = Trace(header={"digest": "d", "mode": "cascade"})
    ref.records.append(TraceRecord(ident, RankMeta(), identity_mapping(tuple(x.shape)), 1, x, "Linear"))
    cand.records.append(TraceRecord(ident, RankMeta(), identity_mapping(tuple(y.shape)), 1, y, "Linear"))
    tol = td.ToleranceMap({ident.encode(): 1.0}, n_samples=1, eps_p=2.0 ** -8)
    cp = CheckPlan(ref, cand, tol, fmt=td.FloatFormat.BF16)
    vec = (cp.plan.segs["flags"] & N.SEG_VEC) != 0
    cells = cp.plan.segs["rows"] * cp.plan.segs["cols"]
    assert cells[vec].sum() >= x.numel() - 7 and cells[~vec].sum() <= 7
    rep = td.check(ref, cand, tol, fmt=td.FloatFormat.BF16)
    want = float(torch.linalg.vector_norm(x.double() - y.double()) / torch.linalg.vector_norm(x.double()))
    assert abs(rep.entries[0].observed - want) <= 1e-12 * want


def test_rel_err_empty_and_scalar():
    """0/0 -> 0 for empty arrays (tensor.py:163-167), 0-d arrays compare."""
    e = torch.zeros(0, device="cuda", dtype=torch.bfloat16)
    assert td.rel_err_arrays(e, e) == 0.0
    assert td.rel_err_arrays(np.zeros(0), np.zeros(0)) == 0.0
    assert td.rel_err_arrays(np.array(2.0), np.array(3.0)) == 0.5


def test_check_plan_cache_with_pinned_host_payloads(cases, golden_trace_bytes):
    """The e2e path: traces in pinned host arenas, the plan cached by the
    first check and reused with the next check's staged copies."""
    from paper_2506_09280_b200 import checker
    from paper_2506_09280_b200.tracestore import pack_pinned
    case = next(c for c in cases["checks"] if c["name"] == "bug_stale_input_k3")
    ref = pack_pinned(trace_from_bytes(golden_trace_bytes(case["ref"])))
    cand = pack_pinned(trace_from_bytes(golden_trace_bytes(case["cand"])))
    tol = td.ToleranceMap.from_json(cases["tols"][case["tol"]])
    fmt = td.FloatFormat(case["fmt"])
    checker._PLAN_CACHE.clear()
    reports = [json.loads(td.render_report(td.check(ref, cand, tol, case["kappa"], fmt=fmt), "json"))
               for _ in range(3)]
    assert len(checker._PLAN_CACHE) == 1
    for rep in reports:
        assert_reports_match(rep, json.loads(case["report"]), "pinned + cached plan")


def test_fuzzed_perturbations_bit_exact():
    """A slice of tools/fuzz_perturb.py: random shapes, column shards with
    odd offsets, row subsets, eps, policies, in/out dtypes and generators —
    td_perturb bit-identical to the oracle."""
    import os
    import random
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import fuzz_perturb
    rnd = random.Random(5)
    for k in range(100):
        fuzz_perturb.run_case(rnd, k)


def test_pageable_host_payloads_through_the_staging_ring():
    """numpy (and pageable torch CPU) payloads above the staging threshold
    cross PCIe through the pinned ring: odd sizes, payloads straddling
    staging buffers, mixed f32 / bf16 / f64 — the report equals the one for
    device-resident copies of the same traces."""
    from paper_2506_09280_b200 import device
    g = np.random.default_rng(21)
    hdr = {"digest": "d", "mode": "cascade"}
    ref, cand, ref_d, cand_d = (Trace(header=dict(hdr)) for _ in range(4))
    shapes = [(4099, 1531), (7,), (3, 5, 7), (1 << 21,), (65537, 33), (12345, 1)]
    for k, shape in enumerate(shapes):
        ident = CanonicalId(0, 0, TensorKind.ACTIVATION_OUT, f"model.m{k}")
        x = g.standard_normal(shape).astype(np.float32)
        y = (x * (1 + 1e-3 * g.standard_normal(shape))).astype(np.float32)
        if k % 3 == 1:
            y_host = torch.from_numpy(y).to(torch.bfloat16)          # pageable torch CPU bf16
        elif k % 3 == 2:
            y_host = y.astype(np.float64)
        else:
            y_host = y
        m = identity_mapping(shape)
        ref.records.append(TraceRecord(ident, RankMeta(), m, 1, x, "Linear"))
        cand.records.append(TraceRecord(ident, RankMeta(), m, 1, y_host, "Linear"))
        ref_d.records.append(TraceRecord(ident, RankMeta(), m, 1, torch.from_numpy(x).cuda(), "Linear"))
        yd = y_host if isinstance(y_host, torch.Tensor) else torch.from_numpy(np.asarray(y_host, np.float32))
        cand_d.records.append(TraceRecord(ident, RankMeta(), m, 1, yd.cuda(), "Linear"))
    assert sum(r.nbytes for r in ref.records) + sum(r.nbytes for r in cand.records) > device._STAGE_MIN
    tol = td.ToleranceMap({}, n_samples=1, eps_p=0.0)
    got = json.loads(td.render_report(td.check(ref, cand, tol, fmt=td.FloatFormat.FP32), "json"))
    want = json.loads(td.render_report(td.check(ref_d, cand_d, tol, fmt=td.FloatFormat.FP32), "json"))
    assert_reports_match(got, want, "staging ring")


def test_read_trace_host_payloads_move_as_pinned_images(cases, golden_trace_bytes, tmp_path, monkeypatch):
    """read_trace(pin=True) on the host returns numpy payloads viewing a
    page-locked file image; check() moves each image with one DMA (no
    staging copies) and the report equals the reference's (and equals the
    default, unpinned read's)."""
    from paper_2506_09280_b200 import device
    case = next(c for c in cases["checks"] if c["name"] == "bug_stale_input_k3")
    paths = {}
    for side in ("ref", "cand"):
        paths[side] = tmp_path / f"{side}.ttrc"
        paths[side].write_bytes(golden_trace_bytes(case[side]))
    ref, cand = td.read_trace(paths["ref"], pin=True), td.read_trace(paths["cand"], pin=True)
    assert all(isinstance(r.payload, np.ndarray) for r in ref.records + cand.records)

    def no_staging(records):
        raise AssertionError("pinned-image payloads went through the staging ring")
    monkeypatch.setattr(device, "_stage_pageable", no_staging)
    tol = td.ToleranceMap.from_json(cases["tols"][case["tol"]])
    rep = td.check(ref, cand, tol, case["kappa"], fmt=td.FloatFormat(case["fmt"]))
    assert_reports_match(json.loads(td.render_report(rep, "json")), json.loads(case["report"]), "pinned image")
    monkeypatch.undo()
    plain = td.check(td.read_trace(paths["ref"]), td.read_trace(paths["cand"]), tol, case["kappa"],
                     fmt=td.FloatFormat(case["fmt"]))
    assert_reports_match(json.loads(td.render_report(plain, "json")), json.loads(case["report"]), "unpinned")


def test_gather_bytes_any_offsets_against_numpy():
    """td_gather_bytes over every source/destination alignment pair (the
    uint4, u32 and funnel-shift paths plus the bytewise heads and tails) and
    ranges longer than one 64 KiB piece: bit-exact against numpy slicing,
    bytes outside the destination ranges untouched."""
    from paper_2506_09280_b200 import _native as N
    rng = np.random.default_rng(11)
    src_h = rng.integers(0, 256, 1 << 21, dtype=np.uint8)
    src = torch.from_numpy(src_h).cuda()
    dst = torch.full((1 << 21,), 0xA5, dtype=torch.uint8, device="cuda")
    table, cur = [], 64
    for so_mod in range(16):
        for do_mod in range(16):
            nb = int(rng.choice([0, 1, 3, 15, 16, 17, 33, 100, 4099]))
            so = int(rng.integers(0, (1 << 21) - 5000)) // 16 * 16 + so_mod
            dof = cur // 16 * 16 + 16 + do_mod
            table.append((so, dof, nb))
            cur = dof + nb + 1
    for so, dof in ((3, cur + 32 + 7), (16, cur + 300000 + 1)):   # multi-piece ranges
        table.append((so, dof, 200001))
        cur = dof + 200001 + 1
    assert cur < (1 << 21)
    ranges = torch.tensor(table, dtype=torch.int64).cuda()
    N.call("td_gather_bytes", src.data_ptr(), dst.data_ptr(), ranges.data_ptr(), len(table), N.stream_handle())
    got = dst.cpu().numpy()
    want = np.full(1 << 21, 0xA5, dtype=np.uint8)
    for so, dof, nb in table:
        want[dof:dof + nb] = src_h[so:so + nb]
    assert np.array_equal(got, want)


def test_write_trace_from_device_is_byte_identical(tmp_path, cases, golden_trace_bytes):
    """write_trace of a CUDA-resident trace (the file image laid out on the
    device, one D2H, parallel pwrites) writes exactly the reference's bytes."""
    from paper_2506_09280_b200.tracestore import read_trace, write_trace
    for name in cases["traces"][:6]:
        raw = golden_trace_bytes(name)
        src = tmp_path / (name + ".in.ttrc")
        src.write_bytes(raw)
        dev = read_trace(src, device="cuda")
        out = tmp_path / (name + ".out.ttrc")
        write_trace(dev, out)
        assert out.read_bytes() == raw, name


def test_concurrent_file_reads_and_host_checks(tmp_path, cases, golden_trace_bytes):
    """The pinned rings (file reader, host staging) are process-wide: two
    threads reading traces to the device and checking host traces at the
    same time get the same results as one thread doing it alone."""
    import concurrent.futures
    from paper_2506_09280_b200 import tracestore
    from paper_2506_09280_b200.tracestore import read_trace
    names = cases["traces"][:4]
    for name in names:
        (tmp_path / (name + ".ttrc")).write_bytes(golden_trace_bytes(name))
    # 64 KiB ring slots x 4: every read spans many slots and wraps the ring,
    # so a reader that refilled a slot before the previous caller's DMA out
    # of it had finished would corrupt that caller's image
    saved = tracestore._RING_PIECE, tracestore._RING_SLOTS, tracestore._RING
    tracestore._RING_PIECE, tracestore._RING_SLOTS, tracestore._RING = 64 << 10, 4, None
    try:
        def job(name):
            dev = read_trace(tmp_path / (name + ".ttrc"), device="cuda")
            return [r.payload.cpu().numpy().tobytes() for r in dev.records]
        want = {n: job(n) for n in names}
        with concurrent.futures.ThreadPoolExecutor(4) as ex:
            for _ in range(3):
                got = dict(zip(names, ex.map(job, names)))
                assert got == want
    finally:
        tracestore._RING_PIECE, tracestore._RING_SLOTS, tracestore._RING = saved


def test_concurrent_checks_share_a_cached_plan(cases, golden_trace_bytes):
    """check() caches one plan per layout, with one pinned staging buffer for
    its tables: threads checking different payloads of the SAME layout at
    once get exactly their own serial reports."""
    import concurrent.futures
    case = next(c for c in cases["checks"] if c["name"] == "clean_tp2_cp2_k3")
    ref = trace_from_bytes(golden_trace_bytes(case["ref"]), device="cuda")
    cand = trace_from_bytes(golden_trace_bytes(case["cand"]), device="cuda")
    tol = td.ToleranceMap.from_json(cases["tols"][case["tol"]])
    fmt = td.FloatFormat(case["fmt"])
    variants = []
    for k in range(6):
        c = Trace(header=cand.header, raw_header=cand.raw_header)
        for j, r in enumerate(cand.records):
            p = r.payload.clone()
            if j == (7 * k) % len(cand.records) and p.numel():
                p.mul_(1.0 + 0.5 * k)
            c.records.append(TraceRecord(r.id, r.rank_meta, r.mapping, r.replica_group_size, p, r.module_class))
        variants.append(c)

    def job(c):
        return td.render_report(td.check(ref, c, tol, case["kappa"], fmt=fmt), "json")
    want = [job(c) for c in variants]
    with concurrent.futures.ThreadPoolExecutor(6) as ex:
        for _ in range(4):
            assert list(ex.map(job, variants)) == want


def _wide_replica_traces(n_copies, corrupt=(), dtype=None):
    """A 16-copy (or any) replica group: reference = one (64, 96) id; the
    candidate holds n_copies identity-mapped copies (replica_group_size =
    n_copies, rank tp = copy index); corrupt = {copy: scale}."""
    dtype = dtype or torch.bfloat16
    ident = CanonicalId(0, 0, TensorKind.ACTIVATION_OUT, "model.layers.0.attn")
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn((64, 96), generator=g, device="cuda").to(dtype)
    y = td.apply_perturbation(x, "cand|" + ident.encode(), td.PerturbSpec(0, 2.0 ** -8), policy="bf16")
    hdr = {"digest": "wide", "mode": "cascade"}
    ref = Trace(dict(hdr), [TraceRecord(ident, RankMeta(), identity_mapping((64, 96)), 1, x, "Attn")])
    cand = Trace(dict(hdr), [])
    for c in range(n_copies):
        p = y.clone()
        if c in dict(corrupt):
            p = (p.float() * dict(corrupt)[c]).to(dtype)
        cand.records.append(TraceRecord(ident, RankMeta(tp=c), identity_mapping((64, 96)), n_copies, p, "Attn"))
    return ref, cand


def _oracle_report(ref, cand, tol, fmt="BF16"):
    def host(t):
        return [O.Rec(r.id.encode(), r.rank_meta.as_tuple(), r.mapping.local_shape, r.mapping.global_shape,
                      [(a.bounds, b.bounds) for a, b in r.mapping.pairs], r.replica_group_size,
                      r.payload.float().cpu().numpy()) for r in t.records]
    return O.check(host(ref), host(cand), ref.header, cand.header, tol.responses, 3.0, fmt)


@pytest.mark.parametrize("n_copies,corrupt", [(16, ()), (16, ((11, 1.5),)), (16, ((3, 1.01), (12, 2.0))),
                                              (9, ((8, 3.0),)), (23, ((15, 1.25), (22, 1.25)))])
def test_replica_groups_beyond_eight_copies(n_copies, corrupt):
    """Replica groups of more than 8 copies (check_replicas walks any number,
    canonical.py:225-247): chunks of 7 replicas per group slot, copy 0
    re-read per chunk, the worst folded with the reference's strict >
    (first maximum wins).  Reports equal the CPU oracle's."""
    ref, cand = _wide_replica_traces(n_copies, corrupt)
    tol = td.ToleranceMap({ref.records[0].id.encode(): 2.0 ** -8}, n_samples=1, eps_p=2.0 ** -8)
    got = json.loads(td.render_report(td.check(ref, cand, tol, fmt=td.FloatFormat.BF16), "json"))
    want = _oracle_report(ref, cand, tol)
    assert_reports_match(got, want, f"{n_copies} copies {corrupt}")
    assert (got["summary"]["replica-mismatch"] == 1) == bool(corrupt)
