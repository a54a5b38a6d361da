"""Generate the golden fixtures by running the REFERENCE implementation.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [/root/reference]

Only this script imports the reference (`traindiff`, from
<reference>/pkg/src); it runs in the build container, never on the GPU box.
Everything it writes under tests/golden/ is small and committed:

  traces/*.ttrc.gz      reference-emulator traces (TTRC bytes, gzip)
  cases.json.gz         check / estimate_tolerance scenarios + the reference's
                        own report JSON and tolerance JSON for each
  shardings.json.gz     randomized shardings (test_acceptance.py:47-112
                        procedure) with the reference merge's witnesses
  layouts.json.gz       id emission / shard-map signatures over the 60-layout
                        grid (test_acceptance.py:118-148) — index-map parity
  vectors.json.gz       RNG, quantizer, perturbation and rel_err known answers
  torchtap.json.gz      the reference torchtap adapter's flushed bytes for small models
"""

from __future__ import annotations

import gzip
import itertools
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = sys.argv[1] if len(sys.argv) > 1 else "/root/reference"
sys.dont_write_bytecode = True
sys.path.insert(0, os.path.join(REF, "pkg", "src"))

from traindiff.bugs import BugInjection  # noqa: E402
from traindiff.canonical import ShardMapping, SliceBox, merge  # noqa: E402
from traindiff.checker import check, estimate_tolerance, render_report  # noqa: E402
from traindiff.engine import (ParallelConfig, PerturbSpec, run_candidate,  # noqa: E402
                              run_reference, validate_parallel)
from traindiff.errors import ConfigInvalid, MergeConflict  # noqa: E402
from traindiff.generation import (SplitMix64, _words, fnv1a_64, seed_from,  # noqa: E402
                                  signed_uniforms)
from traindiff.model import ModelConfig  # noqa: E402
from traindiff.tensor import FloatFormat, quantize_array, rel_err_arrays  # noqa: E402
from traindiff.tracestore import trace_to_bytes  # noqa: E402

TRACES = os.path.join(HERE, "traces")


def cfg(layers=2, precision="bf16", **kw):
    base = dict(layers=layers, d_model=32, n_heads=4, d_ff=64, seq_len=16, vocab=64,
                precision=precision)
    base.update(kw)
    return ModelConfig(**base)


def save_trace(name: str, trace) -> str:
    os.makedirs(TRACES, exist_ok=True)
    path = os.path.join(TRACES, name + ".ttrc.gz")
    with open(path, "wb") as raw, gzip.GzipFile(fileobj=raw, mode="wb", compresslevel=9, mtime=0) as fh:
        fh.write(trace_to_bytes(trace))
    return name


def scenarios() -> dict:
    out = {"traces": [], "checks": [], "estimates": [], "tols": {}}
    saved = set()

    def keep(name, trace):
        if name not in saved:
            save_trace(name, trace)
            saved.add(name)
            out["traces"].append(name)
        return name

    # -- bf16 cascade family (test_checker.py:25-43 scale) -------------------
    c = cfg()
    M = 4
    ref = run_reference(c, microbatches=M).trace
    keep("bf16_ref_m4", ref)
    perturbed = []
    for s in range(3):
        t = run_reference(c, microbatches=M, perturb=PerturbSpec(s, FloatFormat.BF16.eps)).trace
        perturbed.append(keep(f"bf16_ref_m4_pert{s}", t))
    tol = estimate_tolerance(lambda p: run_reference(c, microbatches=M, perturb=p).trace,
                             n_samples=3, eps_p=FloatFormat.BF16.eps)
    out["tols"]["bf16_m4_n3_max"] = tol.to_json().decode()
    out["estimates"].append({"name": "bf16_m4_n3_max", "base": "bf16_ref_m4",
                             "perturbed": perturbed, "eps_p": FloatFormat.BF16.eps,
                             "aggregation": "max", "tol": tol.to_json().decode()})
    tol_mean = estimate_tolerance(lambda p: run_reference(c, microbatches=M, perturb=p).trace,
                                  n_samples=3, eps_p=FloatFormat.BF16.eps, aggregation="mean")
    out["estimates"].append({"name": "bf16_m4_n3_mean", "base": "bf16_ref_m4",
                             "perturbed": perturbed, "eps_p": FloatFormat.BF16.eps,
                             "aggregation": "mean", "tol": tol_mean.to_json().decode()})
    layouts = [
        ("clean_tp2_cp2", ParallelConfig(tp=2, cp=2, microbatches=M), ()),
        ("clean_dp2_tp2", ParallelConfig(dp=2, tp=2, microbatches=M), ()),
        ("clean_tp2_sp", ParallelConfig(tp=2, sp=True, microbatches=M), ()),
        ("clean_dp2_cp2_pp2", ParallelConfig(dp=2, cp=2, pp=2, microbatches=M), ()),
        ("bug_tp_row_allreduce", ParallelConfig(tp=2, microbatches=M), ("MC_TP_ROW_ALLREDUCE",)),
        ("bug_stale_input", ParallelConfig(dp=2, microbatches=M), ("WD_STALE_INPUT",)),
        ("bug_wrong_order_sp", ParallelConfig(tp=2, sp=True, microbatches=M), ("WC_WRONG_ORDER",)),
        ("bug_sp_norm_grad", ParallelConfig(tp=2, sp=True, microbatches=M), ("MC_SP_NORM_GRAD",)),
        ("bug_layout_cp", ParallelConfig(cp=2, microbatches=M), ("WD_LAYOUT",)),
        ("bug_wrong_scale", ParallelConfig(tp=2, microbatches=M), ("WD_WRONG_SCALE",)),
        ("bug_dp_grad", ParallelConfig(dp=2, microbatches=M), ("MC_DP_GRAD",)),
        ("bug_wrong_group", ParallelConfig(dp=2, cp=2, microbatches=M), ("WC_WRONG_GROUP",)),
        ("bug_wrong_reduce_op", ParallelConfig(tp=2, sp=True, microbatches=M), ("WC_WRONG_REDUCE_OP",)),
    ]
    for name, pcfg, bugs in layouts:
        cand = run_candidate(c, pcfg, tuple(BugInjection(b) for b in bugs)).trace
        keep("bf16_" + name, cand)
        for kappa in (3.0,) if name != "bug_wrong_order_sp" else (0.5, 3.0, 1e6):
            rep = check(ref, cand, tol, kappa, fmt=FloatFormat.BF16)
            out["checks"].append({"name": f"{name}_k{kappa:g}", "ref": "bf16_ref_m4",
                                  "cand": "bf16_" + name, "tol": "bf16_m4_n3_max",
                                  "kappa": kappa, "fmt": "BF16",
                                  "report": render_report(rep, "json"),
                                  "text": render_report(rep, "text")})
    # swapped roles (test_checker.py:347-355)
    cand = run_candidate(c, ParallelConfig(dp=2, tp=2, microbatches=M)).trace
    rep = check(cand, ref, tol, fmt=FloatFormat.BF16)
    out["checks"].append({"name": "swapped_dp2_tp2", "ref": "bf16_clean_dp2_tp2", "cand": "bf16_ref_m4",
                          "tol": "bf16_m4_n3_max", "kappa": 3.0, "fmt": "BF16",
                          "report": render_report(rep, "json"), "text": render_report(rep, "text")})
    # -- module-wise mode (test_checker.py:358-372) ----------------------------
    mref = run_reference(c, microbatches=M, rewrite=True).trace
    keep("bf16_modwise_ref_m4", mref)
    mtol = estimate_tolerance(lambda p: run_reference(c, microbatches=M, rewrite=True, perturb=p).trace,
                              n_samples=3, eps_p=FloatFormat.BF16.eps)
    mcand = run_candidate(c, ParallelConfig(tp=2, microbatches=M), (BugInjection("WD_WRONG_SCALE"),),
                          rewrite=True).trace
    keep("bf16_modwise_wrong_scale", mcand)
    out["tols"]["bf16_modwise_m4_n3_max"] = mtol.to_json().decode()
    rep = check(mref, mcand, mtol, fmt=FloatFormat.BF16)
    out["checks"].append({"name": "modwise_wrong_scale", "ref": "bf16_modwise_ref_m4",
                          "cand": "bf16_modwise_wrong_scale", "tol": "bf16_modwise_m4_n3_max",
                          "kappa": 3.0, "fmt": "BF16", "report": render_report(rep, "json"),
                          "text": render_report(rep, "text")})
    # -- config-1 miniature: fp32, reference vs TP=2 -----------------------------
    f = cfg(precision="fp32")
    fref = run_reference(f, microbatches=1).trace
    keep("fp32_ref_m1", fref)
    fpert = [keep(f"fp32_ref_m1_pert{s}",
                  run_reference(f, microbatches=1, perturb=PerturbSpec(s, FloatFormat.FP32.eps)).trace)
             for s in range(2)]
    ftol = estimate_tolerance(lambda p: run_reference(f, microbatches=1, perturb=p).trace,
                              n_samples=2, eps_p=FloatFormat.FP32.eps)
    out["estimates"].append({"name": "fp32_m1_n2_max", "base": "fp32_ref_m1", "perturbed": fpert,
                             "eps_p": FloatFormat.FP32.eps, "aggregation": "max",
                             "tol": ftol.to_json().decode()})
    out["tols"]["fp32_m1_n2_max"] = ftol.to_json().decode()
    fcand = run_candidate(f, ParallelConfig(tp=2, microbatches=1)).trace
    keep("fp32_tp2_m1", fcand)
    rep = check(fref, fcand, ftol, fmt=FloatFormat.FP32)
    out["checks"].append({"name": "fp32_tp2", "ref": "fp32_ref_m1", "cand": "fp32_tp2_m1",
                          "tol": "fp32_m1_n2_max", "kappa": 3.0, "fmt": "FP32",
                          "report": render_report(rep, "json"), "text": render_report(rep, "text")})
    return out


# ---------------------------------------------------------------------------
# randomized shardings with witnesses (test_acceptance.py:47-112 procedure)

def _grid(rng, shape):
    cuts = []
    for n in shape:
        k = int(rng.integers(1, min(n, 3) + 1))
        pts = sorted(rng.choice(np.arange(1, n), size=k - 1, replace=False).tolist()) if k > 1 else []
        edges = [0, *pts, n]
        cuts.append(list(zip(edges, edges[1:])))
    return cuts


def _shards(rng, shape, cuts):
    shards = []
    for col in itertools.product(*cuts[1:]):
        i = 0
        while i < len(cuts[0]):
            group = cuts[0][i:i + int(rng.integers(1, 3))]
            i += len(group)
            height = sum(b - a for a, b in group)
            local_shape = (height,) + tuple(b - a for a, b in col)
            pairs, off = [], 0
            for a, b in group:
                local = SliceBox(((off, off + b - a),) + tuple((0, e - s) for s, e in col))
                pairs.append((local, SliceBox(((a, b),) + col)))
                off += b - a
            shards.append(ShardMapping(local_shape, shape, tuple(pairs)))
    return shards


def _sig(m: ShardMapping):
    return {"local_shape": list(m.local_shape), "global_shape": list(m.global_shape),
            "pairs": [[list(map(list, l.bounds)), list(map(list, g.bounds))] for l, g in m.pairs]}


def _merge_outcome(maps, shape):
    try:
        merge([(m, np.zeros(m.local_shape)) for m in maps], shape)
        return None
    except MergeConflict as exc:
        return {"message": str(exc), "witness": list(exc.witness)}


def shardings() -> list:
    rng = np.random.default_rng(20240817)
    cases = []
    for _ in range(1000):
        shape = tuple(int(rng.integers(1, 7)) for _ in range(int(rng.integers(1, 4))))
        maps = _shards(rng, shape, _grid(rng, shape))
        victim = int(rng.integers(0, len(maps)))
        cases.append({"shape": list(shape), "shards": [_sig(m) for m in maps], "victim": victim,
                      "ok": _merge_outcome(maps, shape),
                      "omitted": _merge_outcome(maps[:victim] + maps[victim + 1:], shape),
                      "doubled": _merge_outcome(maps + [maps[victim]], shape)})
    return cases


# ---------------------------------------------------------------------------
# layout grid: which ids exist, their shard maps and replica sizes

def layouts() -> list:
    c = cfg(layers=4)
    out = []
    for dp, tp, pp, vp, cp, sp in itertools.product((1, 2), (1, 2), (1, 2), (1, 2), (1, 2), (False, True)):
        p = ParallelConfig(dp=dp, tp=tp, pp=pp, vp=vp, cp=cp, sp=sp, microbatches=4)
        try:
            validate_parallel(c, p)
        except ConfigInvalid:
            continue
        trace = run_candidate(c, p).trace
        recs = [[r.id.encode(), list(r.rank_meta.as_tuple()), r.replica_group_size, r.module_class,
                 list(r.mapping.local_shape), list(r.mapping.global_shape),
                 [[list(map(list, l.bounds)), list(map(list, g.bounds))] for l, g in r.mapping.pairs]]
                for r in trace.records]
        out.append({"parallel": p.as_dict(), "model": c.as_dict(), "records": recs})
    return out


# ---------------------------------------------------------------------------
# known-answer vectors

def vectors() -> dict:
    v = {}
    v["fnv1a"] = {s: fnv1a_64(s.encode()) for s in ["", "a", "perturb|s=0|iter=0|mb=0|kind=ActivationOut|mod=model.embedding"]}
    gen = SplitMix64(0)
    v["splitmix_seed0"] = [gen.next_word() for _ in range(3)]
    streams = []
    for seed in (0, 1, 2 ** 64 - 1, 123456789, seed_from("perturb|s=3|iter=0|mb=1|kind=ActivationIn|mod=model.layers.0.mlp")):
        streams.append({"seed": seed, "words": [int(w) for w in _words(seed, 64)]})
    v["splitmix_streams"] = streams
    tags = ["perturb|s=0|iter=0|mb=0|kind=ActivationOut|mod=model.embedding",
            "perturb|s=2|iter=0|mb=3|kind=ActivationIn|mod=model.layers.1.attn"]
    v["signed_uniforms"] = [{"tag": t, "n": 4096,
                             "values_hex": [float(x).hex() for x in signed_uniforms(t, (4096,))]}
                            for t in tags]
    rng = np.random.default_rng(7)
    q = {}
    for fmt in FloatFormat:
        xs = np.concatenate([rng.standard_normal(300), rng.standard_normal(100) * 1e-20,
                             (rng.standard_normal(100) * (1e20 if fmt is not FloatFormat.FP8E4M3 else 100)),
                             np.array([0.0, -0.0, 1.0, -1.0, 0.2, 2.0 ** -60, 257.0, 1 + 2.0 ** -8,
                                       1e39, -1e39, 500.0, -500.0, fmt.max_finite, 5e-324, 1e-310])])
        q[fmt.value] = {"x_hex": [float(x).hex() for x in xs],
                        "y_hex": [float(y).hex() for y in quantize_array(xs, fmt)]}
    v["quantize"] = q
    # perturbation of bf16-grid activations, the reference pipeline end to end
    pert = []
    for eps in (2.0 ** -8, 1e-3, 2.0 ** -24):
        for fmt in (FloatFormat.BF16, FloatFormat.FP32):
            tag = "perturb|s=1|iter=0|mb=0|kind=ActivationOut|mod=model.embedding"
            rows, cols = 16, 64
            x = quantize_array(np.random.default_rng(11).standard_normal((rows, cols)), FloatFormat.BF16)
            pos = np.array([2, 3, 12, 13, 4, 5, 10, 11, 0, 1, 14, 15, 6, 7, 8, 9])
            u = signed_uniforms(tag, (rows, cols))
            y = x * (1.0 + u[pos] * eps)
            if fmt is FloatFormat.BF16:
                y = quantize_array(y, fmt)
            pert.append({"tag": tag, "eps": eps, "fmt": fmt.value, "rows": rows, "cols": cols,
                         "pos": pos.tolist(), "x_hex": [float(a).hex() for a in x.ravel()],
                         "y_hex": [float(a).hex() for a in np.asarray(y).ravel()]})
    v["perturb"] = pert
    rel = []
    r = np.random.default_rng(5)
    for n in (1, 2, 7, 64, 1000, 4099):
        a = r.standard_normal(n).astype(np.float32).astype(np.float64)
        b = (a + r.standard_normal(n) * 1e-3).astype(np.float32).astype(np.float64)
        rel.append({"a_hex": [float(x).hex() for x in a], "b_hex": [float(x).hex() for x in b],
                    "rel": float(rel_err_arrays(a, b)).hex()})
    v["rel_err"] = rel
    from traindiff.canonical import CanonicalId, TensorKind
    from traindiff.generation import GenSpec, Normal, TokenIds, Uniform, generate_full
    gens = []
    for ident, spec, kind in [
            (CanonicalId(0, 0, TensorKind.PARAM, "model.embedding.word"), GenSpec(Normal(0.0, 0.02), (64, 32)), "normal"),
            (CanonicalId(0, 1, TensorKind.ACTIVATION_IN, "model.layers.3.mlp"), GenSpec(Normal(0.0, 0.02), (16, 33)), "normal"),
            (CanonicalId(0, 0, TensorKind.ACTIVATION_IN, "ustats"), GenSpec(Uniform(-2.0, 6.0), (5000,)), "uniform"),
            (CanonicalId(0, 3, TensorKind.ACTIVATION_IN, "model.embedding"), GenSpec(TokenIds(vocab=50257), (4096,)), "tokens")]:
        data = generate_full(ident, spec).data
        gens.append({"ident": ident.encode(), "kind": kind, "shape": list(spec.shape),
                     "params": list(spec.distribution.__dict__.values()),
                     "values_hex": [float(x).hex() for x in data.ravel()]})
    v["generate_full"] = gens
    return v


def torchtap_golden() -> dict:
    """The reference adapter's own capture of small torch models
    (pkg/adapter/tests/test_torchtap.py:10-19 setup), as flushed bytes."""
    sys.path.insert(0, os.path.join(REF, "pkg", "adapter", "src"))
    import torch
    import torchtap
    out = {}
    torch.manual_seed(7)
    net = torch.nn.Sequential(torch.nn.Linear(8, 16, bias=False), torch.nn.Linear(16, 4, bias=False))
    x = torch.randn(5, 8)
    h = torchtap.attach(net, torchtap.TapConfig(patterns=("*",)))
    net(x).square().sum().backward()
    out["two_linear"] = {"seed": 7, "bytes_hex": torchtap.to_bytes(h).hex(),
                         "idents": [r.ident for r in h.records]}
    torch.manual_seed(3)
    mlp = torch.nn.Sequential(torch.nn.LayerNorm(16), torch.nn.Linear(16, 32), torch.nn.GELU(),
                              torch.nn.Linear(32, 16))
    xb = torch.randn(4, 16)
    h = torchtap.attach(mlp, torchtap.TapConfig(patterns=("*",), iteration=2, microbatch=1,
                                                precision="bf16"))
    mlp(xb).sum().backward()
    out["layernorm_mlp"] = {"seed": 3, "bytes_hex": torchtap.to_bytes(h).hex(),
                            "idents": [r.ident for r in h.records]}
    return out


def _dump_gz(name: str, obj, sort_keys: bool = False) -> None:
    with open(os.path.join(HERE, name), "wb") as raw, \
            gzip.GzipFile(fileobj=raw, mode="wb", compresslevel=9, mtime=0) as fh:
        fh.write(json.dumps(obj, sort_keys=sort_keys).encode())


def main():
    os.makedirs(HERE, exist_ok=True)
    _dump_gz("cases.json.gz", scenarios(), sort_keys=True)
    _dump_gz("shardings.json.gz", shardings())
    _dump_gz("layouts.json.gz", layouts())
    _dump_gz("vectors.json.gz", vectors(), sort_keys=True)
    _dump_gz("torchtap.json.gz", torchtap_golden(), sort_keys=True)
    print("wrote golden fixtures to", HERE)


if __name__ == "__main__":
    main()
