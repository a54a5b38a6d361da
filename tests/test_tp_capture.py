"""§8(f) #3: real-TP annotated captures from a live tensor-parallel run.

A Megatron-style TP=2 GPT (tests/tp_gpt.py) runs as two real
torch.distributed ranks (gloo); torchtap.layout_shard tags every capture
with the reference emulator's map for that rank (engine.py:268-296).  The
CPU tests check the annotated candidate against a single-device run with
the CPU oracle (test infrastructure); the GPU tests run the same live job
on cuda:0 (two processes, gloo on CUDA tensors), feed the device-resident
captures to check() and to check_distributed() — each rank passing only its
own records — and compare with the oracle.

Bug site (reference test_checker.py:314-325): with the row-parallel
all-reduce of `model.layers.1.attn` dropped (MC_TP_ROW_ALLREDUCE), the
earliest divergence is that block's ActivationOut, a replica-mismatch whose
observed error clears the tolerance floor by >= 10x.
"""

from __future__ import annotations

import os
import pickle
import socket

import pytest
import torch
import torch.multiprocessing as mp

from oracle import traindiff_oracle as O
from paper_2506_09280_b200 import torchtap
from paper_2506_09280_b200.layout import Layout, ParallelConfig
from paper_2506_09280_b200.torchtap import TapError

from . import tp_gpt

SHAPE = {"layers": 2, "d": 32, "heads": 4, "ff": 64, "seq": 16, "vocab": 64}
# Llama-3 block rules (GQA 8/2, SwiGLU w3, RMSNorm, no position table)
LLAMA = {"layers": 2, "d": 64, "heads": 8, "kv_heads": 2, "ff": 96, "seq": 16, "vocab": 64, "llama": True}
BUG_SITE = "iter=0|mb=0|kind=ActivationOut|mod=model.layers.1.attn"


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _flat(rec) -> dict:
    m = rec.mapping
    return {"ident": rec.ident, "rank": tuple(rec.rank), "local": m.local_shape, "global": m.global_shape,
            "pairs": [(l.bounds, g.bounds) for l, g in m.pairs], "replica": rec.replica,
            "payload": rec.host(), "cls": rec.module_class, "dtype": str(rec.payload.dtype).split(".")[-1]}


def _tp_worker(rank, world, port, out_dir, shape, device, dtype_name, skip, mode, responses=None, kappa=3.0):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if device == "cuda":
            torch.cuda.set_device(0)
        g = tp_gpt.TPGroup(rank, world)
        h = tp_gpt.traced_step(shape, g, device=device, dtype=getattr(torch, dtype_name),
                               skip_reduce=skip, precision=dtype_name)
        result = {"records": [_flat(r) for r in h.records], "header": h.header()}
        if mode == "distributed":
            import paper_2506_09280_b200 as td
            from paper_2506_09280_b200.distributed import (TorchComm, check_distributed, global_trace,
                                                           split_reference)
            ref_h = tp_gpt.traced_step(shape, tp_gpt.TPGroup(), device=device,
                                       dtype=getattr(torch, dtype_name), precision=dtype_name)
            comm = TorchComm()
            cand = h.trace()
            refs = split_reference(ref_h.trace(), global_trace(cand, comm), world)
            fmt = td.FloatFormat.BF16 if dtype_name == "bfloat16" else td.FloatFormat.FP32
            tol = td.ToleranceMap(dict(responses or {}), n_samples=3, eps_p=fmt.eps)
            rep = check_distributed(refs[rank], cand, tol, kappa, fmt=fmt, comm=comm)
            result["report"] = td.render_report(rep, "json")
        with open(os.path.join(out_dir, f"rank{rank}.pkl"), "wb") as fh:
            pickle.dump(result, fh)
    finally:
        dist.destroy_process_group()


def run_tp(tmp_path, shape=SHAPE, world=2, device="cpu", dtype="float32", skip=(), mode="capture",
           responses=None, kappa=3.0):
    mp.start_processes(_tp_worker, args=(world, _free_port(), str(tmp_path), shape, device, dtype,
                                         tuple(skip), mode, responses, kappa),
                       nprocs=world, join=True, start_method="spawn")
    out = []
    for r in range(world):
        with open(tmp_path / f"rank{r}.pkl", "rb") as fh:
            out.append(pickle.load(fh))
    return out


def _oracle_recs(flat_records):
    return [O.Rec(f["ident"], f["rank"], f["local"], f["global"], f["pairs"], f["replica"],
                  f["payload"], f["cls"]) for f in flat_records]


def _single_device(shape=SHAPE, device="cpu", dtype=torch.float32, precision="float32"):
    return tp_gpt.traced_step(shape, tp_gpt.TPGroup(), device=device, dtype=dtype, precision=precision)


def test_layout_shard_maps_are_the_layouts():
    layout = Layout(tp_gpt.model_shape(SHAPE), ParallelConfig(tp=2))
    shard = torchtap.layout_shard(layout, tp=1)
    d, S, V = SHAPE["d"], SHAPE["seq"], SHAPE["vocab"]
    m, rank, rep = shard("model.layers.0.attn.wq", "ParamGrad", torch.empty(d, d // 2))
    assert m.pairs[0][1].bounds == ((0, d), (d // 2, d)) and rep == 1 and rank[1] == 1
    m, _, rep = shard("model.layers.0.attn.wo", "ParamGrad", torch.empty(d // 2, d))
    assert m.pairs[0][1].bounds == ((d // 2, d), (0, d)) and rep == 1
    m, _, rep = shard("model.layers.1.mlp.norm.weight", "ParamGrad", torch.empty(d))
    assert m.global_shape == (d,) and rep == 2
    m, _, rep = shard("model.lm_head", "ActivationOut", torch.empty(S, V // 2))
    assert m.pairs[0][1].bounds == ((0, S), (V // 2, V)) and rep == 1
    m, _, rep = shard("model.layers.0.attn.norm", "ActivationOut", torch.empty(S, d))
    assert m.global_shape == (S, d) and rep == 2
    with pytest.raises(TapError, match="shape"):
        shard("model.layers.0.attn.wq", "ParamGrad", torch.empty(d, d))
    with pytest.raises(TapError, match="no ParamGrad map"):
        shard("model.layers.0.attn.bogus", "ParamGrad", torch.empty(d))
    with pytest.raises(TapError, match="outside"):
        torchtap.layout_shard(layout, tp=2)


@pytest.mark.parametrize("shape", [SHAPE, LLAMA], ids=["gpt", "llama"])
def test_live_tp2_capture_matches_single_device(tmp_path, shape):
    ranks = run_tp(tmp_path, shape=shape)
    ref = _single_device(shape)
    cand = [f for r in ranks for f in r["records"]]
    # every capture carries its rank's map; copies of one id agree on the id set
    assert {f["rank"][1] for f in cand} == {0, 1}
    ids0 = [f["ident"] for f in ranks[0]["records"]]
    assert sorted(ids0) == sorted(f["ident"] for f in ranks[1]["records"])
    assert sorted(set(ids0)) == sorted(r.ident for r in ref.records)
    doc = O.check(_oracle_recs([_flat(r) for r in ref.records]), _oracle_recs(cand),
                  ref.header(), ranks[0]["header"], {}, 3.0, "BF16")
    assert doc["exit_code"] == 0, doc["summary"]
    assert doc["summary"]["pass"] == len(set(ids0)) and doc["summary"]["missing"] == 0
    # fp32 host math: TP=2 differs from one device by reassociation only
    assert max(e["observed"] for e in doc["entries"]) < 1e-5
    # the layout's own id set for this model (layout.emit_records) covers
    # every capture of the tapped kinds
    kinds = ("ActivationIn", "ActivationOut", "ParamGrad")
    want = {sp.ident for sp in Layout(tp_gpt.model_shape(shape), ParallelConfig(tp=2)).records()
            if sp.kind in kinds}
    got = {i for i in ids0 if not i.endswith(".norm")}
    assert got == want


def _dp_tp_worker(rank, world, port, out_dir, shape, tp):
    """Rank r of a dp x tp job: TP group {d*tp .. d*tp+tp-1}, microbatch d."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dp = world // tp
        groups = [dist.new_group(list(range(d * tp, (d + 1) * tp))) for d in range(dp)]
        d, t = divmod(rank, tp)
        h = tp_gpt.traced_step(shape, tp_gpt.TPGroup(t, tp, groups[d]), dp=dp, dp_rank=d, microbatch=d)
        with open(os.path.join(out_dir, f"rank{rank}.pkl"), "wb") as fh:
            pickle.dump({"records": [_flat(r) for r in h.records], "header": h.header()}, fh)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("shape", [SHAPE, LLAMA], ids=["gpt", "llama"])
def test_live_dp2_tp2_microbatches_match_single_device(tmp_path, shape):
    """DP=2 x TP=2 live job (4 gloo ranks, TP sub-groups): DP rank d runs
    microbatch d; every capture carries its (dp, tp) rank and the layout's
    map (ids iter=0|mb=d|...); the union equals a single device running both
    microbatches, per the CPU oracle, and covers the layout's id set."""
    world, tp = 4, 2
    mp.start_processes(_dp_tp_worker, args=(world, _free_port(), str(tmp_path), shape, tp),
                       nprocs=world, join=True, start_method="spawn")
    ranks = []
    for r in range(world):
        with open(tmp_path / f"rank{r}.pkl", "rb") as fh:
            ranks.append(pickle.load(fh))
    cand = [f for r in ranks for f in r["records"]]
    assert {(f["rank"][0], f["rank"][1]) for f in cand} == {(0, 0), (0, 1), (1, 0), (1, 1)}
    assert {f["ident"].split("|")[1] for f in cand} == {"mb=0", "mb=1"}
    ref = [_flat(r) for mb in (0, 1) for r in tp_gpt.traced_step(shape, tp_gpt.TPGroup(), microbatch=mb).records]
    doc = O.check(_oracle_recs(ref), _oracle_recs(cand), ranks[0]["header"], ranks[0]["header"], {}, 3.0, "BF16")
    assert doc["exit_code"] == 0 and doc["summary"]["missing"] == 0, doc["summary"]
    assert max(e["observed"] for e in doc["entries"]) < 1e-5
    kinds = ("ActivationIn", "ActivationOut", "ParamGrad")
    want = {sp.ident for sp in Layout(tp_gpt.model_shape(shape), ParallelConfig(tp=2, dp=2, microbatches=2)).records()
            if sp.kind in kinds}
    assert {f["ident"] for f in cand if not f["ident"].endswith(".norm")} == want


@pytest.mark.parametrize("shape", [SHAPE, LLAMA], ids=["gpt", "llama"])
def test_live_tp2_missing_allreduce_is_a_replica_mismatch_at_the_site(tmp_path, shape):
    ranks = run_tp(tmp_path, shape=shape, skip=("model.layers.1.attn",))
    ref = _single_device(shape)
    cand = [f for r in ranks for f in r["records"]]
    doc = O.check(_oracle_recs([_flat(r) for r in ref.records]), _oracle_recs(cand),
                  ref.header(), ranks[0]["header"], {}, 3.0, "BF16")
    assert doc["earliest_divergence"] == BUG_SITE
    entry = next(e for e in doc["entries"] if e["id"] == BUG_SITE)
    assert entry["verdict"] == "replica-mismatch"
    assert entry["observed"] >= 10 * O.eps_of("BF16")
    assert doc["exit_code"] == 3
    # everything the bug cannot reach stays clean
    before = [e for e in doc["entries"] if "layers.0" in e["id"] and "ActivationOut" in e["id"]]
    assert before and all(e["verdict"] == "pass" for e in before)


GPU_GPT = {"layers": 2, "d": 256, "heads": 8, "ff": 1024, "seq": 128, "vocab": 512}
GPU_LLAMA = {"layers": 2, "d": 256, "heads": 8, "kv_heads": 2, "ff": 768, "seq": 128, "vocab": 512, "llama": True}


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [GPU_GPT, GPU_LLAMA], ids=["gpt", "llama"])
@pytest.mark.parametrize("skip", [(), ("model.layers.1.attn",)], ids=["clean", "missing_allreduce"])
def test_live_tp2_on_gpu_feeds_check_and_check_distributed(tmp_path, skip, shape):
    """Two gloo ranks on cuda:0 run the bf16 TP model; their device-resident
    captures go to check() (union) here and to check_distributed() inside the
    job (each rank its own records); both reports equal the oracle's."""
    _gpu_live_case(tmp_path, shape, "bfloat16", skip, n_samples=3)


# config 1 as BASELINE.json names it: the 2-layer GPT-2-small shape (d=768,
# 12 heads, ff=3072, S=1024, V=50304), fp32, a TP=2 candidate against the
# single-device run, tolerances from perturbation runs (n=5, eps_p = FP32
# eps; config.py:138-141) — here both runs are live PyTorch executions.
# Unlike the reference emulator's fp32 policy (exact float64 arithmetic, so
# a TP run differs from one device by ~1e-16), a real fp32 run carries
# reduction-order round-off of its own: with cuBLAS on the B200 one id —
# ParamGrad of model.final_norm.bias, a sum over all 1024 rows whose
# response to an input nudge is only 1.4e-7 — lands at 1.43x its kappa=3
# threshold (6.0e-7 vs 4.2e-7; 0.7x on the CPU).  kappa=5 leaves every id
# of the clean run passing while the dropped all-reduce still clears its
# threshold by orders of magnitude.
CFG1 = {"layers": 2, "d": 768, "heads": 12, "ff": 3072, "seq": 1024, "vocab": 50304}


@pytest.mark.gpu
@pytest.mark.parametrize("skip", [(), ("model.layers.1.attn",)], ids=["clean", "missing_allreduce"])
def test_config1_live_gpt2_small_tp2_fp32(tmp_path, skip):
    _gpu_live_case(tmp_path, CFG1, "float32", skip, n_samples=5, kappa=5.0)


def _gpu_live_case(tmp_path, shape, dtype, skip, n_samples, kappa=3.0):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import json

    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200.canonical import ShardMapping, SliceBox, parse_canonical
    from paper_2506_09280_b200.tracestore import RankMeta, Trace, TraceRecord
    fmt = td.FloatFormat.BF16 if dtype == "bfloat16" else td.FloatFormat.FP32
    policy = "bf16" if dtype == "bfloat16" else "fp32"
    tdt = getattr(torch, dtype)
    # tolerances the reference way: responses of the single-device run to an
    # eps-nudge of the embedding output (estimate_tolerance)

    def runner(spec):
        pert = None if spec is None else \
            (lambda out, ident: td.apply_perturbation(out, ident, spec, policy=policy))
        return tp_gpt.traced_step(shape, tp_gpt.TPGroup(), device="cuda", dtype=tdt,
                                  precision=dtype, perturb=pert).trace()
    tol = td.estimate_tolerance(runner, n_samples=n_samples, eps_p=fmt.eps)
    assert max(tol.responses.values()) > 0
    ranks = run_tp(tmp_path, shape=shape, device="cuda", dtype=dtype, skip=skip, mode="distributed",
                   responses=dict(tol.responses), kappa=kappa)
    ref_h = _single_device(shape, "cuda", tdt, dtype)
    cand = Trace(header=ranks[0]["header"])
    for f in (f for r in ranks for f in r["records"]):
        pairs = tuple((SliceBox(tuple(map(tuple, l))), SliceBox(tuple(map(tuple, g)))) for l, g in f["pairs"])
        payload = torch.from_numpy(f["payload"]).to("cuda", getattr(torch, f["dtype"]))
        cand.records.append(TraceRecord(parse_canonical(f["ident"]), RankMeta(*f["rank"]),
                                        ShardMapping(tuple(f["local"]), tuple(f["global"]), pairs),
                                        f["replica"], payload, f["cls"]))
    rep = td.check(ref_h.trace(), cand, tol, kappa, fmt=fmt)
    got = json.loads(td.render_report(rep, "json"))
    want = O.check(_oracle_recs([_flat(r) for r in ref_h.records]),
                   _oracle_recs([f for r in ranks for f in r["records"]]),
                   ref_h.header(), ranks[0]["header"], dict(tol.responses), kappa, fmt.value)
    assert got["summary"] == want["summary"] and got["exit_code"] == want["exit_code"]
    assert got["earliest_divergence"] == want["earliest_divergence"]
    for g, w in zip(got["entries"], want["entries"]):
        assert (g["id"], g["verdict"]) == (w["id"], w["verdict"])
        if isinstance(w["observed"], float):
            assert abs(g["observed"] - w["observed"]) <= 1e-12 * max(abs(w["observed"]), 1e-300)
    for r in ranks:
        dist_doc = json.loads(r["report"])
        assert dist_doc["summary"] == want["summary"]
        assert [(e["id"], e["verdict"]) for e in dist_doc["entries"]] == \
            [(e["id"], e["verdict"]) for e in want["entries"]]
    if skip:
        assert want["earliest_divergence"] == BUG_SITE and want["exit_code"] == 3
        entry = next(e for e in want["entries"] if e["id"] == BUG_SITE)
        assert entry["observed"] >= 10 * max(entry["tolerance"], fmt.eps)
    else:
        bad = [(e["id"], e["observed"], e["threshold"]) for e in want["entries"] if e["verdict"] != "pass"]
        assert want["exit_code"] == 0 and want["summary"]["missing"] == 0, bad


@pytest.mark.parametrize("pcfg", [ParallelConfig(tp=2, sp=True, microbatches=2),
                                  ParallelConfig(tp=2, cp=2, microbatches=2),
                                  ParallelConfig(dp=2, tp=2, pp=2, microbatches=4),
                                  ParallelConfig(tp=4, pp=2, vp=2, microbatches=2)],
                         ids=["tp2sp", "tp2cp2", "dp2tp2pp2", "tp4pp2vp2"])
def test_layout_shard_reproduces_every_emitted_map(pcfg):
    """For every rank of SP / CP / PP / VP layouts, layout_shard answers each
    (module, kind) the layout emits for that rank with exactly the emitted
    ShardMapping, RankMeta 6-tuple and declared replica size."""
    shape = dict(SHAPE, layers=4)
    layout = Layout(tp_gpt.model_shape(shape), pcfg)
    specs = list(layout.records())
    n = 0
    for dr in range(pcfg.dp):
        for c in range(pcfg.cp):
            for t in range(pcfg.tp):
                shard = torchtap.layout_shard(layout, dp=dr, tp=t, cp=c)
                for sp in specs:
                    if (sp.rank[0], sp.rank[1], sp.rank[4]) != (dr, t, c) or sp.kind not in \
                            ("ActivationIn", "ActivationOut", "ParamGrad"):
                        continue
                    module = sp.ident.split("|mod=", 1)[1]
                    m, rank, rep = shard(module, sp.kind, torch.empty(sp.mapping.local_shape))
                    assert (m, tuple(rank), rep) == (sp.mapping, sp.rank, sp.replica), sp.ident
                    n += 1
    assert n > 100
