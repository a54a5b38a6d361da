"""Per-GPU shares of a multi-GPU check (synthetic.ShareLayout, StaticComm,
plan.compare_copies) and the batched replica digests (td_fingerprint).

CPU: every rank plans the same global job from metadata alone, the compares
of cross-GPU replica groups are spread over their holders, and each compare
holder has its reference slices.  GPU: all shares run as threads on one GPU
(the whole distributed algorithm, real kernels) and reproduce a single-GPU
check of the union of the shares — clean, and with a replica corrupted on a
GPU whose copy a compare reads (digest mismatch -> copy 0 handed over)."""

import json
import math
import threading

import numpy as np
import pytest
import torch

from paper_2506_09280_b200 import layout as L
from paper_2506_09280_b200 import synthetic
from paper_2506_09280_b200.checker import ToleranceMap
from paper_2506_09280_b200.distributed import DistributedCheckPlan, StaticComm, ThreadComm, _MetaTrace
from paper_2506_09280_b200.tensor import FloatFormat
from paper_2506_09280_b200.tracestore import Trace

SMALL = L.ModelShape(layers=2, d_model=64, n_heads=4, d_ff=128, seq_len=32, vocab=256)
PCFG = L.ParallelConfig(tp=2, dp=2, microbatches=2)
WORLD = 4


def _tol(layout):
    return ToleranceMap({i: 2 * FloatFormat.BF16.eps for i in layout.ids}, n_samples=1,
                        eps_p=FloatFormat.BF16.eps)


def test_share_plans_agree_and_balance():
    lay = synthetic.ShareLayout(SMALL, PCFG, WORLD)
    ref_metas, cand_metas = lay.metas()
    plans = []
    for r in range(WORLD):
        comm = StaticComm(r, WORLD, [ref_metas, cand_metas])
        hdr = {"digest": "x", "mode": "cascade"}
        plans.append(DistributedCheckPlan(_MetaTrace(hdr, ref_metas[r]), _MetaTrace(hdr, cand_metas[r]),
                                          _tol(lay), fmt=FloatFormat.BF16, comm=comm))
    first = plans[0]
    for p in plans[1:]:
        assert p.common == first.common
        assert len(p.plan.groups) == len(first.plan.groups)
        assert p.plan.remote_groups == first.plan.remote_groups
        assert p.plan.compare_reads == first.plan.compare_reads
    assert first.plan.remote_groups, "TP/DP replicas must span GPUs in this layout"
    assert first.plan.compare_reads, "some compares must read a copy other than copy 0"
    reads = [p.plan.algorithmic_bytes + sum(math.prod(m.shape) * 2 for m in cand_metas[r]
                                            if any(m is x for e in p.plan.remote_groups
                                                   for x in p._remote_group_records(e)))
             for r, p in enumerate(plans)]
    assert max(reads) / (sum(reads) / len(reads)) < 1.25, reads


def test_compare_copies_is_copy0_on_one_rank():
    from paper_2506_09280_b200.plan import compare_copies, merge_view
    lay = synthetic.ShareLayout(SMALL, PCFG, WORLD)
    _, cand_metas = lay.metas()
    allm = sorted([m for ms in cand_metas for m in ms], key=lambda m: m.order)
    view = merge_view(_MetaTrace({}, allm))
    assert compare_copies(view, lambda m: 0) == {}
    choice = compare_copies(view, lambda m: m.owner)
    assert choice and any(c > 0 for c in choice.values())
    for (ident, gi), c in choice.items():
        assert 0 <= c < len(view[ident].groups[gi].records)


def _run_threads(world, body):
    hub = ThreadComm.hub(world)
    out, errors = [None] * world, []

    def worker(rank):
        try:
            out[rank] = body(rank, ThreadComm(hub, rank))
        except Exception as exc:  # pragma: no cover - surfaced below
            import traceback
            errors.append(traceback.format_exc())
            hub.barrier.abort()
    threads = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    assert not errors, errors[0]
    return out


def _union(shares, header):
    """The single-process traces the shares split (global execution order)."""
    from paper_2506_09280_b200.distributed import execution_sorted
    ref, cand = Trace(header=dict(header)), Trace(header=dict(header))
    for r, c in shares:
        ref.records.extend(r.records)
        cand.records.extend(c.records)
    ref.records, cand.records = execution_sorted(ref.records), execution_sorted(cand.records)
    return ref, cand


@pytest.mark.gpu
@pytest.mark.parametrize("corrupt", [False, True])
def test_shares_as_threads_match_single_gpu_check(corrupt):
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200.checker import check
    lay = synthetic.ShareLayout(SMALL, PCFG, WORLD)
    shares = [lay.build(r) for r in range(WORLD)]
    tol = _tol(lay)
    ref_metas, cand_metas = lay.metas()
    if corrupt:
        # a replica copy that some compare reads instead of copy 0
        comm = StaticComm(0, WORLD, [ref_metas, cand_metas])
        probe = DistributedCheckPlan(_MetaTrace({"digest": "x", "mode": "cascade"}, ref_metas[0]),
                                     _MetaTrace({"digest": "x", "mode": "cascade"}, cand_metas[0]),
                                     tol, fmt=FloatFormat.BF16, comm=comm)
        ei, gi, c = probe.plan.compare_reads[0]
        meta = probe.plan.entries[ei].y.groups[gi].records[c]
        pos = meta.order[1]
        rec = shares[meta.owner][1].records[pos]
        assert rec.id.encode() == meta.id.encode()
        rec.payload.mul_(2)

    def body(rank, comm):
        ref, cand = shares[rank]
        plan = DistributedCheckPlan(ref, cand, tol, fmt=FloatFormat.BF16, comm=comm)
        return json.loads(td.render_report(plan.run(), "json"))
    reports = _run_threads(WORLD, body)
    ref_all, cand_all = _union(shares, shares[0][0].header)
    want = json.loads(td.render_report(check(ref_all, cand_all, tol, fmt=FloatFormat.BF16), "json"))
    from tests.test_gpu_parity import assert_reports_match
    for rep in reports:
        assert_reports_match(rep, want, f"corrupt={corrupt}")
    if corrupt:
        assert want["summary"]["replica-mismatch"] == 1
    else:
        assert want["summary"]["pass"] == len(want["entries"])


@pytest.mark.gpu
def test_fingerprint_digests():
    from paper_2506_09280_b200.device import Fingerprints, fingerprints
    g = torch.Generator(device="cuda").manual_seed(3)
    a = torch.randn(1 << 20, device="cuda", generator=g).to(torch.bfloat16)
    b = a.clone()
    c = a.clone()
    c.view(torch.int16)[12345] ^= 1                      # one bit
    d = torch.cat([a[1 << 19:], a[:1 << 19]])            # halves swapped (same multiset)
    e = a.view(torch.uint8)[3:3 + 1000003]               # unaligned, odd length
    f = e.clone()
    z = a[:0]
    out = fingerprints([a, b, c, d, e, f, z]).cpu().numpy()
    assert np.array_equal(out[0], out[1])
    assert not np.array_equal(out[0], out[2])
    assert not np.array_equal(out[0], out[3])
    assert np.array_equal(out[4], out[5])                # aligned copy == unaligned view
    assert np.array_equal(out[6], [0, 0])
    # one launch over many items == item by item; replays are deterministic
    parts = [a[k * 1000:(k + 1) * 1000 + 7] for k in range(50)]
    fp = Fingerprints(parts)
    many = fp.run().cpu().numpy()
    again = fp.run().cpu().numpy()
    one = np.stack([fingerprints([p]).cpu().numpy()[0] for p in parts])
    assert np.array_equal(many, one) and np.array_equal(many, again)


@pytest.mark.gpu
def test_digests_fused_in_compare_equal_fingerprints():
    """The digest slots td_segnorm fills while comparing a cross-GPU replica
    group's copy equal td_fingerprint's digest of that copy, and the digest
    rows land in the exchange buffer at the canonical offsets td_combine
    reads (identical on every rank)."""
    from paper_2506_09280_b200.device import fingerprints
    lay = synthetic.ShareLayout(SMALL, PCFG, WORLD)
    ref_metas, cand_metas = lay.metas()
    fused_total = 0
    offsets = None
    for r in range(WORLD):
        ref, cand = lay.build(r)
        dcp = DistributedCheckPlan(ref, cand, _tol(lay), fmt=FloatFormat.BF16,
                                   comm=StaticComm(r, WORLD, [ref_metas, cand_metas]))
        if offsets is None:
            offsets = (dcp.stride, dcp.group_begin, dcp.copy_first.tolist())
        assert (dcp.stride, dcp.group_begin, dcp.copy_first.tolist()) == offsets
        b = dcp.bind()
        b.step()
        torch.cuda.synchronize()
        got = b.local_digests()
        recs = [dcp._remote_group_records(dcp.plan.remote_groups[k])[c].device_payload().reshape(-1)
                for k, c in dcp.where]
        want = fingerprints(recs).cpu().numpy().view(np.uint64)
        for i, kc in enumerate(dcp.where):
            assert got[kc] == (int(want[i, 0]), int(want[i, 1])), (r, kc)
        # canonical rows in the exchange tail (this rank is row 0 of a one-rank gather)
        tail = b.prep.exchange[dcp.n_slots:].view(torch.int64).view(-1, 2).cpu().numpy().view(np.uint64)
        for i, row in enumerate(dcp.canon_rows):
            assert (int(tail[row, 0]), int(tail[row, 1])) == got[dcp.where[i]]
        fused_total += dcp.n_fused
    assert fused_total > 0


@pytest.mark.gpu
def test_fuzzed_shares_match_single_gpu_check():
    """A slice of tools/fuzz_distributed.py: random layouts split into 2-4
    shares run as threads (digests, balanced compares, copy-0 handover), with
    random corruptions — every rank's report == check() of the union."""
    import os
    import random
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import fuzz_distributed
    rnd = random.Random(77)
    for k in range(12):
        fuzz_distributed.run_case(rnd, k)


def _digest_numpy(data: bytes):
    """CPU restatement of the td_fingerprint digest (td_kernels.cu, fp_key_word):
    8-byte little-endian words w_j (tail zero-padded), lane j % 2:
    z_j = (w_j ^ (j+1)*gamma) * M[j % 2], h[j % 2] = sum z_j ^ (z_j >> 32)
    mod 2^64, M = (MIX1, MIX2)."""
    pad = (-len(data)) % 8
    w = np.frombuffer(data + b"\0" * pad, dtype="<u8")
    with np.errstate(over="ignore"):
        j = np.arange(1, len(w) + 1, dtype=np.uint64)
        z = w ^ (j * np.uint64(0x9E3779B97F4A7C15))
        z0 = z[0::2] * np.uint64(0xBF58476D1CE4E5B9)
        z1 = z[1::2] * np.uint64(0x94D049BB133111EB)
        h0 = np.sum(z0 ^ (z0 >> np.uint64(32)), dtype=np.uint64)
        h1 = np.sum(z1 ^ (z1 >> np.uint64(32)), dtype=np.uint64)
    return int(h0), int(h1)


@pytest.mark.gpu
def test_fingerprint_matches_numpy_restatement():
    """td_fingerprint bit-exact against a numpy restatement of the digest, over
    random lengths (multi-chunk, odd tails) and byte offsets (unaligned)."""
    from paper_2506_09280_b200.device import fingerprints
    rng = np.random.default_rng(3)
    blob = torch.from_numpy(rng.integers(0, 256, (3 << 20) + 77, dtype=np.uint8)).cuda()
    host = blob.cpu().numpy().tobytes()
    views, want = [], []
    for _ in range(40):
        off = int(rng.integers(0, 64))
        n = int(rng.choice([0, 1, 7, 8, 15, 16, 17, 1000, (1 << 18) + 3, (1 << 20) + 5, 3 << 20]))
        n = min(n, len(host) - off)
        views.append(blob[off:off + n])
        want.append(_digest_numpy(host[off:off + n]))
    got = fingerprints(views).cpu().numpy().view(np.uint64)
    for g, w in zip(got, want):
        assert (int(g[0]), int(g[1])) == w
    # an equal-and-opposite change of two same-lane words (one bit set in
    # word 0 and cleared in word 2, where their position keys agree): a
    # plain sum of (w ^ k) * M cannot tell the copies apart, the folded
    # digest must
    a, b = _same_lane_swap_pair()
    da, db = fingerprints([torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()]).cpu().numpy().view(np.uint64)
    assert tuple(da) != tuple(db)


def _same_lane_swap_pair():
    gamma = 0x9E3779B97F4A7C15
    k0, k2 = gamma, (3 * gamma) & ((1 << 64) - 1)
    bit = next(i for i in range(64) if ((k0 ^ k2) >> i) & 1 == 0)
    words = np.random.default_rng(5).integers(0, 1 << 62, 8, dtype=np.uint64)
    a, b = words.copy(), words.copy()
    m = np.uint64(1 << bit)
    a[0], a[2] = a[0] | m, a[2] & ~m
    b[0], b[2] = b[0] & ~m, b[2] | m
    return a.view(np.uint8), b.view(np.uint8)


def test_digest_restatement_separates_a_same_lane_swap():
    """The additive-checksum weakness the fold removes (td_kernels.cu,
    fp_key_word), shown on the numpy restatement."""
    a, b = _same_lane_swap_pair()
    with np.errstate(over="ignore"):
        def linear(x):
            w = x.view(np.uint64)
            j = np.arange(1, len(w) + 1, dtype=np.uint64)
            return int(np.sum((w ^ (j * np.uint64(0x9E3779B97F4A7C15)))[0::2] * np.uint64(0xBF58476D1CE4E5B9),
                              dtype=np.uint64))
        assert linear(a) == linear(b)
    assert _digest_numpy(a.tobytes()) != _digest_numpy(b.tobytes())


# config 4's layout (Llama-3-8B rules: L=32, GQA 32/8, SwiGLU w3, RMSNorm, no
# position table; TP=2 x DP=4, M=4, 8 GPUs) at a width that fits all eight
# shares plus the single-GPU union check on one device (d=1024, ff=3584,
# V=32000, S=256 — the parameter-sized ids do not shrink with S)
CFG4_SHAPE = L.ModelShape(layers=32, d_model=1024, n_heads=32, d_ff=3584, seq_len=256, vocab=32000,
                          n_kv_heads=8, gated_mlp=True, norm_bias=False, position_table=False)
CFG4_PCFG = L.ParallelConfig(tp=2, dp=4, microbatches=4)


@pytest.mark.gpu
def test_config4_layout_eight_shares_match_single_gpu_and_oracle():
    """All 8 TP2 x DP4 shares of a config-4-layout check run as ThreadComm
    ranks on one GPU (one all-gather per check, device digest compare), with
    a swapped TP shard (the reference's wrong-order bug: a flag) and one
    corrupted DP replica of a parameter (a cross-GPU digest mismatch: the
    exact bug path, replica-mismatch).  Every rank's report equals a
    single-GPU check() of the union of the shares, and a sample of ids —
    the buggy ones included — equals the CPU oracle's report."""
    import paper_2506_09280_b200 as td
    from oracle import traindiff_oracle as O
    from paper_2506_09280_b200.checker import check
    swapped = "iter=0|mb=1|kind=ParamGrad|mod=model.layers.5.mlp.w1"
    lay = synthetic.ShareLayout(CFG4_SHAPE, CFG4_PCFG, 8)
    shares = [lay.build(r, bugs={swapped: "order"}) for r in range(8)]
    tol = _tol(lay)
    # a DP replica (copy 2 of a column-parallel parameter shard) corrupted
    victim = "iter=0|mb=0|kind=Param|mod=model.layers.20.attn.wk"
    hits = [(r, k) for r, (_, c) in enumerate(shares) for k, rec in enumerate(c.records)
            if rec.id.encode() == victim and rec.rank_meta.dp == 2 and rec.rank_meta.tp == 1]
    assert len(hits) == 1
    r, k = hits[0]
    shares[r][1].records[k].payload.view(torch.int16)[7] ^= 0x40

    def body(rank, comm):
        ref, cand = shares[rank]
        plan = DistributedCheckPlan(ref, cand, tol, fmt=FloatFormat.BF16, comm=comm)
        assert plan.plan.remote_groups
        return json.loads(td.render_report(plan.run(), "json"))
    reports = _run_threads(8, body)
    ref_all, cand_all = _union(shares, shares[0][0].header)
    want = json.loads(td.render_report(check(ref_all, cand_all, tol, fmt=FloatFormat.BF16), "json"))
    from tests.test_gpu_parity import assert_reports_match
    for rep in reports:
        assert_reports_match(rep, want, "config-4 layout, 8 shares")
    verdicts = {e["id"]: e["verdict"] for e in want["entries"]}
    assert verdicts[swapped] == "flag" and verdicts[victim] == "replica-mismatch"
    assert want["summary"]["flag"] == 1 and want["summary"]["replica-mismatch"] == 1
    assert want["summary"]["pass"] == len(want["entries"]) - 2
    # the CPU oracle on a sample of ids (every 97th, plus the two bugs)
    ids = [e["id"] for e in want["entries"]]
    sample = set(ids[::97]) | {swapped, victim}

    def host(recs):
        return [O.Rec(x.id.encode(), x.rank_meta.as_tuple(), x.mapping.local_shape, x.mapping.global_shape,
                      [(lb.bounds, gb.bounds) for lb, gb in x.mapping.pairs], x.replica_group_size,
                      x.payload.float().cpu().numpy()) for x in recs if x.id.encode() in sample]
    doc = O.check(host(ref_all.records), host(cand_all.records), ref_all.header, cand_all.header,
                  tol.responses, 3.0, "BF16")
    got = {e["id"]: e for e in reports[0]["entries"]}
    assert {e["id"] for e in doc["entries"]} == sample
    for w in doc["entries"]:
        g = got[w["id"]]
        assert g["verdict"] == w["verdict"] and g["detail"] == w["detail"], (w["id"], g, w)
        from tests.test_gpu_parity import _close
        assert _close(g["observed"], w["observed"]), (w["id"], g["observed"], w["observed"])


@pytest.mark.gpu
def test_distributed_clean_step_replays_as_one_cuda_graph():
    """The multi-GPU clean path (digests fused in the compare pass and by
    td_fingerprint on a side stream, td_segnorm, slot reduction, the
    exchange, td_combine, td_verdict) has no host synchronisation, so one
    GPU's share of a config-4-layout job captures into ONE CUDA graph;
    replays give the eager step's verdicts, sums and digest table bit for
    bit."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_09280_b200.distributed import StaticComm
    lay = synthetic.ShareLayout(CFG4_SHAPE, CFG4_PCFG, 8)
    ref, cand = lay.build(0)
    rm, cm = lay.metas()
    plan = DistributedCheckPlan(ref, cand, _tol(lay), fmt=FloatFormat.BF16, comm=StaticComm(0, 8, [rm, cm]))
    assert plan.plan.remote_groups and plan.plan.fused_digests
    b = plan.bind()
    b.step()
    idres, gres, ties, n_diff = b.fetch()
    digests = b.local_digests()
    sums = b.prep.slot_sums.clone()
    graph = b.capture()
    for _ in range(3):
        b.prep.slot_sums.zero_()
        graph.replay()
        torch.cuda.synchronize()
        idres2, gres2, ties2, n_diff2 = b.fetch()
        assert idres2.tobytes() == idres.tobytes() and gres2.tobytes() == gres.tobytes()
        assert (ties2, n_diff2) == (ties, n_diff) == (0, 0)
        assert torch.equal(b.prep.slot_sums, sums)
        assert b.local_digests() == digests


@pytest.mark.gpu
@pytest.mark.parametrize("corrupt", [False, True])
def test_graph_step_around_eager_collective_matches_eager_step(corrupt):
    """BoundCheck.capture_parts (what bench.py --gpus N replays): the
    clean-path step as a graph before the all-gather and one after it, the
    collective eager between them — every rank's verdicts, sums and
    digest-mismatch count equal the eager step's, step after step, and the
    bug path run after a replay gives the eager bug path's results."""
    lay = synthetic.ShareLayout(SMALL, PCFG, WORLD)
    shares = [lay.build(r) for r in range(WORLD)]
    if corrupt:
        rec = next(r for r in shares[WORLD - 1][1].records if r.replica_group_size > 1)
        rec.payload.mul_(2)
    tol = _tol(lay)
    lock = threading.Lock()

    def body(rank, comm):
        ref, cand = shares[rank]
        dcp = DistributedCheckPlan(ref, cand, tol, fmt=FloatFormat.BF16, comm=comm)
        b = dcp.bind()
        b.step()
        idres, gres, ties, n_diff = b.fetch()
        sums = b.prep.slot_sums.clone()
        want = dcp._bug_path(b) if n_diff else (idres, gres, ties)
        comm.hub.barrier.wait()
        with lock:                     # one capture at a time: no other thread's CUDA work meanwhile
            torch.cuda.synchronize()
            g = b.capture_parts()
            torch.cuda.synchronize()
        comm.hub.barrier.wait()
        for _ in range(2):
            b.prep.slot_sums.zero_()
            g.replay()
            idres2, gres2, ties2, n_diff2 = b.fetch()
            assert (idres2.tobytes(), gres2.tobytes(), ties2, n_diff2) == \
                (idres.tobytes(), gres.tobytes(), ties, n_diff)
            assert torch.equal(b.prep.slot_sums, sums)
            got = dcp._bug_path(b) if n_diff2 else (idres2, gres2, ties2)
            assert got[0].tobytes() == want[0].tobytes() and got[1].tobytes() == want[1].tobytes()
        return int(n_diff), int((want[0]["verdict"] == 2).sum())
    out = _run_threads(WORLD, body)
    if corrupt:
        assert all(n > 0 for n, _ in out) and all(m == 1 for _, m in out)
    else:
        assert out == [(0, 0)] * WORLD
