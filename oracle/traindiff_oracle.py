"""CPU oracle for the tensor-comparison hot path — TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithm (TTrace `traindiff`,
/root/reference/pkg/src/traindiff), written independently of the product
package so it can check it.  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg may import this module; the
product path (paper_2506_09280_b200) never does.

Parity pinning: tests/test_oracle.py checks this oracle against the golden
fixtures that tests/golden/make_golden.py produced by running the reference
itself (report JSON byte-identical on every scenario, tolerance JSON
byte-identical, every RNG / quantizer / merge-witness vector equal).

Each function cites the reference lines it restates.  The arithmetic
follows the reference's operation order on float64 (numpy pairwise sums),
which is what makes its timing a faithful CPU baseline as well.
"""

from __future__ import annotations

import fnmatch
import gzip
import json
import math
import struct

import numpy as np

M64 = (1 << 64) - 1

# ---------------------------------------------------------------------------
# RNG (generation.py:36-78, 163-167)


def fnv1a64(data: bytes) -> int:
    """generation.py:36-40"""
    h = 0xCBF29CE484222325
    for b in data:
        h = ((h ^ b) * 0x100000001B3) & M64
    return h


def seed_of(tag: str) -> int:
    """generation.py:43-46"""
    return fnv1a64(tag.encode("utf-8"))


def splitmix_words(seed: int, k0: int, n: int) -> np.ndarray:
    """Words k0..k0+n-1: mix(seed + (k+1)*gamma) (generation.py:67-73)."""
    with np.errstate(over="ignore"):
        k = np.arange(k0 + 1, k0 + n + 1, dtype=np.uint64)
        z = np.uint64(seed & M64) + k * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def philox_words(seed: int, k0: int, n: int) -> np.ndarray:
    """Philox4x32-10 keyed by the seed; block b = Philox(counter = b) gives
    word 2b = (out1:out0) and word 2b+1 = (out3:out2).  The opt-in generator
    (not in the reference; restated here so the device stream is checked)."""
    k = np.arange(k0, k0 + n, dtype=np.uint64)
    lane = k & np.uint64(1)
    blk = k >> np.uint64(1)
    c0 = (blk & np.uint64(0xFFFFFFFF)).astype(np.uint64)
    c1 = (blk >> np.uint64(32)).astype(np.uint64)
    c2 = np.zeros_like(c0)
    c3 = np.zeros_like(c0)
    k0_ = np.uint64(seed & 0xFFFFFFFF)
    k1_ = np.uint64((seed >> 32) & 0xFFFFFFFF)
    m32 = np.uint64(0xFFFFFFFF)
    for _ in range(10):
        p0 = np.uint64(0xD2511F53) * c0
        p1 = np.uint64(0xCD9E8D57) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & m32
        hi1, lo1 = p1 >> np.uint64(32), p1 & m32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ k0_) & m32, lo1, (hi0 ^ c3 ^ k1_) & m32, lo0
        k0_ = (k0_ + np.uint64(0x9E3779B9)) & m32
        k1_ = (k1_ + np.uint64(0xBB67AE85)) & m32
    return np.where(lane == 0, (c1 << np.uint64(32)) | c0, (c3 << np.uint64(32)) | c2)


def signed_uniforms(seed: int, n: int, k0: int = 0, generator: str = "splitmix64") -> np.ndarray:
    """2u - 1 with u = (w >> 11) * 2^-53 (generation.py:74-78, 163-167)."""
    w = splitmix_words(seed, k0, n) if generator == "splitmix64" else philox_words(seed, k0, n)
    u = (w >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return 2.0 * u - 1.0


# ---------------------------------------------------------------------------
# numerics (tensor.py:28-77, 144-167)

FORMATS = {"FP32": (24, float(np.finfo(np.float32).max)),
           "BF16": (8, 1.9921875 * 2.0 ** 127),
           "FP8E4M3": (4, 448.0)}


def eps_of(fmt: str) -> float:
    return 2.0 ** -FORMATS[fmt][0]


def quantize(x, fmt: str) -> np.ndarray:
    """RNE to p bits, unbounded exponent, clip (tensor.py:64-77)."""
    x = np.asarray(x, dtype=np.float64)
    if not np.isfinite(x).all():
        raise FloatingPointError("quantize input contains NaN or infinity")
    p, maxf = FORMATS[fmt]
    m, e = np.frexp(x)
    return np.clip(np.ldexp(np.rint(np.ldexp(m, p)), e - p), -maxf, maxf)


def rel_err(a, b) -> float:
    """||a-b|| / ||a|| with 0/0 -> 0, x/0 -> inf (tensor.py:158-167)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError(f"rel_err: {a.shape} vs {b.shape}")
    diff = float(np.sqrt(np.sum(np.square(a - b))))
    ref = float(np.sqrt(np.sum(np.square(a))))
    if ref == 0.0:
        return 0.0 if diff == 0.0 else float("inf")
    return diff / ref


def perturb(x, tag: str, eps: float, positions, full_cols: int, fmt: str | None,
            generator: str = "splitmix64") -> np.ndarray:
    """Emulator._apply_perturbation (engine.py:351-361) on a rank's rows."""
    x = np.asarray(x, dtype=np.float64)
    rows, cols = x.shape
    pos = np.asarray(positions, dtype=np.int64)
    n_rows = int(pos.max()) + 1 if len(pos) else 0
    u = signed_uniforms(seed_of(tag), n_rows * full_cols, 0, generator).reshape(n_rows, full_cols)
    y = x * (1.0 + u[pos, :cols] * eps)
    return quantize(y, fmt) if fmt is not None else y


# ---------------------------------------------------------------------------
# records and geometry (canonical.py:93-247, tracestore.py:51-94)


class Rec:
    """One trace record: id string, rank tuple, mapping, replica size, f32 payload."""

    __slots__ = ("ident", "rank", "local_shape", "global_shape", "pairs", "replica",
                 "payload", "module_class")

    def __init__(self, ident, rank, local_shape, global_shape, pairs, replica, payload,
                 module_class=""):
        self.ident = ident
        self.rank = tuple(rank)
        self.local_shape = tuple(local_shape)
        self.global_shape = tuple(global_shape)
        self.pairs = tuple((tuple(map(tuple, l)), tuple(map(tuple, g))) for l, g in pairs)
        self.replica = int(replica)
        self.payload = np.ascontiguousarray(payload, dtype=np.float32)
        self.module_class = module_class


def _sl(bounds):
    return tuple(slice(a, b) for a, b in bounds)


def _ext(bounds):
    return tuple(b - a for a, b in bounds)


def validate_mapping(local_shape, global_shape, pairs):
    """Error message or None (canonical.py:153-179), via a count array."""
    if not pairs:
        return "mapping has no slice pairs"
    for l, g in pairs:
        if len(l) != len(local_shape) or len(g) != len(global_shape):
            return "box rank differs from shape rank"
        if _ext(l) != _ext(g):
            return f"extent mismatch: local {_ext(l)} vs global {_ext(g)}"
        if not all(b <= n for (_, b), n in zip(l, local_shape)):
            return f"local box {l} exceeds {tuple(local_shape)}"
        if not all(b <= n for (_, b), n in zip(g, global_shape)):
            return f"global box {g} exceeds {tuple(global_shape)}"
    counts = np.zeros(local_shape, dtype=np.int32)
    for l, _ in pairs:
        counts[_sl(l)] += 1
    if (counts > 1).any():
        where = np.argwhere(counts > 1)[0]
        return f"local boxes overlap at {tuple(int(i) for i in where)}"
    return None


def merge(shards, global_shape):
    """(merged f64, None) or (None, (kind, message, witness)) (canonical.py:182-212).
    shards: [(local_shape, pairs, data)]."""
    global_shape = tuple(global_shape)
    out = np.zeros(global_shape, dtype=np.float64)
    counts = np.zeros(global_shape, dtype=np.int32)
    for local_shape, pairs, data in shards:
        msg = validate_mapping(local_shape, global_shape, pairs)
        if msg is not None:
            return None, ("MappingInvalid", msg, None)
        if tuple(data.shape) != tuple(local_shape):
            return None, ("ShapeMismatch",
                          f"shard shape {tuple(data.shape)} != mapping local shape {tuple(local_shape)}", None)
        for l, g in pairs:
            out[_sl(g)] = data[_sl(l)]
            counts[_sl(g)] += 1
    if (counts != 1).any():
        over = np.argwhere(counts > 1)
        if len(over):
            w = tuple(int(i) for i in over[0])
            return None, ("MergeConflict", f"shards overlap at global index {w}", w)
        w = tuple(int(i) for i in np.argwhere(counts == 0)[0])
        return None, ("MergeConflict", f"no shard covers global index {w}", w)
    return out, None


def replica_problem(copies, eps: float):
    """check_replicas (canonical.py:225-247): message or None."""
    if len(copies) <= 1:
        return None
    base = copies[0]
    worst, worst_rank = 0.0, None
    for rank, c in enumerate(copies[1:], start=1):
        err = rel_err(base, c)
        if err > worst:
            worst, worst_rank = err, rank
    if worst > eps:
        return f"replicas diverge: rel_err {worst:.6g} between ranks 0 and {worst_rank}"
    return None


def merge_one(recs, eps: float, replica_check: bool = True):
    """_merge_one (checker.py:151-198) -> dict(values, problem, detail)."""
    out = {"values": None, "problem": None, "detail": ""}
    if len({len(r.global_shape) for r in recs}) != 1:
        out["problem"], out["detail"] = "merge-error", "records disagree on tensor rank"
        return out
    ndim = len(recs[0].global_shape)
    hull = tuple(max(r.global_shape[a] for r in recs) for a in range(ndim))
    groups = {}
    for r in recs:
        groups.setdefault((r.local_shape, r.pairs), []).append(r)
    problems = []
    if replica_check:
        for g in groups.values():
            declared = {r.replica for r in g}
            if declared != {len(g)}:
                problems.append(("replica-mismatch", f"{len(g)} copies of one shard, declared "
                                                      f"replica group size {sorted(declared)}"))
                continue
            msg = replica_problem([r.payload.astype(np.float64) for r in g], eps)
            if msg is not None:
                problems.append(("replica-mismatch", msg))
    values, err = merge([(g[0].local_shape, g[0].pairs, g[0].payload.astype(np.float64))
                         for g in groups.values()], hull)
    out["values"] = values
    if err is not None:
        problems.append(("merge-error", err[1]))
    if problems:
        out["problem"], out["detail"] = problems[0]
    return out


def by_id(records):
    groups = {}
    for k, r in enumerate(records):
        groups.setdefault(r.ident, []).append((k, r))
    return groups


def merge_trace(records, eps: float, replica_check: bool = True, strict: bool = False):
    """_merge_trace (checker.py:201-211)."""
    view = {}
    for ident, entries in by_id(records).items():
        entries = sorted(entries, key=lambda p: p[0])
        m = merge_one([r for _, r in entries], eps, replica_check)
        m["exec"] = entries[0][0]
        if strict and m["problem"] is not None:
            raise RuntimeError(f"{ident}: {m['detail']}")
        view[ident] = m
    return view


# ---------------------------------------------------------------------------
# checker (checker.py:221-365, 446-489)

VERDICTS = ("pass", "flag", "replica-mismatch", "merge-error", "missing")


def _jsonable(v):
    if v is None:
        return None
    if not math.isfinite(v):
        return "inf" if v > 0 else ("-inf" if v < 0 else "nan")
    return v


def check(ref_records, cand_records, ref_header, cand_header, responses: dict, kappa: float,
          fmt: str) -> dict:
    """checker.check -> the report's to_dict() (checker.py:299-309, 312-365)."""
    for key in ("digest", "mode"):
        if ref_header.get(key) != cand_header.get(key):
            raise ValueError(f"traces disagree on {key}")
    eps = eps_of(fmt)
    ref_view = merge_trace(ref_records, eps)
    cand_view = merge_trace(cand_records, eps)
    entries = []
    for ident, got in cand_view.items():
        tol = responses.get(ident, 0.0)
        thr = kappa * max(tol, eps)
        want = ref_view.get(ident)
        if want is None:
            entries.append((ident, "missing", None, tol, thr, "only in candidate trace"))
            continue
        obs = None
        if got["values"] is not None and want["values"] is not None \
                and got["values"].shape == want["values"].shape:
            obs = rel_err(want["values"], got["values"])
        if got["problem"] is not None:
            verdict, detail = got["problem"], got["detail"]
        elif want["problem"] is not None:
            verdict, detail = want["problem"], f"reference side: {want['detail']}"
        elif obs is None:
            verdict = "merge-error"
            detail = (f"merged shapes differ: reference {want['values'].shape} vs candidate "
                      f"{got['values'].shape}")
        else:
            verdict, detail = ("flag" if obs > thr else "pass"), ""
        entries.append((ident, verdict, obs, tol, thr, detail))
    for ident in ref_view:
        if ident not in cand_view:
            tol = responses.get(ident, 0.0)
            entries.append((ident, "missing", None, tol, kappa * max(tol, eps), "only in reference trace"))
    counts = {v: 0 for v in VERDICTS}
    for e in entries:
        counts[e[1]] += 1
    first = lambda vs: next((e[0] for e in entries if e[1] in vs), None)  # noqa: E731
    exit_code = 3 if counts["replica-mismatch"] or counts["merge-error"] else (2 if counts["flag"] else 0)
    return {"report_version": 1, "kind": "check", "mode": str(cand_header.get("mode", "")),
            "kappa": kappa, "format": fmt, "summary": counts,
            "earliest_flag": first(("flag",)),
            "earliest_divergence": first(("flag", "replica-mismatch", "merge-error")),
            "exit_code": exit_code,
            "entries": [{"id": i, "verdict": v, "observed": _jsonable(o), "tolerance": _jsonable(t),
                         "threshold": _jsonable(h), "detail": d} for i, v, o, t, h, d in entries]}


def report_json(doc: dict) -> str:
    return json.dumps(doc, sort_keys=True, separators=(",", ":"))


def estimate_tolerance(traces, n_samples: int, eps_p: float, aggregation: str = "max") -> dict:
    """checker.estimate_tolerance (checker.py:102-138) over pre-recorded runs:
    traces[0] is runner(None), traces[1 + s] is runner(PerturbSpec(s, eps_p))."""
    base = merge_trace(traces[0], eps_of("FP32"), strict=True)
    samples = {i: [] for i in base}
    for s in range(n_samples):
        pert = merge_trace(traces[1 + s], eps_of("FP32"), strict=True)
        for ident, entry in base.items():
            moved = pert.get(ident)
            if moved is None:
                continue
            r = rel_err(entry["values"], moved["values"])
            samples[ident].append(r if math.isfinite(r) else 0.0)
    responses = {}
    for ident, rs in samples.items():
        if not rs:
            responses[ident] = 0.0
        elif aggregation == "max":
            responses[ident] = max(rs)
        else:
            responses[ident] = sum(rs) / len(rs)
    return {"tolerance_version": 1, "n_samples": n_samples, "eps_p": eps_p,
            "aggregation": aggregation, "responses": responses}


def compare_static(ref_records, cand_records, atol: float, rtol: float) -> list:
    """compare_static's verdicts (checker.py:403-443): [(id, verdict)]."""
    ref_view = merge_trace(ref_records, 0.0, replica_check=False)
    cand_view = merge_trace(cand_records, 0.0, replica_check=False)
    out = []
    for ident, got in cand_view.items():
        want = ref_view.get(ident)
        if want is None:
            out.append((ident, "missing"))
        elif got["problem"] is not None or want["problem"] is not None:
            out.append((ident, "merge-error"))
        elif want["values"].shape != got["values"].shape:
            out.append((ident, "merge-error"))
        else:
            close = np.abs(got["values"] - want["values"]) <= atol + rtol * np.abs(want["values"])
            out.append((ident, "pass" if bool(close.all()) else "flag"))
    for ident in ref_view:
        if ident not in cand_view:
            out.append((ident, "missing"))
    return out


# ---------------------------------------------------------------------------
# TTRC reader (tracestore.py:225-284), independent of the product's reader


def read_ttrc(data: bytes):
    """(header dict, [Rec]) from TTRC bytes (gzip accepted)."""
    if data[:2] == b"\x1f\x8b":
        data = gzip.decompress(data)
    assert data[:4] == b"TTRC"
    _, _, hlen = struct.unpack_from("<HHI", data, 4)
    pos = 12
    header = json.loads(data[pos:pos + hlen])
    pos += hlen
    recs = []
    while data[pos:] != b"CRTT":
        (_, id_len) = struct.unpack_from("<BI", data, pos)
        pos += 5
        ident = data[pos:pos + id_len].decode()
        pos += id_len
        rank = struct.unpack_from("<6H", data, pos)
        pos += 12
        (replica, cls_len) = struct.unpack_from("<HI", data, pos)
        pos += 6
        cls = data[pos:pos + cls_len].decode()
        pos += cls_len
        (_, ndim) = struct.unpack_from("<BB", data, pos)
        pos += 2
        dims = struct.unpack_from(f"<{ndim}Q", data, pos)
        pos += 8 * ndim
        (npairs,) = struct.unpack_from("<H", data, pos)
        pos += 2
        pairs = []
        for _ in range(npairs):
            flat = struct.unpack_from(f"<{4 * ndim}Q", data, pos)
            pos += 32 * ndim
            g = tuple((flat[2 * a], flat[2 * a + 1]) for a in range(ndim))
            l = tuple((flat[2 * ndim + 2 * a], flat[2 * ndim + 2 * a + 1]) for a in range(ndim))
            pairs.append((l, g))
        (plen,) = struct.unpack_from("<Q", data, pos)
        pos += 8
        payload = np.frombuffer(data, dtype="<f4", count=plen // 4, offset=pos).reshape(dims)
        pos += plen
        hull = tuple(max(g[a][1] for _, g in pairs) for a in range(ndim))
        recs.append(Rec(ident, rank, dims, hull, pairs, replica, payload, cls))
    return header, recs


def trace_filter(recs, patterns=(), kinds=()):
    """TraceFilter.admits (tracestore.py:116-130)."""
    out = []
    for r in recs:
        kind = r.ident.split("|")[2][len("kind="):]
        mod = r.ident.split("|", 3)[3][len("mod="):]
        if kinds and kind not in kinds:
            continue
        if patterns and not any(fnmatch.fnmatchcase(mod, p) for p in patterns):
            continue
        out.append(r)
    return out
