"""Differential fuzzing of the check's error and edge paths: random layouts
(fuzz_parity.random_case), then 1-3 random structural or numeric faults
injected into the reference or the candidate trace:

  drop_record   a record removed (a shard gap, or a replica copy short of
                its declared group size)
  drop_id       every record of an id removed (only in the other trace)
  extra_id      a record copied under a new module name (only in this trace)
  dup_copy      one more copy of a record (beyond its declared group size),
                bit-identical or perturbed
  declared      a record's declared replica group size changed
  shift_box     a shard's global box moved onto a sibling shard's box of the
                same extent (overlap + gap)
  grow_hull     a record's global shape enlarged (hull mismatch / gap)
  flatten       a record re-declared as a 1-D identity shard of its payload
                (records disagree on tensor rank / merged shapes differ)
  special       one element set to NaN, +inf or -inf (replica copies, the
                compare's strict `>` and NaN handling)
  zero          a payload zeroed (zero reference norm)

Every case: td.check's report on the device traces == the CPU oracle's on
host copies (verdicts, details, thresholds exact; observed within 1e-12,
NaN == NaN), or both raise; about a third of the cases also compare
td.compare_static's verdicts with the oracle's on the same traces.

    python tools/fuzz_faults.py [--cases 500] [--seed 0]      (GPU)
"""

import argparse
import collections
import json
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

FAULTS = ("drop_record", "drop_id", "extra_id", "dup_copy", "declared", "shift_box", "grow_hull",
          "flatten", "special", "zero")


def inject(rnd, trace, fault):
    """Apply one fault in place; returns a short description or None."""
    import torch
    from paper_2506_09280_b200.canonical import ShardMapping, identity_mapping, parse_canonical
    from paper_2506_09280_b200.tracestore import RankMeta, TraceRecord
    recs = trace.records
    if not recs:
        return None
    k = rnd.randrange(len(recs))
    r = recs[k]
    if fault == "drop_record":
        del recs[k]
        return f"drop {r.id.encode()} {r.rank_meta.as_tuple()}"
    if fault == "drop_id":
        ident = r.id.encode()
        trace.records = [x for x in recs if x.id.encode() != ident]
        return f"drop_id {ident}"
    if fault == "extra_id":
        new = parse_canonical(r.id.encode().rsplit("mod=", 1)[0] + f"mod=fuzz.extra{k}")
        recs.insert(rnd.randrange(len(recs) + 1), TraceRecord(new, r.rank_meta, r.mapping, r.replica_group_size,
                                                             r.payload.clone(), r.module_class))
        return f"extra {new.encode()}"
    if fault == "dup_copy":
        p = r.payload.clone()
        if rnd.random() < 0.5 and p.numel():
            p.view(-1)[rnd.randrange(p.numel())] *= 2
        rm = r.rank_meta
        recs.insert(k + 1, TraceRecord(r.id, RankMeta(rm.dp + 7, rm.tp, rm.pp, rm.vp, rm.cp, rm.sp), r.mapping,
                                       r.replica_group_size, p, r.module_class))
        return f"dup {r.id.encode()}"
    if fault == "declared":
        r.replica_group_size = rnd.choice([x for x in (1, 2, 3, 4) if x != r.replica_group_size])
        return f"declared {r.id.encode()} -> {r.replica_group_size}"
    if fault == "shift_box":
        ident = r.id.encode()
        sib = [x for x in recs if x.id.encode() == ident and x is not r
               and x.mapping.local_shape == r.mapping.local_shape and len(x.mapping.pairs) == 1
               and len(r.mapping.pairs) == 1 and x.mapping.pairs_bounds != r.mapping.pairs_bounds]
        if not sib:
            return None
        s = rnd.choice(sib)
        r.mapping = ShardMapping(r.mapping.local_shape, r.mapping.global_shape, s.mapping.pairs)
        return f"shift {ident}"
    if fault == "grow_hull":
        g = list(r.mapping.global_shape)
        if not g:
            return None
        a = rnd.randrange(len(g))
        g[a] += rnd.choice([1, 8])
        r.mapping = ShardMapping(r.mapping.local_shape, tuple(g), r.mapping.pairs)
        return f"grow {r.id.encode()} axis {a}"
    if fault == "flatten":
        p = r.payload.reshape(-1).clone()
        recs[k] = TraceRecord(r.id, r.rank_meta, identity_mapping(tuple(p.shape)), r.replica_group_size, p,
                              r.module_class)
        return f"flatten {r.id.encode()}"
    if fault == "special":
        if not r.payload.numel():
            return None
        v = rnd.choice([float("nan"), float("inf"), float("-inf")])
        p = r.payload.clone()
        p.view(-1)[rnd.randrange(p.numel())] = v
        r.payload = p
        return f"special {r.id.encode()} {v}"
    if fault == "zero":
        r.payload = torch.zeros_like(r.payload)
        return f"zero {r.id.encode()}"
    raise ValueError(fault)


def run(cases: int, seed: int) -> dict:
    """`cases` seeded fault cases; AssertionError (with the case) on the
    first report that differs from the oracle's."""
    import torch
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200 import synthetic
    from fuzz_parity import random_case
    from tests.test_configs_gpu import _oracle_recs
    from tests.test_gpu_parity import assert_reports_match
    from oracle import traindiff_oracle as O
    rnd = random.Random(seed)
    t0 = time.time()
    stats = collections.Counter()
    faults_seen = collections.Counter()
    for k in range(cases):
        m, p, bugs = random_case(rnd)
        dtype = rnd.choice([torch.bfloat16, torch.float32, torch.float16])
        fmt = td.FloatFormat.BF16 if dtype != torch.float32 else td.FloatFormat.FP32
        ref, cand = synthetic.build(m, p, dtype=dtype, seed=k, eps=fmt.eps, bugs=bugs)
        # per-id tolerances: mostly 2 eps, some larger, some never estimated (0: the eps floor)
        tol = td.ToleranceMap({r.id.encode(): rnd.choice([2 * fmt.eps, 2 * fmt.eps, 0.5 * fmt.eps, 30 * fmt.eps])
                               for r in ref.records if rnd.random() < 0.9}, n_samples=1, eps_p=fmt.eps)
        applied = []
        for _ in range(rnd.choice([1, 1, 2, 3])):
            fault = rnd.choice(FAULTS)
            trace = cand if rnd.random() < 0.7 else ref
            what = inject(rnd, trace, fault)
            if what is not None:
                applied.append(("cand: " if trace is cand else "ref: ") + what)
                faults_seen[fault] += 1
        kappa = rnd.choice([0.5, 3.0, 10.0])
        got_err = want_err = None
        try:
            rep = td.check(ref, cand, tol, kappa, fmt=fmt)
            got = json.loads(td.render_report(rep, "json"))
        except Exception as exc:          # noqa: BLE001 — compared with the oracle's outcome
            got_err = type(exc).__name__
        try:
            want = O.check(_oracle_recs(ref), _oracle_recs(cand), ref.header, cand.header, tol.responses, kappa,
                           fmt.value)
        except Exception as exc:          # noqa: BLE001
            want_err = type(exc).__name__
        label = json.dumps({"case": k, "model": str(m), "parallel": str(p), "bugs": bugs, "faults": applied,
                            "dtype": str(dtype), "kappa": kappa})
        if got_err or want_err:
            assert got_err is not None and want_err is not None, (label, got_err, want_err)
            stats["both_raise"] += 1
        else:
            assert_reports_match(got, want, label)
            for v, n in got["summary"].items():
                stats[v] += n
        if rnd.random() < 0.3:
            # compare_static (elementwise |c - r| <= atol + rtol |r|) on the same faulted traces
            atol, rtol = rnd.choice([(0.0, 0.0), (0.0, 1e-2), (1e-3, 1e-1), (10.0, 10.0)])
            got_s = [(e.ident, e.verdict) for e in td.compare_static(ref, cand, atol, rtol).entries]
            want_s = O.compare_static(_oracle_recs(ref), _oracle_recs(cand), atol, rtol)
            assert got_s == want_s, (label, "compare_static", atol, rtol)
            stats["static_cases"] += 1
        stats["cases"] += 1
    out = dict(stats)
    out["faults"] = dict(faults_seen)
    out["seconds"] = round(time.time() - t0, 1)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=500)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    try:
        print(json.dumps(run(args.cases, args.seed)))
    except AssertionError as exc:
        print(json.dumps({"mismatch": str(exc)[:1500]}))
        sys.exit(1)


if __name__ == "__main__":
    main()
