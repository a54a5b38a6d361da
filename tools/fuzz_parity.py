"""Differential fuzzing of the GPU check against the CPU oracle over the
layout space: random small model shapes (GPT-style or Llama-style: GQA,
gated MLP, RMSNorm), random valid parallel layouts (tp, dp, pp, vp, cp, sp,
microbatches; world <= 8), random storage dtype, and random injected bugs
(scale / shard order / missing allreduce on random ids).  Every case: the
report of td.check on the device traces equals the oracle's on host copies
(verdicts, details, thresholds exact; observed within 1e-12).

    python tools/fuzz_parity.py [--cases 200] [--seed 0]     (GPU)
Prints one JSON summary line; exit 1 on the first mismatch (with the case).
"""

import argparse
import json
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def random_case(rnd):
    from paper_2506_09280_b200 import layout as L
    from paper_2506_09280_b200.errors import ConfigInvalid
    while True:
        llama = rnd.random() < 0.5
        heads = rnd.choice([2, 4, 8])
        d = heads * rnd.choice([8, 16])
        m = L.ModelShape(layers=rnd.choice([1, 2, 4]), d_model=d, n_heads=heads,
                         d_ff=d * rnd.choice([2, 4]), seq_len=rnd.choice([16, 32, 64]),
                         vocab=rnd.choice([64, 128, 256]),
                         n_kv_heads=(heads // rnd.choice([1, 2]) if llama else None),
                         gated_mlp=llama, norm_bias=not llama, position_table=not llama)
        p = L.ParallelConfig(tp=rnd.choice([1, 2, 4]), dp=rnd.choice([1, 2]), pp=rnd.choice([1, 2]),
                             vp=rnd.choice([1, 1, 2]), cp=rnd.choice([1, 1, 2]), sp=rnd.random() < 0.3,
                             microbatches=rnd.choice([1, 2, 4]))
        try:
            L.validate_parallel(m, p)
            if m.n_kv_heads and (m.n_kv_heads * m.head_dim) % p.tp:
                continue
            specs = L.emit_records(m, p)
        except (ConfigInvalid, ValueError, AssertionError, ZeroDivisionError):
            continue
        ids = sorted({s.ident for s in specs})
        bugs = {}
        for _ in range(rnd.choice([0, 0, 1, 2])):
            bugs[rnd.choice(ids)] = rnd.choice(["scale", "order", "partial"])
        return m, p, bugs


def scramble_dtypes(rnd, *traces, p=0.15):
    """Widen a random subset of payloads exactly (bf16/f16 -> f32, f32 -> f64):
    mixed-dtype operands and replica groups exercise the widening paths
    (generic walker, per-group common dtype) with unchanged values."""
    import torch
    for trace in traces:
        for rec in trace.records:
            if rnd.random() < p and rec.payload.dtype != torch.float64:
                wider = torch.float64 if rec.payload.dtype == torch.float32 else torch.float32
                rec.payload = rec.payload.to(wider)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=200)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    import torch
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200 import synthetic
    from tests.test_configs_gpu import _oracle_recs
    from tests.test_gpu_parity import assert_reports_match
    from oracle import traindiff_oracle as O
    rnd = random.Random(args.seed)
    t0 = time.time()
    stats = {"cases": 0, "ids": 0, "flag": 0, "replica-mismatch": 0, "merge-error": 0, "layouts": set()}
    for k in range(args.cases):
        m, p, bugs = random_case(rnd)
        dtype = rnd.choice([torch.bfloat16, torch.float32, torch.float16])
        fmt = td.FloatFormat.BF16 if dtype != torch.float32 else td.FloatFormat.FP32
        ref, cand = synthetic.build(m, p, dtype=dtype, seed=k, eps=fmt.eps, bugs=bugs)
        scramble_dtypes(rnd, ref, cand)
        tol = td.ToleranceMap({r.id.encode(): 2 * fmt.eps for r in ref.records}, n_samples=1, eps_p=fmt.eps)
        kappa = rnd.choice([0.5, 3.0, 10.0])
        rep = td.check(ref, cand, tol, kappa, fmt=fmt)
        want = O.check(_oracle_recs(ref), _oracle_recs(cand), ref.header, cand.header, tol.responses, kappa,
                       fmt.value)
        try:
            assert_reports_match(json.loads(td.render_report(rep, "json")), want, f"case {k}")
        except AssertionError as exc:
            print(json.dumps({"mismatch": k, "model": str(m), "parallel": str(p), "bugs": bugs,
                              "dtype": str(dtype), "kappa": kappa, "error": str(exc)[:500]}))
            sys.exit(1)
        stats["cases"] += 1
        stats["ids"] += len(rep.entries)
        for v in ("flag", "replica-mismatch", "merge-error"):
            stats[v] += rep.counts[v]
        stats["layouts"].add((p.tp, p.dp, p.pp, p.vp, p.cp, p.sp, p.microbatches))
    stats["layouts"] = len(stats["layouts"])
    stats["seconds"] = round(time.time() - t0, 1)
    print(json.dumps(stats))


if __name__ == "__main__":
    main()
