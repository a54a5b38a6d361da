"""Differential fuzzing of td_perturb against the oracle's restatement of
Emulator._apply_perturbation (engine.py:351-361): random shapes, column
shards (col0 / full width, odd offsets), row-position subsets (CP / SP
slices), eps (2^-8, 1e-3, 0.3, 2^-24), policy (bf16 / fp32), input and
output dtypes (bf16, f32, f64) and generator (splitmix64, philox).  Values
must be bit-identical (bf16 outputs: outside the bf16-subnormal range, where
no bf16 can hold the reference's unbounded-exponent value).

    python tools/fuzz_perturb.py [--cases 500] [--seed 0]      (GPU)
"""

import argparse
import json
import os
import random
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_case(rnd, k):
    import torch
    import paper_2506_09280_b200 as td
    from oracle import traindiff_oracle as O
    g = torch.Generator(device="cuda").manual_seed(k)
    full_cols = rnd.choice([8, 24, 64, 96, 100, 512, 4096 + 8, 37])
    rows_total = rnd.choice([1, 3, 16, 64, 257])
    cols = rnd.choice([c for c in (full_cols, full_cols // 2, 8, 16, 5) if 0 < c <= full_cols])
    col0 = rnd.randrange(0, full_cols - cols + 1)
    pos = np.array(sorted(rnd.sample(range(rows_total), rnd.randint(1, rows_total))), dtype=np.int64)
    eps = rnd.choice([2.0 ** -8, 1e-3, 0.3, 2.0 ** -24])
    policy = rnd.choice(["bf16", "fp32"])
    in_dt = rnd.choice([torch.bfloat16, torch.float32, torch.float64])
    if policy == "bf16":
        out_dt = rnd.choice([torch.bfloat16, torch.float32, torch.float64])
    else:
        out_dt = rnd.choice([torch.float32, torch.float64])
    generator = rnd.choice(["splitmix64", "philox"])
    scale = rnd.choice([1.0, 1e-3, 1e3])
    x_full = (torch.randn(rows_total, full_cols, device="cuda", generator=g, dtype=torch.float64) * scale).to(in_dt)
    x = x_full[torch.from_numpy(pos).cuda()][:, col0:col0 + cols].contiguous()
    ident = f"iter=0|mb={k % 3}|kind=ActivationIn|mod=model.layers.{k % 7}"
    spec = td.PerturbSpec(k % 5, eps)
    y = torch.empty(x.shape, dtype=out_dt, device="cuda")
    td.apply_perturbation(x, ident, spec, full_cols=full_cols, col0=col0, row_positions=pos, policy=policy,
                          out=y, generator=generator)
    xf = x_full.double().cpu().numpy()[pos]
    want = O.perturb(xf, f"perturb|s={spec.sample}|{ident}", eps, pos, full_cols,
                     "BF16" if policy == "bf16" else None, generator=generator)[:, col0:col0 + cols]
    if out_dt == torch.float32:
        want = want.astype(np.float32).astype(np.float64)
    got = y.double().cpu().numpy()
    mask = np.abs(want) >= 2.0 ** -126 if out_dt == torch.bfloat16 else np.ones(want.shape, bool)
    if not np.array_equal(got[mask], want[mask]):
        bad = np.argwhere((got != want) & mask)[:3].tolist()
        raise AssertionError(json.dumps({"case": k, "rows_total": rows_total, "full_cols": full_cols, "cols": cols,
                                         "col0": col0, "eps": eps, "policy": policy, "in": str(in_dt),
                                         "out": str(out_dt), "generator": generator, "first_bad": bad}))
    return x.numel()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=500)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    rnd = random.Random(args.seed)
    t0 = time.time()
    n = 0
    for k in range(args.cases):
        try:
            n += run_case(rnd, k)
        except AssertionError as exc:
            print(json.dumps({"failed": str(exc)[:1500]}))
            sys.exit(1)
    print(json.dumps({"cases": args.cases, "elements": n, "seconds": round(time.time() - t0, 1)}))


if __name__ == "__main__":
    main()
