"""estimate_tolerance end to end on a real model, config-1 shape: a 2-layer
Pre-LN GPT-2-small-shaped fp32 torch model (d=768, 12 heads, ff=3072,
S=1024, V=50304) — the reference needs 545.6 s for n=2 on its CPU emulator
(SURVEY §6).  Times n_samples+1 traced forward/backward runs with td_perturb
in the embedding hook and the response reductions on the GPU.

    python tools/bench_tolerance.py [--samples 5] [--precision fp32|bf16]
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=5)
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--layers", type=int, default=2)
    args = ap.parse_args()
    import torch
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200.runner import torch_runner
    from paper_2506_09280_b200.torchtap import TapConfig
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from test_runner import Tiny
    torch.manual_seed(0)
    model = Tiny(vocab=50304, d=768, h=12, ff=3072, layers=args.layers, seq=1024).cuda()
    if args.precision == "bf16":
        model = model.bfloat16()
    ids = torch.randint(0, 50304, (1024,), device="cuda")
    labels = torch.roll(ids, -1)

    def step(m):
        torch.nn.functional.cross_entropy(m(ids).float(), labels).backward()
    runner = torch_runner(model, step, embedding="embedding",
                          tap=TapConfig(patterns=("embedding", "layers.*", "final_norm", "head"),
                                        precision=args.precision),
                          policy=args.precision)
    fmt = td.FloatFormat.FP32 if args.precision == "fp32" else td.FloatFormat.BF16
    td.estimate_tolerance(runner, n_samples=1, eps_p=fmt.eps)      # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    tol = td.estimate_tolerance(runner, n_samples=args.samples, eps_p=fmt.eps)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    ref = runner(None)
    t1 = time.perf_counter()
    rep = td.check(ref, runner(None), tol, fmt=fmt)
    torch.cuda.synchronize()
    check_s = time.perf_counter() - t1
    print(json.dumps({"model": f"GPT-2-small shape L={args.layers} S=1024 {args.precision}",
                      "n_samples": args.samples, "estimate_tolerance_seconds": secs,
                      "ids": len(tol.responses), "trace_bytes": ref.nbytes,
                      "check_with_fresh_run_seconds": check_s, "verdicts": rep.counts,
                      "reference_cpu_seconds_n2": 545.6}))


if __name__ == "__main__":
    main()
