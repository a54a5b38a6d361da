"""Config 4's experiment at GPU scale: per-layer gradient tolerance vs depth.

A Llama-shaped bf16 torch model (RMSNorm, GQA attention, SwiGLU w1/w3/w2)
with L layers runs module-wise (every block input regenerated from its id,
then perturbed by td_perturb); estimate_tolerance (n samples) yields each
layer's ParamGrad response, which the paper bounds by c * sqrt(L / l) * eps
(Thm 3; the reference's trend test is test_acceptance.py:258-276).
Prints one JSON line: per-layer responses, Spearman(l, response), and the
least-squares c of the sqrt(L/l) fit with its log-rms residual.

    python tools/depth_sweep.py [--layers 16] [--d 256] [--seq 256] [--samples 5]
"""

import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build(layers, d, seq, vocab, kv):
    import torch

    class RMS(torch.nn.Module):
        def __init__(self, d):
            super().__init__()
            self.weight = torch.nn.Parameter(torch.ones(d))

        def forward(self, x):
            return self.weight * x * torch.rsqrt((x.float() ** 2).mean(-1, keepdim=True) + 1e-5).to(x.dtype)

    class Attn(torch.nn.Module):
        def __init__(self):
            super().__init__()
            self.norm = RMS(d)
            self.h, self.kv, self.hd = 8, kv, d // 8
            self.wq = torch.nn.Linear(d, d, bias=False)
            self.wk = torch.nn.Linear(d, kv * self.hd, bias=False)
            self.wv = torch.nn.Linear(d, kv * self.hd, bias=False)
            self.wo = torch.nn.Linear(d, d, bias=False)

        def forward(self, x):
            a = self.norm(x)
            q = self.wq(a).view(seq, self.h, self.hd).transpose(0, 1)
            k = self.wk(a).view(seq, self.kv, self.hd).transpose(0, 1).repeat_interleave(self.h // self.kv, 0)
            v = self.wv(a).view(seq, self.kv, self.hd).transpose(0, 1).repeat_interleave(self.h // self.kv, 0)
            o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
            return x + self.wo(o.transpose(0, 1).reshape(seq, d))

    class Mlp(torch.nn.Module):
        def __init__(self):
            super().__init__()
            self.norm = RMS(d)
            self.w1 = torch.nn.Linear(d, 4 * d, bias=False)
            self.w3 = torch.nn.Linear(d, 4 * d, bias=False)
            self.w2 = torch.nn.Linear(4 * d, d, bias=False)

        def forward(self, x):
            a = self.norm(x)
            return x + self.w2(torch.nn.functional.silu(self.w1(a)) * self.w3(a))

    class Model(torch.nn.Module):
        def __init__(self):
            super().__init__()
            self.embedding = torch.nn.Embedding(vocab, d)
            self.layers = torch.nn.ModuleList()
            for _ in range(layers):
                self.layers.append(Attn())
                self.layers.append(Mlp())
            self.final_norm = RMS(d)
            self.head = torch.nn.Linear(d, vocab, bias=False)

        def forward(self, ids):
            x = self.embedding(ids)
            for layer in self.layers:
                x = layer(x)
            return self.head(self.final_norm(x))

    return Model()


def spearman(xs, ys):
    def ranks(v):
        order = sorted(range(len(v)), key=lambda i: v[i])
        r = [0.0] * len(v)
        for k, i in enumerate(order):
            r[i] = float(k)
        return r
    rx, ry = ranks(xs), ranks(ys)
    mx, my = sum(rx) / len(rx), sum(ry) / len(ry)
    num = sum((a - mx) * (b - my) for a, b in zip(rx, ry))
    den = math.sqrt(sum((a - mx) ** 2 for a in rx) * sum((b - my) ** 2 for b in ry))
    return num / den


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=16)
    ap.add_argument("--d", type=int, default=256)
    ap.add_argument("--seq", type=int, default=256)
    ap.add_argument("--samples", type=int, default=5)
    args = ap.parse_args()
    import torch
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200.runner import torch_runner
    from paper_2506_09280_b200.torchtap import TapConfig
    torch.manual_seed(0)
    vocab = 1024
    model = build(args.layers, args.d, args.seq, vocab, kv=2).cuda().bfloat16()
    for p in model.parameters():
        torch.nn.init.normal_(p, 0.0, 0.02) if p.dim() > 1 else None
    ids = torch.randint(0, vocab, (args.seq,), device="cuda")
    labels = torch.roll(ids, -1)

    def step(m):
        torch.nn.functional.cross_entropy(m(ids).float(), labels).backward()
    blocks = tuple(f"layers.{i}" for i in range(2 * args.layers))
    runner = torch_runner(model, step, embedding="embedding",
                          tap=TapConfig(patterns=("layers.*",), precision="bf16"),
                          module_inputs=blocks, rewrite=True)
    eps = td.FloatFormat.BF16.eps
    t0 = time.perf_counter()
    tol = td.estimate_tolerance(runner, n_samples=args.samples, eps_p=eps)
    secs = time.perf_counter() - t0
    per_layer = []
    for l in range(args.layers):
        keys = [k for k in tol.responses if "kind=ParamGrad" in k and
                (f"mod=model.layers.{2 * l}." in k or f"mod=model.layers.{2 * l + 1}." in k)]
        vals = [tol.responses[k] for k in keys]
        per_layer.append(math.sqrt(sum(v * v for v in vals) / len(vals)) if vals else 0.0)
    L = args.layers
    basis = [math.sqrt(L / (l + 1)) * eps for l in range(L)]
    c = sum(b * r for b, r in zip(basis, per_layer)) / sum(b * b for b in basis)
    resid = math.sqrt(sum(math.log(max(r, 1e-30) / (c * b)) ** 2 for b, r in zip(basis, per_layer)) / L)
    print(json.dumps({"layers": L, "d_model": args.d, "seq": args.seq, "samples": args.samples,
                      "mode": "module-wise", "estimate_seconds": secs,
                      "per_layer_paramgrad_response_over_eps": [r / eps for r in per_layer],
                      "spearman_layer_vs_response": spearman(list(range(L)), per_layer),
                      "sqrt_bound_fit_c": c, "log_rms_residual": resid,
                      "fit": "response_l ~= c * sqrt(L / l) * eps"}))


if __name__ == "__main__":
    main()
