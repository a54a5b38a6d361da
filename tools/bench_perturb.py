"""td_perturb throughput: y = Q_bf16(x * (1 + u*eps)) on Llama-8B hidden
shapes (S=8192, d=4096) with the splitmix64 (reference) and Philox streams.
Algorithmic bytes = 2 * N * elem_bytes (read x, write y).  Prints JSON lines.

    python tools/bench_perturb.py
"""

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2506_09280_b200 as td
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    for rows, cols in ((8192, 4096), (8192, 2048), (1024, 1024)):
        for gen in ("splitmix64", "philox"):
            x = torch.randn(rows, cols, device="cuda").to(torch.bfloat16)
            y = torch.empty_like(x)
            flag = torch.zeros(1, dtype=torch.int64, device="cuda")
            spec = td.PerturbSpec(0, 2.0 ** -8)
            ident = "iter=0|mb=0|kind=ActivationOut|mod=model.embedding"
            for _ in range(3):
                td.apply_perturbation(x, ident, spec, policy="bf16", out=y, generator=gen,
                                      check=False, nonfinite=flag)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 20
            a.record()
            for _ in range(reps):
                td.apply_perturbation(x, ident, spec, policy="bf16", out=y, generator=gen,
                                      check=False, nonfinite=flag)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / reps
            nbytes = 2 * x.numel() * 2
            print(json.dumps({"rows": rows, "cols": cols, "generator": gen, "ms": ms,
                              "gbs": nbytes / ms / 1e6, "frac_hbm": nbytes / ms / 1e6 / peak,
                              "melem_per_s": x.numel() / ms / 1e3}), flush=True)


if __name__ == "__main__":
    main()
