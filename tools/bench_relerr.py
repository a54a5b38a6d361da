"""Latency of the public rel_err_arrays(a, b) on device tensors (the
reference's basic compare, tensor.py:158-167): per-call wall time through
the Python API, for bf16 tensors of 1 MiB - 1 GiB.  Prints JSON lines."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2506_09280_b200 as td
    for mib in (1, 16, 256, 1024):
        n = (mib << 20) // 2
        a = torch.randn(n, device="cuda").to(torch.bfloat16)
        b = (a.float() * (1 + 1e-3)).to(torch.bfloat16)
        for _ in range(3):
            td.rel_err_arrays(a, b)
        torch.cuda.synchronize()
        reps = 50 if mib < 256 else 10
        t0 = time.perf_counter()
        for _ in range(reps):
            v = td.rel_err_arrays(a, b)
        dt = (time.perf_counter() - t0) / reps
        want = float(torch.linalg.vector_norm((a.double() - b.double())) / torch.linalg.vector_norm(a.double()))
        print(json.dumps({"mib": mib, "us_per_call": dt * 1e6, "gbs": 2 * (mib << 20) / dt / 1e9,
                          "rel_err": v, "torch_fp64": want}), flush=True)


if __name__ == "__main__":
    main()
