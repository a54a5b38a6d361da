"""td_fingerprint throughput: one launch over 64 bf16 tensors of 128 MiB
(8 GiB, >> L2), CUDA events, median of 10.  Prints one JSON line."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2506_09280_b200.device import Fingerprints
    ts = [torch.empty(64 << 20, dtype=torch.bfloat16, device="cuda").normal_() for _ in range(64)]
    fp = Fingerprints(ts)
    for _ in range(3):
        fp.run()
    times = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fp.run()
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
    ms = statistics.median(times)
    print(json.dumps({"bytes": fp.nbytes, "ms": ms, "gbs": fp.nbytes / ms / 1e6}))


if __name__ == "__main__":
    main()
