"""td_gather_bytes on a TTRC-like workload: 3000 ranges with arbitrary
(4-byte-misaligned) source offsets into a 4 GiB image, unpacked into a
256-B-aligned arena (the device reader's step), and the reverse scatter
(the writer's step).  CUDA-event timing after warm-up; prints JSON GB/s
counting bytes read + written."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_2506_09280_b200 import _native as N
    rng = np.random.default_rng(1)
    sizes = rng.integers(1 << 10, 3 << 20, 3000) * 4
    src_off, dst_off, s, d = [], [], 0, 0
    for n in sizes:
        s += int(rng.integers(13, 300))          # a record header of odd length
        src_off.append(s)
        s += int(n)
        d = -(-d // 256) * 256
        dst_off.append(d)
        d += int(n)
    image = torch.empty(s + 16, dtype=torch.uint8, device="cuda")
    arena = torch.empty(d + 16, dtype=torch.uint8, device="cuda")
    out = {}
    for name, a, b, table in (("unpack", image, arena, list(zip(src_off, dst_off, sizes.tolist()))),
                              ("scatter", arena, image, list(zip(dst_off, src_off, sizes.tolist())))):
        ranges = torch.tensor(table, dtype=torch.int64, device="cuda")
        call = lambda: N.call("td_gather_bytes", a.data_ptr(), b.data_ptr(), ranges.data_ptr(), len(table),
                              N.stream_handle())
        for _ in range(3):
            call()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            call()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        out[name] = {"ms": ms, "gbs_rw": 2 * int(sizes.sum()) / (ms / 1e3) / 1e9}
    out["payload_bytes"] = int(sizes.sum())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
