"""Pinned host -> HBM copy bandwidth on this box: one 8 GiB buffer over 1, 2
and 4 streams (chunks split evenly), for the e2e ceiling.  Prints JSON."""
import json
import torch

n = 8 << 30
src = torch.empty(n, dtype=torch.uint8, pin_memory=True)
src.fill_(1)
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
for streams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    chunk = n // streams
    for rep in range(3):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for k, s in enumerate(ss):
            s.wait_event(a)
            with torch.cuda.stream(s):
                dst[k * chunk:(k + 1) * chunk].copy_(src[k * chunk:(k + 1) * chunk], non_blocking=True)
        for s in ss:
            torch.cuda.current_stream().wait_stream(s)
        b.record()
        torch.cuda.synchronize()
    print(json.dumps({"streams": streams, "h2d_gbs": n / (a.elapsed_time(b) / 1e3) / 1e9}), flush=True)
d2h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(); d2h.copy_(dst, non_blocking=True); b.record(); torch.cuda.synchronize()
print(json.dumps({"d2h_gbs": n / (a.elapsed_time(b) / 1e3) / 1e9}))
