"""Host side of the pageable e2e path: how fast T threads copy pageable
memory into a pinned 4 x 64 MiB ring (numpy copyto = glibc memcpy, the GIL
released), alone and with the ring's H2D DMA running, to place
e2e.pageable (33-38 GB/s on config 3) against the host's own ceiling.

    python tools/host_copy_probe.py [--gib 8] [--threads 1,2,4,8,12,16]
"""
import argparse
import concurrent.futures
import json
import time


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=8.0)
    ap.add_argument("--threads", default="1,2,4,8,12,16")
    ap.add_argument("--chunk-mib", type=int, default=64)
    args = ap.parse_args()
    import numpy as np
    import torch
    n = int(args.gib * (1 << 30))
    src = np.empty(n, np.uint8)
    src.fill(3)
    chunk = args.chunk_mib << 20
    ring = [torch.empty(chunk, dtype=torch.uint8).pin_memory() for _ in range(4)]
    host = [r.numpy() for r in ring]
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.Stream()
    out = {"gib": args.gib, "chunk_mib": args.chunk_mib}
    for nt in [int(x) for x in args.threads.split(",")]:
        pool = concurrent.futures.ThreadPoolExecutor(nt)
        for dma in (False, True):
            events = [None] * 4
            t0 = time.perf_counter()
            for k, off in enumerate(range(0, n, chunk)):
                s = k % 4
                if events[s] is not None:
                    events[s].synchronize()
                m = min(chunk, n - off)
                step = -(-m // nt)
                list(pool.map(lambda o: np.copyto(host[s][o:min(o + step, m)], src[off + o:off + min(o + step, m)]),
                              range(0, m, step)))
                if dma:
                    with torch.cuda.stream(stream):
                        dev[off:off + m].copy_(ring[s][:m], non_blocking=True)
                        ev = torch.cuda.Event()
                        ev.record(stream)
                    events[s] = ev
            torch.cuda.synchronize()
            out[f"t{nt}_{'dma' if dma else 'copy'}_gbs"] = round(n / (time.perf_counter() - t0) / 1e9, 2)
        pool.shutdown()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
