"""Pageable host → HBM: what cudaHostRegister (page-lock the caller's memory
in place, then one DMA) costs against the staging-ring copy and the
driver's own pageable cudaMemcpy, per GB.

    python tools/register_probe.py [--gib 4] [--threads 1,4,8]
"""
import argparse
import ctypes
import json
import os
import threading
import time


def cudart():
    import nvidia.cuda_runtime as cr
    base = list(cr.__path__)[0]
    lib = ctypes.CDLL(os.path.join(base, "lib", "libcudart.so.12"))
    lib.cudaHostRegister.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint]
    lib.cudaHostUnregister.argtypes = [ctypes.c_void_p]
    return lib


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=4.0)
    ap.add_argument("--threads", default="1,4,8")
    args = ap.parse_args()
    import torch
    n = int(args.gib * (1 << 30))
    import numpy as np
    raw = np.empty(n + 4096, np.uint8)
    off = (-raw.ctypes.data) % 4096
    host = torch.from_numpy(raw[off:off + n])       # page-aligned, like a trace file's mmap
    host.fill_(7)                                   # pages touched, as a trace's would be
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")
    rt = cudart()
    out = {"gib": args.gib}

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dev.copy_(host)
    torch.cuda.synchronize()
    assert bool((dev[:: 1 << 20] == 7).all())
    out["pageable_memcpy_gbs"] = n / (time.perf_counter() - t0) / 1e9

    for nt in [int(x) for x in args.threads.split(",")]:
        step = -(-n // nt)
        step = -(-step // 4096) * 4096
        pieces = [(o, min(step, n - o)) for o in range(0, n, step)]
        base = host.data_ptr()
        rcs = []

        def reg(o, sz):
            rcs.append(rt.cudaHostRegister(base + o, sz, 0))
        t0 = time.perf_counter()
        ths = [threading.Thread(target=reg, args=p) for p in pieces]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        t1 = time.perf_counter()
        if any(rcs):
            out[f"register_t{nt}"] = {"rc": sorted(set(rcs))}
            continue
        crc = rt.cudaMemcpy(ctypes.c_void_p(dev.data_ptr()), ctypes.c_void_p(base), ctypes.c_size_t(n), 1)
        t2 = time.perf_counter()
        urc = []

        def unreg(o, sz):
            urc.append(rt.cudaHostUnregister(base + o))
        ths = [threading.Thread(target=unreg, args=p) for p in pieces]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        t3 = time.perf_counter()
        out[f"register_t{nt}"] = {"rc": sorted(set(rcs)), "urc": sorted(set(urc)), "copy_rc": crc,
                                  "register_gbs": n / (t1 - t0) / 1e9, "dma_gbs": n / (t2 - t1) / 1e9,
                                  "unregister_gbs": n / (t3 - t2) / 1e9,
                                  "total_gbs": n / (t3 - t0) / 1e9}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
