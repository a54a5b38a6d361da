"""The drop-in host path of a reference user: traces parsed on the host
(numpy f32 payloads, as traindiff.read_trace returns them) passed to
check().  Config-2 traces (16.4 GB of f32 payload).  Prints JSON: seconds
per check (first call plans; later calls hit the plan cache) and GB/s."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    import paper_2506_09280_b200 as td
    from paper_2506_09280_b200.tracestore import trace_from_bytes, trace_to_bytes, write_trace
    _, ref, cand, tol, fmt = bench.workload("cfg2")
    if "--file" in sys.argv:
        # read_trace(path) on the host: payloads view a pinned file image
        tmp = os.environ.get("TMPDIR", "/tmp")
        paths = [os.path.join(tmp, f"bhc_{n}.ttrc") for n in ("ref", "cand")]
        t0 = time.perf_counter()
        write_trace(ref, paths[0])
        write_trace(cand, paths[1])
        write_s = time.perf_counter() - t0
        del ref, cand
        torch.cuda.empty_cache()
        read_dev = []
        for _ in range(2):                      # the CLI's reader: file -> HBM
            t0 = time.perf_counter()
            dref, dcand = td.read_trace(paths[0], device="cuda"), td.read_trace(paths[1], device="cuda")
            torch.cuda.synchronize()
            read_dev.append(time.perf_counter() - t0)
            del dref, dcand
            torch.cuda.empty_cache()
        pin = "--pin" in sys.argv
        t0 = time.perf_counter()
        href, hcand = td.read_trace(paths[0], pin=pin), td.read_trace(paths[1], pin=pin)
        read_s = time.perf_counter() - t0
        for p in paths:
            os.unlink(p)
    else:
        read_s = write_s = read_dev = None
        rb, cb = trace_to_bytes(ref), trace_to_bytes(cand)
        del ref, cand
        torch.cuda.empty_cache()
        href, hcand = trace_from_bytes(rb), trace_from_bytes(cb)
    nbytes = sum(r.nbytes for r in href.records) + sum(r.nbytes for r in hcand.records)
    times = []
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = td.check(href, hcand, tol, fmt=fmt)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    print(json.dumps({"mode": ("file+pin" if "--pin" in sys.argv else "file") if read_s is not None else "bytes", "read_s": read_s, "write_s": write_s, "read_device_s": read_dev,
                      "payload_bytes_f32": nbytes, "first_s": times[0], "cached_s": min(times[1:]),
                      "cached_gbs": nbytes / min(times[1:]) / 1e9, "verdicts": rep.counts}))


if __name__ == "__main__":
    main()
