"""write_trace of a device-resident trace (config-2 reference trace, the
torchtap -> file flow): seconds per call and GB/s of file written, against
the joined-bytes path (trace_to_bytes + one write).  Prints JSON."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import bench
    from paper_2506_09280_b200.tracestore import trace_to_bytes, write_trace
    _, ref, _, _, _ = bench.workload("cfg2")
    path = os.path.join(os.environ.get("TMPDIR", "/tmp"), "bwt.ttrc")
    times = []
    for _ in range(3):
        t0 = time.perf_counter()
        write_trace(ref, path)
        times.append(time.perf_counter() - t0)
    size = os.path.getsize(path)
    t0 = time.perf_counter()
    raw = trace_to_bytes(ref)
    with open(path + ".old", "wb") as fh:
        fh.write(raw)
    old = time.perf_counter() - t0
    same = open(path, "rb").read() == raw
    os.unlink(path)
    os.unlink(path + ".old")
    print(json.dumps({"file_bytes": size, "first_s": times[0], "best_s": min(times),
                      "gbs": size / min(times) / 1e9, "joined_bytes_path_s": old, "identical": same}))


if __name__ == "__main__":
    main()
