"""The reference user's command, end to end: `check --ref R --cand C --tol T`
on config-2 trace files (16.4 GB of f32 payload), run in-process twice (the
first call includes CUDA/library start-up and the plan).  Prints JSON:
seconds per CLI call, exit code, GB/s of file payload."""
import contextlib
import io
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_2506_09280_b200.cli import main as cli
    from paper_2506_09280_b200.tracestore import write_trace
    _, ref, cand, tol, _ = bench.workload("cfg2")
    for t in (ref, cand):                       # the CLI reads the storage format from here
        t.header = dict(t.header, model=dict(t.header.get("model") or {}, precision="bf16"))
        t.raw_header = None
    tmp = os.environ.get("TMPDIR", "/tmp")
    paths = [os.path.join(tmp, f"cli_{n}.ttrc") for n in ("ref", "cand")]
    write_trace(ref, paths[0])
    write_trace(cand, paths[1])
    tpath = os.path.join(tmp, "cli_tol.json")
    with open(tpath, "wb") as fh:
        fh.write(tol.to_json())
    payload = sum(4 * r.payload.numel() for r in ref.records + cand.records)
    del ref, cand
    torch.cuda.empty_cache()
    times, codes = [], []
    for _ in range(3):
        t0 = time.perf_counter()
        with contextlib.redirect_stdout(io.StringIO()):
            codes.append(cli(["check", "--ref", paths[0], "--cand", paths[1], "--tol", tpath, "--json"]))
        times.append(time.perf_counter() - t0)
        torch.cuda.empty_cache()
    for p in paths + [tpath]:
        os.unlink(p)
    print(json.dumps({"payload_bytes_f32": payload, "seconds": times, "exit_codes": codes,
                      "best_gbs": payload / min(times) / 1e9}))


if __name__ == "__main__":
    main()
