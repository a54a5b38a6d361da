"""Condense an `ncu --metrics gpu__time_duration.sum --csv` log into
profiles/ form: every launch of the library's kernels, then per-kernel
totals of the whole process.

    python tools/launch_list.py gpurun_out/prof_cfg2_launches.csv "# header line" > profiles/x.csv
"""
import collections
import csv
import sys

OURS = ("k_segnorm", "k_finalize", "k_reduce", "k_verdict", "k_perturb", "k_generate", "k_gather",
        "k_quantize", "k_signed", "k_fingerprint", "k_box_gather")


def main(path, header):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    head = rows[0]
    ki, mi, vi, ui = head.index("Kernel Name"), head.index("Metric Name"), head.index("Metric Value"), \
        head.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3}
    print(header)
    print("# rows: every launch of the library kernels; per-kernel totals of the whole process below")
    print("id,kernel,duration_us")
    tot = collections.OrderedDict()
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0] if "(" in r[ki] and "<" in r[ki].split("(")[0] else r[ki].split("(")[0]
        us = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        if any(k in name for k in OURS):
            print(f"{r[0]},{name},{us:.3f}")
        c, t = tot.get(name, (0, 0.0))
        tot[name] = (c + 1, t + us)
    print("# launches,total_us,kernel")
    for name, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"# {c},{t:.1f},{name[:200]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "# ncu launch list")
