"""Key columns of an `ncu --page raw --csv` export, one line per launch.

    python tools/ncu_summary.py gpurun_out/prof_cfg2_full_raw.csv
"""
import csv
import sys

COLS = [
    ("gpu__time_duration.sum", "us", 1e-3),
    ("dram__bytes_read.sum", "rd_GB", 1e-9),
    ("dram__bytes_write.sum", "wr_GB", 1e-9),
    ("FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%", 1),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu%", 1),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64%", 1),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu%", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("sm__cycles_elapsed.avg.per_second", "GHz", 1e-9),
]


def main(path):
    with open(path) as fh:
        rows = list(csv.reader(fh))
    head, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(head)}
    print("kernel".ljust(44), " ".join(n.rjust(7) for _, n, _ in COLS), " GB/s")
    for r in rows[2:]:
        name = r[idx["Kernel Name"]].split("(")[0].replace("void <unnamed>::", "")
        vals = []
        for col, _, scale in COLS:
            i = idx.get(col)
            v = r[i].replace(",", "") if i is not None else ""
            try:
                x = float(v)
                u = units[i]
                if col == "gpu__time_duration.sum":
                    x = x * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "ms": 1e6, "us": 1e3, "ns": 1}.get(u, 1)
                if col.startswith("dram__bytes"):
                    x = x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)
                if col.endswith("per_second"):
                    x = x * {"cycle/second": 1, "cycle/nsecond": 1e9, "cycle/usecond": 1e6, "Ghz": 1e9, "Mhz": 1e6, "hz": 1}.get(u, 1)
                vals.append(x * scale)
            except ValueError:
                vals.append(float("nan"))
        gbs = (vals[1] + vals[2]) / (vals[0] * 1e-6) if vals[0] else float("nan")
        print(name[:44].ljust(44), " ".join(f"{v:7.3f}" if v < 100 else f"{v:7.0f}" for v in vals), f"{gbs:6.0f}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(p)
        main(p)
