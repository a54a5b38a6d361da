"""Refresh profiles/segnorm_traffic.json (the bench's roofline.traffic) from
an `ncu --set full` raw page of one check's td_segnorm class launches.

    python tools/traffic_json.py cfg3 profiles/r2_cfg3_segnorm_full_raw.csv 2 <algorithmic bytes>

Takes the first N launches of the capture (one step's classes) and records
dram__bytes_read.sum + dram__bytes_write.sum per launch and per step.
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(cfg, raw, n, alg):
    with open(raw) as fh:
        rows = list(csv.reader(fh))
    head = rows[0]
    idx = {h: i for i, h in enumerate(head)}
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

    def val(r, col):
        return float(r[idx[col]].replace(",", "")) * scale.get(units[idx[col]], 1)
    launches, total = {}, 0
    for r in rows[2:2 + n]:
        name = r[idx["Kernel Name"]].split("(")[0].replace("void <unnamed>::", "")
        rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
        us = float(r[idx["gpu__time_duration.sum"]].replace(",", "")) / (1e3 if units[idx["gpu__time_duration.sum"]] == "ns" else 1)
        launches[name] = {"dram_read": int(rd), "dram_write": int(wr), "us": us}
        total += rd + wr
    path = os.path.join(ROOT, "profiles", "segnorm_traffic.json")
    with open(path) as fh:
        doc = json.load(fh)
    doc["configs"][cfg] = {"launches": launches, "dram_bytes_per_step": int(total),
                           "algorithmic_bytes_per_step": int(alg), "capture": os.path.relpath(raw, ROOT)}
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=2)
    print(cfg, int(total), total / alg)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
