"""Print the headline fields of bench.py JSON lines read from stdin."""
import json
import sys

for line in sys.stdin:
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    r = d.get("roofline", {})
    print(d["config"]["workload"][:40], "value", round(d["value"], 1), "ms", round(d["ms_per_step"], 4),
          "seg", round(r.get("achieved", 0), 1), "frac", round(r.get("frac", 0), 3),
          "e2e", round((d.get("e2e") or {}).get("value", 0), 1), "launches", d.get("gpu_launches"),
          "clk", (d.get("clocks") or {}).get("sm_mhz"), d.get("layer_checks_per_s", ""))
