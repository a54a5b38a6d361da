import json, sys
for line in sys.stdin:
    if line.startswith("{"):
        d = json.loads(line)
        r = d["roofline"]
        print(f"value {d['value']:.0f} GB/s  segnorm {r['achieved']:.0f} GB/s frac {r['frac']:.3f}  ms/step {d['ms_per_step']:.4f}")
    elif "Error" in line:
        print(line.strip())
