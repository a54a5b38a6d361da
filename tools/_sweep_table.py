import json,sys
for l in sys.stdin:
    if l.startswith("{"):
        d=json.loads(l); print(d["mib"], d["maps"], d["shards"], round(d["segnorm_gbs"]), round(d["frac"],3), round(d["check_gbs"]), round(d["checks_per_s"]), round(d["graph_checks_per_s"]))
    else: print(l.strip()[:200])
