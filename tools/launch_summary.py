"""Per-kernel launch counts and mean device time from an ncu launch list
(--metrics gpu__time_duration.sum --csv):  python tools/launch_summary.py launches.csv [out.json]"""
import csv
import json
import sys
from collections import defaultdict

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
acc = defaultdict(list)
for r in csv.DictReader(lines):
    if r["Metric Name"] == "gpu__time_duration.sum":
        v = float(r["Metric Value"].replace(",", ""))
        acc[r["Kernel Name"]].append(v / 1000.0 if r["Metric Unit"] == "ns" else v)
out = {k: {"launches": len(v), "mean_us": sum(v) / len(v), "total_us": sum(v)} for k, v in acc.items()}
tot = sum(o["total_us"] for o in out.values())
for o in out.values():
    o["share"] = o["total_us"] / tot
print(json.dumps(out, indent=1))
if len(sys.argv) > 2:
    json.dump(out, open(sys.argv[2], "w"), indent=1)
