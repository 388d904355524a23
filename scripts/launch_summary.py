"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total device time and share (cold-cache, serialised:
compare SHARES with bench.py's live CUDA-event phase times, not absolutes)."""
import collections
import csv
import json
import sys

path = sys.argv[1]
rows = list(csv.reader(open(path)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"ns": 1.0, "nsecond": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0]
    agg[k][0] += 1
    agg[k][1] += float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
tot = sum(v[1] for v in agg.values())
out = {k: {"launches": v[0], "total_us": round(v[1] / 1e3, 3), "avg_us": round(v[1] / 1e3 / v[0], 3),
           "share": round(v[1] / tot, 4)} for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}
print(json.dumps(out, indent=1))
