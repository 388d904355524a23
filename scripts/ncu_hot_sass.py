"""Top SASS instructions by warp-stall samples from an ncu report (source page),
with the dominant stall reasons:  python scripts/ncu_hot_sass.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = rows[2:]
idx = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") or "Stall" in h and "Sampling" not in h]
tot = sum(float(r[2] or 0) for r in data)
print("total samples", tot, "| stall columns:", len(stall_cols))
agg = {}
for r in data:
    for h in stall_cols:
        try:
            agg[h] = agg.get(h, 0.0) + float(r[idx[h]] or 0)
        except ValueError:
            pass
for h, v in sorted(agg.items(), key=lambda x: -x[1])[:10]:
    print(f"  {h:50s} {v:10.0f}")
top = sorted(data, key=lambda r: -float(r[2] or 0))[:n]
for r in top:
    reasons = sorted(((float(r[idx[h]] or 0), h) for h in stall_cols if (r[idx[h]] or "0") not in ("0", "")),
                     reverse=True)[:3]
    print(f"{float(r[2] or 0):6.0f} {r[1].strip()[:60]:60s} " + " ".join(f"{h.replace('stall_', '')}={v:.0f}" for v, h in reasons))
