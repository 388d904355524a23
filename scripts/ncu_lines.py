"""Warp-stall samples aggregated by CUDA source line (needs -lineinfo and
ncu --import-source on):  python scripts/ncu_lines.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
agg = {}
cur = None
for r in rows:
    if "Source" in r and any("Warp Stall Sampling (All" in h for h in r):
        hdr = r
        ix = {h: i for i, h in enumerate(hdr)}
        key = [h for h in hdr if h.startswith("Warp Stall Sampling (All")][0]
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    src = r[ix["Source"]]
    try:
        v = float(r[ix[key]] or 0)
    except ValueError:
        continue
    line = r[ix["#"]] if "#" in ix else r[0]
    agg[(line, src.strip()[:100])] = agg.get((line, src.strip()[:100]), 0.0) + v
tot = sum(agg.values()) or 1.0
for (line, src), v in sorted(agg.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{100 * v / tot:5.1f}%  {line:>6}  {src}")
