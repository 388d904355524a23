"""Per CUDA source line: warp-stall samples and shared-memory wavefronts (total
and excessive) from `ncu --page source --csv --print-source cuda,sass` output.
    python scripts/ncu_line_wavefronts.py source.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[2]
ix = {}
for i, k in enumerate(h):
    ix.setdefault(k, i)
cur, agg = None, {}
for r in rows[3:]:
    if len(r) < 8:
        continue
    if r[0]:  # a CUDA line row (other kernels / files repeat the header)
        if not r[0].isdigit():
            continue
        cur = (int(r[0]), r[1].strip()[:80])
        agg.setdefault(cur, [0, 0, 0])
        continue
    def num(k):
        try:
            return int(r[ix[k]] or 0)
        except (KeyError, ValueError):
            return 0
    if cur is None:
        continue
    a = agg[cur]
    a[0] += num("Warp Stall Sampling (All Samples)")
    a[1] += num("L1 Wavefronts Shared")
    a[2] += num("L1 Wavefronts Shared Excessive")
ts = sum(v[0] for v in agg.values()) or 1
tw = sum(v[1] for v in agg.values()) or 1
print(f"samples {ts}  smem wavefronts {tw}  excessive {sum(v[2] for v in agg.values())}")
for (ln, src), v in sorted(agg.items(), key=lambda x: -x[1][1])[:n]:
    print(f"{100 * v[1] / tw:5.1f}% wf {100 * v[2] / max(v[1], 1):5.1f}% exc {100 * v[0] / ts:5.1f}% st  L{ln}: {src}")
