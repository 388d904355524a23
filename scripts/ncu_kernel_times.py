"""Per-kernel durations from an `ncu --metrics gpu__time_duration.sum --csv` log.

usage: python scripts/ncu_kernel_times.py LOG.csv [LOG2.csv ...]
"""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, x in enumerate(rows) if "Kernel Name" in x)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    d = collections.defaultdict(list)
    for row in rows[hdr + 1:]:
        d[row[ki].split("(")[0]].append(float(row[vi].replace(",", "")) / 1000)
    print(path)
    for k, v in d.items():
        print("  %-28s n=%-4d mean %8.1f us  first: %s" % (k[:28], len(v), sum(v) / len(v), [round(x, 1) for x in v[:8]]))
