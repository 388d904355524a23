"""Config-2 problem with unquantized values (the ordered Gram path): load it a
few times and print the per-phase load times.  python scripts/gram_raw_run.py [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import nnls_gen as g  # noqa: E402
import paper_cs_0408029_b200 as P  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cfg = int(os.environ.get("CFG", "2"))
shape = dict(m=int(os.environ["M"]), n=int(os.environ["N"]), density=float(os.environ["D"])) if "M" in os.environ else cfg
prob = g.make_problem(shape, seed=0, raw=True)
S = P.setup(prob)
P.timing_enable(S.h)
for _ in range(reps):
    S.load_problem(prob)
t = P.timing_read(S.h)
print({k: round(v[0] / reps, 4) for k, v in t.items() if v[1]})
G, c = S.gram()
print("G checksum", float(np.abs(G).sum()), float(np.abs(c).sum()))
