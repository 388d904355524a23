"""Per-phase timeline of the cluster LSQR (debug hook nnls_debug_lsqr_profile):
average ns per phase over iterations (CTA 0's view)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import nnls_gen as g  # noqa: E402
import paper_cs_0408029_b200 as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prob = g.make_problem(cfg, 0)
S = P.setup(prob)
prof = torch.zeros(64 * 16, dtype=torch.int64, device="cuda")
P.lib.nnls_debug_lsqr_profile.argtypes = [C.c_void_p]
for rep in range(2):
    prof.zero_()
    P.lib.nnls_debug_lsqr_profile(C.c_void_p(prof.data_ptr()))
    x, info = S.solve()
    P.lib.nnls_debug_lsqr_profile(C.c_void_p(0))
p = prof.cpu().numpy().reshape(64, 16).astype(np.float64)
names = ["A.compute", "A.push+bsum", "A.clsync", "B dots | scalars", "B.v update", "B.push+bsum", "B.clsync",
         "ctotal(alpha)", "C.compute", "(C end)"]
# (itn is incremented between stamps 4 and 5: slots 0-4 and 11-13 of an
# iteration are in row r, slots 5-10 in row r + 1)
rows = [r for r in range(1, 62) if p[r, 0] > 0 and p[r + 1, 10] > 0 and p[r + 1, 0] > 0]
d = {n: [] for n in names}
for r in rows:
    q = np.concatenate([p[r, :5], p[r + 1, 5:11]])
    for k in range(10):
        d[names[k]].append(q[k + 1] - q[k])
print("iterations profiled:", len(rows), "lsqr_iterations:", info["lsqr_iterations"])
bd = [p[r, 13] - p[r, 3] for r in rows if p[r, 13] > 0]
if bd:
    print(f"{'  B dots (warp 1)':22s} {np.mean(bd):9.0f} ns")
ws = [p[r, 12] - p[r, 3] for r in rows if p[r, 12] > 0]
if ws:
    print(f"{'  warp0 scalars':22s} {np.mean(ws):9.0f} ns")
pp = [p[r, 11] - p[r, 1] for r in rows if p[r, 11] > 0]
if pp:
    print(f"{'  of which push':22s} {np.mean(pp):9.0f} ns")
tot = 0
for k, v in d.items():
    if v:
        print(f"{k:22s} {np.mean(v):9.0f} ns")
        tot += np.mean(v)
print(f"{'per iteration':22s} {tot:9.0f} ns")

st = p[63]
if st[0] > 0:
    lab = ["entry", "slices", "staged", "loop start", "loop end", "report end"]
    print("setup/epilogue (us from kernel entry):", ", ".join(f"{lab[i]} {(st[i] - st[0]) / 1e3:.2f}" for i in range(6) if st[i] > 0))
