"""Per-phase timeline of the cooperative-grid LSQR (config 2 default):
python scripts/lsqr_grid_profile.py [config]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import nnls_gen as g  # noqa: E402
import paper_cs_0408029_b200 as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
if cfg != 2:
    os.environ["NNLS_NO_CLUSTER"] = "1"
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
# stamps 0-2 of an iteration land in row itn, stamps 3-5 (after ++itn) in row itn+1
rows = [r for r in range(1, 62) if p[r, 0] > 0 and p[r + 1, 5] > 0 and p[r + 1, 0] > 0]
def st(r, k):
    return p[r, k] if k < 3 else p[r + 1, k]
names = ["A spmv", "A blocksum+sync", "A gridsum+test+B spmv", "B blocksum+sync", "B gridsum+C"]
for k, nm in enumerate(names):
    d = [(st(r, k + 1) - st(r, k)) / 1e3 for r in rows]
    print(f"{nm:22s} {np.mean(d):8.2f} us")
if p[rows[0], 6] > 0:
    print("  (A: spmv part %.2f us, partial A^T U %.2f us)" % (np.mean([(p[r, 6] - p[r, 0]) / 1e3 for r in rows]),
                                                          np.mean([(p[r, 1] - p[r, 6]) / 1e3 for r in rows])))
m = p[63]
if m[0] > 0:
    print("kernel: setup %.1f us, to loop end %.1f us, finish %.1f us, total %.1f us" % (
        (m[1] - m[0]) / 1e3 if m[1] > 0 else float("nan"), (m[2] - m[0]) / 1e3 if m[2] > 0 else float("nan"),
        (m[3] - m[2]) / 1e3 if m[2] > 0 else float("nan"), (m[3] - m[0]) / 1e3))
if m[4] > 0:
    print("finish: x out %.1f us, R = Ax-b %.1f us, y' = A^T R %.1f us, reduce %.1f us" % (
        (m[4] - m[2]) / 1e3, (m[5] - m[4]) / 1e3, (m[6] - m[5]) / 1e3, (m[3] - m[6]) / 1e3))
if m[7] > 0:
    print("start: setup end -> first sync arrive %.1f, first sync %.1f, -> loop %.1f us" % (
        (m[8] - m[1]) / 1e3, (m[9] - m[8]) / 1e3, (m[7] - m[9]) / 1e3))
print("per iteration", np.mean([(p[r + 1, 0] - p[r, 0]) / 1e3 for r in rows]), "us; lsqr_iterations", info["lsqr_iterations"])
