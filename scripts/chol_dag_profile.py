"""Per-task timeline of the Cholesky DAG (debug hook nnls_debug_chol_profile):
prints, per task (i,j), start / gathered / updated / L_jj-ready / factored /
published times (us) relative to the first task start.

    python scripts/chol_dag_profile.py [config] [f]
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import nnls_gen as g  # noqa: E402
import paper_cs_0408029_b200 as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
f_target = int(sys.argv[2]) if len(sys.argv) > 2 else 522
prob = g.make_problem(cfg, 0)
S = P.setup(prob)
G, c = S.gram()
n = prob.n
rng = np.random.default_rng(0)
F = np.sort(rng.choice(n, f_target, replace=False)).astype(np.int32)
Gd = torch.tensor(G, device="cuda")
cd = torch.tensor(c, device="cuda")
Fd = torch.tensor(F, device="cuda")
xF = torch.empty(f_target, dtype=torch.float64, device="cuda")
prof = torch.zeros(20000 * 8, dtype=torch.int64, device="cuda")
P.lib.nnls_debug_chol_profile.argtypes = [C.c_void_p]
P.lib.nnls_debug_chol_profile.restype = C.c_int32
for rep in range(3):
    prof.zero_()
    P.lib.nnls_debug_chol_profile(C.c_void_p(prof.data_ptr()))
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    P.step_normal_solve(n, Gd, cd, Fd, xF)
    t1.record()
    torch.cuda.synchronize()
    P.lib.nnls_debug_chol_profile(C.c_void_p(0))
print("step_normal_solve ms", t0.elapsed_time(t1))
allp = prof.cpu().numpy().reshape(-1, 8)
hp = allp[1000:1200]
p = allp[:600]
p = p[p[:, 0] > 0]
base = p[:, 0].min()
# chain CTA: one row per tile column j
print("   j    start  factored  trtri-16 trtri-done    joined  gemm-done  end (us)")
for j, r in enumerate(p):
    v = [(x - base) / 1e3 if x > 0 else float("nan") for x in (r[0], r[1], r[7], r[3], r[2], r[4], r[5])]
    print(f"{j:4d} " + " ".join(f"{x:9.1f}" for x in v))
if len(p) > 1:
    d = np.diff(p[:, 0]) / 1e3
    print("per-column period us: mean %.2f  min %.2f  max %.2f" % (d.mean(), d.min(), d.max()))
    q = p[:-1]
    print("potrf (+deferred SYRK) %.2f  trtri (7 warps) %.2f [diag+L8+L16 %.2f, L32 %.2f]  "
          "join (wait partials) %.2f  gemm %.2f  end %.2f" % (
        ((q[:, 1] - q[:, 0]) / 1e3).mean(), ((q[:, 3] - q[:, 1]) / 1e3).mean(),
        ((q[:, 7] - q[:, 1]) / 1e3).mean(), ((q[:, 3] - q[:, 7]) / 1e3).mean(),
        ((q[:, 2] - q[:, 3]) / 1e3).mean(),
        ((q[:, 4] - q[:, 2]) / 1e3).mean(), ((q[:, 5] - q[:, 4]) / 1e3).mean()))
print("helpers, per column j (us, same base): P(j+1,j) last-update-start / published, T(j+1,j-1) published, P(j+1,j+1)... ")
for j in range(len(p)):
    h = hp[j]
    def us(x):
        return (x - base) / 1e3 if x > 0 else float("nan")
    print(f"{j:4d}  P(j+1,j) upd-done {us(h[4]):8.1f} pub {us(h[0]):8.1f} | T(j+1,j-1) pub {us(h[1]):8.1f} | "
          f"P(j,j) pub {us(h[2]):8.1f} | chain needs sub at {us(p[j][2]):8.1f}")
# POTRF panels of the chain (rows 600+4j, clock64 cycles: after (a), warp 0
# panel done, (c) warps done; row 600+4j+3 slot 0: POTRF entry)
pp = allp[600:600 + 4 * len(p)].reshape(len(p), 4, 8).astype(np.int64)
print("POTRF per panel (cycles): (a) lookahead incl. previous sync | (b) panel factor (warp 0) | (c) strips (warp 2)")
for j in [jj for jj in (1, 2, 3, 30, 50) if jj < len(p)]:
    t_start = [pp[j][3][0] if k == 0 else pp[j][1][k - 1] for k in range(8)]
    row = []
    for k in range(8):
        if pp[j][0][k] <= 0:
            break
        row.append("%d: %d|%d|%s" % (k, pp[j][0][k] - t_start[k], pp[j][1][k] - pp[j][0][k],
                                     str(pp[j][2][k] - pp[j][0][k]) if pp[j][2][k] > 0 else "-"))
    print("  j=%d total %d  " % (j, pp[j][1][7] - pp[j][3][0]) + "  ".join(row))
# back substitution chain (rows 900+J, slot 0): x_J computed on the chain CTA
bs = allp[900:900 + 100, 0]
idx = np.flatnonzero(bs > 0)
if idx.size:
    t = bs[idx]
    order = np.argsort(t)
    print("backsolve chain: x_J done at (us from the first):",
          " ".join("J%d:%.2f" % (idx[k], (t[k] - t.min()) / 1e3) for k in order))
    full = allp[900:900 + 100]
    t0 = t.min()
    print("  J   N armed   a_J in   x_J done   x_J published (us)")
    for k in order:
        J = idx[k]
        r = full[J]
        print("  %2d  %8.2f %8.2f %8.2f %8.2f" % (J, *[(v - t0) / 1e3 if v > 0 else float('nan') for v in (r[2], r[1], r[0], r[3])]))
