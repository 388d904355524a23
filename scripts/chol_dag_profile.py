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
p = prof.cpu().numpy().reshape(-1, 8)
p = p[p[:, 0] > 0]
base = p[:, 0].min()
print(" task   i   j  sm    start gathered  updated  Ljj-rdy factored published (us)")
for t, r in enumerate(p):
    meta = int(r[7])
    i, j, sm = meta >> 40, (meta >> 20) & 0xFFFFF, meta & 0xFFFFF

    def us(x):
        return (x - base) / 1e3 if x > 0 else float("nan")
    print(f"{t:5d} {i:3d} {j:3d} {sm:3d} {us(r[0]):8.1f} {us(r[1]):8.1f} {us(r[2]):8.1f} "
          f"{us(r[3]):8.1f} {us(r[4]):8.1f} {us(r[5]):9.1f}")
