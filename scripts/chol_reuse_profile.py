"""Timeline of the LAST factorization of a full solve (the one with the
longest kept prefix): chain rows from the restart column, and the restart
task D(jq).  Debug hook nnls_debug_chol_profile."""
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
S.solve()
prof = torch.zeros(1200 * 8, dtype=torch.int64, device="cuda")
P.lib.nnls_debug_chol_profile.argtypes = [C.c_void_p]
P.lib.nnls_debug_chol_profile.restype = C.c_int32
P.lib.nnls_debug_chol_profile(C.c_void_p(prof.data_ptr()))
x, info = S.solve()
torch.cuda.synchronize()
P.lib.nnls_debug_chol_profile(C.c_void_p(0))
a = prof.cpu().numpy().reshape(-1, 8).astype(np.float64)
t0 = a[1198, 0]
print("iterations", info["iterations"], "free", info["free_count"])
print("restart task D(jq): start %.2f  published %.2f us" % ((a[1199, 0] - t0) / 1e3, (a[1199, 1] - t0) / 1e3))
print("   j    start  factored   joined  trtri-16 trtri-done  gemm-done  syrk-w0   end (us)")
for j in range(600):
    r = a[j]
    if r[0] > 0 and r[0] >= t0:
        v = [(x - t0) / 1e3 if x > 0 else float("nan") for x in (r[0], r[1], r[2], r[7], r[3], r[4], r[6], r[5])]
        print(f"{j:4d} " + " ".join(f"{x:9.1f}" for x in v))
