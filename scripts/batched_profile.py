"""Per-phase cycles of the batched kernel (CTA 0's problems; debug hook
nnls_debug_batched_profile):  python scripts/batched_profile.py [count]"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import nnls_gen as g  # noqa: E402
import paper_cs_0408029_b200 as P  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
B = g.make_batch(seed=0, start=0, count=count)
S = P.BatchedSolver().load_batch(B)
S.solve()
prof = torch.zeros(16, dtype=torch.int64, device="cuda")
P.lib.nnls_debug_batched_profile.argtypes = [C.c_void_p]
P.lib.nnls_debug_batched_profile(C.c_void_p(prof.data_ptr()))
out = S.solve()
P.lib.nnls_debug_batched_profile(C.c_void_p(0))
p = prof.cpu().numpy()
nprob = max(int(p[9]), 1)
names = ["load", "column view", "Gram", "decide+compact", "gather+Cholesky", "back subst",
         "scatter+dual", "hand-off", "-", "-", "B: load", "B: LSQR", "B: output+KKT"]
tot = p[:8].sum() + p[10:13].sum()
print(f"CTA 0 problems: {nprob}; cycles per problem {tot / nprob:.0f} ({tot / nprob / 1965:.1f} us at 1965 MHz)")
for i, nm in enumerate(names):
    if nm == "-":
        continue
    cnt = max(int(p[13]), 1) if i >= 10 else nprob
    print(f"  {nm:18s} {p[i] / cnt:9.0f} cycles  {100 * p[i] / tot:5.1f}%")
print("mean pivot iterations", float(out["info"]["iterations"].mean()), "mean lsqr itn",
      float(out["info"]["lsqr_iterations"].mean()), "mean f", float(out["info"]["free_count"].mean()))
