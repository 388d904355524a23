"""Time step_normal_solve (factor + back-solve) for several |F| on one Gram:
python scripts/chol_timing_sweep.py [config] f1 f2 ..."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import nnls_gen as g  # noqa: E402
import paper_cs_0408029_b200 as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
fs = [int(v) for v in sys.argv[2:]] or [1000, 2000, 3000, 3981, 4500, 5000]
prob = g.make_problem(cfg, 0)
S = P.setup(prob, trace=1)
x, info = S.solve()
print("solve trace f:", [t["f"] for t in S.trace()])
G, c = S.gram()
Gd = torch.tensor(G, device="cuda")
cd = torch.tensor(c, device="cuda")
rng = np.random.default_rng(0)
for f in fs:
    F = np.sort(rng.choice(prob.n, f, replace=False)).astype(np.int32)
    Fd = torch.tensor(F, device="cuda")
    xF = torch.empty(f, dtype=torch.float64, device="cuda")
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        P.step_normal_solve(prob.n, Gd, cd, Fd, xF)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"f={f}: {dt * 1e3:.2f} ms")
