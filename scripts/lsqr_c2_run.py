"""Config-2 solves on the host-driven loop (NNLS_NO_GRAPH) for ncu captures of
the final LSQR kernel: python scripts/lsqr_c2_run.py [reps]"""
import os
import sys

os.environ["NNLS_NO_GRAPH"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import nnls_gen as g  # noqa: E402
import paper_cs_0408029_b200 as P  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
prob = g.make_problem(2, 0)
S = P.setup(prob)
for _ in range(reps):
    x, info = S.solve()
torch.cuda.synchronize()
print(info)
