"""Load one problem (CSR upload + validation + CSC + Gram) through the C ABI,
for profiling the ingest kernels:  python scripts/run_load.py [config] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import nnls_gen as g  # noqa: E402
import paper_cs_0408029_b200 as P  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
prob = g.make_problem(cfg, 0)
for _ in range(reps):
    S = P.setup(prob)
print("ok")
