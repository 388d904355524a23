"""Wall time of the pipelined batched run (pinned host in/out) per chunk size."""
import time, numpy as np, torch
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import nnls_gen as g, paper_cs_0408029_b200 as P
B = g.make_batch(seed=0)
arrs = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (B.nnz_off, B.rowptr, B.colind, B.vals, B.b)]
x = torch.empty(B.count * B.n, dtype=torch.float64).pin_memory()
S = P.BatchedSolver()
for chunk in (2048, 4096, 8192, 16384, 65536):
    for _ in range(2): S.run(B.count, B.m, B.n, *arrs, x_out=x, want_info=False, chunk=chunk)
    t = time.perf_counter()
    for _ in range(5): S.run(B.count, B.m, B.n, *arrs, x_out=x, want_info=False, chunk=chunk)
    dt = (time.perf_counter() - t) / 5
    print(chunk, round(dt * 1e3, 2), "ms", round(B.count / dt), "solves/s")
