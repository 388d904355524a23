#!/usr/bin/env python
"""Writes tests/golden/config2_seed{0,1,2}.npz: the CPU oracle's result on the
full BASELINE config-2 problem (40000 x 8000 CSR, 0.5% nonzeros) for seeds 0-2.

Calls ONLY oracle/ (and the seeded input generator nnls_gen/); nothing here
comes from the CUDA path.  The oracle needs ~25 s per solve, too long to run
inside the GPU parity test three times, so its output is cached here (SURVEY.md
§8(c)/(d): "run it once per seed and cache F, iterations and x for the GPU
parity re-checks").  F and the iteration count are defined only by the
algorithm (the pseudo-code), which the oracle follows step by step.

    python tests/golden/make_config2_golden.py [seed ...]

Stored per seed: the final F (packed bits), iterations, single exchanges,
|F|, the per-iteration trace (k, branch, |F|, nearest values below/above the
1e-12 tolerance), the final x (LSQR mode 1), the last normal-equations
x, LSQR iteration count, objective and a sha256 of the input arrays (so a
changed generator is detected instead of silently comparing other inputs).
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import nnls_gen as g  # noqa: E402
import oracle as O  # noqa: E402


def input_digest(prob) -> str:
    h = hashlib.sha256()
    for a in (prob.rowptr, prob.colind, prob.vals, prob.b):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def solve_golden(seed: int) -> dict:
    prob = g.make_problem(2, seed=seed)
    r = O.solve(prob, trace_cap=10 * prob.n + 2)
    tr = r["trace"]
    return dict(
        seed=np.int64(seed),
        digest=np.array(input_digest(prob)),
        mask_bits=np.packbits(r["mask"].astype(np.uint8)),
        n=np.int64(prob.n),
        status=np.int64(r["status"]),
        iterations=np.int64(r["iterations"]),
        single_exchanges=np.int64(r["single_exchanges"]),
        free_count=np.int64(r["free_count"]),
        lsqr_iterations=np.int64(r["lsqr_iterations"]),
        objective=np.float64(r["objective"]),
        trace_kbf=np.array([[t["k"], t["branch"], t["f"]] for t in tr], dtype=np.int64),
        trace_below=np.array([t["below_tol"] for t in tr]),
        trace_above=np.array([t["above_tol"] for t in tr]),
        x=r["x"],
        x_ne=r["x_ne"],
    )


def main(seeds):
    for s in seeds:
        t0 = time.time()
        d = solve_golden(s)
        path = os.path.join(HERE, f"config2_seed{s}.npz")
        np.savez_compressed(path, **d)
        print(f"seed {s}: iterations={int(d['iterations'])} |F|={int(d['free_count'])} "
              f"lsqr={int(d['lsqr_iterations'])} ({time.time() - t0:.1f} s) -> {path}")


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [0, 1, 2])
