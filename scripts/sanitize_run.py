"""Small solves for compute-sanitizer (memcheck / racecheck / synccheck):
config 0 (graph path and host-driven loop), config 1 (restart chains, the
cluster LSQR), a config-2-shaped problem at reduced size for the grid LSQR,
and a 64-problem config-4 batch -- each checked against the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import nnls_gen as g  # noqa: E402
import oracle as O  # noqa: E402
import paper_cs_0408029_b200 as P  # noqa: E402


def check(prob, **kw):
    S = P.setup(prob, trace=1)
    x, info = S.solve()
    r = O.solve(prob)
    assert info["status"] == r["status"] and np.array_equal(S.free_set(), r["mask"]), "parity"
    assert np.abs(x - r["x"]).max() <= 1e-9 * max(np.abs(r["x"]).max(), 1e-300)
    return info


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    print("config0", check(g.make_problem(0, 0))["iterations"])
    if which != "quick":
        os.environ["NNLS_NO_GRAPH"] = "1"
        print("config0 host loop", check(g.make_problem(0, 1))["iterations"])
        del os.environ["NNLS_NO_GRAPH"]
        print("config1", check(g.make_problem(1, 0))["iterations"])
        os.environ["NNLS_NO_CLUSTER"] = "1"
        print("grid lsqr", check(g.make_problem(dict(m=1200, n=600, density=0.02), 2))["iterations"])
        del os.environ["NNLS_NO_CLUSTER"]
    B = g.make_batch(seed=0, start=0, count=64)
    out = P.BatchedSolver().load_batch(B).solve()
    rb = O.solve_batched(B, threads=1)
    assert np.array_equal(out["mask"].reshape(64, B.n), rb["mask"])
    print("batched 64 ok")


if __name__ == "__main__":
    main()
