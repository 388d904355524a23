"""Writes tests/golden/single_exchange_seeds.json: seeds of
nnls_gen.make_correlated(seed, 0.05) on which the CPU ORACLE (only) takes the
single-exchange branch of P:98-99 at least once with p_max = 3, and on which
brute force (oracle.brute_force) finds exactly one feasible partition.
Run: python tests/golden/make_single_exchange_seeds.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import nnls_gen as g  # noqa: E402
import oracle as O  # noqa: E402

out = []
for seed in range(4000):
    p = g.make_correlated(seed, 0.05)
    r = O.solve(p, lsqr_mode=0)
    if r["status"] == 0 and r["single_exchanges"] > 0:
        cnt, masks, _ = O.brute_force(p)
        if cnt == 1 and np.array_equal(masks[0], r["mask"]):
            out.append(dict(seed=seed, n=p.n, m=p.m, iterations=r["iterations"],
                            single_exchanges=r["single_exchanges"]))
    if len(out) >= 40:
        break
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "single_exchange_seeds.json")
with open(path, "w") as fh:
    json.dump({"generator": "nnls_gen.make_correlated(seed, corr=0.05)",
               "source": "oracle.solve(lsqr_mode=0) + oracle.brute_force", "cases": out}, fh, indent=1)
print(len(out), "cases ->", path)
