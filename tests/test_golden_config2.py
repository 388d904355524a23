"""Pins for the cached config-2 oracle results (tests/golden/config2_seed*.npz,
written by tests/golden/make_config2_golden.py from oracle/ only), -m "not gpu":

* the file is what the oracle produces today (seed 0 re-solved, bitwise);
* its x satisfies the KKT conditions of Eq. 3 recomputed
  independently with scipy.sparse (x >= 0, y' = A^T(Ax - b) >= 0, x_i y'_i ~ 0),
  its F is the support structure of x, and the trace is a valid run of
  P:89-101 (|F| matches, the branch rule and the N/p counters are consistent).
"""
import os

import numpy as np
import pytest

sp = pytest.importorskip("scipy.sparse")

import nnls_gen as g  # noqa: E402
import oracle as O  # noqa: E402

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(seed):
    return np.load(os.path.join(HERE, f"config2_seed{seed}.npz"))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_golden_kkt_and_trace(seed):
    gold = load(seed)
    prob = g.make_problem(2, seed)
    n = prob.n
    mask = np.unpackbits(gold["mask_bits"])[:n].astype(bool)
    x = gold["x"]
    A = sp.csr_matrix((prob.vals, prob.colind, prob.rowptr), shape=(prob.m, n))
    c = A.T @ prob.b
    y = A.T @ (A @ x - prob.b)
    scale = np.abs(c).max()
    assert int(gold["status"]) == 0 and mask.sum() == int(gold["free_count"])
    assert x.min() >= 0 and np.all(x[~mask] == 0)
    assert np.abs(y[mask]).max() <= 1e-9 * scale
    assert y[~mask].min() >= -1e-9 * scale
    # trace: iteration i's |F| is the last one's for the final F; block exchanges
    # follow P:91-97 (N strictly decreases on branch 0, p counts down on 1)
    kbf = gold["trace_kbf"]
    assert len(kbf) == int(gold["iterations"]) and kbf[-1][2] == mask.sum()
    N, p = n + 1, 3
    for k, br, _ in kbf:
        if k < N:
            assert br == 0
            N, p = k, 3
        elif p > 0:
            assert br == 1
            p -= 1
        else:
            assert br == 2
    # decision margins: nothing within 1e3 x of the 1e-12 tolerance
    assert gold["trace_below"].max() < 1e-15 and gold["trace_above"].min() > 1e-9


def test_golden_is_current_oracle_output():
    """Seed 0 re-solved by the oracle (~40 s): every stored field bit-equal."""
    gold = load(0)
    prob = g.make_problem(2, 0)
    r = O.solve(prob, trace_cap=10 * prob.n + 2)
    assert np.array_equal(np.packbits(r["mask"].astype(np.uint8)), gold["mask_bits"])
    assert r["iterations"] == int(gold["iterations"])
    assert np.array_equal(r["x"], gold["x"]) and np.array_equal(r["x_ne"], gold["x_ne"])
    assert [(t["k"], t["branch"], t["f"]) for t in r["trace"]] == [tuple(v) for v in gold["trace_kbf"].tolist()]
