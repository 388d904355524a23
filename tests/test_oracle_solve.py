"""Pins for the oracle's whole block-principal-pivoting solve (-m "not gpu").

* hand examples, closed forms (A = I, n = 1,
  A^T b <= 0 -> 0 iterations, disjoint column supports -> 1 iteration,
  b = A x* with x* >= 0 -> x = x*);
* brute force over all 2^n complementary partitions (n <= 12): the feasible
  partition is unique for nondegenerate instances and equals the oracle's F;
* scipy.optimize.nnls (Lawson-Hanson, an independent algorithm) on the same
  unique minimiser, at the BASELINE config shapes;
* KKT / LCP invariants of Eq. 3, reading c18;
* the single-exchange fallback on seed-searched instances
  (tests/golden/single_exchange_seeds.json), checked against brute force.
"""
import json
import os

import numpy as np
import pytest
from scipy.optimize import nnls as scipy_nnls

import nnls_gen as g
import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
SINGLES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "single_exchange_seeds.json")))


def rel(a, b):
    d = np.abs(b).max()
    return np.abs(a - b).max() / (d if d > 0 else 1.0)


def kkt_ok(prob, r):
    x = r["x"]
    A = prob.dense()
    c = A.T @ prob.b
    yp = A.T @ (A @ x - prob.b)
    cs = max(1.0, np.abs(c).max())
    assert x.min() >= 0.0
    assert yp.min() >= -1e-10 * cs
    assert abs(x @ yp) <= 1e-10 * max(1.0, np.abs(x).max() * np.abs(c).max())
    # the algorithm's own (x, y) are exactly complementary
    assert np.all(r["x"][r["mask"] == 0] == 0) and np.all(r["y"][r["mask"] == 1] == 0)


@pytest.mark.parametrize("case", GOLD["bpp_solve"], ids=lambda c: c["cite"])
def test_bpp_golden(case):
    p = g.from_dense(case["A"], case["b"])
    r = O.solve(p)
    assert r["status"] == 0
    assert np.allclose(r["x"], case["x"], atol=1e-14)
    assert np.allclose(r["y"], case["y"], atol=1e-14)
    if "objective" in case:
        assert abs(r["objective"] - case["objective"]) < 1e-14


def test_identity_closed_form():
    rng = np.random.default_rng(0)
    b = np.round(rng.standard_normal(30) * 64) / 64
    r = O.solve(g.from_dense(np.eye(30), b), lsqr_mode=0)
    assert np.array_equal(r["x"], np.maximum(b, 0))
    r1 = O.solve(g.from_dense(np.eye(30), b))                 # + final LSQR
    assert np.allclose(r1["x"], np.maximum(b, 0), rtol=1e-15, atol=0)
    assert np.array_equal(r["y"], np.maximum(-b, 0) * (r["mask"] == 0))
    assert r["iterations"] == 1


def test_single_column_closed_form():
    rng = np.random.default_rng(1)
    for _ in range(10):
        a = np.round(rng.standard_normal((9, 1)) * 16) / 16
        b = np.round(rng.standard_normal(9) * 16) / 16
        r = O.solve(g.from_dense(a, b), lsqr_mode=0)
        want = max((a[:, 0] @ b) / (a[:, 0] @ a[:, 0]), 0.0)
        assert abs(r["x"][0] - want) <= 1e-15 * max(1, abs(want))


def test_nonpositive_atb_zero_iterations():
    A = np.array([[1.0, 2.0], [0.5, 1.0], [0.0, 3.0]])
    b = -A @ np.array([1.0, 0.5])          # A^T b = -A^T A (1, .5) < 0 componentwise
    assert np.all(A.T @ b < 0)
    r = O.solve(g.from_dense(A, b))
    assert r["iterations"] == 0 and r["free_count"] == 0
    assert np.all(r["x"] == 0)


def test_disjoint_supports_one_iteration():
    """Columns with disjoint row supports: G is diagonal, x_i = max(c_i/G_ii, 0),
    reached in exactly one block exchange."""
    rng = np.random.default_rng(2)
    n, per = 12, 3
    A = np.zeros((n * per, n))
    for j in range(n):
        A[j * per:(j + 1) * per, j] = np.round(rng.standard_normal(per) * 32) / 32 + 0.0
    A[A == 0] = 0.0
    b = np.round(rng.standard_normal(n * per) * 32) / 32
    r = O.solve(g.from_dense(A, b), lsqr_mode=0)
    G = (A * A).sum(0)
    c = A.T @ b
    assert r["iterations"] == 1
    assert np.allclose(r["x"], np.maximum(c / G, 0), rtol=1e-15, atol=0)


def test_exact_nonnegative_rhs_recovers_x():
    """b = A x* with x* >= 0 (BASELINE north_star's closed form): x = x*,
    residual 0.  Config-3-like generator at test size."""
    p = g.make_problem(dict(m=300, n=150, density=0.05, rhs="degenerate"), seed=4)
    r = O.solve(p)
    assert r["status"] == 0
    assert rel(r["x"], p.x_gen) < 1e-12
    assert r["objective"] < 1e-20
    assert np.all(r["mask"][p.x_gen > 0] == 1)       # supp(x*) subset of F


@pytest.mark.parametrize("seed", range(60))
def test_brute_force_unique_partition(seed):
    rng = np.random.default_rng([seed, 5])
    n = int(rng.integers(2, 13))
    m = n + int(rng.integers(1, 8))
    d = float(rng.choice([1.0, 0.6, 0.35]))
    p = g.make_problem(dict(m=m, n=n, density=d), seed=seed)
    r = O.solve(p, lsqr_mode=0)
    cnt, masks, x_bf = O.brute_force(p)
    assert r["status"] == 0
    assert cnt == 1, "nondegenerate instance has a unique feasible partition"
    assert np.array_equal(masks[0], r["mask"])
    assert rel(r["x"], x_bf) < 1e-12
    kkt_ok(p, r)


@pytest.mark.parametrize("case", SINGLES["cases"][:25], ids=lambda c: f"seed{c['seed']}")
def test_single_exchange_branch(case):
    """P:98-99 fallback: instances (found by the committed script, oracle-only)
    whose block exchanges stall; the final F still equals brute force's."""
    p = g.make_correlated(case["seed"], 0.05)
    r = O.solve(p, lsqr_mode=0, trace_cap=200)
    assert r["status"] == 0
    assert r["single_exchanges"] == case["single_exchanges"] >= 1
    assert any(t["branch"] == 2 for t in r["trace"])
    cnt, masks, x_bf = O.brute_force(p)
    assert cnt == 1 and np.array_equal(masks[0], r["mask"])
    # N is non-increasing and p stays in [0, 3]
    ks = [t["k"] for t in r["trace"]]
    Nrun, best = [], 10**9
    for k in ks:
        best = min(best, k)
        Nrun.append(best)
    assert all(a >= b for a, b in zip(Nrun, Nrun[1:]))


@pytest.mark.parametrize("cfg,seed", [(0, 0), (0, 1), (0, 2), (1, 0), (3, 0)])
def test_matches_scipy_nnls(cfg, seed):
    p = g.make_problem(cfg, seed)
    r = O.solve(p)
    assert r["status"] == 0
    xs, _ = scipy_nnls(p.dense(), p.b, maxiter=50 * p.n)
    assert rel(r["x"], xs) < 1e-9
    assert rel(r["x_ne"], xs) < 1e-9
    kkt_ok(p, r)


def test_batch_matches_scipy_and_single():
    B = g.make_batch(seed=0, start=0, count=48)
    out = O.solve_batched(B, threads=2)
    for q in range(0, 48, 7):
        p = B.problem(q)
        r = O.solve(p)
        assert np.array_equal(out["x"][q], r["x"]) and np.array_equal(out["mask"][q], r["mask"])
        xs, _ = scipy_nnls(p.dense(), p.b, maxiter=50 * p.n)
        assert rel(r["x"], xs) < 1e-9
        kkt_ok(p, r)
    assert np.all(out["status"] == 0)


def test_iteration_limit_and_not_pd():
    p = g.make_problem(0, 0)
    r = O.solve(p, max_iter=1)
    assert r["status"] == 8 and r["iterations"] == 1          # reading c12
    A = p.dense()
    A = np.concatenate([A, A[:, :1]], axis=1)                  # duplicate column: rank deficient
    q = g.from_dense(A, p.b)
    r = O.solve(q)
    # column 0 and its duplicate both enter F only if both are infeasible at the
    # start; c_0 = c_dup so they move together -> NOT_PD on that solve
    if (A.T @ p.b)[0] > 0:
        assert r["status"] == 7


# ---------------------------------------------------------------- or_kkt pins
# KKT report of Eq. 3 with the independent dual y' = A^T (A x - b).
# Hand-computed on the S:334 matrix A = [[1,0],[0,1],[1,1]], b = (-1,1,0):
#   x = (0, .5):  r = A x - b = (1, -.5, .5),  y' = A^T r = (1.5, 0)
#   x = (1, 1):   r = (2, 0, 2),               y' = (4, 2)
#   x = (.5, -1): r = (1.5, -2, -.5),          y' = (1, -2.5)
# Every field is distinct across the cases, so a sign error in y' (or r), a
# dropped |.| in the complementarity, or a min/max swap fails one of them.
KKT_HAND = [
    ((0.0, 0.5), dict(objective=0.75, kkt_min_x=0.0, kkt_min_y=0.0, kkt_max_comp=0.0, kkt_dot=0.0)),
    ((1.0, 1.0), dict(objective=4.0, kkt_min_x=1.0, kkt_min_y=2.0, kkt_max_comp=4.0, kkt_dot=6.0)),
    ((0.5, -1.0), dict(objective=3.25, kkt_min_x=-1.0, kkt_min_y=-2.5, kkt_max_comp=2.5, kkt_dot=3.0)),
]


@pytest.mark.parametrize("x,want", KKT_HAND, ids=["S334-optimum", "x=(1,1)", "x=(.5,-1)"])
def test_kkt_hand_cases(x, want):
    p = g.from_dense([[1, 0], [0, 1], [1, 1]], [-1, 1, 0])
    got = O.kkt(p, np.array(x))
    for k, v in want.items():
        assert got[k] == v, (k, got[k], v)


def test_kkt_matches_dense_definition():
    """Random x on a config-0 problem: every field equals its definition
    evaluated densely with numpy (y' = A^T (A x - b))."""
    p = g.make_problem(0, 3)
    rng = np.random.default_rng(9)
    x = rng.standard_normal(p.n)
    A = p.dense()
    r = A @ x - p.b
    yp = A.T @ r
    got = O.kkt(p, x)
    assert abs(got["objective"] - 0.5 * r @ r) <= 1e-12 * (r @ r)
    assert got["kkt_min_x"] == x.min()
    assert abs(got["kkt_min_y"] - yp.min()) <= 1e-12 * np.abs(yp).max()
    assert abs(got["kkt_max_comp"] - np.abs(x * yp).max()) <= 1e-12 * np.abs(x * yp).max()
    assert abs(got["kkt_dot"] - x @ yp) <= 1e-12 * np.abs(x * yp).sum()


# --------------------------------------------------------- or_brute_force pins
def test_brute_force_identity_closed_form():
    """A = I: the feasible partition is unique, F = {i : b_i > 0},
    x = max(b, 0); every b_i = 0 exactly doubles the count (i in F or in G
    both give x_i = y_i = 0)."""
    b = np.array([3.0, -2.0, 0.5, -0.25, 1.0, -7.0])
    cnt, masks, x = O.brute_force(g.from_dense(np.eye(6), b))
    assert cnt == 1
    assert np.array_equal(masks[0], (b > 0).astype(np.uint8))
    assert np.array_equal(x, np.maximum(b, 0))
    b0 = np.array([3.0, 0.0, -1.0, 0.0])
    cnt, masks, _ = O.brute_force(g.from_dense(np.eye(4), b0))
    assert cnt == 4
    got = sorted(tuple(m) for m in masks)
    assert got == sorted([(1, a, 0, c) for a in (0, 1) for c in (0, 1)])


def test_brute_force_diagonal_gram_closed_form():
    """Columns with disjoint row supports: G = diag(g_i), y_i = g_i x_i - c_i,
    so F = {i : c_i > 0} and x_i = c_i / g_i there (no enumeration needed)."""
    rng = np.random.default_rng(12)
    n, per = 9, 2
    A = np.zeros((n * per, n))
    for j in range(n):
        A[j * per:(j + 1) * per, j] = np.round(rng.standard_normal(per) * 16) / 16 + 2.0
    b = np.round(rng.standard_normal(n * per) * 16) / 16
    c = A.T @ b
    gd = (A * A).sum(0)
    cnt, masks, x = O.brute_force(g.from_dense(A, b))
    assert cnt == 1
    assert np.array_equal(masks[0], (c > 0).astype(np.uint8))
    assert np.allclose(x, np.where(c > 0, c / gd, 0.0), rtol=1e-15, atol=0)


def test_brute_force_counts_all_feasible_partitions():
    """A problem with two KKT points is impossible for full-rank A (unique
    minimiser), so a rank-deficient A (two equal columns) with c > 0 on them
    has exactly the F's that put the weight on either copy -- but both copies
    together make the Gram singular (skipped, NOT_PD).  Expect 2 partitions."""
    A = np.array([[1.0, 1.0], [2.0, 2.0], [0.0, 0.0]])
    b = np.array([1.0, 1.0, 0.0])
    cnt, masks, _ = O.brute_force(g.from_dense(A, b))
    assert cnt == 2
    assert sorted(tuple(m) for m in masks) == [(0, 1), (1, 0)]
