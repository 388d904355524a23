"""Pins for the NEXT-2 oracle extension (-m "not gpu"):

* or_condest -- the 1-norm condition estimate of M = L L^T that P:129 (Section
  3) takes from LAPACK dpocon (Hager's estimator with Higham's refinements,
  dlacn2's steps): SPEC's closed forms, soundness against the
  exact kappa_1 from a dense inverse (an estimator of ||M^-1||_1 never exceeds
  it), quality on a random SPD suite;
* lsqr_mode 3 (adaptive, "to determine when a switch to a final step
  with LSQR is necessary"): below the threshold x is the normal-equations x
  bit for bit (mode 0), above it the LSQR x bit for bit (mode 1);
* notpd_fallback ("may fail entirely"): a rank-deficient A_F no
  longer aborts the solve; the objective reaches the constrained optimum.
"""
import numpy as np
import pytest
from scipy.optimize import nnls as scipy_nnls

import nnls_gen as g
import oracle as O


def exact_kappa1(M):
    return np.abs(M).sum(0).max() * np.abs(np.linalg.inv(M)).sum(0).max()


@pytest.mark.parametrize("d,norm,want", [([1.0, 1.0, 1.0], 1.0, 1.0),
                                         ([1.0, 100.0], 100.0, 100.0),
                                         ([1.0, 1e-6], 1.0, 1e6)])
def test_condest_closed_forms(d, norm, want):
    L, rc = O.cholesky(np.diag(d))
    assert rc == 0
    assert O.condest(L, norm) == pytest.approx(want, rel=1e-14)


def test_norm1_definition():
    M = np.array([[4.0, -2.0, 1.0], [-2.0, 5.0, 0.5], [1.0, 0.5, 3.0]])
    assert O.norm1(M) == 7.5                     # column 1: 2 + 5 + 0.5


def test_condest_sound_and_sharp():
    """Random SPD suite (dimension <= 50, kappa up to ~1e8): the estimate never
    exceeds the exact kappa_1 (beyond rounding) and is within 10x of it on >= 95%."""
    rng = np.random.default_rng(123)
    ratios = []
    for t in range(200):
        f = int(rng.integers(1, 51))
        B = rng.standard_normal((f + int(rng.integers(0, 20)), f))
        B[:, : max(1, f // 4)] *= 10.0 ** rng.uniform(-4, 0)      # spread the column scales
        M = B.T @ B + 1e-3 * np.eye(f)
        L, rc = O.cholesky(M)
        assert rc == 0
        est = O.condest(L, O.norm1(M))
        ex = exact_kappa1(M)
        assert est <= ex * (1 + 1e-9), (t, est, ex)
        assert est >= 1.0 - 1e-12
        ratios.append(est / ex)
    assert np.mean(np.array(ratios) >= 0.1) >= 0.95


def _ill_conditioned(seed, scale):
    """A with one column scaled by `scale`: kappa(A^T A) ~ 1/scale^2; b = A x
    with x >= 1, so every column stays in F."""
    rng = np.random.default_rng(seed)
    A = np.round(rng.standard_normal((40, 8)) * 64) / 64
    A[:, 0] *= scale
    x = 1.0 + np.abs(rng.standard_normal(8))
    b = A @ x + 1e-9 * rng.standard_normal(40)
    return g.from_dense(A, b)


def test_adaptive_mode_switch():
    well = g.make_problem(0, 2)
    r0 = O.solve(well, lsqr_mode=0)
    r1 = O.solve(well, lsqr_mode=1)
    r3 = O.solve(well, lsqr_mode=3)
    assert r3["refined"] == 0 and 1.0 <= r3["kappa"] < 1e4
    assert np.array_equal(r3["x"], r0["x"]) and r3["lsqr_iterations"] == 0
    ill = _ill_conditioned(5, 1e-5)
    assert O.solve(ill)["free_count"] == 8
    s0 = O.solve(ill, lsqr_mode=0)
    s1 = O.solve(ill, lsqr_mode=1)
    s3 = O.solve(ill, lsqr_mode=3)
    assert s3["kappa"] * 2.0 ** -52 > 1e-8 and s3["refined"] == 1
    assert np.array_equal(s3["x"], s1["x"]) and s3["lsqr_iterations"] == s1["lsqr_iterations"]
    assert np.array_equal(s3["mask"], s0["mask"])          # the pivoting is mode-independent
    assert r1["refined"] == 1 and r0["refined"] == 0
    # the estimate is the final (A^T A)_FF's: recompute it from the final F
    F = np.flatnonzero(s3["mask"])
    A = ill.dense()
    M = A[:, F].T @ A[:, F]
    assert s3["kappa"] <= exact_kappa1(M) * 1.01 and s3["kappa"] >= exact_kappa1(M) / 10


def test_notpd_fallback_reaches_optimum():
    """Duplicate column (rank-deficient A): without the fallback the solve
    stops at NOT_PD (reading c13); with it the loop continues on an LSQR x_F
    and reaches the optimal objective (unique even when x is not)."""
    p = g.make_problem(0, 0)
    A = p.dense()
    A = np.concatenate([A, A[:, :1]], axis=1)
    q = g.from_dense(A, p.b)
    if (A.T @ p.b)[0] <= 0:
        pytest.skip("column 0 never enters F")
    r = O.solve(q)
    assert r["status"] == 7
    rf = O.solve(q, notpd_fallback=1)
    assert rf["status"] == 0 and rf["lsqr_fallbacks"] >= 1
    xs, _ = scipy_nnls(A, q.b, maxiter=50 * q.n)
    opt = 0.5 * np.sum((A @ xs - q.b) ** 2)
    assert rf["objective"] <= opt * (1 + 1e-9) + 1e-12
    assert rf["x"].min() >= 0.0
