"""Pins for the CPU oracle's step functions (-m "not gpu").

Each check ties the oracle to something other than itself: hand examples
(tests/golden/spec_examples.json, cited), exact integer arithmetic, library
routines (numpy / scipy), or invariants that a dropped term, wrong sign or
transposed operand would break.
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse
import scipy.sparse.linalg

import nnls_gen as g
import oracle as O

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _dense_problem(A, b=None):
    A = np.asarray(A, dtype=float)
    if b is None:
        b = np.zeros(A.shape[0])
    return g.from_dense(A, b)


# ----------------------------------------------------------------- Gram (a1)
@pytest.mark.parametrize("case", GOLD["gram"], ids=lambda c: c["cite"])
def test_gram_golden(case):
    G, c = O.gram(_dense_problem(case["A"]))
    assert np.array_equal(G, np.array(case["G"], dtype=float))


@pytest.mark.parametrize("cfg", [dict(m=60, n=25, density=0.3), dict(m=200, n=100, density=0.1)])
def test_gram_exact_integer(cfg):
    """Quantized inputs: G and c are exact, so they equal the integer-arithmetic
    product bit for bit (pins both the terms and the symmetric layout)."""
    p = g.make_problem(cfg, seed=3)
    G, c = O.gram(p)
    Ai = np.round(p.dense() * g.Q_A).astype(object)
    bi = np.round(p.b * g.Q_B).astype(np.int64).astype(object)
    Gi = Ai.T.dot(Ai)
    ci = Ai.T.dot(bi)
    assert np.array_equal(G, np.array(Gi, dtype=float) / g.Q_A**2)
    assert np.array_equal(c, np.array(ci, dtype=float) / (g.Q_A * g.Q_B))
    assert np.array_equal(G, G.T)


def test_gram_raw_matches_numpy():
    p = g.make_problem(dict(m=80, n=30, density=0.4), seed=1, raw=True)
    G, c = O.gram(p)
    A = p.dense()
    assert np.allclose(G, A.T @ A, rtol=1e-14, atol=1e-13)
    assert np.allclose(c, A.T @ p.b, rtol=1e-14, atol=1e-13)


# ----------------------------------------------------------- gather (a4)
@pytest.mark.parametrize("case", GOLD["gram_submatrix"], ids=lambda c: c["cite"])
def test_gather_golden(case):
    G, _ = O.gram(_dense_problem(case["A"]))
    assert np.array_equal(O.gather(G, case["sel"]), np.array(case["M"], dtype=float))


def test_gather_equals_fancy_index():
    rng = np.random.default_rng(0)
    G = rng.standard_normal((40, 40))
    F = np.sort(rng.choice(40, 17, replace=False))
    assert np.array_equal(O.gather(G, F), G[np.ix_(F, F)])


# --------------------------------------------------------- Cholesky (a5, a6)
@pytest.mark.parametrize("case", GOLD["factorize"], ids=lambda c: c["cite"])
def test_cholesky_golden(case):
    L, rc = O.cholesky(np.array(case["M"], dtype=float))
    if "not_pd_column" in case:
        assert rc == -(case["not_pd_column"] + 1)
    else:
        assert rc == 0
        assert np.array_equal(L, np.array(case["L"], dtype=float))


@pytest.mark.parametrize("case", GOLD["solve"], ids=lambda c: c["cite"])
def test_chol_solve_golden(case):
    L, rc = O.cholesky(np.array(case["M"], dtype=float))
    assert rc == 0
    assert np.allclose(O.chol_solve(L, case["rhs"]), case["x"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("seed", range(5))
def test_cholesky_random_spd(seed):
    rng = np.random.default_rng(seed)
    f = 5 + 11 * seed
    B = rng.standard_normal((f + 7, f))
    M = B.T @ B + f * np.eye(f)
    L, rc = O.cholesky(M)
    assert rc == 0
    n1 = np.abs(M).sum(0).max()
    assert np.abs(L @ L.T - M).sum(0).max() <= 1e-12 * n1
    assert np.array_equal(L, np.tril(L))
    assert np.allclose(L, np.linalg.cholesky(M), rtol=1e-12, atol=1e-12)
    r = rng.standard_normal(f)
    x = O.chol_solve(L, r)
    assert np.abs(M @ x - r).max() <= 1e-10 * n1 * np.abs(r).max()
    assert np.allclose(x, np.linalg.solve(M, r), rtol=1e-10, atol=1e-12)


def test_cholesky_not_pd_rank_deficient():
    A = np.array([[1.0, 2.0, 1.0], [0.0, 1.0, 1.0], [1.0, 3.0, 2.0], [2.0, 0.0, 2.0]])
    A[:, 2] = A[:, 0] + A[:, 1] * 0.0 + A[:, 0] * 0.0  # duplicate column 0
    G, _ = O.gram(_dense_problem(A))
    _, rc = O.cholesky(G)
    assert rc == -3


# ------------------------------------------------ unconstrained LS on F (Eq.4)
@pytest.mark.parametrize("case", GOLD["unconstrained_ls_normal_eq"], ids=lambda c: c["cite"])
def test_normal_eq_golden(case):
    p = _dense_problem(case["A"], case["b"])
    G, c = O.gram(p)
    sel = np.array(case["sel"])
    L, rc = O.cholesky(O.gather(G, sel))
    assert rc == 0
    assert np.allclose(O.chol_solve(L, c[sel]), case["xF"], atol=1e-15)


def test_normal_eq_matches_lstsq():
    """x_F from the normal equations equals lstsq(A_F, b) within c*kappa^2*eps."""
    p = g.make_problem(dict(m=300, n=120, density=0.1), seed=5)
    G, c = O.gram(p)
    F = np.arange(0, 120, 2)
    L, rc = O.cholesky(O.gather(G, F))
    xf = O.chol_solve(L, c[F])
    A = p.dense()[:, F]
    ref = np.linalg.lstsq(A, p.b, rcond=None)[0]
    kappa = np.linalg.cond(A)
    assert np.abs(xf - ref).max() / np.abs(ref).max() <= 10 * kappa**2 * 2.0**-52


# ----------------------------------------------------------- dual (Eq. 5)
@pytest.mark.parametrize("case", GOLD["dual_vector"], ids=lambda c: c["cite"])
def test_dual_golden(case):
    p = _dense_problem(case["A"], case["b"])
    n = p.n
    mask = np.zeros(n, dtype=np.uint8)
    mask[case["F"]] = 1
    x = np.zeros(n)
    x[case["F"]] = case["xF"]
    G, c = O.gram(p)
    for y in (O.dual_gram(G, c, mask, x), O.dual_eq5(p, mask, x)):
        assert np.allclose(y[case["G"]], case["yG"], atol=1e-15)
        assert np.all(y[case["F"]] == 0)


@pytest.mark.parametrize("seed", range(3))
def test_dual_gram_form_equals_eq5(seed):
    """Reading c4: (A^T A)_GF x_F - (A^T b)_G == A_G^T (A_F x_F - b) up to rounding."""
    p = g.make_problem(dict(m=400, n=150, density=0.08), seed=seed)
    rng = np.random.default_rng(seed)
    mask = (rng.random(p.n) < 0.5).astype(np.uint8)
    x = np.where(mask == 1, rng.standard_normal(p.n), 0.0)
    G, c = O.gram(p)
    y1 = O.dual_gram(G, c, mask, x)
    y2 = O.dual_eq5(p, mask, x)
    scale = np.abs(G).max() * np.abs(x).sum() + np.abs(c).max()
    assert np.abs(y1 - y2).max() <= 1e-13 * scale
    A = p.dense()
    Fm, Gm = mask == 1, mask == 0
    ref = A[:, Gm].T @ (A[:, Fm] @ x[Fm] - p.b)
    assert np.allclose(y1[Gm], ref, rtol=1e-12, atol=1e-12 * scale)


# ------------------------------------------------------------ clamp
@pytest.mark.parametrize("case", GOLD["zero_clamp"], ids=lambda c: c["cite"])
def test_clamp_golden(case):
    assert np.array_equal(O.clamp(case["v"], case["tol"]), np.array(case["out"], dtype=float))


# ---------------------------------------------------- exchange
@pytest.mark.parametrize("case", GOLD["exchange_infeasible"], ids=lambda c: c["cite"])
def test_exchange_golden(case):
    n = case["n"]
    mask = np.zeros(n, dtype=np.uint8)
    mask[case["F"]] = 1
    x, y = np.zeros(n), np.zeros(n)
    for k, v in case["x"].items():
        x[int(k)] = v
    for k, v in case["y"].items():
        y[int(k)] = v
    # "all" = branch 0 (k < N); "single" = p exhausted and no improvement
    N, p = (n + 1, 3) if case["rule"] == "all" else (0, 0)
    k, m2, N2, p2, br = O.exchange(mask, x, y, N, p)
    assert br == (0 if case["rule"] == "all" else 2)
    assert sorted(np.nonzero(m2)[0].tolist()) == case["F_out"]


def test_exchange_branches():
    n = 6
    mask = np.array([1, 1, 0, 0, 1, 0], dtype=np.uint8)
    x = np.array([-1.0, 2.0, 0.0, 0.0, -3.0, 0.0])
    y = np.array([0.0, 0.0, -1.0, 4.0, 0.0, -2.0])      # infeasible: 0, 2, 4, 5 -> k = 4
    # (i) k < N: reset p, flip all
    k, m2, N2, p2, br = O.exchange(mask, x, y, 5, 1)
    assert (k, br, N2, p2) == (4, 0, 4, 3)
    assert m2.tolist() == [0, 1, 1, 0, 0, 1]
    # (ii) k >= N, p > 0: p decrements, flip all, N unchanged
    k, m2, N2, p2, br = O.exchange(mask, x, y, 4, 2)
    assert (k, br, N2, p2) == (4, 1, 4, 1)
    assert m2.tolist() == [0, 1, 1, 0, 0, 1]
    # (iii) k >= N, p == 0: only the largest original index (5, in G) moves
    k, m2, N2, p2, br = O.exchange(mask, x, y, 3, 0)
    assert (k, br, N2, p2) == (4, 2, 3, 0)
    assert m2.tolist() == [1, 1, 0, 0, 1, 1]
    # largest infeasible index inside F
    y2 = y.copy()
    y2[5] = 1.0
    k, m2, _, _, br = O.exchange(mask, x, y2, 1, 0)
    assert (k, br) == (3, 2) and m2.tolist() == [1, 1, 0, 0, 0, 0]
    # feasible state: nothing changes
    k, m2, N2, p2, br = O.exchange(mask, np.abs(x), np.abs(y), 2, 1)
    assert (k, br, N2, p2) == (0, -1, 2, 1) and np.array_equal(m2, mask)
    # zero is feasible (strict negativity, reading c5)
    k, *_ = O.exchange(np.zeros(2, np.uint8), np.zeros(2), np.array([0.0, -0.0]), 3, 3)
    assert k == 0


# ------------------------------------------------------------- LSQR (a10)
@pytest.mark.parametrize("case", GOLD["lsqr"], ids=lambda c: c["cite"])
def test_lsqr_golden(case):
    p = _dense_problem(case["A"], case["b"])
    r = O.lsqr(p, itn_limit=50)
    assert np.allclose(r["x"], case["x"], atol=1e-13)
    if "rnorm" in case:
        assert abs(r["rnorm"] - case["rnorm"]) <= 1e-13


@pytest.mark.parametrize("seed", range(4))
def test_lsqr_matches_scipy_and_lstsq(seed):
    p = g.make_problem(dict(m=300, n=100, density=0.1), seed=seed)
    A = p.dense()
    r = O.lsqr(p)
    ref = np.linalg.lstsq(A, p.b, rcond=None)[0]
    assert np.abs(r["x"] - ref).max() / np.abs(ref).max() < 1e-10
    sp = scipy.sparse.linalg.lsqr(scipy.sparse.csr_matrix(A), p.b, atol=1e-15, btol=1e-15,
                                  conlim=1e8, iter_lim=400)
    assert np.abs(r["x"] - sp[0]).max() / np.abs(ref).max() < 1e-10
    h = r["rnorm_hist"]
    assert np.all(np.diff(h) <= 1e-12 * h[0])                       # S:236 monotone
    assert r["istop"] in (1, 2, 4, 5)
    # masked columns: LSQR on A_F equals lstsq(A_F)
    mask = (np.arange(p.n) % 3 != 0).astype(np.uint8)
    r2 = O.lsqr(p, mask=mask)
    ref2 = np.linalg.lstsq(A[:, mask == 1], p.b, rcond=None)[0]
    assert np.all(r2["x"][mask == 0] == 0)
    assert np.abs(r2["x"][mask == 1] - ref2).max() / np.abs(ref2).max() < 1e-10


def test_lsqr_adjoint_consistency():
    """<A v, u> == <v, A^T u> for the oracle's masked products (via dual_eq5)."""
    p = g.make_problem(dict(m=120, n=60, density=0.2), seed=2, raw=True)
    rng = np.random.default_rng(1)
    v = rng.standard_normal(p.n)
    u = rng.standard_normal(p.m)
    # dual_eq5 with mask=all ones in F gives nothing; use G-mask all zeros:
    # y = A^T (0 - b') with b' = -u  ->  A^T u
    q = g.Problem(p.m, p.n, p.rowptr, p.colind, p.vals, -u, p.x_gen, "raw", 0)
    Atu = O.dual_eq5(q, np.zeros(p.n, np.uint8), np.zeros(p.n))
    Av = p.dense() @ v
    assert abs(Av @ u - v @ Atu) <= 1e-13 * np.abs(p.vals).sum() * np.abs(v).max() * np.abs(u).max()
