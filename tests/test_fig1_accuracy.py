"""NEXT-3: the accuracy experiment of PAPER.md Section 4 / Fig. 1.

-m "not gpu": the P(m,n,d,x) generator (nnls_gen.make_p_problem, SPEC gen_p
substitute) is pinned by its definition -- singular values from a dense SVD,
r orthogonal to range(A), x_true the NNLS solution (scipy) -- and the oracle
reproduces the paper's error model: the normal equations' relative error
~ 0.1 kappa^2 eps (accepted within [1e-3, 10] kappa^2 eps, SPEC
acceptance 1), LSQR recompute at least one order better on small-residual
problems ("2 or 3 orders"; SPEC acceptance 2), and kappa = 1e8 (kappa^2
eps >= 1) completing without a crash (SPEC acceptance 3).
-m gpu: the same error model on the B200 path (modes 0 and 1).
"""
import numpy as np
import pytest
from scipy.optimize import nnls as scipy_nnls

import nnls_gen as g
import oracle as O

EPS = 2.0 ** -52


def rel(x, xt):
    return np.abs(np.asarray(x) - xt).max() / np.abs(xt).max()


@pytest.mark.parametrize("m,n,d,cond", [(4, 2, 1, 1.0), (6, 3, 1, 100.0), (80, 70, 4, 1e4), (40, 30, 3, 1e6)])
def test_p_generator_definition(m, n, d, cond):
    p = g.make_p_problem(m, n, d, cond, seed=3)
    A = p.dense()
    s = np.linalg.svd(A, compute_uv=False)
    k = (n + d - 1) // d
    want = np.repeat(cond ** (-np.arange(k) / max(k - 1, 1)) if k > 1 else np.ones(1), d)[:n]
    assert np.allclose(np.sort(s)[::-1], np.sort(want)[::-1], rtol=1e-10, atol=0)
    assert abs(s[0] / s[-1] - cond) <= 0.01 * cond
    r = p.b - A @ p.x_gen
    assert np.abs(A.T @ r).max() <= 1e-12 * np.abs(A).sum(0).max() * np.abs(r).max()
    assert abs(np.linalg.norm(r) - 0.25 * np.linalg.norm(A @ p.x_gen)) <= 1e-12 * np.linalg.norm(r)
    assert p.x_gen.min() > 0


def test_p_generator_solution_is_x_true():
    p = g.make_p_problem(80, 70, 4, 100.0, seed=1)
    xs, _ = scipy_nnls(p.dense(), p.b, maxiter=5000)
    assert rel(xs, p.x_gen) < 1e-12


@pytest.mark.parametrize("resid", [0.25, 1e-4])
def test_oracle_reproduces_error_model(resid):
    for kap in (1e2, 1e4, 1e6):
        ne, ls = [], []
        for seed in range(3):
            p = g.make_p_problem(80, 70, 4, kap, seed, resid=resid)
            ne.append(rel(O.solve(p, lsqr_mode=0)["x"], p.x_gen))
            ls.append(rel(O.solve(p, lsqr_mode=1)["x"], p.x_gen))
        m_ne, m_ls = np.median(ne), np.median(ls)
        assert 1e-3 * kap * kap * EPS <= m_ne <= 10 * kap * kap * EPS, (kap, m_ne)
        if resid < 1e-2 and kap >= 1e3:
            assert m_ls <= m_ne / 10, (kap, m_ne, m_ls)       # SPEC acceptance 2 (2-3 orders)
        assert m_ls <= 2 * m_ne


def test_oracle_extreme_conditioning_completes():
    p = g.make_p_problem(80, 70, 4, 1e8, 0)
    for mode in (0, 1):
        r = O.solve(p, lsqr_mode=mode)
        assert r["status"] in (0, 7, 8)


@pytest.mark.gpu
@pytest.mark.parametrize("resid", [0.25, 1e-4])
def test_gpu_reproduces_error_model(resid):
    pytest.importorskip("torch")
    import paper_cs_0408029_b200 as P
    for kap in (1e2, 1e4, 1e6):
        ne, ls = [], []
        for seed in range(3):
            p = g.make_p_problem(80, 70, 4, kap, seed, resid=resid)
            r = O.solve(p, lsqr_mode=0)
            S = P.setup(p, lsqr_mode=0)
            x0, info = S.solve()
            assert np.array_equal(S.free_set(), r["mask"]) and info["iterations"] == r["iterations"]
            ne.append(rel(x0, p.x_gen))
            x1, _ = P.setup(p, lsqr_mode=1).solve()
            ls.append(rel(x1, p.x_gen))
        m_ne, m_ls = np.median(ne), np.median(ls)
        assert 1e-3 * kap * kap * EPS <= m_ne <= 10 * kap * kap * EPS, (kap, m_ne)
        if resid < 1e-2 and kap >= 1e3:
            assert m_ls <= m_ne / 10, (kap, m_ne, m_ls)
    p = g.make_p_problem(80, 70, 4, 1e8, 0)
    _, info = P.setup(p).solve(check=False)
    assert info["status"] in (0, P.ERR_NOT_PD, P.ITERATION_LIMIT)
