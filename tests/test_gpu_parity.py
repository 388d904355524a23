"""GPU parity tests (-m gpu): the CUDA path, called through the C ABI, against
the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star): final free set F and pivot-iteration count
identical, x within relative inf-norm 1e-9 (FP64).  The Gram matrix and A^T b
are compared BITWISE (exact for the quantized inputs, and the kernel also
keeps the oracle's summation order).  Integer decisions (branch per
iteration, infeasible counts, |F|) are compared exactly via the trace.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

import nnls_gen as g  # noqa: E402
import oracle as O  # noqa: E402

TOL_X = 1e-9
HERE = os.path.dirname(os.path.abspath(__file__))
SINGLES = json.load(open(os.path.join(HERE, "golden", "single_exchange_seeds.json")))


@pytest.fixture(scope="module")
def P():
    import paper_cs_0408029_b200 as pkg
    assert pkg.device_info()["cc"] >= 100
    return pkg


def rel(a, b):
    d = np.abs(b).max() if np.size(b) else 0.0
    return np.abs(np.asarray(a) - np.asarray(b)).max() / (d if d > 0 else 1.0) if np.size(b) else 0.0


def run_gpu(P, prob, **kw):
    S = P.setup(prob, trace=1, **kw)
    x, info = S.solve()
    return dict(x=x, info=info, mask=S.free_set(), x_ne=S.x_ne(), trace=S.trace(), S=S)


def assert_parity(P, prob, check_trace=True, **kw):
    r = O.solve(prob, trace_cap=10 * prob.n + 2, **kw)
    gpu = run_gpu(P, prob, **kw)
    info = gpu["info"]
    assert info["status"] == r["status"], (info["status"], r["status"])
    assert np.array_equal(gpu["mask"], r["mask"]), "final free set differs"
    assert info["iterations"] == r["iterations"]
    assert info["single_exchanges"] == r["single_exchanges"]
    assert info["free_count"] == r["free_count"]
    if check_trace:
        tg, to = gpu["trace"], r["trace"]
        assert [(t["k"], t["branch"], t["f"]) for t in tg] == [(t["k"], t["branch"], t["f"]) for t in to]
    assert rel(gpu["x_ne"], r["x_ne"]) <= TOL_X
    assert rel(gpu["x"], r["x"]) <= TOL_X
    if r["status"] == 0:
        assert gpu["x"].min() >= 0.0
    if r["status"] == 0 and info["free_count"] > 0 and kw.get("lsqr_mode", 1) == 1:
        assert info["lsqr_iterations"] > 0
    return gpu, r


# ------------------------------------------------------------------- Gram
@pytest.mark.parametrize("cfg", [0, 1, 3, dict(m=333, n=129, density=0.07), dict(m=50, n=50, density=1.0)])
def test_gram_bitwise(P, cfg):
    prob = g.make_problem(cfg, seed=1)
    S = P.setup(prob)
    G, c = S.gram()
    Go, co = O.gram(prob)
    assert np.array_equal(G, Go) and np.array_equal(c, co)


def test_gram_bitwise_raw_inputs(P):
    """Unquantized values: the kernel keeps the oracle's term order and rounding."""
    prob = g.make_problem(dict(m=400, n=150, density=0.05), seed=2, raw=True)
    G, c = P.setup(prob).gram()
    Go, co = O.gram(prob)
    assert np.array_equal(G, Go) and np.array_equal(c, co)


@pytest.mark.parametrize("shape", [dict(m=400, n=150, density=0.05), dict(m=900, n=40, density=0.3),
                                   dict(m=2500, n=1100, density=0.02), dict(m=320, n=300, density=0.15), dict(m=320, n=300, density=0.25),
                                   dict(m=400, n=300, density=0.38), dict(m=5, n=5, density=1.0),
                                   dict(m=6000, n=100, density=0.3), dict(m=1100, n=90, density=0.5)])
def test_gram_claim_ordered_path_bitwise(P, shape, monkeypatch):
    """General (unquantized) values on the CTA-per-G-row kernel that applies
    each batch of rows by claims (equal j's in increasing row order): the
    oracle's bits (rows <= 128 entries in 2-4 per lane; columns longer
    than the 512-tuple stage -- the last two shapes: ~1800 and ~550 entries -- in segments).  The second
    shape packs ~270 entries into each of 40 columns, so most tuples of a batch
    collide and wait several passes; NNLS_CLAIM_MIN_N forces the path at small n."""
    monkeypatch.setenv("NNLS_CLAIM_MIN_N", "1")
    prob = g.make_problem(shape, seed=6, raw=True)
    G, c = P.setup(prob).gram()
    Go, co = O.gram(prob)
    assert np.array_equal(G, Go) and np.array_equal(c, co)
    monkeypatch.setenv("NNLS_CLAIM_MIN_N", "1000000")      # the warp-per-row kernel: same bits
    Gw, cw = P.setup(prob).gram()
    assert np.array_equal(Gw, Go) and np.array_equal(cw, co)


def test_gram_claim_ordered_row_shard_packed(P, monkeypatch):
    """The claim-ordered kernel over a row block, packed-triangle output (the
    row-shard partial): equal to the oracle's Gram of that block."""
    from paper_cs_0408029_b200.dist import gram_tensor, row_shards
    monkeypatch.setenv("NNLS_CLAIM_MIN_N", "1")
    prob = g.make_problem(dict(m=1200, n=260, density=0.04), seed=8, raw=True)
    (r0, r1) = row_shards(prob.m, 3)[1]
    S = P.ShardSolver(prob.m, prob.n, prob.rowptr, prob.colind, prob.vals, prob.b, r0, r1)
    buf = gram_tensor(S).cpu().numpy()
    lo, hi = prob.rowptr[r0], prob.rowptr[r1]
    blk = g.Problem(r1 - r0, prob.n, prob.rowptr[r0:r1 + 1] - lo, prob.colind[lo:hi], prob.vals[lo:hi],
                    prob.b[r0:r1], prob.x_gen, prob.kind, prob.seed)
    Gb, cb = O.gram(blk)
    n = prob.n
    assert np.array_equal(buf[:n * (n + 1) // 2], Gb[np.tril_indices(n)])
    assert np.array_equal(buf[n * (n + 1) // 2:], cb)


@pytest.mark.parametrize("cfg", [1, dict(m=3000, n=12, density=0.5)])
def test_gram_exact_and_ordered_paths_agree(P, cfg, monkeypatch):
    """Quantized inputs take the exact-arithmetic Gram (any summation order,
    integer accumulation) unless a column is too long for it (the second case:
    columns of ~1500 entries); NNLS_NO_EXACT_GRAM forces the row-ordered
    kernel.  Both must give the oracle's bits."""
    prob = g.make_problem(cfg, seed=4)
    Ge, ce = P.setup(prob).gram()
    monkeypatch.setenv("NNLS_NO_EXACT_GRAM", "1")
    Gs, cs = P.setup(prob).gram()
    Go, co = O.gram(prob)
    assert np.array_equal(Ge, Go) and np.array_equal(ce, co)
    assert np.array_equal(Gs, Go) and np.array_equal(cs, co)


def test_step_gram_device_buffers(P):
    prob = g.make_problem(dict(m=300, n=97, density=0.1), seed=3)
    dev = "cuda"
    rp = torch.tensor(prob.rowptr, device=dev)
    ci = torch.tensor(prob.colind, device=dev)
    v = torch.tensor(prob.vals, device=dev)
    b = torch.tensor(prob.b, device=dev)
    ldg = 100
    G = torch.full((prob.n, ldg), -7.0, dtype=torch.float64, device=dev)
    c = torch.empty(prob.n, dtype=torch.float64, device=dev)
    P.step_gram(prob.m, prob.n, rp, ci, v, b, G, c, ldg=ldg)
    Go, co = O.gram(prob)
    assert np.array_equal(G[:, :prob.n].cpu().numpy(), Go)
    assert np.array_equal(c.cpu().numpy(), co)


# --------------------------------------------------- normal solve (a5, a6)
@pytest.mark.parametrize("f", [1, 2, 63, 64, 65, 127, 128, 129, 191, 257])
def test_normal_solve_tile_edges(P, f):
    prob = g.make_problem(dict(m=900, n=300, density=0.06), seed=f)
    Go, co = O.gram(prob)
    rng = np.random.default_rng(f)
    F = np.sort(rng.choice(prob.n, f, replace=False)).astype(np.int32)
    L, rc = O.cholesky(O.gather(Go, F))
    assert rc == 0
    want = O.chol_solve(L, co[F])
    G = torch.tensor(Go, device="cuda")
    c = torch.tensor(co, device="cuda")
    xF = torch.empty(f, dtype=torch.float64, device="cuda")
    st, col = P.step_normal_solve(prob.n, G, c, torch.tensor(F, device="cuda"), xF)
    assert st == P.OK and col == -1
    assert rel(xF.cpu().numpy(), want) <= 1e-12


def test_normal_solve_not_pd(P):
    A = np.random.default_rng(0).standard_normal((40, 6))
    A[:, 4] = A[:, 1]
    prob = g.from_dense(np.round(A * 64) / 64, np.ones(40))
    Go, co = O.gram(prob)
    F = np.array([0, 1, 2, 4], dtype=np.int32)
    _, rc = O.cholesky(O.gather(Go, F))
    xF = torch.empty(4, dtype=torch.float64, device="cuda")
    st, col = P.step_normal_solve(6, torch.tensor(Go, device="cuda"), torch.tensor(co, device="cuda"),
                                  torch.tensor(F, device="cuda"), xF)
    assert st == P.ERR_NOT_PD and col == -rc - 1 == 3


# ---------------------------------------------------- exchange (a3, a4)
def _exchange_gpu(P, mask, x, y, N, p, p_max=3):
    m = torch.tensor(mask, dtype=torch.uint8, device="cuda")
    state = [N, p, 0, 0]
    k, br = P.step_exchange(len(mask), m, torch.tensor(x, device="cuda"), torch.tensor(y, device="cuda"),
                            state, p_max=p_max)
    return k, m.cpu().numpy(), state[0], state[1], br


def test_exchange_hand_states(P):
    mask = np.array([1, 1, 0, 0, 1, 0], dtype=np.uint8)
    x = np.array([-1.0, 2.0, 0.0, 0.0, -3.0, 0.0])
    y = np.array([0.0, 0.0, -1.0, 4.0, 0.0, -2.0])
    for N, p in [(5, 1), (4, 2), (3, 0), (1, 0), (4, 0)]:
        kg, mg, Ng, pg, bg = _exchange_gpu(P, mask, x, y, N, p)
        ko, mo, No, po, bo = O.exchange(mask, x, y, N, p)
        assert (kg, Ng, pg, bg) == (ko, No, po, bo) and np.array_equal(mg, mo)
    kg, mg, _, _, bg = _exchange_gpu(P, mask, np.abs(x), np.abs(y), 2, 1)
    assert kg == 0 and bg == -1 and np.array_equal(mg, mask)


@pytest.mark.parametrize("n", [1, 31, 32, 33, 1023, 1024, 1025, 5000])
def test_exchange_random_states(P, n):
    rng = np.random.default_rng(n)
    for trial in range(4):
        mask = (rng.random(n) < 0.5).astype(np.uint8)
        x = np.where(mask == 1, rng.standard_normal(n), 0.0)
        y = np.where(mask == 0, rng.standard_normal(n), 0.0)
        N = int(rng.integers(0, n + 2))
        p = int(rng.integers(0, 4))
        kg, mg, Ng, pg, bg = _exchange_gpu(P, mask, x, y, N, p)
        ko, mo, No, po, bo = O.exchange(mask, x, y, N, p)
        assert (kg, Ng, pg, bg) == (ko, No, po, bo) and np.array_equal(mg, mo)


# ------------------------------------------------------- dual (a7, a8)
@pytest.mark.parametrize("seed", range(3))
def test_dual_matches_oracle(P, seed):
    prob = g.make_problem(dict(m=500, n=200, density=0.05), seed=seed)
    Go, co = O.gram(prob)
    rng = np.random.default_rng(seed)
    mask = (rng.random(prob.n) < 0.5).astype(np.uint8)
    x = np.where(mask == 1, rng.standard_normal(prob.n), 0.0)
    x[np.nonzero(mask)[0][:3]] = [3e-13, -5e-13, 1e-12]          # zeroing boundary cases
    yo = O.dual_gram(Go, co, mask, x)
    xo = x.copy()
    for i in range(prob.n):
        if mask[i] and abs(xo[i]) < 1e-12:
            xo[i] = 0.0
        if not mask[i] and abs(yo[i]) < 1e-12:
            yo[i] = 0.0
    xd = torch.tensor(x, device="cuda")
    yd = torch.full((prob.n,), 9.0, dtype=torch.float64, device="cuda")
    P.step_dual(prob.n, torch.tensor(Go, device="cuda"), torch.tensor(co, device="cuda"),
                torch.tensor(mask, device="cuda"), xd, yd)
    assert np.array_equal(xd.cpu().numpy(), xo)
    yg = yd.cpu().numpy()
    assert np.all(yg[mask == 1] == 0)
    scale = np.abs(Go).max() * np.abs(x).sum() + np.abs(co).max()
    assert np.abs(yg - yo).max() <= 1e-14 * scale


# ----------------------------------------------------- whole solve parity
@pytest.mark.parametrize("cfg,seed", [(0, s) for s in range(5)] + [(1, s) for s in range(3)] +
                         [(3, s) for s in range(3)])
def test_solve_parity_configs(P, cfg, seed):
    gpu, r = assert_parity(P, g.make_problem(cfg, seed))
    i = gpu["info"]
    assert abs(i["objective"] - r["objective"]) <= 1e-9 * max(1.0, r["objective"])
    assert i["kkt_min_x"] >= 0.0


@pytest.mark.parametrize("n", [63, 64, 65, 127, 128, 129, 192])
def test_solve_all_free_tile_edges(P, n):
    """b = A x* with x* > 0: every column ends in F, so |F| = n hits each ragged tile edge."""
    prob = g.make_problem(dict(m=3 * n, n=n, density=0.08, rhs="degenerate"), seed=n)
    x = prob.x_gen.copy()
    x[x == 0] = 0.75                       # all strictly positive
    A = prob.dense()
    b = np.round(A @ x * (1 << 24)) / (1 << 24)
    q = g.from_dense(A, b)
    gpu, r = assert_parity(P, q)
    assert r["free_count"] == n


@pytest.mark.parametrize("seed", range(12))
def test_solve_parity_random_shapes(P, seed):
    rng = np.random.default_rng([seed, 9])
    n = int(rng.integers(2, 300))
    m = n + int(rng.integers(1, 3 * n))
    d = float(rng.choice([0.02, 0.1, 0.5]))
    assert_parity(P, g.make_problem(dict(m=m, n=n, density=max(d, 2.0 / n)), seed=seed))


@pytest.mark.parametrize("seed", range(8))
def test_solve_parity_reuse_shapes(P, seed):
    """|F| of a few hundred to ~700: later pivot iterations keep a factor
    prefix (factor reuse) -- restart row chains by half or whole tiles, the
    bordered row landing anywhere relative to the kept columns."""
    rng = np.random.default_rng([seed, 17])
    n = int(rng.integers(300, 1300))
    m = n + int(rng.integers(n // 2, 3 * n))
    d = float(rng.choice([0.03, 0.06, 0.12]))
    assert_parity(P, g.make_problem(dict(m=m, n=n, density=d), seed=100 + seed))


@pytest.mark.parametrize("case", SINGLES["cases"][:20], ids=lambda c: f"seed{c['seed']}")
def test_single_exchange_parity(P, case):
    gpu, r = assert_parity(P, g.make_correlated(case["seed"], 0.05), lsqr_mode=0)
    assert gpu["info"]["single_exchanges"] >= 1


@pytest.mark.parametrize("mode", [0, 2])
def test_lsqr_modes(P, mode):
    assert_parity(P, g.make_problem(0, 7), lsqr_mode=mode)


def test_edge_cases(P):
    # A^T b <= 0: zero iterations, x = 0
    A = np.array([[1.0, 2.0], [0.5, 1.0], [0.0, 3.0]])
    b = -A @ np.array([1.0, 0.5])
    gpu, r = assert_parity(P, g.from_dense(A, b))
    assert gpu["info"]["iterations"] == 0 and np.all(gpu["x"] == 0)
    # n = 1, m = 1
    assert_parity(P, g.from_dense(np.array([[2.0]]), np.array([3.0])))
    assert_parity(P, g.from_dense(np.array([[2.0], [1.0]]), np.array([-3.0, 1.0])))
    # identity: x = max(b, 0) exactly, one iteration
    bb = np.round(np.random.default_rng(1).standard_normal(70) * 64) / 64
    gpu, _ = assert_parity(P, g.from_dense(np.eye(70), bb), lsqr_mode=0)
    assert np.array_equal(gpu["x"], np.maximum(bb, 0)) and gpu["info"]["iterations"] == 1
    # iteration limit (reading c12)
    gpu, r = assert_parity(P, g.make_problem(0, 0), max_iter=1)
    assert gpu["info"]["status"] == 8


def test_not_pd_status(P):
    p = g.make_problem(0, 0)
    A = p.dense()
    A = np.concatenate([A, A[:, :1]], axis=1)
    q = g.from_dense(A, p.b)
    r = O.solve(q)
    gpu = run_gpu(P, q)
    assert gpu["info"]["status"] == r["status"]
    assert gpu["info"]["iterations"] == r["iterations"]
    if r["status"] == 7:
        assert gpu["info"]["not_pd_column"] >= 0


def test_invalid_inputs(P):
    p = g.make_problem(dict(m=20, n=10, density=0.3), seed=0)
    S = P.Solver()
    bad = p.colind.copy()
    bad[3] = 10
    with pytest.raises(P.NNLSError) as e:
        S.load(p.m, p.n, p.rowptr, bad, p.vals, p.b)
    assert e.value.status == P.ERR_INDEX
    rp = p.rowptr.copy()
    rp[-1] -= 1
    with pytest.raises(P.NNLSError) as e:
        S.load(p.m, p.n, rp, p.colind, p.vals, p.b)
    assert e.value.status == P.ERR_DIMENSION
    v = p.vals.copy()
    v[0] = np.nan
    with pytest.raises(P.NNLSError) as e:
        S.load(p.m, p.n, p.rowptr, p.colind, v, p.b)
    assert e.value.status == P.ERR_NONFINITE
    with pytest.raises(P.NNLSError) as e:
        S.solve()
    assert e.value.status == P.ERR_STATE
    # a valid load afterwards works on the same handle
    S.load_problem(p)
    x, info = S.solve()
    assert info["status"] == 0


def test_repeated_solves_and_reload(P):
    """Handles are reusable: reload different problems into one handle (buffer reuse)."""
    S = P.Solver(trace=1)
    for cfg, seed in [(0, 1), (dict(m=700, n=300, density=0.05), 2), (0, 3)]:
        prob = g.make_problem(cfg, seed)
        S.load_problem(prob)
        for _ in range(2):
            x, info = S.solve()
            r = O.solve(prob)
            assert np.array_equal(S.free_set(), r["mask"]) and info["iterations"] == r["iterations"]
            assert rel(x, r["x"]) <= TOL_X


def test_device_resident_inputs_and_outputs(P):
    prob = g.make_problem(1, 4)
    t = {k: torch.tensor(getattr(prob, k), device="cuda") for k in ("rowptr", "colind", "vals", "b")}
    S = P.Solver().load(prob.m, prob.n, t["rowptr"], t["colind"], t["vals"], t["b"])
    xd = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    S.solve(x_out=xd)
    r = O.solve(prob)
    assert rel(xd.cpu().numpy(), r["x"]) <= TOL_X


# ---------------------------------------------------------------- batched
def _batched_parity(P, B, **kw):
    out = P.BatchedSolver(**kw).load_batch(B).solve()
    ref = O.solve_batched(B, O.default_params(**kw), threads=0)
    x = out["x"].reshape(B.count, B.n)
    mask = out["mask"].reshape(B.count, B.n)
    info = out["info"]
    assert np.array_equal(info["status"], ref["status"])
    assert np.array_equal(mask, ref["mask"])
    assert np.array_equal(info["iterations"], ref["iterations"])
    assert np.array_equal(info["single_exchanges"], ref["single_exchanges"])
    scale = np.maximum(np.abs(ref["x"]).max(axis=1), 1e-300)
    err = np.abs(x - ref["x"]).max(axis=1) / np.where(np.abs(ref["x"]).max(axis=1) > 0, scale, 1.0)
    assert err.max() <= TOL_X
    return out, ref


def test_batched_invalid_inputs(P):
    """Batched validation: each corruption is reported with its own status,
    wherever in the batch it sits (first / middle / last problem, first /
    last row), and a clean batch after it loads on the same handle."""
    B = g.make_batch(seed=5, start=0, count=40)
    S = P.BatchedSolver()

    def expect(status, **over):
        kw = dict(nnz_off=B.nnz_off, rowptr=B.rowptr, colind=B.colind, vals=B.vals, b=B.b)
        kw.update(over)
        with pytest.raises(P.NNLSError) as e:
            S.load(B.count, B.m, B.n, kw["nnz_off"], kw["rowptr"], kw["colind"], kw["vals"], kw["b"])
        assert e.value.status == status

    def row_span(prob, r):
        base = int(B.nnz_off[prob])
        rp = B.rowptr[prob * (B.m + 1):(prob + 1) * (B.m + 1)]
        return base + int(rp[r]), base + int(rp[r + 1])

    for prob in (0, 17, B.count - 1):
        ci = B.colind.copy()
        ci[row_span(prob, B.m - 1)[1] - 1] = B.n  # out of range
        expect(P.ERR_INDEX, colind=ci)
        for r in (0, B.m // 2, B.m - 1):
            lo, hi = row_span(prob, r)
            if hi - lo < 2:
                continue
            ci = B.colind.copy()
            ci[lo], ci[lo + 1] = ci[lo + 1], ci[lo]  # out of order inside a row
            expect(P.ERR_INDEX, colind=ci)
            ci = B.colind.copy()
            ci[hi - 1] = ci[hi - 2]  # repeated column
            expect(P.ERR_INDEX, colind=ci)
        v = B.vals.copy()
        v[row_span(prob, 3)[0]] = np.inf
        expect(P.ERR_NONFINITE, vals=v)
        bb = B.b.copy()
        bb[prob * B.m + B.m - 1] = np.nan
        expect(P.ERR_NONFINITE, b=bb)
        rp = B.rowptr.copy()
        rp[prob * (B.m + 1) + B.m] -= 1  # last row end != nnz of the problem
        expect(P.ERR_DIMENSION, rowptr=rp)
    S.load_batch(B)
    out = S.solve()
    assert (out["info"]["status"] == 0).all()


@pytest.mark.parametrize("chunk", [1, 7, 100, 0])
def test_batched_pipelined_run_matches_load_solve(P, chunk):
    """nnls_run_batched (chunked copy/compute pipeline) gives the bits of
    load + solve, pinned or pageable host buffers alike."""
    B = g.make_batch(seed=6, start=0, count=300)
    ref = P.BatchedSolver().load_batch(B).solve()
    S = P.BatchedSolver()
    for pinned in (False, True):
        arrs = [B.nnz_off, B.rowptr, B.colind, B.vals, B.b]
        if pinned:
            arrs = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in arrs]
        x = torch.empty(B.count * B.n, dtype=torch.float64).pin_memory() if pinned else None
        out = S.run(B.count, B.m, B.n, *arrs, x_out=x, chunk=chunk)
        xo = out["x"].numpy() if pinned else out["x"]
        assert np.array_equal(xo, ref["x"])
        assert np.array_equal(out["mask"], ref["mask"])
        for k in ref["info"]:
            assert np.array_equal(out["info"][k], ref["info"][k], equal_nan=True), k
    # the handle is loaded afterwards: a plain solve repeats the result
    again = S.solve()
    assert np.array_equal(again["x"], ref["x"])


def test_batched_pipelined_run_invalid_chunk(P):
    """A corrupt problem in a middle chunk: the call reports it, the other
    chunks still run, and the handle works for the next batch."""
    B = g.make_batch(seed=7, start=0, count=64)
    S = P.BatchedSolver()
    ci = B.colind.copy()
    ci[int(B.nnz_off[40]) + 5] = -1
    with pytest.raises(P.NNLSError) as e:
        S.run(B.count, B.m, B.n, B.nnz_off, B.rowptr, ci, B.vals, B.b, chunk=16)
    assert e.value.status == P.ERR_INDEX
    v = B.vals.copy()
    v[int(B.nnz_off[63]) + 1] = np.nan
    with pytest.raises(P.NNLSError) as e:
        S.run(B.count, B.m, B.n, B.nnz_off, B.rowptr, B.colind, v, B.b, chunk=16)
    assert e.value.status == P.ERR_NONFINITE
    out = S.run_batch(B, chunk=16)
    ref = O.solve_batched(B, O.default_params(), threads=0)
    assert np.array_equal(out["mask"].reshape(B.count, B.n), ref["mask"])


@pytest.mark.parametrize("m,n,density,count", [(256, 64, 0.2, 64), (64, 64, 0.3, 64), (10, 1, 0.5, 33),
                                               (33, 17, 0.25, 100), (200, 40, 0.05, 50)])
def test_batched_shapes(P, m, n, density, count):
    """Batched limits and odd shapes (m = n, n = 1, m at its 256 cap, very
    sparse rows incl. empty ones): parity with the oracle, through both the
    load + solve path and the pipelined run."""
    B = g.make_batch(seed=8, start=0, count=count, m=m, n=n, density=density, total=count)
    out, ref = _batched_parity(P, B)
    run = P.BatchedSolver().run_batch(B, chunk=16)
    assert np.array_equal(run["x"], out["x"]) and np.array_equal(run["mask"], out["mask"])


def test_batched_config4_slice(P):
    B = g.make_batch(seed=0, start=0, count=2048)
    out, ref = _batched_parity(P, B)
    assert out["info"]["kkt_min_x"].min() >= 0


def test_batched_slices_independent_of_position(P):
    """A problem's result does not depend on its batch neighbours (sharding invariance)."""
    B = g.make_batch(seed=1, start=0, count=300)
    full = P.BatchedSolver().load_batch(B).solve()
    C = g.make_batch(seed=1, start=100, count=57)
    part = P.BatchedSolver().load_batch(C).solve()
    assert np.array_equal(full["x"].reshape(300, 64)[100:157], part["x"].reshape(57, 64))


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_batched_lsqr_modes(P, mode):
    _batched_parity(P, g.make_batch(seed=2, start=0, count=256), lsqr_mode=mode)


def test_batched_x_ne_matches_oracle(P):
    """NE path of the batched kernel (mode 0): Gram and factor keep the
    oracle's operation order (bit-identical), the back substitution is a
    column sweep (different summation order) -> F exact, x to 1e-12."""
    B = g.make_batch(seed=3, start=0, count=512)
    out = P.BatchedSolver(lsqr_mode=0).load_batch(B).solve()
    ref = O.solve_batched(B, O.default_params(lsqr_mode=0), threads=0)
    assert np.array_equal(out["mask"].reshape(512, 64), ref["mask"])
    x = out["x"].reshape(512, 64)
    scale = np.maximum(np.abs(ref["x"]).max(axis=1, keepdims=True), 1e-300)
    assert (np.abs(x - ref["x"]) / scale).max() <= 1e-12


def test_batched_single_exchange_cases(P):
    for case in SINGLES["cases"][:10]:
        p = g.make_correlated(case["seed"], 0.05)
        B = g.Batch(p.m, p.n, 1, np.array([0, p.nnz], dtype=np.int64), p.rowptr, p.colind, p.vals, p.b,
                    np.zeros(p.n), 0, 0)
        _batched_parity(P, B, lsqr_mode=0)


@pytest.mark.parametrize("cfg,seed", [(0, 3), (1, 1), (3, 1)])
def test_lsqr_full_grid_path(P, cfg, seed, monkeypatch):
    """The cluster-resident LSQR is used when A fits in one cluster's shared
    memory; force the full-grid cooperative kernel and check it too."""
    monkeypatch.setenv("NNLS_NO_CLUSTER", "1")
    assert_parity(P, g.make_problem(cfg, seed))


@pytest.mark.parametrize("cfg,seed", [(0, 4), (1, 2), (3, 2)])
def test_host_driven_loop_path(P, cfg, seed, monkeypatch):
    """The pivot loop normally runs device-resident (CUDA-graph WHILE node);
    the host-driven loop (used for per-phase timing) must agree."""
    monkeypatch.setenv("NNLS_NO_GRAPH", "1")
    assert_parity(P, g.make_problem(cfg, seed))


@pytest.mark.parametrize("cfg,seed", [(0, 5), (1, 0), (3, 0)])
def test_index_order_path(P, cfg, seed, monkeypatch):
    """By default the factorization order keeps the previous iteration's
    surviving prefix and reuses its factor tiles;
    the plain index-order factorization (NNLS_NO_REUSE) must agree too."""
    monkeypatch.setenv("NNLS_NO_REUSE", "1")
    assert_parity(P, g.make_problem(cfg, seed))


@pytest.mark.parametrize("cfg,seed", [(0, 6), (1, 3), (3, 3)])
@pytest.mark.parametrize("graph", [True, False])
def test_unfused_decide_path(P, cfg, seed, graph, monkeypatch):
    """By default the dual kernel also counts the infeasibles and its last CTA
    takes the branch and applies the exchange (north_star step 4); the
    separate count + exchange pass of the decide kernel (NNLS_NO_FUSED_DUAL)
    must agree, in the graph loop and the host-driven loop."""
    monkeypatch.setenv("NNLS_NO_FUSED_DUAL", "1")
    if not graph:
        monkeypatch.setenv("NNLS_NO_GRAPH", "1")
    assert_parity(P, g.make_problem(cfg, seed))


def test_graph_replay_across_loads(P):
    """One handle, the captured solve graph is reused / rebuilt across loads."""
    S = P.Solver(trace=1)
    for cfg, seed in [(1, 0), (1, 0), (0, 2), (1, 1), (3, 0)]:
        prob = g.make_problem(cfg, seed)
        S.load_problem(prob)
        x, info = S.solve()
        r = O.solve(prob, trace_cap=10 * prob.n + 2)
        assert np.array_equal(S.free_set(), r["mask"]) and info["iterations"] == r["iterations"]
        assert [t["branch"] for t in S.trace()] == [t["branch"] for t in r["trace"]]
        assert rel(x, r["x"]) <= TOL_X


@pytest.mark.parametrize("world", [2, 3])
def test_row_sharded_gram_path(P, world):
    """Root ShardSolver (full A, its own rows) + BlockSolver ranks (ONLY their
    row block uploaded) -> packed partial [G | c] buffers, summed here by torch
    on one GPU (what dist.reduce_gram does across GPUs) -> nnls_gram_finalize:
    the packed partials equal the oracle's row-block Grams, the finalized Gram
    is bitwise the full one and the solve matches the oracle."""
    from paper_cs_0408029_b200.dist import gram_tensor, packed_count, row_block, row_shards
    prob = g.make_problem(1, 5)
    sh = row_shards(prob.m, world)
    root = P.ShardSolver(prob.m, prob.n, prob.rowptr, prob.colind, prob.vals, prob.b, *sh[0])
    blocks = []
    for r0, r1 in sh[1:]:
        rp, ci, v, b = row_block(prob.rowptr, prob.colind, prob.vals, prob.b, r0, r1)
        blocks.append((P.BlockSolver().load_block(r1 - r0, prob.n, rp, ci, v, b), (rp, ci, v, b, r1 - r0)))
    torch.cuda.synchronize()
    with pytest.raises(P.NNLSError):
        root.solve()                                       # not finalized yet
    with pytest.raises(P.NNLSError):
        blocks[0][0].solve()                               # a block-only handle never solves
    n = prob.n
    tril = np.tril_indices(n)
    for S, (rp, ci, v, b, mb) in blocks:                   # packed layout: row i = G[i, :i+1]
        buf = gram_tensor(S).cpu().numpy()
        assert buf.size == packed_count(n)
        Gb, cb = O.gram(g.Problem(mb, n, rp, ci, v, b, prob.x_gen, prob.kind, prob.seed))
        assert np.array_equal(buf[:n * (n + 1) // 2], Gb[tril]) and np.array_equal(buf[n * (n + 1) // 2:], cb)
    acc = gram_tensor(root)
    for S, _ in blocks:
        acc += gram_tensor(S)
    torch.cuda.synchronize()
    root.finalize()
    G, c = root.gram()
    Go, co = O.gram(prob)
    assert np.array_equal(G, Go) and np.array_equal(c, co)
    x, info = root.solve()
    r = O.solve(prob)
    assert np.array_equal(root.free_set(), r["mask"]) and info["iterations"] == r["iterations"]
    assert rel(x, r["x"]) <= TOL_X


# ------------------------------------------------------------------ NEXT-2
# lsqr_mode 3 (adaptive final step) and the NOT_PD LSQR fallback
# against the oracle extension (oracle/nnls_oracle.c or_condest).
# kappa: the forward solve is bit-identical to the oracle's, the backward
# sweep sums in another order -> relative 1e-6 (decisions are far from it).
@pytest.mark.parametrize("cfg,seed", [(0, 0), (1, 0), (3, 1), ("ill", 5)])
@pytest.mark.parametrize("thr", [1e-8, 1e-14])
def test_adaptive_mode_single(P, cfg, seed, thr):
    if cfg == "ill":
        rng = np.random.default_rng(seed)
        A = np.round(rng.standard_normal((200, 60)) * 64) / 64
        A[:, 0] *= 1e-5
        b = A @ (1.0 + np.abs(rng.standard_normal(60))) + 1e-9 * rng.standard_normal(200)
        prob = g.from_dense(A, b)
    else:
        prob = g.make_problem(cfg, seed)
    r = O.solve(prob, lsqr_mode=3, adaptive_threshold=thr, trace_cap=10 * prob.n + 2)
    S = P.setup(prob, lsqr_mode=3, adaptive_threshold=thr)
    x, info = S.solve()
    assert info["status"] == r["status"] == 0
    assert np.array_equal(S.free_set(), r["mask"]) and info["iterations"] == r["iterations"]
    assert info["refined"] == r["refined"]
    assert abs(info["kappa"] - r["kappa"]) <= 1e-6 * r["kappa"]
    assert rel(x, r["x"]) <= TOL_X
    if not r["refined"]:
        assert info["lsqr_iterations"] == 0 and rel(x, S.x_ne()) == 0.0


def test_adaptive_mode_batched(P):
    B = g.make_batch(seed=2, start=0, count=512)
    thr = 1e-14                              # kappa ~ 10-100 at config 4: some refine, some not
    out = P.BatchedSolver(lsqr_mode=3, adaptive_threshold=thr).load_batch(B).solve()
    info = out["info"]
    xs = out["x"].reshape(B.count, B.n)
    nref = 0
    for q in range(B.count):
        r = O.solve(B.problem(q), lsqr_mode=3, adaptive_threshold=thr)
        assert info["refined"][q] == r["refined"], q
        assert abs(info["kappa"][q] - r["kappa"]) <= 1e-6 * r["kappa"], q
        assert rel(xs[q], r["x"]) <= TOL_X, q
        nref += r["refined"]
    assert 0 < nref < B.count


def test_notpd_fallback_single(P):
    """Duplicate column: the default stops at NOT_PD (as the oracle); with
    notpd_fallback the LSQR solve replaces the failed factorization and the
    solve reaches the oracle's F, iteration count and optimal objective."""
    base = g.make_problem(0, 0)
    A = base.dense()
    A = np.concatenate([A, A[:, :1]], axis=1)
    prob = g.from_dense(A, base.b)
    S = P.setup(prob)
    _, info = S.solve()
    assert info["status"] == P.ERR_NOT_PD
    r = O.solve(prob, notpd_fallback=1)
    S2 = P.setup(prob, notpd_fallback=1)
    x, info2 = S2.solve()
    assert info2["status"] == r["status"] == 0
    assert info2["lsqr_fallbacks"] == r["lsqr_fallbacks"] >= 1
    assert info2["iterations"] == r["iterations"]
    assert np.array_equal(S2.free_set(), r["mask"])
    assert abs(info2["objective"] - r["objective"]) <= 1e-9 * r["objective"]
    assert x.min() >= 0.0


# ------------------------------------------------------------------ NEXT-1
# The Fig. 2 workloads (n x (n-10), density 1 and 0.01).  Density 1
# takes the dense DMMA SYRK Gram (gram_dense.cu): with exact inputs its sums
# are bitwise the oracle's, for the full Gram and for a row shard's packed one.
@pytest.mark.parametrize("n,d", [(100, 1.0), (300, 1.0), (700, 1.0), (1000, 1.0), (800, 0.01), (1420, 0.01)])
def test_fig2_workloads(P, n, d):
    prob = g.make_fig2(n, d, seed=1)
    S = P.Solver(trace=1)
    P.timing_enable(S.h, True)
    S.load_problem(prob)
    gram_launches = P.timing_read(S.h)["gram"][1]
    P.timing_enable(S.h, False)
    assert gram_launches == (4 if d == 1.0 else 1)      # density 1: the dense DMMA SYRK path
    G, c = S.gram()
    Go, co = O.gram(prob)
    assert np.array_equal(G, Go) and np.array_equal(c, co)
    x, info = S.solve()
    r = O.solve(prob, trace_cap=10 * prob.n + 2)
    assert info["status"] == r["status"] == 0
    assert np.array_equal(S.free_set(), r["mask"]) and info["iterations"] == r["iterations"]
    assert rel(x, r["x"]) <= TOL_X


def test_dense_gram_row_shard_packed(P):
    from paper_cs_0408029_b200.dist import gram_tensor, row_block, row_shards
    prob = g.make_fig2(400, 1.0, seed=2)
    n = prob.n
    tril = np.tril_indices(n)
    for r0, r1 in row_shards(prob.m, 3)[1:]:
        rp, ci, v, b = row_block(prob.rowptr, prob.colind, prob.vals, prob.b, r0, r1)
        S = P.BlockSolver()
        P.timing_enable(S.h, True)
        S.load_block(r1 - r0, n, rp, ci, v, b)
        assert P.timing_read(S.h)["gram"][1] == 4            # the dense path, packed output
        buf = gram_tensor(S).cpu().numpy()
        Gb, cb = O.gram(g.Problem(r1 - r0, n, rp, ci, v, b, prob.x_gen, prob.kind, prob.seed))
        assert np.array_equal(buf[:n * (n + 1) // 2], Gb[tril]) and np.array_equal(buf[n * (n + 1) // 2:], cb)


@pytest.mark.parametrize("lsqr_mode", [1, 2, 0])
def test_large_shape_lsqr_modes(P, lsqr_mode):
    """The grid-resident LSQR's warm start (mode 2: the correction from the NE
    x, U = b - A_F x_NE from the row slices) and mode 0 (the NE x, no LSQR:
    the global report path) at a shape beyond one cluster."""
    assert_parity(P, g.make_problem(dict(m=30000, n=3001, density=0.003), seed=8), lsqr_mode=lsqr_mode)


@pytest.mark.parametrize("shape", [dict(m=30000, n=3001, density=0.003), dict(m=12000, n=2049, density=0.01)])
def test_large_odd_shapes(P, shape):
    """Shapes beyond one cluster's shared memory with an odd n >= 2048: the
    grid-resident LSQR (row slices of A_F in every SM), the dual streaming
    whole G rows (16-byte loads plus the odd last column), ragged Cholesky
    tiles and factor reuse -- F, the iteration count and the trace identical
    to the oracle, x within the north_star bar."""
    assert_parity(P, g.make_problem(shape, seed=7))


def test_invalid_inputs_large(P):
    """From 1M entries the CSR is validated by the flat two-count kernel: an
    out-of-range, a repeated and an out-of-order column inside a row, a
    descending pair across a row boundary (valid), a non-finite value or b,
    and a bad rowptr must give the same status codes as the small-input path."""
    p = g.make_problem(dict(m=40000, n=8000, density=0.004), seed=3)
    assert p.nnz >= (1 << 20)
    S = P.Solver()
    r = int(p.rowptr[20000])  # a row in the middle
    lo, hi = int(p.rowptr[20000]), int(p.rowptr[20001])
    assert hi - lo >= 3
    cases = []
    bad = p.colind.copy(); bad[lo + 1] = p.n; cases.append((p.rowptr, bad, p.vals, p.b, P.ERR_INDEX))
    bad = p.colind.copy(); bad[lo + 1] = bad[lo]; cases.append((p.rowptr, bad, p.vals, p.b, P.ERR_INDEX))
    bad = p.colind.copy(); bad[lo], bad[lo + 1] = bad[lo + 1], bad[lo]; cases.append((p.rowptr, bad, p.vals, p.b, P.ERR_INDEX))
    v = p.vals.copy(); v[r + 2] = np.inf; cases.append((p.rowptr, p.colind, v, p.b, P.ERR_NONFINITE))
    bb = p.b.copy(); bb[7] = np.nan; cases.append((p.rowptr, p.colind, p.vals, bb, P.ERR_NONFINITE))
    rp = p.rowptr.copy(); rp[-1] -= 1; cases.append((rp, p.colind, p.vals, p.b, P.ERR_DIMENSION))
    for rowptr, colind, vals, b, code in cases:
        with pytest.raises(P.NNLSError) as e:
            S.load(p.m, p.n, rowptr, colind, vals, b)
        assert e.value.status == code
    S.load_problem(p)  # valid afterwards (descents at row starts are allowed)
    x, info = S.solve()
    assert info["status"] == 0 and info["kkt_min_x"] >= 0.0


@pytest.mark.parametrize("cfg", [1, 3])
def test_bitwise_repeatable(P, cfg):
    """Configs 1 and 3 (cluster LSQR, restart chains by half tiles and whole
    tiles): repeated solves bitwise identical (fixed-order reductions)."""
    prob = g.make_problem(cfg, 2)
    x0, i0 = P.setup(prob).solve()
    x0 = np.array(x0)
    for _ in range(4):
        x, info = P.setup(prob).solve()
        assert np.array_equal(np.array(x), x0)
        assert info["iterations"] == i0["iterations"] and info["lsqr_iterations"] == i0["lsqr_iterations"]


def test_batched_bitwise_repeatable(P):
    """The batched kernels (per-CTA problems, fixed-order sums): two solves of
    the same 2048-problem slice, and the pipelined run, bitwise identical."""
    B = g.make_batch(seed=5, start=0, count=2048)
    o1 = P.BatchedSolver().load_batch(B).solve()
    o2 = P.BatchedSolver().load_batch(B).solve()
    o3 = P.BatchedSolver().run_batch(B)
    for o in (o2, o3):
        assert np.array_equal(np.asarray(o["x"]), np.asarray(o1["x"]))
        assert np.array_equal(np.asarray(o["mask"]), np.asarray(o1["mask"]))
        assert np.array_equal(o["info"]["iterations"], o1["info"]["iterations"])
