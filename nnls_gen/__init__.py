"""Seeded synthetic NNLS inputs shared by the CPU oracle and the CUDA path.

This module holds NO arithmetic of the method (no Gram, no factorization, no
pivoting, no LSQR).  It only draws random problems shaped like BASELINE.json's
configs and packs them as CSR arrays + b.  Both sides of every parity test (and
bench.py) receive the same arrays from here.

Recipe (DESIGN.md §"Input recipe"):
  * sparsity: exactly round(d*m*n) distinct positions, uniform without
    replacement, rows sorted, columns sorted within a row (CSR);
  * values: N(0,1) quantized to the 2^-12 grid (redraw exact zeros, clip to
    [-8, 8]) -- quantization makes A^T A and A^T b exact in FP64 in any
    summation order, so the Gram is bitwise comparable across implementations;
  * x0 (configs 0,1,2,4): floor(n/2) entries U(0,1), the rest U(-1,0), random
    permutation, quantized to 2^-12 ("roughly half the variables end
    constrained", BASELINE.json configs[0]);
  * noise: 0.01*N(0,1) quantized to 2^-24; b = A x0 + noise computed exactly in
    integer units of 2^-24;
  * config 3 (degenerate): x* has exactly 40% zeros, the rest U(0.5,1) quantized
    to 2^-12; b = A x* exactly (no noise);
  * raw=True skips every quantization (robustness variant).

The paper's own timing inputs were MATLAB `sprandn` matrices;
these seeded matrices stand in for them.
"""
from __future__ import annotations

import dataclasses
import numpy as np

Q_A = 4096.0            # 2^12: grid of A entries and x0
Q_B = float(1 << 24)    # 2^24: grid of b (a*x products) and noise
A_CLIP = 8.0

# BASELINE.json "configs" (index -> shape, density, rhs kind, batch)
CONFIGS = {
    0: dict(m=200, n=100, density=0.10, rhs="noisy", batch=1),
    1: dict(m=2000, n=1000, density=0.05, rhs="noisy", batch=1),
    2: dict(m=40000, n=8000, density=0.005, rhs="noisy", batch=1),
    3: dict(m=3000, n=1500, density=0.02, rhs="degenerate", batch=1),
    4: dict(m=128, n=64, density=0.20, rhs="noisy", batch=65536),
}


@dataclasses.dataclass
class Problem:
    m: int
    n: int
    rowptr: np.ndarray   # int32[m+1]
    colind: np.ndarray   # int32[nnz]
    vals: np.ndarray     # float64[nnz]
    b: np.ndarray        # float64[m]
    x_gen: np.ndarray    # float64[n]: x0 (noisy) or x* (degenerate) used to build b
    kind: str
    seed: int

    @property
    def nnz(self) -> int:
        return int(self.colind.shape[0])

    def dense(self) -> np.ndarray:
        A = np.zeros((self.m, self.n))
        rows = np.repeat(np.arange(self.m), np.diff(self.rowptr))
        A[rows, self.colind] = self.vals
        return A


@dataclasses.dataclass
class Batch:
    """`count` independent problems of identical shape m x n (config 4)."""
    m: int
    n: int
    count: int
    nnz_off: np.ndarray  # int64[count+1]
    rowptr: np.ndarray   # int32[count*(m+1)], local to each problem
    colind: np.ndarray   # int32[total nnz]
    vals: np.ndarray     # float64[total nnz]
    b: np.ndarray        # float64[count*m]
    x_gen: np.ndarray    # float64[count*n]
    seed: int
    start: int

    def problem(self, p: int) -> Problem:
        lo, hi = int(self.nnz_off[p]), int(self.nnz_off[p + 1])
        return Problem(self.m, self.n,
                       self.rowptr[p * (self.m + 1):(p + 1) * (self.m + 1)].copy(),
                       self.colind[lo:hi].copy(), self.vals[lo:hi].copy(),
                       self.b[p * self.m:(p + 1) * self.m].copy(),
                       self.x_gen[p * self.n:(p + 1) * self.n].copy(),
                       "noisy", self.seed)


def _quantized_normal(rng, size, raw):
    z = rng.standard_normal(size)
    if raw:
        z[z == 0.0] = 1.0 / Q_A
        return z
    q = np.clip(np.round(z * Q_A), -A_CLIP * Q_A, A_CLIP * Q_A)
    bad = q == 0
    while bad.any():                      # "redraw if 0"
        q[bad] = np.clip(np.round(rng.standard_normal(int(bad.sum())) * Q_A),
                         -A_CLIP * Q_A, A_CLIP * Q_A)
        bad = q == 0
    return q / Q_A


def _x_noisy(rng, n, raw):
    half = n // 2
    x = np.concatenate([rng.uniform(0.0, 1.0, half), rng.uniform(-1.0, 0.0, n - half)])
    x = x[rng.permutation(n)]
    return x if raw else np.round(x * Q_A) / Q_A


def _x_degenerate(rng, n, raw, zero_frac=0.4):
    nz = int(round(zero_frac * n))
    x = rng.uniform(0.5, 1.0, n)
    if not raw:
        x = np.round(x * Q_A) / Q_A
    x[rng.permutation(n)[:nz]] = 0.0
    return x


def _rhs(rowptr, colind, vals, x, noise, raw):
    """b = A x + noise, computed exactly (integer units of 2^-24) unless raw."""
    m = rowptr.shape[0] - 1
    if raw:
        prod = vals * x[colind]
        b = np.zeros(m)
        nz = np.diff(rowptr) > 0
        b[nz] = np.add.reduceat(prod, rowptr[:-1][nz]) if prod.size else 0.0
        return b + noise
    ai = np.round(vals * Q_A).astype(np.int64)
    xi = np.round(x * Q_A).astype(np.int64)
    prod = ai * xi[colind]                      # units 2^-24, |.| <= 2^27
    bi = np.zeros(m, dtype=np.int64)
    nz = np.diff(rowptr) > 0
    if prod.size:
        bi[nz] = np.add.reduceat(prod, rowptr[:-1][nz])
    bi += np.round(noise * Q_B).astype(np.int64)
    assert np.abs(bi).max(initial=0) < (1 << 52)
    return bi.astype(np.float64) / Q_B


def _check_exact_budget(rowptr, colind, vals, b, n):
    """Quantized inputs only: sum_r |a_ri*b_r| < 2^53 units of 2^-36 per column,
    so A^T b is exact in FP64 in any order (likewise A^T A, bounded below)."""
    rows = np.repeat(np.arange(rowptr.shape[0] - 1), np.diff(rowptr))
    mag = np.abs(vals) * np.abs(b[rows]) * (Q_A * Q_B)
    col_budget = np.bincount(colind, weights=mag, minlength=n)
    assert col_budget.max(initial=0) < 2.0 ** 52, "A^T b not exactly representable"
    g_budget = np.bincount(colind, weights=vals * vals * Q_A * Q_A, minlength=n)
    assert g_budget.max(initial=0) < 2.0 ** 52


def make_problem(cfg: int | dict, seed: int = 0, raw: bool = False) -> Problem:
    """One seeded problem of BASELINE.json config `cfg` (0..3) or a dict
    {m, n, density, rhs} for test sizes."""
    spec = CONFIGS[cfg] if isinstance(cfg, int) else dict(cfg)
    m, n, d = int(spec["m"]), int(spec["n"]), float(spec["density"])
    kind = spec.get("rhs", "noisy")
    cfg_id = cfg if isinstance(cfg, int) else 100 + (m * 7919 + n) % 100000
    for attempt in range(100):
        rng = np.random.default_rng([int(seed), int(cfg_id), attempt])
        nnz = int(round(d * m * n))
        pos = np.sort(rng.choice(m * n, size=nnz, replace=False))
        rows, cols = pos // n, pos % n
        if np.bincount(cols, minlength=n).min(initial=1) == 0 and n > 0:
            continue                                   # every column non-empty
        vals = _quantized_normal(rng, nnz, raw)
        rowptr = np.zeros(m + 1, dtype=np.int32)
        np.cumsum(np.bincount(rows, minlength=m), out=rowptr[1:])
        colind = cols.astype(np.int32)
        if kind == "degenerate":
            x = _x_degenerate(rng, n, raw)
            noise = np.zeros(m)
        else:
            x = _x_noisy(rng, n, raw)
            noise = 0.01 * rng.standard_normal(m)
            if not raw:
                noise = np.round(noise * Q_B) / Q_B
        b = _rhs(rowptr, colind, vals, x, noise, raw)
        if not raw:
            _check_exact_budget(rowptr, colind, vals, b, n)
        return Problem(m, n, rowptr, colind, vals.astype(np.float64), b, x, kind, int(seed))
    raise RuntimeError("could not draw a problem with non-empty columns")


def from_dense(A: np.ndarray, b: np.ndarray) -> Problem:
    """Pack a small dense (hand-built) test matrix as CSR."""
    A = np.asarray(A, dtype=np.float64)
    m, n = A.shape
    rows, cols = np.nonzero(A)
    rowptr = np.zeros(m + 1, dtype=np.int32)
    np.cumsum(np.bincount(rows, minlength=m), out=rowptr[1:])
    return Problem(m, n, rowptr, cols.astype(np.int32), A[rows, cols].astype(np.float64),
                   np.asarray(b, dtype=np.float64).copy(), np.zeros(n), "hand", -1)


_CHUNK = 1024


def _batch_chunk(seed, m, n, d, chunk_id, count, raw):
    rng = np.random.default_rng([int(seed), 4, int(chunk_id)])
    nnz = int(round(d * m * n))
    keys = rng.random((count, m * n))
    pos = np.sort(np.argpartition(keys, nnz - 1, axis=1)[:, :nnz], axis=1)
    cols = pos % n
    # redraw (deterministically) any problem with an empty column
    for p in range(count):
        attempt = 0
        while np.bincount(cols[p], minlength=n).min() == 0:
            r2 = np.random.default_rng([int(seed), 4, int(chunk_id), p, attempt])
            pos[p] = np.sort(r2.choice(m * n, size=nnz, replace=False))
            cols[p] = pos[p] % n
            attempt += 1
    rows = pos // n
    vals = _quantized_normal(rng, (count, nnz), raw)
    xs = np.stack([_x_noisy(rng, n, raw) for _ in range(count)]) if count else np.zeros((0, n))
    noise = 0.01 * rng.standard_normal((count, m))
    if not raw:
        noise = np.round(noise * Q_B) / Q_B
    return rows, cols, vals, xs, noise


def make_batch(seed: int = 0, start: int = 0, count: int | None = None, raw: bool = False,
               m: int = 128, n: int = 64, density: float = 0.20, total: int = 65536) -> Batch:
    """Problems [start, start+count) of config 4's batch.  Problem p is a pure
    function of (seed, p): generated in chunks of 1024 so any slice (a rank's
    shard) can be drawn without the others."""
    if count is None:
        count = total - start
    nnz = int(round(density * m * n))
    rowptr_all = np.zeros((count, m + 1), dtype=np.int32)
    colind_all = np.zeros((count, nnz), dtype=np.int32)
    vals_all = np.zeros((count, nnz))
    b_all = np.zeros((count, m))
    x_all = np.zeros((count, n))
    p = start
    while p < start + count:
        chunk = p // _CHUNK
        c0 = chunk * _CHUNK
        csize = min(_CHUNK, total - c0) if total > c0 else _CHUNK
        rows, cols, vals, xs, noise = _batch_chunk(seed, m, n, density, chunk, csize, raw)
        lo = p - c0
        hi = min(csize, start + count - c0)
        for q in range(lo, hi):
            o = c0 + q - start
            rp = np.zeros(m + 1, dtype=np.int32)
            np.cumsum(np.bincount(rows[q], minlength=m), out=rp[1:])
            rowptr_all[o] = rp
            colind_all[o] = cols[q]
            vals_all[o] = vals[q]
            x_all[o] = xs[q]
            b_all[o] = _rhs(rp, cols[q].astype(np.int32), vals[q], xs[q], noise[q], raw)
        p = c0 + hi
    nnz_off = np.arange(count + 1, dtype=np.int64) * nnz
    return Batch(m, n, count, nnz_off, rowptr_all.reshape(-1), colind_all.reshape(-1),
                 vals_all.reshape(-1), b_all.reshape(-1), x_all.reshape(-1), int(seed), int(start))


def make_correlated(seed: int, corr: float = 0.05, nmin: int = 4, nmax: int = 9, grid: float = 256.0) -> Problem:
    """Tiny dense problems whose columns share a rank-2 component plus
    `corr` * N(0,1): nearly collinear, so block exchanges can fail to reduce
    the infeasible count and the single-exchange fallback fires.
    Entries quantized to 1/grid."""
    rng = np.random.default_rng([int(seed), 78])
    n = int(rng.integers(nmin, nmax))
    m = n + int(rng.integers(1, 5))
    base = rng.standard_normal((m, 2))
    A = np.round((base @ rng.standard_normal((2, n)) + corr * rng.standard_normal((m, n))) * grid) / grid
    b = np.round(rng.standard_normal(m) * grid) / grid
    p = from_dense(A, b)
    p.seed = int(seed)
    p.kind = "correlated"
    return p


def _householder_apply(vs, M):
    """(H_1 H_2 ... H_k) M for reflections H_i = I - 2 v v^T / v^T v (v in vs)."""
    for v in reversed(vs):
        M = M - np.outer(2.0 * v / (v @ v), v @ M)
    return M


def make_p_problem(m: int = 80, n: int = 70, d: int = 4, cond: float = 1e4, seed: int = 0,
                   resid: float = 0.25) -> Problem:
    """The paper's accuracy test family P(m, n, d, x) (Section 4:
    "each singular value is repeated 4 times, and x is a parameter which
    controls the condition number"; the original LSQR generator is not
    available -- this is SPEC.md's gen_p substitute):
    A = Y D Z^T with Y (m x m), Z (n x n) products of seeded Householder
    reflections, D = diag of ceil(n/d) singular values geometrically spaced
    from 1 down to 1/cond, each repeated d times; x_true_j = 1 + j/n; b =
    A x_true + r with r = Y (0_n; c) orthogonal to range(A), ||r|| = resid *
    ||A x_true|| (SPEC's 1/4 by default; the LSQR generator's residual size is
    not in the paper) -- so the NNLS solution is exactly x_true (y = A^T r = 0)
    and kappa(A) = cond.  Dense, unquantized (stored as CSR)."""
    assert m > n >= 1 and d >= 1 and cond >= 1.0
    rng = np.random.default_rng([int(seed), 8080, m, n, d])
    k = (n + d - 1) // d
    levels = cond ** (-np.arange(k) / max(k - 1, 1)) if k > 1 else np.ones(1)
    sig = np.repeat(levels, d)[:n]
    Y = _householder_apply([rng.standard_normal(m) for _ in range(m)], np.eye(m))
    Z = _householder_apply([rng.standard_normal(n) for _ in range(n)], np.eye(n))
    A = (Y[:, :n] * sig) @ Z.T
    x_true = 1.0 + np.arange(n) / n
    Ax = A @ x_true
    c = rng.standard_normal(m - n)
    r = Y[:, n:] @ c
    r *= (resid * np.linalg.norm(Ax)) / np.linalg.norm(r)
    p = from_dense(A, Ax + r)
    p.x_gen = x_true
    p.kind = "p_family"
    p.seed = int(seed)
    return p


def make_fig2(n: int, density: float, seed: int = 0) -> Problem:
    """The paper's timing workloads (Fig. 2): "randomly
    generated, well-conditioned matrices from MATLAB's sprandn ... of size
    n x (n-10)", density 1 ("general dense") and 0.01 ("sparse").  Stand-in:
    this module's seeded N(0,1) recipe (2^-12 grid) at that shape; the paper
    does not say how b was drawn -- b = A x0 + 0.01 N(0,1) as for the BASELINE
    configs (reading c25)."""
    return make_problem(dict(m=int(n), n=int(n) - 10, density=float(density)), seed=seed)
