"""ctypes wrapper around the plain C CPU oracle (oracle/nnls_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs are the only callers.  The product path
(paper_cs_0408029_b200) never imports this package; the oracle shares no code
with it.  The library is compiled with gcc -O2 -ffp-contract=off on first use
(or by __graft_entry__.build()).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nnls_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

STATUS = {0: "OK", 6: "OOM", 7: "NOT_PD", 8: "ITERATION_LIMIT"}


class Params(C.Structure):
    _fields_ = [("zero_tol", C.c_double), ("p_max", C.c_int32), ("max_iter", C.c_int32),
                ("lsqr_mode", C.c_int32), ("lsqr_atol", C.c_double), ("lsqr_btol", C.c_double),
                ("lsqr_conlim", C.c_double), ("lsqr_itn_limit", C.c_int32), ("notpd_fallback", C.c_int32),
                ("adaptive_threshold", C.c_double)]


class Info(C.Structure):
    _fields_ = [("status", C.c_int32), ("iterations", C.c_int32), ("single_exchanges", C.c_int32),
                ("free_count", C.c_int32), ("lsqr_iterations", C.c_int32), ("lsqr_stop", C.c_int32),
                ("infeasible_after_lsqr", C.c_int32), ("pad", C.c_int32),
                ("objective", C.c_double), ("kkt_min_x", C.c_double), ("kkt_min_y", C.c_double),
                ("kkt_max_comp", C.c_double), ("kkt_dot", C.c_double), ("kappa", C.c_double),
                ("refined", C.c_int32), ("lsqr_fallbacks", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad"}


class TraceRec(C.Structure):
    _fields_ = [("iter", C.c_int32), ("k", C.c_int32), ("branch", C.c_int32), ("f", C.c_int32),
                ("below_tol", C.c_double), ("above_tol", C.c_double)]


def build(force: bool = False) -> str:
    with _lock:
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
                                   "-o", tmp, _SRC, "-lm"])
            os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        P = C.c_void_p
        i32 = C.c_int32
        L.or_gram.argtypes = [i32, i32, P, P, P, P, P, P]
        L.or_gather.argtypes = [i32, P, i32, P, P]
        L.or_cholesky.argtypes = [i32, P, P]
        L.or_cholesky.restype = i32
        L.or_chol_solve.argtypes = [i32, P, P, P]
        L.or_dual_gram.argtypes = [i32, P, P, P, P, P]
        L.or_dual_eq5.argtypes = [i32, i32, P, P, P, P, P, P, P]
        L.or_clamp.argtypes = [i32, P, C.c_double]
        L.or_exchange.argtypes = [i32, P, P, P, P, P, i32, P]
        L.or_exchange.restype = i32
        L.or_lsqr.argtypes = [i32, i32, P, P, P, P, P, C.c_double, C.c_double, C.c_double, i32,
                              P, P, P, P, P, i32]
        L.or_lsqr.restype = i32
        L.or_kkt.argtypes = [i32, i32, P, P, P, P, P, P]
        L.or_condest.argtypes = [i32, P, C.c_double]
        L.or_condest.restype = C.c_double
        L.or_norm1.argtypes = [i32, P]
        L.or_norm1.restype = C.c_double
        L.or_bpp_solve.argtypes = [i32, i32, P, P, P, P, P, P, P, P, P, P, P, i32]
        L.or_bpp_solve.restype = i32
        L.or_bpp_solve_batched.argtypes = [i32, i32, i32, P, P, P, P, P, P, P, P, P, i32]
        L.or_bpp_solve_batched.restype = i32
        L.or_brute_force.argtypes = [i32, i32, P, P, P, P, C.c_double, P, P, i32]
        L.or_brute_force.restype = i32
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _csr(prob):
    return (np.ascontiguousarray(prob.rowptr, dtype=np.int32),
            np.ascontiguousarray(prob.colind, dtype=np.int32),
            np.ascontiguousarray(prob.vals, dtype=np.float64),
            np.ascontiguousarray(prob.b, dtype=np.float64))


def default_params(**kw) -> Params:
    p = Params(zero_tol=1e-12, p_max=3, max_iter=0, lsqr_mode=1, lsqr_atol=1e-15,
               lsqr_btol=1e-15, lsqr_conlim=1e8, lsqr_itn_limit=0, notpd_fallback=0,
               adaptive_threshold=1e-8)
    for k, v in kw.items():
        setattr(p, k, v)
    return p


# ---------------------------------------------------------------- step level
def gram(prob):
    rp, ci, v, b = _csr(prob)
    G = np.empty((prob.n, prob.n))
    c = np.empty(prob.n)
    lib().or_gram(prob.m, prob.n, _p(rp), _p(ci), _p(v), _p(b), _p(G), _p(c))
    return G, c


def gather(G, Fidx):
    G = np.ascontiguousarray(G, dtype=np.float64)
    F = np.ascontiguousarray(Fidx, dtype=np.int32)
    M = np.empty((F.size, F.size))
    lib().or_gather(G.shape[0], _p(G), F.size, _p(F), _p(M))
    return M


def cholesky(M):
    M = np.ascontiguousarray(M, dtype=np.float64)
    L = np.empty_like(M)
    rc = lib().or_cholesky(M.shape[0], _p(M), _p(L))
    return L, int(rc)


def chol_solve(L, rhs):
    L = np.ascontiguousarray(L, dtype=np.float64)
    r = np.ascontiguousarray(rhs, dtype=np.float64)
    x = np.empty_like(r)
    lib().or_chol_solve(L.shape[0], _p(L), _p(r), _p(x))
    return x


def dual_gram(G, c, mask, x):
    G = np.ascontiguousarray(G, dtype=np.float64)
    c = np.ascontiguousarray(c, dtype=np.float64)
    mk = np.ascontiguousarray(mask, dtype=np.uint8)
    xx = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(G.shape[0])
    lib().or_dual_gram(G.shape[0], _p(G), _p(c), _p(mk), _p(xx), _p(y))
    return y


def dual_eq5(prob, mask, x):
    rp, ci, v, b = _csr(prob)
    mk = np.ascontiguousarray(mask, dtype=np.uint8)
    xx = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(prob.n)
    lib().or_dual_eq5(prob.m, prob.n, _p(rp), _p(ci), _p(v), _p(b), _p(mk), _p(xx), _p(y))
    return y


def clamp(v, tol=1e-12):
    out = np.array(v, dtype=np.float64, copy=True)
    lib().or_clamp(out.size, _p(out), tol)
    return out


def exchange(mask, x, y, N, p, p_max=3):
    """Returns (k, new_mask, N, p, branch)."""
    mk = np.array(mask, dtype=np.uint8, copy=True)
    xx = np.ascontiguousarray(x, dtype=np.float64)
    yy = np.ascontiguousarray(y, dtype=np.float64)
    Nc, pc, br = C.c_int32(N), C.c_int32(p), C.c_int32(-1)
    k = lib().or_exchange(mk.size, _p(mk), _p(xx), _p(yy), C.byref(Nc), C.byref(pc), p_max, C.byref(br))
    return int(k), mk, Nc.value, pc.value, br.value


def lsqr(prob, mask=None, rhs=None, atol=1e-15, btol=1e-15, conlim=1e8, itn_limit=0):
    rp, ci, v, b = _csr(prob)
    mk = np.ones(prob.n, dtype=np.uint8) if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
    r = b if rhs is None else np.ascontiguousarray(rhs, dtype=np.float64)
    if itn_limit <= 0:
        itn_limit = 4 * max(1, int(mk.sum()))
    x = np.empty(prob.n)
    itn, rn, arn = C.c_int32(0), C.c_double(0), C.c_double(0)
    hist = np.zeros(itn_limit)
    istop = lib().or_lsqr(prob.m, prob.n, _p(rp), _p(ci), _p(v), _p(mk), _p(r), atol, btol, conlim,
                          itn_limit, _p(x), C.byref(itn), C.byref(rn), C.byref(arn), _p(hist), itn_limit)
    return dict(x=x, istop=int(istop), itn=itn.value, rnorm=rn.value, arnorm=arn.value,
                rnorm_hist=hist[:itn.value].copy())


def condest(L, norm1_M):
    """kappa_1 estimate of M = L L^T (Hager/Higham, as LAPACK dpocon): norm1_M * est(||M^-1||_1)."""
    L = np.ascontiguousarray(L, dtype=np.float64)
    return float(lib().or_condest(L.shape[0], _p(L), float(norm1_M)))


def norm1(M):
    M = np.ascontiguousarray(M, dtype=np.float64)
    return float(lib().or_norm1(M.shape[0], _p(M)))


def kkt(prob, x):
    rp, ci, v, b = _csr(prob)
    xx = np.ascontiguousarray(x, dtype=np.float64)
    info = Info()
    lib().or_kkt(prob.m, prob.n, _p(rp), _p(ci), _p(v), _p(b), _p(xx), C.byref(info))
    return info.as_dict()


def brute_force(prob, tol=1e-12, cap=64):
    """All feasible complementary partitions (as bit masks) for n <= 20."""
    rp, ci, v, b = _csr(prob)
    feas = np.zeros(cap, dtype=np.uint32)
    x0 = np.zeros(prob.n)
    cnt = lib().or_brute_force(prob.m, prob.n, _p(rp), _p(ci), _p(v), _p(b), tol, _p(feas), _p(x0), cap)
    if cnt < 0:
        raise ValueError("n > 20")
    masks = [np.array([(int(s) >> i) & 1 for i in range(prob.n)], dtype=np.uint8) for s in feas[:min(cnt, cap)]]
    return int(cnt), masks, x0


# ---------------------------------------------------------------- whole solve
def solve(prob, params: Params | None = None, trace_cap: int = 0, **kw):
    """The block principal pivoting algorithm + final LSQR."""
    prm = params if params is not None else default_params(**kw)
    rp, ci, v, b = _csr(prob)
    n = prob.n
    x = np.empty(n)
    x_ne = np.empty(n)
    mask = np.empty(n, dtype=np.uint8)
    y = np.empty(n)
    info = Info()
    tr = (TraceRec * max(trace_cap, 1))()
    lib().or_bpp_solve(prob.m, n, _p(rp), _p(ci), _p(v), _p(b), C.byref(prm), _p(x), _p(x_ne),
                       _p(mask), _p(y), C.byref(info), tr if trace_cap > 0 else None, trace_cap)
    out = info.as_dict()
    out.update(x=x, x_ne=x_ne, mask=mask, y=y)
    if trace_cap > 0:
        out["trace"] = [dict(iter=t.iter, k=t.k, branch=t.branch, f=t.f, below_tol=t.below_tol,
                             above_tol=t.above_tol) for t in tr[:min(info.iterations, trace_cap)]]
    return out


def solve_batched(batch, params: Params | None = None, threads: int = 0, **kw):
    prm = params if params is not None else default_params(**kw)
    x = np.empty(batch.count * batch.n)
    mask = np.empty(batch.count * batch.n, dtype=np.uint8)
    infos = (Info * max(batch.count, 1))()
    nnz_off = np.ascontiguousarray(batch.nnz_off, dtype=np.int64)
    used = lib().or_bpp_solve_batched(batch.count, batch.m, batch.n, _p(nnz_off),
                                      _p(np.ascontiguousarray(batch.rowptr, dtype=np.int32)),
                                      _p(np.ascontiguousarray(batch.colind, dtype=np.int32)),
                                      _p(np.ascontiguousarray(batch.vals, dtype=np.float64)),
                                      _p(np.ascontiguousarray(batch.b, dtype=np.float64)),
                                      C.byref(prm), _p(x), _p(mask), infos, threads)
    return dict(x=x.reshape(batch.count, batch.n), mask=mask.reshape(batch.count, batch.n),
                iterations=np.array([i.iterations for i in infos[:batch.count]]),
                single_exchanges=np.array([i.single_exchanges for i in infos[:batch.count]]),
                status=np.array([i.status for i in infos[:batch.count]]),
                threads=int(used))
