"""Python binding of libnnls_b200.so -- the B200 (sm_100a) hot path of tsnnls'
block principal pivoting NNLS solver (Cantarella & Piatek, arXiv cs/0408029).

Argument marshalling only: every arithmetic step runs in the library's CUDA
kernels (see include/nnls.h).  Arrays may be numpy arrays (host) or torch
tensors (host or CUDA); their data pointers are passed to the C ABI, which
copies what it needs.  There is no CPU fallback: if the shared library is
missing or cannot load, importing this package raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnnls_b200.so")
HEADER = os.path.join(os.path.dirname(_HERE), "include", "nnls.h")

OK, ERR_INVALID_ARG, ERR_DIMENSION, ERR_INDEX, ERR_NONFINITE, ERR_CUDA, ERR_OOM, ERR_NOT_PD, \
    ITERATION_LIMIT, ERR_STATE = range(10)
STATUS_NAMES = ["OK", "ERR_INVALID_ARG", "ERR_DIMENSION", "ERR_INDEX", "ERR_NONFINITE", "ERR_CUDA",
                "ERR_OOM", "ERR_NOT_PD", "ITERATION_LIMIT", "ERR_STATE"]


NPHASES = 16
PHASES = ["upload", "validate", "csc", "gram", "init", "decide", "chol_factor", "chol_solve", "dual",
          "lsqr", "download", "batched"]


class NNLSError(RuntimeError):
    def __init__(self, status, where=""):
        self.status = int(status)
        name = STATUS_NAMES[self.status] if 0 <= self.status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{where}: {name}")


class Params(C.Structure):
    _fields_ = [("zero_tol", C.c_double), ("p_max", C.c_int32), ("max_iter", C.c_int32),
                ("lsqr_mode", C.c_int32), ("lsqr_itn_limit", C.c_int32), ("lsqr_atol", C.c_double),
                ("lsqr_btol", C.c_double), ("lsqr_conlim", C.c_double), ("trace", C.c_int32),
                ("kkt", C.c_int32), ("adaptive_threshold", C.c_double), ("notpd_fallback", C.c_int32),
                ("reserved", C.c_int32)]


class Info(C.Structure):
    _fields_ = [("status", C.c_int32), ("iterations", C.c_int32), ("single_exchanges", C.c_int32),
                ("free_count", C.c_int32), ("lsqr_iterations", C.c_int32), ("lsqr_stop", C.c_int32),
                ("infeasible_after_lsqr", C.c_int32), ("not_pd_column", C.c_int32),
                ("objective", C.c_double), ("kkt_min_x", C.c_double), ("kkt_min_y", C.c_double),
                ("kkt_max_comp", C.c_double), ("kkt_dot", C.c_double), ("kappa", C.c_double),
                ("refined", C.c_int32), ("lsqr_fallbacks", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class IterRec(C.Structure):
    _fields_ = [("iter", C.c_int32), ("k", C.c_int32), ("branch", C.c_int32), ("f", C.c_int32),
                ("below_tol", C.c_double), ("above_tol", C.c_double), ("kept", C.c_int32),
                ("pad", C.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(python paper_cs_0408029_b200/build.py); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    P, i32, i64, d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "nnls_status_string": ([i32], C.c_char_p),
        "nnls_params_default": ([P], i32),
        "nnls_device_info": ([P, P, P], i32),
        "nnls_create": ([P, P, P], i32),
        "nnls_load": ([P, i32, i32, i64, P, P, P, P], i32),
        "nnls_setup": ([P, i32, i32, i64, P, P, P, P, P, P], i32),
        "nnls_solve": ([P, P, P], i32),
        "nnls_set_params": ([P, P], i32),
        "nnls_get_free_set": ([P, P], i32),
        "nnls_get_x_ne": ([P, P], i32),
        "nnls_get_trace": ([P, P, i32, P], i32),
        "nnls_get_gram": ([P, P, P], i32),
        "nnls_destroy": ([P], i32),
        "nnls_setup_shard": ([P, i32, i32, i64, P, P, P, P, i32, i32, P, P], i32),
        "nnls_gram_buffer": ([P, P, P], i32),
        "nnls_load_block": ([P, i32, i32, i64, P, P, P, P], i32),
        "nnls_load_shard": ([P, i32, i32, i64, P, P, P, P, i32, i32], i32),
        "nnls_gram_finalize": ([P], i32),
        "nnls_setup_batched": ([P, i32, i32, i32, P, P, P, P, P, P, P], i32),
        "nnls_create_batched": ([P, P, P], i32),
        "nnls_load_batched": ([P, i32, i32, i32, P, P, P, P, P], i32),
        "nnls_solve_batched": ([P, P, P, P], i32),
        "nnls_run_batched": ([P, i32, i32, i32, P, P, P, P, P, P, P, P, i32], i32),
        "nnls_step_gram": ([i32, i32, i64, P, P, P, P, P, i32, P, P], i32),
        "nnls_step_normal_solve": ([i32, P, i32, P, i32, P, P, P, P], i32),
        "nnls_step_exchange": ([i32, P, P, P, i32, P, P, P, P], i32),
        "nnls_step_dual": ([i32, P, i32, P, P, P, P, d, P], i32),
        "nnls_timing_enable": ([P, i32], i32),
        "nnls_timing_read": ([P, P, P, i32], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    return L


lib = _load()


def header_symbols():
    """Names of every function include/nnls.h declares."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^NNLS_API\s+[\w\s\*]+?\b(nnls_\w+)\s*\(", txt, flags=re.M)))


def _ptr(a):
    """Data pointer of a numpy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return C.c_void_p(a.ctypes.data)
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return C.c_void_p(a.data_ptr())
    raise TypeError(f"unsupported array type {type(a)}")


def _as(a, dtype):
    if hasattr(a, "data_ptr"):
        return a
    return np.ascontiguousarray(a, dtype=dtype)


def _stream_ptr(stream):
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


def _check(st, where):
    if st != OK:
        raise NNLSError(st, where)


def default_params(**kw) -> Params:
    p = Params()
    _check(lib.nnls_params_default(C.byref(p)), "nnls_params_default")
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def device_info():
    sms, cc, dev = C.c_int32(), C.c_int32(), C.c_int32()
    _check(lib.nnls_device_info(C.byref(sms), C.byref(cc), C.byref(dev)), "nnls_device_info")
    return dict(sm_count=sms.value, cc=cc.value, device=dev.value)


class Solver:
    """One problem: nnls_create / nnls_load / nnls_solve (configs 0-3)."""

    def __init__(self, params: Params | None = None, stream=None, **kw):
        self.params = params if params is not None else default_params(**kw)
        self.h = C.c_void_p()
        _check(lib.nnls_create(C.byref(self.h), C.byref(self.params), _stream_ptr(stream)), "nnls_create")
        self.m = self.n = 0

    def load(self, m, n, rowptr, colind, vals, b):
        rp, ci, v, bb = _as(rowptr, np.int32), _as(colind, np.int32), _as(vals, np.float64), _as(b, np.float64)
        nnz = int(ci.shape[0])
        _check(lib.nnls_load(self.h, int(m), int(n), nnz, _ptr(rp), _ptr(ci), _ptr(v), _ptr(bb)), "nnls_load")
        self.m, self.n = int(m), int(n)
        return self

    def load_problem(self, prob):
        return self.load(prob.m, prob.n, prob.rowptr, prob.colind, prob.vals, prob.b)

    def set_params(self, params: Params | None = None, **kw):
        if params is None:
            params = self.params
            for k, v in kw.items():
                setattr(params, k, v)
        self.params = params
        _check(lib.nnls_set_params(self.h, C.byref(params)), "nnls_set_params")

    def solve(self, x_out=None, check=True):
        """Returns (x, info dict).  x_out may be a host array or a CUDA tensor."""
        x = x_out if x_out is not None else np.empty(self.n)
        info = Info()
        st = lib.nnls_solve(self.h, _ptr(x), C.byref(info))
        if check and st not in (OK, ERR_NOT_PD, ITERATION_LIMIT):
            raise NNLSError(st, "nnls_solve")
        return x, info.as_dict()

    def free_set(self, out=None):
        mk = out if out is not None else np.empty(self.n, dtype=np.uint8)
        _check(lib.nnls_get_free_set(self.h, _ptr(mk)), "nnls_get_free_set")
        return mk

    def x_ne(self, out=None):
        x = out if out is not None else np.empty(self.n)
        _check(lib.nnls_get_x_ne(self.h, _ptr(x)), "nnls_get_x_ne")
        return x

    def trace(self, cap=100000):
        recs = (IterRec * cap)()
        cnt = C.c_int32()
        _check(lib.nnls_get_trace(self.h, recs, cap, C.byref(cnt)), "nnls_get_trace")
        return [dict(iter=r.iter, k=r.k, branch=r.branch, f=r.f, below_tol=r.below_tol,
                     above_tol=r.above_tol, kept=r.kept) for r in recs[:cnt.value]]

    def gram(self):
        G = np.empty((self.n, self.n))
        c = np.empty(self.n)
        _check(lib.nnls_get_gram(self.h, _ptr(G), _ptr(c)), "nnls_get_gram")
        return G, c

    def close(self):
        if self.h:
            lib.nnls_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def timing_enable(handle, on=True):
    _check(lib.nnls_timing_enable(handle, 1 if on else 0), "nnls_timing_enable")


def timing_read(handle):
    """{phase: (ms, launches)} accumulated since timing_enable."""
    ms = (C.c_double * NPHASES)()
    nl = (C.c_int64 * NPHASES)()
    _check(lib.nnls_timing_read(handle, ms, nl, NPHASES), "nnls_timing_read")
    return {name: (ms[i], nl[i]) for i, name in enumerate(PHASES)}


def setup(prob, params: Params | None = None, stream=None, **kw) -> Solver:
    return Solver(params, stream, **kw).load_problem(prob)


class ShardSolver(Solver):
    """Row-sharded Gram, shard ROOT (include/nnls.h): holds the full A and b,
    forms the packed partial Gram of its own rows [row_begin, row_end); after
    the ranks' reduction (paper_cs_0408029_b200.dist.reduce_gram) finalize()
    expands it and solve() runs the pivot loop."""

    def __init__(self, m, n, rowptr, colind, vals, b, row_begin, row_end, params=None, stream=None, **kw):
        self.params = params if params is not None else default_params(**kw)
        self.h = C.c_void_p()
        rp, ci, v, bb = _as(rowptr, np.int32), _as(colind, np.int32), _as(vals, np.float64), _as(b, np.float64)
        _check(lib.nnls_setup_shard(C.byref(self.h), int(m), int(n), int(ci.shape[0]), _ptr(rp), _ptr(ci),
                                    _ptr(v), _ptr(bb), int(row_begin), int(row_end),
                                    C.byref(self.params), _stream_ptr(stream)), "nnls_setup_shard")
        self.m, self.n = int(m), int(n)

    def load_shard(self, m, n, rowptr, colind, vals, b, row_begin, row_end):
        rp, ci, v, bb = _as(rowptr, np.int32), _as(colind, np.int32), _as(vals, np.float64), _as(b, np.float64)
        _check(lib.nnls_load_shard(self.h, int(m), int(n), int(ci.shape[0]), _ptr(rp), _ptr(ci), _ptr(v),
                                   _ptr(bb), int(row_begin), int(row_end)), "nnls_load_shard")
        self.m, self.n = int(m), int(n)
        return self

    def gram_buffer(self):
        """(device pointer, element count) of the packed [G lower | c] partial."""
        p, cnt = C.c_void_p(), C.c_size_t()
        _check(lib.nnls_gram_buffer(self.h, C.byref(p), C.byref(cnt)), "nnls_gram_buffer")
        return p.value, cnt.value

    def finalize(self):
        _check(lib.nnls_gram_finalize(self.h), "nnls_gram_finalize")


class BlockSolver(Solver):
    """Row-sharded Gram, NON-ROOT rank: only its row block (local CSR of
    m_block rows and b_block) is uploaded; it contributes the packed partial
    Gram to the reduction and never solves."""

    def load_block(self, m_block, n, rowptr, colind, vals, b_block):
        rp, ci, v, bb = _as(rowptr, np.int32), _as(colind, np.int32), _as(vals, np.float64), _as(b_block, np.float64)
        _check(lib.nnls_load_block(self.h, int(m_block), int(n), int(ci.shape[0]), _ptr(rp), _ptr(ci), _ptr(v),
                                   _ptr(bb)), "nnls_load_block")
        self.m, self.n = int(m_block), int(n)
        return self

    gram_buffer = ShardSolver.gram_buffer


class BatchedSolver:
    """Independent problems of one shape (config 4): nnls_*_batched."""

    def __init__(self, params: Params | None = None, stream=None, **kw):
        self.params = params if params is not None else default_params(**kw)
        self.h = C.c_void_p()
        _check(lib.nnls_create_batched(C.byref(self.h), C.byref(self.params), _stream_ptr(stream)),
               "nnls_create_batched")
        self.batch = self.m = self.n = 0

    def load(self, batch, m, n, nnz_off, rowptr, colind, vals, b):
        off, rp = _as(nnz_off, np.int64), _as(rowptr, np.int32)
        ci, v, bb = _as(colind, np.int32), _as(vals, np.float64), _as(b, np.float64)
        _check(lib.nnls_load_batched(self.h, int(batch), int(m), int(n), _ptr(off), _ptr(rp), _ptr(ci),
                                     _ptr(v), _ptr(bb)), "nnls_load_batched")
        self.batch, self.m, self.n = int(batch), int(m), int(n)
        return self

    def load_batch(self, B):
        return self.load(B.count, B.m, B.n, B.nnz_off, B.rowptr, B.colind, B.vals, B.b)

    def solve(self, x_out=None, mask_out=None, want_info=True, check=True):
        x = x_out if x_out is not None else np.empty(self.batch * self.n)
        mk = mask_out if mask_out is not None else (np.empty(self.batch * self.n, dtype=np.uint8)
                                                    if want_info else None)
        infos = (Info * self.batch)() if want_info else None
        st = lib.nnls_solve_batched(self.h, _ptr(x), infos, _ptr(mk))
        if check and st not in (OK, ERR_NOT_PD, ITERATION_LIMIT):
            raise NNLSError(st, "nnls_solve_batched")
        out = dict(x=x, mask=mk, status=st)
        if want_info:
            out["info"] = {k: np.array([getattr(i, k) for i in infos]) for k, _ in Info._fields_}
        return out

    def run(self, batch, m, n, nnz_off, rowptr, colind, vals, b, x_out=None, mask_out=None,
            want_info=True, chunk=0, check=True):
        """load + solve in one pipelined call (nnls_run_batched): chunk k+1's
        inputs copy in and chunk k-1's x copies out while chunk k solves.
        Same results as load(...) then solve(...)."""
        off, rp = _as(nnz_off, np.int64), _as(rowptr, np.int32)
        ci, v, bb = _as(colind, np.int32), _as(vals, np.float64), _as(b, np.float64)
        x = x_out if x_out is not None else np.empty(int(batch) * int(n))
        mk = mask_out if mask_out is not None else (np.empty(int(batch) * int(n), dtype=np.uint8)
                                                    if want_info else None)
        infos = (Info * int(batch))() if want_info else None
        st = lib.nnls_run_batched(self.h, int(batch), int(m), int(n), _ptr(off), _ptr(rp), _ptr(ci), _ptr(v),
                                  _ptr(bb), _ptr(x), infos, _ptr(mk), int(chunk))
        if check and st not in (OK, ERR_NOT_PD, ITERATION_LIMIT):
            raise NNLSError(st, "nnls_run_batched")
        self.batch, self.m, self.n = int(batch), int(m), int(n)
        out = dict(x=x, mask=mk, status=st)
        if want_info:
            out["info"] = {k: np.array([getattr(i, k) for i in infos]) for k, _ in Info._fields_}
        return out

    def run_batch(self, B, **kw):
        return self.run(B.count, B.m, B.n, B.nnz_off, B.rowptr, B.colind, B.vals, B.b, **kw)

    def close(self):
        if self.h:
            lib.nnls_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------- step level
def step_gram(m, n, rowptr, colind, vals, b, G, c, ldg=None, stream=None):
    """Device buffers (torch CUDA tensors)."""
    _check(lib.nnls_step_gram(int(m), int(n), int(colind.shape[0]), _ptr(rowptr), _ptr(colind), _ptr(vals),
                              _ptr(b), _ptr(G), int(ldg or n), _ptr(c), _stream_ptr(stream)), "nnls_step_gram")


def step_normal_solve(n, G, c, Fidx, xF, ldg=None, stream=None):
    col = C.c_int32(-1)
    st = lib.nnls_step_normal_solve(int(n), _ptr(G), int(ldg or n), _ptr(c), int(Fidx.shape[0]), _ptr(Fidx),
                                    _ptr(xF), C.byref(col), _stream_ptr(stream))
    if st not in (OK, ERR_NOT_PD):
        raise NNLSError(st, "nnls_step_normal_solve")
    return st, col.value


def step_exchange(n, mask, x, y, state, p_max=3, stream=None):
    """state: [N, p, iter, singles] (updated in place, host list/array)."""
    s = (C.c_int32 * 4)(*[int(v) for v in state])
    k, br = C.c_int32(), C.c_int32()
    _check(lib.nnls_step_exchange(int(n), _ptr(mask), _ptr(x), _ptr(y), int(p_max), s, C.byref(k),
                                  C.byref(br), _stream_ptr(stream)), "nnls_step_exchange")
    for i in range(4):
        state[i] = s[i]
    return k.value, br.value


def step_dual(n, G, c, mask, x, y, tol=1e-12, ldg=None, stream=None):
    _check(lib.nnls_step_dual(int(n), _ptr(G), int(ldg or n), _ptr(c), _ptr(mask), _ptr(x), _ptr(y),
                              float(tol), _stream_ptr(stream)), "nnls_step_dual")
