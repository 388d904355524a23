/*
 * nnls.h -- C ABI of the B200-native (sm_100a) hot path of tsnnls, the
 * block-principal-pivoting solver for sparse nonnegative least squares
 *
 *          min_x  1/2 || A x - b ||_2^2   subject to  x >= 0          (Eq. 1)
 *
 * (Cantarella & Piatek, arXiv cs/0408029; "P:n" = PAPER.md line n, "S:n" =
 * SPEC.md line n, readings c1..c21 = DESIGN.md §Readings).
 *
 * The library is libnnls_b200.so (paper_cs_0408029_b200/).  Every step of the
 * solve runs in hand-written sm_100a kernels; there is no CPU fallback: on a
 * machine without a usable B200 every call returns NNLS_ERR_CUDA.
 *
 * Conventions
 *   - All functions return an nnls_status; 0 = success.  Nothing throws.
 *   - Matrices are CSR: rowptr int32[m+1] (rowptr[0] = 0, nondecreasing,
 *     rowptr[m] = nnz), colind int32[nnz] (strictly increasing within a row,
 *     0 <= colind < n), vals float64[nnz] (finite).  b is float64[m].
 *   - Input pointers may be HOST or DEVICE memory (detected with
 *     cudaPointerGetAttributes).  nnls_setup* copies what it needs and keeps
 *     no caller pointer after it returns.  Output pointers (x_out, mask_out)
 *     may be host or device, caller-allocated.
 *   - Work is ordered on the CUDA stream given at setup (NULL = the legacy
 *     default stream).  Calls that return host outputs synchronize that
 *     stream before returning.
 *   - A handle is not thread-safe; distinct handles are independent.
 */
#ifndef NNLS_B200_H
#define NNLS_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define NNLS_API __attribute__((visibility("default")))
#else
#define NNLS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NNLS_OK = 0,
  NNLS_ERR_INVALID_ARG = 1,  /* NULL pointer, bad size, m < n, n < 1          */
  NNLS_ERR_DIMENSION = 2,    /* rowptr[0] != 0, rowptr decreasing, rowptr[m] != nnz */
  NNLS_ERR_INDEX = 3,        /* colind out of range or not strictly increasing in a row */
  NNLS_ERR_NONFINITE = 4,    /* a value of A or b is NaN/Inf                  */
  NNLS_ERR_CUDA = 5,         /* no device / kernel or runtime failure         */
  NNLS_ERR_OOM = 6,          /* device allocation failed                      */
  NNLS_ERR_NOT_PD = 7,       /* Cholesky pivot <= 0 or < 1e-300 (c13)   */
  NNLS_ITERATION_LIMIT = 8,  /* max_iter pivots without feasibility (c12); the
                                last iterate is returned                      */
  NNLS_ERR_STATE = 9         /* call out of order (e.g. solve before setup)   */
} nnls_status;

/* Solver parameters.  Fill with nnls_params_default. */
typedef struct {
  double zero_tol;        /* 1e-12: |v| < zero_tol -> 0 after every update
                             (strict, reading c1)               */
  int32_t p_max;          /* 3: the no-progress counter p of P:87, P:92 --
                             block exchanges allowed without reducing the
                             infeasible count before the single-exchange
                             fallback of P:98-99                             */
  int32_t max_iter;       /* 0 -> 10*n pivot iterations (reading c12)       */
  int32_t lsqr_mode;      /* 0: return the last normal-equations x;
                             1 (default): recompute x on the final F with
                             LSQR from x = 0 ("recomputing the final
                             solution");  2: LSQR correction started from
                             the normal-equations x;  3: adaptive -- a
                             1-norm condition estimate kappa of the final
                             (A^T A)_FF from its Cholesky factor (P:129,
                             LAPACK dpocon's estimator) decides: LSQR as in
                             mode 1 iff kappa * 2^-52 > adaptive_threshold,
                             else the normal-equations x                    */
  int32_t lsqr_itn_limit; /* 0 -> 4*|F|                              */
  double lsqr_atol;       /* 1e-15                                   */
  double lsqr_btol;       /* 1e-15                                           */
  double lsqr_conlim;     /* 1e8                                             */
  int32_t trace;          /* != 0: record one nnls_iter_rec per pivot       */
  int32_t kkt;            /* != 0 (default): fill the KKT fields of nnls_info */
  double adaptive_threshold; /* lsqr_mode 3: predicted relative error above
                                which LSQR runs (default 1e-8)       */
  int32_t notpd_fallback; /* != 0: a Cholesky failure ("may fail
                             entirely when kappa^2 eps >= 1") no longer ends
                             the solve: that iteration's x_F comes from LSQR
                             on A_F (cold start, the lsqr_* tolerances) and
                             pivoting continues.  Single-problem
                             handles only; batched handles return NOT_PD. */
  int32_t reserved;
} nnls_params;

/* Per-solve report. */
typedef struct {
  int32_t status;             /* nnls_status of the solve                   */
  int32_t iterations;         /* pivot iterations = normal-equations solves
                                 (reading c11; 0 when A^T b <= 0)           */
  int32_t single_exchanges;   /* times the P:98-99 branch was taken         */
  int32_t free_count;         /* |F| at exit                                */
  int32_t lsqr_iterations;
  int32_t lsqr_stop;          /* LSQR istop (0..7)                          */
  int32_t infeasible_after_lsqr; /* 1 if some x_F < 0 after LSQR + clamp (c16) */
  int32_t not_pd_column;      /* failing pivot position in F (NOT_PD), else -1 */
  double objective;           /* 1/2 ||A x - b||^2                          */
  double kkt_min_x;           /* min_i x_i                                  */
  double kkt_min_y;           /* min_i y'_i, y' = A^T (A x - b) recomputed  */
  double kkt_max_comp;        /* max_i |x_i y'_i|                           */
  double kkt_dot;             /* <x, y'>                                    */
  double kappa;               /* lsqr_mode 3: the condition estimate of the
                                 final (A^T A)_FF (0 in the other modes)    */
  int32_t refined;            /* 1 if the final x came from LSQR            */
  int32_t lsqr_fallbacks;     /* NOT_PD iterations solved by LSQR instead   */
} nnls_info;

/* One pivot iteration (for parity tests against the oracle's trace). */
typedef struct {
  int32_t iter;       /* 1-based iteration number                           */
  int32_t k;          /* infeasible count before the exchange        */
  int32_t branch;     /* 0: k < N; 1: p > 0; 2: single */
  int32_t f;          /* |F| after the exchange                            */
  double below_tol;   /* largest |v| < zero_tol over x_F, y_G before zeroing (0 if none) */
  double above_tol;   /* smallest |v| >= zero_tol over x_F, y_G (inf if none) */
  int32_t kept;       /* leading rows/columns of the previous iteration's
                         Cholesky factor reused unchanged by this one (factor
                         reuse, reading c22; 0 = full factorization).
                         Implementation record, not part of the paper's state */
  int32_t pad;
} nnls_iter_rec;

typedef struct nnls_handle nnls_handle;

NNLS_API const char* nnls_status_string(nnls_status s);
NNLS_API nnls_status nnls_params_default(nnls_params* p);
/* Device / library facts: number of SMs, compute capability (e.g. 100). */
NNLS_API nnls_status nnls_device_info(int32_t* sm_count, int32_t* cc, int32_t* device);

/* ---------------------------------------------------------------------------
 * Single problem (configs 0-3).
 *
 * nnls_setup: validates and uploads CSR A (m x n, m >= n >= 1; P:42 assumes
 * m > n and full column rank -- rank deficiency is detected only as NOT_PD),
 * builds a device CSC copy, and forms the Gram matrix G = A^T A (full
 * symmetric, FP64) and c = A^T b ONCE (P:126 caching).  p may be NULL
 * (defaults).  cuda_stream: cudaStream_t or NULL.  On error *h is NULL.
 */
NNLS_API nnls_status nnls_setup(nnls_handle** h, int32_t m, int32_t n, int64_t nnz,
                       const int32_t* rowptr, const int32_t* colind, const double* vals,
                       const double* b, const nnls_params* p, void* cuda_stream);

/* nnls_setup split in two: nnls_create makes an empty handle bound to a
 * stream; nnls_load (re)loads a problem into it -- validation, CSC build and
 * Gram formation run again on the new data; device buffers are reused when
 * large enough.  nnls_setup = nnls_create + nnls_load. */
NNLS_API nnls_status nnls_create(nnls_handle** h, const nnls_params* p, void* cuda_stream);
NNLS_API nnls_status nnls_load(nnls_handle* h, int32_t m, int32_t n, int64_t nnz,
                      const int32_t* rowptr, const int32_t* colind, const double* vals,
                      const double* b);

/* Runs the pivot loop of P:86-104 on the cached Gram (normal equations with a
 * blocked FP64 Cholesky, Gram-form dual y_G = (A^T A)_GF x_F - (A^T b)_G,
 * zeroing, exchange with single-exchange fallback), then the final LSQR of
 * P:124 per params.lsqr_mode.  x_out: float64[n] (host or device) receives
 * x >= 0 (on NNLS_ITERATION_LIMIT / NNLS_ERR_NOT_PD: the last iterate, which
 * may be infeasible, resp. x = 0).  info_out may be NULL.  May be called repeatedly (each call
 * restarts from F = {} on the cached Gram). */
NNLS_API nnls_status nnls_solve(nnls_handle* h, double* x_out, nnls_info* info_out);

/* Replace the parameters used by subsequent nnls_solve calls. */
NNLS_API nnls_status nnls_set_params(nnls_handle* h, const nnls_params* p);
/* Final free set F as a mask (1 = free), uint8[n], host or device. */
NNLS_API nnls_status nnls_get_free_set(nnls_handle* h, uint8_t* mask_out);
/* The last normal-equations x (before LSQR), float64[n], host or device. */
NNLS_API nnls_status nnls_get_x_ne(nnls_handle* h, double* x_out);
/* Copies min(cap, iterations) trace records of the last solve to host recs. */
NNLS_API nnls_status nnls_get_trace(nnls_handle* h, nnls_iter_rec* recs, int32_t cap, int32_t* count);
/* Copies the cached Gram (n x n row-major, full symmetric) and c = A^T b to
 * host or device buffers (either may be NULL).  For parity tests. */
NNLS_API nnls_status nnls_get_gram(nnls_handle* h, double* G_out, double* c_out);
NNLS_API nnls_status nnls_destroy(nnls_handle* h);

/* ---------------------------------------------------------------------------
 * Row-sharded Gram (config 2 across GPUs, BASELINE north_star; "A^T A
 * ... is computed once": the one step of the method that shards).  The Gram
 * is a sum over rows, G = sum_r a_r a_r^T, c = sum_r a_r b_r, so rank k forms
 * the partial sums of its row block and the ranks SUM them with one
 * collective through torch.distributed / NCCL (a reduce to the root, or an
 * all-reduce); only the root runs the pivot loop.
 *
 *   root:      nnls_setup_shard / nnls_load_shard with the FULL A and b (kept
 *              for the final LSQR and the report) and its own row range
 *              [row_begin, row_end);
 *   non-root:  nnls_create + nnls_load_block with ONLY its row block (local
 *              CSR of m_block rows, its slice of b; m_block < n allowed);
 *   all:       reduce (SUM, float64) the device buffer of nnls_gram_buffer;
 *   root:      nnls_gram_finalize, then nnls_solve.
 *
 * The buffer is the PACKED lower triangle (row i = G[i][0..i] at offset
 * i(i+1)/2) followed by c (n): n(n+1)/2 + n doubles, half the bytes of the
 * square.  With quantized (exact-sum) inputs the reduced Gram is bitwise
 * identical for any rank count.  nnls_solve before nnls_gram_finalize, and
 * finalize/solve on a block-only handle, return NNLS_ERR_STATE.
 */
NNLS_API nnls_status nnls_setup_shard(nnls_handle** h, int32_t m, int32_t n, int64_t nnz,
                             const int32_t* rowptr, const int32_t* colind, const double* vals,
                             const double* b, int32_t row_begin, int32_t row_end,
                             const nnls_params* p, void* cuda_stream);
/* Reload a (new) problem into a handle as the shard root (as nnls_load, the
 * partial Gram over rows [row_begin, row_end) only; finalize required again). */
NNLS_API nnls_status nnls_load_shard(nnls_handle* h, int32_t m, int32_t n, int64_t nnz,
                                     const int32_t* rowptr, const int32_t* colind,
                                     const double* vals, const double* b, int32_t row_begin,
                                     int32_t row_end);
/* A non-root rank's row block: CSR of m_block rows (rowptr local, starting
 * at 0), b_block[m_block]; validated like nnls_load (same error codes), then
 * its packed partial Gram is formed.  The handle can only serve
 * nnls_gram_buffer afterwards. */
NNLS_API nnls_status nnls_load_block(nnls_handle* h, int32_t m_block, int32_t n, int64_t nnz,
                                     const int32_t* rowptr, const int32_t* colind,
                                     const double* vals, const double* b_block);
/* Device pointer and element count (n(n+1)/2 + n) of the packed [G | c]
 * partial of a shard or block handle (owned by the handle; valid until the
 * next load or destroy). */
NNLS_API nnls_status nnls_gram_buffer(nnls_handle* h, double** dev_ptr, size_t* count);
/* Root only, after the reduction: expands the packed sum into the full
 * symmetric Gram the pivot loop reads (stream-ordered). */
NNLS_API nnls_status nnls_gram_finalize(nnls_handle* h);

/* ---------------------------------------------------------------------------
 * Batched independent problems (config 4; config 0 with batch = 1 also
 * fits): `batch` problems of identical shape m x n, CSR blocks concatenated.
 * nnz_off int64[batch+1] (nnz_off[0] = 0) gives each problem's slice of
 * colind/vals; rowptr is int32[batch*(m+1)] with problem-local offsets; b is
 * float64[batch*m].  Limits: n <= 64, m <= 256 (one CTA holds a problem on
 * chip).  nnls_solve_batched writes x_out float64[batch*n] and, if not
 * NULL, info_out[batch] (host) and mask_out uint8[batch*n].
 */
NNLS_API nnls_status nnls_setup_batched(nnls_handle** h, int32_t batch, int32_t m, int32_t n,
                               const int64_t* nnz_off, const int32_t* rowptr,
                               const int32_t* colind, const double* vals, const double* b,
                               const nnls_params* p, void* cuda_stream);
NNLS_API nnls_status nnls_solve_batched(nnls_handle* h, double* x_out, nnls_info* info_out,
                               uint8_t* mask_out);
/* nnls_load_batched + nnls_solve_batched as one pipelined call: the batch is
 * cut into chunks of `chunk` problems (<= 0: 8192); chunk k+1's inputs copy
 * host->device on one stream and chunk k-1's x_out / mask_out copy back on
 * another while chunk k is validated and solved on the handle's stream.
 * Arguments and results as the two calls (inputs host -- pinned for overlap
 * -- or device; outputs likewise).  A chunk that fails validation is not
 * solved (a device-side guard) and the call returns the first failing
 * chunk's status after all chunks finished; outputs are then unspecified.
 * Returns after the outputs are written (the stream is synchronized). */
NNLS_API nnls_status nnls_run_batched(nnls_handle* h, int32_t batch, int32_t m, int32_t n,
                             const int64_t* nnz_off, const int32_t* rowptr, const int32_t* colind,
                             const double* vals, const double* b, double* x_out,
                             nnls_info* info_out, uint8_t* mask_out, int32_t chunk);
/* nnls_setup_batched split in two, as nnls_create / nnls_load. */
NNLS_API nnls_status nnls_create_batched(nnls_handle** h, const nnls_params* p, void* cuda_stream);
NNLS_API nnls_status nnls_load_batched(nnls_handle* h, int32_t batch, int32_t m, int32_t n,
                              const int64_t* nnz_off, const int32_t* rowptr, const int32_t* colind,
                              const double* vals, const double* b);

/* ---------------------------------------------------------------------------
 * Step-level entry points on caller DEVICE buffers, for kernel unit tests
 * against the oracle's steps.  All sizes are element counts; all pointers are
 * device pointers; work is ordered on `stream` and synchronized on return.
 */
/* G (n x ldg row-major, full symmetric) and c = A^T b from device CSR. */
NNLS_API nnls_status nnls_step_gram(int32_t m, int32_t n, int64_t nnz, const int32_t* rowptr,
                           const int32_t* colind, const double* vals, const double* b,
                           double* G, int32_t ldg, double* c, void* stream);
/* Normal-equations solve on F: factor (A^T A)_FF gathered from G
 * via Fidx int32[f] (sorted) and solve for x_F (float64[f]) with rhs c[Fidx].
 * Returns NNLS_ERR_NOT_PD (with *not_pd_col set) on a failed pivot. */
NNLS_API nnls_status nnls_step_normal_solve(int32_t n, const double* G, int32_t ldg, const double* c,
                                   int32_t f, const int32_t* Fidx, double* xF,
                                   int32_t* not_pd_col, void* stream);
/* One count/decide/exchange step on device state mask uint8[n],
 * x, y float64[n]; state int32[4] = {N, p, iter, singles} in/out.  Writes
 * *k_out (infeasible count) and *branch_out (-1 feasible, 0, 1, 2). */
NNLS_API nnls_status nnls_step_exchange(int32_t n, uint8_t* mask, const double* x, const double* y,
                               int32_t p_max, int32_t* state, int32_t* k_out,
                               int32_t* branch_out, void* stream);
/* Gram-form dual (Eq. 5, north_star (4)) + zeroing: y_j for j not in
 * F from x (x_G = 0), then |x_F|,|y_G| < tol -> 0; writes y_F = 0. */
NNLS_API nnls_status nnls_step_dual(int32_t n, const double* G, int32_t ldg, const double* c,
                           const uint8_t* mask, double* x, double* y, double tol, void* stream);

/* ---------------------------------------------------------------------------
 * Instrumentation: per-phase CUDA-event timing on the handle's stream and
 * kernel-launch counts (the bench's roofline and gpu_launches evidence).
 * nnls_timing_enable(h, 1) resets the accumulators and records an event pair
 * around every phase; nnls_timing_read syncs the stream and returns the
 * accumulated milliseconds and launch counts per phase (cap entries).
 * Launch counts are kept even when timing is off.
 */
#define NNLS_NPHASES 16
enum {
  NNLS_PH_UPLOAD = 0,      /* input copies into the handle (H2D or D2D)          */
  NNLS_PH_VALIDATE = 1,    /* a0 CSR validation                                  */
  NNLS_PH_CSC = 2,         /* a0 CSR -> CSC (4 kernels)                          */
  NNLS_PH_GRAM = 3,        /* a1 A^T A, A^T b                                    */
  NNLS_PH_INIT = 4,        /* a2                                                 */
  NNLS_PH_DECIDE = 5,      /* a3 + a4 count/decide/exchange/compaction           */
  NNLS_PH_CHOL_FACTOR = 6, /* a5 (+ forward solve via the bordered row)          */
  NNLS_PH_CHOL_SOLVE = 7,  /* a6 back substitution                               */
  NNLS_PH_DUAL = 8,        /* a7 + a8                                            */
  NNLS_PH_LSQR = 9,        /* a10 + a11 report                                   */
  NNLS_PH_DOWNLOAD = 10,   /* x_out copy                                         */
  NNLS_PH_BATCHED = 11     /* batched whole-solve kernel                         */
};
NNLS_API nnls_status nnls_timing_enable(nnls_handle* h, int32_t on);
NNLS_API nnls_status nnls_timing_read(nnls_handle* h, double* ms, int64_t* launches, int32_t cap);

#ifdef __cplusplus
}
#endif
#endif /* NNLS_B200_H */
