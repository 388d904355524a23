// kernels.cuh -- host-side launchers of the sm_100a kernels (one .cu per step).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace nnls {

constexpr int kTile = 64;  // Cholesky tile edge (T x T FP64 tiles, DMMA 8x8x4 updates)

// ---- a0 ingest (ingest_gram.cu) ------------------------------------------
// Validation error bits written to *err (device int): 1 dimension, 2 index,
// 4 non-finite.
cudaError_t launch_validate(int m, int n, int64_t nnz, const int32_t* rowptr, const int32_t* colind,
                            const double* vals, const double* b, int* err, cudaStream_t s);
// CSR -> CSC (rows sorted within each column).  colcnt: int32[n+1] scratch,
// tmp_row/tmp_val: nnz scratch.
// colcount + scan only (safe on unvalidated CSR: out-of-range columns are
// skipped), then the rest of the CSC build after validation.
cudaError_t launch_csc_count(int m, int n, int64_t nnz, const int32_t* colind, int32_t* colptr,
                             int32_t* cursor, cudaStream_t s, int* maxcnt);
cudaError_t launch_csc_fill(int m, int n, const int32_t* rowptr, const int32_t* colind,
                            const double* vals, const int32_t* colptr, int32_t* rowind,
                            double* cvals, int32_t* cursor, int32_t* tmp_row, double* tmp_val,
                            cudaStream_t s, int maxcnt = -1);
// four device-to-device copies (src[q] -> dst[q], bytes[q]) in one launch
cudaError_t launch_upload_copy(const void* const* src, void* const* dst, const size_t* bytes, int sm_count,
                               cudaStream_t s);
// the same CSC by a stable radix sort on the column (CUB): temp_bytes from
// csc_sort_temp_bytes (0: not available, use launch_csc_fill)
size_t csc_sort_temp_bytes(int64_t nnz, int n);
cudaError_t launch_csc_fill_sorted(int m, int n, int64_t nnz, const int32_t* rowptr, const int32_t* colind,
                                   const double* vals, int32_t* rowind, double* cvals, int32_t* tmp_row,
                                   double* tmp_val, void* temp, size_t temp_bytes, cudaStream_t s);
cudaError_t launch_csr_to_csc(int m, int n, int64_t nnz, const int32_t* rowptr,
                              const int32_t* colind, const double* vals, int32_t* colptr,
                              int32_t* rowind, double* cvals, int32_t* cursor, int32_t* tmp_row,
                              double* tmp_val, cudaStream_t s, int* maxcnt = nullptr);
// ---- a1 Gram + c (ingest_gram.cu) ---------------------------------------
// G (n rows of stride ldg) = A_R^T A_R and c = A_R^T b_R over rows R =
// [row_begin, row_end) (all rows: 0, m).
// err[kErrExp..+3]: exponent statistics of A and b from validate (see
// exact_bits); gram_is_exact(err) -> every Gram/c sum is exact in FP64.
constexpr int kErrExp = 48;
bool gram_is_exact(const int* err);    // exact AND the column fits gram_exact_kernel
bool gram_bits_exact(const int* err);  // exact (bit budget only): A^T A and A^T b
bool gram_A_exact(const int* err);     // A^T A exact
bool gram_c_exact(const int* err);     // A^T b exact
inline int gram_exact_lmin(const int* err) { return 2048 - err[kErrExp + 1]; }  // L_A
// ldg <= 0: G is the packed lower triangle (row i = entries j <= i at offset
// i(i+1)/2) -- the row-shard partial Gram that ranks reduce.
// launch_gram_unpack: packed -> full symmetric n x ldg.
cudaError_t launch_gram_unpack(int n, const double* P, double* G, int ldg, int sm_count, cudaStream_t s);
// dense A (gram_dense.cu): G = A^T A over rows [row_begin, row_end) as a DMMA
// SYRK on a tiled dense copy At (gram_dense_doubles(rows, n) doubles), c from
// the CSC.  Exact-arithmetic inputs only (the order differs from the oracle's).
size_t gram_dense_doubles(int rows, int n);
// c_exact: A^T b exact in any order (else summed per column in increasing
// row order, the oracle's order: bitwise either way)
cudaError_t launch_gram_dense(int n, const int32_t* rowptr, const int32_t* colind, const double* vals,
                              const int32_t* colptr, const int32_t* rowind, const double* cvals, const double* b,
                              int row_begin, int row_end, double* At, double* G, int ldg, double* c, int sm_count,
                              cudaStream_t s, bool c_exact);
cudaError_t launch_gram(int m, int n, const int32_t* rowptr, const int32_t* colind,
                        const double* vals, const int32_t* colptr, const int32_t* rowind,
                        const double* cvals, const double* b, int row_begin, int row_end,
                        double* G, int ldg, double* c, int sm_count, cudaStream_t s, bool exact = false, int exact_lmin = 0,
                        int max_row = 0, int max_col = 0);

// ---- a2/a3/a4/a7/a8 pivot steps (pivot.cu) -----------------------------
cudaError_t launch_init(int n, const double* c, uint8_t* mask, double* x, double* y, double tol,
                        DevState* st, int p_max, int max_iter, cudaStream_t s, int32_t* pos = nullptr);
// count + decide + exchange + compaction (one CTA); records trace[iter] head.
// loop != nullptr: the kernel runs inside a CUDA-graph WHILE node and clears
// its condition when the pivot loop ends (feasible, limit, or failure).
// pos == nullptr: Fidx = F in index order.  pos != nullptr (factor reuse):
// pos[i] = position of i in the previous factorization order (-1: not in
// F); Fidx keeps the previous order's longest prefix that survived the
// exchange and appends the rest by predicted stability; st->reuse_cols =
// the whole tile columns of that prefix (see cholesky.cu).
cudaError_t launch_decide(int n, uint8_t* mask, const double* x, const double* y, int32_t* Fidx,
                          int32_t* Gidx, DevState* st, TraceRec* trace, int trace_cap,
                          cudaStream_t s, const cudaGraphConditionalHandle* loop = nullptr,
                          int32_t* pos = nullptr, int32_t* Fs = nullptr, double* xs = nullptr);
cudaError_t launch_compact(int n, const uint8_t* mask, const double* x, int32_t* Fidx,
                           int32_t* Gidx, double* xF, DevState* st, cudaStream_t s);
// y_G = G_GF x_F - c_G (Gram form of Eq. 5), zeroing, scatter x_F into x.
// Fs/xs (factor reuse): F in index order and x_F scattered by index.
cudaError_t launch_dual(int n, const double* G, int ldg, const double* c, const int32_t* Fidx,
                        const int32_t* Gidx, const double* xF, uint8_t* mask, double* x,
                        double* y, double tol, DevState* st, int sm_count, cudaStream_t s,
                        const int32_t* Fs = nullptr, const double* xs = nullptr,
                        int32_t* inflist = nullptr);

// ---- a5/a6 Cholesky + solves (cholesky.cu) -------------------------------
size_t chol_tile_doubles(int n);
size_t chol_flag_count(int n);
cudaError_t chol_debug_set_profile(unsigned long long* p);  // tiles needed for |F| <= n (bordered, lower)
// Factor the bordered matrix [[G_FF, .], [c_F^T, .]] (gathered from G via
// Fidx) into tiles Lt, then back-substitute L^T x_F = z.  f read from st.
cudaError_t launch_cholesky_solve(int n, const double* G, int ldg, const double* c,
                                  const int32_t* Fidx, double* Lt, int* flags, double* xF,
                                  DevState* st, int sm_count, cudaStream_t s);
cudaError_t launch_chol_factor(int n, const double* G, int ldg, const double* c, const int32_t* Fidx,
                               double* Lt, int* flags, DevState* st, int sm_count, cudaStream_t s);
// xs != nullptr: also xs[Fidx[a]] = x_F[a] (the dual's index-order view)
cudaError_t launch_chol_backsolve(int n, const double* Lt, int* flags, double* xF, DevState* st,
                                  int sm_count, cudaStream_t s, const int32_t* Fidx = nullptr,
                                  double* xs = nullptr);

// ---- NEXT-2 condition estimate (condest.cu) --------------------------------
// kappa_1 estimate of the final (A^T A)_FF = L L^T from the factor tiles Lt
// (layout of cholesky.cu, n = the handle's size), written to st->kappa, and
// st->refined = kappa * 2^-52 > threshold.  work: 6 n doubles; norm1: one u64.
cudaError_t launch_condest(const double* G, int ldg, const int32_t* Fidx, const double* Lt, int n, DevState* st,
                           double* work, unsigned long long* norm1, double threshold, int sm_count, cudaStream_t s);
// NOT_PD fallback steps (pivot.cu): before the LSQR on the failed F (status
// cleared, done raised so the LSQR kernels take it as a final F) and after it
// (x_F from the LSQR x, done cleared, counter).
cudaError_t launch_fallback_prep(DevState* st, cudaStream_t s);
cudaError_t launch_fallback_fixup(int n, const int32_t* Fidx, const double* xl, double* xF, double* xs,
                                  DevState* st, cudaStream_t s);

// ---- a10 LSQR + final report (lsqr.cu) ----------------------------------
struct LsqrArgs {
  int m, n;
  const int32_t *rowptr, *colind;
  const double* vals;
  const int32_t *colptr, *rowind;
  const double* cvals;
  const double* b;
  const uint8_t* mask;
  const double* x_ne;   // normal-equations x (length n, zero on G)
  double* x_out;        // final x (length n)
  double *U, *V, *W, *X;   // work: U[m], V/W/X[n]
  double* R;            // work[m] (residual for the report)
  double* partials;     // work[gridDim * 8]
  DevState* st;
  int mode;             // 0 none, 1 cold, 2 warm
  int itn_limit;        // <= 0 -> 4 f
  double atol, btol, conlim, tol;
  int kkt;
  const double* G; int ldg; const double* c;   // for y (report)
  // rows of A restricted to the final F, compacted in place of each row
  // (row r: Fcnt[r] entries from offset rowptr[r]); built by launch_lsqr_compact
  double* Fval; int32_t* Fcol; int32_t* Fcnt;
  const int32_t* Fidx;  // the final F (f entries; from the last decide)
  const int32_t* Gidx;  // the final G (n - f entries, index order; the resident report)
  const int* plan;      // cluster slice plan (lsqr_plan_kernel: maxima, row bounds, column bounds)
  int res_cap;          // resident LSQR: slice budget override in bytes (0: the kernel's maximum)
};
cudaError_t launch_lsqr_compact(const LsqrArgs& a, int sm_count, cudaStream_t s);
cudaError_t launch_lsqr_final(const LsqrArgs& a, int sm_count, cudaStream_t s);
// Cluster-resident variant for problems whose CSR + CSC slices fit in the
// shared memory of one thread-block cluster (max_row / max_col: longest
// row / column).  Returns cudaErrorNotSupported when it does not fit.
cudaError_t lsqr_debug_set_profile(unsigned long long* p);
cudaError_t launch_lsqr_plan(int m, int n, const int32_t* rowptr, const int32_t* colptr, int* out,
                             cudaStream_t s);
size_t lsqr_cluster_smem(int m, int n, const int* plan);
cudaError_t launch_lsqr_cluster_planned(const LsqrArgs& a, const int* plan_host, cudaStream_t s);

// ---- batched whole solve (batched.cu) ------------------------------------
constexpr int kInfoI = 10, kInfoD = 6;  // per-problem report slots of the batched kernels
struct BatchArgs {
  int batch, m, n;
  const int64_t* nnz_off;
  const int32_t* rowptr;
  const int32_t* colind;
  const double* vals;
  const double* b;
  double* x_out;
  uint8_t* mask_out;
  int32_t* info_i;   // batch * kInfoI ints: status, iter, singles, f, lsqr_itn, lsqr_stop, infeas, notpd, refined, -
  double* info_d;    // batch * kInfoD doubles: objective, min_x, min_y, max_comp, dot, kappa
  double tol, atol, btol, conlim;
  int p_max, max_iter, lsqr_mode, itn_limit, kkt;
  double adaptive_threshold;  // lsqr_mode 3
  int lsqr_cap_pct;           // LSQR kernel: SELL capacity in % of nnz_max (env NNLS_BATCH_CAP, default 90)
  uint8_t* colview;  // scratch: per problem the column view (batched_colview_stride bytes)
  size_t cv_stride;
  double* gram;      // scratch: one packed Gram per CTA (batched_gram_scratch bytes)
  const int* guard;  // non-null: skip the whole launch when *guard != 0 (validation failed)
};
size_t batched_colview_stride(int n, int nnz_max);
size_t batched_gram_scratch(int n, int sm_count);
size_t batched_smem_bytes(int m, int n, int nnz_max);
// err: 6 ints, zeroed: [0] error bits (an out-of-order / repeated column
// inside a row sets bit 2 via the [2..5] descent counts).  The problems of
// this slice: nnz_off / rowptr / b at its first problem; its entries are
// [g_begin, g_end) of colind / vals (absolute offsets; the pipelined path
// validates chunks).
cudaError_t launch_validate_batched(int batch, int m, int n, const int64_t* nnz_off, int64_t g_begin,
                                    int64_t g_end, const int32_t* rowptr, const int32_t* colind,
                                    const double* vals, const double* b, int* err, cudaStream_t s);
cudaError_t launch_batched_nnz(const BatchArgs& a, int nnz_max, int sm_count, cudaStream_t s);
cudaError_t batched_debug_set_profile(long long* p);

}  // namespace nnls
