// api.cu -- the C ABI (include/nnls.h) and the host-side driver of the solve.
//
// The driver only orders kernels on the caller's stream and reads back one
// small status block per pivot iteration (the loop test "while (x_F, y_G) is
// infeasible"); every arithmetic step of the method runs in the sm_100a
// kernels of this directory.  There is no CPU fallback.
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <new>
#include <vector>

#include "../../include/nnls.h"
#include "common.cuh"
#include "kernels.cuh"

using namespace nnls;

namespace {

struct Buf {
  void* p = nullptr;
  size_t cap = 0;
};

cudaError_t ensure(Buf& b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.cap >= bytes) return cudaSuccess;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
  cudaError_t e = cudaMalloc(&b.p, bytes);
  if (e == cudaSuccess) b.cap = bytes;
  return e;
}

template <class T>
T* P(Buf& b) {
  return static_cast<T*>(b.p);
}

nnls_status map_cuda(cudaError_t e) {
  if (e == cudaSuccess) return NNLS_OK;
  if (e == cudaErrorMemoryAllocation) return NNLS_ERR_OOM;
  return NNLS_ERR_CUDA;
}

#define CK(expr)                                                                             \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess) {                                                                 \
      if (getenv("NNLS_DEBUG")) fprintf(stderr, "[nnls] %s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      return map_cuda(e_);                                                                   \
    }                                                                                        \
  } while (0)

int round_up(int v, int q) { return (v + q - 1) / q * q; }

// env switch: set to anything but "" or "0"
bool env_on(const char* name) {
  const char* v = getenv(name);
  return v && v[0] && !(v[0] == '0' && v[1] == 0);
}

}  // namespace

struct HostState {
  DevState st;
  int err[64];  // device err block: [0] bits, [1] longest row, [2] longest column, [4..] LSQR plan, [48..] exponents
  int plan[4];  // cluster LSQR slice maxima (rows, CSR nnz, cols, CSC nnz)
};

struct Timing {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  struct Pend {
    int phase, b, e;
  };
  std::vector<Pend> pending;
  double ms[NNLS_NPHASES] = {0};
  long long launches[NNLS_NPHASES] = {0};
};

struct nnls_handle {
  Timing tm;
  cudaStream_t stream = nullptr;
  int device = 0, sms = 148;
  nnls_params prm{};
  // problem
  int m = 0, n = 0, ldg = 0;
  int64_t nnz = 0;
  bool loaded = false, gram_ready = false;
  Buf rowptr, colind, vals, b;           // CSR + rhs
  Buf colptr, rowind, cvals, cursor, tmp_row, tmp_val, csc_temp;  // CSC (csc_temp: radix-sort scratch)
  Buf Gc;                                 // G (n x ldg) followed by c (n)
  Buf Gp;                                 // row-shard partial: packed lower G (n(n+1)/2) then c (n)
  int shard = 0;                          // 0 whole problem, 1 shard root (full A), 2 row block only
  Buf mask, x, y, xF, Fidx, Gidx;         // pivot state
  Buf inflist;                            // fused dual: the iteration's infeasible indices
  Buf pos, Fs, xs;                        // factor reuse: order positions, F sorted, x_F by index
  Buf Lt, flags;                          // Cholesky tiles + DAG flags
  Buf U, V, W, X, R, partials, xfin;      // LSQR / report
  Buf Fval, Fcol, Fcnt;                   // A restricted to the final F (cluster LSQR)
  Buf cwork;                              // condest vectors (6 n doubles) + ||M||_1 bits; fallback x
  Buf Adense;                             // tiled dense copy of A (dense Gram path)
  bool gram_dense = false;                // the last load formed G with the dense DMMA SYRK
  Buf st, err, trace;
  int trace_cap = 0;
  HostState* h = nullptr;                 // pinned readback
  bool no_cluster = false;  // force the full-grid LSQR (tests / env NNLS_NO_CLUSTER)
  bool no_graph = false;    // host-driven pivot loop (env NNLS_NO_GRAPH, or capture failed)
  bool no_reuse = false;    // F in index order, no factor reuse across iterations (env NNLS_NO_REUSE)
  bool no_fuse = false;     // separate count/exchange pass in decide (env NNLS_NO_FUSED_DUAL)
  bool no_exact_gram = false;  // always the row-ordered Gram kernel (env NNLS_NO_EXACT_GRAM)
  int claim_min_n = 2048;  // general values: the CTA-per-row claim-ordered Gram kernel from this n (env NNLS_CLAIM_MIN_N)
  bool no_sort_csc = false;    // CSC by scatter + rank instead of the radix sort (env NNLS_NO_SORT_CSC)
  cudaGraphExec_t gexec = nullptr;
  std::vector<double> gkey;
  cudaStream_t gstream = nullptr;
  cudaEvent_t gev[2] = {nullptr, nullptr};
  // batched
  bool batched = false;
  int batch = 0;
  Buf b_nnz_off, b_info_i, b_info_d, b_x, b_mask, b_colview, b_gram;
  std::vector<int64_t> b_hoff;            // host copy of nnz_off
  cudaStream_t s_in = nullptr, s_out = nullptr;  // pipelined batched: copy streams
  std::vector<cudaEvent_t> pev;           // pipelined batched: per-chunk events
};

namespace {

int tm_event(nnls_handle* h) {
  Timing& t = h->tm;
  if (t.used == t.pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    t.pool.push_back(e);
  }
  return (int)t.used++;
}
int tm_begin(nnls_handle* h) {
  if (!h->tm.on) return -1;
  const int i = tm_event(h);
  if (i >= 0) cudaEventRecord(h->tm.pool[i], h->stream);
  return i;
}
void tm_end(nnls_handle* h, int phase, int ib, int nlaunch) {
  h->tm.launches[phase] += nlaunch;
  if (ib < 0) return;
  const int ie = tm_event(h);
  if (ie < 0) return;
  cudaEventRecord(h->tm.pool[ie], h->stream);
  h->tm.pending.push_back({phase, ib, ie});
}
// resolve recorded pairs (after a stream sync) to free the event pool
void tm_flush(nnls_handle* h) {
  Timing& t = h->tm;
  if (t.pending.empty()) {
    t.used = 0;
    return;
  }
  cudaStreamSynchronize(h->stream);
  for (const auto& p : t.pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, t.pool[p.b], t.pool[p.e]) == cudaSuccess) t.ms[p.phase] += ms;
  }
  t.pending.clear();
  t.used = 0;
}

#define TIMED(phase, nl, expr)            \
  do {                                    \
    const int ib_ = tm_begin(h);          \
    CK(expr);                             \
    tm_end(h, (phase), ib_, (nl));        \
  } while (0)

nnls_status set_stream_device(nnls_handle* h, void* stream) {
  h->stream = static_cast<cudaStream_t>(stream);
  int dev = 0;
  CK(cudaGetDevice(&dev));
  h->device = dev;
  CK(cudaDeviceGetAttribute(&h->sms, cudaDevAttrMultiProcessorCount, dev));
  int major = 0;
  CK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major < 10) return NNLS_ERR_CUDA;  // sm_100a code only
  return NNLS_OK;
}

nnls_status check_params(const nnls_params* p) {
  if (!(p->zero_tol >= 0.0) || p->p_max < 0 || p->max_iter < 0 || p->lsqr_mode < 0 ||
      p->lsqr_mode > 3 || !(p->adaptive_threshold >= 0.0))
    return NNLS_ERR_INVALID_ARG;
  return NNLS_OK;
}

nnls_status map_err_bits(int e) {
  if (e & 1) return NNLS_ERR_DIMENSION;
  if (e & 2) return NNLS_ERR_INDEX;
  if (e & 4) return NNLS_ERR_NONFINITE;
  return NNLS_OK;
}

// upload + validate + CSC + Gram over rows [r0, r1)
// shard: 0 whole problem (full Gram); 1 shard root (full A kept for the
// loop and LSQR, packed partial Gram over rows [r0, r1)); 2 a row block only
// (packed partial Gram over all its rows; m < n allowed; cannot solve)
nnls_status load_impl(nnls_handle* h, int32_t m, int32_t n, int64_t nnz, const int32_t* rowptr,
                      const int32_t* colind, const double* vals, const double* b, int r0, int r1,
                      int shard = 0) {
  if (!h || m < 1 || n < 1 || (m < n && shard != 2) || nnz < 0 || !rowptr || !b) return NNLS_ERR_INVALID_ARG;
  if (nnz > 0 && (!colind || !vals)) return NNLS_ERR_INVALID_ARG;
  if (nnz > 0x7fffffffLL) return NNLS_ERR_INVALID_ARG;
  if ((int64_t)n * 8 > 200 * 1024) return NNLS_ERR_INVALID_ARG;  // Gram row accumulator in smem
  if (r0 < 0 || r1 > m || r0 > r1) return NNLS_ERR_INVALID_ARG;
  cudaStream_t s = h->stream;
  h->m = m;
  h->n = n;
  h->nnz = nnz;
  h->ldg = round_up(n, 4);
  h->gram_ready = false;
  h->loaded = false;
  h->shard = shard;
  CK(ensure(h->rowptr, sizeof(int32_t) * (size_t)(m + 1)));
  CK(ensure(h->colind, sizeof(int32_t) * (size_t)nnz));
  CK(ensure(h->vals, sizeof(double) * (size_t)nnz));
  CK(ensure(h->b, sizeof(double) * (size_t)m));
  CK(ensure(h->colptr, sizeof(int32_t) * (size_t)(n + 1)));
  CK(ensure(h->cursor, sizeof(int32_t) * (size_t)(n + 1)));
  CK(ensure(h->rowind, sizeof(int32_t) * (size_t)nnz));
  CK(ensure(h->cvals, sizeof(double) * (size_t)nnz));
  CK(ensure(h->tmp_row, sizeof(int32_t) * (size_t)nnz));
  CK(ensure(h->tmp_val, sizeof(double) * (size_t)nnz));
  // (the radix sort's fixed cost of several passes loses to scatter + rank
  // below ~1M entries: config 1, 100K entries, 39 -> 62 us)
  const size_t csc_tb = (h->no_sort_csc || nnz < (1 << 20)) ? 0 : csc_sort_temp_bytes(nnz, n);
  if (csc_tb > 0) CK(ensure(h->csc_temp, csc_tb));
  CK(ensure(h->Gc, sizeof(double) * ((size_t)n * h->ldg + n)));
  CK(ensure(h->mask, (size_t)n));
  CK(ensure(h->x, sizeof(double) * (size_t)n));
  CK(ensure(h->y, sizeof(double) * (size_t)n));
  CK(ensure(h->xF, sizeof(double) * (size_t)(n + kTile)));
  CK(ensure(h->Fidx, sizeof(int32_t) * (size_t)n));
  CK(ensure(h->Gidx, sizeof(int32_t) * (size_t)n));
  CK(ensure(h->inflist, sizeof(int32_t) * (size_t)n));
  CK(ensure(h->pos, sizeof(int32_t) * (size_t)n));
  CK(ensure(h->Fs, sizeof(int32_t) * (size_t)n));
  CK(ensure(h->xs, sizeof(double) * (size_t)n));
  const size_t nflags = chol_flag_count(n);
  if (h->flags.cap < sizeof(int) * nflags) {
    CK(ensure(h->flags, sizeof(int) * nflags));
    CK(cudaMemsetAsync(h->flags.p, 0, h->flags.cap, s));
    // a fresh flag array must not alias a reused epoch: reset the epoch too
    CK(ensure(h->st, sizeof(DevState)));
    CK(cudaMemsetAsync(h->st.p, 0, sizeof(DevState), s));
  }
  CK(ensure(h->Lt, sizeof(double) * chol_tile_doubles(n)));
  CK(ensure(h->U, sizeof(double) * (size_t)m));
  CK(ensure(h->R, sizeof(double) * (size_t)m));
  CK(ensure(h->Fval, sizeof(double) * (size_t)(nnz > 0 ? nnz : 1)));
  CK(ensure(h->Fcol, sizeof(int32_t) * (size_t)(nnz > 0 ? nnz : 1)));
  CK(ensure(h->Fcnt, sizeof(int32_t) * (size_t)m));
  CK(ensure(h->V, sizeof(double) * (size_t)n));
  CK(ensure(h->W, sizeof(double) * (size_t)n));
  CK(ensure(h->X, sizeof(double) * (size_t)n));
  CK(ensure(h->xfin, sizeof(double) * (size_t)n));
  CK(ensure(h->cwork, sizeof(double) * (7 * (size_t)n + 1)));
  CK(ensure(h->partials, sizeof(double) * 8 * (size_t)(h->sms * 4)));
  CK(ensure(h->st, sizeof(DevState)));
  CK(ensure(h->err, sizeof(int) * 64));  // [0..3] error bits / longest row, column; [4..] LSQR plan
  const int cap = h->prm.trace ? (h->prm.max_iter > 0 ? h->prm.max_iter : 10 * n) + 1 : 0;
  h->trace_cap = cap;
  if (cap > 0) CK(ensure(h->trace, sizeof(TraceRec) * (size_t)cap));

  int ib = tm_begin(h);
  // device-resident inputs: one copy kernel; otherwise (host memory) the copy engines
  bool all_dev = true;
  for (const void* ptr : {(const void*)rowptr, (const void*)colind, (const void*)vals, (const void*)b}) {
    cudaPointerAttributes pa;
    if (ptr == nullptr) continue;
    if (cudaPointerGetAttributes(&pa, ptr) != cudaSuccess || pa.type != cudaMemoryTypeDevice) all_dev = false;
    cudaGetLastError();
  }
  if (all_dev) {
    const void* src[4] = {rowptr, colind, vals, b};
    void* dst[4] = {h->rowptr.p, h->colind.p, h->vals.p, h->b.p};
    const size_t by[4] = {sizeof(int32_t) * (size_t)(m + 1), nnz > 0 ? sizeof(int32_t) * (size_t)nnz : 0,
                          nnz > 0 ? sizeof(double) * (size_t)nnz : 0, sizeof(double) * (size_t)m};
    CK(launch_upload_copy(src, dst, by, h->sms, s));
  } else {
    CK(cudaMemcpyAsync(h->rowptr.p, rowptr, sizeof(int32_t) * (size_t)(m + 1), cudaMemcpyDefault, s));
    if (nnz > 0) {
      CK(cudaMemcpyAsync(h->colind.p, colind, sizeof(int32_t) * (size_t)nnz, cudaMemcpyDefault, s));
      CK(cudaMemcpyAsync(h->vals.p, vals, sizeof(double) * (size_t)nnz, cudaMemcpyDefault, s));
    }
    CK(cudaMemcpyAsync(h->b.p, b, sizeof(double) * (size_t)m, cudaMemcpyDefault, s));
  }
  CK(cudaMemsetAsync(h->err.p, 0, sizeof(int) * 64, s));
  tm_end(h, NNLS_PH_UPLOAD, ib, 0);
  TIMED(NNLS_PH_VALIDATE, 1,
        launch_validate(m, n, nnz, P<int32_t>(h->rowptr), P<int32_t>(h->colind), P<double>(h->vals),
                        P<double>(h->b), P<int>(h->err), s));
  // column counts (guarded against invalid indices) and the cluster-LSQR
  // slice plan are computed before the validation readback, so ONE host sync
  // returns the error bits, the longest row/column and the plan together
  TIMED(NNLS_PH_CSC, nnz > 0 ? 2 : 1,
        launch_csc_count(m, n, nnz, P<int32_t>(h->colind), P<int32_t>(h->colptr),
                         P<int32_t>(h->cursor), s, P<int>(h->err) + 2));
  // (the cluster LSQR keeps replicas of u and v in every CTA's shared memory:
  // no plan when those alone exceed it)
  const bool cl_possible = 8 * ((size_t)m + n) < 220 * 1024;
  if (cl_possible)
    CK(launch_lsqr_plan(m, n, P<int32_t>(h->rowptr), P<int32_t>(h->colptr), P<int>(h->err) + 4, s));
  tm_end(h, NNLS_PH_CSC, -1, 1);
  CK(cudaMemcpyAsync(h->h->err, h->err.p, sizeof(int) * 64, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const int herr = h->h->err[0];
  if (herr) return map_err_bits(herr);
  memcpy(h->h->plan, h->h->err + 4, sizeof(h->h->plan));  // cluster LSQR slice maxima
  if (!cl_possible) {  // maxima that no cluster holds: the grid LSQR runs
    h->h->plan[0] = m;
    h->h->plan[1] = (int)(nnz < INT32_MAX ? nnz : INT32_MAX);
    h->h->plan[2] = n;
    h->h->plan[3] = h->h->plan[1];
  }
  if (csc_tb > 0) {
    TIMED(NNLS_PH_CSC, 3,
          launch_csc_fill_sorted(m, n, nnz, P<int32_t>(h->rowptr), P<int32_t>(h->colind), P<double>(h->vals),
                                 P<int32_t>(h->rowind), P<double>(h->cvals), P<int32_t>(h->tmp_row),
                                 P<double>(h->tmp_val), h->csc_temp.p, h->csc_temp.cap, s));
  } else {
    TIMED(NNLS_PH_CSC, 2,
          launch_csc_fill(m, n, P<int32_t>(h->rowptr), P<int32_t>(h->colind), P<double>(h->vals),
                          P<int32_t>(h->colptr), P<int32_t>(h->rowind), P<double>(h->cvals),
                          P<int32_t>(h->cursor), P<int32_t>(h->tmp_row), P<double>(h->tmp_val), s,
                          h->h->err[2]));
  }
  double* G = P<double>(h->Gc);
  double* c = G + (size_t)n * h->ldg;
  int ldg = h->ldg;
  if (shard != 0) {  // packed partial [P | c]: what the ranks reduce (half the bytes of the square)
    CK(ensure(h->Gp, sizeof(double) * ((size_t)n * (n + 1) / 2 + n)));
    G = P<double>(h->Gp);
    c = G + (size_t)n * (n + 1) / 2;
    ldg = 0;
  }
  const bool exact = gram_is_exact(h->h->err) && !h->no_exact_gram;
  const bool a_exact = gram_A_exact(h->h->err) && !h->no_exact_gram;
  // dense A (NEXT-1, the Fig. 2 density-1 workloads): the Gram is an O(m n^2)
  // SYRK -> DMMA on a tiled dense copy; exact inputs only (bitwise = oracle)
  const double density = (double)nnz / ((double)m * (double)n);
  const size_t dense_bytes = sizeof(double) * gram_dense_doubles(r1 - r0, n);
  if (a_exact && density >= 0.25 && n >= 32 && dense_bytes <= ((size_t)16 << 30) && !env_on("NNLS_NO_DENSE_GRAM")) {
    CK(ensure(h->Adense, dense_bytes));
    TIMED(NNLS_PH_GRAM, 4,
          launch_gram_dense(n, P<int32_t>(h->rowptr), P<int32_t>(h->colind), P<double>(h->vals),
                            P<int32_t>(h->colptr), P<int32_t>(h->rowind), P<double>(h->cvals), P<double>(h->b), r0,
                            r1, P<double>(h->Adense), G, ldg, c, h->sms, s, gram_c_exact(h->h->err)));
    h->gram_dense = true;
  } else {
    TIMED(NNLS_PH_GRAM, 1,
          launch_gram(m, n, P<int32_t>(h->rowptr), P<int32_t>(h->colind), P<double>(h->vals),
                      P<int32_t>(h->colptr), P<int32_t>(h->rowind), P<double>(h->cvals),
                      P<double>(h->b), r0, r1, G, ldg, c, h->sms, s, exact, gram_exact_lmin(h->h->err),
                      n >= h->claim_min_n ? h->h->err[1] : 0, h->h->err[2]));
    h->gram_dense = false;
  }
  h->loaded = true;
  return NNLS_OK;
}

nnls_status create_impl(nnls_handle** out, const nnls_params* p, void* stream) {
  if (!out) return NNLS_ERR_INVALID_ARG;
  *out = nullptr;
  nnls_handle* h = new (std::nothrow) nnls_handle();
  if (!h) return NNLS_ERR_OOM;
  nnls_params_default(&h->prm);
  if (p) {
    nnls_status ps = check_params(p);
    if (ps != NNLS_OK) {
      delete h;
      return ps;
    }
    h->prm = *p;
  }
  nnls_status s = set_stream_device(h, stream);
  if (s == NNLS_OK && cudaMallocHost(&h->h, sizeof(HostState)) != cudaSuccess) s = NNLS_ERR_OOM;
  if (s != NNLS_OK) {
    if (h->h) cudaFreeHost(h->h);
    delete h;
    return s;
  }
  memset(h->h, 0, sizeof(HostState));
  h->no_cluster = env_on("NNLS_NO_CLUSTER");
  h->no_graph = env_on("NNLS_NO_GRAPH");
  h->no_reuse = env_on("NNLS_NO_REUSE");
  h->no_fuse = env_on("NNLS_NO_FUSED_DUAL");
  h->no_exact_gram = env_on("NNLS_NO_EXACT_GRAM");
  if (const char* v = getenv("NNLS_CLAIM_MIN_N")) h->claim_min_n = atoi(v);
  h->no_sort_csc = env_on("NNLS_NO_SORT_CSC");
  *out = h;
  return NNLS_OK;
}

void free_buf(Buf& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
}

nnls_status read_state(nnls_handle* h) {
  CK(cudaMemcpyAsync(&h->h->st, h->st.p, sizeof(DevState), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (h->tm.pending.size() > 256) tm_flush(h);
  return NNLS_OK;
}


}  // namespace

extern "C" {

const char* nnls_status_string(nnls_status s) {
  switch (s) {
    case NNLS_OK: return "ok";
    case NNLS_ERR_INVALID_ARG: return "invalid argument";
    case NNLS_ERR_DIMENSION: return "CSR dimension error";
    case NNLS_ERR_INDEX: return "CSR column index error";
    case NNLS_ERR_NONFINITE: return "non-finite value";
    case NNLS_ERR_CUDA: return "CUDA error";
    case NNLS_ERR_OOM: return "out of device memory";
    case NNLS_ERR_NOT_PD: return "Cholesky pivot not positive (A_F rank deficient or kappa^2 eps >= 1)";
    case NNLS_ITERATION_LIMIT: return "iteration limit";
    case NNLS_ERR_STATE: return "call out of order";
  }
  return "unknown";
}

nnls_status nnls_params_default(nnls_params* p) {
  if (!p) return NNLS_ERR_INVALID_ARG;
  memset(p, 0, sizeof(*p));
  p->zero_tol = 1e-12;
  p->p_max = 3;
  p->max_iter = 0;
  p->lsqr_mode = 1;
  p->lsqr_itn_limit = 0;
  p->lsqr_atol = 1e-15;
  p->lsqr_btol = 1e-15;
  p->lsqr_conlim = 1e8;
  p->trace = 0;
  p->kkt = 1;
  p->adaptive_threshold = 1e-8;
  p->notpd_fallback = 0;
  return NNLS_OK;
}

nnls_status nnls_device_info(int32_t* sm_count, int32_t* cc, int32_t* device) {
  int dev = 0, ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return NNLS_ERR_CUDA;
  CK(cudaGetDevice(&dev));
  int sms = 0, ma = 0, mi = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&ma, cudaDevAttrComputeCapabilityMajor, dev));
  CK(cudaDeviceGetAttribute(&mi, cudaDevAttrComputeCapabilityMinor, dev));
  if (sm_count) *sm_count = sms;
  if (cc) *cc = ma * 10 + mi;
  if (device) *device = dev;
  return NNLS_OK;
}

nnls_status nnls_create(nnls_handle** h, const nnls_params* p, void* cuda_stream) {
  return create_impl(h, p, cuda_stream);
}

nnls_status nnls_load(nnls_handle* h, int32_t m, int32_t n, int64_t nnz, const int32_t* rowptr,
                      const int32_t* colind, const double* vals, const double* b) {
  if (!h || h->batched) return NNLS_ERR_INVALID_ARG;
  nnls_status s = load_impl(h, m, n, nnz, rowptr, colind, vals, b, 0, m);
  if (s == NNLS_OK) h->gram_ready = true;
  return s;
}

nnls_status nnls_setup(nnls_handle** h, int32_t m, int32_t n, int64_t nnz, const int32_t* rowptr,
                       const int32_t* colind, const double* vals, const double* b,
                       const nnls_params* p, void* cuda_stream) {
  nnls_status s = create_impl(h, p, cuda_stream);
  if (s != NNLS_OK) return s;
  s = nnls_load(*h, m, n, nnz, rowptr, colind, vals, b);
  if (s != NNLS_OK) {
    nnls_destroy(*h);
    *h = nullptr;
  }
  return s;
}

nnls_status nnls_setup_shard(nnls_handle** h, int32_t m, int32_t n, int64_t nnz,
                             const int32_t* rowptr, const int32_t* colind, const double* vals,
                             const double* b, int32_t row_begin, int32_t row_end,
                             const nnls_params* p, void* cuda_stream) {
  nnls_status s = create_impl(h, p, cuda_stream);
  if (s != NNLS_OK) return s;
  s = load_impl(*h, m, n, nnz, rowptr, colind, vals, b, row_begin, row_end, 1);
  if (s != NNLS_OK) {
    nnls_destroy(*h);
    *h = nullptr;
  }
  return s;
}

nnls_status nnls_load_shard(nnls_handle* h, int32_t m, int32_t n, int64_t nnz, const int32_t* rowptr,
                            const int32_t* colind, const double* vals, const double* b,
                            int32_t row_begin, int32_t row_end) {
  if (!h || h->batched) return NNLS_ERR_INVALID_ARG;
  return load_impl(h, m, n, nnz, rowptr, colind, vals, b, row_begin, row_end, 1);
}

nnls_status nnls_load_block(nnls_handle* h, int32_t m_block, int32_t n, int64_t nnz, const int32_t* rowptr,
                            const int32_t* colind, const double* vals, const double* b) {
  if (!h || h->batched) return NNLS_ERR_INVALID_ARG;
  return load_impl(h, m_block, n, nnz, rowptr, colind, vals, b, 0, m_block, 2);
}

nnls_status nnls_gram_buffer(nnls_handle* h, double** dev_ptr, size_t* count) {
  if (!h || !h->loaded || h->batched || h->shard == 0) return NNLS_ERR_STATE;
  if (dev_ptr) *dev_ptr = P<double>(h->Gp);
  if (count) *count = (size_t)h->n * (h->n + 1) / 2 + h->n;
  return NNLS_OK;
}

nnls_status nnls_gram_finalize(nnls_handle* h) {
  if (!h || !h->loaded || h->batched || h->shard != 1) return NNLS_ERR_STATE;
  const int n = h->n;
  const double* Pk = P<double>(h->Gp);
  double* G = P<double>(h->Gc);
  int ib = tm_begin(h);
  CK(launch_gram_unpack(n, Pk, G, h->ldg, h->sms, h->stream));
  CK(cudaMemcpyAsync(G + (size_t)n * h->ldg, Pk + (size_t)n * (n + 1) / 2, sizeof(double) * (size_t)n,
                     cudaMemcpyDeviceToDevice, h->stream));
  tm_end(h, NNLS_PH_GRAM, ib, 1);
  h->gram_ready = true;
  return NNLS_OK;
}

nnls_status nnls_set_params(nnls_handle* h, const nnls_params* p) {
  if (!h || !p) return NNLS_ERR_INVALID_ARG;
  nnls_status s = check_params(p);
  if (s != NNLS_OK) return s;
  h->prm = *p;
  if (h->loaded && !h->batched) {
    const int cap = p->trace ? (p->max_iter > 0 ? p->max_iter : 10 * h->n) + 1 : 0;
    h->trace_cap = cap;
    if (cap > 0) CK(ensure(h->trace, sizeof(TraceRec) * (size_t)cap));
  }
  return NNLS_OK;
}

}  // extern "C"

namespace {
LsqrArgs lsqr_args(nnls_handle* h) {
  const int n = h->n;
  const nnls_params& p = h->prm;
  double* G = P<double>(h->Gc);
  LsqrArgs a{};
  a.m = h->m;
  a.n = n;
  a.rowptr = P<int32_t>(h->rowptr);
  a.colind = P<int32_t>(h->colind);
  a.vals = P<double>(h->vals);
  a.colptr = P<int32_t>(h->colptr);
  a.rowind = P<int32_t>(h->rowind);
  a.cvals = P<double>(h->cvals);
  a.b = P<double>(h->b);
  a.mask = P<uint8_t>(h->mask);
  a.x_ne = P<double>(h->x);
  a.x_out = P<double>(h->xfin);
  a.U = P<double>(h->U);
  a.V = P<double>(h->V);
  a.W = P<double>(h->W);
  a.X = P<double>(h->X);
  a.R = P<double>(h->R);
  a.partials = P<double>(h->partials);
  a.st = P<DevState>(h->st);
  a.mode = p.lsqr_mode;
  a.itn_limit = p.lsqr_itn_limit;
  a.atol = p.lsqr_atol;
  a.btol = p.lsqr_btol;
  a.conlim = p.lsqr_conlim;
  a.tol = p.zero_tol;
  a.kkt = p.kkt;
  a.G = G;
  a.ldg = h->ldg;
  a.c = G + (size_t)n * h->ldg;
  a.Fval = P<double>(h->Fval);
  a.Fcol = P<int32_t>(h->Fcol);
  a.Fcnt = P<int32_t>(h->Fcnt);
  a.Fidx = h->no_reuse ? P<int32_t>(h->Fidx) : P<int32_t>(h->Fs);  // F (index order when reusing)
  a.Gidx = P<int32_t>(h->Gidx);  // G in index order (decide)
  a.plan = P<int>(h->err) + 4;
  return a;
}

// cluster-resident LSQR when A's slices fit in one 16-CTA cluster's shared
// memory (configs 0, 1, 3); the full-grid cooperative kernel otherwise
cudaError_t launch_lsqr_args(nnls_handle* h, const LsqrArgs& a, cudaStream_t s);
double* xs_or_null(nnls_handle* h);
// NOT_PD fallback (notpd_fallback): x_F of the failed iteration from
// a cold LSQR on A_F (no report), then the pivot loop continues; the next
// factorization starts from scratch (the failed factor's prefix is not reused)
cudaError_t launch_fallback(nnls_handle* h, cudaStream_t s) {
  DevState* st = P<DevState>(h->st);
  double* xl = P<double>(h->cwork);
  cudaError_t e = launch_fallback_prep(st, s);
  if (e != cudaSuccess) return e;
  LsqrArgs a = lsqr_args(h);
  a.mode = 1;
  a.kkt = 0;
  a.x_out = xl;
  e = launch_lsqr_args(h, a, s);
  if (e != cudaSuccess) return e;
  e = launch_fallback_fixup(h->n, P<int32_t>(h->Fidx), xl, P<double>(h->xF), xs_or_null(h), st, s);
  return e;
}
// the final step: (mode 3) the condition estimate, then LSQR + report
cudaError_t launch_condest_h(nnls_handle* h, cudaStream_t s) {
  const int n = h->n;
  double* w = P<double>(h->cwork);
  return launch_condest(P<double>(h->Gc), h->ldg, P<int32_t>(h->Fidx), P<double>(h->Lt), n, P<DevState>(h->st),
                        w, reinterpret_cast<unsigned long long*>(w + 7 * (size_t)n), h->prm.adaptive_threshold,
                        h->sms, s);
}
cudaError_t launch_lsqr(nnls_handle* h, cudaStream_t s) {
  if (h->prm.lsqr_mode == 3) {
    cudaError_t ec = launch_condest_h(h, s);
    if (ec != cudaSuccess) return ec;
  }
  return launch_lsqr_args(h, lsqr_args(h), s);
}
cudaError_t launch_lsqr_args(nnls_handle* h, const LsqrArgs& a, cudaStream_t s) {
  cudaError_t e = launch_lsqr_compact(a, h->sms, s);  // A restricted to F (both paths)
  if (e != cudaSuccess) return e;
  e = h->no_cluster ? cudaErrorNotSupported : launch_lsqr_cluster_planned(a, h->h->plan, s);
  if (e == cudaErrorNotSupported) {
    cudaGetLastError();
    e = launch_lsqr_final(a, h->sms, s);
  }
  return e;
}

}  // namespace
bool nnls::pdl_enabled() {
  static const bool on = !env_on("NNLS_NO_PDL");
  return on;
}
namespace {
int32_t* pos_or_null(nnls_handle* h) { return h->no_reuse ? nullptr : P<int32_t>(h->pos); }
int32_t* fs_or_null(nnls_handle* h) { return h->no_reuse ? nullptr : P<int32_t>(h->Fs); }
double* xs_or_null(nnls_handle* h) { return h->no_reuse ? nullptr : P<double>(h->xs); }
int32_t* inflist_or_null(nnls_handle* h) { return h->no_fuse ? nullptr : P<int32_t>(h->inflist); }

// one pivot iteration: decide -> (gather + Cholesky + forward) -> back solve -> dual
cudaError_t launch_iteration(nnls_handle* h, cudaStream_t s, const cudaGraphConditionalHandle* loop) {
  const int n = h->n;
  double* G = P<double>(h->Gc);
  double* c = G + (size_t)n * h->ldg;
  DevState* st = P<DevState>(h->st);
  TraceRec* trace = h->trace_cap > 0 ? P<TraceRec>(h->trace) : nullptr;
  cudaError_t e = launch_decide(n, P<uint8_t>(h->mask), P<double>(h->x), P<double>(h->y),
                                P<int32_t>(h->Fidx), P<int32_t>(h->Gidx), st, trace, h->trace_cap, s, loop,
                                pos_or_null(h), fs_or_null(h), xs_or_null(h));
  if (e == cudaSuccess)
    e = launch_chol_factor(n, G, h->ldg, c, P<int32_t>(h->Fidx), P<double>(h->Lt), P<int>(h->flags), st,
                           h->sms, s);
  if (e == cudaSuccess)
    e = launch_chol_backsolve(n, P<double>(h->Lt), P<int>(h->flags), P<double>(h->xF), st, h->sms, s,
                              P<int32_t>(h->Fidx), xs_or_null(h));
  if (e == cudaSuccess)
    e = launch_dual(n, G, h->ldg, c, P<int32_t>(h->Fidx), P<int32_t>(h->Gidx), P<double>(h->xF),
                    P<uint8_t>(h->mask), P<double>(h->x), P<double>(h->y), h->prm.zero_tol, st, h->sms, s,
                    fs_or_null(h), xs_or_null(h), inflist_or_null(h));
  return e;
}

// Everything a captured solve graph depends on.
std::vector<double> graph_key(nnls_handle* h) {
  const nnls_params& p = h->prm;
  std::vector<double> k = {(double)h->m, (double)h->n, (double)h->nnz, (double)h->ldg,
                           (double)h->h->plan[0], (double)h->h->plan[1], (double)h->h->plan[2],
                           (double)h->h->plan[3], p.zero_tol, (double)p.p_max, (double)p.max_iter,
                           (double)p.lsqr_mode, (double)p.lsqr_itn_limit, p.lsqr_atol, p.lsqr_btol,
                           p.lsqr_conlim, (double)p.kkt, (double)h->trace_cap, (double)h->no_cluster,
                           (double)h->no_reuse, (double)h->no_fuse, p.adaptive_threshold, (double)p.notpd_fallback};
  const Buf* bufs[] = {&h->rowptr, &h->colind, &h->vals, &h->b, &h->colptr, &h->rowind, &h->cvals,
                       &h->Gc, &h->mask, &h->x, &h->y, &h->xF, &h->Fidx, &h->Gidx, &h->inflist, &h->pos, &h->Fs, &h->xs, &h->Lt, &h->flags,
                       &h->U, &h->V, &h->W, &h->X, &h->R, &h->partials, &h->xfin, &h->st, &h->trace,
                       &h->Fval, &h->Fcol, &h->Fcnt, &h->cwork};
  for (const Buf* b : bufs) k.push_back((double)(uintptr_t)b->p);
  return k;
}

void drop_graph(nnls_handle* h) {
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  h->gexec = nullptr;
  h->gkey.clear();
}

// Device-resident solve: init -> WHILE(decide clears the condition) { one
// pivot iteration } -> LSQR, captured once per problem shape / buffer set and
// replayed with one graph launch (no host round trip per pivot iteration).
#define GDBG(msg)                                                                         \
  do {                                                                                    \
    if (env_on("NNLS_DEBUG")) fprintf(stderr, "[nnls graph] %s: %s\n", msg, cudaGetErrorString(e)); \
  } while (0)
cudaError_t build_graph(nnls_handle* h, cudaStream_t s) {
  drop_graph(h);
  const int n = h->n;
  const nnls_params& p = h->prm;
  const int max_iter = p.max_iter > 0 ? p.max_iter : 10 * n;
  double* G = P<double>(h->Gc);
  double* c = G + (size_t)n * h->ldg;
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaGraphCreate(&g, 0);
  if (e != cudaSuccess) return e;
  cudaGraphConditionalHandle cond;
  cudaGraphNode_t init_node = nullptr, cond_node = nullptr;
  e = cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault);
  GDBG("handle");
  if (env_on("NNLS_DEBUG")) {
    fprintf(stderr, "[nnls graph] stream %p graph %p query %d\n", (void*)s, (void*)g, (int)cudaStreamQuery(s));
    fflush(stderr);
  }
  if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  GDBG("begin1");
  if (e == cudaSuccess) {
    cudaError_t el = launch_init(n, c, P<uint8_t>(h->mask), P<double>(h->x), P<double>(h->y), p.zero_tol,
                                 P<DevState>(h->st), p.p_max, max_iter, s, pos_or_null(h));
    cudaGraph_t gg = g;
    e = cudaStreamEndCapture(s, &gg);
    if (e == cudaSuccess) e = el;
  }
  GDBG("init");
  if (e == cudaSuccess) {
    size_t nn = 0;
    e = cudaGraphGetRootNodes(g, nullptr, &nn);
    if (e == cudaSuccess && nn != 1) e = cudaErrorNotSupported;
    if (e == cudaSuccess) e = cudaGraphGetRootNodes(g, &init_node, &nn);
  }
  GDBG("roots");
  cudaGraph_t body = nullptr;
  if (e == cudaSuccess) {
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    e = cudaGraphAddNode(&cond_node, g, &init_node, 1, &cp);
    if (e == cudaSuccess) body = cp.conditional.phGraph_out[0];
  }
  GDBG("cond");
  if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  if (e == cudaSuccess) {
    cudaError_t el = launch_iteration(h, s, &cond);
    cudaGraph_t bb = body;
    e = cudaStreamEndCapture(s, &bb);
    if (e == cudaSuccess) e = el;
  }
  GDBG("body");
  if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(s, g, &cond_node, nullptr, 1, cudaStreamCaptureModeRelaxed);
  if (e == cudaSuccess) {
    cudaError_t el = launch_lsqr(h, s);
    cudaGraph_t gg = g;
    e = cudaStreamEndCapture(s, &gg);
    if (e == cudaSuccess) e = el;
  }
  GDBG("lsqr");
  if (e == cudaSuccess) e = cudaGraphInstantiate(&h->gexec, g, 0);
  GDBG("instantiate");
  cudaGraphDestroy(g);
  if (e != cudaSuccess) {
    cudaGetLastError();
    h->gexec = nullptr;
    return e;
  }
  h->gkey = graph_key(h);
  return cudaSuccess;
}
}  // namespace

extern "C" {

nnls_status nnls_solve(nnls_handle* h, double* x_out, nnls_info* info) {
  if (!h || h->batched) return NNLS_ERR_INVALID_ARG;
  if (!h->loaded || !h->gram_ready) return NNLS_ERR_STATE;
  cudaStream_t s = h->stream;
  const int n = h->n;
  const nnls_params& p = h->prm;
  const int max_iter = p.max_iter > 0 ? p.max_iter : 10 * n;
  double* G = P<double>(h->Gc);
  double* c = G + (size_t)n * h->ldg;
  DevState* st = P<DevState>(h->st);
  bool done_graph = false;
  if (!h->tm.on && !h->no_graph && !p.notpd_fallback) {
    // device-resident loop (one graph launch); per-phase timing uses the host
    // loop, and so does the NOT_PD fallback (it needs the host between steps)
    // graphs are captured and launched on a private stream fenced to the
    // caller's stream with events (capture is not allowed on the legacy stream)
    if (!h->gstream) {
      if (cudaStreamCreateWithFlags(&h->gstream, cudaStreamNonBlocking) != cudaSuccess ||
          cudaEventCreateWithFlags(&h->gev[0], cudaEventDisableTiming) != cudaSuccess ||
          cudaEventCreateWithFlags(&h->gev[1], cudaEventDisableTiming) != cudaSuccess)
        h->no_graph = true;
    }
    if (!h->no_graph && (!h->gexec || h->gkey != graph_key(h))) {
      CK(cudaStreamSynchronize(s));
      if (build_graph(h, h->gstream) != cudaSuccess) h->no_graph = true;  // fall back for this handle
    }
    if (!h->no_graph && h->gexec) {
      CK(cudaEventRecord(h->gev[0], s));
      CK(cudaStreamWaitEvent(h->gstream, h->gev[0], 0));
      CK(cudaGraphLaunch(h->gexec, h->gstream));
      CK(cudaEventRecord(h->gev[1], h->gstream));
      CK(cudaStreamWaitEvent(s, h->gev[1], 0));
      h->tm.launches[NNLS_PH_INIT] += 1;
      done_graph = true;
    }
  }
  if (!done_graph) {
    TIMED(NNLS_PH_INIT, 1,
          launch_init(n, c, P<uint8_t>(h->mask), P<double>(h->x), P<double>(h->y), p.zero_tol, st,
                      p.p_max, max_iter, s, pos_or_null(h)));
    TraceRec* trace = h->trace_cap > 0 ? P<TraceRec>(h->trace) : nullptr;
    for (;;) {
      TIMED(NNLS_PH_DECIDE, 1,
            launch_decide(n, P<uint8_t>(h->mask), P<double>(h->x), P<double>(h->y),
                          P<int32_t>(h->Fidx), P<int32_t>(h->Gidx), st, trace, h->trace_cap, s, nullptr,
                          pos_or_null(h), fs_or_null(h), xs_or_null(h)));
      nnls_status rs = read_state(h);
      if (rs != NNLS_OK) return rs;
      const DevState& hs = h->h->st;
      if (hs.done || hs.status != 0) break;
      if (hs.f > 0) {
        TIMED(NNLS_PH_CHOL_FACTOR, 1,
              launch_chol_factor(n, G, h->ldg, c, P<int32_t>(h->Fidx), P<double>(h->Lt),
                                 P<int>(h->flags), st, h->sms, s));
        TIMED(NNLS_PH_CHOL_SOLVE, 1,
              launch_chol_backsolve(n, P<double>(h->Lt), P<int>(h->flags), P<double>(h->xF), st,
                                    h->sms, s, P<int32_t>(h->Fidx), xs_or_null(h)));
        if (p.notpd_fallback) {
          nnls_status rs2 = read_state(h);
          if (rs2 != NNLS_OK) return rs2;
          if (h->h->st.status == 7) TIMED(NNLS_PH_LSQR, 2, launch_fallback(h, s));
        }
      }
      TIMED(NNLS_PH_DUAL, 1,
            launch_dual(n, G, h->ldg, c, P<int32_t>(h->Fidx), P<int32_t>(h->Gidx), P<double>(h->xF),
                        P<uint8_t>(h->mask), P<double>(h->x), P<double>(h->y), p.zero_tol, st,
                        h->sms, s, fs_or_null(h), xs_or_null(h), inflist_or_null(h)));
    }
    {
      const int ib = tm_begin(h);
      CK(launch_lsqr(h, s));
      tm_end(h, NNLS_PH_LSQR, ib, 1);
    }
  }
  if (x_out) {
    const int ib = tm_begin(h);
    CK(cudaMemcpyAsync(x_out, h->xfin.p, sizeof(double) * (size_t)n, cudaMemcpyDefault, s));
    tm_end(h, NNLS_PH_DOWNLOAD, ib, 0);
  }
  nnls_status rs = read_state(h);
  if (rs != NNLS_OK) return rs;
  const DevState& hs = h->h->st;
  if (done_graph) {  // kernels the graph ran (the WHILE body runs iterations + 1 times)
    const int body = hs.iter + 1;
    h->tm.launches[NNLS_PH_DECIDE] += body;
    h->tm.launches[NNLS_PH_CHOL_FACTOR] += body;
    h->tm.launches[NNLS_PH_CHOL_SOLVE] += body;
    h->tm.launches[NNLS_PH_DUAL] += body;
    h->tm.launches[NNLS_PH_LSQR] += 1;
  }
  nnls_status status = NNLS_OK;
  if (hs.status == 7) status = NNLS_ERR_NOT_PD;
  else if (hs.status == 8) status = NNLS_ITERATION_LIMIT;
  if (info) {
    memset(info, 0, sizeof(*info));
    info->status = status;
    info->iterations = hs.iter;
    info->single_exchanges = hs.singles;
    info->free_count = hs.free_count;
    info->lsqr_iterations = hs.lsqr_iterations;
    info->lsqr_stop = hs.lsqr_stop;
    info->infeasible_after_lsqr = hs.infeasible_after_lsqr;
    info->not_pd_column = hs.status == 7 ? hs.not_pd_col : -1;
    info->objective = hs.objective;
    info->kkt_min_x = hs.kkt_min_x;
    info->kkt_min_y = hs.kkt_min_y;
    info->kkt_max_comp = hs.kkt_max_comp;
    info->kkt_dot = hs.kkt_dot;
    info->kappa = hs.kappa;
    info->refined = (hs.status == 0 && hs.free_count > 0 &&
                     (h->prm.lsqr_mode == 1 || h->prm.lsqr_mode == 2 || (h->prm.lsqr_mode == 3 && hs.refined)))
                        ? 1 : 0;
    info->lsqr_fallbacks = hs.lsqr_fallbacks;
  }
  return status;
}

nnls_status nnls_get_free_set(nnls_handle* h, uint8_t* mask_out) {
  if (!h || !mask_out) return NNLS_ERR_INVALID_ARG;
  if (!h->loaded || h->batched) return NNLS_ERR_STATE;
  CK(cudaMemcpyAsync(mask_out, h->mask.p, (size_t)h->n, cudaMemcpyDefault, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return NNLS_OK;
}

nnls_status nnls_get_x_ne(nnls_handle* h, double* x_out) {
  if (!h || !x_out) return NNLS_ERR_INVALID_ARG;
  if (!h->loaded || h->batched) return NNLS_ERR_STATE;
  CK(cudaMemcpyAsync(x_out, h->x.p, sizeof(double) * (size_t)h->n, cudaMemcpyDefault, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return NNLS_OK;
}

nnls_status nnls_get_trace(nnls_handle* h, nnls_iter_rec* recs, int32_t cap, int32_t* count) {
  if (!h || (cap > 0 && !recs)) return NNLS_ERR_INVALID_ARG;
  if (!h->loaded || h->batched) return NNLS_ERR_STATE;
  nnls_status rs = read_state(h);
  if (rs != NNLS_OK) return rs;
  int it = h->h->st.iter;
  int cnt = it < h->trace_cap ? it : h->trace_cap;
  if (cnt > cap) cnt = cap;
  if (count) *count = cnt;
  if (cnt > 0) {
    static_assert(sizeof(nnls_iter_rec) == sizeof(TraceRec), "trace layout");
    CK(cudaMemcpyAsync(recs, h->trace.p, sizeof(TraceRec) * (size_t)cnt, cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
  }
  return NNLS_OK;
}

nnls_status nnls_get_gram(nnls_handle* h, double* G_out, double* c_out) {
  if (!h) return NNLS_ERR_INVALID_ARG;
  if (!h->loaded || h->batched) return NNLS_ERR_STATE;
  const int n = h->n;
  double* G = P<double>(h->Gc);
  if (G_out)
    CK(cudaMemcpy2DAsync(G_out, sizeof(double) * n, G, sizeof(double) * h->ldg, sizeof(double) * n,
                         n, cudaMemcpyDefault, h->stream));
  if (c_out)
    CK(cudaMemcpyAsync(c_out, G + (size_t)n * h->ldg, sizeof(double) * n, cudaMemcpyDefault,
                       h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return NNLS_OK;
}

// debug hook (not in nnls.h): per-task timestamps of the Cholesky DAG
NNLS_API nnls_status nnls_debug_chol_profile(unsigned long long* dev_buf) {
  CK(chol_debug_set_profile(dev_buf));
  return NNLS_OK;
}

NNLS_API nnls_status nnls_debug_lsqr_profile(unsigned long long* dev_buf) {
  CK(lsqr_debug_set_profile(dev_buf));
  return NNLS_OK;
}

NNLS_API nnls_status nnls_debug_batched_profile(long long* dev_buf) {
  CK(batched_debug_set_profile(dev_buf));
  return NNLS_OK;
}

nnls_status nnls_timing_enable(nnls_handle* h, int32_t on) {
  if (!h) return NNLS_ERR_INVALID_ARG;
  tm_flush(h);
  for (int i = 0; i < NNLS_NPHASES; ++i) {
    h->tm.ms[i] = 0.0;
    h->tm.launches[i] = 0;
  }
  h->tm.on = on != 0;
  return NNLS_OK;
}

nnls_status nnls_timing_read(nnls_handle* h, double* ms, int64_t* launches, int32_t cap) {
  if (!h) return NNLS_ERR_INVALID_ARG;
  tm_flush(h);
  for (int i = 0; i < NNLS_NPHASES && i < cap; ++i) {
    if (ms) ms[i] = h->tm.ms[i];
    if (launches) launches[i] = h->tm.launches[i];
  }
  return NNLS_OK;
}

nnls_status nnls_destroy(nnls_handle* h) {
  if (!h) return NNLS_OK;
  if (h->stream) cudaStreamSynchronize(h->stream);
  Buf* bufs[] = {&h->rowptr, &h->colind, &h->vals, &h->b, &h->colptr, &h->rowind, &h->cvals,
                 &h->cursor, &h->tmp_row, &h->tmp_val, &h->csc_temp, &h->Gc, &h->mask, &h->x, &h->y, &h->xF,
                 &h->Fidx, &h->Gidx, &h->Lt, &h->flags, &h->U, &h->V, &h->W, &h->X, &h->R,
                 &h->partials, &h->xfin, &h->st, &h->err, &h->trace, &h->b_nnz_off, &h->b_info_i,
                 &h->b_info_d, &h->b_x, &h->b_mask, &h->Fval, &h->Fcol, &h->Fcnt, &h->b_colview, &h->b_gram,
                 &h->pos, &h->Fs, &h->xs, &h->Gp, &h->cwork, &h->Adense};
  for (Buf* b : bufs) free_buf(*b);
  if (h->s_in) cudaStreamSynchronize(h->s_in);
  if (h->s_out) cudaStreamSynchronize(h->s_out);
  for (cudaEvent_t e : h->pev) cudaEventDestroy(e);
  if (h->s_in) cudaStreamDestroy(h->s_in);
  if (h->s_out) cudaStreamDestroy(h->s_out);
  for (cudaEvent_t e : h->tm.pool) cudaEventDestroy(e);
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->gstream) cudaStreamDestroy(h->gstream);
  for (cudaEvent_t e : h->gev)
    if (e) cudaEventDestroy(e);
  if (h->h) cudaFreeHost(h->h);
  delete h;
  return NNLS_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Step-level entry points (device buffers) for kernel unit tests.
namespace {
struct TmpBufs {
  Buf bufs[12];
  ~TmpBufs() {
    for (Buf& b : bufs) free_buf(b);
  }
};
nnls_status upload_state(DevState* d, const DevState& hs, cudaStream_t s) {
  CK(cudaMemcpyAsync(d, &hs, sizeof(DevState), cudaMemcpyHostToDevice, s));
  return NNLS_OK;
}
nnls_status download_state(DevState& hs, const DevState* d, cudaStream_t s) {
  CK(cudaMemcpyAsync(&hs, d, sizeof(DevState), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return NNLS_OK;
}
int sm_count_now() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}
}  // namespace

extern "C" {

nnls_status nnls_step_gram(int32_t m, int32_t n, int64_t nnz, const int32_t* rowptr,
                           const int32_t* colind, const double* vals, const double* b, double* G,
                           int32_t ldg, double* c, void* stream) {
  if (m < 1 || n < 1 || nnz < 0 || !rowptr || !b || !G || !c || ldg < n) return NNLS_ERR_INVALID_ARG;
  if ((int64_t)n * 8 > 200 * 1024) return NNLS_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  TmpBufs t;
  CK(ensure(t.bufs[0], sizeof(int32_t) * (size_t)(n + 1)));
  CK(ensure(t.bufs[1], sizeof(int32_t) * (size_t)(n + 1)));
  CK(ensure(t.bufs[2], sizeof(int32_t) * (size_t)nnz));
  CK(ensure(t.bufs[3], sizeof(double) * (size_t)nnz));
  CK(ensure(t.bufs[4], sizeof(int32_t) * (size_t)nnz));
  CK(ensure(t.bufs[5], sizeof(double) * (size_t)nnz));
  CK(launch_csr_to_csc(m, n, nnz, rowptr, colind, vals, P<int32_t>(t.bufs[0]), P<int32_t>(t.bufs[2]),
                       P<double>(t.bufs[3]), P<int32_t>(t.bufs[1]), P<int32_t>(t.bufs[4]),
                       P<double>(t.bufs[5]), s));
  CK(launch_gram(m, n, rowptr, colind, vals, P<int32_t>(t.bufs[0]), P<int32_t>(t.bufs[2]),
                 P<double>(t.bufs[3]), b, 0, m, G, ldg, c, sm_count_now(), s));
  CK(cudaStreamSynchronize(s));
  return NNLS_OK;
}

nnls_status nnls_step_normal_solve(int32_t n, const double* G, int32_t ldg, const double* c,
                                   int32_t f, const int32_t* Fidx, double* xF, int32_t* not_pd_col,
                                   void* stream) {
  if (n < 1 || f < 0 || f > n || !G || !c || ldg < n || (f > 0 && (!Fidx || !xF)))
    return NNLS_ERR_INVALID_ARG;
  if (f == 0) return NNLS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  TmpBufs t;
  CK(ensure(t.bufs[0], sizeof(double) * chol_tile_doubles(n)));
  CK(ensure(t.bufs[1], sizeof(int) * chol_flag_count(n)));
  CK(ensure(t.bufs[2], sizeof(DevState)));
  CK(ensure(t.bufs[3], sizeof(double) * (size_t)(f + kTile)));
  CK(cudaMemsetAsync(t.bufs[1].p, 0, t.bufs[1].cap, s));
  DevState hs;
  memset(&hs, 0, sizeof(hs));
  hs.f = f;
  hs.g = n - f;
  hs.epoch = 1;
  hs.not_pd_col = -1;
  nnls_status r = upload_state(P<DevState>(t.bufs[2]), hs, s);
  if (r != NNLS_OK) return r;
  CK(launch_cholesky_solve(n, G, ldg, c, Fidx, P<double>(t.bufs[0]), P<int>(t.bufs[1]),
                           P<double>(t.bufs[3]), P<DevState>(t.bufs[2]), sm_count_now(), s));
  CK(cudaMemcpyAsync(xF, t.bufs[3].p, sizeof(double) * (size_t)f, cudaMemcpyDeviceToDevice, s));
  r = download_state(hs, P<DevState>(t.bufs[2]), s);
  if (r != NNLS_OK) return r;
  if (not_pd_col) *not_pd_col = hs.status == 7 ? hs.not_pd_col : -1;
  return hs.status == 7 ? NNLS_ERR_NOT_PD : NNLS_OK;
}

nnls_status nnls_step_exchange(int32_t n, uint8_t* mask, const double* x, const double* y,
                               int32_t p_max, int32_t* state, int32_t* k_out, int32_t* branch_out,
                               void* stream) {
  if (n < 1 || !mask || !x || !y || !state) return NNLS_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  TmpBufs t;
  CK(ensure(t.bufs[0], sizeof(DevState)));
  CK(ensure(t.bufs[1], sizeof(int32_t) * (size_t)n));
  CK(ensure(t.bufs[2], sizeof(int32_t) * (size_t)n));
  DevState hs;
  memset(&hs, 0, sizeof(hs));
  hs.N = state[0];
  hs.p = state[1];
  hs.iter = state[2];
  hs.singles = state[3];
  hs.max_iter = 0x7fffffff;
  hs.p_max = p_max;
  nnls_status r = upload_state(P<DevState>(t.bufs[0]), hs, s);
  if (r != NNLS_OK) return r;
  CK(launch_decide(n, mask, x, y, P<int32_t>(t.bufs[1]), P<int32_t>(t.bufs[2]),
                   P<DevState>(t.bufs[0]), nullptr, 0, s));
  r = download_state(hs, P<DevState>(t.bufs[0]), s);
  if (r != NNLS_OK) return r;
  state[0] = hs.N;
  state[1] = hs.p;
  state[2] = hs.iter;
  state[3] = hs.singles;
  if (k_out) *k_out = hs.k;
  if (branch_out) *branch_out = hs.done ? -1 : hs.branch;
  return NNLS_OK;
}

nnls_status nnls_step_dual(int32_t n, const double* G, int32_t ldg, const double* c,
                           const uint8_t* mask, double* x, double* y, double tol, void* stream) {
  if (n < 1 || !G || !c || !mask || !x || !y || ldg < n) return NNLS_ERR_INVALID_ARG;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  TmpBufs t;
  CK(ensure(t.bufs[0], sizeof(DevState)));
  CK(ensure(t.bufs[1], sizeof(int32_t) * (size_t)n));
  CK(ensure(t.bufs[2], sizeof(int32_t) * (size_t)n));
  CK(ensure(t.bufs[3], sizeof(double) * (size_t)n));
  CK(cudaMemsetAsync(t.bufs[0].p, 0, sizeof(DevState), s));
  CK(launch_compact(n, mask, x, P<int32_t>(t.bufs[1]), P<int32_t>(t.bufs[2]), P<double>(t.bufs[3]),
                    P<DevState>(t.bufs[0]), s));
  CK(launch_dual(n, G, ldg, c, P<int32_t>(t.bufs[1]), P<int32_t>(t.bufs[2]), P<double>(t.bufs[3]),
                 const_cast<uint8_t*>(mask), x, y, tol, P<DevState>(t.bufs[0]), sm_count_now(), s));
  CK(cudaStreamSynchronize(s));
  return NNLS_OK;
}

}  // extern "C"

namespace {

// host checks of the batch shape and nnz offsets, device buffers for the
// whole batch; h->b_hoff = nnz_off on the host
nnls_status batched_prepare(nnls_handle* h, int32_t batch, int32_t m, int32_t n, const int64_t* nnz_off,
                            const int32_t* rowptr, const int32_t* colind, const double* vals,
                            const double* b) {
  if (!h || !h->batched) return NNLS_ERR_INVALID_ARG;
  if (batch < 1 || n < 1 || m < n || n > 64 || m > 256 || !nnz_off || !rowptr || !b)
    return NNLS_ERR_INVALID_ARG;
  h->loaded = false;
  // nnz offsets are needed on the host to size shared memory (nnz_max)
  std::vector<int64_t>& hoff = h->b_hoff;
  hoff.resize((size_t)batch + 1);
  if (cudaMemcpy(hoff.data(), nnz_off, sizeof(int64_t) * (size_t)(batch + 1), cudaMemcpyDefault) !=
      cudaSuccess)
    return NNLS_ERR_CUDA;
  int64_t nnz_max = 0;
  bool bad = hoff[0] != 0;
  for (int q = 0; q < batch && !bad; ++q) {
    const int64_t d = hoff[q + 1] - hoff[q];
    if (d < 0 || d > (int64_t)m * n) bad = true;
    if (d > nnz_max) nnz_max = d;
  }
  if (bad) return NNLS_ERR_DIMENSION;
  const int64_t total = hoff[batch];
  if (total > 0 && (!colind || !vals)) return NNLS_ERR_INVALID_ARG;
  if (batched_smem_bytes(m, n, (int)nnz_max) > 220 * 1024) return NNLS_ERR_INVALID_ARG;
  h->m = m;
  h->n = n;
  h->batch = batch;
  h->nnz = total;
  h->ldg = (int)nnz_max;  // batched: ldg holds nnz_max
  CK(ensure(h->b_nnz_off, sizeof(int64_t) * (size_t)(batch + 1)));
  CK(ensure(h->rowptr, sizeof(int32_t) * (size_t)batch * (m + 1)));
  CK(ensure(h->colind, sizeof(int32_t) * (size_t)total));
  CK(ensure(h->vals, sizeof(double) * (size_t)total));
  CK(ensure(h->b, sizeof(double) * (size_t)batch * m));
  CK(ensure(h->b_x, sizeof(double) * (size_t)batch * n));
  CK(ensure(h->b_mask, (size_t)batch * n));
  CK(ensure(h->b_colview, batched_colview_stride(n, (int)nnz_max) * (size_t)batch));
  CK(ensure(h->b_gram, batched_gram_scratch(n, h->sms)));
  CK(ensure(h->b_info_i, sizeof(int32_t) * kInfoI * (size_t)batch));
  CK(ensure(h->b_info_d, sizeof(double) * kInfoD * (size_t)batch));
  return NNLS_OK;
}

BatchArgs batched_args(nnls_handle* h) {
  const nnls_params& p = h->prm;
  BatchArgs a{};
  a.batch = h->batch;
  a.m = h->m;
  a.n = h->n;
  a.nnz_off = P<int64_t>(h->b_nnz_off);
  a.rowptr = P<int32_t>(h->rowptr);
  a.colind = P<int32_t>(h->colind);
  a.vals = P<double>(h->vals);
  a.b = P<double>(h->b);
  a.x_out = P<double>(h->b_x);
  a.mask_out = P<uint8_t>(h->b_mask);
  a.info_i = P<int32_t>(h->b_info_i);
  a.info_d = P<double>(h->b_info_d);
  a.tol = p.zero_tol;
  a.atol = p.lsqr_atol;
  a.btol = p.lsqr_btol;
  a.conlim = p.lsqr_conlim;
  a.p_max = p.p_max;
  a.max_iter = p.max_iter > 0 ? p.max_iter : 10 * h->n;
  a.lsqr_mode = p.lsqr_mode;
  a.itn_limit = p.lsqr_itn_limit;
  a.kkt = p.kkt;
  a.adaptive_threshold = p.adaptive_threshold;
  {
    const char* cp = getenv("NNLS_BATCH_CAP");
    a.lsqr_cap_pct = (cp && cp[0]) ? atoi(cp) : 90;
    if (a.lsqr_cap_pct < 10) a.lsqr_cap_pct = 10;
  }
  a.colview = P<uint8_t>(h->b_colview);
  a.cv_stride = batched_colview_stride(h->n, h->ldg);
  a.gram = P<double>(h->b_gram);
  a.guard = nullptr;
  return a;
}

// per-problem info of problems [p0, p0 + count) from the device arrays
nnls_status batched_info(nnls_handle* h, int p0, int count, nnls_info* info_out, cudaStream_t s) {
  const size_t nb = (size_t)count;
  std::vector<int32_t> ii(kInfoI * nb);
  std::vector<double> dd(kInfoD * nb);
  CK(cudaMemcpyAsync(ii.data(), P<int32_t>(h->b_info_i) + (size_t)p0 * kInfoI, sizeof(int32_t) * kInfoI * nb,
                     cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(dd.data(), P<double>(h->b_info_d) + (size_t)p0 * kInfoD, sizeof(double) * kInfoD * nb,
                     cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  nnls_status worst = NNLS_OK;
  for (size_t q = 0; q < nb; ++q) {
    nnls_info& o = info_out[q];
    memset(&o, 0, sizeof(o));
    const int st = ii[q * kInfoI + 0];
    o.status = st == 7 ? NNLS_ERR_NOT_PD : (st == 8 ? NNLS_ITERATION_LIMIT : NNLS_OK);
    if (o.status != NNLS_OK && worst == NNLS_OK) worst = (nnls_status)o.status;
    o.iterations = ii[q * kInfoI + 1];
    o.single_exchanges = ii[q * kInfoI + 2];
    o.free_count = ii[q * kInfoI + 3];
    o.lsqr_iterations = ii[q * kInfoI + 4];
    o.lsqr_stop = ii[q * kInfoI + 5];
    o.infeasible_after_lsqr = ii[q * kInfoI + 6];
    o.not_pd_column = ii[q * kInfoI + 7];
    o.objective = dd[q * kInfoD + 0];
    o.kkt_min_x = dd[q * kInfoD + 1];
    o.kkt_min_y = dd[q * kInfoD + 2];
    o.kkt_max_comp = dd[q * kInfoD + 3];
    o.kkt_dot = dd[q * kInfoD + 4];
    o.refined = ii[q * kInfoI + 8];
    o.kappa = dd[q * kInfoD + 5];
  }
  return worst;
}

}  // namespace

extern "C" {

nnls_status nnls_load_batched(nnls_handle* h, int32_t batch, int32_t m, int32_t n,
                              const int64_t* nnz_off, const int32_t* rowptr, const int32_t* colind,
                              const double* vals, const double* b) {
  nnls_status st = batched_prepare(h, batch, m, n, nnz_off, rowptr, colind, vals, b);
  if (st != NNLS_OK) return st;
  cudaStream_t s = h->stream;
  const int64_t total = h->nnz;
  CK(ensure(h->err, sizeof(int) * 8));
  CK(cudaMemcpyAsync(h->b_nnz_off.p, nnz_off, sizeof(int64_t) * (size_t)(batch + 1), cudaMemcpyDefault, s));
  CK(cudaMemcpyAsync(h->rowptr.p, rowptr, sizeof(int32_t) * (size_t)batch * (m + 1), cudaMemcpyDefault, s));
  if (total > 0) {
    CK(cudaMemcpyAsync(h->colind.p, colind, sizeof(int32_t) * (size_t)total, cudaMemcpyDefault, s));
    CK(cudaMemcpyAsync(h->vals.p, vals, sizeof(double) * (size_t)total, cudaMemcpyDefault, s));
  }
  CK(cudaMemcpyAsync(h->b.p, b, sizeof(double) * (size_t)batch * m, cudaMemcpyDefault, s));
  CK(cudaMemsetAsync(h->err.p, 0, sizeof(int) * 6, s));
  TIMED(NNLS_PH_VALIDATE, 3,
        launch_validate_batched(batch, m, n, P<int64_t>(h->b_nnz_off), 0, total, P<int32_t>(h->rowptr),
                                P<int32_t>(h->colind), P<double>(h->vals), P<double>(h->b),
                                P<int>(h->err), s));
  CK(cudaMemcpyAsync(h->h->err, h->err.p, sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (h->h->err[0]) return map_err_bits(h->h->err[0]);
  h->loaded = true;
  return NNLS_OK;
}

nnls_status nnls_setup_batched(nnls_handle** h, int32_t batch, int32_t m, int32_t n,
                               const int64_t* nnz_off, const int32_t* rowptr, const int32_t* colind,
                               const double* vals, const double* b, const nnls_params* p,
                               void* cuda_stream) {
  nnls_status s = create_impl(h, p, cuda_stream);
  if (s != NNLS_OK) return s;
  (*h)->batched = true;
  s = nnls_load_batched(*h, batch, m, n, nnz_off, rowptr, colind, vals, b);
  if (s != NNLS_OK) {
    nnls_destroy(*h);
    *h = nullptr;
  }
  return s;
}

nnls_status nnls_create_batched(nnls_handle** h, const nnls_params* p, void* cuda_stream) {
  nnls_status s = create_impl(h, p, cuda_stream);
  if (s == NNLS_OK) (*h)->batched = true;
  return s;
}

nnls_status nnls_solve_batched(nnls_handle* h, double* x_out, nnls_info* info_out,
                               uint8_t* mask_out) {
  if (!h || !h->batched) return NNLS_ERR_INVALID_ARG;
  if (!h->loaded) return NNLS_ERR_STATE;
  cudaStream_t s = h->stream;
  BatchArgs a = batched_args(h);
  TIMED(NNLS_PH_BATCHED, 2, launch_batched_nnz(a, h->ldg, h->sms, s));
  const size_t nb = (size_t)h->batch;
  const int ibd = tm_begin(h);
  if (x_out) CK(cudaMemcpyAsync(x_out, h->b_x.p, sizeof(double) * nb * h->n, cudaMemcpyDefault, s));
  if (mask_out) CK(cudaMemcpyAsync(mask_out, h->b_mask.p, nb * h->n, cudaMemcpyDefault, s));
  tm_end(h, NNLS_PH_DOWNLOAD, ibd, 0);
  if (info_out) return batched_info(h, 0, h->batch, info_out, s);
  CK(cudaStreamSynchronize(s));
  return NNLS_OK;
}

nnls_status nnls_run_batched(nnls_handle* h, int32_t batch, int32_t m, int32_t n, const int64_t* nnz_off,
                             const int32_t* rowptr, const int32_t* colind, const double* vals,
                             const double* b, double* x_out, nnls_info* info_out, uint8_t* mask_out,
                             int32_t chunk) {
  nnls_status st = batched_prepare(h, batch, m, n, nnz_off, rowptr, colind, vals, b);
  if (st != NNLS_OK) return st;
  if (chunk <= 0) chunk = 8192;
  if (chunk > batch) chunk = batch;  // (a huge chunk means one chunk; no int overflow below)
  const int nch = (batch + chunk - 1) / chunk;
  cudaStream_t s = h->stream;
  if (!h->s_in) CK(cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking));
  if (!h->s_out) CK(cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking));
  while (h->pev.size() < (size_t)(2 * nch + 1)) {
    cudaEvent_t e;
    CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    h->pev.push_back(e);
  }
  CK(ensure(h->err, sizeof(int) * 8 * (size_t)nch));
  const std::vector<int64_t>& off = h->b_hoff;
  // the copy streams start after everything already queued on the stream
  // (an earlier call still reading these buffers)
  cudaEvent_t e0 = h->pev[2 * nch];
  CK(cudaEventRecord(e0, s));
  CK(cudaStreamWaitEvent(h->s_in, e0, 0));
  CK(cudaMemsetAsync(h->err.p, 0, sizeof(int) * 8 * (size_t)nch, s));
  CK(cudaMemcpyAsync(h->b_nnz_off.p, nnz_off, sizeof(int64_t) * (size_t)(batch + 1), cudaMemcpyDefault,
                     h->s_in));
  BatchArgs a0 = batched_args(h);
  const size_t cvs = a0.cv_stride;
  for (int c = 0; c < nch; ++c) {
    const int p0 = c * chunk, p1 = p0 + chunk < batch ? p0 + chunk : batch, cnt = p1 - p0;
    const int64_t o0 = off[p0], o1 = off[p1];
    // stage c in: its CSR slice and b
    CK(cudaMemcpyAsync(P<int32_t>(h->rowptr) + (size_t)p0 * (m + 1), rowptr + (size_t)p0 * (m + 1),
                       sizeof(int32_t) * (size_t)cnt * (m + 1), cudaMemcpyDefault, h->s_in));
    if (o1 > o0) {
      CK(cudaMemcpyAsync(P<int32_t>(h->colind) + o0, colind + o0, sizeof(int32_t) * (size_t)(o1 - o0),
                         cudaMemcpyDefault, h->s_in));
      CK(cudaMemcpyAsync(P<double>(h->vals) + o0, vals + o0, sizeof(double) * (size_t)(o1 - o0),
                         cudaMemcpyDefault, h->s_in));
    }
    CK(cudaMemcpyAsync(P<double>(h->b) + (size_t)p0 * m, b + (size_t)p0 * m, sizeof(double) * (size_t)cnt * m,
                       cudaMemcpyDefault, h->s_in));
    CK(cudaEventRecord(h->pev[2 * c], h->s_in));
    // stage c compute: validate, then solve unless validation failed
    CK(cudaStreamWaitEvent(s, h->pev[2 * c], 0));
    int* err = P<int>(h->err) + 8 * c;
    TIMED(NNLS_PH_VALIDATE, 3,
          launch_validate_batched(cnt, m, n, P<int64_t>(h->b_nnz_off) + p0, o0, o1,
                                  P<int32_t>(h->rowptr) + (size_t)p0 * (m + 1), P<int32_t>(h->colind),
                                  P<double>(h->vals), P<double>(h->b) + (size_t)p0 * m, err, s));
    BatchArgs a = a0;
    a.batch = cnt;
    a.nnz_off = a0.nnz_off + p0;
    a.rowptr = a0.rowptr + (size_t)p0 * (m + 1);
    a.b = a0.b + (size_t)p0 * m;
    a.x_out = a0.x_out + (size_t)p0 * n;
    a.mask_out = a0.mask_out + (size_t)p0 * n;
    a.info_i = a0.info_i + (size_t)p0 * kInfoI;
    a.info_d = a0.info_d + (size_t)p0 * kInfoD;
    a.colview = a0.colview + (size_t)p0 * cvs;
    a.guard = err;
    TIMED(NNLS_PH_BATCHED, 2, launch_batched_nnz(a, h->ldg, h->sms, s));
    CK(cudaEventRecord(h->pev[2 * c + 1], s));
    // stage c out
    CK(cudaStreamWaitEvent(h->s_out, h->pev[2 * c + 1], 0));
    if (x_out)
      CK(cudaMemcpyAsync(x_out + (size_t)p0 * n, a.x_out, sizeof(double) * (size_t)cnt * n, cudaMemcpyDefault,
                         h->s_out));
    if (mask_out)
      CK(cudaMemcpyAsync(mask_out + (size_t)p0 * n, a.mask_out, (size_t)cnt * n, cudaMemcpyDefault, h->s_out));
  }
  // the stream orders after the outputs (the caller's view of completion)
  CK(cudaEventRecord(h->pev[2 * nch], h->s_out));
  CK(cudaStreamWaitEvent(s, h->pev[2 * nch], 0));
  std::vector<int> herr(8 * (size_t)nch);
  CK(cudaMemcpyAsync(herr.data(), h->err.p, sizeof(int) * 8 * (size_t)nch, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int c = 0; c < nch; ++c)
    if (herr[8 * c]) return map_err_bits(herr[8 * c]);
  h->loaded = true;
  if (info_out) return batched_info(h, 0, batch, info_out, s);
  return NNLS_OK;
}

}  // extern "C"
