// pivot.cu -- the pivoting steps of the block principal pivoting algorithm
// that surround the normal-equations solve:
//   a2 init      F = {}, x = 0, y = -A^T b (zeroed), p = p_max, N = n+1
//   a3 decide    count infeasibles, choose the branch, exchange
//   a4 compact   Fidx / Gidx by warp ballot + block prefix scan
//   a7/a8 dual   y_G = (A^T A)_GF x_F - (A^T b)_G (Eq. 5, Gram form), then
//                |x_F|, |y_G| < tol -> 0 (reading c1); inside the
//                pivot loop the same kernel also counts the infeasibles
//                (warp/block reductions + one atomic per CTA), and its last
//                CTA chooses the branch and applies the exchange,
//                so decide is left with the compaction (a4)
#include <cuda_runtime.h>
#include <math.h>

#include <cub/block/block_radix_sort.cuh>

#include "common.cuh"
#include "kernels.cuh"

namespace nnls {

// ---------------------------------------------------------------- init (a2)
__global__ void init_kernel(int n, const double* __restrict__ c, uint8_t* mask, double* x,
                            double* y, double tol, DevState* st, int p_max, int max_iter, int32_t* pos) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    mask[i] = 0;
    if (pos != nullptr) pos[i] = -1;
    x[i] = 0.0;
    const double v = -c[i];
    y[i] = fabs(v) < tol ? 0.0 : v;  // reading c2: the initial y is zeroed too
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->k = 0;
    st->N = n + 1;  // reading c8: N = infinity
    st->p = p_max;
    st->iter = 0;
    st->singles = 0;
    st->f = 0;
    st->g = n;
    st->branch = -1;
    st->done = 0;
    st->status = 0;
    st->not_pd_col = -1;
    st->max_iter = max_iter;
    st->p_max = p_max;
    st->below_bits = 0ull;
    st->above_bits = dbits(INFINITY);
    st->lsqr_iterations = 0;
    st->lsqr_stop = 0;
    st->infeasible_after_lsqr = 0;
    st->reuse_cols = 0;
    st->kappa = 0.0;
    st->refined = 0;
    st->lsqr_fallbacks = 0;
    st->decided = 0;
    st->inf_count = 0;
    st->inf_last1 = 0;
    st->dual_ticket = 0u;
  }
}

cudaError_t launch_init(int n, const double* c, uint8_t* mask, double* x, double* y, double tol,
                        DevState* st, int p_max, int max_iter, cudaStream_t s, int32_t* pos) {
  int blocks = (n + 255) / 256;
  if (blocks > 1024) blocks = 1024;
  if (blocks < 1) blocks = 1;
  init_kernel<<<blocks, 256, 0, s>>>(n, c, mask, x, y, tol, st, p_max, max_iter, pos);
  return cudaGetLastError();
}

// Fidx = sorted F, Gidx = sorted G (warp ballot + block prefix scan over
// chunks of blockDim.x).  Called by all threads of one CTA; *carryF/*carryG
// (shared, zero on entry) end as |F| and |G|.
__device__ void block_compact(int n, const uint8_t* __restrict__ mask, int32_t* __restrict__ Fidx,
                              int32_t* __restrict__ Gidx, int* s_wF, int* s_wG, int* s_cnt,
                              int* carryF, int* carryG) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + tid;
    const bool valid = i < n;
    const bool inF = valid && mask[i];
    const bool inG = valid && !mask[i];
    const unsigned bF = __ballot_sync(kFull, inF), bG = __ballot_sync(kFull, inG);
    if (lane == 0) {
      s_wF[wid] = __popc(bF);
      s_wG[wid] = __popc(bG);
    }
    __syncthreads();
    if (wid == 0) {
      const int nw = blockDim.x >> 5;
      int a = lane < nw ? s_wF[lane] : 0, bb = lane < nw ? s_wG[lane] : 0;
      int ia = a, ib = bb;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int ya = __shfl_up_sync(kFull, ia, o), yb = __shfl_up_sync(kFull, ib, o);
        if (lane >= o) {
          ia += ya;
          ib += yb;
        }
      }
      s_wF[lane] = ia - a;  // exclusive
      s_wG[lane] = ib - bb;
      if (lane == 31) {
        s_cnt[0] = ia;  // chunk totals
        s_cnt[1] = ib;
      }
    }
    __syncthreads();
    if (inF) Fidx[*carryF + s_wF[wid] + __popc(bF & lt)] = i;
    if (inG) Gidx[*carryG + s_wG[wid] + __popc(bG & lt)] = i;
    __syncthreads();
    if (tid == 0) {
      *carryF += s_cnt[0];
      *carryG += s_cnt[1];
    }
    __syncthreads();
  }
}

// ------------------------------------------- factorization order (reuse)
// The Cholesky factor of the permuted (A^T A)_FF is as valid as that of the
// sorted one (the paper's TAUCS / colamd solvers factor permuted matrices,
// P:131); choosing the order lets consecutive pivot iterations share
// a factor prefix: if the first q members of the previous order are all
// still in F, the leading q x q block of L -- and every tile of it -- is
// unchanged (left-looking Cholesky: column k of L only depends on the
// leading (k+1) x (k+1) block).  New order = that prefix, then the other
// members of F sorted by predicted stability: old members by decreasing x
// (those with x near 0 are the likeliest to leave next), then the newly
// added ones in index order -- so the first factorization is in index order,
// exactly the oracle's.  (|F|, the iterates and the termination are those of
// P:86-104; only rounding differs.)
constexpr int kOrderMax = 8192;  // largest sorted tail; longer tails stay in index order

constexpr int kDecideThreads = 1024;
__device__ __forceinline__ unsigned order_key(double v) {  // monotone 16-bit key of (float)v
  unsigned u = __float_as_uint((float)v);
  u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return u >> 16;
}
template <int IPT>
using TailSort = cub::BlockRadixSort<unsigned, kDecideThreads, IPT, int>;  // 4 passes of 4 bits

template <int IPT>
__device__ void sort_tail(int32_t* __restrict__ tail, int r, const double* __restrict__ x,
                          const int32_t* __restrict__ pos, void* smem) {
  unsigned key[IPT];
  int val[IPT];
#pragma unroll
  for (int k = 0; k < IPT; ++k) {  // blocked: element e = tid * IPT + k (index order)
    const int e = threadIdx.x * IPT + k;
    if (e < r) {
      const int i = tail[e];
      key[k] = pos[i] >= 0 ? order_key(-x[i]) : 0xFFFFu;
      val[k] = i;
    } else {
      key[k] = 0xFFFFu;  // after every real element (stable)
      val[k] = -1;
    }
  }
  __syncthreads();  // (tail[] is rewritten below)
  TailSort<IPT>(*reinterpret_cast<typename TailSort<IPT>::TempStorage*>(smem))
      .SortBlockedToStriped(key, val, 4, 16);  // the top 12 key bits (3 radix passes)
#pragma unroll
  for (int k = 0; k < IPT; ++k) {  // striped: rank = k * threads + tid
    const int rank = k * kDecideThreads + threadIdx.x;
    if (rank < r) tail[rank] = val[k];
  }
}
// Short tails (r <= threads): rank by comparison, element t -> position
// #{u : (key_u, i_u) < (key_t, i_t)} -- the same stable order as sort_tail
// (12-bit key, index ties), r broadcast reads per thread instead of the
// radix sort's fixed passes.
__device__ void rank_tail(int32_t* __restrict__ tail, int r, const double* __restrict__ x,
                          const int32_t* __restrict__ pos, void* smem) {
  unsigned* sk = reinterpret_cast<unsigned*>(smem);  // (key << 20) | element index t (t < 2^20)
  const int t = threadIdx.x;
  int i = 0;
  unsigned kt = 0xFFFFFFFFu;
  if (t < r) {
    i = tail[t];
    const unsigned key = (pos[i] >= 0 ? order_key(-x[i]) : 0xFFFFu) >> 4;  // top 12 bits
    kt = (key << 20) | (unsigned)t;  // tail[] is in index order: t breaks ties like the index
    sk[t] = kt;
  }
  __syncthreads();  // (tail[] is rewritten below)
  if (t < r) {
    int rank = 0;
#pragma unroll 8
    for (int u = 0; u < r; ++u) rank += sk[u] < kt;
    tail[rank] = i;
  }
}

constexpr size_t kTailSortSmem = sizeof(typename TailSort<kOrderMax / kDecideThreads>::TempStorage) >
                                         sizeof(typename TailSort<1>::TempStorage)
                                     ? sizeof(typename TailSort<kOrderMax / kDecideThreads>::TempStorage)
                                     : sizeof(typename TailSort<1>::TempStorage);

// Called by all threads of the decide CTA after the exchange.  fprev: |F| of
// the previous order.  Writes Fidx (order), Gidx (sorted G), pos; returns f
// in *s_f and the prefix length in *s_q.
__device__ void order_free_set(int n, const uint8_t* __restrict__ mask, const double* __restrict__ x,
                               const double* __restrict__ y, int32_t* __restrict__ pos,
                               int32_t* __restrict__ Fidx, int32_t* __restrict__ Gidx,
                               int32_t* __restrict__ Fs, double* __restrict__ xs, int fprev, int* s_wF,
                               int* s_wG, int* s_wS,
                               int* s_cnt, int* s_f, int* s_g, int* s_s, int* s_q, int* s_old,
                               void* sort_smem) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  // Each thread owns kE consecutive indices per sweep (n <= 1024 kE: one
  // sweep), its (mask, pos) held in registers from (1) to (2): one block
  // reduction and one block scan per sweep instead of per 1024 indices.
  constexpr int kE = 8;
  const int E = min(kE, max(1, (n + (int)blockDim.x - 1) / (int)blockDim.x));
  const int span = E * (int)blockDim.x;
  // (1) q = first position of the previous order whose member left F
  int qloc = fprev;
  for (int base = 0; base < n; base += span) {
    const int i0 = base + E * tid;
#pragma unroll
    for (int e = 0; e < kE; ++e) {
      const int i = i0 + e;
      if (e < E && i < n) {
        const int pi = pos[i];
        if (pi >= 0 && !mask[i]) qloc = min(qloc, pi);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) qloc = min(qloc, __shfl_xor_sync(kFull, qloc, o));
  if (lane == 0) s_cnt[wid] = qloc;
  __syncthreads();
  if (wid == 0) {
    int v = lane < nw ? s_cnt[lane] : fprev;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(kFull, v, o));
    if (lane == 0) {
      *s_q = v;
      *s_f = v;  // running |F| (the prefix stays in place)
      *s_g = 0;
      *s_s = 0;
      *s_old = 0;
    }
  }
  __syncthreads();
  const int q = *s_q;
  // (2) the tail R = F minus the prefix -> Fidx[q..) in index order; G ->
  // Gidx, F -> Fs (both in index order)
  for (int base = 0; base < n; base += span) {
    const int i0 = base + E * tid;
    unsigned fR = 0u, fG = 0u, fS = 0u;
    int cR = 0, cG = 0, cS = 0, cO = 0;
#pragma unroll
    for (int e = 0; e < kE; ++e) {
      const int i = i0 + e;
      if (e < E && i < n) {
        const bool inF = mask[i] != 0;
        const int pi = pos[i];
        const bool inR = inF && !(pi >= 0 && pi < q);
        fR |= (inR ? 1u : 0u) << e;
        fG |= (inF ? 0u : 1u) << e;
        fS |= (inF ? 1u : 0u) << e;
        cO += (inR && pi >= 0) ? 1 : 0;
      }
    }
    cR = __popc(fR);
    cG = __popc(fG);
    cS = __popc(fS);
    // block exclusive scan of (cR, cG, cS)
    int ia = cR, ib = cG, ic = cS;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int ya = __shfl_up_sync(kFull, ia, o), yb = __shfl_up_sync(kFull, ib, o),
                yc = __shfl_up_sync(kFull, ic, o);
      if (lane >= o) {
        ia += ya;
        ib += yb;
        ic += yc;
      }
    }
    cO = warp_sum_i(cO);
    if (lane == 31) {
      s_wF[wid] = ia;
      s_wG[wid] = ib;
      s_wS[wid] = ic;
    }
    if (lane == 0 && cO != 0) atomicAdd(s_old, cO);
    __syncthreads();
    if (wid == 0) {
      int a = lane < nw ? s_wF[lane] : 0, bb = lane < nw ? s_wG[lane] : 0, cc = lane < nw ? s_wS[lane] : 0;
      int xa = a, xb = bb, xc = cc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int ya = __shfl_up_sync(kFull, xa, o), yb = __shfl_up_sync(kFull, xb, o),
                  yc = __shfl_up_sync(kFull, xc, o);
        if (lane >= o) {
          xa += ya;
          xb += yb;
          xc += yc;
        }
      }
      s_wF[lane] = xa - a;
      s_wG[lane] = xb - bb;
      s_wS[lane] = xc - cc;
      if (lane == 31) {
        s_cnt[0] = xa;
        s_cnt[1] = xb;
        s_cnt[2] = xc;
      }
    }
    __syncthreads();
    int oR = *s_f + s_wF[wid] + ia - cR, oG = *s_g + s_wG[wid] + ib - cG, oS = *s_s + s_wS[wid] + ic - cS;
#pragma unroll
    for (int e = 0; e < kE; ++e) {
      const int i = i0 + e;
      if ((fR >> e) & 1u) Fidx[oR++] = i;
      if ((fS >> e) & 1u) Fs[oS++] = i;
      if ((fG >> e) & 1u) {
        Gidx[oG++] = i;
        pos[i] = -1;
        if (xs != nullptr) xs[i] = 0.0;  // (the dual streams whole G rows against xs: zero off F)
      }
    }
    __syncthreads();
    if (tid == 0) {
      *s_f += s_cnt[0];
      *s_g += s_cnt[1];
      *s_s += s_cnt[2];
    }
    __syncthreads();
  }
  const int f = *s_f, r = f - q;
  // (3) stable sort of the tail by the top 12 bits of a 16-bit key (the order
  // is a heuristic: 3 mantissa bits give the same kept prefixes as the exact
  // sort at configs 1 and 2): old members (pos >= 0) by decreasing x, new
  // members after them in index order (the first factorization is thus in
  // index order, as the oracle's); pos[] still holds the previous positions.
#ifndef NO_ORDER_SORT
  if (r > 1 && r <= kOrderMax && *s_old > 0) {  // (no old member: already in order)
    if (r <= kDecideThreads) rank_tail(Fidx + q, r, x, pos, sort_smem);
    else sort_tail<kOrderMax / kDecideThreads>(Fidx + q, r, x, pos, sort_smem);
    __syncthreads();
  }
#endif
  for (int t = tid; t < r; t += blockDim.x) pos[Fidx[q + t]] = q + t;
}

// ------------------------------------------------- decide + exchange (a3, a4)
// The branch of P:89-101 from the infeasible count kk of this iteration (one
// thread): -1 feasible (k = 0, the while-loop ends) or the iteration limit
// (reading c12); 0 block exchange with progress; 1 block exchange
// within the p no-progress budget; 2 single exchange.
__device__ int choose_branch(DevState* st, int kk) {
  int branch;
  st->k = kk;
  if (kk == 0) {
    st->done = 1;
    branch = -1;
  } else if (st->iter >= st->max_iter) {
    st->status = 8;  // ITERATION_LIMIT
    branch = -1;
  } else if (kk < st->N) {
    st->N = kk;
    st->p = st->p_max;
    branch = 0;
  } else if (st->p > 0) {
    st->p -= 1;
    branch = 1;
  } else {
    st->singles += 1;
    branch = 2;
  }
  st->branch = branch;
  return branch;
}

// One CTA of 1024 threads.  Each thread owns the indices i = tid + 1024 q, so
// the "snapshot before any flip" of reading c10 is automatic: a thread reads
// its own (mask, x, y) and flips only its own entries after the block-wide
// decision.
__global__ void __launch_bounds__(kDecideThreads) decide_kernel(
    int n, uint8_t* __restrict__ mask, const double* __restrict__ x,
    const double* __restrict__ y, int32_t* __restrict__ Fidx, int32_t* __restrict__ Gidx,
    DevState* st, TraceRec* trace, int trace_cap, cudaGraphConditionalHandle loop, int use_loop,
    int32_t* pos, int32_t* Fs, double* xs) {
  extern __shared__ __align__(16) unsigned char s_sort[];  // (pos != nullptr) the tail sort's storage
  pdl_wait();
  __shared__ int s_cnt[32], s_max[32];
  __shared__ int s_wF[32], s_wG[32], s_wS[32];
  __shared__ int s_branch, s_last, s_carryF, s_carryG, s_carryS, s_q, s_fprev, s_old;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  // close the previous iteration's trace record (extremes from the dual kernel)
  if (tid == 0 && trace != nullptr) {
    const int it = st->iter;
    if (it > 0 && it - 1 < trace_cap) {
      trace[it - 1].below_tol = __longlong_as_double((long long)st->below_bits);
      trace[it - 1].above_tol = __longlong_as_double((long long)st->above_bits);
    }
  }
  if (st->status != 0 || st->done) {
    if (use_loop && tid == 0) cudaGraphSetConditional(loop, 0);  // leave the device-side loop
    return;
  }

  // (fused) the dual kernel already counted, chose the branch and exchanged
  if (tid == 0) s_branch = st->decided ? st->branch : -2;
  __syncthreads();
  int branch = s_branch;
  if (branch == -2) {
    // pass 1: k = #{i in F: x_i < 0} + #{j in G: y_j < 0} (reading c5);
    // largest infeasible original index (reading c6)
    int k = 0, last = -1;
    for (int i = tid; i < n; i += kDecideThreads) {
      const bool inf = mask[i] ? (x[i] < 0.0) : (y[i] < 0.0);
      if (inf) {
        ++k;
        last = i;
      }
    }
    k = warp_sum_i(k);
    last = warp_max_i(last);
    if (lane == 0) {
      s_cnt[wid] = k;
      s_max[wid] = last;
    }
    __syncthreads();
    if (wid == 0) {
      int kk = s_cnt[lane], ll = s_max[lane];
      kk = warp_sum_i(kk);
      ll = warp_max_i(ll);
      if (lane == 0) {
        s_branch = choose_branch(st, kk);
        s_last = ll;
      }
    }
    __syncthreads();
    branch = s_branch;
    if (branch < 0) {
      if (use_loop && tid == 0) cudaGraphSetConditional(loop, 0);  // feasible / iteration limit
      return;
    }
    const int lastidx = s_last;
    // pass 2: exchange (from the snapshot: each thread re-reads its own entries)
    for (int i = tid; i < n; i += kDecideThreads) {
      const uint8_t mi = mask[i];
      const bool inf = mi ? (x[i] < 0.0) : (y[i] < 0.0);
      const bool flip = (branch == 2) ? (i == lastidx) : inf;
      if (flip) mask[i] = mi ? 0 : 1;
    }
  }
  if (tid == 0) {
    st->decided = 0;
    s_fprev = st->keep_none ? 0 : st->f;  // (keep_none: the previous factor failed, nothing is kept)
    st->keep_none = 0;
    s_carryF = 0;
    s_carryG = 0;
  }
  __syncthreads();

  if (pos == nullptr) {
    block_compact(n, mask, Fidx, Gidx, s_wF, s_wG, s_cnt, &s_carryF, &s_carryG);
  } else {
    order_free_set(n, mask, x, y, pos, Fidx, Gidx, Fs, xs, s_fprev, s_wF, s_wG, s_wS, s_cnt, &s_carryF,
                   &s_carryG, &s_carryS, &s_q, &s_old, s_sort);
  }
  if (tid == 0) {
    const int f = s_carryF;
    st->f = f;
    // whole tile columns of the kept prefix (the factorization keeps at least
    // its last tile column to itself)
    int jq = 0;
    if (pos != nullptr && f > 0) jq = min(s_q / kTile, (f + kTile - 1) / kTile - 1);
    st->reuse_cols = jq > 0 ? jq : 0;
    st->g = s_carryG;
    st->epoch += 1;
    st->tile_counter = 0;
    st->solve_counter = 0;
    st->role_factor = 0;
    st->role_solve = 0;
    st->below_bits = 0ull;
    st->above_bits = dbits(INFINITY);
    const int it = st->iter;
    if (trace != nullptr && it < trace_cap) {
      trace[it].iter = it + 1;
      trace[it].k = st->k;
      trace[it].branch = branch;
      trace[it].f = f;
      trace[it].below_tol = 0.0;
      trace[it].above_tol = INFINITY;
      trace[it].kept = (jq > 0 ? jq : 0) * kTile;
      trace[it].pad = 0;
    }
  }
}

// Step-API helper: Fidx/Gidx/f/g from a given mask, and x_F = x[Fidx].
__global__ void __launch_bounds__(kDecideThreads) compact_kernel(int n, const uint8_t* mask,
                                                                 const double* x, int32_t* Fidx,
                                                                 int32_t* Gidx, double* xF,
                                                                 DevState* st) {
  __shared__ int s_cnt[32], s_wF[32], s_wG[32];
  __shared__ int s_carryF, s_carryG;
  if (threadIdx.x == 0) {
    s_carryF = 0;
    s_carryG = 0;
  }
  __syncthreads();
  block_compact(n, mask, Fidx, Gidx, s_wF, s_wG, s_cnt, &s_carryF, &s_carryG);
  const int f = s_carryF;
  for (int a = threadIdx.x; a < f; a += blockDim.x) xF[a] = x[Fidx[a]];
  if (threadIdx.x == 0) {
    st->f = f;
    st->g = s_carryG;
  }
}

cudaError_t launch_compact(int n, const uint8_t* mask, const double* x, int32_t* Fidx,
                           int32_t* Gidx, double* xF, DevState* st, cudaStream_t s) {
  compact_kernel<<<1, kDecideThreads, 0, s>>>(n, mask, x, Fidx, Gidx, xF, st);
  return cudaGetLastError();
}

cudaError_t launch_decide(int n, uint8_t* mask, const double* x, const double* y, int32_t* Fidx,
                          int32_t* Gidx, DevState* st, TraceRec* trace, int trace_cap,
                          cudaStream_t s, const cudaGraphConditionalHandle* loop, int32_t* pos,
                          int32_t* Fs, double* xs) {
  const size_t smem = pos != nullptr ? kTailSortSmem : 0;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(decide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  return launch_pdl(decide_kernel, dim3(1), dim3(kDecideThreads), smem, s, n, mask, x, y, Fidx, Gidx, st, trace,
                    trace_cap, loop ? *loop : cudaGraphConditionalHandle{}, loop ? 1 : 0, pos, Fs, xs);
  return cudaGetLastError();
}

// --------------------------------------------------------- dual (a7, a8)
// Warps over G: y_j = sum_a G[j, Fidx[a]] x_F[a] - c_j, from the UNCLAMPED
// x_F (reading c3), then zeroing.  Threads over F: scatter the zeroed x_F.
//
// Fused count + exchange (inflist != nullptr, the pivot loop): every entry
// found infeasible after the zeroing (x_i < 0 for i in F, y_j < 0 for j in
// G -- the count of P:90 over the same snapshot as the decide kernel's pass)
// is appended to inflist through a per-CTA shared-memory list (one global
// atomic per CTA); the largest such index is a block max, then one atomicMax.
// The last CTA to finish (a ticket after a release fence) takes the branch of
// P:89-101 and flips the listed entries (block exchange) or only the
// largest one (single exchange); decide then only compacts and orders
// the new F.  (The dual kernel never reads mask, so flipping it in its own
// last CTA cannot race with the other CTAs.)
constexpr int kDualThreads = 256;
constexpr int kDualList = 512;  // per-CTA infeasible list; overflow goes straight to global

__device__ __forceinline__ void dual_note_infeasible(int i, int* s_n, int* s_list, DevState* st,
                                                     int32_t* inflist) {
  const int slot = atomicAdd(s_n, 1);
  if (slot < kDualList) s_list[slot] = i;
  else inflist[atomicAdd(&st->inf_count, 1)] = i;
}

__global__ void __launch_bounds__(kDualThreads) dual_kernel(
    int n, const double* __restrict__ G, int ldg, const double* __restrict__ c,
    const int32_t* __restrict__ Fidx, const int32_t* __restrict__ Gidx,
    const double* __restrict__ xF, uint8_t* __restrict__ mask, double* __restrict__ x,
    double* __restrict__ y, double tol, DevState* st, const int32_t* __restrict__ Fs,
    const double* __restrict__ xs, int32_t* __restrict__ inflist) {
  __shared__ int s_n, s_lastinf, s_base, s_islast, s_branch, s_k;
  __shared__ int s_list[kDualList];
  const bool fused = inflist != nullptr;
  if (threadIdx.x == 0) {
    s_n = 0;
    s_lastinf = -1;
  }
  __syncthreads();
  // Before waiting for the back substitution (PDL: it lets this grid start
  // once it runs): gather this warp's first G row entries G[j, F] into
  // registers -- G, F and the sets come from earlier kernels (decide).
  // With the factor-reuse views (Fs, xs: x_F scattered by index, zero on G
  // -- decide zeroes the G entries, the back substitution writes F), row j
  // of G is streamed WHOLE with 16-byte loads against xs: the same DRAM
  // sectors as gathering its F entries (about two of the four doubles of
  // every sector are in F), read in order; the G terms add exact zeros.
  constexpr int PF = 8;  // prefetched double2 per lane
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int f = st->f, g = st->g;
  const int n2 = n >> 1;
  // (dense rows only when G streams from DRAM: for a small, L2-resident G the
  // F-entry gathers read half the bytes -- config 1: 43 vs 61 us)
  const bool dense = Fs != nullptr && n >= 2048;
  const bool pre = dense && !st->done && gwarp < g;
  double2 pg[PF];
#pragma unroll
  for (int k = 0; k < PF; ++k) pg[k] = make_double2(0.0, 0.0);
  if (pre) {
    const double2* G2 = reinterpret_cast<const double2*>(G + (size_t)Gidx[gwarp] * ldg);
#pragma unroll
    for (int k = 0; k < PF; ++k)
      if (lane + 32 * k < n2) pg[k] = __ldcs(&G2[lane + 32 * k]);
  }
  // (sparse rows: the first row's F entries G[j, Fs[a]] gathered ahead instead)
  constexpr int PS = 16;
  const bool pres = Fs != nullptr && !dense && !st->done && gwarp < g;
  double ps[PS];
  int pi[PS];
#pragma unroll
  for (int k = 0; k < PS; ++k) {
    pi[k] = 0;
    ps[k] = 0.0;
  }
  if (pres) {
    const double* Gj = G + (size_t)Gidx[gwarp] * ldg;
#pragma unroll
    for (int k = 0; k < PS; ++k) {
      const int a = lane + 32 * k;
      if (a < f) {
        pi[k] = __ldg(&Fs[a]);
        ps[k] = Gj[pi[k]];
      }
    }
  }
  pdl_wait();
  const int status = st->status;
  if (status != 0) {
    if (status == 7) {  // NOT_PD: the solve failed, x = 0 (as the oracle)
      for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        x[i] = 0.0;
    }
    return;
  }
  if (st->done) return;
  const double2* __restrict__ X2 = reinterpret_cast<const double2*>(xs);
  // the prefetched entries (then dead)
  double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
  int pa = lane;
  if (pres) {
#pragma unroll
    for (int k = 0; k < PS; k += 4) {
      const int a0 = lane + 32 * k;
      if (a0 + 96 < f) {
        p0 = fma(ps[k], xs[pi[k]], p0);
        p1 = fma(ps[k + 1], xs[pi[k + 1]], p1);
        p2 = fma(ps[k + 2], xs[pi[k + 2]], p2);
        p3 = fma(ps[k + 3], xs[pi[k + 3]], p3);
      } else {  // the tail (p0), then nothing is left
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (a0 + 32 * q < f) p0 = fma(ps[k + q], xs[pi[k + q]], p0);
      }
    }
    pa = (lane + 32 * (PS - 4) + 96 < f) ? lane + 32 * PS : f;  // (continue after a full last group)
  }
  if (pre) {
#pragma unroll
    for (int k = 0; k < PF; ++k) {
      if (lane + 32 * k < n2) {
        const double2 xv = __ldg(&X2[lane + 32 * k]);
        p0 = fma(pg[k].x, xv.x, p0);
        p1 = fma(pg[k].y, xv.y, p1);
      }
    }
  }
  double below = 0.0, above = INFINITY;
  for (int jj = gwarp; jj < g; jj += nwarps) {
    const int j = Gidx[jj];
    const double* Gj = G + (size_t)j * ldg;
    // four independent partial sums: four loads of G_j (and of Fidx, x_F,
    // which every warp shares through L1) in flight per lane.  With a
    // permuted factorization order (Fs != nullptr) the sum runs over F in
    // index order (Fs) with x_F scattered to xs, so G_j is read in order.
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int a = lane;
    if (dense) {
      const double2* __restrict__ G2 = reinterpret_cast<const double2*>(Gj);
      int t = lane;
      if (jj == gwarp && pre) {
        s0 = p0;
        s1 = p1;
        t = lane + 32 * PF;
      }
      // eight 16-byte loads of the row in flight per lane (a warp streams a
      // whole 64 KB row: its memory-level parallelism sets the pace)
      for (; t + 32 * 7 < n2; t += 32 * 8) {
        double2 gv[8], xv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) gv[u] = __ldcs(&G2[t + 32 * u]);
#pragma unroll
        for (int u = 0; u < 8; ++u) xv[u] = __ldg(&X2[t + 32 * u]);
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
          s0 = fma(gv[u].x, xv[u].x, s0);
          s1 = fma(gv[u].y, xv[u].y, s1);
          s2 = fma(gv[u + 1].x, xv[u + 1].x, s2);
          s3 = fma(gv[u + 1].y, xv[u + 1].y, s3);
        }
      }
      for (; t < n2; t += 32) {
        const double2 g0 = __ldcs(&G2[t]), x0 = __ldg(&X2[t]);
        s0 = fma(g0.x, x0.x, s0);
        s1 = fma(g0.y, x0.y, s1);
      }
      if ((n & 1) && lane == 0) s0 = fma(Gj[n - 1], xs[n - 1], s0);
    } else if (Fs != nullptr) {  // F in index order (Fs) against x scattered to xs: G_j read in order
      if (jj == gwarp && pres) {
        s0 = p0;
        s1 = p1;
        s2 = p2;
        s3 = p3;
        a = pa;
      }
#pragma unroll 4
      for (; a + 96 < f; a += 128) {
        const int i0 = __ldg(&Fs[a]), i1 = __ldg(&Fs[a + 32]), i2 = __ldg(&Fs[a + 64]), i3 = __ldg(&Fs[a + 96]);
        s0 = fma(Gj[i0], xs[i0], s0);
        s1 = fma(Gj[i1], xs[i1], s1);
        s2 = fma(Gj[i2], xs[i2], s2);
        s3 = fma(Gj[i3], xs[i3], s3);
      }
      for (; a < f; a += 32) {
        const int i = __ldg(&Fs[a]);
        s0 = fma(Gj[i], xs[i], s0);
      }
    } else {
      for (; a + 96 < f; a += 128) {
        const int i0 = __ldg(&Fidx[a]), i1 = __ldg(&Fidx[a + 32]), i2 = __ldg(&Fidx[a + 64]), i3 = __ldg(&Fidx[a + 96]);
        s0 = fma(Gj[i0], __ldg(&xF[a]), s0);
        s1 = fma(Gj[i1], __ldg(&xF[a + 32]), s1);
        s2 = fma(Gj[i2], __ldg(&xF[a + 64]), s2);
        s3 = fma(Gj[i3], __ldg(&xF[a + 96]), s3);
      }
      for (; a < f; a += 32) s0 = fma(Gj[__ldg(&Fidx[a])], __ldg(&xF[a]), s0);
    }
    const double s = warp_sum((s0 + s1) + (s2 + s3));
    if (lane == 0) {
      const double v = s - c[j];
      const double av = fabs(v);
      if (av < tol) {
        below = fmax(below, av);
        y[j] = 0.0;
      } else {
        above = fmin(above, av);
        y[j] = v;
      }
      x[j] = 0.0;
      if (fused && v < 0.0 && av >= tol) {  // y_j < 0 after the zeroing
        dual_note_infeasible(j, &s_n, s_list, st, inflist);
        atomicMax(&s_lastinf, j);
      }
    }
  }
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < f; a += gridDim.x * blockDim.x) {
    const int i = Fidx[a];
    const double v = xF[a];
    const double av = fabs(v);
    if (av < tol) {
      below = fmax(below, av);
      x[i] = 0.0;
    } else {
      above = fmin(above, av);
      x[i] = v;
      if (fused && v < 0.0) {  // x_i < 0 after the zeroing
        dual_note_infeasible(i, &s_n, s_list, st, inflist);
        atomicMax(&s_lastinf, i);
      }
    }
    y[i] = 0.0;
  }
  // trace extremes: warp, then block, then ONE atomic pair per block (a
  // global atomic per warp on the same two words serialised ~10 us here)
  __shared__ double s_below[8], s_above[8];
  below = warp_max(below);
  above = warp_min(above);
  const int wid = threadIdx.x >> 5;
  if (lane == 0) {
    s_below[wid] = below;
    s_above[wid] = above;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    double bl = lane < (int)(blockDim.x >> 5) ? s_below[lane] : 0.0;
    double ab = lane < (int)(blockDim.x >> 5) ? s_above[lane] : INFINITY;
    bl = warp_max(bl);
    ab = warp_min(ab);
    if (lane == 0) {
      if (bl > 0.0) atomicMax(&st->below_bits, dbits(bl));
      if (ab < INFINITY) atomicMin(&st->above_bits, dbits(ab));
    }
  }
  if (!fused) {
    if (blockIdx.x == 0 && threadIdx.x == 0) st->iter += 1;
    return;
  }
  // (the __syncthreads above also published s_n / s_list / s_lastinf)
  const int nloc = min(s_n, kDualList);
  if (threadIdx.x == 0) {
    s_base = nloc > 0 ? atomicAdd(&st->inf_count, nloc) : 0;
    if (s_lastinf >= 0) atomicMax(&st->inf_last1, s_lastinf + 1);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nloc; e += blockDim.x) inflist[s_base + e] = s_list[e];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();  // release: this CTA's x, y, list entries before its ticket
    s_islast = atomicAdd(&st->dual_ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_islast) return;
  __threadfence();  // acquire: every CTA's entries
  if (threadIdx.x == 0) {
    st->iter += 1;  // (the completed solve of this iteration, reading c11)
    const int kk = atomicAdd(&st->inf_count, 0);
    const int branch = choose_branch(st, kk);
    st->decided = 1;
    s_branch = branch;
    s_k = kk;
    s_lastinf = atomicAdd(&st->inf_last1, 0) - 1;
    st->inf_count = 0;  // (ready for the next iteration: every CTA is done)
    st->inf_last1 = 0;
    st->dual_ticket = 0u;
  }
  __syncthreads();
  const int branch = s_branch;
  if (branch == 0 || branch == 1) {  // block exchange of every infeasible entry
    for (int e = threadIdx.x; e < s_k; e += blockDim.x) {
      const int i = __ldcg(&inflist[e]);
      mask[i] = mask[i] ? 0 : 1;
    }
  } else if (branch == 2 && threadIdx.x == 0) {  // single exchange of the largest index
    const int i = s_lastinf;
    mask[i] = mask[i] ? 0 : 1;
  }
}

cudaError_t launch_dual(int n, const double* G, int ldg, const double* c, const int32_t* Fidx,
                        const int32_t* Gidx, const double* xF, uint8_t* mask, double* x,
                        double* y, double tol, DevState* st, int sm_count, cudaStream_t s,
                        const int32_t* Fs, const double* xs, int32_t* inflist) {
  int blocks = (n + 7) / 8;  // one warp per G index upper bound
  if (blocks > sm_count * 8) blocks = sm_count * 8;
  if (blocks < 1) blocks = 1;
  return launch_pdl(dual_kernel, dim3(blocks), dim3(kDualThreads), 0, s, n, G, ldg, c, Fidx, Gidx, xF, mask, x, y,
                    tol, st, Fs, xs, inflist);
}

// --------------------------------------------- NOT_PD fallback
__global__ void fallback_prep_kernel(DevState* st) {
  st->status = 0;
  st->done = 1;  // the LSQR kernels take the current F as the final one
}
__global__ void __launch_bounds__(256) fallback_fixup_kernel(int n, const int32_t* __restrict__ Fidx,
                                                             const double* __restrict__ xl, double* __restrict__ xF,
                                                             double* __restrict__ xs, DevState* st) {
  const int f = st->f;
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < f; a += gridDim.x * blockDim.x) xF[a] = xl[Fidx[a]];
  if (xs != nullptr)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) xs[i] = xl[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->done = 0;
    st->lsqr_fallbacks += 1;
    st->keep_none = 1;  // the failed factor's prefix is not reused by the next decide
  }
}
cudaError_t launch_fallback_prep(DevState* st, cudaStream_t s) {
  fallback_prep_kernel<<<1, 1, 0, s>>>(st);
  return cudaGetLastError();
}
cudaError_t launch_fallback_fixup(int n, const int32_t* Fidx, const double* xl, double* xF, double* xs,
                                  DevState* st, cudaStream_t s) {
  int blocks = (n + 255) / 256;
  if (blocks > 64) blocks = 64;
  fallback_fixup_kernel<<<blocks, 256, 0, s>>>(n, Fidx, xl, xF, xs, st);
  return cudaGetLastError();
}

}  // namespace nnls
