// batched.cu -- the whole block-principal-pivoting solve of one small problem
// per CTA, for batches of independent problems (BASELINE config 4: 65536
// problems of 128 x 64, 20% dense; "one warp-group per problem").
//
// Two kernels, one 128-thread CTA per problem each (grid-stride over the
// batch); everything but the Gram lives in shared memory.  Steps, following
// PAPER.md:
//   batched_kernel (the pivot loop):
//   a1 Gram  G_ij = sum over rows set in mask_i & mask_j (a column
//                    view of per-column row bitmasks), increasing row order,
//                    separate multiply/add -> the oracle's terms, order and
//                    roundings (bit-identical); packed, in a per-CTA global
//                    scratch that stays L2-resident, so the CSR's smem region
//                    is reused by the factor (~24 KB per problem).
//   a2 init, a3 decide/exchange, a4 compaction (ballot)
//   a5 Cholesky of the bordered [G_FF; c_F^T], LEFT-looking by columns in the
//                    oracle's jki order (bit-identical factor) on warp 0
//                    alone (a lane owns two rows; one __syncwarp per column,
//                    the other warps wait once)
//   a6 back substitution L^T x = z by a column sweep on one warp (lane k
//                    owns z_k; its summation order differs from the oracle's)
//   a7/a8 dual y_G = G_GF x_F - c_G (oracle order per entry), zeroing
//   NEXT-2 (lsqr_mode 3) the condition estimate of the final factor on warp 0
//   batched_lsqr_kernel:
//   a10 LSQR on the final F on all four warps (thread r owns row r,
//                    2-4 threads per F column; three CTA barriers per
//                    iteration), A restricted to F (rows stored F entries
//                    first)
//   a11 report (objective, KKT of Eq. 3)
// Problems are independent: CTAs grid-stride over the batch; no inter-CTA
// communication.
#include <cuda_runtime.h>
#include <math.h>

#include "common.cuh"
#include "kernels.cuh"

namespace nnls {

namespace {
constexpr int BT = 128;  // one warp-group per problem

__device__ __forceinline__ int pk(int i, int j) {  // packed lower index, any order
  return i >= j ? i * (i + 1) / 2 + j : j * (j + 1) / 2 + i;
}

// Kernel A's shared memory: the phase-1 region (CSR, column view, b: load,
// Gram) and the phase-2 region (bordered factor, pivot vectors) overlap --
// A is not needed after the Gram (which goes to a per-CTA global scratch,
// L2-resident) -- so ~24 KB per problem at config 4: 9 problems per SM.
struct Lay {
  // byte offsets
  size_t c;                                         // persistent: c (n)
  size_t rv, bb, cm, co, rp, ci, crow, cpos;        // phase 1
  size_t L, colk, xF, x, y, Fidx, Gidx, mk;         // phase 2
  size_t bytes;
};
__host__ __device__ inline size_t al16(size_t v) { return (v + 15) & ~(size_t)15; }
__host__ __device__ inline Lay layout(int m, int n, int nnz_max) {
  Lay L;
  const int W = (m + 31) / 32;
  size_t o = 0;
  L.c = o; o = al16(o + 8 * (size_t)n);
  const size_t base = o;
  L.rv = o; o = al16(o + 8 * (size_t)nnz_max);
  L.bb = o; o = al16(o + 8 * (size_t)m);
  L.cm = o; o = al16(o + 4 * (size_t)n * W);
  L.co = o; o = al16(o + 4 * (size_t)(n + 1));
  L.rp = o; o = al16(o + 4 * (size_t)(m + 1));
  L.ci = o; o = al16(o + (size_t)nnz_max);
  L.crow = o; o = al16(o + (size_t)nnz_max);
  L.cpos = o; o = al16(o + 2 * (size_t)nnz_max);
  const size_t end1 = o;
  o = base;
  L.L = o; o = al16(o + 8 * (size_t)(n + 1) * (n + 2) / 2);
  L.colk = o; o = al16(o + 8 * (size_t)(n + 1));
  L.xF = o; o = al16(o + 8 * (size_t)(n + 1));
  L.x = o; o = al16(o + 8 * (size_t)n);
  L.y = o; o = al16(o + 8 * (size_t)n);
  L.Fidx = o; o = al16(o + 4 * (size_t)n);
  L.Gidx = o; o = al16(o + 4 * (size_t)n);
  L.mk = o; o = al16(o + (size_t)n);
  L.bytes = end1 > o ? end1 : o;
  return L;
}

__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  return (red[0] + red[1]) + (red[2] + red[3]);
}
__device__ double block_min(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_min(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  return fmin(fmin(red[0], red[1]), fmin(red[2], red[3]));
}
__device__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  return fmax(fmax(red[0], red[1]), fmax(red[2], red[3]));
}
// next packed-lower position (i, j) -> (i, j + step), wrapping rows
__device__ __forceinline__ void pk_step(int& i, int& j, int step) {
  j += step;
  while (j > i) {
    j -= i + 1;
    ++i;
  }
}
}  // namespace

// Debug hook (not part of the ABI): accumulated clock64 cycles per phase of
// CTA 0's problems, enabled by nnls_debug_batched_profile(ptr).
__device__ long long* g_batch_prof = nullptr;
#define BP_MARK(slot)                                                      \
  do {                                                                     \
    if (g_batch_prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {  \
      const long long t_ = clock64();                                      \
      g_batch_prof[slot] += t_ - bp_t;                                     \
      bp_t = t_;                                                           \
    }                                                                      \
  } while (0)

__global__ void __launch_bounds__(BT, 9) batched_kernel(BatchArgs a, int nnz_max) {
  long long bp_t = clock64();
  extern __shared__ __align__(16) double sm[];
  unsigned char* smb = reinterpret_cast<unsigned char*>(sm);
  const int m = a.m, n = a.n, W = (m + 31) / 32;
  const Lay Ly = layout(m, n, nnz_max);
  double* c = reinterpret_cast<double*>(smb + Ly.c);
  double* rv = reinterpret_cast<double*>(smb + Ly.rv);
  double* bb = reinterpret_cast<double*>(smb + Ly.bb);
  unsigned* cm = reinterpret_cast<unsigned*>(smb + Ly.cm);
  int* co = reinterpret_cast<int*>(smb + Ly.co);
  int* rp = reinterpret_cast<int*>(smb + Ly.rp);
  uint8_t* ci = smb + Ly.ci;
  uint8_t* crow = smb + Ly.crow;
  uint16_t* cpos = reinterpret_cast<uint16_t*>(smb + Ly.cpos);
  double* L = reinterpret_cast<double*>(smb + Ly.L);
  double* colk = reinterpret_cast<double*>(smb + Ly.colk);
  double* xF = reinterpret_cast<double*>(smb + Ly.xF);
  double* x = reinterpret_cast<double*>(smb + Ly.x);
  double* y = reinterpret_cast<double*>(smb + Ly.y);
  int* Fidx = reinterpret_cast<int*>(smb + Ly.Fidx);
  int* Gidx = reinterpret_cast<int*>(smb + Ly.Gidx);
  uint8_t* mk = smb + Ly.mk;
  // the Gram of the current problem: per-CTA global scratch (L2-resident)
  double* G = a.gram + (size_t)blockIdx.x * ((size_t)n * (n + 1) / 2);
  __shared__ int s_last, s_f, s_bad;
  __shared__ unsigned s_bF[BT / 32], s_bG[BT / 32];
  __shared__ int s_scan[BT / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double tol = a.tol;

  if (a.guard && *(volatile const int*)a.guard) return;  // invalid input (pipelined path)
  for (int prob = blockIdx.x; prob < a.batch; prob += gridDim.x) {
    // ---------------------------------------------------------- load
    const int64_t e0 = a.nnz_off[prob];
    const int nz = (int)(a.nnz_off[prob + 1] - e0);
    for (int r = tid; r <= m; r += BT) rp[r] = a.rowptr[(size_t)prob * (m + 1) + r];
    for (int e = tid; e < nz; e += BT) ci[e] = (uint8_t)a.colind[e0 + e];
    for (int r = tid; r < m; r += BT) bb[r] = a.b[(size_t)prob * m + r];
    for (int q = tid; q < n * W; q += BT) cm[q] = 0u;
    __syncthreads();
    BP_MARK(0);  // load
    // column view: row bitmasks, counts (block scan), row lists in row order
    for (int r = tid; r < m; r += BT)
      for (int e = rp[r]; e < rp[r + 1]; ++e) atomicOr(&cm[(r >> 5) * n + ci[e]], 1u << (r & 31));
    __syncthreads();
    {
      // each thread owns a contiguous run of columns; block-wide exclusive scan
      const int per = (n + BT - 1) / BT;
      const int j0 = tid * per, j1 = min(n, j0 + per);
      int run = 0;
      for (int j = j0; j < j1; ++j)
        for (int q = 0; q < W; ++q) run += __popc(cm[q * n + j]);
      int incl = run;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int yv = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += yv;
      }
      if (lane == 31) s_scan[wid] = incl;
      __syncthreads();
      int base = 0;
      for (int q = 0; q < wid; ++q) base += s_scan[q];
      int acc = base + incl - run;
      for (int j = j0; j < j1; ++j) {
        co[j] = acc;
        for (int q = 0; q < W; ++q) acc += __popc(cm[q * n + j]);
      }
      if (tid == BT - 1) co[n] = base + incl;
    }
    __syncthreads();
    for (int r = tid; r < m; r += BT) {
      const int wr = r >> 5;
      const unsigned below = (1u << (r & 31)) - 1u;
      for (int e = rp[r]; e < rp[r + 1]; ++e) {
        const int j = ci[e];
        int rank = co[j];
        for (int q = 0; q < wr; ++q) rank += __popc(cm[q * n + j]);
        rank += __popc(cm[wr * n + j] & below);
        crow[rank] = (uint8_t)r;
        cpos[rank] = (uint16_t)e;
        rv[rank] = a.vals[e0 + e];  // values in COLUMN order (the Gram reads them by rank)
      }
    }
    __syncthreads();
    BP_MARK(1);  // column view
    // ---------------------------------------------------------- a1 Gram, c
    // rows i and n-1-i are folded (i+1 + n-i = n+1 pairs per fold): the work
    // index decodes without a square root
    {
      const int nf = (n + 1) / 2, np1 = n + 1;
      for (int wk = tid; wk < nf * np1; wk += BT) {
        const int fo = wk / np1, k = wk - fo * np1;
        const int i1 = fo, i2 = n - 1 - fo;
        int i, j;
        if (k <= i1) {
          i = i1;
          j = k;
        } else {
          if (i2 == i1) continue;  // odd n: the middle row is alone
          i = i2;
          j = k - i1 - 1;
        }
        double sacc = 0.0;
        int ki = co[i], kj = co[j];
        for (int wq = 0; wq < W; ++wq) {
          const unsigned mi = cm[wq * n + i], mj = cm[wq * n + j];
          unsigned both = mi & mj;
          while (both) {
            const int bpos = __ffs(both) - 1;
            const unsigned bl = (1u << bpos) - 1u;
            const double vi = rv[ki + __popc(mi & bl)];
            const double vj = rv[kj + __popc(mj & bl)];
            sacc = __dadd_rn(sacc, __dmul_rn(vi, vj));
            both &= both - 1u;
          }
          ki += __popc(mi);
          kj += __popc(mj);
        }
        G[i * (i + 1) / 2 + j] = sacc;
      }
    }
    for (int j = tid; j < n; j += BT) {
      double sacc = 0.0;
      for (int t = co[j]; t < co[j + 1]; ++t) sacc = __dadd_rn(sacc, __dmul_rn(rv[t], bb[crow[t]]));
      c[j] = sacc;
    }
    // the column view goes to kernel B now (phase 2 overwrites it)
    {
      int32_t* cvw = reinterpret_cast<int32_t*>(a.colview + (size_t)prob * a.cv_stride);
      uint16_t* cvr = reinterpret_cast<uint16_t*>(cvw + (n + 1));
      for (int j = tid; j <= n; j += BT) cvw[j] = co[j];
      for (int t = tid; t < nz; t += BT) {
        cvr[t] = crow[t];
        cvr[nnz_max + t] = cpos[t];
      }
    }
    __syncthreads();
    BP_MARK(2);  // Gram
    // ---------------------------------------------------------- a2 init
    for (int j = tid; j < n; j += BT) {
      mk[j] = 0;
      x[j] = 0.0;
      const double vv = -c[j];
      y[j] = fabs(vv) < tol ? 0.0 : vv;
    }
    int N = n + 1, p = a.p_max, iter = 0, singles = 0, status = 0, f = 0, not_pd = -1;
    __syncthreads();
    // ---------------------------------------------------------- pivot loop
    for (;;) {
      // a3 count + decide (every thread reaches the same decision)
      bool inf = false;
      if (tid < n) inf = mk[tid] ? (x[tid] < 0.0) : (y[tid] < 0.0);
      if (tid == 0) s_last = -1;
      __syncthreads();
      if (inf) atomicMax(&s_last, tid);
      const int k = __syncthreads_count(inf);
      const int last = s_last;
      if (k == 0) break;
      if (iter >= a.max_iter) {
        status = 8;
        break;
      }
      int branch;
      if (k < N) {
        N = k;
        p = a.p_max;
        branch = 0;
      } else if (p > 0) {
        p -= 1;
        branch = 1;
      } else {
        singles += 1;
        branch = 2;
      }
      if (tid < n && ((branch == 2) ? (tid == last) : inf)) mk[tid] ^= 1;
      __syncthreads();
      // a4 compaction (n <= BT)
      const bool inF = (tid < n) && mk[tid];
      const bool inG = (tid < n) && !mk[tid];
      const unsigned bF = __ballot_sync(kFull, inF);
      const unsigned bG = __ballot_sync(kFull, inG);
      if (lane == 0) {
        s_bF[wid] = bF;
        s_bG[wid] = bG;
      }
      __syncthreads();
      {
        const unsigned lt = (1u << lane) - 1u;
        int offF = 0, offG = 0;
        for (int q = 0; q < wid; ++q) {
          offF += __popc(s_bF[q]);
          offG += __popc(s_bG[q]);
        }
        if (inF) Fidx[offF + __popc(bF & lt)] = tid;
        if (inG) Gidx[offG + __popc(bG & lt)] = tid;
      }
      if (tid == 0) {
        int ff = 0;
        for (int q = 0; q < BT / 32; ++q) ff += __popc(s_bF[q]);
        s_f = ff;
      }
      __syncthreads();
      f = s_f;
      BP_MARK(3);  // decide + compaction
      // a5 Cholesky of the bordered (f+1) x (f+1) matrix [G_FF; c_F^T], packed
      // lower (no (f, f) entry)
      const int fa = f + 1;
      const int ne = fa * (fa + 1) / 2 - 1;  // entries (i, j), j <= i, j < f
      {
        int i = 0, jx = 0;
        pk_step(i, jx, tid);
        for (int e = tid; e < ne; e += BT) {
          double val = (i < f) ? G[pk(Fidx[i], Fidx[jx])] : c[Fidx[jx]];
          L[e] = val;
          pk_step(i, jx, BT);
        }
      }
      // left-looking by columns (the oracle's jki order per entry, so the
      // factor is bit-identical) on warp 0 alone (f <= n <= 64: lane owns rows
      // jj+1+lane and jj+33+lane of step jj): in step jj the owner of row
      // i > jj finishes L(i, jj) with a sequential dot in increasing k and
      // subtracts L(i, jj)^2 from its diagonal entry (the pivot's sum, kept
      // running in place: the same terms in the same order as the oracle's
      // dot); the owner of row jj+1 then takes the square root of the now
      // complete next pivot -> one warp barrier per column, the other warps
      // wait once
      __syncthreads();  // the gathered L
      if (wid == 0) {
        if (lane == 0) {
          s_bad = -1;
          if (f > 0) {
            const double d = L[0];
            if (!(d > 0.0) || d < 1e-300 || !isfinite(d)) s_bad = 0;
            L[0] = sqrt(d);
          }
        }
        __syncwarp();
        for (int jj = 0; jj < f; ++jj) {
          const int rj = jj * (jj + 1) / 2;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int i = jj + 1 + lane + 32 * h;
            if (i <= f) {
              const int ri = i * (i + 1) / 2;
              double sacc = L[ri + jj];
              for (int k = 0; k < jj; ++k) sacc = __dsub_rn(sacc, __dmul_rn(L[ri + k], L[rj + k]));
              sacc = sacc / L[rj + jj];
              L[ri + jj] = sacc;
              if (i < f) {  // the pivot's running sum: d_i -= L(i,jj)^2 (increasing k, as the oracle)
                const double d = __dsub_rn(L[ri + i], __dmul_rn(sacc, sacc));
                if (i == jj + 1) {  // the next pivot, complete
                  if (!(d > 0.0) || d < 1e-300 || !isfinite(d)) atomicMin(&s_bad, i);
                  L[ri + i] = sqrt(d);
                } else {
                  L[ri + i] = d;
                }
              }
            }
          }
          __syncwarp();
        }
      }
      __syncthreads();
      {
        const int bad = s_bad;
        if (bad >= 0) {
          status = 7;
          not_pd = bad;
        }
      }
      if (status == 7) {
        for (int j = tid; j < n; j += BT) x[j] = 0.0;
        __syncthreads();
        break;
      }
      BP_MARK(4);  // gather + Cholesky
      // a6 back substitution L^T x_F = z (z = row f): column sweep on warp 0
      if (wid == 0) {
        double zr[4];  // lane owns k = lane + 32 q (f <= 128)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int kq = lane + 32 * q;
          zr[q] = kq < f ? L[f * (f + 1) / 2 + kq] : 0.0;
        }
        for (int i = lane; i < f; i += 32) colk[i] = 1.0 / L[i * (i + 1) / 2 + i];
        __syncwarp();
        for (int i = f - 1; i >= 0; --i) {
          const int qi = i >> 5, li = i & 31;
          double zi = 0.0;
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (q == qi) zi = zr[q];
          zi = __shfl_sync(kFull, zi, li);
          const double xi = zi * colk[i];
          if (lane == 0) xF[i] = xi;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int kq = lane + 32 * q;
            if (kq < i) zr[q] = __dsub_rn(zr[q], __dmul_rn(L[i * (i + 1) / 2 + kq], xi));
          }
        }
      }
      __syncthreads();
      BP_MARK(5);  // back substitution
      // scatter x_F, x_G = 0
      for (int aa = tid; aa < n; aa += BT) {
        if (aa < f) x[Fidx[aa]] = xF[aa];
        else x[Gidx[aa - f]] = 0.0;
      }
      __syncthreads();
      // a7 y_G = G_GF x_F - c_G (from the unclamped x_F), y_F = 0; a8 zeroing
      if (tid < n) {
        const int j = tid;
        if (mk[j]) {
          y[j] = 0.0;
        } else {
          double sacc = 0.0;
          for (int aa = 0; aa < f; ++aa) sacc = __dadd_rn(sacc, __dmul_rn(G[pk(j, Fidx[aa])], xF[aa]));
          const double vv = sacc - c[j];
          y[j] = fabs(vv) < tol ? 0.0 : vv;
        }
      }
      __syncthreads();
      if (tid < n && mk[tid] && fabs(x[tid]) < tol) x[tid] = 0.0;
      __syncthreads();
      ++iter;
    }
    BP_MARK(6);  // scatter + dual (+ loop exit)
    // ---------------------------------------------------------- NEXT-2
    // lsqr_mode 3: Hager/Higham estimate of kappa_1((A^T A)_FF) from the
    // final factor (dpocon's estimator, LAPACK dlacn2's steps) on warp 0,
    // vectors in registers (lane l holds entries l and l+32; f <= 64).
    double kappa = 0.0;
    int refined = (status == 0 && f > 0 && (a.lsqr_mode == 1 || a.lsqr_mode == 2)) ? 1 : 0;
    if (a.lsqr_mode == 3 && status == 0 && f > 0) {
      if (wid == 0) {
        // ||M||_1: column j's sum in increasing i (the oracle's order), then the max
        double cs = 0.0;
        for (int jq = lane; jq < f; jq += 32) {
          double t = 0.0;
          for (int i = 0; i < f; ++i) t += fabs(G[pk(Fidx[i], Fidx[jq])]);
          cs = fmax(cs, t);
        }
        const double norm1 = warp_max(cs);
        // B v = M^-1 v: forward L z = v (column sweep: each z_i gets its terms in
        // increasing k, as the oracle), then L^T x = z (column sweep, descending)
        auto applyB = [&](double v0, double v1, double& o0, double& o1) {
          double s0 = v0, s1 = v1;
          for (int j = 0; j < f; ++j) {
            const int rj = j * (j + 1) / 2;
            const double own = (j < 32) ? s0 : s1;
            const double zj = __shfl_sync(kFull, own, j & 31) / L[rj + j];
            if (lane == (j & 31)) {
              if (j < 32) s0 = zj;
              else s1 = zj;
            }
            const int i0 = lane, i1 = lane + 32;
            if (i0 > j && i0 < f) s0 = __dsub_rn(s0, __dmul_rn(L[i0 * (i0 + 1) / 2 + j], zj));
            if (i1 > j && i1 < f) s1 = __dsub_rn(s1, __dmul_rn(L[i1 * (i1 + 1) / 2 + j], zj));
          }
          for (int i = f - 1; i >= 0; --i) {
            const int ri = i * (i + 1) / 2;
            const double own = (i < 32) ? s0 : s1;
            const double xi_ = __shfl_sync(kFull, own, i & 31) / L[ri + i];
            if (lane == (i & 31)) {
              if (i < 32) s0 = xi_;
              else s1 = xi_;
            }
            const int k0 = lane, k1 = lane + 32;
            if (k0 < i) s0 = __dsub_rn(s0, __dmul_rn(L[ri + k0], xi_));
            if (k1 < i) s1 = __dsub_rn(s1, __dmul_rn(L[ri + k1], xi_));
          }
          o0 = (lane < f) ? s0 : 0.0;
          o1 = (lane + 32 < f) ? s1 : 0.0;
        };
        auto asum = [&](double a0, double a1) { return warp_sum(fabs(a0) + fabs(a1)); };
        auto iamax = [&](double a0, double a1) {  // first index of max |v|
          double b = fabs(a0);
          int bi = lane;
          if (lane + 32 < f && fabs(a1) > b) {
            b = fabs(a1);
            bi = lane + 32;
          }
          if (lane >= f) b = -1.0;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(kFull, b, o);
            const int oi = __shfl_xor_sync(kFull, bi, o);
            if (ob > b || (ob == b && oi < bi)) {
              b = ob;
              bi = oi;
            }
          }
          return bi;
        };
        auto sgn = [](double v) { return v >= 0.0 ? 1.0 : -1.0; };
        const double inv_f = 1.0 / (double)f;
        double x0 = lane < f ? inv_f : 0.0, x1 = lane + 32 < f ? inv_f : 0.0, y0, y1;
        applyB(x0, x1, y0, y1);
        double est;
        if (f == 1) {
          est = fabs(__shfl_sync(kFull, y0, 0));
        } else {
          est = asum(y0, y1);
          double xi0 = lane < f ? sgn(y0) : 0.0, xi1 = lane + 32 < f ? sgn(y1) : 0.0;
          applyB(xi0, xi1, y0, y1);
          int jj = iamax(y0, y1), iter = 2;
          for (;;) {
            x0 = (lane == jj) ? 1.0 : 0.0;
            x1 = (lane + 32 == jj) ? 1.0 : 0.0;
            applyB(x0, x1, y0, y1);
            const double est_old = est;
            est = asum(y0, y1);
            const bool diff = (lane < f && sgn(y0) != xi0) || (lane + 32 < f && sgn(y1) != xi1);
            if (!__any_sync(kFull, diff) || est <= est_old) break;
            xi0 = lane < f ? sgn(y0) : 0.0;
            xi1 = lane + 32 < f ? sgn(y1) : 0.0;
            applyB(xi0, xi1, y0, y1);
            const int jlast = jj;
            jj = iamax(y0, y1);
            const double zl = __shfl_sync(kFull, jlast < 32 ? y0 : y1, jlast & 31);
            const double zj = __shfl_sync(kFull, jj < 32 ? y0 : y1, jj & 31);
            if (zl != fabs(zj) && iter < 5) {
              ++iter;
              continue;
            }
            break;
          }
          x0 = lane < f ? ((lane & 1) ? -1.0 : 1.0) * (1.0 + (double)lane / (double)(f - 1)) : 0.0;
          x1 = lane + 32 < f ? (((lane + 32) & 1) ? -1.0 : 1.0) * (1.0 + (double)(lane + 32) / (double)(f - 1))
                             : 0.0;
          applyB(x0, x1, y0, y1);
          const double temp = 2.0 * asum(y0, y1) / (3.0 * (double)f);
          if (temp > est) est = temp;
        }
        if (lane == 0) colk[0] = norm1 * est;
      }
      __syncthreads();
      kappa = colk[0];
      refined = (kappa * 0x1p-52 > a.adaptive_threshold) ? 1 : 0;
      __syncthreads();
    }
    // ---------------------------------------------------------- hand-off
    // the NE solution, F and the counters go to global memory with the
    // column view; batched_lsqr_kernel (a smaller on-chip footprint, so more
    // problems per SM) runs a10/a11
    for (int j = tid; j < n; j += BT) {
      a.x_out[(size_t)prob * n + j] = mk[j] ? x[j] : 0.0;
      a.mask_out[(size_t)prob * n + j] = mk[j];
    }
    if (tid == 0) {
      int32_t* ii = a.info_i + (size_t)prob * kInfoI;
      ii[0] = status;
      ii[1] = iter;
      ii[2] = singles;
      ii[3] = f;
      ii[7] = status == 7 ? not_pd : -1;
      ii[8] = refined;
      ii[9] = 0;
      a.info_d[(size_t)prob * kInfoD + 5] = kappa;
    }
    __syncthreads();
    BP_MARK(7);  // hand-off
    if (g_batch_prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0) g_batch_prof[9] += 1;
  }
}

// a10 LSQR on the final F and a11 report, one problem per 128-thread
// CTA.  A restricted to F is held in shared memory twice, both as SLICED
// ELL (SELL-32) blocks: by rows (thread r owns row r; warp slice w holds its
// 32 rows' F entries entry-major, padded to the slice's longest row) and by
// F columns (a column's entries dealt round-robin to its tpc threads; slices
// of 32 thread slots).  Every value / index load of the two products is then
// one conflict-free wavefront pair, and the column product needs no
// indirection through the row storage; only the gathers of v and u are
// random.  (ncu on the previous CSR/CSC layout: the two products were 78 % of
// the kernel's shared-memory wavefronts, over half of them bank conflicts.)
// Built straight from the global CSR and the pivot kernel's column view;
// a problem whose padded blocks exceed the capacity (very uneven rows) runs
// its products from global memory instead.  The report reads global memory.
struct LLay {
  int ors, ocs, ou, ov, ow, oX, ored;  // double offsets
  int doubles;
  int iri, icr, irof, icof, ifl, ircnt, irp, icp, imk;  // byte offsets in the int area
  int cap;                             // entries per SELL block
  size_t bytes;
};
__host__ __device__ inline LLay llayout(int m, int n, int nnz_max, int cap_pct) {
  LLay L;
  // padded F blocks: ~1.1 nnz_F, nnz_F ~ nnz f/n (config 4: f/n ~ 0.5, up to
  // 0.7); cap_pct = 90 covers every problem of the config-4 batch (measured:
  // 70 % -> 34 ms, 80 % -> 24 ms, 90 % -> 21.8 ms, 100 % -> 22.7 ms per batch);
  // a problem that does not fit takes the global-memory path
  L.cap = ((nnz_max * cap_pct / 100 + 31) / 32) * 32 + 32;  // (sorted slices pad ~10 %)
  int o = 0;
  L.ors = o; o += L.cap;
  L.ocs = o; o += L.cap;
  L.ou = o; o += m;
  L.ov = o; o += n;
  L.ow = o; o += n;
  L.oX = o; o += n;
  L.ored = o; o += 32;
  L.doubles = o;
  int q = 0;  // bytes
  L.iri = q; q += L.cap;                        // row SELL column indices (u8)
  L.icr = q; q += L.cap;                        // column SELL row indices (u8)
  q = (q + 15) & ~15;
  L.irof = q; q += 4 * 12;                      // row slice offsets (<= 8 slices + 1)
  L.icof = q; q += 4 * 8;                       // column slice offsets (4 slices + 1)
  L.ifl = q; q += 4 * (n + 1);                  // F columns, index order
  L.ircnt = q; q += 4 * (m > n ? m : n);        // F entries per row / per F column (sort keys)
  L.irp = q; q += m;                            // rows by decreasing F count (SELL-sigma)
  L.icp = q; q += n;                            // F columns by decreasing length
  L.imk = q; q += n;
  q = (q + 15) & ~15;
  L.bytes = sizeof(double) * (size_t)L.doubles + (size_t)q;
  return L;
}

__global__ void __launch_bounds__(BT, 8) batched_lsqr_kernel(BatchArgs a, int nnz_max) {
  long long bp_t = clock64();
  extern __shared__ double sm[];
  const int m = a.m, n = a.n;
  const LLay Ly = llayout(m, n, nnz_max, a.lsqr_cap_pct);
  double* rS = sm + Ly.ors;
  double* cS = sm + Ly.ocs;
  double* u = sm + Ly.ou;
  double* v = sm + Ly.ov;
  double* w = sm + Ly.ow;
  double* X = sm + Ly.oX;
  double* red = sm + Ly.ored;
  unsigned char* ib = reinterpret_cast<unsigned char*>(sm + Ly.doubles);
  uint8_t* rI = ib + Ly.iri;
  uint8_t* cR = ib + Ly.icr;
  int* roff = reinterpret_cast<int*>(ib + Ly.irof);
  int* coff = reinterpret_cast<int*>(ib + Ly.icof);
  int* fl = reinterpret_cast<int*>(ib + Ly.ifl);
  int* kcnt = reinterpret_cast<int*>(ib + Ly.ircnt);
  uint8_t* rperm = ib + Ly.irp;
  uint8_t* cperm = ib + Ly.icp;
  uint8_t* mk = ib + Ly.imk;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double tol = a.tol;
  __shared__ int s_istop, s_ws[8], s_wc[4], s_over;
  if (a.guard && *(volatile const int*)a.guard) return;  // invalid input (pipelined path)
  const int nsl = (m + 31) / 32;  // row slices (<= 8)
  for (int prob = blockIdx.x; prob < a.batch; prob += gridDim.x) {
    const int64_t e0 = a.nnz_off[prob];
    const int status = a.info_i[(size_t)prob * kInfoI + 0];
    const int f = a.info_i[(size_t)prob * kInfoI + 3];
    const int32_t* rpg = a.rowptr + (size_t)prob * (m + 1);
    const int32_t* gci = a.colind + e0;
    const double* gvl = a.vals + e0;
    const double* bb = a.b + (size_t)prob * m;       // b (global)
    const double* x = a.x_out + (size_t)prob * n;    // the NE x (global; overwritten by the output below)
    const int32_t* cvw = reinterpret_cast<const int32_t*>(a.colview + (size_t)prob * a.cv_stride);
    const uint16_t* cvr = reinterpret_cast<const uint16_t*>(cvw + (n + 1));
    for (int j = tid; j < n; j += BT) {
      mk[j] = a.mask_out[(size_t)prob * n + j];
      v[j] = 0.0;
      X[j] = 0.0;
    }
    if (tid == 0) s_over = 0;
    __syncthreads();
    if (wid == 0) {  // F columns in index order
      int base = 0;
      for (int j0 = 0; j0 < n; j0 += 32) {
        const int j = j0 + lane;
        const bool inF = j < n && mk[j];
        const unsigned bal = __ballot_sync(kFull, inF);
        if (inF) fl[base + __popc(bal & ((1u << lane) - 1u))] = j;
        base += __popc(bal);
      }
      if (lane == 0) fl[n] = base;
    }
    __syncthreads();
    const int nF = fl[n];
    const int tpc = nF <= 32 ? 4 : 2;  // threads per F column
    // ---- row SELL-sigma: rows sorted by decreasing F count (rank = rows
    //      with more entries, ties by index), so a 32-row slice's padding to
    //      its longest row stays small; thread t then owns row rperm[t]
    for (int r = tid; r < m; r += BT) {
      int c = 0;
      for (int e = rpg[r]; e < rpg[r + 1]; ++e) c += mk[gci[e]];
      kcnt[r] = c;
    }
    __syncthreads();
    for (int r = tid; r < m; r += BT) {
      const int c = kcnt[r];
      int rank = 0;
      for (int q = 0; q < m; ++q) {
        const int cq = kcnt[q];
        rank += (cq > c) || (cq == c && q < r);
      }
      rperm[rank] = (uint8_t)r;
    }
    __syncthreads();
    int cntr[2] = {0, 0};
    for (int h = 0; h < 2; ++h) {
      const int t = tid + BT * h;
      if (t < m) cntr[h] = kcnt[rperm[t]];
    }
    for (int h = 0; h < 2; ++h) {
      const int wmax = warp_max_i(cntr[h]);
      if (lane == 0 && wid + 4 * h < nsl) s_ws[wid + 4 * h] = wmax;
    }
    __syncthreads();
    // ---- column SELL: F columns sorted by decreasing length; slot tid =
    //      (group, sub) takes entries k = sub (mod tpc) of its group's column
    for (int g = tid; g < nF; g += BT) kcnt[g] = cvw[fl[g] + 1] - cvw[fl[g]];
    __syncthreads();
    for (int g = tid; g < nF; g += BT) {
      const int c = kcnt[g];
      int rank = 0;
      for (int q = 0; q < nF; ++q) {
        const int cq = kcnt[q];
        rank += (cq > c) || (cq == c && q < g);
      }
      cperm[rank] = (uint8_t)g;
    }
    __syncthreads();
    const int grp = tid / tpc, sub = tid % tpc;
    const bool colgrp = grp < nF;
    const int jc = colgrp ? fl[cperm[grp]] : 0;
    const int c0 = colgrp ? cvw[jc] : 0, c1 = colgrp ? cvw[jc + 1] : 0;
    const int cntc = colgrp ? max(0, (c1 - c0 - sub + tpc - 1) / tpc) : 0;
    {
      const int wmax = warp_max_i(cntc);
      if (lane == 0) s_wc[wid] = wmax;
    }
    __syncthreads();
    if (tid == 0) {
      int o = 0;
      for (int sl = 0; sl < 8; ++sl) {
        if (sl >= nsl) s_ws[sl] = 0;  // (warps with no second slice read width 0)
        roff[sl] = o;
        o += 32 * s_ws[sl];
      }
      roff[8] = o;
      int oc = 0;
      for (int sl = 0; sl < 4; ++sl) {
        coff[sl] = oc;
        oc += 32 * s_wc[sl];
      }
      coff[4] = oc;
      s_over = (o > Ly.cap || oc > Ly.cap) ? 1 : 0;
    }
    __syncthreads();
    const bool sell = !s_over;
    if (sell) {
      for (int h = 0; h < 2; ++h) {
        const int t = tid + BT * h, sl = wid + 4 * h;
        if (sl >= nsl) continue;
        const int r = t < m ? rperm[t] : m;
        const int base = roff[sl] + lane, W = s_ws[sl];
        int k = 0;
        if (r < m)
          for (int e = rpg[r]; e < rpg[r + 1]; ++e) {
            const int j = gci[e];
            if (mk[j]) {
              rS[base + 32 * k] = gvl[e];
              rI[base + 32 * k] = (uint8_t)j;
              ++k;
            }
          }
        for (; k < W; ++k) {
          rS[base + 32 * k] = 0.0;
          rI[base + 32 * k] = 0;
        }
      }
      {
        const int base = coff[wid] + lane, W = s_wc[wid];
        int k = 0;
        for (int t = c0 + sub; t < c1; t += tpc, ++k) {
          cS[base + 32 * k] = gvl[cvr[nnz_max + t]];
          cR[base + 32 * k] = (uint8_t)cvr[t];
        }
        for (; k < W; ++k) {
          cS[base + 32 * k] = 0.0;
          cR[base + 32 * k] = 0;
        }
      }
    }
    __syncthreads();
    BP_MARK(10);  // LSQR kernel: load
    // ---------------------------------------------------------- a10 LSQR
    // All 4 warps.  Thread r owns row r (u); a group of tpc threads owns the
    // F column fl[grp] (v, w, X; the group splits A^T u).  Three CTA barriers
    // per iteration: the norm reductions (|u|^2 | |v|^2, |d|^2, |x|^2) each
    // end with one, and the vectors a thread reads from others were written
    // before it; the stopping test of an iteration is evaluated after the next
    // barrier (it needs only scalars, and x is not touched in between).
    int itn = 0, istop = 0;
    const int mode0 = (status == 0 && f > 0) ? a.lsqr_mode : 0;
    // mode 3 (adaptive): the pivot kernel's condition estimate decided
    const int mode = mode0 == 3 ? (a.info_i[(size_t)prob * kInfoI + 8] ? 1 : 0) : mode0;
    if (mode != 0) {
      const int itn_limit = a.itn_limit > 0 ? a.itn_limit : 4 * f;
      int rslot = 0;  // red[] double-buffering: red[rslot*16 + 4*q + warp]
      auto reduce3 = [&](double v0, double v1, double v2, int nv, double* out) {
        v0 = warp_sum(v0);
        if (nv > 1) v1 = warp_sum(v1);
        if (nv > 2) v2 = warp_sum(v2);
        double* rr = red + rslot * 16;
        if (lane == 0) {
          rr[wid] = v0;
          if (nv > 1) rr[4 + wid] = v1;
          if (nv > 2) rr[8 + wid] = v2;
        }
        __syncthreads();
        out[0] = (rr[0] + rr[1]) + (rr[2] + rr[3]);
        if (nv > 1) out[1] = (rr[4] + rr[5]) + (rr[6] + rr[7]);
        if (nv > 2) out[2] = (rr[8] + rr[9]) + (rr[10] + rr[11]);
        rslot ^= 1;
      };
      // row product s = A_F(r, :) vec (h: the thread's second row when m > 128)
      auto row_dot = [&](int h, const double* vec) {
        const int t = tid + BT * h, sl = wid + 4 * h;
        const int r = t < m ? rperm[t] : m;
        double s0 = 0.0, s1 = 0.0;
        if (sell) {
          const int base = roff[sl] + lane, W = s_ws[sl];
          int k = 0;
          for (; k + 1 < W; k += 2) {
            s0 = fma(rS[base + 32 * k], vec[rI[base + 32 * k]], s0);
            s1 = fma(rS[base + 32 * (k + 1)], vec[rI[base + 32 * (k + 1)]], s1);
          }
          if (k < W) s0 = fma(rS[base + 32 * k], vec[rI[base + 32 * k]], s0);
        } else if (r < m) {
          for (int e = rpg[r]; e < rpg[r + 1]; ++e) {
            const int j = gci[e];
            if (mk[j]) s0 = fma(gvl[e], vec[j], s0);
          }
        }
        return s0 + s1;
      };
      // column product over the F columns: the slot's entries, then the group's sum
      auto col_dot = [&](const double* vec) {
        double s0 = 0.0, s1 = 0.0;
        if (sell) {
          const int base = coff[wid] + lane, W = s_wc[wid];
          int k = 0;
          for (; k + 1 < W; k += 2) {
            s0 = fma(cS[base + 32 * k], vec[cR[base + 32 * k]], s0);
            s1 = fma(cS[base + 32 * (k + 1)], vec[cR[base + 32 * (k + 1)]], s1);
          }
          if (k < W) s0 = fma(cS[base + 32 * k], vec[cR[base + 32 * k]], s0);
        } else if (colgrp) {
          for (int t = c0 + sub; t < c1; t += tpc) s0 = fma(gvl[cvr[nnz_max + t]], vec[cvr[t]], s0);
        }
        double sacc = s0 + s1;
        sacc += __shfl_xor_sync(kFull, sacc, 1);
        if (tpc == 4) sacc += __shfl_xor_sync(kFull, sacc, 2);
        return sacc;
      };
      const bool colown = colgrp && sub == 0;
      double tot[3];
      // beta u = b - A x (mode 2) or b
      double pu = 0.0;
      for (int h = 0; h < 2; ++h) {
        const int t = tid + BT * h;
        if (BT * h >= m) continue;
        const int r = t < m ? rperm[t] : m;
        const double sacc = (mode == 2) ? row_dot(h, x) : 0.0;  // (uniform per warp slice)
        if (r < m) {
          const double uu = bb[r] - sacc;
          u[r] = uu;
          pu += uu * uu;
        }
      }
      reduce3(pu, 0.0, 0.0, 1, tot);  // B: u complete
      double beta = sqrt(tot[0]);
      const double bnorm = beta;
      double ibt = beta > 0.0 ? 1.0 / beta : 0.0;
      // alpha v = A^T u
      double pv = 0.0;
      {
        const double sacc = beta > 0.0 ? col_dot(u) : 0.0;
        if (colown) {
          const double vv = sacc * ibt;
          v[jc] = vv;
          pv = vv * vv;
        }
      }
      reduce3(pv, 0.0, 0.0, 1, tot);  // B: every read of u done
      double alpha = sqrt(tot[0]);
      const double ia0 = alpha > 0.0 ? 1.0 / alpha : 0.0;
      for (int r = tid; r < m; r += BT) u[r] *= ibt;  // own rows
      if (colown) {
        v[jc] *= ia0;
        w[jc] = v[jc];
      }
      __syncthreads();  // v, u complete
      double rhobar = alpha, phibar = beta, anorm = 0.0, ddnorm = 0.0;
      const double ctol = a.conlim > 0.0 ? 1.0 / a.conlim : 0.0;
      if (tid == 0) s_istop = 0;
      if (alpha * beta != 0.0) {
        for (;;) {
          // u' = A v - alpha u (own rows)
          const bool more = itn < itn_limit;
          pu = 0.0;
          if (more)
            for (int h = 0; h < 2; ++h) {
              const int t = tid + BT * h;
              if (BT * h >= m) continue;
              const int r = t < m ? rperm[t] : m;
              const double rd = row_dot(h, v);
              if (r < m) {
                const double uu = rd - alpha * u[r];
                u[r] = uu;
                pu += uu * uu;
              }
            }
          reduce3(pu, 0.0, 0.0, 1, tot);  // B1: u' complete; the previous test visible
          istop = s_istop;
          if (istop != 0) break;
          ++itn;
          beta = sqrt(tot[0]);
          double alpha_new = alpha;
          if (beta > 0.0) {
            ibt = 1.0 / beta;
            anorm = sqrt(anorm * anorm + alpha * alpha + beta * beta);
            // v' = A^T u' / beta - beta v (own columns)
            const double sacc = col_dot(u);
            pv = 0.0;
            if (colown) {
              const double vv = sacc * ibt - beta * v[jc];
              v[jc] = vv;
              pv = vv * vv;
            }
            reduce3(pv, 0.0, 0.0, 1, tot);  // B2: every read of u' done
            alpha_new = sqrt(tot[0]);
            for (int r = tid; r < m; r += BT) u[r] *= ibt;  // own rows
            if (alpha_new > 0.0 && colown) v[jc] *= 1.0 / alpha_new;
          }
          const double rho = sqrt(rhobar * rhobar + beta * beta);
          const double irho = 1.0 / rho;
          const double cs = rhobar * irho, sn = beta * irho;
          const double theta = sn * alpha_new;
          rhobar = -cs * alpha_new;
          const double phi = cs * phibar;
          phibar = sn * phibar;
          const double t1 = phi * irho, t2 = -theta * irho;
          double pd = 0.0, px = 0.0;
          if (colown) {  // own column: w, x
            const double ww = w[jc];
            const double dd = ww * irho;
            pd = dd * dd;
            const double xx = X[jc] + t1 * ww;
            X[jc] = xx;
            w[jc] = v[jc] + t2 * ww;
            px = xx * xx;
          }
          alpha = alpha_new;
          reduce3(pd, px, 0.0, 2, tot);  // B3: v, w, x complete
          ddnorm += tot[0];
          if (tid == 0) {
            const double xnorm = sqrt(tot[1]);
            const double acond = anorm * sqrt(ddnorm);
            const double rnorm = phibar;
            const double arnorm = alpha * fabs(sn * phi);
            const double test1 = bnorm > 0.0 ? rnorm / bnorm : 0.0;
            const double test2 = (anorm * rnorm) > 0.0 ? arnorm / (anorm * rnorm) : 0.0;
            const double test3 = acond > 0.0 ? 1.0 / acond : 0.0;
            const double tt1 = bnorm > 0.0 ? test1 / (1.0 + anorm * xnorm / bnorm) : 0.0;
            const double rtol = a.btol + (bnorm > 0.0 ? a.atol * anorm * xnorm / bnorm : 0.0);
            int st = 0;
            if (itn >= itn_limit) st = 7;
            if (1.0 + test3 <= 1.0) st = 6;
            if (1.0 + test2 <= 1.0) st = 5;
            if (1.0 + tt1 <= 1.0) st = 4;
            if (test3 <= ctol) st = 3;
            if (test2 <= a.atol) st = 2;
            if (test1 <= rtol) st = 1;
            s_istop = st;
          }
        }
      }
      __syncthreads();
    }
    BP_MARK(11);  // LSQR
    // ---------------------------------------------------------- a11 output
    bool infeas = false;
    for (int j = tid; j < n; j += BT) {
      double vv;
      if (!mk[j]) vv = 0.0;
      else if (mode == 1) vv = X[j];
      else if (mode == 2) vv = x[j] + X[j];
      else vv = x[j];
      if (fabs(vv) < tol) vv = 0.0;
      if (vv < 0.0) infeas = true;
      w[j] = vv;  // final x staged in w
      a.x_out[(size_t)prob * n + j] = vv;
    }
    const int any_infeas = __syncthreads_or(infeas);
    double obj = 0.0, mx = INFINITY, my = INFINITY, mc = 0.0, dot = 0.0;
    if (a.kkt) {  // the report over all of A, from global memory (once per problem)
      double po = 0.0;
      for (int r = tid; r < m; r += BT) {
        double sacc = 0.0;
        for (int e = rpg[r]; e < rpg[r + 1]; ++e) sacc = fma(gvl[e], w[gci[e]], sacc);
        const double rr = sacc - bb[r];
        u[r] = rr;
        po += rr * rr;
      }
      obj = block_sum(po, red);
      double lmx = INFINITY, lmy = INFINITY, lmc = 0.0, ld = 0.0;
      for (int j = tid; j < n; j += BT) {
        double sacc = 0.0;
        for (int t = cvw[j]; t < cvw[j + 1]; ++t) sacc = fma(gvl[cvr[nnz_max + t]], u[cvr[t]], sacc);
        const double xj = w[j];
        lmx = fmin(lmx, xj);
        lmy = fmin(lmy, sacc);
        lmc = fmax(lmc, fabs(xj * sacc));
        ld += xj * sacc;
      }
      mx = block_min(lmx, red);
      my = block_min(lmy, red);
      mc = block_max(lmc, red);
      dot = block_sum(ld, red);
    }
    if (tid == 0) {
      int32_t* ii = a.info_i + (size_t)prob * kInfoI;
      ii[4] = itn;
      ii[5] = istop;
      ii[6] = (mode != 0 && any_infeas) ? 1 : 0;
      double* dd = a.info_d + (size_t)prob * kInfoD;
      dd[0] = 0.5 * obj;
      dd[1] = mx;
      dd[2] = my;
      dd[3] = mc;
      dd[4] = dot;
    }
    __syncthreads();
    BP_MARK(12);  // output + KKT
    if (g_batch_prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0) g_batch_prof[13] += 1;
  }
}

cudaError_t batched_debug_set_profile(long long* p) {
  return cudaMemcpyToSymbol(g_batch_prof, &p, sizeof(p));
}

// Validation in two coalesced passes (no warp per row: rows hold ~13
// entries).  The per-row "columns strictly increasing" test is turned into a
// count: over the whole concatenated colind, D = #{g >= 1 : colind[g] <=
// colind[g-1]} (entry pass); a valid batch has such descents only at the
// first entry of a non-empty row, Ds of them (row pass) -> valid iff D == Ds
// (rows partition each problem's entries once rowptr passes its own checks).
// cnt[0] = D, cnt[1] = Ds.
__global__ void validate_entries_kernel(int64_t g_begin, int64_t g_end, int n,
                                        const int32_t* __restrict__ colind,
                                        const double* __restrict__ vals, int* err,
                                        unsigned long long* cnt) {
  // entries [g_begin, g_end) of the (16-byte aligned) arrays
  __shared__ int s_e;
  __shared__ unsigned s_d;
  if (threadIdx.x == 0) {
    s_e = 0;
    s_d = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int e_local = 0;
  unsigned d_local = 0;
  // aligned quads of 4 entries per thread (16-byte colind, 2 x 16-byte vals
  // loads); whole warps iterate together (the shuffle below)
  const int64_t qa = g_begin / 4, qb = (g_end + 3) / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t span = (qb - qa + 31) / 32 * 32;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < span; q += stride) {
    const int64_t g0 = 4 * (qa + q);
    int c[4];
    double v[4];
    if (g0 >= g_begin && g0 + 3 < g_end) {
      const int4 c4 = *reinterpret_cast<const int4*>(colind + g0);
      const double2 v0 = *reinterpret_cast<const double2*>(vals + g0);
      const double2 v1 = *reinterpret_cast<const double2*>(vals + g0 + 2);
      c[0] = c4.x; c[1] = c4.y; c[2] = c4.z; c[3] = c4.w;
      v[0] = v0.x; v[1] = v0.y; v[2] = v1.x; v[3] = v1.y;
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool in = g0 + k >= g_begin && g0 + k < g_end;
        c[k] = in ? colind[g0 + k] : 0;
        v[k] = in ? vals[g0 + k] : 0.0;
      }
    }
    int prev = __shfl_up_sync(kFull, c[3], 1);
    if (lane == 0 && g0 > g_begin && g0 <= g_end) prev = colind[g0 - 1];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t gk = g0 + k;
      if (gk >= g_begin && gk < g_end) {
        if (c[k] < 0 || c[k] >= n) e_local |= 2;
        if (!isfinite(v[k])) e_local |= 4;
        if (gk > g_begin && c[k] <= (k ? c[k - 1] : prev)) ++d_local;
      }
    }
  }
  d_local = warp_sum_i((int)d_local);
  if (e_local) atomicOr(&s_e, e_local);
  if (lane == 0 && d_local) atomicAdd(&s_d, d_local);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_e) atomicOr(err, s_e);
    if (s_d) atomicAdd(cnt, (unsigned long long)s_d);
  }
}

__global__ void validate_rows_kernel(int batch, int m, const int64_t* __restrict__ nnz_off,
                                     const int32_t* __restrict__ rowptr,
                                     const int32_t* __restrict__ colind,
                                     const double* __restrict__ b, int* err,
                                     unsigned long long* cnt, int64_t g_begin) {
  __shared__ int s_e;
  __shared__ unsigned s_d;
  if (threadIdx.x == 0) {
    s_e = 0;
    s_d = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int e_local = 0;
  unsigned d_local = 0;
  const int64_t rows = (int64_t)batch * m;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool small = rows < (1ll << 31);
  for (int64_t gr = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; gr < rows; gr += stride) {
    const int prob = small ? (int)((unsigned)gr / (unsigned)m) : (int)(gr / m);
    const int r = (int)(gr - (int64_t)prob * m);
    const int64_t base = nnz_off[prob];
    const int64_t nz = nnz_off[prob + 1] - base;
    const int64_t lo = rowptr[(size_t)prob * (m + 1) + r], hi = rowptr[(size_t)prob * (m + 1) + r + 1];
    if (r == 0 && lo != 0) e_local |= 1;
    if (r == m - 1 && hi != nz) e_local |= 1;
    if (!isfinite(b[gr])) e_local |= 4;
    if (hi < lo || lo < 0 || hi > nz) {
      e_local |= 1;
      continue;
    }
    const int64_t g = base + lo;
    if (hi > lo && g > g_begin && colind[g] <= colind[g - 1]) ++d_local;
  }
  d_local = warp_sum_i((int)d_local);
  if (e_local) atomicOr(&s_e, e_local);
  if (lane == 0 && d_local) atomicAdd(&s_d, d_local);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_e) atomicOr(err, s_e);
    if (s_d) atomicAdd(cnt + 1, (unsigned long long)s_d);
  }
}

__global__ void validate_finalize_kernel(int* err) {
  const unsigned long long* cnt = reinterpret_cast<const unsigned long long*>(err + 2);
  if (cnt[0] != cnt[1]) err[0] |= 2;
}

cudaError_t launch_validate_batched(int batch, int m, int n, const int64_t* nnz_off, int64_t g_begin,
                                    int64_t g_end, const int32_t* rowptr, const int32_t* colind,
                                    const double* vals, const double* b, int* err, cudaStream_t s) {
  // err[0] bits, err[2..5] the two 64-bit descent counts (zeroed by the caller)
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(err + 2);
  const int64_t quads = (g_end + 3) / 4 - g_begin / 4;
  int blocks = (int)((quads + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  if (g_end > g_begin)
    validate_entries_kernel<<<blocks, 256, 0, s>>>(g_begin, g_end, n, colind, vals, err, cnt);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t rows = (int64_t)batch * m;
  blocks = (int)((rows + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  validate_rows_kernel<<<blocks, 256, 0, s>>>(batch, m, nnz_off, rowptr, colind, b, err, cnt, g_begin);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  validate_finalize_kernel<<<1, 1, 0, s>>>(err);
  return cudaGetLastError();
}

size_t batched_smem_bytes(int m, int n, int nnz_max) { return layout(m, n, nnz_max).bytes; }
size_t batched_gram_scratch(int n, int sm_count) { return sizeof(double) * (size_t)n * (n + 1) / 2 * (size_t)sm_count * 16; }

size_t batched_colview_stride(int n, int nnz_max) {
  return ((sizeof(int32_t) * (size_t)(n + 1) + sizeof(uint16_t) * 2 * (size_t)nnz_max) + 15) & ~(size_t)15;
}

cudaError_t launch_batched_nnz(const BatchArgs& a, int nnz_max, int sm_count, cudaStream_t s) {
  const size_t smem = layout(a.m, a.n, nnz_max).bytes;
  const size_t smem2 = llayout(a.m, a.n, nnz_max, a.lsqr_cap_pct).bytes;
  if (smem > 220 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(batched_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(batched_lsqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
  if (e != cudaSuccess) return e;
  int per_sm = 0, per_sm2 = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, batched_kernel, BT, smem);
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, batched_lsqr_kernel, BT, smem2);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  if (per_sm2 < 1) per_sm2 = 1;
  if (per_sm > 16) per_sm = 16;  // the Gram scratch holds 16 CTAs per SM
  int grid = sm_count * per_sm;
  if (grid > a.batch) grid = a.batch;
  if (grid < 1) grid = 1;
  batched_kernel<<<grid, BT, smem, s>>>(a, nnz_max);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int grid2 = sm_count * per_sm2;
  if (grid2 > a.batch) grid2 = a.batch;
  if (grid2 < 1) grid2 = 1;
  batched_lsqr_kernel<<<grid2, BT, smem2, s>>>(a, nnz_max);
  return cudaGetLastError();
}

}  // namespace nnls
