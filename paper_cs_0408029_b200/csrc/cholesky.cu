// cholesky.cu -- a5/a6: the normal-equations solve on the free set F
// ("solves A^T A x = A^T b using a Cholesky factorization
// of the symmetric matrix A^T A"), on the principal submatrix (A^T A)_FF of
// the cached Gram.
//
// B200 design
//   * Bordered system: the factorization runs on the (f+1) x (f+1) matrix
//     [[G_FF, .], [c_F^T, .]], whose last row of L is z^T = (L^-1 c_F)^T, so
//     the forward substitution L z = c_F comes out of the factorization and
//     only L^T x_F = z remains (one triangular solve instead of two).
//   * Gather fused into the factorization: each tile task reads
//     G[Fidx[r], Fidx[c]] directly -- (A^T A)_FF is never materialised.
//   * Tiled left-looking Cholesky, T = 64, as a dependency DAG executed by a
//     persistent kernel: tasks (i, j) are claimed in column-major order from
//     an atomic counter and wait on per-tile "ready" flags (release/acquire),
//     so there is no grid-wide barrier; a task only waits for the tiles it
//     reads.  Since tasks are claimed in topological order by running CTAs,
//     the DAG cannot deadlock.
//   * Every O(T^3) step runs on the FP64 tensor pipe, mma.sync.m8n8k4.f64
//     (SASS DMMA.8x8x4 -- the only FP64 tensor path on sm_100a, tcgen05 has no
//     f64 kind): the left-looking update C_ij -= L_ik L_jk^T, and the
//     triangular solve of the off-diagonal tiles, done as a product with the
//     explicit inverse of the diagonal tile, X = C_ij L_jj^-T.
//   * The diagonal task factors its tile (2 x 2 blocks of 32: POTRF, TRSM,
//     SYRK, POTRF in one warp) and inverts it (TRTRI of the two 32-blocks by
//     two warps, off-diagonal block by products).  Column-sequential work is
//     thereby confined to the diagonal tile; the off-diagonal tiles never run
//     a column-sequential loop.  Pivot <= 0, < 1e-300 or non-finite -> NOT_PD
//     (reading c13).
//   * L^T x = z by a second DAG kernel over column tiles (last to first), each
//     step a GEMV with the published inverse diagonal tile.
#include <cuda_runtime.h>
#include <math.h>

#include "common.cuh"
#include "kernels.cuh"

namespace nnls {

namespace {
constexpr int T = kTile;
constexpr int LDS = T + 4;  // smem row stride (doubles): conflict-free 8x4 fragment reads
constexpr int kThreads = 256;
constexpr int kSmemDoubles = 4 * T * LDS;

__host__ __device__ inline int tidx(int i, int j) { return i * (i + 1) / 2 + j; }
inline int tri_tiles(int n) {
  const int ntr = (n + 1 + T - 1) / T;
  return ntr * (ntr + 1) / 2;
}
}  // namespace

// Debug hook (not part of the ABI): per-task %globaltimer stamps of the
// factorization DAG, enabled by nnls_debug_chol_profile(ptr).
__device__ unsigned long long* g_chol_prof = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PROF_STAMP(task, slot)                                                                  \
  do {                                                                                          \
    if (g_chol_prof != nullptr && threadIdx.x == 0) g_chol_prof[(task) * 8 + (slot)] = gtimer(); \
  } while (0)

// Lower tiles L(i,j) followed by one inverse tile per tile column.
size_t chol_tile_count(int n) {
  const int ntr = (n + 1 + T - 1) / T;
  return (size_t)tri_tiles(n) + ntr;
}

// load a T x T tile (row-major, contiguous) from global into smem (stride LDS)
__device__ __forceinline__ void load_tile(double* __restrict__ dst, const double* __restrict__ src) {
  const double2* s2 = reinterpret_cast<const double2*>(src);
  for (int e = threadIdx.x; e < T * T / 2; e += kThreads) {
    const int r = (2 * e) / T, c = (2 * e) % T;
    const double2 v = __ldcg(&s2[e]);  // written by other CTAs: bypass L1
    dst[r * LDS + c] = v.x;
    dst[r * LDS + c + 1] = v.y;
  }
}

__device__ __forceinline__ void store_tile(double* __restrict__ dst, const double* __restrict__ src) {
  double2* d2 = reinterpret_cast<double2*>(dst);
  for (int e = threadIdx.x; e < T * T / 2; e += kThreads) {
    const int r = (2 * e) / T, c = (2 * e) % T;
    d2[e] = make_double2(src[r * LDS + c], src[r * LDS + c + 1]);
  }
}

// asynchronous 16-byte copies global -> shared (cp.async.cg: L2 only)
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void tile_async(double* __restrict__ dst, const double* __restrict__ src) {
  for (int e = threadIdx.x; e < T * T / 2; e += kThreads) {
    const int r = (2 * e) / T, c = (2 * e) % T;
    cp_async16(dst + r * LDS + c, src + 2 * e);
  }
}

// acc (16 x 32 per warp) += sign * A B^T for 64 x 64 tiles in smem (B given
// by rows: C[m][n] += sum_k A[m][k] B[n][k]), on DMMA 8x8x4.
template <bool kNegate>
__device__ __forceinline__ void dmma_tile(double (&acc)[2][4][2], const double* __restrict__ A,
                                          const double* __restrict__ B, int lane, int rb0, int cb0) {
#pragma unroll 4
  for (int kk = 0; kk < T; kk += 4) {
    double av[2], bv[4];
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const double v = A[(rb0 + 8 * a + (lane >> 2)) * LDS + kk + (lane & 3)];
      av[a] = kNegate ? -v : v;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) bv[q] = B[(cb0 + 8 * q + (lane >> 2)) * LDS + kk + (lane & 3)];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int q = 0; q < 4; ++q) dmma8x8x4(acc[a][q][0], acc[a][q][1], av[a], bv[q]);
  }
}
__device__ __forceinline__ void acc_load(double (&acc)[2][4][2], const double* S, int lane, int rb0,
                                         int cb0) {
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int v = 0; v < 2; ++v)
        acc[a][q][v] = S[(rb0 + 8 * a + (lane >> 2)) * LDS + cb0 + 8 * q + 2 * (lane & 3) + v];
}
__device__ __forceinline__ void acc_store(const double (&acc)[2][4][2], double* S, int lane, int rb0,
                                          int cb0) {
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int v = 0; v < 2; ++v)
        S[(rb0 + 8 * a + (lane >> 2)) * LDS + cb0 + 8 * q + 2 * (lane & 3) + v] = acc[a][q][v];
}

// POTRF of a 32-row block held by one warp, lane = row, a[t] = A[lane][t].
// Columns c < ncols are pivots; rows >= ncols (e.g. the bordered row c_F^T)
// are eliminated as off-diagonal rows.  Right-looking, updates applied in
// increasing c.  The finished column is broadcast through shared memory
// (colbuf: broadcast loads at immediate offsets); updates are predicated,
// never divergent.  The column loop is rolled 4 columns at a time with a
// register shift (register arrays are indexed by compile-time constants only;
// a fully unrolled loop is instruction-bound, not cheaper).  Writes L[lane][c]
// to out[lane*LDS + c] (0 above the diagonal and in non-pivot columns),
// 1/l_cc to rinv[c].  Returns the first bad pivot or -1.
__device__ __forceinline__ int warp_potrf32(double (&a)[32], int ncols, int lane, double* rinv,
                                            double* out, double* colbuf) {
  int bad = -1;
#pragma unroll 1
  for (int c0 = 0; c0 < ncols; c0 += 4) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int c = c0 + u;
      if (c < ncols) {
        const double d = __shfl_sync(kFull, a[u], c);
        if ((!(d > 0.0) || d < 1e-300 || !isfinite(d)) && bad < 0) bad = c;
        const double inv = rsqrt(d);
        const double lic = (lane == c) ? d * inv : ((lane > c) ? a[u] * inv : 0.0);
        colbuf[lane] = lic;
        if (lane == 0) rinv[c] = inv;
        out[lane * LDS + c] = lic;
        __syncwarp();
        const double* cb = colbuf + c;             // cb[t] = l_{c+t, c}
        const int lim = min(lane, ncols - 1) - c;  // update columns c+t, 1 <= t <= lim
#pragma unroll
        for (int t = 1; u + t < 32; ++t) {
          const double v = cb[t];
          if (t <= lim) a[u + t] = fma(-lic, v, a[u + t]);
        }
        __syncwarp();
      }
    }
#pragma unroll
    for (int t = 0; t < 28; ++t) a[t] = a[t + 4];
    a[28] = a[29] = a[30] = a[31] = 0.0;
  }
  for (int col = ncols; col < 32; ++col) out[lane * LDS + col] = 0.0;
  return bad;
}

// Inverse of a 32 x 32 lower-triangular block (smem, stride LDS) with
// reciprocal diagonal rinvb: lane = column c computes X[:, c] by forward
// substitution, x_i = (delta_ic - sum_{k<i} L_ik x_k) / L_ii.  ncols pivots;
// rows/columns >= ncols are zero.  Writes X (lower) to out (stride LDS).
__device__ __forceinline__ void warp_trtri32(const double* __restrict__ Lb,
                                             const double* __restrict__ rinvb, int ncols, int lane,
                                             double* __restrict__ out, double* __restrict__ outT) {
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    double s = (i == lane) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) s = fma(-Lb[i * LDS + k], x[k], s);
    x[i] = (i < ncols && lane < ncols) ? s * rinvb[i] : 0.0;
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) out[i * LDS + lane] = x[i];
  if (outT != nullptr) {
#pragma unroll
    for (int i = 0; i < 32; ++i) outT[lane * LDS + i] = x[i];
  }
}

// Cholesky of the diagonal 64 x 64 tile S (smem, rows < rv, pivot columns
// < cv; a row >= cv is the bordered row c_F^T and is only eliminated) by all
// 256 threads.  Thread t owns the lower-triangle entries e = t + 256 s of the
// tile in registers.  Column c: the owners of column c publish it into a
// ping-pong buffer, ONE barrier, then every thread updates its own entries
// with l_rc l_kc = b_r b_k / d (and finalises column c).  Writes L back into S
// (zero above the diagonal / beyond cv), 1/l_cc into rinv.  Returns the first
// bad pivot column or -1.
__device__ __forceinline__ int block_potrf64(double* __restrict__ S, int rv, int cv,
                                             double* __restrict__ rinv, double (*colbuf)[T]) {
  constexpr int NS = (T * (T + 1) / 2 + kThreads - 1) / kThreads;  // 9 slots
  const int tid = threadIdx.x;
  double a[NS];
  int rs[NS], ks[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int e = tid + kThreads * s;
    int r = (int)((sqrtf(8.0f * e + 1.0f) - 1.0f) * 0.5f);
    while (r * (r + 1) / 2 > e) --r;
    while ((r + 1) * (r + 2) / 2 <= e) ++r;
    const int k = e - r * (r + 1) / 2;
    const bool valid = e < T * (T + 1) / 2 && r < rv && k < cv;
    rs[s] = valid ? r : 0;
    ks[s] = valid ? k : T;  // k = T: never updated (and never published)
    a[s] = valid ? S[r * LDS + k] : 0.0;
  }
  int bad = -1;
  // branch-free column loop: every slot computes both candidates and selects
  // (divergent if/else per slot cost ~1.7K cycles per column)
#pragma unroll 1
  for (int c = 0; c < cv; ++c) {
    double* buf = colbuf[c & 1];
#pragma unroll
    for (int s = 0; s < NS; ++s)
      if (ks[s] == c) buf[rs[s]] = a[s];
    __syncthreads();
    const double d = buf[c];
    if (!(d > 0.0) || d < 1e-300 || !isfinite(d)) bad = (bad < 0) ? c : bad;
    const double inv = rsqrt(d);
    if (tid == 0) rinv[c] = inv;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int k = ks[s];
      const double br = buf[rs[s]], bk = buf[min(k, T - 1)];
      const double upd = fma(-(br * inv), bk * inv, a[s]);
      const double fin = (rs[s] == c) ? d * inv : a[s] * inv;
      a[s] = (k == c) ? fin : ((k > c && k < T) ? upd : a[s]);
    }
  }
  __syncthreads();
  for (int e = tid; e < T * T; e += kThreads) S[(e / T) * LDS + (e % T)] = 0.0;
  __syncthreads();
#pragma unroll
  for (int s = 0; s < NS; ++s)
    if (ks[s] < T) S[rs[s] * LDS + ks[s]] = a[s];
  return bad;
}

// Cholesky of the diagonal 64 x 64 tile S (smem; rows < rv, pivot columns
// < cv; a row >= cv is the bordered row c_F^T and is only eliminated), by
// panels of 8 columns: warp 0 factors the 8-wide panel in registers (lane l
// holds rows 8p+l and 8p+l+32; 8 shuffle-broadcast columns), then all 8
// warps apply the rank-8 trailing update with DMMA.  Column-sequential work
// per lane is 8 wide instead of 32/64 (the column chain is latency-bound).
// Writes L into S (lower; the strict upper part is cleared by the caller),
// 1/l_cc into rinv; returns the first bad pivot column or -1.
__device__ __forceinline__ void panel8_update_block(double* __restrict__ S, int c0, int r0, int k0,
                                                    int lane) {
  // S[r0..r0+8)[k0..k0+8) -= S[r0..][c0..c0+8) S[k0..][c0..c0+8)^T  (one DMMA block, K = 8)
  double* Cp = S + (r0 + (lane >> 2)) * LDS + k0 + 2 * (lane & 3);
  double c0v = Cp[0], c1v = Cp[1];
#pragma unroll
  for (int kk = 0; kk < 8; kk += 4) {
    const double av = -S[(r0 + (lane >> 2)) * LDS + c0 + kk + (lane & 3)];
    const double bv = S[(k0 + (lane >> 2)) * LDS + c0 + kk + (lane & 3)];
    dmma8x8x4(c0v, c1v, av, bv);
  }
  Cp[0] = c0v;
  Cp[1] = c1v;
}

__device__ __forceinline__ int potrf64_panel8(double* __restrict__ S, int rv, int cv,
                                              double* __restrict__ rinv, int* s_bad) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) *s_bad = -1;
  const int np = (cv + 7) >> 3;
  const int nbr = (rv + 7) >> 3;  // 8-row blocks holding valid rows
  __syncthreads();
#pragma unroll 1
  for (int p = 0; p < np; ++p) {
    const int c0 = 8 * p;
    // (a) critical: apply panel p-1's update to column block p (blocks (I, p))
    if (p > 0) {
      for (int I = p + w; I < nbr; I += 8) panel8_update_block(S, c0 - 8, 8 * I, c0, lane);
      __syncthreads();
    }
    if (w == 0) {
      // (b) warp 0 factors panel p in registers: lane l holds rows c0+l, c0+32+l
      const int R0 = c0 + lane, R1 = c0 + 32 + lane;
      const bool v0 = R0 < rv, v1 = R1 < rv;
      double a0[8], a1[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        a0[c] = v0 ? S[R0 * LDS + c0 + c] : 0.0;
        a1[c] = v1 ? S[R1 * LDS + c0 + c] : 0.0;
      }
      int bad = -1;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c0 + c < cv) {
          const double d = __shfl_sync(kFull, a0[c], c);
          if (!(d > 0.0) || d < 1e-300 || !isfinite(d)) bad = (bad < 0) ? c0 + c : bad;
          const double inv = rsqrt(d);
          if (lane == 0) rinv[c0 + c] = inv;
          a0[c] = (lane == c) ? d * inv : ((lane > c) ? a0[c] * inv : 0.0);
          a1[c] *= inv;
#pragma unroll
          for (int c2 = c + 1; c2 < 8; ++c2) {
            const double x = __shfl_sync(kFull, a0[c], c2);  // l_{c0+c2, c0+c}
            if (c0 + c2 < cv) {
              if (lane >= c2) a0[c2] = fma(-a0[c], x, a0[c2]);
              a1[c2] = fma(-a1[c], x, a1[c2]);
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (v0) S[R0 * LDS + c0 + c] = (c0 + c < cv) ? a0[c] : 0.0;
        if (v1) S[R1 * LDS + c0 + c] = (c0 + c < cv) ? a1[c] : 0.0;
      }
      if (lane == 0 && bad >= 0 && *s_bad < 0) *s_bad = bad;
    } else if (p > 0) {
      // (c) meanwhile warps 1..7: the rest of panel p-1's trailing update
      //     (blocks (I, J) with I >= J >= p+1), disjoint from panel p
      const int nb = nbr - (p + 1);
      const int nblk = nb > 0 ? nb * (nb + 1) / 2 : 0;
      for (int bq = w - 1; bq < nblk; bq += 7) {
        int I = (int)((sqrtf(8.0f * bq + 1.0f) - 1.0f) * 0.5f);
        while (I * (I + 1) / 2 > bq) --I;
        while ((I + 1) * (I + 2) / 2 <= bq) ++I;
        const int J = bq - I * (I + 1) / 2;
        if (8 * (p + 1 + J) < cv) panel8_update_block(S, c0 - 8, 8 * (p + 1 + I), 8 * (p + 1 + J), lane);
      }
    }
    __syncthreads();
  }
  return *s_bad;
}

// acc[q] (rows 8w.. of a 32 x 32 product, cols 8q..) += A B^T, A and B
// 32 x 32 row-major (B by rows n: C[m][n] += sum_k A[m][k] B[n][k]).
__device__ __forceinline__ void dmma32(double (&acc)[4][2], const double* __restrict__ A,
                                       const double* __restrict__ B, int lane, int w) {
#pragma unroll
  for (int kk = 0; kk < 32; kk += 4) {
    const double av = A[(8 * w + (lane >> 2)) * LDS + kk + (lane & 3)];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double bv = B[(8 * q + (lane >> 2)) * LDS + kk + (lane & 3)];
      dmma8x8x4(acc[q][0], acc[q][1], av, bv);
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1) chol_factor_kernel(
    const double* __restrict__ G, int ldg, const double* __restrict__ cvec,
    const int32_t* __restrict__ Fidx, double* __restrict__ Lt, double* __restrict__ Linv,
    int* __restrict__ flags, DevState* st) {
  extern __shared__ double smem[];
  // four T x LDS buffers: BUF(0) = S (task tile) and, during the update loop,
  // the second (i,k)/(j,k) operand pair with BUF(1); BUF(2)/BUF(3) = first pair.
#define BUF(q) (smem + (q) * (T * LDS))
  double* S = BUF(0);
  __shared__ double rinv[T];
  __shared__ int s_task, s_ready, s_bad;

  const int f = st->f;
  const int epoch = st->epoch;
  if (f <= 0 || st->done || st->status != 0) return;  // (graph loop: nothing to solve)
  const int ntc = (f + T - 1) / T;      // tile columns to factor
  const int ntr = (f + 1 + T - 1) / T;  // tile rows (incl. the rhs row f)
  const int total = ntc * ntr - ntc * (ntc - 1) / 2;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int rb0 = (w >> 1) * 16;  // warp tile of the DMMA products: rows rb0..rb0+15
  const int cb0 = (w & 1) * 32;   //                                 cols cb0..cb0+31

  for (;;) {
    if (tid == 0) s_task = atomicAdd(&st->tile_counter, 1);
    __syncthreads();
    int t = s_task;
    if (t >= total) break;
    int j = 0;
    while (t >= ntr - j) {
      t -= ntr - j;
      ++j;
    }
    const int i = j + t;
    const int rv = min(T, f + 1 - i * T);  // valid rows in this tile (incl. rhs row)
    const int cv = min(T, f - j * T);      // valid (factored) columns
    const int task = s_task;
    PROF_STAMP(task, 0);
    if (g_chol_prof != nullptr && tid == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      g_chol_prof[task * 8 + 7] = ((unsigned long long)i << 40) | ((unsigned long long)j << 20) | smid;
    }

    // 1) gather A(i,j) = [G_FF; c_F^T] block straight from the cached Gram
    for (int e = tid; e < T * T; e += kThreads) {
      const int r = e / T, cc = e % T;
      const int gi = i * T + r, gj = j * T + cc;
      double v = 0.0;
      if (r < rv && cc < cv && (i != j || cc <= r)) {
        v = (gi < f) ? G[(size_t)Fidx[gi] * ldg + Fidx[gj]] : cvec[Fidx[gj]];
      }
      S[r * LDS + cc] = v;
    }
    __syncthreads();
    PROF_STAMP(task, 1);

    // 2) left-looking update S -= sum_{k<j} L(i,k) L(j,k)^T on the DMMA pipe,
    //    operand tiles double-buffered with cp.async
    if (j > 0) {
      double acc[2][4][2];
      acc_load(acc, S, lane, rb0, cb0);
      __syncthreads();  // BUF(0) is reused as an operand buffer below
      bool have_next = false;
      for (int k = 0; k < j; ++k) {
        double* LA = BUF((k & 1) ? 0 : 2);
        double* LB = BUF((k & 1) ? 1 : 3);
        if (!have_next) {
          if (tid == 0) {
            wait_flag(&flags[tidx(i, k)], epoch);
            wait_flag(&flags[tidx(j, k)], epoch);
          }
          __syncthreads();
          tile_async(LA, Lt + (size_t)tidx(i, k) * T * T);
          tile_async(LB, Lt + (size_t)tidx(j, k) * T * T);
          cp_async_commit();
        }
        // try to prefetch k+1 into the other pair if its tiles are ready
        have_next = false;
        if (k + 1 < j) {
          if (tid == 0)
            s_ready = (ld_acquire(&flags[tidx(i, k + 1)]) == epoch) &&
                      (ld_acquire(&flags[tidx(j, k + 1)]) == epoch);
          __syncthreads();
          if (s_ready) {
            tile_async(BUF((k & 1) ? 2 : 0), Lt + (size_t)tidx(i, k + 1) * T * T);
            tile_async(BUF((k & 1) ? 3 : 1), Lt + (size_t)tidx(j, k + 1) * T * T);
            cp_async_commit();
            have_next = true;
          }
        }
        if (have_next) cp_async_wait<1>();
        else cp_async_wait<0>();
        __syncthreads();
        dmma_tile<true>(acc, LA, LB, lane, rb0, cb0);
        __syncthreads();
      }
      acc_store(acc, S, lane, rb0, cb0);
      __syncthreads();
    }
    PROF_STAMP(task, 2);

    if (i == j) {
      // 3a) diagonal tile: L_jj = chol(A_jj) by all 256 threads (block_potrf64,
      //     one barrier per column), then Linv_jj = L_jj^-1 (published for the
      //     TRSM tasks and the solve): TRTRI of the two 32-blocks by two warps,
      //     the off-diagonal block -X22 L21 X11 by two 32^3 DMMA products.
      double* X = BUF(1);    // inverse
      double* X11t = BUF(2); // X11^T
      double* Tmt = BUF(3);  // (L21 X11)^T
      const int n1 = min(32, cv), n2 = cv - 32;
      const int bad = potrf64_panel8(S, rv, cv, rinv, &s_bad);
      for (int e = tid; e < T * T; e += kThreads)  // strict upper part
        if ((e % T) > (e / T)) S[(e / T) * LDS + (e % T)] = 0.0;
      __syncthreads();
      if (w == 0) {
        warp_trtri32(S, rinv, n1, lane, X, X11t);
      } else if (w == 1) {
        if (n2 > 0) {
          warp_trtri32(S + 32 * LDS + 32, rinv + 32, n2, lane, X + 32 * LDS + 32, nullptr);
        } else {
          for (int r = 0; r < 32; ++r) X[(32 + r) * LDS + 32 + lane] = 0.0;
        }
      }
      __syncthreads();
      if (w < 4) {  // Tm = L21 X11 (rows 32.., stored transposed)
        double acc[4][2] = {};
        dmma32(acc, S + 32 * LDS, X11t, lane, w);
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int v = 0; v < 2; ++v)
            Tmt[(8 * q + 2 * (lane & 3) + v) * LDS + 8 * w + (lane >> 2)] = acc[q][v];
      }
      __syncthreads();
      if (w < 4) {  // Linv21 = -X22 Tm
        double acc[4][2] = {};
        dmma32(acc, X + 32 * LDS + 32, Tmt, lane, w);
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int v = 0; v < 2; ++v)
            X[(32 + 8 * w + (lane >> 2)) * LDS + 8 * q + 2 * (lane & 3) + v] = -acc[q][v];
      } else {
        for (int e = tid - 128; e < 32 * 32; e += 128) X[(e >> 5) * LDS + 32 + (e & 31)] = 0.0;
      }
      __syncthreads();
      if (tid == 0 && bad >= 0) {
        if (atomicCAS(&st->status, 0, 7) == 0) st->not_pd_col = j * T + bad;
      }
      store_tile(Linv + (size_t)j * T * T, X);
    } else {
      // 3b) TRSM as a product with the inverse diagonal tile: S <- S Linv_jj^T
      double* LB = BUF(1);
      if (tid == 0) wait_flag(&flags[tidx(j, j)], epoch);
      __syncthreads();
      PROF_STAMP(task, 3);
      load_tile(LB, Linv + (size_t)j * T * T);
      __syncthreads();
      double acc[2][4][2] = {};
      dmma_tile<false>(acc, S, LB, lane, rb0, cb0);
      __syncthreads();
      acc_store(acc, S, lane, rb0, cb0);
      __syncthreads();
    }
    PROF_STAMP(task, 4);
    // 4) publish
    store_tile(Lt + (size_t)tidx(i, j) * T * T, S);
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release(&flags[tidx(i, j)], epoch);
    PROF_STAMP(task, 5);
  }
#undef BUF
}

cudaError_t chol_debug_set_profile(unsigned long long* p) {
  return cudaMemcpyToSymbol(g_chol_prof, &p, sizeof(p));
}

// L^T x = z, z = row f of the bordered factor.  Column tiles J from the last
// to the first; task J waits for x_I (I > J), subtracts L_IJ^T x_I, then
// x_J = Linv_JJ^T s (a GEMV, no sequential substitution).  xflags[J] == epoch:
// x_J published.
__global__ void __launch_bounds__(kThreads) chol_backsolve_kernel(const double* __restrict__ Lt,
                                                                   const double* __restrict__ Linv,
                                                                   int* __restrict__ xflags,
                                                                   double* __restrict__ xF,
                                                                   DevState* st) {
  extern __shared__ double bsm[];
  double* Lnext = bsm;        // L(J+1, J): the only tile on the critical path
  double* Xinv = bsm + T * T; // Linv(J, J)
  __shared__ double part[4 * T];
  __shared__ double s_rhs[T];
  __shared__ double s_x[T];
  __shared__ int s_task;
  const int f = st->f;
  const int epoch = st->epoch;
  if (f <= 0 || st->done || st->status != 0) return;  // (graph loop: nothing to solve)
  const int ntc = (f + T - 1) / T;
  const int Rf = f / T, rf = f % T;  // tile row / local row of the rhs row
  const int tid = threadIdx.x;
  const int c = tid & (T - 1), rg = tid >> 6;  // column, 4 row groups
  for (;;) {
    if (tid == 0) s_task = atomicAdd(&st->solve_counter, 1);
    __syncthreads();
    const int t = s_task;
    if (t >= ntc) break;
    const int J = ntc - 1 - t;
    const int cv = min(T, f - J * T);
    // prefetch the critical-path tiles (the factorization is complete)
    for (int e = tid; e < T * T / 2; e += kThreads) {
      cp_async16(Xinv + 2 * e, Linv + (size_t)J * T * T + 2 * e);
      if (J + 1 < ntc) cp_async16(Lnext + 2 * e, Lt + (size_t)tidx(J + 1, J) * T * T + 2 * e);
    }
    cp_async_commit();
    if (tid < T) s_rhs[tid] = (tid < cv) ? __ldcg(&Lt[(size_t)tidx(Rf, J) * T * T + rf * T + tid]) : 0.0;
    __syncthreads();
    // subtract L_IJ^T x_I for I = ntc-1 .. J+2 straight from L2 (off the critical path)
    for (int I = ntc - 1; I > J + 1; --I) {
      if (tid == 0) wait_flag(&xflags[I], epoch);
      __syncthreads();
      const int rvI = min(T, f - I * T);  // rows of L_IJ that are < f
      if (tid < T) s_x[tid] = (tid < rvI) ? __ldcg(&xF[I * T + tid]) : 0.0;
      __syncthreads();
      const double* L = Lt + (size_t)tidx(I, J) * T * T;
      double p = 0.0;
      for (int r = rg; r < rvI; r += 4) p = fma(__ldcg(&L[r * T + c]), s_x[r], p);
      part[rg * T + c] = p;
      __syncthreads();
      if (tid < T) s_rhs[tid] -= (part[tid] + part[T + tid]) + (part[2 * T + tid] + part[3 * T + tid]);
      __syncthreads();
    }
    cp_async_wait<0>();
    __syncthreads();
    if (J + 1 < ntc) {  // the critical step: x_{J+1} from the previous task
      if (tid == 0) wait_flag(&xflags[J + 1], epoch);
      __syncthreads();
      const int rvI = min(T, f - (J + 1) * T);
      if (tid < T) s_x[tid] = (tid < rvI) ? __ldcg(&xF[(J + 1) * T + tid]) : 0.0;
      __syncthreads();
      double p = 0.0;
#pragma unroll 4
      for (int r = rg; r < T; r += 4) p = fma(Lnext[r * T + c], s_x[r], p);
      part[rg * T + c] = p;
      __syncthreads();
      if (tid < T) s_rhs[tid] -= (part[tid] + part[T + tid]) + (part[2 * T + tid] + part[3 * T + tid]);
      __syncthreads();
    }
    // x_J = Linv_JJ^T s : x[c] = sum_{r >= c} Linv[r][c] s[r]  (Linv is zero beyond cv)
    double p = 0.0;
#pragma unroll 4
    for (int r = rg; r < T; r += 4) p = fma(Xinv[r * T + c], s_rhs[r], p);
    part[rg * T + c] = p;
    __syncthreads();
    if (tid < cv) xF[J * T + tid] = (part[tid] + part[T + tid]) + (part[2 * T + tid] + part[3 * T + tid]);
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release(&xflags[J], epoch);
  }
}

static cudaError_t set_attrs() {
  static bool attr_set = false;
  if (attr_set) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(chol_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(sizeof(double) * kSmemDoubles));
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(chol_backsolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(sizeof(double) * 2 * T * T));
  if (e != cudaSuccess) return e;
  attr_set = true;
  return cudaSuccess;
}

cudaError_t launch_chol_factor(int n, const double* G, int ldg, const double* c, const int32_t* Fidx,
                               double* Lt, int* flags, DevState* st, int sm_count, cudaStream_t s) {
  cudaError_t e = set_attrs();
  if (e != cudaSuccess) return e;
  // grid sized for the largest possible DAG; tasks are claimed dynamically
  const int tasks = tri_tiles(n);
  int grid = sm_count;  // 136 KB smem per CTA: one persistent CTA per SM
  if (grid > tasks) grid = tasks;
  double* Linv = Lt + (size_t)tri_tiles(n) * T * T;
  chol_factor_kernel<<<grid, kThreads, sizeof(double) * kSmemDoubles, s>>>(G, ldg, c, Fidx, Lt, Linv,
                                                                          flags, st);
  return cudaGetLastError();
}

cudaError_t launch_chol_backsolve(int n, const double* Lt, int* flags, double* xF, DevState* st,
                                  int sm_count, cudaStream_t s) {
  const int ntr = (n + 1 + T - 1) / T;
  int* xflags = flags + tri_tiles(n);
  const double* Linv = Lt + (size_t)tri_tiles(n) * T * T;
  const int g2 = ntr < sm_count ? ntr : sm_count;
  cudaError_t e = set_attrs();
  if (e != cudaSuccess) return e;
  chol_backsolve_kernel<<<g2, kThreads, sizeof(double) * 2 * T * T, s>>>(Lt, Linv, xflags, xF, st);
  return cudaGetLastError();
}

cudaError_t launch_cholesky_solve(int n, const double* G, int ldg, const double* c,
                                  const int32_t* Fidx, double* Lt, int* flags, double* xF,
                                  DevState* st, int sm_count, cudaStream_t s) {
  cudaError_t e = launch_chol_factor(n, G, ldg, c, Fidx, Lt, flags, st, sm_count, s);
  if (e != cudaSuccess) return e;
  return launch_chol_backsolve(n, Lt, flags, xF, st, sm_count, s);
}

}  // namespace nnls
