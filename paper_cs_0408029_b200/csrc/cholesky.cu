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
//   * The tile update  C_ij -= L_ik L_jk^T  (the O(f^3) work) runs on the FP64
//     tensor pipe: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), the only FP64 tensor
//     path on sm_100a (tcgen05 has no f64 kind).  8 warps, each a 16 x 32
//     register accumulator; operands staged in shared memory.
//   * Diagonal tiles are factored (POTRF) and off-diagonal tiles triangular-
//     solved (TRSM) in shared memory, column by column.  Pivot <= 0,
//     < 1e-300 or non-finite -> NOT_PD (reading c13).
//   * L^T x = z by a second DAG kernel over column tiles (last to first).
#include <cuda_runtime.h>
#include <math.h>

#include "common.cuh"
#include "kernels.cuh"

namespace nnls {

namespace {
constexpr int T = kTile;
constexpr int LDS = T + 4;  // smem row stride (doubles): conflict-free 8x4 fragment reads
constexpr int kThreads = 256;
constexpr int kSmemDoubles = 3 * T * LDS;

__host__ __device__ inline int tidx(int i, int j) { return i * (i + 1) / 2 + j; }
}  // namespace

size_t chol_tile_count(int n) {
  const int ntr = (n + 1 + T - 1) / T;
  return (size_t)ntr * (ntr + 1) / 2;
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

__global__ void __launch_bounds__(kThreads) chol_factor_kernel(
    const double* __restrict__ G, int ldg, const double* __restrict__ cvec,
    const int32_t* __restrict__ Fidx, double* __restrict__ Lt, int* __restrict__ flags,
    DevState* st) {
  extern __shared__ double smem[];
  double* S = smem;               // task tile (accumulator / result)
  double* LA = smem + T * LDS;    // L(i,k)
  double* LB = smem + 2 * T * LDS;  // L(j,k) or L(j,j)
  __shared__ int s_task;

  const int f = st->f;
  const int epoch = st->epoch;
  if (f <= 0) return;
  const int ntc = (f + T - 1) / T;      // tile columns to factor
  const int ntr = (f + 1 + T - 1) / T;  // tile rows (incl. the rhs row f)
  const int total = ntc * ntr - ntc * (ntc - 1) / 2;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int rb0 = (w >> 1) * 16;  // warp tile: rows rb0..rb0+15
  const int cb0 = (w & 1) * 32;   //            cols cb0..cb0+31

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

    // 2) left-looking update S -= sum_{k<j} L(i,k) L(j,k)^T on the DMMA pipe
    if (j > 0) {
      double acc[2][4][2];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int v = 0; v < 2; ++v)
            acc[a][q][v] = S[(rb0 + 8 * a + (lane >> 2)) * LDS + cb0 + 8 * q + 2 * (lane & 3) + v];
      for (int k = 0; k < j; ++k) {
        if (tid == 0) {
          wait_flag(&flags[tidx(i, k)], epoch);
          wait_flag(&flags[tidx(j, k)], epoch);
        }
        __syncthreads();
        load_tile(LA, Lt + (size_t)tidx(i, k) * T * T);
        load_tile(LB, Lt + (size_t)tidx(j, k) * T * T);
        __syncthreads();
#pragma unroll 4
        for (int kk = 0; kk < T; kk += 4) {
          double av[2], bv[4];
#pragma unroll
          for (int a = 0; a < 2; ++a) av[a] = -LA[(rb0 + 8 * a + (lane >> 2)) * LDS + kk + (lane & 3)];
#pragma unroll
          for (int q = 0; q < 4; ++q) bv[q] = LB[(cb0 + 8 * q + (lane >> 2)) * LDS + kk + (lane & 3)];
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int q = 0; q < 4; ++q) dmma8x8x4(acc[a][q][0], acc[a][q][1], av[a], bv[q]);
        }
        __syncthreads();
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int v = 0; v < 2; ++v)
            S[(rb0 + 8 * a + (lane >> 2)) * LDS + cb0 + 8 * q + 2 * (lane & 3) + v] = acc[a][q][v];
      __syncthreads();
    }

    if (i == j) {
      // 3a) POTRF of the diagonal tile (rows may include the rhs row f)
      for (int c = 0; c < cv; ++c) {
        const double d = S[c * LDS + c];
        const bool bad = !(d > 0.0) || d < 1e-300 || !isfinite(d);
        if (bad && tid == 0) {
          if (atomicCAS(&st->status, 0, 7) == 0) st->not_pd_col = j * T + c;
        }
        const double l = sqrt(d);
        __syncthreads();
        if (tid > c && tid < rv) S[tid * LDS + c] = S[tid * LDS + c] / l;
        if (tid == 0) S[c * LDS + c] = l;
        __syncthreads();
        // trailing update of the tile: S[r][q] -= S[r][c] S[q][c], c < q <= r
        const int nr = rv - c - 1;
        for (int e = tid; e < nr * (cv - c - 1); e += kThreads) {
          const int r = c + 1 + e / (cv - c - 1);
          const int q = c + 1 + e % (cv - c - 1);
          if (q <= r) S[r * LDS + q] -= S[r * LDS + c] * S[q * LDS + c];
        }
        __syncthreads();
      }
      for (int e = tid; e < T * T; e += kThreads) {  // clear the strict upper part
        const int r = e / T, q = e % T;
        if (q > r) S[r * LDS + q] = 0.0;
      }
      __syncthreads();
    } else {
      // 3b) TRSM: S <- S L(j,j)^-T, column by column
      if (tid == 0) wait_flag(&flags[tidx(j, j)], epoch);
      __syncthreads();
      load_tile(LB, Lt + (size_t)tidx(j, j) * T * T);
      __syncthreads();
      for (int c = 0; c < cv; ++c) {
        if (tid < rv) S[tid * LDS + c] = S[tid * LDS + c] / LB[c * LDS + c];
        __syncthreads();
        const int nq = cv - c - 1;
        for (int e = tid; e < rv * nq; e += kThreads) {
          const int r = e / nq, q = c + 1 + e % nq;
          S[r * LDS + q] -= S[r * LDS + c] * LB[q * LDS + c];
        }
        __syncthreads();
      }
    }
    // 4) publish
    store_tile(Lt + (size_t)tidx(i, j) * T * T, S);
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release(&flags[tidx(i, j)], epoch);
  }
}

// L^T x = z, z = row f of the bordered factor.  Column tiles J from the last
// to the first; task J waits for x_I (I > J), subtracts L_IJ^T x_I, then
// solves with L_JJ^T.  xflags[J] == epoch: x_J published.
__global__ void __launch_bounds__(kThreads) chol_backsolve_kernel(const double* __restrict__ Lt,
                                                                   int* __restrict__ xflags,
                                                                   double* __restrict__ xF,
                                                                   DevState* st) {
  extern __shared__ double smem[];
  double* Ls = smem;             // tile L(J,J) or L(I,J), stride LDS
  double* part = smem + T * LDS;  // 4 x T partial sums
  __shared__ double s_rhs[T];
  __shared__ double s_x[T];
  __shared__ int s_task;
  const int f = st->f;
  const int epoch = st->epoch;
  if (f <= 0) return;
  const int ntc = (f + T - 1) / T;
  const int Rf = f / T, rf = f % T;  // tile row / local row of the rhs row
  const int tid = threadIdx.x;
  for (;;) {
    if (tid == 0) s_task = atomicAdd(&st->solve_counter, 1);
    __syncthreads();
    const int t = s_task;
    if (t >= ntc) break;
    const int J = ntc - 1 - t;
    const int cv = min(T, f - J * T);
    // z_J
    if (tid < T) s_rhs[tid] = (tid < cv) ? __ldcg(&Lt[(size_t)tidx(Rf, J) * T * T + rf * T + tid]) : 0.0;
    __syncthreads();
    // subtract L_IJ^T x_I for I = ntc-1 .. J+1 (the latest-ready block last)
    for (int I = ntc - 1; I > J; --I) {
      if (tid == 0) wait_flag(&xflags[I], epoch);
      __syncthreads();
      const int rvI = min(T, f - I * T);  // rows of L_IJ that are < f
      if (tid < T) s_x[tid] = (tid < rvI) ? __ldcg(&xF[I * T + tid]) : 0.0;
      __syncthreads();
      const double* L = Lt + (size_t)tidx(I, J) * T * T;
      const int c = tid & (T - 1), rg = tid >> 6;  // 4 row groups
      double p = 0.0;
      for (int r = rg; r < rvI; r += 4) p = fma(__ldcg(&L[r * T + c]), s_x[r], p);
      part[rg * T + c] = p;
      __syncthreads();
      if (tid < T) s_rhs[tid] -= (part[tid] + part[T + tid]) + (part[2 * T + tid] + part[3 * T + tid]);
      __syncthreads();
    }
    // diagonal: L_JJ^T x_J = s_rhs (backward substitution), one warp
    load_tile(Ls, Lt + (size_t)tidx(J, J) * T * T);
    __syncthreads();
    if (tid < 32) {
      const int l = tid;
      double s0 = s_rhs[l], s1 = s_rhs[l + 32];
      for (int c = cv - 1; c >= 0; --c) {
        const double own = (c < 32) ? s0 : s1;
        const double sc = __shfl_sync(kFull, own, c & 31);
        const double xc = sc / Ls[c * LDS + c];
        if (l == 0) s_x[c] = xc;
        // s_t -= L[c][t] x_c for t < c
        if (l < c) s0 = fma(-Ls[c * LDS + l], xc, s0);
        if (l + 32 < c) s1 = fma(-Ls[c * LDS + l + 32], xc, s1);
      }
    }
    __syncthreads();
    if (tid < cv) xF[J * T + tid] = s_x[tid];
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
                           (int)(sizeof(double) * (T * LDS + 4 * T)));
  if (e != cudaSuccess) return e;
  attr_set = true;
  return cudaSuccess;
}

cudaError_t launch_chol_factor(int n, const double* G, int ldg, const double* c, const int32_t* Fidx,
                               double* Lt, int* flags, DevState* st, int sm_count, cudaStream_t s) {
  cudaError_t e = set_attrs();
  if (e != cudaSuccess) return e;
  // grid sized for the largest possible DAG; tasks are claimed dynamically
  const int ntr = (n + 1 + T - 1) / T;
  const int tasks = ntr * (ntr + 1) / 2;
  int grid = sm_count * 2;
  if (grid > tasks) grid = tasks;
  chol_factor_kernel<<<grid, kThreads, sizeof(double) * kSmemDoubles, s>>>(G, ldg, c, Fidx, Lt, flags, st);
  return cudaGetLastError();
}

cudaError_t launch_chol_backsolve(int n, const double* Lt, int* flags, double* xF, DevState* st,
                                  int sm_count, cudaStream_t s) {
  cudaError_t e = set_attrs();
  if (e != cudaSuccess) return e;
  const int ntr = (n + 1 + T - 1) / T;
  int* xflags = flags + chol_tile_count(n);
  const int g2 = ntr < sm_count ? ntr : sm_count;
  chol_backsolve_kernel<<<g2, kThreads, sizeof(double) * (T * LDS + 4 * T), s>>>(Lt, xflags, xF, st);
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
