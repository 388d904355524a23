// Microbenchmark of the Cholesky tile primitives (cycle counts on one SM,
// fresh SPD tile copied in before every repetition; the copy is timed alone
// and subtracted): potrf64_panel8, potrf_r8<2>, potrf_r8<4> (128-row panel),
// trsm_rows / trsm_blocked (64x64), the DMMA 64x64x64 update, load_tile.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o bench/mb_chol bench/microbench_chol_tile.cu
#include <cstdio>

#include "../paper_cs_0408029_b200/csrc/cholesky.cu"

#include "trsm_blocked.cuh"

using namespace nnls;
bool nnls::pdl_enabled() { return false; }

// reference versions (previous product code) for timing / cross-checks
namespace nnls {
__device__ __forceinline__ int potrf64_panel8(double* __restrict__ S, int rv, int cv,
                                              double* __restrict__ rinv, int* s_bad) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) *s_bad = -1;
  const int np = (cv + 7) >> 3;
  const int nbr = (rv + 7) >> 3;  // 8-row blocks holding valid rows
  csync();
#pragma unroll 1
  for (int p = 0; p < np; ++p) {
    const int c0 = 8 * p;
    // (a) critical: apply panel p-1's update to column block p (blocks (I, p))
    if (p > 0) {
      for (int I = p + w; I < nbr; I += 8) panel8_update_block(S, c0 - 8, 8 * I, c0, lane);
      csync();
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
    csync();
  }
  return *s_bad;
}

// X := X L^-T for a 64x64 smem tile X (rows independent) and lower L with
// 1/l_cc in rinv.  Thread (r = tid/4, q = tid%4) holds X[r][4m+q] in
// registers; column c is finished by its owner, broadcast over the 4 lanes
// of the row by one shuffle, and folded into the later columns with FMAs
// (right-looking substitution; the column loop is unrolled so every
// register index is static).
__device__ __forceinline__ void trsm_rows(double* __restrict__ X, const double* __restrict__ L,
                                          const double* __restrict__ rinv, int cv) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int r = tid >> 2, q = tid & 3;
  double a[16];
#pragma unroll
  for (int m = 0; m < 16; ++m) a[m] = X[r * LDS + 4 * m + q];
#pragma unroll
  for (int c = 0; c < T; ++c) {
    if (c < cv) {
      const int q0 = c & 3, m0 = c >> 2;
      const double own = a[m0] * rinv[c];
      if (q == q0) a[m0] = own;
      const double xc = __shfl_sync(kFull, own, (lane & ~3) | q0);
      if (q > q0) a[m0] = fma(-xc, L[(4 * m0 + q) * LDS + c], a[m0]);
#pragma unroll
      for (int m = m0 + 1; m < 16; ++m) a[m] = fma(-xc, L[(4 * m + q) * LDS + c], a[m]);
    }
  }
#pragma unroll
  for (int m = 0; m < 16; ++m) X[r * LDS + 4 * m + q] = a[m];
}
}  // namespace nnls

__device__ void copy_in(double* dst, const double* src, int rows) {
  for (int e = threadIdx.x; e < rows * LDS; e += 256) dst[e] = src[e];
  __syncthreads();
}

__global__ void __launch_bounds__(256, 1) tile_bench(double* out, long long* cyc, const double* gsrc, int reps) {
  extern __shared__ double sm[];
  double* S = sm;                  // 128 rows
  double* B = sm + 2 * T * LDS;    // 128-row backup
  double* L = sm + 4 * T * LDS;
  __shared__ double rinv[T];
  __shared__ int sbad;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  for (int e = tid; e < 2 * T * LDS; e += 256) {
    const int r = e / LDS, c = e % LDS;
    B[e] = (c >= T) ? 0.0 : (r == c ? 100.0 + r : 1.0 / (1.0 + r + c));
  }
  for (int e = tid; e < T * LDS; e += 256) {
    const int r = e / LDS, c = e % LDS;
    L[e] = (c >= T) ? 0.0 : ((r == c) ? 10.0 : (c < r ? 0.01 * (r - c) : 0.0));
  }
  if (tid < T) rinv[tid] = 0.1;
  __syncthreads();
  long long t[9];
  t[0] = clock64();
  for (int rep = 0; rep < reps; ++rep) copy_in(S, B, 2 * T);
  t[1] = clock64();
  for (int rep = 0; rep < reps; ++rep) { copy_in(S, B, 2 * T); potrf64_panel8(S, 64, 64, rinv, &sbad); __syncthreads(); }
  t[2] = clock64();
  for (int rep = 0; rep < reps; ++rep) { copy_in(S, B, 2 * T); potrf_r8<2>(S, 64, 64, rinv, &sbad); __syncthreads(); }
  t[3] = clock64();
  for (int rep = 0; rep < reps; ++rep) { copy_in(S, B, 2 * T); potrf_r8<1, 8, true>(S, 64, 64, rinv, &sbad); __syncthreads(); }
  t[4] = clock64();
  for (int rep = 0; rep < reps; ++rep) { copy_in(S, B, 2 * T); trsm_rows(S, L, rinv, 64); __syncthreads(); }
  t[5] = clock64();
  double acc[2][4][2] = {};
  const int rb0 = (w >> 1) * 16, cb0 = (w & 1) * 32;
  for (int rep = 0; rep < reps; ++rep) {
    copy_in(S, B, 2 * T);
    acc_load(acc, S, lane, rb0, cb0);
    dmma_tile<true>(acc, L, L, lane, rb0, cb0);
    __syncthreads();
    acc_store(acc, S, lane, rb0, cb0);
    __syncthreads();
  }
  t[6] = clock64();
  for (int rep = 0; rep < reps; ++rep) { load_tile(S, gsrc + (rep & 7) * T * T); __syncthreads(); }
  t[7] = clock64();
  for (int rep = 0; rep < reps; ++rep) { copy_in(S, B, 2 * T); trsm_blocked(S, L, rinv, 64); __syncthreads(); }
  t[8] = clock64();

  if (tid == 0) {
    const long long cp = (t[1] - t[0]) / reps;
    cyc[0] = cp;
    for (int q = 1; q < 6; ++q) cyc[q] = (t[q + 1] - t[q]) / reps - cp;
    cyc[6] = (t[7] - t[6]) / reps;
    cyc[7] = (t[8] - t[7]) / reps - cp;
  }
  out[tid] = S[tid] + S[70 * LDS + (tid & 63)] + acc[0][0][0];
}

__global__ void __launch_bounds__(256, 1) stamp_run(double* out) {
  extern __shared__ double sm[];
  double* S = sm;
  double* L = sm + 4 * T * LDS;
  __shared__ double rinv[T];
  __shared__ int sbad;
  const int tid = threadIdx.x;
  for (int e = tid; e < 2 * T * LDS; e += 256) {
    const int r = e / LDS, c = e % LDS;
    S[e] = (c >= T) ? 0.0 : (r == c ? 100.0 + r : 1.0 / (1.0 + r + c));
  }
  for (int e = tid; e < T * LDS; e += 256) {
    const int r = e / LDS, c = e % LDS;
    L[e] = (c >= T) ? 0.0 : ((r == c) ? 10.0 : (c < r ? 0.01 * (r - c) : 0.0));
  }
  __syncthreads();
  potrf_r8<2>(S, 64, 64, rinv, &sbad);
  __syncthreads();
  trsm_blocked(S + T * LDS, L, rinv, 64);
  __syncthreads();
  // warp 0's panel code alone, 8 panels back to back, no other warps
  long long t0 = clock64();
  int bad = 0;
  if (tid < 32)
    for (int p = 0; p < 8; ++p) bad += panel_factor8<2, true>(S, 8 * p, 8 * p, 64, 64, rinv, tid & 31, true);
  __syncthreads();
  long long t1 = clock64();
  if (tid < 32)
    for (int p = 0; p < 8; ++p) bad += panel_factor8<2, false>(S, 8 * p, 8 * p, 64, 61, rinv, tid & 31, true);
  __syncthreads();
  long long t2 = clock64();
  if (tid == 0) { out[300] = (t1 - t0) / 8; out[301] = (t2 - t1) / 8; }
  out[tid] = S[tid] + bad;
}


// debug variants of potrf_r8: MODE 1 = (c) after warp 0 (serialised),
// MODE 2 = no (c); trailing update done by (a)-style full left-looking
template <int MODE>
__device__ int potrf_dbg(double* __restrict__ S, int rv, int cv, double* __restrict__ rinv, int* s_bad) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) *s_bad = -1;
  const int np = (cv + 7) >> 3;
  const int nbr = (rv + 7) >> 3;
  __syncthreads();
  for (int p = 0; p < np; ++p) {
    const int c0 = 8 * p;
    if (MODE == 2) {
      for (int q = 0; q < p; ++q) {
        for (int I = p + w; I < nbr; I += 8) panel8_update_block(S, 8 * q, 8 * I, c0, lane);
        __syncthreads();
      }
    } else if (p > 0) {
      for (int I = p + w; I < nbr; I += 8) panel8_update_block(S, c0 - 8, 8 * I, c0, lane);
      __syncthreads();
    }
    if (w == 0) {
      const int bad = (c0 + 8 <= cv) ? panel_factor8<2, true>(S, c0, c0, rv, cv, rinv, lane, true)
                                     : panel_factor8<2, false>(S, c0, c0, rv, cv, rinv, lane, true);
      if (lane == 0 && bad >= 0 && *s_bad < 0) *s_bad = bad;
    }
    __syncthreads();
    if (MODE == 1 && w > 0 && p > 0) {
      const int ncb = (cv + 7) >> 3;
      for (int I = p + w; I < nbr; I += 7) {
        const int j1 = min(I + 1, ncb);
        if (p + 1 < j1) strip8_gemm(S, S, S, c0 - 8, 8 * I, p + 1, j1, lane);
      }
    }
    __syncthreads();
  }
  return *s_bad;
}

// 64x64x64 update with 32x32 per warp on warps 0..3 (4 A + 4 B fragment
// loads per 16 DMMAs instead of 2 + 4 per 8)
__device__ __forceinline__ void dmma_tile32(double (&acc)[4][4][2], const double* __restrict__ A,
                                            const double* __restrict__ B, int lane, int rb0, int cb0) {
#pragma unroll 2
  for (int kk = 0; kk < T; kk += 4) {
    double av[4], bv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) av[a] = -A[(rb0 + 8 * a + (lane >> 2)) * LDS + kk + (lane & 3)];
#pragma unroll
    for (int q = 0; q < 4; ++q) bv[q] = B[(cb0 + 8 * q + (lane >> 2)) * LDS + kk + (lane & 3)];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int q = 0; q < 4; ++q) dmma8x8x4(acc[a][q][0], acc[a][q][1], av[a], bv[q]);
  }
}
__global__ void __launch_bounds__(256, 1) dmma_bench(double* out, long long* cyc, int reps) {
  extern __shared__ double sm[];
  double* S = sm;
  double* L = sm + T * LDS;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  for (int e = tid; e < T * LDS; e += 256) {
    S[e] = 0.001 * e;
    L[e] = 0.002 * (e % 97);
  }
  __syncthreads();
  long long t0 = clock64();
  double acc[2][4][2] = {};
  const int rb0 = (w >> 1) * 16, cb0 = (w & 1) * 32;
  for (int rep = 0; rep < reps; ++rep) {
    dmma_tile<true>(acc, L, L, lane, rb0, cb0);
    __syncthreads();
  }
  long long t1 = clock64();
  double acc4[4][4][2] = {};
  for (int rep = 0; rep < reps; ++rep) {
    if (w < 4) dmma_tile32(acc4, L, L, lane, (w >> 1) * 32, (w & 1) * 32);
    __syncthreads();
  }
  long long t2 = clock64();
  if (tid == 0) {
    cyc[0] = (t1 - t0) / reps;
    cyc[1] = (t2 - t1) / reps;
  }
  out[tid] = acc[0][0][0] + acc[1][3][1] + acc4[0][0][0] + acc4[3][3][1];
}

// correctness: residual max |(L L^T)[r][c] - A[r][c]| (c <= r, c < cv) of
// potrf64_panel8 and potrf_r8<2>, and trsm_blocked vs trsm_rows
__global__ void __launch_bounds__(256, 1) check(double* err, int cv, int dbg) {
  extern __shared__ double sm[];
  double* S1 = sm;
  double* S2 = sm + T * LDS;
  double* A = sm + 2 * T * LDS;
  double* X1 = sm + 4 * T * LDS;
  double* X2 = sm + 5 * T * LDS;
  __shared__ double rinv1[T], rinv2[T];
  __shared__ int sbad;
  const int tid = threadIdx.x;
  for (int e = tid; e < T * LDS; e += 256) {
    const int r = e / LDS, c = e % LDS;
    const int lo = r < c ? r : c, hi = r < c ? c : r;
    const double v = (c >= T) ? 0.0 : (r == c ? 40.0 + 0.1 * r : sin(0.37 * hi + 1.3 * lo) * 0.5);
    S1[e] = v;
    S2[e] = v;
    A[e] = v;
  }
  for (int e = tid; e < T * LDS; e += 256) X1[e] = X2[e] = cos(0.11 * e);
  __syncthreads();
  potrf64_panel8(S1, 64, cv, rinv1, &sbad);
  __syncthreads();
  if (dbg == 0) potrf_r8<2>(S2, 64, cv, rinv2, &sbad);
  else if (dbg == 1) potrf_r8<1, 8, true>(S2, 64, cv, rinv2, &sbad);
  else potrf_dbg<2>(S2, 64, cv, rinv2, &sbad);
  __syncthreads();
  if (dbg == 0 && cv == 64 && tid == 0) {
    int cnt = 0;
    for (int c = 0; c < 64 && cnt < 40; ++c)
      for (int r = c; r < 64 && cnt < 40; ++r)
        if (fabs(S1[r * LDS + c] - S2[r * LDS + c]) > 1e-9 * fabs(S1[r * LDS + c]) + 1e-12) {
          printf("diff r %d c %d: %.6g vs %.6g\n", r, c, S1[r * LDS + c], S2[r * LDS + c]);
          ++cnt;
        }
  }
  double m1 = 0.0, m2 = 0.0;
  for (int e = tid; e < T * T; e += 256) {
    const int r = e / T, c = e % T;
    if (c <= r && c < cv) {
      double s1 = 0.0, s2 = 0.0;
      for (int t = 0; t <= c; ++t) {
        s1 += S1[r * LDS + t] * S1[c * LDS + t];
        s2 += S2[r * LDS + t] * S2[c * LDS + t];
      }
      m1 = fmax(m1, fabs(s1 - A[r * LDS + c]));
      m2 = fmax(m2, fabs(s2 - A[r * LDS + c]));
    }
  }
  trsm_rows(X1, S1, rinv1, cv);
  __syncthreads();
  trsm_blocked(X2, S1, rinv1, cv);
  __syncthreads();
  double m3 = 0.0;
  for (int e = tid; e < T * T; e += 256) {
    const int r = e / T, c = e % T;
    if (c < cv) m3 = fmax(m3, fabs(X1[r * LDS + c] - X2[r * LDS + c]) / (fabs(X1[r * LDS + c]) + 1e-3));
  }
  atomicMax((unsigned long long*)&err[0], __double_as_longlong(m1));
  atomicMax((unsigned long long*)&err[1], __double_as_longlong(m2));
  atomicMax((unsigned long long*)&err[2], __double_as_longlong(m3));
}

int main() {
  double *out, *src, *err;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&src, 8 * 64 * 64 * 8);
  cudaMalloc(&err, 64);
  cudaMemset(err, 0, 64);
  cudaMemset(src, 0, 8 * 64 * 64 * 8);
  cudaMalloc(&cyc, 80 * 8);
  const int smem = 6 * T * LDS * 8;
  cudaFuncSetAttribute(tile_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(check, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  check<<<1, 256, smem>>>(err, 64, 0);
  check<<<1, 256, smem>>>(err + 3, 60, 0);
  {
    double* e2; cudaMalloc(&e2, 64); cudaMemset(e2, 0, 64);
    check<<<1, 256, smem>>>(e2, 64, 1);
    check<<<1, 256, smem>>>(e2 + 3, 64, 2);
    double hh[6]; cudaMemcpy(hh, e2, 48, cudaMemcpyDeviceToHost);
    printf("split potrf resid %.2e   dbg2 (left-looking, no c) resid %.2e\n", hh[1], hh[4]);
  }
  tile_bench<<<1, 256, smem>>>(out, cyc, src, 2);
  tile_bench<<<1, 256, smem>>>(out, cyc, src, 20);
  cudaDeviceSynchronize();
  long long h[8];
  double he[6];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  cudaMemcpy(he, err, sizeof(he), cudaMemcpyDeviceToHost);
  printf("{\"copy128_cycles\": %lld, \"potrf64_panel8\": %lld, \"potrf_r8_64\": %lld, \"potrf_r8_split64\": %lld, "
         "\"trsm_rows64\": %lld, \"dmma_update_64x64x64\": %lld, \"load_tile_L2\": %lld, \"trsm_blocked64\": %lld, "
         "\"resid_panel8\": [%.2e, %.2e], \"resid_r8\": [%.2e, %.2e], \"trsm_blocked_vs_rows\": [%.2e, %.2e], \"err\": \"%s\"}\n",
         h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], he[0], he[3], he[1], he[4], he[2], he[5],
         cudaGetErrorString(cudaGetLastError()));
  {
    cudaFuncSetAttribute(dmma_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    dmma_bench<<<1, 256, smem>>>(out, cyc, 4);
    dmma_bench<<<1, 256, smem>>>(out, cyc, 50);
    cudaDeviceSynchronize();
    long long hd[2];
    cudaMemcpy(hd, cyc, sizeof(hd), cudaMemcpyDeviceToHost);
    printf("64x64x64 DMMA update: 16x32 per warp (8 warps) %lld cycles; 32x32 per warp (4 warps) %lld cycles\n",
           hd[0], hd[1]);
  }
  cudaFuncSetAttribute(stamp_run, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  stamp_run<<<1, 256, smem>>>(out);
  stamp_run<<<1, 256, smem>>>(out);
  cudaDeviceSynchronize();
  {
    double o[2]; cudaMemcpy(o, out + 300, 16, cudaMemcpyDeviceToHost);
    printf("panel_factor8 alone (warp 0 only): FULL %.0f  partial %.0f cycles/panel\n", o[0], o[1]);
  }
  return 0;
}
