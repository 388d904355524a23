// condest.cu -- NEXT-2: the condition estimate that decides
// whether the final LSQR is needed.
//
// PAPER.md P:129 (Section 3): "We can estimate the relative error kappa^2 eps
// of each normal equations solution by computing the condition number
// kappa^2 of A_F^T A_F with the LAPACK function dpocon.  Since we have
// already computed the Cholesky factorization ... this takes very little
// additional time.  This is used to determine when a switch to a final step
// with LSQR is necessary for error control."  dpocon = ||M||_1 times
// Hager's estimate of ||M^-1||_1 with Higham's refinements (LAPACK dlacn2),
// M = (A^T A)_FF = L L^T, M^-1 applied by two triangular solves with the
// factor the pivot loop already holds (the tiles of cholesky.cu).  The step
// order is dlacn2's: x = 1/f; y = B x; xi = sign(y); z = B xi; j = argmax|z|;
// then up to 5 rounds of x = e_j (stop on a repeated sign vector or no
// growth), and the alternating-sign vector's 2||B x||_1/(3f) as a floor.
//
// B200 design: one 8-CTA thread-block cluster runs the whole estimator (at
// most 11 applications of M^-1, i.e. 22 triangular solves).  A tile solve
// L z = v walks the tile columns J: the CTA owning tile row J forms
// z_J = Linv_JJ s_J (the inverse diagonal tiles exist already), publishes it
// through global memory, one cluster barrier, and every CTA updates its own
// tile rows s_I -= L(I,J) z_J (tile rows are dealt round-robin, so the
// updates of a step are spread over the cluster); the owner of J+1 updates
// s_{J+1} and forms z_{J+1} FIRST, so one barrier per tile column is the
// whole critical path.  L^T x = z is the mirror image with tile COLUMNS
// dealt round-robin.  Every CTA then runs dlacn2's scalar control flow
// redundantly on the same global vectors with the same fixed-order
// reductions, so all take identical decisions.  ||M||_1 comes from a
// grid-wide kernel over G's rows (symmetry: column j of M = row Fidx[j] of G
// restricted to F), combined with an order-independent atomic max.
#include <cuda_runtime.h>
#include <math.h>

#include "common.cuh"
#include "kernels.cuh"

namespace nnls {

namespace {
constexpr int T = kTile;
constexpr int LDS = T + 4;
constexpr int TS = T * LDS;
constexpr int kCl = 8;       // cluster size
constexpr int kCT = 256;     // threads per CTA
__host__ __device__ inline int tidx(int i, int j) { return i * (i + 1) / 2 + j; }

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

// out[r] (r < rv) = base[r] - sum_{c < cv} A[r][c] v[c]   (A: one tile, global)
// (base == nullptr: out[r] = sum A[r][c] v[c]).  Thread t: row t/4, 16 columns.
__device__ __forceinline__ void tile_gemv(double* __restrict__ out, const double* __restrict__ base,
                                          const double* __restrict__ A, const double* __restrict__ v, int rv,
                                          int cv) {
  const int t = threadIdx.x, r = t >> 2, q = t & 3;
  double s = 0.0;
  if (r < rv) {
#pragma unroll
    for (int c2 = 0; c2 < 16; c2 += 2) {
      const int c = 16 * q + c2;
      if (c < cv) {
        const double2 a = __ldcg(reinterpret_cast<const double2*>(A + r * LDS + c));
        s = fma(a.x, __ldcg(&v[c]), s);
        if (c + 1 < cv) s = fma(a.y, __ldcg(&v[c + 1]), s);
      }
    }
  }
  s += __shfl_xor_sync(kFull, s, 1);
  s += __shfl_xor_sync(kFull, s, 2);
  if (q == 0 && r < rv) out[r] = base != nullptr ? __ldcg(&base[r]) - s : s;
}
// out[c] (c < cv) = base[c] - sum_{r < rv} A[r][c] v[r]   (the transposed tile)
__device__ __forceinline__ void tile_gemv_t(double* __restrict__ out, const double* __restrict__ base,
                                            const double* __restrict__ A, const double* __restrict__ v, int rv,
                                            int cv, double* red) {
  const int t = threadIdx.x, c = t & 63, q = t >> 6;
  double s = 0.0;
  if (c < cv)
    for (int r = 16 * q; r < 16 * q + 16 && r < rv; ++r) s = fma(__ldcg(&A[r * LDS + c]), __ldcg(&v[r]), s);
  red[q * 64 + c] = s;
  __syncthreads();
  if (t < cv) {
    const double tot = (red[t] + red[64 + t]) + (red[128 + t] + red[192 + t]);
    out[t] = base != nullptr ? __ldcg(&base[t]) - tot : tot;
  }
  __syncthreads();
}

// z = L^-1 v (forward).  s: scratch f, owned tile rows only.
__device__ void tile_forward(const double* __restrict__ Lt, const double* __restrict__ Linv, int f,
                             const double* __restrict__ v, double* __restrict__ s, double* __restrict__ z,
                             unsigned me) {
  const int nt = (f + T - 1) / T;
  for (int I = (int)me; I < nt; I += kCl)  // s_I = v_I
    for (int r = threadIdx.x; r < min(T, f - I * T); r += kCT) s[I * T + r] = __ldcg(&v[I * T + r]);
  __syncthreads();
  if (me == 0) {  // z_0
    tile_gemv(z, nullptr, Linv, s, min(T, f), min(T, f));
  }
  __threadfence();
  cluster_sync_all();
  for (int J = 0; J < nt; ++J) {
    const int cvJ = min(T, f - J * T);
    const double* zJ = z + J * T;
    // the owner of J+1: its update and z_{J+1} first (the critical path)
    if (J + 1 < nt && (J + 1) % kCl == (int)me) {
      const int rv = min(T, f - (J + 1) * T);
      tile_gemv(s + (J + 1) * T, s + (J + 1) * T, Lt + (size_t)tidx(J + 1, J) * TS, zJ, rv, cvJ);
      __syncthreads();
      tile_gemv(z + (J + 1) * T, nullptr, Linv + (size_t)(J + 1) * TS, s + (J + 1) * T, rv, rv);
      __threadfence();
    }
    for (int I = (int)me; I < nt; I += kCl) {
      if (I <= J + 1) continue;
      tile_gemv(s + I * T, s + I * T, Lt + (size_t)tidx(I, J) * TS, zJ, min(T, f - I * T), cvJ);
    }
    __syncthreads();
    cluster_sync_all();
  }
}

// x = L^-T z (backward).  t: scratch f, owned tile columns only.
__device__ void tile_backward(const double* __restrict__ Lt, const double* __restrict__ Linv, int f,
                              const double* __restrict__ z, double* __restrict__ t, double* __restrict__ x,
                              unsigned me, double* red) {
  const int nt = (f + T - 1) / T;
  for (int K = (int)me; K < nt; K += kCl)
    for (int r = threadIdx.x; r < min(T, f - K * T); r += kCT) t[K * T + r] = __ldcg(&z[K * T + r]);
  __syncthreads();
  const int L0 = nt - 1;
  if (L0 % kCl == (int)me) {
    const int cv = min(T, f - L0 * T);
    tile_gemv_t(x + L0 * T, nullptr, Linv + (size_t)L0 * TS, t + L0 * T, cv, cv, red);
  }
  __threadfence();
  cluster_sync_all();
  for (int J = nt - 1; J >= 0; --J) {
    const int rvJ = min(T, f - J * T);
    const double* xJ = x + J * T;
    if (J - 1 >= 0 && (J - 1) % kCl == (int)me) {  // t_{J-1} and x_{J-1} first
      const int cv = min(T, f - (J - 1) * T);
      tile_gemv_t(t + (J - 1) * T, t + (J - 1) * T, Lt + (size_t)tidx(J, J - 1) * TS, xJ, rvJ, cv, red);
      tile_gemv_t(x + (J - 1) * T, nullptr, Linv + (size_t)(J - 1) * TS, t + (J - 1) * T, cv, cv, red);
      __threadfence();
    }
    for (int K = (int)me; K < nt; K += kCl) {
      if (K >= J - 1) continue;
      tile_gemv_t(t + K * T, t + K * T, Lt + (size_t)tidx(J, K) * TS, xJ, rvJ, min(T, f - K * T), red);
    }
    __syncthreads();
    cluster_sync_all();
  }
}

// fixed-order block reductions (identical results in every CTA)
__device__ double block_sum_abs(const double* v, int f, double* red) {
  double s = 0.0;
  for (int i = threadIdx.x; i < f; i += kCT) s += fabs(__ldcg(&v[i]));
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  double tot = 0.0;
  for (int w = 0; w < kCT / 32; ++w) tot += red[w];
  __syncthreads();
  return tot;
}
// first index of max |v_i| (LAPACK idamax)
__device__ int block_iamax(const double* v, int f, double* redv, int* redi) {
  double best = -1.0;
  int bi = 0;
  for (int i = threadIdx.x; i < f; i += kCT) {
    const double a = fabs(__ldcg(&v[i]));
    if (a > best) {
      best = a;
      bi = i;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(kFull, best, o);
    const int oi = __shfl_xor_sync(kFull, bi, o);
    if (ob > best || (ob == best && oi < bi)) {
      best = ob;
      bi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    redv[threadIdx.x >> 5] = best;
    redi[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  double b = redv[0];
  int j = redi[0];
  for (int w = 1; w < kCT / 32; ++w)
    if (redv[w] > b || (redv[w] == b && redi[w] < j)) {
      b = redv[w];
      j = redi[w];
    }
  __syncthreads();
  return j;
}
}  // namespace

// ||M||_1 = max_j sum_{i in F} |G[Fidx[j]][Fidx[i]]| (symmetric: row Fidx[j]).
__global__ void __launch_bounds__(256) condest_norm1_kernel(const double* __restrict__ G, int ldg,
                                                            const int32_t* __restrict__ Fidx, DevState* st,
                                                            unsigned long long* out) {
  const int f = st->f;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  double mx = 0.0;
  for (int j = gw; j < f; j += nw) {
    const double* Gj = G + (size_t)Fidx[j] * ldg;
    double s = 0.0;
    for (int i = lane; i < f; i += 32) s += fabs(Gj[Fidx[i]]);
    s = warp_sum(s);
    mx = fmax(mx, s);
  }
  if (lane == 0 && mx > 0.0) atomicMax(out, dbits(mx));
}

struct CondArgs {
  const double* Lt;
  const double* Linv;
  DevState* st;
  const unsigned long long* norm1;  // bits of ||M||_1
  double* work;                     // 6 f doubles: x, y, xi, s, z, t
  double threshold;                 // refine iff kappa * 2^-52 > threshold
};

__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kCT) condest_kernel(CondArgs a) {
  __shared__ double red[256];
  __shared__ int redi[8];
  DevState* st = a.st;
  const int f = st->f;
  if (st->status != 0 || f <= 0) return;  // (uniform over the cluster)
  const unsigned me = cluster_rank();
  double* x = a.work;
  double* y = x + f;
  double* xi = y + f;
  double* s = xi + f;
  double* z = s + f;
  double* t = z + f;
  const int tid = threadIdx.x;
  // B v = M^-1 v = L^-T L^-1 v  (in -> out; z, s, t scratch)
  auto applyB = [&](const double* in, double* out) {
    tile_forward(a.Lt, a.Linv, f, in, s, z, me);
    tile_backward(a.Lt, a.Linv, f, z, t, out, me, red);
  };
  // step 1: x = 1/f
  for (int i = tid; i < f; i += kCT)
    if (me == 0) x[i] = 1.0 / (double)f;
  __threadfence();
  cluster_sync_all();
  applyB(x, y);
  double est;
  if (f == 1) {
    est = fabs(__ldcg(&y[0]));
  } else {
    est = block_sum_abs(y, f, red);
    // step 2: xi = sign(y); z = B xi; j = argmax |z|
    if (me == 0)
      for (int i = tid; i < f; i += kCT) xi[i] = __ldcg(&y[i]) >= 0.0 ? 1.0 : -1.0;
    __threadfence();
    cluster_sync_all();
    applyB(xi, y);
    int j = block_iamax(y, f, red, redi), iter = 2;
    for (;;) {  // step 3
      cluster_sync_all();  // (everyone read y / xi)
      if (me == 0)
        for (int i = tid; i < f; i += kCT) x[i] = (i == j) ? 1.0 : 0.0;
      __threadfence();
      cluster_sync_all();
      applyB(x, y);
      const double est_old = est;
      est = block_sum_abs(y, f, red);
      int diff = 0;
      for (int i = tid; i < f; i += kCT) diff |= ((__ldcg(&y[i]) >= 0.0 ? 1.0 : -1.0) != __ldcg(&xi[i]));
      const int same = !__syncthreads_or(diff);
      if (same || est <= est_old) break;
      cluster_sync_all();  // (everyone compared against xi)
      if (me == 0)
        for (int i = tid; i < f; i += kCT) xi[i] = __ldcg(&y[i]) >= 0.0 ? 1.0 : -1.0;
      __threadfence();
      cluster_sync_all();
      applyB(xi, y);
      const int jlast = j;
      j = block_iamax(y, f, red, redi);
      if (__ldcg(&y[jlast]) != fabs(__ldcg(&y[j])) && iter < 5) {
        ++iter;
        continue;
      }
      break;
    }
    // step 5: the alternating-sign vector
    cluster_sync_all();
    if (me == 0)
      for (int i = tid; i < f; i += kCT) x[i] = ((i & 1) ? -1.0 : 1.0) * (1.0 + (double)i / (double)(f - 1));
    __threadfence();
    cluster_sync_all();
    applyB(x, y);
    const double temp = 2.0 * block_sum_abs(y, f, red) / (3.0 * (double)f);
    if (temp > est) est = temp;
  }
  if (me == 0 && tid == 0) {
    const double n1 = __longlong_as_double((long long)*a.norm1);
    const double kappa = n1 * est;
    st->kappa = kappa;
    st->refined = (kappa * 0x1p-52 > a.threshold) ? 1 : 0;
  }
}

cudaError_t launch_condest(const double* G, int ldg, const int32_t* Fidx, const double* Lt, int n, DevState* st,
                           double* work, unsigned long long* norm1, double threshold, int sm_count, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(norm1, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  int blocks = (n + 7) / 8;
  if (blocks > sm_count * 8) blocks = sm_count * 8;
  if (blocks < 1) blocks = 1;
  condest_norm1_kernel<<<blocks, 256, 0, s>>>(G, ldg, Fidx, st, norm1);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int ntr = (n + 1 + T - 1) / T;
  const int tri = ntr * (ntr + 1) / 2;
  CondArgs a;
  a.Lt = Lt;
  a.Linv = Lt + (size_t)tri * TS;
  a.st = st;
  a.norm1 = norm1;
  a.work = work;
  a.threshold = threshold;
  condest_kernel<<<kCl, kCT, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace nnls
