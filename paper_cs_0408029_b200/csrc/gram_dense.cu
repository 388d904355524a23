// gram_dense.cu -- a1 for dense A (NEXT-1: the Fig. 2
// workloads at density 1.0): G = A^T A as a DSYRK on the
// FP64 tensor pipe.
//
// "For an m x n dense matrix A, the matrix multiplication required to
// form A^T A requires n^2 m flops" -- at density 1 the Gram is the dominant
// O(m n^2) step (the sparse scatter kernels of ingest_gram.cu are built for
// m d^2 ~ 1-5 MACs per output entry).  Used when the load's exactness check
// passes for A (gram_A_exact: every product and partial sum of A^T A exact in
// FP64, as for BASELINE's 2^-12-quantized inputs), so the DMMA summation
// order gives the same bits as the oracle's sequential sum; and when A is
// dense enough.
//
// B200 design
//   * densify: CSR rows [r0, r1) -> a TILED dense copy, tile (kb, jb) = rows
//     64 kb.., columns 64 jb.. stored as one contiguous 64 x 68 block (the
//     shared-memory layout), zero padded -- one bulk copy per operand tile.
//   * SYRK: one CTA per lower tile (I, J) of G (persistent over tiles).  A
//     producer warp streams At(kb, I) and At(kb, J), kb = 0 .. M/64-1, into a
//     2-stage mbarrier ring with cp.async.bulk; 8 consumer warps accumulate
//     G_IJ += At(kb,I)^T At(kb,J) with DMMA 8x8x4 (16 x 32 accumulators per
//     warp, operands read transposed from shared memory -- with the 68-double
//     row stride every fragment load is the minimal 2 wavefronts).  The tile
//     leaves through shared memory: the lower block row-coalesced, its mirror
//     transposed (full symmetric output), or only j <= i into the packed row
//     shard buffer.
//   * c = A^T b: a warp per column over the CSC when its sums are exact, else
//     a thread per column in increasing row order (the oracle's sequence).
#include <cuda_runtime.h>

#include "common.cuh"
#include "kernels.cuh"

namespace nnls {

namespace {
constexpr int T = kTile;
constexpr int LDS = T + 4;
constexpr int TS = T * LDS;
constexpr int kStagesD = 2;   // (2 stages x 2 operand tiles + the output staging tile: 174 KB)
constexpr int kCons = 256;            // consumer threads
constexpr int kThr = kCons + 32;      // + the producer warp

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mb_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mb_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned parity) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(saddr(b)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void bulk_tile(double* dst, const double* src, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   saddr(dst)),
               "l"(src), "n"(TS * 8), "r"(saddr(b))
               : "memory");
}
__device__ __forceinline__ void bar_cons() { asm volatile("bar.sync 1, %0;\n" ::"n"(kCons) : "memory"); }
__device__ __forceinline__ void bar_all() { asm volatile("bar.sync 2, %0;\n" ::"n"(kThr) : "memory"); }

// acc (16 x 32 per warp) += X^T Y over K = 64 for 64 x 64 smem tiles stored
// k-major (X[k][m], Y[k][n]): G_IJ[m][n] += sum_k X[k][m] Y[k][n].
__device__ __forceinline__ void dmma_tile_tn(double (&acc)[2][4][2], const double* __restrict__ X,
                                             const double* __restrict__ Y, int lane, int rb0, int cb0) {
  const int rq = lane >> 2, kq = lane & 3;
#pragma unroll 4
  for (int kk = 0; kk < T; kk += 4) {
    double av[2], bv[4];
#pragma unroll
    for (int a = 0; a < 2; ++a) av[a] = X[(kk + kq) * LDS + rb0 + 8 * a + rq];
#pragma unroll
    for (int q = 0; q < 4; ++q) bv[q] = Y[(kk + kq) * LDS + cb0 + 8 * q + rq];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int q = 0; q < 4; ++q) dmma8x8x4(acc[a][q][0], acc[a][q][1], av[a], bv[q]);
  }
}
}  // namespace

// rows [r0, r1) of the CSR into the tiled dense copy (zeroed by the caller):
// a warp per row, lanes over its entries
__global__ void __launch_bounds__(256) densify_kernel(const int32_t* __restrict__ rowptr,
                                                      const int32_t* __restrict__ colind,
                                                      const double* __restrict__ vals, int r0, int r1, int ntc,
                                                      double* __restrict__ At) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = r0 + gw; r < r1; r += nw) {
    const int rl = r - r0, kb = rl / T, ri = rl % T;
    for (int e = rowptr[r] + lane; e < rowptr[r + 1]; e += 32) {
      const int c = colind[e];
      At[((size_t)kb * ntc + c / T) * TS + ri * LDS + c % T] = vals[e];
    }
  }
}

// c_i = sum over column i of a_ri b_r in increasing row order, separate
// multiply / add (the oracle's sequence: bitwise for any inputs) -- a thread
// per column, for when the products or sums are not exact
__global__ void __launch_bounds__(128) dense_c_ordered_kernel(int n, const int32_t* __restrict__ colptr,
                                                              const int32_t* __restrict__ rowind,
                                                              const double* __restrict__ cvals,
                                                              const double* __restrict__ b, int r0, int r1,
                                                              double* __restrict__ c) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int t = colptr[j]; t < colptr[j + 1]; ++t) {
      const int r = rowind[t];
      if (r >= r0 && r < r1) s = __dadd_rn(s, __dmul_rn(cvals[t], b[r]));
    }
    c[j] = s;
  }
}

// c_i = sum over column i of a_ri b_r, rows [r0, r1) (CSC; exact inputs)
__global__ void __launch_bounds__(256) dense_c_kernel(int n, const int32_t* __restrict__ colptr,
                                                      const int32_t* __restrict__ rowind,
                                                      const double* __restrict__ cvals, const double* __restrict__ b,
                                                      int r0, int r1, double* __restrict__ c) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (int j = gw; j < n; j += nw) {
    double s = 0.0;
    for (int t = colptr[j] + lane; t < colptr[j + 1]; t += 32) {
      const int r = rowind[t];
      if (r >= r0 && r < r1) s += cvals[t] * b[r];
    }
    s = warp_sum(s);
    if (lane == 0) c[j] = s;
  }
}

// G (n rows of stride ldg; ldg <= 0: packed lower) = At^T At over nkb row tiles
__global__ void __launch_bounds__(kThr, 1) dense_syrk_kernel(const double* __restrict__ At, int nkb, int ntc, int n,
                                                               double* __restrict__ G, int ldg) {
  extern __shared__ __align__(128) double sm[];
  __shared__ unsigned long long full[kStagesD], empty[kStagesD];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    for (int k = 0; k < kStagesD; ++k) {
      mb_init(&full[k], 1);
      mb_init(&empty[k], kCons / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  bar_all();
  double* S = sm + (size_t)2 * kStagesD * TS;  // output staging
  const int ntiles = ntc * (ntc + 1) / 2;
  unsigned cnt = 0;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    int I = (int)((sqrt(8.0 * tile + 1.0) - 1.0) * 0.5);
    while (I * (I + 1) / 2 > tile) --I;
    while ((I + 1) * (I + 2) / 2 <= tile) ++I;
    const int J = tile - I * (I + 1) / 2;
    const bool diag = I == J;
    if (w == kCons / 32) {  // ---- producer
      if (lane == 0) {
        for (int kb = 0; kb < nkb; ++kb, ++cnt) {
          const int s = (int)(cnt % kStagesD);
          const unsigned use = cnt / kStagesD;
          if (use > 0) mb_wait(&empty[s], (use - 1) & 1);
          double* slot = sm + (size_t)(2 * s) * TS;
          mb_expect(&full[s], (diag ? 1u : 2u) * TS * 8);
          bulk_tile(slot, At + ((size_t)kb * ntc + I) * TS, &full[s]);
          if (!diag) bulk_tile(slot + TS, At + ((size_t)kb * ntc + J) * TS, &full[s]);
        }
      } else {
        cnt += nkb;
      }
    } else {  // ---- consumers
      const int rb0 = (w >> 1) * 16, cb0 = (w & 1) * 32;
      double acc[2][4][2] = {};
      for (int kb = 0; kb < nkb; ++kb, ++cnt) {
        const int s = (int)(cnt % kStagesD);
        mb_wait(&full[s], (cnt / kStagesD) & 1);
        const double* slot = sm + (size_t)(2 * s) * TS;
        dmma_tile_tn(acc, slot, diag ? slot : slot + TS, lane, rb0, cb0);
        __syncwarp();
        if (lane == 0) mb_arrive(&empty[s]);
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int v = 0; v < 2; ++v)
            S[(rb0 + 8 * a + (lane >> 2)) * LDS + cb0 + 8 * q + 2 * (lane & 3) + v] = acc[a][q][v];
      bar_cons();
      const int rv = min(T, n - I * T), cv = min(T, n - J * T);
      for (int e = tid; e < T * T; e += kCons) {
        const int i = e / T, j = e % T;  // lower block, row-coalesced
        if (i < rv && j < cv) {
          const int gi = I * T + i, gj = J * T + j;
          if (ldg > 0) G[(size_t)gi * ldg + gj] = S[i * LDS + j];
          else if (gj <= gi) G[(size_t)gi * (gi + 1) / 2 + gj] = S[i * LDS + j];
        }
      }
      if (ldg > 0 && !diag)
        for (int e = tid; e < T * T; e += kCons) {
          const int j = e / T, i = e % T;  // mirror: row J*T + j of G, columns I*T + i
          if (i < rv && j < cv) G[(size_t)(J * T + j) * ldg + I * T + i] = S[i * LDS + j];
        }
      bar_cons();
    }
  }
}

size_t gram_dense_doubles(int rows, int n) {
  const size_t nkb = (size_t)(rows + T - 1) / T, ntc = (size_t)(n + T - 1) / T;
  return nkb * ntc * TS;
}

cudaError_t launch_gram_dense(int n, const int32_t* rowptr, const int32_t* colind, const double* vals,
                              const int32_t* colptr, const int32_t* rowind, const double* cvals, const double* b,
                              int row_begin, int row_end, double* At, double* G, int ldg, double* c, int sm_count,
                              cudaStream_t s, bool c_exact) {
  const int rows = row_end - row_begin;
  const int nkb = (rows + T - 1) / T, ntc = (n + T - 1) / T;
  cudaError_t e = cudaMemsetAsync(At, 0, sizeof(double) * gram_dense_doubles(rows, n), s);
  if (e != cudaSuccess) return e;
  int blocks = (rows + 7) / 8;
  if (blocks > sm_count * 16) blocks = sm_count * 16;
  if (blocks < 1) blocks = 1;
  densify_kernel<<<blocks, 256, 0, s>>>(rowptr, colind, vals, row_begin, row_end, ntc, At);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  int cb = (n + 7) / 8;
  if (cb > sm_count * 8) cb = sm_count * 8;
  if (cb < 1) cb = 1;
  if (c_exact) dense_c_kernel<<<cb, 256, 0, s>>>(n, colptr, rowind, cvals, b, row_begin, row_end, c);
  else dense_c_ordered_kernel<<<(n + 127) / 128, 128, 0, s>>>(n, colptr, rowind, cvals, b, row_begin, row_end, c);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const size_t smem = sizeof(double) * (size_t)(2 * kStagesD + 1) * TS;
  static DeviceOnce once;
  if (!device_once(once, [&]() {
        e = cudaFuncSetAttribute(dense_syrk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        return e == cudaSuccess ? 1 : 0;
      }))
    return e;
  const int ntiles = ntc * (ntc + 1) / 2;
  int grid = ntiles < sm_count ? ntiles : sm_count;
  if (grid < 1) grid = 1;
  dense_syrk_kernel<<<grid, kThr, smem, s>>>(At, nkb, ntc, n, G, ldg);
  return cudaGetLastError();
}

}  // namespace nnls
