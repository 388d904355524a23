// Microbenchmark of the Cholesky tile primitives (cycle counts on one SM):
// warp_potrf32, trsm_rows (64x64), the DMMA 64x64x64 update.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb_chol bench/microbench_chol_tile.cu
#include <cstdio>

#include "../paper_cs_0408029_b200/csrc/cholesky.cu"

using namespace nnls;

__global__ void __launch_bounds__(256, 1) tile_bench(double* out, long long* cyc, int reps) {
  extern __shared__ double sm[];
  double* S = sm;
  double* L = sm + T * LDS;
  __shared__ double rinv[T];
  __shared__ double colbuf[64];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // SPD tile: diagonally dominant
  for (int e = tid; e < T * T; e += 256) {
    const int r = e / T, c = e % T;
    S[r * LDS + c] = (r == c) ? 100.0 + r : 1.0 / (1.0 + r + c);
    L[r * LDS + c] = (r == c) ? 10.0 : (c < r ? 0.01 * (r - c) : 0.0);
  }
  if (tid < T) rinv[tid] = 0.1;
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (w == 0) {
      double a[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) a[k] = S[lane * LDS + k];
      warp_potrf32(a, 32, lane, rinv, L, colbuf);
    }
    __syncthreads();
  }
  long long t1 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (w == 0) warp_trtri32(S, rinv, 32, lane, L + 32, nullptr);
    __syncthreads();
  }
  long long t2 = clock64();
  double acc[2][4][2] = {};
  const int rb0 = (w >> 1) * 16, cb0 = (w & 1) * 32;
  for (int rep = 0; rep < reps; ++rep) {
#pragma unroll 4
    for (int kk = 0; kk < T; kk += 4) {
      double av[2], bv[4];
#pragma unroll
      for (int a = 0; a < 2; ++a) av[a] = -S[(rb0 + 8 * a + (lane >> 2)) * LDS + kk + (lane & 3)];
#pragma unroll
      for (int q = 0; q < 4; ++q) bv[q] = L[(cb0 + 8 * q + (lane >> 2)) * LDS + kk + (lane & 3)];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int q = 0; q < 4; ++q) dmma8x8x4(acc[a][q][0], acc[a][q][1], av[a], bv[q]);
    }
    __syncthreads();
  }
  long long t3 = clock64();
  __shared__ int sbad;
  for (int rep = 0; rep < reps; ++rep) {
    potrf64_panel8(L, 64, 64, rinv, &sbad);
    __syncthreads();
  }
  long long t4 = clock64();
  for (int rep = 0; rep < reps * 64; ++rep) {
    __syncthreads();
  }
  long long t5 = clock64();
  if (tid == 0) cyc[4] = (t5 - t4) / (reps * 64);
  if (tid == 0) {
    cyc[0] = (t1 - t0) / reps;
    cyc[1] = (t2 - t1) / reps;
    cyc[2] = (t3 - t2) / reps;
    cyc[3] = (t4 - t3) / reps;
  }
  out[tid] = S[tid] + L[tid] + acc[0][0][0] + acc[1][3][1];
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMemset(out, 0, 1 << 20);
  cudaMalloc(&cyc, 64);
  const int smem = 4 * T * LDS * 8;
  cudaFuncSetAttribute(tile_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  tile_bench<<<1, 256, smem>>>(out, cyc, 2);
  tile_bench<<<1, 256, smem>>>(out, cyc, 20);
  cudaDeviceSynchronize();
  long long h[5];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("{\"syncthreads256_cycles\": %lld}\n", h[4]);
  printf("{\"potrf32_cycles\": %lld, \"trsm_rows64_cycles\": %lld, \"dmma_64x64x64_cycles\": %lld, "
         "\"load_tile_cycles\": %lld, \"err\": \"%s\"}\n",
         h[0], h[1], h[2], h[3], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
