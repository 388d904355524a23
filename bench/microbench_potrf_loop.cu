// Long-running loop of one Cholesky tile primitive, for ncu source-level
// stall sampling: ./mb_potrf_loop <0: potrf_r8<2> | 1: trsm_blocked | 2: dmma update>
#include <cstdio>
#include <cstdlib>

#include "../paper_cs_0408029_b200/csrc/cholesky.cu"
#include "trsm_blocked.cuh"

using namespace nnls;

__global__ void __launch_bounds__(256, 1) loop_kernel(double* out, int reps, int mode) {
  extern __shared__ double sm[];
  double* S = sm;
  double* B = sm + T * LDS;
  double* L = sm + 2 * T * LDS;
  __shared__ double rinv[T];
  __shared__ int sbad;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  for (int e = tid; e < T * LDS; e += 256) {
    const int r = e / LDS, c = e % LDS;
    B[e] = (c >= T) ? 0.0 : (r == c ? 100.0 + r : 1.0 / (1.0 + r + c));
    L[e] = (c >= T) ? 0.0 : ((r == c) ? 10.0 : (c < r ? 0.01 * (r - c) : 0.0));
  }
  if (tid < T) rinv[tid] = 0.1;
  __syncthreads();
  double acc[2][4][2] = {};
  const int rb0 = (w >> 1) * 16, cb0 = (w & 1) * 32;
  for (int rep = 0; rep < reps; ++rep) {
    for (int e = tid; e < T * LDS; e += 256) S[e] = B[e];
    __syncthreads();
    if (mode == 0) potrf_r8<2>(S, 64, 64, rinv, &sbad);
    else if (mode == 1) trsm_blocked(S, L, rinv, 64);
    else dmma_tile<true>(acc, L, L, lane, rb0, cb0);
    __syncthreads();
  }
  out[tid] = S[tid] + acc[0][0][0];
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 0;
  double* out;
  cudaMalloc(&out, 1 << 16);
  const int smem = 3 * T * LDS * 8;
  cudaFuncSetAttribute(loop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  loop_kernel<<<1, 256, smem>>>(out, 2000, mode);
  cudaDeviceSynchronize();
  printf("mode %d: %s\n", mode, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
