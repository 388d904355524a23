// Latency probes on one SM: dependent DMMA.8x8x4 chain, independent DMMAs
// (1 warp / 4 warps / 8 warps), LDS.64 -> use, STS -> bar.sync -> LDS round trip,
// bar.sync alone, DFMA chain.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench/mb_dmma_lat bench/microbench_dmma_lat.cu
#include <cstdio>
#include "../paper_cs_0408029_b200/csrc/common.cuh"
using namespace nnls;

__global__ void probe(double* out, long long* cyc, int reps, int nwarps_active) {
  __shared__ double sm[4096];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int e = tid; e < 4096; e += blockDim.x) sm[e] = 1e-3 * (e & 63);
  __syncthreads();
  double c0 = 0, c1 = 0, d[8][2] = {};
  const double a = sm[lane], b = sm[lane + 32];
  long long t0 = clock64();
  if (w < nwarps_active)
    for (int r = 0; r < reps; ++r) dmma8x8x4(c0, c1, a, b);  // dependent chain
  __syncthreads();
  long long t1 = clock64();
  if (w < nwarps_active)
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int q = 0; q < 8; ++q) dmma8x8x4(d[q][0], d[q][1], a, b);  // 8 independent
    }
  __syncthreads();
  long long t2 = clock64();
  // LDS -> dependent address chain
  int idx = lane;
  volatile int* ism = reinterpret_cast<volatile int*>(sm);
  if (tid == 0) for (int e = 0; e < 64; ++e) ism[e] = (e + 1) & 63;
  __syncthreads();
  long long t3 = clock64();
  for (int r = 0; r < reps; ++r) idx = ism[idx];
  long long t4 = clock64();
  // STS -> bar -> LDS round trip (values through smem between two warps)
  double v = lane;
  for (int r = 0; r < reps; ++r) {
    if (w == 0) sm[lane] = v + 1.0;
    __syncthreads();
    v = sm[(lane + 1) & 31];
    __syncthreads();
  }
  long long t5 = clock64();
  for (int r = 0; r < reps; ++r) __syncthreads();
  long long t6 = clock64();
  double x = lane * 1e-3;
  for (int r = 0; r < reps; ++r) x = fma(x, 1.0000001, 1e-9);
  long long t7 = clock64();
  if (tid == 0) {
    cyc[0] = (t1 - t0) / reps;
    cyc[1] = (t2 - t1) / reps;
    cyc[2] = (t4 - t3) / reps;
    cyc[3] = (t5 - t4) / reps;
    cyc[4] = (t6 - t5) / reps;
    cyc[5] = (t7 - t6) / reps;
  }
  out[tid] = c0 + c1 + d[3][1] + d[7][0] + idx + v + x;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 16);
  cudaMalloc(&cyc, 64);
  for (int nw : {1, 2, 4, 8}) {
    probe<<<1, 256>>>(out, cyc, 16, nw);
    probe<<<1, 256>>>(out, cyc, 512, nw);
    cudaDeviceSynchronize();
    long long h[6];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    printf("active warps %d: dependent DMMA %lld cyc/op; 8 independent DMMAs per warp %lld cyc/iter; "
           "LDS chain %lld; STS-bar-LDS-bar %lld; bar.sync %lld; DFMA chain %lld\n",
           nw, h[0], h[1], h[2], h[3], h[4], h[5]);
  }
  return 0;
}
