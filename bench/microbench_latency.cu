// Single-warp dependent-chain latencies on B200 (cycles per op): DFMA, DMUL,
// FFMA, SHFL (64-bit), rsqrt(double), 1.0/x, LDS.64.
#include <cstdio>
__global__ void lat(double* out, long long* cyc, int n) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  sm[lane] = lane; sm[lane + 32] = lane;
  __syncwarp();
  double x = 1.0 + lane * 1e-9, y = 0.999999;
  float xf = 1.0f + lane * 1e-6f;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 1e-9);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = x * y;
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) xf = fmaf(xf, 0.9999f, 1e-6f);
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffff, x, (lane + 1) & 31);
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x + 1.0);
  long long t5 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.0);
  long long t6 = clock64();
  int idx = lane;
  for (int i = 0; i < n; ++i) { double v = sm[idx]; idx = ((int)v + 1) & 63; }
  long long t7 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
  long long t8 = clock64();
  if (lane == 0) {
    cyc[0] = (t1 - t0) / n; cyc[1] = (t2 - t1) / n; cyc[2] = (t3 - t2) / n; cyc[3] = (t4 - t3) / n;
    cyc[4] = (t5 - t4) / n; cyc[5] = (t6 - t5) / n; cyc[6] = (t7 - t6) / n; cyc[7] = (t8 - t7) / n;
  }
  out[lane] = x + xf + idx;
}
// throughput of independent DFMA from ONE warp (16 chains)
__global__ void thr(double* out, long long* cyc, int n) {
  double a[16];
  for (int k = 0; k < 16; ++k) a[k] = threadIdx.x + k;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) a[k] = fma(a[k], 0.999, 1e-9);
  }
  long long t1 = clock64();
  double s = 0; for (int k = 0; k < 16; ++k) s += a[k];
  if (threadIdx.x == 0) cyc[8] = (t1 - t0) / (n * 16);
  out[threadIdx.x + 64] = s;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 4096); cudaMalloc(&cyc, 128);
  lat<<<1, 32>>>(out, cyc, 100); lat<<<1, 32>>>(out, cyc, 1000);
  thr<<<1, 32>>>(out, cyc, 100); thr<<<1, 32>>>(out, cyc, 1000);
  cudaDeviceSynchronize();
  long long h[9]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  printf("{\"dfma_lat\": %lld, \"dmul_lat\": %lld, \"ffma_lat\": %lld, \"shfl64_lat\": %lld, \"rsqrt_d_lat\": %lld, \"rcp_d_lat\": %lld, \"lds64_lat\": %lld, \"sqrt_d_lat\": %lld, \"dfma_1warp_cpi\": %lld}\n",
         h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8]);
}
