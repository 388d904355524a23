// M1: FP64 peak microbenchmark for B200 (sm_100a) -- the roofline denominator
// that MEASURED_PEAKS.json lacks.
//
// Measures, on the whole chip:
//   * DFMA throughput  (independent FMA chains in registers)
//   * DMMA throughput  (mma.sync.aligned.m8n8k4.row.col.f64, the only FP64
//                       tensor path on sm_100a; tcgen05 has no f64 kind)
//   * cooperative grid.sync() latency at one CTA per SM
//   * empty-kernel launch latency (stream and CUDA graph)
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench_fp64 microbench_fp64.cu
// Prints one JSON line.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(1);} } while (0)

constexpr int kChains = 8;

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[4][2];
#pragma unroll
  for (int t = 0; t < 4; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(c[t][0]), "+d"(c[t][1])
          : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void gridsync_kernel(int reps, unsigned long long* cycles) {
  cg::grid_group g = cg::this_grid();
  long long t0 = clock64();
  for (int i = 0; i < reps; ++i) g.sync();
  long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) cycles[0] = (unsigned long long)(t1 - t0);
}

__global__ void empty_kernel() {}

int main() {
  int dev = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  const int sms = prop.multiProcessorCount;
  double* dout;
  CK(cudaMalloc(&dout, 64));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  float ms;

  // ---- DFMA ----
  const int threads = 512, blocks_per_sm = 4;
  const int dfma_iters = 1 << 16;
  dfma_kernel<<<sms * blocks_per_sm, threads>>>(dout, 1024, 1.0000001, 1e-9);
  CK(cudaDeviceSynchronize());
  float best_dfma = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    dfma_kernel<<<sms * blocks_per_sm, threads>>>(dout, dfma_iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best_dfma) best_dfma = ms;
  }
  double dfma_flops = 2.0 * kChains * (double)dfma_iters * threads * sms * blocks_per_sm;
  double dfma_tf = dfma_flops / (best_dfma * 1e-3) / 1e12;

  // ---- DMMA ----
  const int dmma_iters = 1 << 14;
  dmma_kernel<<<sms * blocks_per_sm, threads>>>(dout, 256);
  CK(cudaDeviceSynchronize());
  float best_dmma = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    dmma_kernel<<<sms * blocks_per_sm, threads>>>(dout, dmma_iters);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best_dmma) best_dmma = ms;
  }
  // per warp per mma: 8*8*4 = 256 FMA = 512 flop
  double dmma_flops = 512.0 * 4 * (double)dmma_iters * (threads / 32) * sms * blocks_per_sm;
  double dmma_tf = dmma_flops / (best_dmma * 1e-3) / 1e12;

  // ---- grid sync ----
  unsigned long long* dcyc;
  CK(cudaMalloc(&dcyc, 8));
  int reps = 1000;
  double gs_us[3];
  int gs_threads[3] = {256, 512, 1024};
  for (int k = 0; k < 3; ++k) {
    void* args[] = {&reps, &dcyc};
    int nthr = gs_threads[k];
    CK(cudaLaunchCooperativeKernel((void*)gridsync_kernel, dim3(sms), dim3(nthr), args, 0, 0));
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    CK(cudaLaunchCooperativeKernel((void*)gridsync_kernel, dim3(sms), dim3(nthr), args, 0, 0));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    gs_us[k] = ms * 1e3 / reps;
  }

  // ---- launch latency ----
  for (int i = 0; i < 100; ++i) empty_kernel<<<1, 32>>>();
  CK(cudaDeviceSynchronize());
  const int nl = 2000;
  CK(cudaEventRecord(e0));
  for (int i = 0; i < nl; ++i) empty_kernel<<<sms, 128>>>();
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  CK(cudaEventElapsedTime(&ms, e0, e1));
  double launch_us = ms * 1e3 / nl;
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int i = 0; i < 100; ++i) empty_kernel<<<sms, 128, 0, s>>>();
  CK(cudaStreamEndCapture(s, &graph));
  CK(cudaGraphInstantiate(&exec, graph, 0));
  CK(cudaGraphLaunch(exec, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaEventRecord(e0, s));
  for (int i = 0; i < 20; ++i) CK(cudaGraphLaunch(exec, s));
  CK(cudaEventRecord(e1, s));
  CK(cudaEventSynchronize(e1));
  CK(cudaEventElapsedTime(&ms, e0, e1));
  double graph_us = ms * 1e3 / 2000;

  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %zu, \"clock_khz_attr\": %d, "
         "\"dfma_tflops\": %.3f, \"dmma_tflops\": %.3f, \"dfma_ms\": %.3f, \"dmma_ms\": %.3f, "
         "\"grid_sync_us\": {\"256\": %.3f, \"512\": %.3f, \"1024\": %.3f}, "
         "\"launch_us_stream\": %.3f, \"launch_us_graph\": %.3f}\n",
         prop.name, sms, prop.l2CacheSize, prop.sharedMemPerBlockOptin, clk_khz, dfma_tf, dmma_tf,
         best_dfma, best_dmma, gs_us[0], gs_us[1], gs_us[2], launch_us, graph_us);
  return 0;
}
