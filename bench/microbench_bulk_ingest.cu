// Per-SM ingest rate of cp.async.bulk (global -> shared) from L2-resident
// data: one CTA streams 32 KB tiles through a ring of S stages (S copies in
// flight), as the Cholesky/back-substitution chains do.  Also G CTAs at once
// (aggregate).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench/mb_bulk bench/microbench_bulk_ingest.cu
#include <cstdio>
#include <cstdint>
constexpr int TB = 32768;  // bytes per copy
__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
template <int S>
__global__ void ingest(const char* src, size_t span, int iters, long long* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) unsigned long long mb[S];
  if (threadIdx.x == 0) {
    for (int k = 0; k < S; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&mb[k])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t base = ((size_t)blockIdx.x * 7919 * TB) % (span - (size_t)iters * TB % span);
  long long t0 = clock64();
  for (int i = 0; i < iters + S; ++i) {
    if (i >= S) {  // wait for copy i - S
      const int k = (i - S) % S;
      const unsigned par = ((i - S) / S) & 1;
      unsigned done = 0;
      while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(sa(&mb[k])), "r"(par) : "memory");
    }
    if (i < iters) {
      const int k = i % S;
      const char* g = src + (base + (size_t)i * TB) % (span - TB);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&mb[k])), "r"(TB) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(sm + (size_t)k * TB)), "l"(g), "r"(TB), "r"(sa(&mb[k])) : "memory");
    }
  }
  long long t1 = clock64();
  out[blockIdx.x] = t1 - t0;
}
int main() {
  const size_t span = 64ull << 20;  // 64 MB: L2-resident after the warm-up
  char* src; cudaMalloc(&src, span); cudaMemset(src, 1, span);
  long long* out; cudaMalloc(&out, 4096 * 8);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 400;
  auto run = [&](auto kern, int S, int grid) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, S * TB);
    kern<<<grid, 32, S * TB>>>(src, span, iters, out);  // warm
    kern<<<grid, 32, S * TB>>>(src, span, iters, out);
    cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, out, grid * 8, cudaMemcpyDeviceToHost);
    long long mx = 0; for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
    const double sec = (double)mx / (clk * 1e3);
    printf("{\"stages\": %d, \"ctas\": %d, \"per_cta_GBps\": %.1f, \"aggregate_GBps\": %.1f}\n", S, grid,
           (double)iters * TB / sec / 1e9, (double)iters * TB * grid / sec / 1e9);
  };
  run(ingest<1>, 1, 1); run(ingest<2>, 2, 1); run(ingest<3>, 3, 1); run(ingest<6>, 6, 1);
  run(ingest<3>, 3, 148); run(ingest<6>, 6, 148);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
