// Effective SM clock (MHz) seen by a lightly loaded GPU: spin N cycles on
// clock64() in 1 CTA (or many), measure %globaltimer.
#include <cstdio>
__global__ void spin(long long n, unsigned long long* out) {
  unsigned long long g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  long long t0 = clock64();
  while (clock64() - t0 < n) {}
  long long t1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = g1 - g0; }
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16);
  unsigned long long h[2];
  int grids[4] = {1, 16, 148, 1};
  for (int k = 0; k < 4; ++k) {
    for (int rep = 0; rep < 3; ++rep) {
      spin<<<grids[k], 32>>>(20000000LL, d);
      cudaDeviceSynchronize();
    }
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("grid %d: %llu cycles in %llu ns -> %.0f MHz\n", grids[k], h[0], h[1], 1e3 * h[0] / (double)h[1]);
  }
  return 0;
}
