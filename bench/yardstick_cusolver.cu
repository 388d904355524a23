// yardstick_cusolver.cu -- library yardsticks for SURVEY.md §8(d): cuSOLVER
// DPOTRF and cuBLAS DSYRK in FP64 at the sizes this build's own kernels run
// (the config-2 free-set size f ~ 3980, the full n = 8000, the Fig. 2 dense
// Gram 16384 x 8000).  Not on any product path: the numbers sit beside the
// bench's chol_factor / dense-SYRK rates in profiles/.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 bench/yardstick_cusolver.cu \
//        -lcusolver -lcublas -o bench/yardstick_cusolver
//   ./bench/yardstick_cusolver            (one JSON line per measurement)
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    auto e_ = (x);                                                             \
    if ((int)e_ != 0) {                                                        \
      fprintf(stderr, "%s:%d error %d\n", __FILE__, __LINE__, (int)e_);        \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

// SPD test matrix: M = B^T B / k + n I from a random B (only the lower
// triangle matters for DPOTRF), built on the device with DSYRK.
static void make_spd(cublasHandle_t cb, double* M, int n, double* B, int k) {
  const double alpha = 1.0 / k, beta = 0.0;
  CK(cublasDsyrk(cb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, n, k, &alpha, B, k, &beta, M, n));
  for (int i = 0; i < n; ++i) {
    double d;
    CK(cudaMemcpy(&d, M + (size_t)i * n + i, sizeof(double), cudaMemcpyDeviceToHost));
    d += 1.0;
    CK(cudaMemcpy(M + (size_t)i * n + i, &d, sizeof(double), cudaMemcpyHostToDevice));
  }
}

__global__ void fill(double* p, size_t cnt, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < cnt; i += (size_t)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)i * 2654435761u ^ seed;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    p[i] = (double)(h & 0xFFFFFF) / 16777216.0 - 0.5;
  }
}

int main() {
  cublasHandle_t cb;
  cusolverDnHandle_t cs;
  CK(cublasCreate(&cb));
  CK(cusolverDnCreate(&cs));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));

  // ---- DPOTRF (lower) at f = 1000, 2000, 3980, 8000: flops f^3/3 + f^2/2
  const int fs[] = {1000, 2000, 3980, 8000};
  for (int f : fs) {
    const int k = f + 64;
    double *B, *M, *W;
    int* dinfo;
    CK(cudaMalloc(&B, sizeof(double) * (size_t)k * f));
    CK(cudaMalloc(&M, sizeof(double) * (size_t)f * f));
    CK(cudaMalloc(&W, sizeof(double) * (size_t)f * f));
    CK(cudaMalloc(&dinfo, sizeof(int)));
    fill<<<1024, 256>>>(B, (size_t)k * f, 17u + f);
    make_spd(cb, M, f, B, k);
    int lwork = 0;
    CK(cusolverDnDpotrf_bufferSize(cs, CUBLAS_FILL_MODE_LOWER, f, W, f, &lwork));
    double* work;
    CK(cudaMalloc(&work, sizeof(double) * (size_t)lwork));
    const int reps = 5;
    float best = 1e30f, total = 0.f;
    for (int r = 0; r < reps + 2; ++r) {
      CK(cudaMemcpy(W, M, sizeof(double) * (size_t)f * f, cudaMemcpyDeviceToDevice));
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      CK(cusolverDnDpotrf(cs, CUBLAS_FILL_MODE_LOWER, f, W, f, work, lwork, dinfo));
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r >= 2) {
        total += ms;
        if (ms < best) best = ms;
      }
    }
    int hinfo = -1;
    CK(cudaMemcpy(&hinfo, dinfo, sizeof(int), cudaMemcpyDeviceToHost));
    const double flops = (double)f * f * f / 3.0 + (double)f * f / 2.0;
    printf("{\"op\": \"cusolverDnDpotrf\", \"n\": %d, \"info\": %d, \"ms_mean\": %.4f, \"ms_best\": %.4f, "
           "\"tflops_mean\": %.3f}\n",
           f, hinfo, total / reps, best, flops / (total / reps * 1e-3) / 1e12);
    CK(cudaFree(B));
    CK(cudaFree(M));
    CK(cudaFree(W));
    CK(cudaFree(work));
    CK(cudaFree(dinfo));
  }

  // ---- DSYRK C = A^T A (lower), A k x n column-major: flops k n (n+1)
  const int shapes[][2] = {{16384, 8000}, {40000, 8000}, {2000, 1000}};
  for (auto& sh : shapes) {
    const int k = sh[0], n = sh[1];
    double *A, *C;
    CK(cudaMalloc(&A, sizeof(double) * (size_t)k * n));
    CK(cudaMalloc(&C, sizeof(double) * (size_t)n * n));
    fill<<<1024, 256>>>(A, (size_t)k * n, 99u + k);
    const double alpha = 1.0, beta = 0.0;
    const int reps = 3;
    float total = 0.f;
    for (int r = 0; r < reps + 1; ++r) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      CK(cublasDsyrk(cb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_T, n, k, &alpha, A, k, &beta, C, n));
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      if (r >= 1) total += ms;
    }
    const double flops = (double)k * n * (n + 1);
    printf("{\"op\": \"cublasDsyrk\", \"k\": %d, \"n\": %d, \"ms_mean\": %.4f, \"tflops_mean\": %.3f}\n", k, n,
           total / reps, flops / (total / reps * 1e-3) / 1e12);
    CK(cudaFree(A));
    CK(cudaFree(C));
  }
  return 0;
}
