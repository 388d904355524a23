// common.cuh -- device helpers shared by the sm_100a kernels of libnnls_b200.
// (Not shared with the CPU oracle: oracle/ and csrc/ have no code in common.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>

#define NNLS_DEV __device__ __forceinline__

namespace nnls {

constexpr unsigned kFull = 0xffffffffu;

// Device-resident solver state of one problem (one 128-byte line).
struct DevState {
  int32_t k;            // infeasible count of the last decide
  int32_t N;            // best infeasible count so far (N = inf -> n+1)
  int32_t p;            // no-progress counter
  int32_t iter;         // completed normal-equation solves (reading c11)
  int32_t singles;      // single exchanges taken
  int32_t f, g;         // |F|, |G| after the last exchange
  int32_t branch;       // -1 feasible, 0, 1, 2
  int32_t done;         // 1: feasible (k == 0), stop
  int32_t status;       // 0 ok, 7 NOT_PD, 8 ITERATION_LIMIT
  int32_t not_pd_col;   // failing pivot position in F
  int32_t epoch;        // Cholesky DAG epoch (flags == epoch mean "ready")
  int32_t tile_counter; // DAG work counter of the factorization
  int32_t solve_counter;// DAG work counter of the back substitution
  int32_t max_iter;
  int32_t p_max;
  unsigned long long below_bits;  // trace: max |v| < tol (as ordered bits)
  unsigned long long above_bits;  // trace: min |v| >= tol
  // final-step report
  int32_t lsqr_iterations, lsqr_stop, infeasible_after_lsqr, free_count;
  double objective, kkt_min_x, kkt_min_y, kkt_max_comp, kkt_dot;
  int32_t reuse_cols;   // leading tile columns of the last factor still valid (factor reuse)
  int32_t role_factor;  // CTA role tickets of the factorization / back-substitution kernels:
  int32_t role_solve;   // the first CTA to run takes the chain (reset with the task counters)
  int32_t keep_none;      // 1: the next decide keeps no factor prefix (set after a NOT_PD fallback)
  double kappa;           // lsqr_mode 3: condition estimate of the final (A^T A)_FF (condest.cu)
  int32_t refined;        // 1: the final x comes from LSQR
  int32_t lsqr_fallbacks; // NOT_PD iterations solved by LSQR instead (notpd_fallback)
  // fused dual + exchange (pivot.cu dual_kernel with an infeasible list)
  int32_t decided;        // 1: the dual kernel counted, chose the branch and exchanged; decide only compacts
  int32_t inf_count;      // infeasible entries appended to the list so far (= k at the end)
  int32_t inf_last1;      // 1 + the largest infeasible index (0: none)
  uint32_t dual_ticket;   // CTAs of the dual kernel that finished (the last one decides)
};

struct TraceRec {
  int32_t iter, k, branch, f;
  double below_tol, above_tol;
  int32_t kept;   // leading columns of the previous factor reused (0: full factorization)
  int32_t pad;
};

NNLS_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
NNLS_DEV int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
NNLS_DEV int warp_max_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
NNLS_DEV double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(kFull, v, o));
  return v;
}
NNLS_DEV double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// D(8x8) += A(8x4) * B(4x8) in FP64 on the tensor pipe (SASS DMMA.8x8x4).
// Fragments (lane = l): a = A[l>>2][l&3]; b = B[k=l&3][n=l>>2];
// c0,c1 = C[l>>2][2*(l&3) + {0,1}].
NNLS_DEV void dmma8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

NNLS_DEV int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
NNLS_DEV int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
NNLS_DEV void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
NNLS_DEV int ld_volatile(const int* p) { return *(volatile const int*)p; }

// spin (one thread) until *flag == want
NNLS_DEV void wait_flag(const int* flag, int want) {
  int spins = 0;
  while (ld_acquire(flag) != want) {
    if (++spins > 64) __nanosleep(40);
  }
}

// non-negative doubles compare like their bit patterns
NNLS_DEV unsigned long long dbits(double v) { return (unsigned long long)__double_as_longlong(v); }

// Programmatic dependent launch: a kernel launched with launch_pdl starts
// (CTA rasterisation, shared-memory carve-out) while its predecessor in the
// stream drains, and waits here before touching the predecessor's results.
// A no-op for a kernel launched without the attribute.
NNLS_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }

// Per-device cached host setup (kernel attributes set with
// cudaFuncSetAttribute are per device): state[dev] = the value init()
// returned for the CURRENT device (0 = not yet / failed: retried next call),
// computed once under a mutex.
constexpr int kMaxDevices = 64;
struct DeviceOnce {
  std::atomic<int> state[kMaxDevices];
  std::mutex mu;
  DeviceOnce() {
    for (auto& v : state) v.store(0, std::memory_order_relaxed);
  }
};
template <typename F>
inline int device_once(DeviceOnce& o, F init) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return init();
  int v = o.state[dev].load(std::memory_order_acquire);
  if (v != 0) return v;
  std::lock_guard<std::mutex> g(o.mu);
  v = o.state[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    v = init();
    o.state[dev].store(v, std::memory_order_release);
  }
  return v;
}

bool pdl_enabled();  // (env NNLS_NO_PDL=1 disables; api.cu)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

}  // namespace nnls
