// trsm_blocked: the substitution TRSM the factorization chain used before it
// switched to an explicit Linv_jj (trtri64); kept for the microbenchmarks.
#pragma once
namespace nnls {
// (moved here from the product: the chain now inverts L_jj, see trtri64)
struct NoHook {
  __device__ __forceinline__ void operator()(int, int) const {}
};

// X := X L^-T for a 64x64 smem tile X and lower L (cv valid columns), in
// 8-column panels: warps 0-1 solve the panel row by row (thread per row,
// the 8x8 diagonal block of L in registers), then every warp folds the
// panel into the later column blocks with DMMA (warp w: rows 8w..8w+7).
// hook(p, lane) runs on warp 7 during the solve phase of panel p.
template <class Hook = NoHook>
__device__ __forceinline__ void trsm_blocked(double* __restrict__ X, const double* __restrict__ L,
                                             const double* __restrict__ rinv, int cv,
                                             const Hook& hook = Hook()) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int np = (cv + 7) >> 3;
#pragma unroll 1
  for (int p = 0; p < np; ++p) {
    const int c0 = 8 * p;
    if (tid < 64) {
      double Ld[8][8], ri[8], x[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        ri[c] = (c0 + c < cv) ? rinv[c0 + c] : 0.0;
#pragma unroll
        for (int c2 = c + 1; c2 < 8; ++c2) Ld[c2][c] = L[(c0 + c2) * LDS + c0 + c];
        x[c] = X[tid * LDS + c0 + c];
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        x[c] *= ri[c];
#pragma unroll
        for (int c2 = c + 1; c2 < 8; ++c2) x[c2] = fma(-x[c], Ld[c2][c], x[c2]);
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) X[tid * LDS + c0 + c] = x[c];
    } else if (w == 7) {
      hook(p, lane);  // warp 7 is idle in the solve phase
    }
    csync();
    if (p + 1 < np) {  // X(rows of warp w, J) -= X(., panel) L(J, panel)^T for J in (p, np)
      strip8_gemm(X, X, L, c0, 8 * w, p + 1, np, lane);
      csync();
    }
  }
}

}  // namespace nnls
