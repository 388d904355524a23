// lsqr.cu -- a10: the final solve on the final free set F with LSQR
// ("using the method of normal equations for the intermediate
// solutions ... and then recomputing the final solution using the more
// accurate LSQR solver"), followed by the a11 report: zeroing of x_F (c16),
// objective 1/2||Ax-b||^2 and the KKT residuals of Eq. 3 with an
// independently recomputed y' = A^T (A x - b).
//
// B200 design: one cooperative persistent kernel (1 CTA per SM) runs the
// whole Golub-Kahan/LSQR recurrence without returning to the host.  Each
// iteration has three grid-wide phases separated by grid.sync():
//   A  rows:    U = A v - alpha u        (CSR SpMV, warp per row)     |U|^2
//   B  cols F:  V = A_F^T u - beta v     (CSC SpMV, warp per column)  |V|^2
//   C  cols F:  v, x, w updates (Givens rotation scalars replicated)  |d|^2,|x|^2
// Norms are reduced deterministically: every CTA writes a partial, every CTA
// re-reduces all partials in the same fixed order, so all CTAs hold identical
// scalars and take identical stopping decisions.  u and v are kept
// unnormalised (U = beta u) and scaled on the fly.  Stopping rules are the
// standard LSQR tests: test1 <= btol + atol |A||x|/|b|, test2 <= atol,
// test3 <= 1/conlim, their machine-precision forms, or itn == itn_limit.
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace nnls {

namespace {
constexpr int kThreads = 512;
constexpr int kSlots = 8;

// block-reduce v (sum) and write partials[blockIdx*kSlots + slot]
__device__ void block_partial_sum(double v, double* partials, int slot, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double s = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    s = warp_sum(s);
    if (lane == 0) partials[blockIdx.x * kSlots + slot] = s;
  }
}
__device__ void block_partial_minmax(double v, double* partials, int slot, double* red, bool is_min) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = is_min ? warp_min(v) : warp_max(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double s = lane < (int)(blockDim.x >> 5) ? red[lane] : (is_min ? INFINITY : -INFINITY);
    s = is_min ? warp_min(s) : warp_max(s);
    if (lane == 0) partials[blockIdx.x * kSlots + slot] = s;
  }
}
// all CTAs: sum partials[*][slot .. slot+nv) (nv <= 3) with every thread of
// the block (fixed order per thread, then a fixed block reduction: the
// result is identical in every CTA).  red[] holds 3 x 32 doubles.
__device__ void grid_sum3(const double* partials, int slot, int nv, double* out, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double sv[3] = {0.0, 0.0, 0.0};
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
    for (int q = 0; q < nv; ++q) sv[q] += __ldcg(&partials[b * kSlots + slot + q]);
  for (int q = 0; q < nv; ++q) sv[q] = warp_sum(sv[q]);
  __syncthreads();
  if (lane == 0)
    for (int q = 0; q < nv; ++q) red[32 * q + wid] = sv[q];
  __syncthreads();
  for (int q = 0; q < nv; ++q) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[32 * q + w];
    out[q] = t;
  }
}
// block-reduce nv (<= 3) values into partials[blockIdx][slot ..]
__device__ void block_partial_sum3(const double* v, int nv, double* partials, int slot, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double x[3] = {0.0, 0.0, 0.0};
  for (int q = 0; q < nv; ++q) x[q] = warp_sum(v[q]);
  __syncthreads();
  if (lane == 0)
    for (int q = 0; q < nv; ++q) red[32 * q + wid] = x[q];
  __syncthreads();
  if (wid == 0) {
    for (int q = 0; q < nv; ++q) {
      double y = lane < (int)(blockDim.x >> 5) ? red[32 * q + lane] : 0.0;
      y = warp_sum(y);
      if (lane == 0) partials[blockIdx.x * kSlots + slot + q] = y;
    }
  }
}
// all CTAs: reduce partials[*][slot] in a fixed order (result identical in every CTA)
__device__ double grid_total(const double* partials, int slot, double* bcast, int kind) {
  // kind 0 sum, 1 min, 2 max
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    double s = kind == 0 ? 0.0 : (kind == 1 ? INFINITY : -INFINITY);
    for (int b = lane; b < (int)gridDim.x; b += 32) {
      const double v = __ldcg(&partials[b * kSlots + slot]);
      s = kind == 0 ? s + v : (kind == 1 ? fmin(s, v) : fmax(s, v));
    }
    s = kind == 0 ? warp_sum(s) : (kind == 1 ? warp_min(s) : warp_max(s));
    if (lane == 0) *bcast = s;
  }
  __syncthreads();
  const double r = *bcast;
  __syncthreads();
  return r;
}
}  // namespace

// debug hook: per-phase %globaltimer stamps of CTA 0 (nnls_debug_lsqr_profile)
__device__ unsigned long long* g_lsqr_prof = nullptr;
#define LG_MARK(slot)                                                                      \
  do {                                                                                     \
    if (g_lsqr_prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {                   \
      unsigned long long t_;                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
      g_lsqr_prof[63 * 16 + (slot)] = t_;                                                  \
    }                                                                                      \
  } while (0)
#define LG_STAMP(slot)                                                                     \
  do {                                                                                     \
    if (g_lsqr_prof != nullptr && blockIdx.x == 0 && threadIdx.x == 0 && itn < 64) {        \
      unsigned long long t_;                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
      g_lsqr_prof[itn * 16 + (slot)] = t_;                                                 \
    }                                                                                      \
  } while (0)

// The global-memory LSQR iteration (any cooperative grid): A_F from the
// compacted rows (Fval/Fcol/Fcnt) and the CSC in global memory / L2.  On
// return X[j] (j in F) holds the LSQR x.
__device__ void lsqr_iterate_global(const LsqrArgs& a, cg::grid_group& grid, int mode, int f, double* red,
                                    double* bcast_p, int& itn, int& istop) {
  double& bcast = *bcast_p;
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nthr = gridDim.x * blockDim.x;
  const int m = a.m, n = a.n;
  const uint8_t* __restrict__ mask = a.mask;
  const int itn_limit = a.itn_limit > 0 ? a.itn_limit : 4 * f;
  // ---- start: U = rhs (cold: b; warm: b - A_F x_ne); beta = |U|
  double p = 0.0;
  for (int r = gwarp; r < m; r += nwarps) {
    double s = 0.0;
    if (mode == 2) {
      for (int t = a.rowptr[r] + lane; t < a.rowptr[r + 1]; t += 32) {
        const int j = a.colind[t];
        if (mask[j]) s = fma(a.vals[t], a.x_ne[j], s);
      }
      s = warp_sum(s);
    }
    if (lane == 0) {
      const double u = a.b[r] - s;
      a.U[r] = u;
      p += u * u;
    }
  }
  for (int j = gtid; j < n; j += nthr) {
    a.V[j] = 0.0;
    a.W[j] = 0.0;
    a.X[j] = 0.0;
  }
  block_partial_sum(p, a.partials, 0, red);
  grid.sync();
  double beta = sqrt(grid_total(a.partials, 0, &bcast, 0));
  const double bnorm = beta;
  // V = A_F^T u (u = U / beta); alpha = |V|
  p = 0.0;
  if (beta > 0.0) {
    const double ib = 1.0 / beta;
    for (int j = gwarp; j < n; j += nwarps) {
      if (!mask[j]) continue;
      double s = 0.0;
      for (int t = a.colptr[j] + lane; t < a.colptr[j + 1]; t += 32)
        s = fma(a.cvals[t], __ldcg(&a.U[a.rowind[t]]), s);
      s = warp_sum(s) * ib;
      if (lane == 0) {
        a.V[j] = s;
        p += s * s;
      }
    }
  }
  block_partial_sum(p, a.partials, 1, red);
  grid.sync();
  double alpha = beta > 0.0 ? sqrt(grid_total(a.partials, 1, &bcast, 0)) : 0.0;
  if (alpha > 0.0) {
    const double ia = 1.0 / alpha;
    for (int j = gtid; j < n; j += nthr) {
      if (!mask[j]) continue;
      const double v = __ldcg(&a.V[j]) * ia;
      a.V[j] = v;
      a.W[j] = v;
    }
  }
  grid.sync();
  double rhobar = alpha, phibar = beta, anorm = 0.0, ddnorm = 0.0;
  const double ctol = a.conlim > 0.0 ? 1.0 / a.conlim : 0.0;
  // Two grid barriers per iteration: the |d|^2, |x|^2 partials of
  // iteration t ride on iteration t+1's first barrier, and t's stopping
  // test is taken there (x is not touched in between).
  double pd = 0.0, px = 0.0, last_phi = 0.0, last_sn = 0.0;
  bool pending = false;
  const int32_t* __restrict__ Fidx = a.Fidx;
  // V holds v unnormalised (V = v / vscale) from phase B on, so phase C
  // never writes it: phase A of the next iteration reads V with no barrier
  // after phase C
  double vscale = 1.0;
  if (alpha * beta != 0.0) {
    for (;;) {
      const bool more = itn < itn_limit;
      LG_STAMP(0);
      // ---- phase A: U = A v - alpha u, u = U / beta.  Four rows per warp
      //      pass (8 lanes each), so four rows' gathers are in flight at once
      const double au = beta > 0.0 ? alpha / beta : 0.0;
      p = 0.0;
      if (more) {
        const int sub = lane >> 3, sl = lane & 7;
        for (int r0 = gwarp * 4; r0 < m; r0 += nwarps * 4) {
          const int r = r0 + sub;
          double s = 0.0;
          if (r < m) {  // A restricted to F (lsqr_compact_kernel): V is zero off F
            const int t0 = a.rowptr[r], t1 = t0 + __ldcg(&a.Fcnt[r]);
#pragma unroll 2
            for (int t = t0 + sl; t < t1; t += 8) s = fma(__ldcg(&a.Fval[t]), __ldcg(&a.V[__ldcg(&a.Fcol[t])]), s);
          }
          s += __shfl_xor_sync(kFull, s, 4);
          s += __shfl_xor_sync(kFull, s, 2);
          s += __shfl_xor_sync(kFull, s, 1);
          if (sl == 0 && r < m) {
            const double u = s * vscale - au * a.U[r];
            a.U[r] = u;
            p += u * u;
          }
        }
      }
      LG_STAMP(1);
      {
        const double v3[3] = {p, pd, px};
        block_partial_sum3(v3, 3, a.partials, 0, red);
      }
      grid.sync();
      LG_STAMP(2);
      double gt[3];
      grid_sum3(a.partials, 0, 3, gt, red);
      if (pending) {  // stopping test of the previous iteration
        ddnorm += gt[1];
        const double xnorm = sqrt(gt[2]);
        const double acond = anorm * sqrt(ddnorm);
        const double rnorm = phibar;
        const double arnorm = alpha * fabs(last_sn * last_phi);
        const double test1 = bnorm > 0.0 ? rnorm / bnorm : 0.0;
        const double test2 = (anorm * rnorm) > 0.0 ? arnorm / (anorm * rnorm) : 0.0;
        const double test3 = acond > 0.0 ? 1.0 / acond : 0.0;
        const double tt1 = bnorm > 0.0 ? test1 / (1.0 + anorm * xnorm / bnorm) : 0.0;
        const double rtol = a.btol + (bnorm > 0.0 ? a.atol * anorm * xnorm / bnorm : 0.0);
        if (itn >= itn_limit) istop = 7;
        if (1.0 + test3 <= 1.0) istop = 6;
        if (1.0 + test2 <= 1.0) istop = 5;
        if (1.0 + tt1 <= 1.0) istop = 4;
        if (test3 <= ctol) istop = 3;
        if (test2 <= a.atol) istop = 2;
        if (test1 <= rtol) istop = 1;
        if (istop != 0) break;
      }
      ++itn;
      const double beta_new = sqrt(gt[0]);
      // ---- phase B: V' = A_F^T u - beta v (warp per F column)
      double alpha_new = alpha;
      if (beta_new > 0.0) {
        anorm = sqrt(anorm * anorm + alpha * alpha + beta_new * beta_new);
        const double ib = 1.0 / beta_new;
        p = 0.0;
        for (int k = gwarp; k < f; k += nwarps) {
          const int j = Fidx[k];
          double s = 0.0;
          const int c1 = a.colptr[j + 1];
#pragma unroll 2
          for (int t = a.colptr[j] + lane; t < c1; t += 32) s = fma(a.cvals[t], __ldcg(&a.U[a.rowind[t]]), s);
          s = warp_sum(s) * ib;
          if (lane == 0) {
            const double v = s - beta_new * (__ldcg(&a.V[j]) * vscale);
            a.V[j] = v;  // unnormalised
            p += v * v;
          }
        }
        LG_STAMP(3);
        block_partial_sum(p, a.partials, 4, red);
        grid.sync();
        LG_STAMP(4);
        grid_sum3(a.partials, 4, 1, gt, red);
        alpha_new = sqrt(gt[0]);
      }
      beta = beta_new;
      // ---- rotation (replicated scalars)
      const double rho = sqrt(rhobar * rhobar + beta * beta);
      const double irho = 1.0 / rho;
      const double cs = rhobar * irho, sn = beta * irho;
      const double theta = sn * alpha_new;
      rhobar = -cs * alpha_new;
      const double phi = cs * phibar;
      phibar = sn * phibar;
      const double t1 = phi * irho, t2 = -theta * irho;
      // ---- phase C: v = V'/alpha, x += t1 w, w = v + t2 w (F columns; V not written)
      if (beta_new > 0.0 && alpha_new > 0.0) vscale = 1.0 / alpha_new;
      pd = 0.0;
      px = 0.0;
      for (int k = gtid; k < f; k += nthr) {
        const int j = Fidx[k];
        const double v = __ldcg(&a.V[j]) * vscale;
        const double w = a.W[j];
        const double d = w * irho;
        pd += d * d;
        const double x = a.X[j] + t1 * w;
        a.X[j] = x;
        a.W[j] = v + t2 * w;
        px += x * x;
      }
      alpha = alpha_new;
      last_phi = phi;
      last_sn = sn;
      pending = true;
      LG_STAMP(5);
    }
  }
}

// x (LSQR result on F, correction, or the NE x), zeroing (c16), and the
// a11 report; every CTA of the cooperative grid
__device__ void lsqr_finish(const LsqrArgs& a, cg::grid_group& grid, int mode, int f, int itn, int istop,
                            double* red, double* bcast_p) {
  double& bcast = *bcast_p;
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nthr = gridDim.x * blockDim.x;
  const int m = a.m, n = a.n;
  const uint8_t* __restrict__ mask = a.mask;
  // ---- x: LSQR result on F (mode 1), correction (mode 2) or NE x; zeroing (c16)
  double pinf = 0.0;
  for (int j = gtid; j < n; j += nthr) {
    double v;
    if (!mask[j]) v = 0.0;
    else if (mode == 1) v = a.X[j];
    else if (mode == 2) v = a.x_ne[j] + a.X[j];
    else v = a.x_ne[j];
    if (fabs(v) < a.tol) v = 0.0;
    if (v < 0.0) pinf = 1.0;
    a.x_out[j] = v;
  }
  block_partial_minmax(pinf, a.partials, 4, red, false);
  grid.sync();
  LG_MARK(4);
  const double infeas = grid_total(a.partials, 4, &bcast, 2);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.st->lsqr_iterations = itn;
    a.st->lsqr_stop = istop;
    a.st->infeasible_after_lsqr = (mode != 0 && infeas > 0.0) ? 1 : 0;
    a.st->free_count = f;
  }
  if (!a.kkt) return;
  // ---- report: R = A x - b, objective; y' = A^T R; KKT residuals (Eq. 3)
  double po = 0.0;
  {  // eight lanes per row, four rows per warp pass (latency-bound gathers in flight)
    const int sub = lane >> 3, sl = lane & 7;
    for (int r0 = gwarp * 4; r0 < m; r0 += nwarps * 4) {
      const int r = r0 + sub;
      double s = 0.0;
      if (r < m) {
        const int t1 = a.rowptr[r + 1];
#pragma unroll 2
        for (int t = a.rowptr[r] + sl; t < t1; t += 8) s = fma(a.vals[t], __ldcg(&a.x_out[a.colind[t]]), s);
      }
      s += __shfl_xor_sync(kFull, s, 4);
      s += __shfl_xor_sync(kFull, s, 2);
      s += __shfl_xor_sync(kFull, s, 1);
      if (sl == 0 && r < m) {
        const double rr = s - a.b[r];
        a.R[r] = rr;
        po += rr * rr;
      }
    }
  }
  block_partial_sum(po, a.partials, 0, red);
  grid.sync();
  LG_MARK(5);
  double mx = INFINITY, my = INFINITY, mc = 0.0, dot = 0.0;
  for (int j = gwarp; j < n; j += nwarps) {
    double s = 0.0;
    const int t1 = a.colptr[j + 1];
#pragma unroll 4
    for (int t = a.colptr[j] + lane; t < t1; t += 32) s = fma(a.cvals[t], __ldcg(&a.R[a.rowind[t]]), s);
    s = warp_sum(s);
    if (lane == 0) {
      const double xj = __ldcg(&a.x_out[j]);
      mx = fmin(mx, xj);
      my = fmin(my, s);
      mc = fmax(mc, fabs(xj * s));
      dot += xj * s;
    }
  }
  block_partial_minmax(mx, a.partials, 1, red, true);
  block_partial_minmax(my, a.partials, 2, red, true);
  block_partial_minmax(mc, a.partials, 3, red, false);
  block_partial_sum(dot, a.partials, 4, red);
  grid.sync();
  LG_MARK(6);
  if (blockIdx.x == 0) {
    const double obj = grid_total(a.partials, 0, &bcast, 0);
    const double gmx = grid_total(a.partials, 1, &bcast, 1);
    const double gmy = grid_total(a.partials, 2, &bcast, 1);
    const double gmc = grid_total(a.partials, 3, &bcast, 2);
    const double gd = grid_total(a.partials, 4, &bcast, 0);
    if (threadIdx.x == 0) {
      a.st->objective = 0.5 * obj;
      a.st->kkt_min_x = gmx;
      a.st->kkt_min_y = gmy;
      a.st->kkt_max_comp = gmc;
      a.st->kkt_dot = gd;
    }
  }
}

__device__ __forceinline__ int lsqr_mode_of(const LsqrArgs& a, int f) {
  const int mode0 = (a.st->status == 0 && a.st->done && f > 0) ? a.mode : 0;
  // mode 3 (adaptive): condest.cu decided -- LSQR as mode 1, or the NE x
  return mode0 == 3 ? (a.st->refined ? 1 : 0) : mode0;
}

__global__ void __launch_bounds__(kThreads) lsqr_final_kernel(LsqrArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[96];
  __shared__ double bcast;
  LG_MARK(0);
  const int f = a.st->f;
  const int mode = lsqr_mode_of(a, f);
  int itn = 0, istop = 0;
  if (mode != 0) lsqr_iterate_global(a, grid, mode, f, red, &bcast, itn, istop);
  LG_MARK(2);
  lsqr_finish(a, grid, mode, f, itn, istop, red, &bcast);
  LG_MARK(3);
}

// ===========================================================================
// Grid-resident LSQR (config 2 and other problems too large for one
// cluster): one CTA per SM (kResThreads) keeps, for the whole solve, a row
// slice of A_F (rows [r0,r1), columns renumbered to their position in F) in
// two orders -- by row for A_F v, and the same entries by F column for this
// slice's share of A_F^T u -- plus its piece of u, the pieces of v, w, x of
// its F columns [k0,k1), and a replica of all of v, in shared memory.
// Per iteration:
//   A  rows:  U = A_F v - alpha u; the slice's partial sums of A_F^T U,
//             written as part[cta][k] (shared memory only until that store)  |U|^2
//   -- grid barrier --
//   B  cols:  V = A_F^T u - beta v for own columns: the G partials of each
//             column summed in a fixed order (L2 reads, deterministic)  |V|^2
//   -- grid barrier --
//   C  cols:  x, w updates; the v replica refreshed from V (f doubles, L2)
// No u or v element is gathered from global memory.  The scalar recurrence,
// the vscale bookkeeping, the deterministic norm reductions and the
// stopping tests are those of lsqr_iterate_global, so both paths compute the
// same LSQR iterates up to the summation order of the two products.  The
// slice sizes are planned in the kernel (F is only known on the device); if
// any CTA's slices exceed kResSmem (or G f > nnz: the partials live in
// Fval), every CTA takes the global-memory iteration instead (the decision
// is grid-uniform).
// ===========================================================================
#ifndef NNLS_RES_THREADS
#define NNLS_RES_THREADS 512
#endif
constexpr int kResThreads = NNLS_RES_THREADS;
constexpr int kResSmem = 222 * 1024;

__device__ __forceinline__ size_t res_al(size_t b) { return (b + 15) & ~(size_t)15; }

// block-wide sum returned to every thread
__device__ double block_sum_all(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < nw; ++w) t += red[w];
  __syncthreads();
  return t;
}
// block-wide exclusive scan of one int per thread; *total = the block sum
__device__ int block_scan_excl(int v, int* wsum, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int t = lane < nw ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, t, o);
      if (lane >= o) t += y;
    }
    wsum[lane] = t;
  }
  __syncthreads();
  *total = wsum[nw - 1];
  return (wid > 0 ? wsum[wid - 1] : 0) + x - v;
}

// false (grid-uniform): the slices do not fit, nothing but the map was written
__device__ bool lsqr_iterate_resident(const LsqrArgs& a, cg::grid_group& grid, int mode, int f, double* red,
                                      double* bcast, int* wsum, int& itn, int& istop) {
  extern __shared__ __align__(16) unsigned char rsm[];
  const int tid = threadIdx.x, nb = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5, nw = nb >> 5;
  const int G = gridDim.x, bid = blockIdx.x;
  const int m = a.m;
  const int32_t* __restrict__ Fidx = a.Fidx;
  int* map = reinterpret_cast<int*>(a.R);  // j -> position of j in F (R is free until the report)
  // per-CTA partial sums of A_F^T U, [cta][k] (coalesced stores): in Fval
  // (its entries are in shared memory after the setup; the plan checks G f <= nnz)
  double* part = a.Fval;
  const int r0 = (int)((long long)m * bid / G), r1 = (int)((long long)m * (bid + 1) / G);
  const int k0 = (int)((long long)f * bid / G), k1 = (int)((long long)f * (bid + 1) / G);
  const int R = r1 - r0, C = k1 - k0;
  // ---- plan
  for (int k = bid * nb + tid; k < f; k += G * nb) map[Fidx[k]] = k;
  double nzr = 0.0;
  for (int r = r0 + tid; r < r1; r += nb) nzr += (double)a.Fcnt[r];
  const size_t NZR = (size_t)block_sum_all(nzr, red);
  const size_t o_ul = res_al(8 * (size_t)f), o_vo = o_ul + res_al(8 * (size_t)R);
  const size_t o_wo = o_vo + res_al(8 * (size_t)C), o_xo = o_wo + res_al(8 * (size_t)C);
  const size_t o_rv = o_xo + res_al(8 * (size_t)C), o_qv = o_rv + res_al(8 * NZR);
  const size_t o_rp = o_qv + res_al(8 * NZR), o_rc = o_rp + res_al(4 * (size_t)(R + 1));
  const size_t o_qp = o_rc + res_al(4 * NZR), o_qr = o_qp + res_al(4 * (size_t)(f + 1));
  // column totals: nch chunks of CTAs per own column, then the chunk sums in order
  const int nch = C > 0 ? max(1, min(G, nb / C)) : 1;
  const size_t o_ct = o_qr + res_al(4 * max(NZR, (size_t)R + 1));
  const size_t need = o_ct + res_al(8 * ((size_t)nch * C + C));
  if (tid == 0) a.partials[bid * kSlots + 7] = (double)need;
  grid.sync();
  const bool fits = (long long)G * f <= (long long)a.rowptr[m] && R < (1 << 30);
  const double cap = (a.res_cap > 0 && a.res_cap < kResSmem) ? (double)a.res_cap : (double)kResSmem;
  if (!fits || grid_total(a.partials, 7, bcast, 2) > cap) return false;
  double* vs = reinterpret_cast<double*>(rsm);
  double* ul = reinterpret_cast<double*>(rsm + o_ul);
  double* Vo = reinterpret_cast<double*>(rsm + o_vo);
  double* Wo = reinterpret_cast<double*>(rsm + o_wo);
  double* Xo = reinterpret_cast<double*>(rsm + o_xo);
  double* rv = reinterpret_cast<double*>(rsm + o_rv);  // row slice: values, F positions
  double* qv = reinterpret_cast<double*>(rsm + o_qv);  // the same entries by F column: values, local rows
  int* rp = reinterpret_cast<int*>(rsm + o_rp);
  int* rc = reinterpret_cast<int*>(rsm + o_rc);
  int* qp = reinterpret_cast<int*>(rsm + o_qp);
  int* qr = reinterpret_cast<int*>(rsm + o_qr);
  double* ctot = reinterpret_cast<double*>(rsm + o_ct);  // [C] totals, then [nch][C] chunk sums
  // ---- slices.  Row pointers by a block scan of the F counts (the global
  // row starts staged beside them); the entries copied one per thread (row
  // by a binary search of the pointers); the column view of the same entries
  // by a counting sort on the F position, each column's few entries then put
  // in row order (a deterministic summation order for partial_AtU).
  int* rsrc = qr;  // (staging: the global start of each row; qr is filled last)
  {
    int run = 0, tot = 0;
    for (int base = 0; base < R; base += nb) {
      const int i = base + tid;
      const int cnt = i < R ? a.Fcnt[r0 + i] : 0;
      const int ex = block_scan_excl(cnt, wsum, &tot);
      if (i < R) {
        rp[i] = run + ex;
        rsrc[i] = a.rowptr[r0 + i];
      }
      run += tot;
    }
    if (tid == 0) rp[R] = run;
  }
  int* cur = reinterpret_cast<int*>(vs);  // (column counters; vs is filled after the setup)
  for (int k = tid; k <= f; k += nb) cur[k] = 0;
  __syncthreads();
#pragma unroll 4
  for (int t = tid; t < (int)NZR; t += nb) {
    int lo = 0, hi = R;  // row i: rp[i] <= t < rp[i+1]
    while (hi - lo > 1) {
      const int md = (lo + hi) >> 1;
      if (rp[md] <= t) lo = md; else hi = md;
    }
    const int src = rsrc[lo] + (t - rp[lo]);
    rv[t] = a.Fval[src];
    const int k = __ldcg(&map[a.Fcol[src]]);
    rc[t] = k;
    atomicAdd(&cur[k], 1);
  }
  __syncthreads();
  {
    int run = 0, tot = 0;
    for (int base = 0; base < f; base += nb) {
      const int k = base + tid;
      const int cnt = k < f ? cur[k] : 0;
      const int ex = block_scan_excl(cnt, wsum, &tot);
      if (k < f) {
        qp[k] = run + ex;
        cur[k] = run + ex;
      }
      run += tot;
    }
    if (tid == 0) qp[f] = run;
  }
  __syncthreads();
  for (int i = wid; i < R; i += nw)
    for (int t = rp[i] + lane; t < rp[i + 1]; t += 32) {
      const int d = atomicAdd(&cur[rc[t]], 1);
      qv[d] = rv[t];
      qr[d] = i;
    }
  __syncthreads();
  for (int k = tid; k < f; k += nb) {  // insertion sort of column k's entries by row
    const int q0 = qp[k], q1 = qp[k + 1];
    for (int t = q0 + 1; t < q1; ++t) {
      const int rr = qr[t];
      const double vv = qv[t];
      int u = t - 1;
      while (u >= q0 && qr[u] > rr) {
        qr[u + 1] = qr[u];
        qv[u + 1] = qv[u];
        --u;
      }
      qr[u + 1] = rr;
      qv[u + 1] = vv;
    }
  }
  for (int c = tid; c < C; c += nb) {
    Vo[c] = 0.0;
    Wo[c] = 0.0;
    Xo[c] = 0.0;
  }
  if (mode == 2)
    for (int k = tid; k < f; k += nb) vs[k] = a.x_ne[Fidx[k]];
  __syncthreads();
  LG_MARK(1);
  const int itn_limit = a.itn_limit > 0 ? a.itn_limit : 4 * f;
  // partial A_F^T U of this CTA's rows, column k -> part[bid * f + k] (fixed order per column)
  auto partial_AtU = [&]() {
    double* dst = part + (size_t)bid * f;
    for (int k = tid; k < f; k += 2 * nb) {  // columns k and k + nb interleaved
      const int k2 = k + nb;
      const int a0 = qp[k], a1 = qp[k + 1];
      const int b0 = k2 < f ? qp[k2] : 0, b1 = k2 < f ? qp[k2 + 1] : 0;
      double s = 0.0, s2 = 0.0;
      for (int t = 0; t < max(a1 - a0, b1 - b0); ++t) {
        if (a0 + t < a1) s = fma(qv[a0 + t], ul[qr[a0 + t]], s);
        if (b0 + t < b1) s2 = fma(qv[b0 + t], ul[qr[b0 + t]], s2);
      }
      dst[k] = s;
      if (k2 < f) dst[k2] = s2;
    }
  };
  // own columns: ctot[c] = the G partials of column k0 + c, summed over CTAs
  // [G h / nch, G (h+1) / nch) per chunk h, then over h in order (the same
  // order in every run); consecutive threads read consecutive columns
  auto column_totals = [&]() {
    double* cs = ctot + C;
    for (int idx = tid; idx < nch * C; idx += nb) {
      const int c = idx % C, h = idx / C;
      const int b1 = (int)((long long)G * (h + 1) / nch);
      double s = 0.0;
      for (int b = (int)((long long)G * h / nch); b < b1; b += 8) {  // eight loads in flight, summed in order
        double pv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) pv[u] = b + u < b1 ? __ldcg(&part[(size_t)(b + u) * f + k0 + c]) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (b + u < b1) s += pv[u];
      }
      cs[idx] = s;
    }
    __syncthreads();
    for (int c = tid; c < C; c += nb) {
      double s = 0.0;
      for (int h = 0; h < nch; ++h) s += cs[h * C + c];
      ctot[c] = s;
    }
  };
  // ---- start: U = rhs (cold: b; warm: b - A_F x_ne); beta = |U|
  double p = 0.0;
  for (int i = tid; i < R; i += nb) {
    double s = 0.0;
    if (mode == 2)
      for (int t = rp[i]; t < rp[i + 1]; ++t) s = fma(rv[t], vs[rc[t]], s);
    const double u = a.b[r0 + i] - s;
    ul[i] = u;
    p += u * u;
  }
  block_partial_sum(p, a.partials, 0, red);  // (its barriers order ul before the partial products)
  LG_MARK(8);
  grid.sync();                               // every CTA's Fval reads done: part may be written
  LG_MARK(9);
  partial_AtU();
  grid.sync();
  double beta = sqrt(grid_total(a.partials, 0, bcast, 0));
  const double bnorm = beta;
  // V = A_F^T u (u = U / beta); alpha = |V|
  p = 0.0;
  if (beta > 0.0) {
    const double ib = 1.0 / beta;
    column_totals();
    for (int c = tid; c < C; c += nb) {
      const double s = ctot[c] * ib;
      Vo[c] = s;
      a.V[k0 + c] = s;
      p += s * s;
    }
  }
  block_partial_sum(p, a.partials, 1, red);
  grid.sync();
  double alpha = beta > 0.0 ? sqrt(grid_total(a.partials, 1, bcast, 0)) : 0.0;
  if (alpha > 0.0) {
    const double ia = 1.0 / alpha;
    for (int c = tid; c < C; c += nb) {
      const double v = Vo[c] * ia;
      Vo[c] = v;
      Wo[c] = v;
    }
    for (int k = tid; k < f; k += nb) vs[k] = __ldcg(&a.V[k]) * ia;
  }
  __syncthreads();
  double rhobar = alpha, phibar = beta, anorm = 0.0, ddnorm = 0.0;
  const double ctol = a.conlim > 0.0 ? 1.0 / a.conlim : 0.0;
  double pd = 0.0, px = 0.0, last_phi = 0.0, last_sn = 0.0;
  bool pending = false;
  double vscale = 1.0;  // Vo, vs and V hold v unnormalised (v = V vscale), as in lsqr_iterate_global
  if (alpha * beta != 0.0) {
    const int g4 = tid >> 2, s4 = tid & 3, ng4 = nb >> 2;
    LG_MARK(7);
    for (;;) {
      const bool more = itn < itn_limit;
      LG_STAMP(0);
      // ---- phase A: U = A_F v - alpha u (four lanes per row), then this
      //      slice's partial A_F^T U (phase B's products) -- shared memory only
      const double au = beta > 0.0 ? alpha / beta : 0.0;
      p = 0.0;
      if (more) {
        if (R <= nb) {  // a thread per row, four independent gathers in flight
          if (tid < R) {
            const int t0 = rp[tid], t1 = rp[tid + 1];
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int t = t0;
            for (; t + 4 <= t1; t += 4) {
              s0 = fma(rv[t], vs[rc[t]], s0);
              s1 = fma(rv[t + 1], vs[rc[t + 1]], s1);
              s2 = fma(rv[t + 2], vs[rc[t + 2]], s2);
              s3 = fma(rv[t + 3], vs[rc[t + 3]], s3);
            }
            for (; t < t1; ++t) s0 = fma(rv[t], vs[rc[t]], s0);
            const double s = (s0 + s1) + (s2 + s3);
            const double u = s * vscale - au * ul[tid];
            ul[tid] = u;
            p += u * u;
          }
        } else {
          for (int base = 0; base < R; base += ng4) {
            const int i = base + g4;
            double s = 0.0;
            if (i < R) {
              const int t1 = rp[i + 1];
              for (int t = rp[i] + s4; t < t1; t += 4) s = fma(rv[t], vs[rc[t]], s);
            }
            s += __shfl_xor_sync(kFull, s, 2);
            s += __shfl_xor_sync(kFull, s, 1);
            if (s4 == 0 && i < R) {
              const double u = s * vscale - au * ul[i];
              ul[i] = u;
              p += u * u;
            }
          }
        }
        LG_STAMP(6);
        __syncthreads();
        partial_AtU();
      }
      LG_STAMP(1);
      {
        const double v3[3] = {p, pd, px};
        block_partial_sum3(v3, 3, a.partials, 0, red);
      }
      grid.sync();
      LG_STAMP(2);
      double gt[3];
      grid_sum3(a.partials, 0, 3, gt, red);
      if (pending) {  // stopping test of the previous iteration
        ddnorm += gt[1];
        const double xnorm = sqrt(gt[2]);
        const double acond = anorm * sqrt(ddnorm);
        const double rnorm = phibar;
        const double arnorm = alpha * fabs(last_sn * last_phi);
        const double test1 = bnorm > 0.0 ? rnorm / bnorm : 0.0;
        const double test2 = (anorm * rnorm) > 0.0 ? arnorm / (anorm * rnorm) : 0.0;
        const double test3 = acond > 0.0 ? 1.0 / acond : 0.0;
        const double tt1 = bnorm > 0.0 ? test1 / (1.0 + anorm * xnorm / bnorm) : 0.0;
        const double rtol = a.btol + (bnorm > 0.0 ? a.atol * anorm * xnorm / bnorm : 0.0);
        if (itn >= itn_limit) istop = 7;
        if (1.0 + test3 <= 1.0) istop = 6;
        if (1.0 + test2 <= 1.0) istop = 5;
        if (1.0 + tt1 <= 1.0) istop = 4;
        if (test3 <= ctol) istop = 3;
        if (test2 <= a.atol) istop = 2;
        if (test1 <= rtol) istop = 1;
        if (istop != 0) break;
      }
      ++itn;
      const double beta_new = sqrt(gt[0]);
      // ---- phase B: V' = A_F^T u - beta v, own columns: the G partials summed (L2, coalesced)
      double alpha_new = alpha;
      if (beta_new > 0.0) {
        anorm = sqrt(anorm * anorm + alpha * alpha + beta_new * beta_new);
        const double ib = 1.0 / beta_new;
        p = 0.0;
        column_totals();
        for (int c = tid; c < C; c += nb) {
          const double v = ctot[c] * ib - beta_new * (Vo[c] * vscale);
          Vo[c] = v;  // unnormalised
          a.V[k0 + c] = v;
          p += v * v;
        }
        LG_STAMP(3);
        block_partial_sum(p, a.partials, 4, red);
        grid.sync();
        LG_STAMP(4);
        grid_sum3(a.partials, 4, 1, gt, red);
        alpha_new = sqrt(gt[0]);
      }
      beta = beta_new;
      // ---- rotation (replicated scalars)
      const double rho = sqrt(rhobar * rhobar + beta * beta);
      const double irho = 1.0 / rho;
      const double cs = rhobar * irho, sn = beta * irho;
      const double theta = sn * alpha_new;
      rhobar = -cs * alpha_new;
      const double phi = cs * phibar;
      phibar = sn * phibar;
      const double t1 = phi * irho, t2 = -theta * irho;
      // ---- phase C: v = V'/alpha, x += t1 w, w = v + t2 w (own columns); v replica
      if (beta_new > 0.0 && alpha_new > 0.0) vscale = 1.0 / alpha_new;
      pd = 0.0;
      px = 0.0;
      for (int c = tid; c < C; c += nb) {
        const double v = Vo[c] * vscale;
        const double w = Wo[c];
        const double d = w * irho;
        pd += d * d;
        const double x = Xo[c] + t1 * w;
        Xo[c] = x;
        Wo[c] = v + t2 * w;
        px += x * x;
      }
      if (beta_new > 0.0)
        for (int k = tid; k < f; k += nb) vs[k] = __ldcg(&a.V[k]);
      __syncthreads();
      alpha = alpha_new;
      last_phi = phi;
      last_sn = sn;
      pending = true;
      LG_STAMP(5);
    }
  }
  LG_MARK(2);
  // ---- x (zeroing, c16) and the a11 report from the resident slices: x is
  // zero off F, so R = A x - b needs only the row slice (x_F replicated in
  // shared memory), A^T R on the F columns is the partial-sum pass of
  // phase B, and only the G columns gather R from global memory (CSC).
  double pinf = 0.0;
  for (int c = tid; c < C; c += nb) {
    const int j = Fidx[k0 + c];
    double v = mode == 2 ? a.x_ne[j] + Xo[c] : Xo[c];
    if (fabs(v) < a.tol) v = 0.0;
    if (v < 0.0) pinf = 1.0;
    a.x_out[j] = v;
    a.V[k0 + c] = v;  // (compact copy for the replicas)
    Wo[c] = v;
  }
  const int g = a.n - f;
  const int32_t* __restrict__ Gidx = a.Gidx;
  const int q0 = (int)((long long)g * bid / G), q1 = (int)((long long)g * (bid + 1) / G);
  for (int t = q0 + tid; t < q1; t += nb) a.x_out[Gidx[t]] = 0.0;
  block_partial_minmax(pinf, a.partials, 4, red, false);
  grid.sync();
  LG_MARK(4);
  const double infeas = grid_total(a.partials, 4, bcast, 2);
  if (bid == 0 && tid == 0) {
    a.st->lsqr_iterations = itn;
    a.st->lsqr_stop = istop;
    a.st->infeasible_after_lsqr = (infeas > 0.0) ? 1 : 0;
    a.st->free_count = f;
  }
  if (!a.kkt) return true;
  for (int k = tid; k < f; k += nb) vs[k] = __ldcg(&a.V[k]);
  __syncthreads();
  double po = 0.0;
  for (int i = tid; i < R; i += nb) {  // R = A_F x_F - b on own rows
    double s0 = 0.0, s1 = 0.0;
    const int t1 = rp[i + 1];
    int t = rp[i];
    for (; t + 2 <= t1; t += 2) {
      s0 = fma(rv[t], vs[rc[t]], s0);
      s1 = fma(rv[t + 1], vs[rc[t + 1]], s1);
    }
    if (t < t1) s0 = fma(rv[t], vs[rc[t]], s0);
    const double rr = (s0 + s1) - a.b[r0 + i];
    ul[i] = rr;
    a.R[r0 + i] = rr;
    po += rr * rr;
  }
  __syncthreads();
  partial_AtU();  // this slice's partial A_F^T R
  block_partial_sum(po, a.partials, 0, red);
  grid.sync();
  LG_MARK(5);
  double mx = INFINITY, my = INFINITY, mc = 0.0, dot = 0.0;
  column_totals();  // own F columns: y'_j
  for (int c = tid; c < C; c += nb) {
    const double xj = Wo[c], yj = ctot[c];
    mx = fmin(mx, xj);
    my = fmin(my, yj);
    mc = fmax(mc, fabs(xj * yj));
    dot += xj * yj;
  }
  for (int t = q0 + wid; t < q1; t += nw) {  // own G columns: y'_j = A_j^T R (x_j = 0)
    const int j = Gidx[t];
    double sj = 0.0;
    const int t1 = a.colptr[j + 1];
#pragma unroll 4
    for (int e = a.colptr[j] + lane; e < t1; e += 32) sj = fma(a.cvals[e], __ldcg(&a.R[a.rowind[e]]), sj);
    sj = warp_sum(sj);
    if (lane == 0) {
      mx = fmin(mx, 0.0);
      my = fmin(my, sj);
    }
  }
  block_partial_minmax(mx, a.partials, 1, red, true);
  block_partial_minmax(my, a.partials, 2, red, true);
  block_partial_minmax(mc, a.partials, 3, red, false);
  block_partial_sum(dot, a.partials, 4, red);
  grid.sync();
  LG_MARK(6);
  if (bid == 0 && wid < 5) {  // five totals at once (a warp each, fixed order)
    const int kind = wid == 0 || wid == 4 ? 0 : (wid == 3 ? 2 : 1);
    double v = kind == 0 ? 0.0 : (kind == 1 ? INFINITY : -INFINITY);
    for (int b = lane; b < G; b += 32) {
      const double u = __ldcg(&a.partials[b * kSlots + wid]);
      v = kind == 0 ? v + u : (kind == 1 ? fmin(v, u) : fmax(v, u));
    }
    v = kind == 0 ? warp_sum(v) : (kind == 1 ? warp_min(v) : warp_max(v));
    if (lane == 0) {
      if (wid == 0) a.st->objective = 0.5 * v;
      else if (wid == 1) a.st->kkt_min_x = v;
      else if (wid == 2) a.st->kkt_min_y = v;
      else if (wid == 3) a.st->kkt_max_comp = v;
      else a.st->kkt_dot = v;
    }
  }
  return true;
}

__global__ void __launch_bounds__(kResThreads, 1) lsqr_resident_kernel(LsqrArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[96];
  __shared__ double bcast;
  __shared__ int wsum[32];
  LG_MARK(0);
  const int f = a.st->f;
  const int mode = lsqr_mode_of(a, f);
  int itn = 0, istop = 0;
  if (mode != 0) {
    if (lsqr_iterate_resident(a, grid, mode, f, red, &bcast, wsum, itn, istop)) {
      LG_MARK(3);  // (x and the report done from the slices)
      return;
    }
    lsqr_iterate_global(a, grid, mode, f, red, &bcast, itn, istop);
  }
  LG_MARK(2);
  lsqr_finish(a, grid, mode, f, itn, istop, red, &bcast);
  LG_MARK(3);
}

cudaError_t launch_lsqr_final(const LsqrArgs& a, int sm_count, cudaStream_t s) {
  LsqrArgs args = a;
  void* params[] = {&args};
  // (read per launch: a handle captures its solve graph once, so a test can
  // select the path per handle)
  const char* ev = getenv("NNLS_NO_RESIDENT_LSQR");
  const bool no_res = ev != nullptr && ev[0] != 0 && ev[0] != '0';
  const char* cv = getenv("NNLS_RESIDENT_CAP");  // shared-memory budget of the slices (bytes; test hook)
  args.res_cap = (cv != nullptr && cv[0] != 0) ? atoi(cv) : 0;
  if (!no_res) {
    static DeviceOnce once;
    const int ok = device_once(once, [] {
      if (cudaFuncSetAttribute(lsqr_resident_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kResSmem) !=
          cudaSuccess)
        return -1;
      int per = 0;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, lsqr_resident_kernel, kResThreads, kResSmem) !=
              cudaSuccess ||
          per < 1)
        return -1;
      return 1;
    });
    if (ok == 1)
      return cudaLaunchCooperativeKernel((void*)lsqr_resident_kernel, dim3(sm_count), dim3(kResThreads), params,
                                         (size_t)kResSmem, s);
    cudaGetLastError();
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lsqr_final_kernel, kThreads, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorLaunchOutOfResources;
  if (per_sm > 4) per_sm = 4;  // partials[] holds 4 CTAs per SM
  int grid = sm_count * per_sm;  // every co-resident CTA (latency-bound gathers)
  return cudaLaunchCooperativeKernel((void*)lsqr_final_kernel, dim3(grid), dim3(kThreads), params, 0, s);
}

// ===========================================================================
// Cluster-resident LSQR (configs 0, 1, 3: A fits in the shared memory of one
// 16-CTA thread-block cluster).  Each CTA keeps its CSR row slice and CSC
// column slice (balanced by nonzeros) in shared memory for the whole solve,
// plus full replicas of u (m) and v (n).  Vector pieces are exchanged by
// pushing them into every CTA's replica through distributed shared memory
// (st.shared::cluster), norms by reading the 16 partials from each CTA's
// shared memory in a fixed order (deterministic, identical in every CTA).
// Two cluster barriers per iteration (the stopping test of iteration i is
// evaluated after the first barrier of iteration i+1; no extra state is
// touched before it, so the result is the standard LSQR iterate).
// ===========================================================================
namespace {
constexpr int kCT = 512;
constexpr int kMaxC = 16;

struct ClSlices {
  int r0, r1, e0, e1;   // rows [r0,r1), CSR entries [e0,e1)
  int j0, j1, f0, f1;   // cols [j0,j1), CSC entries [f0,f1)
};

struct ClLayout {
  int rows_max, cols_max, nzr_max, nzc_max;
  size_t bytes;
};

__host__ __device__ inline ClLayout cl_layout(int m, int n, const int* mx) {
  ClLayout L;
  L.rows_max = mx[0];
  L.nzr_max = mx[1];
  L.cols_max = mx[2];
  L.nzc_max = mx[3];
  size_t d = (size_t)m + n + L.nzr_max + L.nzc_max + 4 * (size_t)L.cols_max + 3 * 32;
  size_t i = (size_t)L.nzr_max + L.nzc_max + L.rows_max + 1 + L.cols_max + 1 + 2 * (size_t)L.cols_max;
  L.bytes = 8 * d + 4 * i + 64;
  return L;
}
}  // namespace

// plan: per-CTA slice bounds and maxima for cluster size C.  out[0..3] =
// max rows, CSR nnz, cols, CSC nnz of a slice; out[4 .. 4+C] = row bounds,
// out[5+C .. 5+2C] = column bounds (slice k: rows [rb[k], rb[k+1])).  Bound k
// is the first row r with rowptr[r] >= nnz*k/C (nnz-balanced), found by
// every thread checking its own rows against all C thresholds (no serial
// binary searches).
__global__ void __launch_bounds__(1024) lsqr_plan_kernel(int m, int n, const int32_t* rowptr,
                                                         const int32_t* colptr, int C, int* out) {
  __shared__ int thr[kMaxC];
  pdl_wait();
  int* rb = out + 4;
  int* cb = out + 5 + C;
  const int tid = threadIdx.x;
  if (tid < C) thr[tid] = (int)((long long)rowptr[m] * tid / C);
  __syncthreads();
  for (int r = tid; r <= m; r += blockDim.x) {
    const int v = rowptr[r], vp = r > 0 ? rowptr[r - 1] : (-0x7fffffff - 1);
    if (v == vp) continue;  // (an empty row is never a first crossing)
    for (int k = 1; k < C; ++k)
      if (vp < thr[k] && v >= thr[k]) rb[k] = r;
  }
  for (int j = tid; j <= n; j += blockDim.x) {
    const int v = colptr[j], vp = j > 0 ? colptr[j - 1] : (-0x7fffffff - 1);
    if (v == vp) continue;
    for (int k = 1; k < C; ++k)
      if (vp < thr[k] && v >= thr[k]) cb[k] = j;
  }
  if (tid == 0) {
    rb[0] = 0;
    rb[C] = m;
    cb[0] = 0;
    cb[C] = n;
  }
  __syncthreads();
  if (tid < 32) {
    int v[4] = {0, 0, 0, 0};
    if (tid < C) {
      const int r0 = rb[tid], r1 = max(rb[tid + 1], r0), j0 = cb[tid], j1 = max(cb[tid + 1], j0);
      v[0] = r1 - r0;
      v[1] = rowptr[r1] - rowptr[r0];
      v[2] = j1 - j0;
      v[3] = colptr[j1] - colptr[j0];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int x = warp_max_i(v[q]);
      if (tid == 0) out[q] = x;
    }
  }
}

// setup / epilogue stamps go to row 63 (slots 0..)
#define LQ_STAMP_SETUP(slot)                                                               \
  do {                                                                                     \
    if (g_lsqr_prof != nullptr && kr == 0 && threadIdx.x == 0) {                           \
      unsigned long long t_;                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
      g_lsqr_prof[63 * 16 + (slot)] = t_;                                                  \
    }                                                                                      \
  } while (0)
#define LQ_STAMP(slot)                                                                     \
  do {                                                                                     \
    if (g_lsqr_prof != nullptr && kr == 0 && threadIdx.x == 0 && itn < 64) {               \
      unsigned long long t_;                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
      g_lsqr_prof[itn * 16 + (slot)] = t_;                                                 \
    }                                                                                      \
  } while (0)
cudaError_t lsqr_debug_set_profile(unsigned long long* p) {
  return cudaMemcpyToSymbol(g_lsqr_prof, &p, sizeof(p));
}

// Sub-warp segmented dot products: segment q (a row of the CSR slice or a
// column of the CSC slice) is handled by a group of g lanes (g = power of two
// sized so that all segments of the slice are processed in ONE pass by the
// 512 threads), each lane striding over the segment; the group reduces with
// xor-shuffles.  emit(q, s) is called by the group's first lane.
template <class Emit>
__device__ __forceinline__ void seg_dots(int nseg, int g, const int* __restrict__ sp,
                                         const double* __restrict__ val, const int* __restrict__ idx,
                                         const double* __restrict__ vec, const int* __restrict__ skip,
                                         Emit emit, int t0 = 0) {
  if ((int)threadIdx.x < t0) return;  // (whole warps: t0 is a multiple of 32)
  const int tid = threadIdx.x - t0, sl = tid & (g - 1);
  const int per = (kCT - t0) / g;
  for (int base = 0; base < nseg; base += per) {
    const int q = base + tid / g;
    double s = 0.0;
    if (q < nseg && (skip == nullptr || skip[q])) {
      const int t1 = sp[q + 1];
#pragma unroll 4
      for (int t = sp[q] + sl; t < t1; t += g) s = fma(val[t], vec[idx[t]], s);
    }
    for (int o = g >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(kFull, s, o);
    if (sl == 0 && q < nseg) emit(q, s);
  }
}
__device__ __forceinline__ int seg_group(int nseg, int nthreads = kCT) {
  int g = 32;
  while (g > 1 && (long long)nseg * g > nthreads) g >>= 1;
  return g;
}

__global__ void __launch_bounds__(kCT, 1) lsqr_cluster_kernel(LsqrArgs a, ClLayout Ly) {
  cg::cluster_group cl = cg::this_cluster();
  const int C = (int)cl.num_blocks(), kr = (int)cl.block_rank();
  extern __shared__ double smem[];
  __shared__ double red[2][4][32];  // (double-buffered by publish call parity)
  __shared__ double parts[8][kMaxC];  // [slot][source CTA] partials, pushed by every CTA
  pdl_wait();
  const int m = a.m, n = a.n;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int NW = kCT / 32;
  LQ_STAMP_SETUP(0);
  ClSlices S;  // this CTA's slice, from the plan (lsqr_plan_kernel)
  {
    const int* rb = a.plan + 4;
    const int* cbd = a.plan + 5 + C;
    S.r0 = rb[kr];
    S.r1 = max(rb[kr + 1], S.r0);
    S.j0 = cbd[kr];
    S.j1 = max(cbd[kr + 1], S.j0);
    S.e0 = a.rowptr[S.r0];
    S.e1 = a.rowptr[S.r1];
    S.f0 = a.colptr[S.j0];
    S.f1 = a.colptr[S.j1];
  }
  const int nrows = S.r1 - S.r0, ncols = S.j1 - S.j0;
  LQ_STAMP_SETUP(1);
  const int gR = seg_group(nrows);
  // ---- shared memory carve-up
  double* Urep = smem;                 // m  (u replica, unnormalised)
  double* Vrep = Urep + m;             // n  (v replica, unnormalised)
  double* sv = Vrep + n;               // nzr (CSR values of own rows)
  double* scv = sv + Ly.nzr_max;       // nzc (CSC values of own columns)
  double* vo = scv + Ly.nzc_max;       // own columns: v (normalised)
  double* wo = vo + Ly.cols_max;       //              w
  double* xo = wo + Ly.cols_max;       //              x
  double* scr = xo + Ly.cols_max;      //              scratch
  int* sci = reinterpret_cast<int*>(scr + Ly.cols_max + 3 * 32);
  int* sri = sci + Ly.nzr_max;         // CSC row indices
  int* srp = sri + Ly.nzc_max;         // local rowptr (nrows + 1)
  int* scp = srp + Ly.rows_max + 1;    // local colptr (ncols + 1)
  int* smk = scp + Ly.cols_max + 1;    // own column mask
  int* fcol = smk + Ly.cols_max;       // own F columns (local index), in order
  const uint8_t* __restrict__ mask = a.mask;
  __shared__ int s_nfc;

  // ---- stage the slices (once per solve).  Every CSR product of the path
  //      multiplies a vector that is zero outside F (v, x_ne, x), so the row
  //      slice keeps only the F columns; the CSC slice (A^T u, y') is kept whole.
  // the CSC slice keeps only the F columns (every A^T product of the loop is
  // needed on F only; the report's y' over all columns reads the global CSC)
  for (int j = tid; j < ncols; j += kCT) smk[j] = mask[S.j0 + j];
  if (wid == 0) {
    int carry = 0;
    for (int b0 = 0; b0 < ncols; b0 += 32) {
      const int j = b0 + lane;
      const bool inF = j < ncols && mask[S.j0 + j];
      const unsigned bal = __ballot_sync(kFull, inF);
      if (inF) fcol[carry + __popc(bal & ((1u << lane) - 1u))] = j;
      carry += __popc(bal);
    }
    if (lane == 0) s_nfc = carry;
  }
  __syncthreads();
  const int nfc = s_nfc;
  for (int q = tid; q < nfc; q += kCT) scp[q + 1] = a.colptr[S.j0 + fcol[q] + 1] - a.colptr[S.j0 + fcol[q]];
  if (tid == 0) scp[0] = 0;
  __syncthreads();
  if (wid == 0) {  // inclusive scan of the F-column lengths (one warp)
    int carry = 0;
    for (int b0 = 0; b0 < nfc; b0 += 32) {
      int v = (b0 + lane < nfc) ? scp[b0 + lane + 1] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v += y;
      }
      if (b0 + lane < nfc) scp[b0 + lane + 1] = v + carry;
      carry += __shfl_sync(kFull, v, 31);
    }
  }
  __syncthreads();
  for (int q = wid; q < nfc; q += NW) {  // copy the F columns (warp per column, coalesced)
    const int src = a.colptr[S.j0 + fcol[q]], dst = scp[q], cnt = scp[q + 1] - dst;
    for (int t = lane; t < cnt; t += 32) {
      scv[dst + t] = a.cvals[src + t];
      sri[dst + t] = a.rowind[src + t];
    }
  }
  for (int r = tid; r < nrows; r += kCT) srp[r + 1] = __ldcg(&a.Fcnt[S.r0 + r]);  // F-entries per row
  if (tid == 0) srp[0] = 0;
  __syncthreads();
  if (wid == 0) {  // inclusive scan of the row counts (one warp)
    int carry = 0;
    for (int b0 = 0; b0 < nrows; b0 += 32) {
      int v = (b0 + lane < nrows) ? srp[b0 + lane + 1] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(kFull, v, o);
        if (lane >= o) v += y;
      }
      if (b0 + lane < nrows) srp[b0 + lane + 1] = v + carry;
      carry += __shfl_sync(kFull, v, 31);
    }
  }
  __syncthreads();
  for (int r = wid; r < nrows; r += NW) {  // copy the compacted rows (warp per row, coalesced)
    const int pos = srp[r], cnt = srp[r + 1] - pos, base = a.rowptr[S.r0 + r];
    for (int t = lane; t < cnt; t += 32) {
      sv[pos + t] = __ldcg(&a.Fval[base + t]);
      sci[pos + t] = __ldcg(&a.Fcol[base + t]);
    }
  }
  __shared__ double sc[16];  // scalars computed by warp 0, broadcast after a barrier
  __syncthreads();
  LQ_STAMP_SETUP(2);

  // Cluster reductions without remote loads: every CTA reduces its values
  // block-wide and warp 0 PUSHES the block totals into slot [slot+q][kr] of
  // every CTA's parts[][] array; after the cluster barrier each thread sums
  // its local copy in rank order (deterministic, identical everywhere).
  // (red is double-buffered: the readers of call t finish before call t+1's
  // barrier, so call t+2 may overwrite it -- one barrier per call)
  int red_par = 0;
  auto publish = [&](int nv, const double* v, const int* kind, int slot) {
    double (*rb)[32] = red[red_par];
    red_par ^= 1;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      if (q < nv) {
        double x = v[q];
        x = kind[q] == 0 ? warp_sum(x) : (kind[q] == 1 ? warp_min(x) : warp_max(x));
        if (lane == 0) rb[q][wid] = x;
      }
    }
    __syncthreads();
    if (wid < nv) {
      const int k = kind[wid];
      double x = lane < NW ? rb[wid][lane] : (k == 0 ? 0.0 : (k == 1 ? INFINITY : -INFINITY));
      x = k == 0 ? warp_sum(x) : (k == 1 ? warp_min(x) : warp_max(x));
      if (lane < C) *cl.map_shared_rank(&parts[slot + wid][kr], lane) = x;
    }
  };
  // cluster totals of parts[slot..slot+nv): lane r < C loads source r's
  // partial, one xor-butterfly per value (fixed order: identical in every CTA
  // and every warp).  Called by whole warps.
  auto ctotal = [&](int nv, const int* kind, int slot, double* out) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      if (q < nv) {
        const int k = kind[q];
        double x = (lane < C) ? parts[slot + q][lane] : (k == 0 ? 0.0 : (k == 1 ? INFINITY : -INFINITY));
        if (k == 0) x = warp_sum(x);
        else if (k == 1) x = warp_min(x);
        else x = warp_max(x);
        out[q] = x;
      }
    }
  };
  const int K_SUM[3] = {0, 0, 0};
  // push own rows/cols of a replica to every CTA's copy
  // (all 512 threads share the (destination, element) space: a loop over
  //  destinations with only `cnt` active threads was 4x slower)
  auto push = [&](double* rep, int base, int cnt) {  // warp per destination
    for (int d = wid; d < C - 1; d += NW) {
      const int q = d + (d >= kr);  // skip self
      double* dst = cl.map_shared_rank(rep, q);
      for (int i = lane; i < cnt; i += 32) dst[base + i] = rep[base + i];
    }
  };

  const int f = a.st->f;
  const int status = a.st->status;
  const int mode0 = (status == 0 && a.st->done && f > 0) ? a.mode : 0;
  // mode 3 (adaptive): condest.cu decided -- LSQR as mode 1, or the NE x
  const int mode = mode0 == 3 ? (a.st->refined ? 1 : 0) : mode0;
  int itn = 0, istop = 0;

  if (mode != 0) {
    const int itn_limit = a.itn_limit > 0 ? a.itn_limit : 4 * f;
    // U' = rhs on own rows (mode 2: b - A_F x_ne)
    if (mode == 2) {
      for (int j = tid; j < n; j += kCT) Vrep[j] = mask[j] ? __ldcg(&a.x_ne[j]) : 0.0;
      __syncthreads();
    }
    seg_dots(nrows, gR, srp, sv, sci, Vrep, nullptr, [&](int r, double s) {
      Urep[S.r0 + r] = a.b[S.r0 + r] - (mode == 2 ? s : 0.0);
    });
    __syncthreads();
    double p = 0.0;
    for (int r = tid; r < nrows; r += kCT) p += Urep[S.r0 + r] * Urep[S.r0 + r];
    push(Urep, S.r0, nrows);
    publish(1, &p, K_SUM, 0);
    cl.sync();
    double tot[3];
    ctotal(1, K_SUM, 0, tot);
    double beta = sqrt(tot[0]);
    const double bnorm = beta;
    // V' = A_F^T u on own columns
    const double ib0 = beta > 0.0 ? 1.0 / beta : 0.0;
    seg_dots(nfc, seg_group(nfc), scp, scv, sri, Urep, nullptr,
             [&](int q, double s) { Vrep[S.j0 + fcol[q]] = s * ib0; });
    __syncthreads();
    p = 0.0;
    for (int j = tid; j < ncols; j += kCT) {
      if (!smk[j]) Vrep[S.j0 + j] = 0.0;
      p += Vrep[S.j0 + j] * Vrep[S.j0 + j];
    }
    __syncthreads();
    push(Vrep, S.j0, ncols);
    publish(1, &p, K_SUM, 4);
    cl.sync();
    ctotal(1, K_SUM, 4, tot);
    double alpha = beta > 0.0 ? sqrt(tot[0]) : 0.0;
    const double ia0 = alpha > 0.0 ? 1.0 / alpha : 0.0;
    for (int j = tid; j < ncols; j += kCT) {
      const double v = Vrep[S.j0 + j] * ia0;
      vo[j] = v;
      wo[j] = v;
      xo[j] = 0.0;
    }
    double rhobar = alpha, phibar = beta, anorm = 0.0, ddnorm = 0.0;
    double vscale = ia0;  // Vrep * vscale = v
    const double ctol = a.conlim > 0.0 ? 1.0 / a.conlim : 0.0;
    double last_phi = 0.0, last_sn = 0.0;  // for the deferred stopping test
    bool pending = false;
    double pd = 0.0, px = 0.0;
    const int gCw = seg_group(nfc, kCT - 32);  // phase B runs on warps 1.. (warp 0: scalars)
    __syncthreads();
    LQ_STAMP_SETUP(3);
    if (alpha * beta != 0.0) {
      for (;;) {
        // ---- phase A (iteration itn+1): U' = A_F v - alpha u on own rows
        LQ_STAMP(0);
        const bool more = itn < itn_limit;
        if (more) {
          const double au = beta > 0.0 ? alpha / beta : 0.0;
          const double vs = vscale;
          seg_dots(nrows, gR, srp, sv, sci, Vrep, nullptr, [&](int r, double s) {
            Urep[S.r0 + r] = s * vs - au * Urep[S.r0 + r];  // own slot
          });
        }
        __syncthreads();
        LQ_STAMP(1);
        double pu = 0.0;
        if (more) {
          for (int r = tid; r < nrows; r += kCT) pu += Urep[S.r0 + r] * Urep[S.r0 + r];
          push(Urep, S.r0, nrows);
        }
        LQ_STAMP(11);
        {
          const double v3[3] = {pu, pd, px};
          publish(3, v3, K_SUM, 0);  // parts 0 (|U'|^2), 1 (|d|^2), 2 (|x|^2)
        }
        LQ_STAMP(2);
        cl.sync();
        LQ_STAMP(3);
        // ---- warp 0: deferred stopping test of the previous iteration, beta;
        //      warps 1..: the A_F^T U' dots of phase B (no scalar dependency)
        if (wid == 0) {
          double t3[3];
          ctotal(3, K_SUM, 0, t3);
          int stop = 0;
          if (pending) {
            ddnorm += t3[1];
            const double xnorm = sqrt(t3[2]);
            const double acond = anorm * sqrt(ddnorm);
            const double rnorm = phibar;
            const double arnorm = alpha * fabs(last_sn * last_phi);
            const double test1 = bnorm > 0.0 ? rnorm / bnorm : 0.0;
            const double test2 = (anorm * rnorm) > 0.0 ? arnorm / (anorm * rnorm) : 0.0;
            const double test3 = acond > 0.0 ? 1.0 / acond : 0.0;
            const double axb = bnorm > 0.0 ? anorm * xnorm / bnorm : 0.0;
            const double tt1 = bnorm > 0.0 ? test1 / (1.0 + axb) : 0.0;
            const double rtol = a.btol + a.atol * axb;
            if (itn >= itn_limit) stop = 7;
            if (1.0 + test3 <= 1.0) stop = 6;
            if (1.0 + test2 <= 1.0) stop = 5;
            if (1.0 + tt1 <= 1.0) stop = 4;
            if (test3 <= ctol) stop = 3;
            if (test2 <= a.atol) stop = 2;
            if (test1 <= rtol) stop = 1;
          }
          if (lane == 0) {
            const double bn = sqrt(t3[0]);  // beta_new
            sc[0] = bn;
            sc[1] = (double)stop;
            sc[2] = ddnorm;
            // the part of the rotation that does not depend on alpha_new
            // (formed here, in the shadow of the other warps' dots)
            const double rho = sqrt(rhobar * rhobar + bn * bn);
            sc[3] = rho;
            sc[4] = rhobar / rho;  // cs
            sc[5] = bn / rho;      // sn
            sc[6] = (sc[4] * phibar) / rho;  // t1 = phi / rho
            sc[7] = 1.0 / rho;
          }
          LQ_STAMP(12);
        } else if (more) {
          seg_dots(nfc, gCw, scp, scv, sri, Urep, nullptr, [&](int q, double s) { scr[fcol[q]] = s; }, 32);
          if (g_lsqr_prof != nullptr && kr == 0 && threadIdx.x == 32 && itn < 64) {
            unsigned long long t_;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
            g_lsqr_prof[itn * 16 + 13] = t_;
          }
        }
        __syncthreads();
        LQ_STAMP(4);
        istop = (int)sc[1];
        ddnorm = sc[2];
        if (istop != 0) break;
        ++itn;
        const double beta_new = sc[0];
        const double rho = sc[3], cs = sc[4], sn = sc[5], t1 = sc[6], irho = sc[7];
        const double phi = cs * phibar;
        // ---- phase B: V' = A_F^T u - beta v on own columns (u = U'/beta_new)
        double alpha_new = alpha;
        if (beta_new > 0.0) {
          anorm = sqrt(anorm * anorm + alpha * alpha + beta_new * beta_new);
          const double ib = 1.0 / beta_new;
          double pv = 0.0;
          for (int j = tid; j < ncols; j += kCT) {
            if (!smk[j]) continue;
            const double v = scr[j] * ib - beta_new * vo[j];
            Vrep[S.j0 + j] = v;
            pv += v * v;
          }
          __syncthreads();
          LQ_STAMP(5);
          push(Vrep, S.j0, ncols);
          publish(1, &pv, K_SUM, 3);
          LQ_STAMP(6);
          cl.sync();
          LQ_STAMP(7);
          {  // every warp forms the same total (same inputs, same butterfly): no barrier
            double t1v[3];
            ctotal(1, K_SUM, 3, t1v);
            alpha_new = sqrt(t1v[0]);
          }
          LQ_STAMP(8);
        } else {
          cl.sync();  // keep the two-barrier rhythm (partials are reused)
        }
        beta = beta_new;
        // ---- rotation (replicated scalars; rho, cs, sn, phi, t1 formed above)
        const double theta = sn * alpha_new;
        rhobar = -cs * alpha_new;
        phibar = sn * phibar;
        const double t2 = -theta / rho;
        // ---- phase C: v, x, w on own columns (partials ride on the next barrier)
        const bool newv = beta_new > 0.0;
        const double ia = (newv && alpha_new > 0.0) ? 1.0 / alpha_new : 1.0;
        pd = 0.0;
        px = 0.0;
        for (int j = tid; j < ncols; j += kCT) {
          if (!smk[j]) continue;
          double v = vo[j];
          if (newv) {
            v = Vrep[S.j0 + j] * ia;
            vo[j] = v;
          }
          const double w = wo[j];
          const double d = w * irho;
          pd += d * d;
          const double x = xo[j] + t1 * w;
          xo[j] = x;
          wo[j] = v + t2 * w;
          px += x * x;
        }
        if (newv) vscale = ia;
        alpha = alpha_new;
        last_phi = phi;
        last_sn = sn;
        pending = true;
        LQ_STAMP(9);
        LQ_STAMP(10);
      }
    }
  }

  // ---- x on own columns, zeroing (c16), write out, replicate into Vrep
  LQ_STAMP_SETUP(4);
  cl.sync();  // every CTA is done reading the replicas
  double pinf = 0.0;
  for (int j = tid; j < ncols; j += kCT) {
    const int g = S.j0 + j;
    double v;
    if (!mask[g]) v = 0.0;
    else if (mode == 1) v = xo[j];
    else if (mode == 2) v = __ldcg(&a.x_ne[g]) + xo[j];
    else v = __ldcg(&a.x_ne[g]);
    if (fabs(v) < a.tol) v = 0.0;
    if (v < 0.0) pinf = 1.0;
    a.x_out[g] = v;
    Vrep[g] = v;
  }
  __syncthreads();
  push(Vrep, S.j0, ncols);
  {
    const int K_MAX[1] = {2};
    publish(1, &pinf, K_MAX, 6);
    cl.sync();
    double t[3];
    ctotal(1, K_MAX, 6, t);
    if (kr == 0 && tid == 0) {
      a.st->lsqr_iterations = itn;
      a.st->lsqr_stop = istop;
      a.st->infeasible_after_lsqr = (mode != 0 && t[0] > 0.0) ? 1 : 0;
      a.st->free_count = f;
    }
  }
  if (a.kkt) {
    // ---- report: R = A x - b on own rows -> Urep; y' = A^T R on own columns
    seg_dots(nrows, gR, srp, sv, sci, Vrep, nullptr, [&](int r, double s) {
      Urep[S.r0 + r] = s - a.b[S.r0 + r];
    });
    __syncthreads();
    double po = 0.0;
    for (int r = tid; r < nrows; r += kCT) po += Urep[S.r0 + r] * Urep[S.r0 + r];
    push(Urep, S.r0, nrows);
    publish(1, &po, K_SUM, 0);
    cl.sync();
    seg_dots(ncols, seg_group(ncols), a.colptr + S.j0, a.cvals, a.rowind, Urep, nullptr,
             [&](int j, double s) { scr[j] = s; });  // all own columns, global CSC
    __syncthreads();
    double mx = INFINITY, my = INFINITY, mc = 0.0, dot = 0.0;
    for (int j = tid; j < ncols; j += kCT) {
      const double xj = Vrep[S.j0 + j], yj = scr[j];
      mx = fmin(mx, xj);
      my = fmin(my, yj);
      mc = fmax(mc, fabs(xj * yj));
      dot += xj * yj;
    }
    const int K3[3] = {1, 1, 2};
    const double v3[3] = {mx, my, mc};
    publish(3, v3, K3, 1);
    publish(1, &dot, K_SUM, 5);
    cl.sync();
    double o1[3], o3[3], o5[3];
    ctotal(1, K_SUM, 0, o1);
    ctotal(3, K3, 1, o3);
    ctotal(1, K_SUM, 5, o5);
    if (kr == 0 && tid == 0) {
      a.st->objective = 0.5 * o1[0];
      a.st->kkt_min_x = o3[0];
      a.st->kkt_min_y = o3[1];
      a.st->kkt_max_comp = o3[2];
      a.st->kkt_dot = o5[0];
    }
  }
  LQ_STAMP_SETUP(5);
  cl.sync();  // keep every CTA's shared memory alive until remote reads finish
}

// A restricted to the final F, row by row (warp per row, ballot compaction
// keeps the entries in column order), written in place of each row.
__global__ void lsqr_compact_kernel(int m, const int32_t* __restrict__ rowptr,
                                    const int32_t* __restrict__ colind, const double* __restrict__ vals,
                                    const uint8_t* __restrict__ mask, double* __restrict__ Fval,
                                    int32_t* __restrict__ Fcol, int32_t* __restrict__ Fcnt) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < m; r += warps) {
    const int t0 = rowptr[r], t1 = rowptr[r + 1];
    int cnt = 0;
    for (int tb = t0; tb < t1; tb += 32) {
      const int t = tb + lane;
      int j = 0;
      double v = 0.0;
      bool keep = false;
      if (t < t1) {
        j = colind[t];
        v = vals[t];
        keep = mask[j] != 0;
      }
      const unsigned bal = __ballot_sync(kFull, keep);
      if (keep) {
        const int pos = t0 + cnt + __popc(bal & ((1u << lane) - 1u));
        Fval[pos] = v;
        Fcol[pos] = j;
      }
      cnt += __popc(bal);
    }
    if (lane == 0) Fcnt[r] = cnt;
  }
}

cudaError_t launch_lsqr_compact(const LsqrArgs& a, int sm_count, cudaStream_t s) {
  int blocks = (a.m + 7) / 8;
  if (blocks > sm_count * 8) blocks = sm_count * 8;
  if (blocks < 1) blocks = 1;
  lsqr_compact_kernel<<<blocks, 256, 0, s>>>(a.m, a.rowptr, a.colind, a.vals, a.mask, a.Fval, a.Fcol, a.Fcnt);
  return cudaGetLastError();
}

cudaError_t launch_lsqr_plan(int m, int n, const int32_t* rowptr, const int32_t* colptr, int* out,
                             cudaStream_t s) {
  return launch_pdl(lsqr_plan_kernel, dim3(1), dim3(1024), 0, s, m, n, rowptr, colptr, (int)kMaxC, out);
}

size_t lsqr_cluster_smem(int m, int n, const int* plan) { return cl_layout(m, n, plan).bytes; }

cudaError_t launch_lsqr_cluster_planned(const LsqrArgs& a, const int* plan_host, cudaStream_t s) {
  const ClLayout Ly = cl_layout(a.m, a.n, plan_host);
  if (Ly.bytes > 220 * 1024) return cudaErrorNotSupported;
  // attributes and the co-residency check are host round trips: do them once
  // at the maximum shared-memory size (valid for every smaller launch)
  static DeviceOnce once;  // per device: 1 supported, -1 not supported
  constexpr size_t kMaxSmem = 220 * 1024;
  const int checked = device_once(once, [&]() {
    cudaError_t e = cudaFuncSetAttribute(lsqr_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kMaxSmem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(lsqr_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int nclusters = 0;
    if (e == cudaSuccess) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(kMaxC);
      q.blockDim = dim3(kCT);
      q.dynamicSmemBytes = kMaxSmem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = kMaxC;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      q.attrs = at;
      q.numAttrs = 1;
      e = cudaOccupancyMaxActiveClusters(&nclusters, lsqr_cluster_kernel, &q);
    }
    cudaGetLastError();
    return (e == cudaSuccess && nclusters >= 1) ? 1 : -1;
  });
  if (checked < 0) return cudaErrorNotSupported;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kMaxC);
  cfg.blockDim = dim3(kCT);
  cfg.dynamicSmemBytes = Ly.bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kMaxC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // (see launch_pdl)
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, lsqr_cluster_kernel, a, Ly);
}

}  // namespace nnls
