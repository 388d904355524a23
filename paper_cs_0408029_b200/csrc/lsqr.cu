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

__global__ void __launch_bounds__(kThreads) lsqr_final_kernel(LsqrArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[32];
  __shared__ double bcast;
  const int lane = threadIdx.x & 31;
  const int gwarp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nthr = gridDim.x * blockDim.x;
  const int m = a.m, n = a.n;
  const int status = a.st->status;
  const int f = a.st->f;
  const uint8_t* __restrict__ mask = a.mask;
  const int mode = (status == 0 && a.st->done && f > 0) ? a.mode : 0;

  int itn = 0, istop = 0;
  if (mode != 0) {
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
    if (alpha * beta != 0.0) {
      while (itn < itn_limit) {
        ++itn;
        // ---- phase A: U = A v - alpha u, u = U / beta
        const double au = beta > 0.0 ? alpha / beta : 0.0;
        p = 0.0;
        for (int r = gwarp; r < m; r += nwarps) {
          double s = 0.0;
          for (int t = a.rowptr[r] + lane; t < a.rowptr[r + 1]; t += 32)
            s = fma(a.vals[t], __ldcg(&a.V[a.colind[t]]), s);
          s = warp_sum(s);
          if (lane == 0) {
            const double u = s - au * a.U[r];
            a.U[r] = u;
            p += u * u;
          }
        }
        block_partial_sum(p, a.partials, 0, red);
        grid.sync();
        const double beta_new = sqrt(grid_total(a.partials, 0, &bcast, 0));
        // ---- phase B: V' = A_F^T u - beta v
        double alpha_new = alpha;
        if (beta_new > 0.0) {
          anorm = sqrt(anorm * anorm + alpha * alpha + beta_new * beta_new);
          const double ib = 1.0 / beta_new;
          p = 0.0;
          for (int j = gwarp; j < n; j += nwarps) {
            if (!mask[j]) continue;
            double s = 0.0;
            for (int t = a.colptr[j] + lane; t < a.colptr[j + 1]; t += 32)
              s = fma(a.cvals[t], __ldcg(&a.U[a.rowind[t]]), s);
            s = warp_sum(s) * ib;
            if (lane == 0) {
              const double v = s - beta_new * __ldcg(&a.V[j]);
              a.V[j] = v;
              p += v * v;
            }
          }
          block_partial_sum(p, a.partials, 1, red);
          grid.sync();
          alpha_new = sqrt(grid_total(a.partials, 1, &bcast, 0));
        }
        beta = beta_new;
        // ---- rotation (replicated scalars)
        const double rho = sqrt(rhobar * rhobar + beta * beta);
        const double cs = rhobar / rho, sn = beta / rho;
        const double theta = sn * alpha_new;
        rhobar = -cs * alpha_new;
        const double phi = cs * phibar;
        phibar = sn * phibar;
        const double t1 = phi / rho, t2 = -theta / rho;
        // ---- phase C: v = V'/alpha, x += t1 w, w = v + t2 w
        const double ia = alpha_new > 0.0 ? 1.0 / alpha_new : 0.0;
        double pd = 0.0, px = 0.0;
        for (int j = gtid; j < n; j += nthr) {
          if (!mask[j]) continue;
          double v = __ldcg(&a.V[j]);
          if (beta_new > 0.0 && alpha_new > 0.0) {
            v *= ia;
            a.V[j] = v;
          }
          const double w = a.W[j];
          const double d = w / rho;
          pd += d * d;
          const double x = a.X[j] + t1 * w;
          a.X[j] = x;
          a.W[j] = v + t2 * w;
          px += x * x;
        }
        alpha = alpha_new;
        block_partial_sum(pd, a.partials, 2, red);
        block_partial_sum(px, a.partials, 3, red);
        grid.sync();
        ddnorm += grid_total(a.partials, 2, &bcast, 0);
        const double xnorm = sqrt(grid_total(a.partials, 3, &bcast, 0));
        const double acond = anorm * sqrt(ddnorm);
        const double rnorm = phibar;
        const double arnorm = alpha * fabs(sn * phi);
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
    }
  }

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
  for (int r = gwarp; r < m; r += nwarps) {
    double s = 0.0;
    for (int t = a.rowptr[r] + lane; t < a.rowptr[r + 1]; t += 32)
      s = fma(a.vals[t], __ldcg(&a.x_out[a.colind[t]]), s);
    s = warp_sum(s);
    if (lane == 0) {
      const double rr = s - a.b[r];
      a.R[r] = rr;
      po += rr * rr;
    }
  }
  block_partial_sum(po, a.partials, 0, red);
  grid.sync();
  double mx = INFINITY, my = INFINITY, mc = 0.0, dot = 0.0;
  for (int j = gwarp; j < n; j += nwarps) {
    double s = 0.0;
    for (int t = a.colptr[j] + lane; t < a.colptr[j + 1]; t += 32)
      s = fma(a.cvals[t], __ldcg(&a.R[a.rowind[t]]), s);
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

cudaError_t launch_lsqr_final(const LsqrArgs& a, int sm_count, cudaStream_t s) {
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lsqr_final_kernel, kThreads, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorLaunchOutOfResources;
  int grid = sm_count;  // one CTA per SM
  LsqrArgs args = a;
  void* params[] = {&args};
  return cudaLaunchCooperativeKernel((void*)lsqr_final_kernel, dim3(grid), dim3(kThreads), params, 0, s);
}

}  // namespace nnls
