// batched.cu -- the whole block-principal-pivoting solve of one small problem
// per CTA, for batches of independent problems (BASELINE config 4: 65536
// problems of 128 x 64, 20% dense; "one warp-group per problem").
//
// Everything for a problem lives in shared memory: CSR rows, a column view
// (per-column row bitmasks + values in row order), the packed Gram, the
// packed bordered factor and all vectors.  Steps, following PAPER.md:
//   a1 Gram  G_ij = sum over rows set in mask_i & mask_j, increasing
//                    row order, separate multiply/add -> same terms, same
//                    order, same roundings as the CPU oracle (bit-identical).
//   a2 init, a3 decide/exchange, a4 compaction (ballot)
//   a5/a6 Cholesky of the bordered [G_FF; c_F^T] (right-looking, updates
//                    applied in increasing k with separate mul/sub -> the same
//                    rounding sequence as the oracle's jki loop) and the back
//                    substitution L^T x = z (sequential, oracle order)
//   a7/a8 dual y_G = G_GF x_F - c_G (sequential over F, oracle order), zeroing
//   a10 LSQR on the final F, block reductions for the norms
//   a11 report (objective, KKT of Eq. 3)
// Problems are independent: CTAs grid-stride over the batch; no inter-CTA
// communication.
#include <cuda_runtime.h>
#include <math.h>

#include "common.cuh"
#include "kernels.cuh"

namespace nnls {

namespace {
constexpr int BT = 128;  // one warp-group per problem

__device__ __forceinline__ int pk(int i, int j) {  // packed lower index, any order
  return i >= j ? i * (i + 1) / 2 + j : j * (j + 1) / 2 + i;
}

struct Lay {
  int oG, oL, ocv, orv, ob, ou, oc, ox, oy, oxF, ov, ow, oX, ored;  // double offsets
  int doubles;
  int irp, ici, icm, ico, iF, iG, imk;  // int offsets (after doubles)
  int ints;
  size_t bytes;
};

__host__ __device__ inline Lay layout(int m, int n, int nnz_max) {
  Lay L;
  int o = 0;
  L.oG = o; o += n * (n + 1) / 2;
  L.oL = o; o += (n + 1) * (n + 2) / 2;
  L.ocv = o; o += nnz_max;
  L.orv = o; o += nnz_max;
  L.ob = o; o += m;
  L.ou = o; o += m;
  L.oc = o; o += n;
  L.ox = o; o += n;
  L.oy = o; o += n;
  L.oxF = o; o += n;
  L.ov = o; o += n;
  L.ow = o; o += n;
  L.oX = o; o += n;
  L.ored = o; o += 64;
  L.doubles = o;
  const int W = (m + 31) / 32;
  int q = 0;
  L.irp = q; q += m + 1;
  L.ici = q; q += nnz_max;
  L.icm = q; q += n * W;
  L.ico = q; q += n + 1;
  L.iF = q; q += n;
  L.iG = q; q += n;
  L.imk = q; q += (n + 3) / 4;
  L.ints = q + 8;
  L.bytes = sizeof(double) * (size_t)L.doubles + sizeof(int) * (size_t)L.ints;
  return L;
}

__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  return (red[0] + red[1]) + (red[2] + red[3]);
}
__device__ double block_min(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_min(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  return fmin(fmin(red[0], red[1]), fmin(red[2], red[3]));
}
__device__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  return fmax(fmax(red[0], red[1]), fmax(red[2], red[3]));
}
}  // namespace

__global__ void __launch_bounds__(BT) batched_kernel(BatchArgs a, int nnz_max) {
  extern __shared__ double sm[];
  const int m = a.m, n = a.n, W = (m + 31) / 32;
  const Lay Ly = layout(m, n, nnz_max);
  double* G = sm + Ly.oG;
  double* L = sm + Ly.oL;
  double* cv = sm + Ly.ocv;
  double* rv = sm + Ly.orv;
  double* bb = sm + Ly.ob;
  double* u = sm + Ly.ou;
  double* c = sm + Ly.oc;
  double* x = sm + Ly.ox;
  double* y = sm + Ly.oy;
  double* xF = sm + Ly.oxF;
  double* v = sm + Ly.ov;
  double* w = sm + Ly.ow;
  double* X = sm + Ly.oX;
  double* red = sm + Ly.ored;
  int* ib = reinterpret_cast<int*>(sm + Ly.doubles);
  int* rp = ib + Ly.irp;
  int* ci = ib + Ly.ici;
  unsigned* cm = reinterpret_cast<unsigned*>(ib + Ly.icm);
  int* co = ib + Ly.ico;
  int* Fidx = ib + Ly.iF;
  int* Gidx = ib + Ly.iG;
  uint8_t* mk = reinterpret_cast<uint8_t*>(ib + Ly.imk);
  __shared__ int s_last, s_f;
  __shared__ unsigned s_bF[2], s_bG[2];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double tol = a.tol;

  for (int prob = blockIdx.x; prob < a.batch; prob += gridDim.x) {
    // ---------------------------------------------------------- load
    const int64_t e0 = a.nnz_off[prob];
    const int nz = (int)(a.nnz_off[prob + 1] - e0);
    for (int r = tid; r <= m; r += BT) rp[r] = a.rowptr[(size_t)prob * (m + 1) + r];
    for (int e = tid; e < nz; e += BT) {
      ci[e] = a.colind[e0 + e];
      rv[e] = a.vals[e0 + e];
    }
    for (int r = tid; r < m; r += BT) bb[r] = a.b[(size_t)prob * m + r];
    for (int q = tid; q < n * W; q += BT) cm[q] = 0u;
    __syncthreads();
    // column view: row bitmasks, counts, values in row order
    for (int r = tid; r < m; r += BT)
      for (int e = rp[r]; e < rp[r + 1]; ++e) atomicOr(&cm[ci[e] * W + (r >> 5)], 1u << (r & 31));
    __syncthreads();
    if (tid == 0) {
      int acc = 0;
      for (int j = 0; j < n; ++j) {
        co[j] = acc;
        for (int q = 0; q < W; ++q) acc += __popc(cm[j * W + q]);
      }
      co[n] = acc;
    }
    __syncthreads();
    for (int r = tid; r < m; r += BT) {
      const int wr = r >> 5;
      const unsigned below = (1u << (r & 31)) - 1u;
      for (int e = rp[r]; e < rp[r + 1]; ++e) {
        const int j = ci[e];
        int rank = co[j];
        for (int q = 0; q < wr; ++q) rank += __popc(cm[j * W + q]);
        rank += __popc(cm[j * W + wr] & below);
        cv[rank] = rv[e];
      }
    }
    __syncthreads();
    // ---------------------------------------------------------- a1 Gram, c
    const int npair = n * (n + 1) / 2;
    for (int q = tid; q < npair; q += BT) {
      int i = (int)((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
      while (i * (i + 1) / 2 > q) --i;
      while ((i + 1) * (i + 2) / 2 <= q) ++i;
      const int j = q - i * (i + 1) / 2;
      double s = 0.0;
      int ki = co[i], kj = co[j];
      for (int wq = 0; wq < W; ++wq) {
        const unsigned mi = cm[i * W + wq], mj = cm[j * W + wq];
        unsigned both = mi & mj;
        while (both) {
          const int bpos = __ffs(both) - 1;
          const unsigned below = (1u << bpos) - 1u;
          const double vi = cv[ki + __popc(mi & below)];
          const double vj = cv[kj + __popc(mj & below)];
          s = __dadd_rn(s, __dmul_rn(vi, vj));
          both &= both - 1u;
        }
        ki += __popc(mi);
        kj += __popc(mj);
      }
      G[q] = s;
    }
    for (int j = tid; j < n; j += BT) {
      double s = 0.0;
      int k = co[j];
      for (int wq = 0; wq < W; ++wq) {
        unsigned bits = cm[j * W + wq];
        while (bits) {
          const int r = wq * 32 + __ffs(bits) - 1;
          s = __dadd_rn(s, __dmul_rn(cv[k++], bb[r]));
          bits &= bits - 1u;
        }
      }
      c[j] = s;
    }
    __syncthreads();
    // ---------------------------------------------------------- a2 init
    for (int j = tid; j < n; j += BT) {
      mk[j] = 0;
      x[j] = 0.0;
      const double vv = -c[j];
      y[j] = fabs(vv) < tol ? 0.0 : vv;
    }
    int N = n + 1, p = a.p_max, iter = 0, singles = 0, status = 0, f = 0, not_pd = -1;
    __syncthreads();
    // ---------------------------------------------------------- pivot loop
    for (;;) {
      // a3 count + decide (every thread reaches the same decision)
      bool inf = false;
      if (tid < n) inf = mk[tid] ? (x[tid] < 0.0) : (y[tid] < 0.0);
      if (tid == 0) s_last = -1;
      __syncthreads();
      if (inf) atomicMax(&s_last, tid);
      const int k = __syncthreads_count(inf);
      const int last = s_last;
      if (k == 0) break;
      if (iter >= a.max_iter) {
        status = 8;
        break;
      }
      int branch;
      if (k < N) {
        N = k;
        p = a.p_max;
        branch = 0;
      } else if (p > 0) {
        p -= 1;
        branch = 1;
      } else {
        singles += 1;
        branch = 2;
      }
      if (tid < n && ((branch == 2) ? (tid == last) : inf)) mk[tid] ^= 1;
      __syncthreads();
      // a4 compaction (n <= 64: two warps)
      const bool inF = (tid < n) && mk[tid];
      const bool inG = (tid < n) && !mk[tid];
      const unsigned bF = __ballot_sync(kFull, inF);
      const unsigned bG = __ballot_sync(kFull, inG);
      if (lane == 0 && wid < 2) {
        s_bF[wid] = bF;
        s_bG[wid] = bG;
      }
      __syncthreads();
      if (wid < 2) {
        const unsigned lt = (1u << lane) - 1u;
        const int offF = wid == 1 ? __popc(s_bF[0]) : 0;
        const int offG = wid == 1 ? __popc(s_bG[0]) : 0;
        if (inF) Fidx[offF + __popc(bF & lt)] = tid;
        if (inG) Gidx[offG + __popc(bG & lt)] = tid;
      }
      if (tid == 0) s_f = __popc(s_bF[0]) + __popc(s_bF[1]);
      __syncthreads();
      f = s_f;
      // a5 Cholesky of the bordered (f+1) x (f+1) matrix, packed lower
      const int fa = f + 1;
      for (int q = tid; q < fa * (fa + 1) / 2; q += BT) {
        int i = (int)((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
        while (i * (i + 1) / 2 > q) --i;
        while ((i + 1) * (i + 2) / 2 <= q) ++i;
        const int j = q - i * (i + 1) / 2;
        double val = 0.0;
        if (j < f) val = (i < f) ? G[pk(Fidx[i], Fidx[j])] : c[Fidx[j]];
        L[q] = val;
      }
      __syncthreads();
      for (int kk = 0; kk < f; ++kk) {
        const double d = L[pk(kk, kk)];
        if (!(d > 0.0) || d < 1e-300 || !isfinite(d)) {
          if (status == 0) not_pd = kk;
          status = 7;
        }
        const double l = sqrt(d);
        __syncthreads();
        for (int i = kk + 1 + tid; i <= f; i += BT) L[pk(i, kk)] = L[pk(i, kk)] / l;
        if (tid == 0) L[pk(kk, kk)] = l;
        __syncthreads();
        // trailing update, rows i in (kk, f], cols jj in (kk, min(i, f-1)]
        const int nr = f - kk;  // rows kk+1..f
        const int tot = nr * (nr + 1) / 2;
        for (int q = tid; q < tot; q += BT) {
          int ii = (int)((sqrt(8.0 * q + 1.0) - 1.0) * 0.5);
          while (ii * (ii + 1) / 2 > q) --ii;
          while ((ii + 1) * (ii + 2) / 2 <= q) ++ii;
          const int jj = q - ii * (ii + 1) / 2;
          const int i = kk + 1 + ii, j = kk + 1 + jj;
          if (j < f) L[pk(i, j)] = __dsub_rn(L[pk(i, j)], __dmul_rn(L[pk(i, kk)], L[pk(j, kk)]));
        }
        __syncthreads();
      }
      if (status == 7) {
        for (int j = tid; j < n; j += BT) x[j] = 0.0;
        __syncthreads();
        break;
      }
      // a6 back substitution L^T x_F = z (z = row f), oracle order
      if (tid == 0) {
        for (int i = f - 1; i >= 0; --i) {
          double s = L[pk(f, i)];
          for (int kq = i + 1; kq < f; ++kq) s = __dsub_rn(s, __dmul_rn(L[pk(kq, i)], xF[kq]));
          xF[i] = s / L[pk(i, i)];
        }
      }
      __syncthreads();
      // scatter x_F, x_G = 0
      for (int aa = tid; aa < n; aa += BT) {
        if (aa < f) x[Fidx[aa]] = xF[aa];
        else x[Gidx[aa - f]] = 0.0;
      }
      __syncthreads();
      // a7 y_G = G_GF x_F - c_G (from the unclamped x_F), y_F = 0; a8 zeroing
      if (tid < n) {
        const int j = tid;
        if (mk[j]) {
          y[j] = 0.0;
        } else {
          double s = 0.0;
          for (int aa = 0; aa < f; ++aa) s = __dadd_rn(s, __dmul_rn(G[pk(j, Fidx[aa])], xF[aa]));
          const double vv = s - c[j];
          y[j] = fabs(vv) < tol ? 0.0 : vv;
        }
      }
      __syncthreads();
      if (tid < n && mk[tid] && fabs(x[tid]) < tol) x[tid] = 0.0;
      __syncthreads();
      ++iter;
    }
    // ---------------------------------------------------------- a10 LSQR
    int itn = 0, istop = 0;
    const int mode = (status == 0 && f > 0) ? a.lsqr_mode : 0;
    if (mode != 0) {
      const int itn_limit = a.itn_limit > 0 ? a.itn_limit : 4 * f;
      for (int r = tid; r < m; r += BT) {
        double s = 0.0;
        if (mode == 2)
          for (int e = rp[r]; e < rp[r + 1]; ++e)
            if (mk[ci[e]]) s = fma(rv[e], x[ci[e]], s);
        u[r] = bb[r] - s;
      }
      double pu = 0.0;
      for (int r = tid; r < m; r += BT) pu += u[r] * u[r];
      double beta = sqrt(block_sum(pu, red));
      const double bnorm = beta;
      if (beta > 0.0)
        for (int r = tid; r < m; r += BT) u[r] /= beta;
      __syncthreads();
      double pv = 0.0;
      for (int j = tid; j < n; j += BT) {
        double s = 0.0;
        if (mk[j] && beta > 0.0) {
          int k = co[j];
          for (int wq = 0; wq < W; ++wq) {
            unsigned bits = cm[j * W + wq];
            while (bits) {
              const int r = wq * 32 + __ffs(bits) - 1;
              s = fma(cv[k++], u[r], s);
              bits &= bits - 1u;
            }
          }
        }
        v[j] = s;
        X[j] = 0.0;
        pv += s * s;
      }
      double alpha = sqrt(block_sum(pv, red));
      if (alpha > 0.0)
        for (int j = tid; j < n; j += BT) v[j] /= alpha;
      __syncthreads();
      for (int j = tid; j < n; j += BT) w[j] = v[j];
      __syncthreads();
      double rhobar = alpha, phibar = beta, anorm = 0.0, ddnorm = 0.0;
      const double ctol = a.conlim > 0.0 ? 1.0 / a.conlim : 0.0;
      if (alpha * beta != 0.0) {
        while (itn < itn_limit) {
          ++itn;
          pu = 0.0;
          for (int r = tid; r < m; r += BT) {
            double s = 0.0;
            for (int e = rp[r]; e < rp[r + 1]; ++e) s = fma(rv[e], v[ci[e]], s);  // v_G = 0
            const double uu = s - alpha * u[r];
            u[r] = uu;
            pu += uu * uu;
          }
          beta = sqrt(block_sum(pu, red));
          if (beta > 0.0) {
            for (int r = tid; r < m; r += BT) u[r] /= beta;
            anorm = sqrt(anorm * anorm + alpha * alpha + beta * beta);
            __syncthreads();
            pv = 0.0;
            for (int j = tid; j < n; j += BT) {
              if (!mk[j]) continue;
              double s = 0.0;
              int k = co[j];
              for (int wq = 0; wq < W; ++wq) {
                unsigned bits = cm[j * W + wq];
                while (bits) {
                  const int r = wq * 32 + __ffs(bits) - 1;
                  s = fma(cv[k++], u[r], s);
                  bits &= bits - 1u;
                }
              }
              const double vv = s - beta * v[j];
              v[j] = vv;
              pv += vv * vv;
            }
            alpha = sqrt(block_sum(pv, red));
            if (alpha > 0.0)
              for (int j = tid; j < n; j += BT)
                if (mk[j]) v[j] /= alpha;
          }
          const double rho = sqrt(rhobar * rhobar + beta * beta);
          const double cs = rhobar / rho, sn = beta / rho;
          const double theta = sn * alpha;
          rhobar = -cs * alpha;
          const double phi = cs * phibar;
          phibar = sn * phibar;
          const double t1 = phi / rho, t2 = -theta / rho;
          __syncthreads();
          double pd = 0.0, px = 0.0;
          for (int j = tid; j < n; j += BT) {
            if (!mk[j]) continue;
            const double ww = w[j];
            const double d = ww / rho;
            pd += d * d;
            const double xx = X[j] + t1 * ww;
            X[j] = xx;
            w[j] = v[j] + t2 * ww;
            px += xx * xx;
          }
          ddnorm += block_sum(pd, red);
          const double xnorm = sqrt(block_sum(px, red));
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
          __syncthreads();
          if (istop != 0) break;
        }
      }
    }
    // ---------------------------------------------------------- a11 output
    bool infeas = false;
    for (int j = tid; j < n; j += BT) {
      double vv;
      if (!mk[j]) vv = 0.0;
      else if (mode == 1) vv = X[j];
      else if (mode == 2) vv = x[j] + X[j];
      else vv = x[j];
      if (fabs(vv) < tol) vv = 0.0;
      if (vv < 0.0) infeas = true;
      w[j] = vv;  // final x staged in w
      a.x_out[(size_t)prob * n + j] = vv;
      if (a.mask_out) a.mask_out[(size_t)prob * n + j] = mk[j];
    }
    const int any_infeas = __syncthreads_or(infeas);
    double obj = 0.0, mx = INFINITY, my = INFINITY, mc = 0.0, dot = 0.0;
    if (a.kkt) {
      double po = 0.0;
      for (int r = tid; r < m; r += BT) {
        double s = 0.0;
        for (int e = rp[r]; e < rp[r + 1]; ++e) s = fma(rv[e], w[ci[e]], s);
        const double rr = s - bb[r];
        u[r] = rr;
        po += rr * rr;
      }
      obj = block_sum(po, red);
      double lmx = INFINITY, lmy = INFINITY, lmc = 0.0, ld = 0.0;
      for (int j = tid; j < n; j += BT) {
        double s = 0.0;
        int k = co[j];
        for (int wq = 0; wq < W; ++wq) {
          unsigned bits = cm[j * W + wq];
          while (bits) {
            const int r = wq * 32 + __ffs(bits) - 1;
            s = fma(cv[k++], u[r], s);
            bits &= bits - 1u;
          }
        }
        const double xj = w[j];
        lmx = fmin(lmx, xj);
        lmy = fmin(lmy, s);
        lmc = fmax(lmc, fabs(xj * s));
        ld += xj * s;
      }
      mx = block_min(lmx, red);
      my = block_min(lmy, red);
      mc = block_max(lmc, red);
      dot = block_sum(ld, red);
    }
    if (tid == 0) {
      int32_t* ii = a.info_i + (size_t)prob * 8;
      ii[0] = status;
      ii[1] = iter;
      ii[2] = singles;
      ii[3] = f;
      ii[4] = itn;
      ii[5] = istop;
      ii[6] = (mode != 0 && any_infeas) ? 1 : 0;
      ii[7] = status == 7 ? not_pd : -1;
      double* dd = a.info_d + (size_t)prob * 5;
      dd[0] = 0.5 * obj;
      dd[1] = mx;
      dd[2] = my;
      dd[3] = mc;
      dd[4] = dot;
    }
    __syncthreads();
  }
}

__global__ void validate_batched_kernel(int batch, int m, int n, const int64_t* __restrict__ nnz_off,
                                        const int32_t* __restrict__ rowptr,
                                        const int32_t* __restrict__ colind,
                                        const double* __restrict__ vals,
                                        const double* __restrict__ b, int* err) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int e_local = 0;
  for (int64_t gr = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; gr < (int64_t)batch * m;
       gr += warps) {
    const int prob = (int)(gr / m), r = (int)(gr % m);
    const int64_t base = nnz_off[prob];
    const int64_t nz = nnz_off[prob + 1] - base;
    const int64_t lo = rowptr[(size_t)prob * (m + 1) + r], hi = rowptr[(size_t)prob * (m + 1) + r + 1];
    if (lane == 0) {
      if (r == 0 && lo != 0) e_local |= 1;
      if (r == m - 1 && hi != nz) e_local |= 1;
      if (!isfinite(b[gr])) e_local |= 4;
    }
    if (hi < lo || lo < 0 || hi > nz) {
      e_local |= 1;
      continue;
    }
    for (int64_t t = lo + lane; t < hi; t += 32) {
      const int cidx = colind[base + t];
      if (cidx < 0 || cidx >= n) e_local |= 2;
      if (t > lo && colind[base + t - 1] >= cidx) e_local |= 2;
      if (!isfinite(vals[base + t])) e_local |= 4;
    }
  }
  if (e_local) atomicOr(err, e_local);
}

cudaError_t launch_validate_batched(int batch, int m, int n, const int64_t* nnz_off,
                                    const int32_t* rowptr, const int32_t* colind,
                                    const double* vals, const double* b, int* err, cudaStream_t s) {
  int64_t warps = (int64_t)batch * m;
  int blocks = (int)((warps * 32 + 255) / 256);
  if (blocks > 8192) blocks = 8192;
  if (blocks < 1) blocks = 1;
  validate_batched_kernel<<<blocks, 256, 0, s>>>(batch, m, n, nnz_off, rowptr, colind, vals, b, err);
  return cudaGetLastError();
}

size_t batched_smem_bytes(int m, int n, int nnz_max) { return layout(m, n, nnz_max).bytes; }

cudaError_t launch_batched_nnz(const BatchArgs& a, int nnz_max, int sm_count, cudaStream_t s) {
  const size_t smem = layout(a.m, a.n, nnz_max).bytes;
  if (smem > 220 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(batched_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, batched_kernel, BT, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  int grid = sm_count * per_sm;
  if (grid > a.batch) grid = a.batch;
  if (grid < 1) grid = 1;
  batched_kernel<<<grid, BT, smem, s>>>(a, nnz_max);
  return cudaGetLastError();
}

}  // namespace nnls
