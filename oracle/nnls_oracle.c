/*
 * nnls_oracle.c -- plain, slow, obviously-correct CPU oracle for the tsnnls
 * block-principal-pivoting NNLS hot path (Cantarella & Piatek, arXiv
 * cs/0408029; "P:n" = /root/reference/PAPER.md line n).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  It
 * shares no code, header, table or helper with the CUDA path
 * (paper_cs_0408029_b200/csrc); neither includes the other.
 *
 * Conventions: FP64 throughout, sequential loops in increasing index order,
 * no BLAS, compiled with -O2 -ffp-contract=off (no FMA contraction) so each
 * expression rounds exactly as written.  Every function cites the passage it
 * follows; readings of ambiguous passages are DESIGN.md §"Readings" c1..c21.
 *
 * Pins (tests/test_oracle_*.py, -m "not gpu"):
 *   or_gram          -- hand examples, exact integer arithmetic, numpy dense A^T A
 *   or_cholesky      -- hand examples, reconstruction, numpy.linalg.cholesky
 *   or_chol_solve    -- hand example, residual, numpy.linalg.solve
 *   or_dual_gram     -- equals the Eq.5 form (or_dual_eq5) within eps bound
 *   or_clamp / or_exchange -- hand examples + all branches on hand states
 *   or_bpp_solve     -- brute force 2^n (n<=12), closed forms, scipy nnls, KKT
 *   or_lsqr          -- hand examples, scipy.sparse.linalg.lsqr, numpy lstsq
 *   or_brute_force   -- closed forms (identity, diagonal G)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---- status codes (values mirror the ABI's meaning, defined independently) */
enum {
  OR_OK = 0,
  OR_NOT_PD = 7,
  OR_ITERATION_LIMIT = 8,
  OR_OOM = 6
};

typedef struct {
  double zero_tol;      /* 1e-12                          */
  int32_t p_max;        /* 3                              */
  int32_t max_iter;     /* <=0 -> 10*n (reading c12)                  */
  int32_t lsqr_mode;    /* 0 none, 1 cold recompute, 2 warm   */
  double lsqr_atol, lsqr_btol, lsqr_conlim;
  int32_t lsqr_itn_limit; /* <=0 -> 4*|F|                             */
  int32_t notpd_fallback; /* 1: a failed Cholesky is replaced by an
                             LSQR solve on A_F for that iteration  */
  double adaptive_threshold; /* lsqr_mode 3: LSQR iff kappa*2^-52 > this
                                ("when a switch ... is necessary";
                                default 1e-8)                      */
} or_params;

typedef struct {
  int32_t status, iterations, single_exchanges, free_count;
  int32_t lsqr_iterations, lsqr_stop, infeasible_after_lsqr, pad;
  double objective, kkt_min_x, kkt_min_y, kkt_max_comp, kkt_dot;
  double kappa;                /* lsqr_mode 3: condition estimate of the final
                                  (A^T A)_FF (or_condest); else 0           */
  int32_t refined;             /* 1 if the final x came from LSQR           */
  int32_t lsqr_fallbacks;      /* NOT_PD iterations solved by LSQR instead  */
} or_info;

typedef struct {
  int32_t iter, k, branch, f; /* branch 0: k<N all; 1: p>0 all; 2: single */
  double below_tol;           /* largest |v| < tol over x_F u y_G (0 if none) */
  double above_tol;           /* smallest |v| >= tol over x_F u y_G (inf)     */
} or_trace_rec;

/* ------------------------------------------------------------------------ */
/* Gram matrix and A^T b.  P:126: "A^T A_ij is just the dot product of the
 * i-th and j-th columns of A" -- G_ij = sum_r a_ri a_rj.  We accumulate the
 * terms for every (i,j) in increasing row order r (the same order a dense
 * triple loop i,j,r would use; zero terms are skipped).  Output: full
 * symmetric n x n row-major G and c = A^T b (c_i = sum_r a_ri b_r).          */
void or_gram(int32_t m, int32_t n, const int32_t* rowptr, const int32_t* colind,
             const double* vals, const double* b, double* G, double* c) {
  memset(G, 0, sizeof(double) * (size_t)n * n);
  memset(c, 0, sizeof(double) * (size_t)n);
  for (int32_t r = 0; r < m; ++r) {
    for (int32_t e1 = rowptr[r]; e1 < rowptr[r + 1]; ++e1) {
      int32_t i = colind[e1];
      for (int32_t e2 = rowptr[r]; e2 < rowptr[r + 1]; ++e2) {
        int32_t j = colind[e2];
        G[(size_t)i * n + j] += vals[e1] * vals[e2];
      }
      c[i] += vals[e1] * b[r];
    }
  }
}

/* Principal submatrix (A^T A)_FF, "pass submatrices".               */
void or_gather(int32_t n, const double* G, int32_t f, const int32_t* Fidx, double* M) {
  for (int32_t a = 0; a < f; ++a)
    for (int32_t bb = 0; bb < f; ++bb)
      M[(size_t)a * f + bb] = G[(size_t)Fidx[a] * n + Fidx[bb]];
}

/* Unblocked column-by-column (jki) Cholesky M = L L^T.  L is the
 * full f x f row-major lower factor (upper part zeroed).  Returns 0, or
 * -(j+1) when pivot j is <= 0, < 1e-300 or not finite (NOT_PD; reading c13,
 * "may fail entirely when kappa^2 eps >= 1").                         */
int32_t or_cholesky(int32_t f, const double* M, double* L) {
  memset(L, 0, sizeof(double) * (size_t)f * f);
  for (int32_t j = 0; j < f; ++j) {
    double d = M[(size_t)j * f + j];
    for (int32_t k = 0; k < j; ++k) d -= L[(size_t)j * f + k] * L[(size_t)j * f + k];
    if (!(d > 0.0) || d < 1e-300 || !isfinite(d)) return -(j + 1);
    double ljj = sqrt(d);
    L[(size_t)j * f + j] = ljj;
    for (int32_t i = j + 1; i < f; ++i) {
      double s = M[(size_t)i * f + j];
      for (int32_t k = 0; k < j; ++k) s -= L[(size_t)i * f + k] * L[(size_t)j * f + k];
      L[(size_t)i * f + j] = s / ljj;
    }
  }
  return 0;
}

/* Forward then back substitution: L z = rhs, L^T x = z.        */
void or_chol_solve(int32_t f, const double* L, const double* rhs, double* x) {
  double* z = (double*)malloc(sizeof(double) * (size_t)(f > 0 ? f : 1));
  for (int32_t i = 0; i < f; ++i) {
    double s = rhs[i];
    for (int32_t k = 0; k < i; ++k) s -= L[(size_t)i * f + k] * z[k];
    z[i] = s / L[(size_t)i * f + i];
  }
  for (int32_t i = f - 1; i >= 0; --i) {
    double s = z[i];
    for (int32_t k = i + 1; k < f; ++k) s -= L[(size_t)k * f + i] * x[k];
    x[i] = s / L[(size_t)i * f + i];
  }
  free(z);
}

/* Eq. 5 in Gram form (BASELINE.json north_star (4)):
 *   y_G = (A^T A)_GF x_F - (A^T b)_G, sequential sum over F in increasing
 * index order.  x is length n with x_G = 0; writes y_j for j in G, y_F = 0.  */
void or_dual_gram(int32_t n, const double* G, const double* c, const uint8_t* mask,
                  const double* x, double* y) {
  for (int32_t j = 0; j < n; ++j) {
    if (mask[j]) { y[j] = 0.0; continue; }
    double s = 0.0;
    for (int32_t i = 0; i < n; ++i)
      if (mask[i]) s += G[(size_t)j * n + i] * x[i];
    y[j] = s - c[j];
  }
}

/* Eq. 5 as printed: y_G = A_G^T (A_F x_F - b).  Used only to pin the
 * Gram form (reading c4).                                                   */
void or_dual_eq5(int32_t m, int32_t n, const int32_t* rowptr, const int32_t* colind,
                 const double* vals, const double* b, const uint8_t* mask,
                 const double* x, double* y) {
  double* r = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  for (int32_t i = 0; i < m; ++i) {
    double s = 0.0;
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e)
      if (mask[colind[e]]) s += vals[e] * x[colind[e]];
    r[i] = s - b[i];
  }
  for (int32_t j = 0; j < n; ++j) y[j] = 0.0;
  for (int32_t i = 0; i < m; ++i)
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e)
      if (!mask[colind[e]]) y[colind[e]] += vals[e] * r[i];
  free(r);
}

/* Zeroing of P:77 / P:103, reading c1: |v| < tol -> 0 (strict).           */
void or_clamp(int32_t len, double* v, double tol) {
  for (int32_t i = 0; i < len; ++i)
    if (fabs(v[i]) < tol) v[i] = 0.0;
}

/* Count + decide + exchange, P:89-101 (readings c5-c10).  State: mask (1 =
 * in F), x (x_F on F), y (y_G on G), *N, *p.  Returns the infeasible count k
 * (k = 0: feasible, nothing changed).  *branch: 0 "n < N", 1 "p > 0",
 * 2 single exchange of the largest original index.                           */
int32_t or_exchange(int32_t n, uint8_t* mask, const double* x, const double* y,
                    int32_t* N, int32_t* p, int32_t p_max, int32_t* branch) {
  uint8_t* infeas = (uint8_t*)malloc((size_t)(n > 0 ? n : 1));
  int32_t k = 0, last = -1;
  for (int32_t i = 0; i < n; ++i) {          /* snapshot before any flip (c10) */
    infeas[i] = mask[i] ? (x[i] < 0.0) : (y[i] < 0.0);
    if (infeas[i]) { ++k; last = i; }
  }
  if (k == 0) { free(infeas); *branch = -1; return 0; }
  if (k < *N) {
    *N = k; *p = p_max; *branch = 0;
    for (int32_t i = 0; i < n; ++i) if (infeas[i]) mask[i] = (uint8_t)!mask[i];
  } else if (*p > 0) {
    *p -= 1; *branch = 1;
    for (int32_t i = 0; i < n; ++i) if (infeas[i]) mask[i] = (uint8_t)!mask[i];
  } else {                                   /* P:98-99, reading c6 */
    *branch = 2;
    mask[last] = (uint8_t)!mask[last];
  }
  free(infeas);
  return k;
}

/* ------------------------------------------------------------------------ */
/* 1-norm condition estimate of M = L L^T (Section 3: "We can estimate
 * the relative error kappa^2 eps of each normal equations solution by
 * computing the condition number kappa^2 of A_F^T A_F with the LAPACK
 * function dpocon").  dpocon returns 1/(||M||_1 est(||M^-1||_1)) where est is
 * Hager's estimator with Higham's refinements (LAPACK dlacn2, at most 5
 * iterations, then the alternating-sign test vector); B = M^-1 is applied by
 * the forward and back substitutions of or_chol_solve (M is symmetric, so
 * B^T = B).  Written out step by step in dlacn2's order:
 *   1. x = (1/f, ..., 1/f); y = B x; est = ||y||_1 (f == 1: est = |y_1|, stop)
 *   2. xi = sign(y); z = B xi; j = argmax_i |z_i|; iter = 2
 *   3. x = e_j; y = B x; est_old = est; est = ||y||_1
 *      if sign(y) == xi or est <= est_old: go to 5
 *      xi = sign(y); z = B xi; jlast = j; j = argmax |z_i|
 *      if z_jlast != |z_j| and iter < 5: iter += 1, go to 3
 *   5. x_i = (-1)^(i) (1 + i/(f-1)), i = 0..f-1 (x_0 = +1); y = B x;
 *      est = max(est, 2 ||y||_1 / (3 f))
 * sign(0) = +1 (dlacn2).  Returns kappa = norm1_M * est (>= 1 for SPD M). */
static double asum(int32_t f, const double* v) {
  double s = 0.0;
  for (int32_t i = 0; i < f; ++i) s += fabs(v[i]);
  return s;
}
static int32_t iamax(int32_t f, const double* v) {
  int32_t j = 0;
  for (int32_t i = 1; i < f; ++i)
    if (fabs(v[i]) > fabs(v[j])) j = i;
  return j;
}
double or_condest(int32_t f, const double* L, double norm1_M) {
  if (f <= 0) return 0.0;
  double* x = (double*)malloc(sizeof(double) * (size_t)f);
  double* y = (double*)malloc(sizeof(double) * (size_t)f);
  double* xi = (double*)malloc(sizeof(double) * (size_t)f);
  double est;
  for (int32_t i = 0; i < f; ++i) x[i] = 1.0 / (double)f;
  or_chol_solve(f, L, x, y);                                     /* step 1 */
  if (f == 1) {
    est = fabs(y[0]);
  } else {
    est = asum(f, y);
    for (int32_t i = 0; i < f; ++i) xi[i] = y[i] >= 0.0 ? 1.0 : -1.0; /* step 2 */
    or_chol_solve(f, L, xi, y);
    int32_t j = iamax(f, y), iter = 2;
    for (;;) {                                                   /* step 3 */
      for (int32_t i = 0; i < f; ++i) x[i] = (i == j) ? 1.0 : 0.0;
      or_chol_solve(f, L, x, y);
      const double est_old = est;
      est = asum(f, y);
      int32_t same = 1;
      for (int32_t i = 0; i < f; ++i)
        if ((y[i] >= 0.0 ? 1.0 : -1.0) != xi[i]) { same = 0; break; }
      if (same || est <= est_old) break;   /* converged / cycling (dlacn2 keeps est) */
      for (int32_t i = 0; i < f; ++i) xi[i] = y[i] >= 0.0 ? 1.0 : -1.0;
      or_chol_solve(f, L, xi, y);
      const int32_t jlast = j;
      j = iamax(f, y);
      if (y[jlast] != fabs(y[j]) && iter < 5) { iter += 1; continue; }   /* (signed z_jlast, as dlacn2) */
      break;
    }
    double sgn = 1.0;                                            /* step 5 */
    for (int32_t i = 0; i < f; ++i) { x[i] = sgn * (1.0 + (double)i / (double)(f - 1)); sgn = -sgn; }
    or_chol_solve(f, L, x, y);
    const double temp = 2.0 * asum(f, y) / (3.0 * (double)f);
    if (temp > est) est = temp;
  }
  free(x); free(y); free(xi);
  return norm1_M * est;
}

/* ||M||_1 = max_j sum_i |M_ij| (M symmetric f x f, row-major).            */
double or_norm1(int32_t f, const double* M) {
  double mx = 0.0;
  for (int32_t j = 0; j < f; ++j) {
    double s = 0.0;
    for (int32_t i = 0; i < f; ++i) s += fabs(M[(size_t)i * f + j]);
    if (s > mx) mx = s;
  }
  return mx;
}

/* ------------------------------------------------------------------------ */
/* LSQR (Paige & Saunders; the solver P:124 embeds) on A_F = columns of A with
 * mask[j] = 1, rhs u0, starting from 0.  damp = 0.  Stopping rules (SPEC
 * S:228 / standard LSQR): test1 = ||r||/||b|| <= btol + atol*||A||*||x||/||b||,
 * test2 = ||A^T r||/(||A|| ||r||) <= atol, test3 = 1/cond(A) <= 1/conlim,
 * the machine-precision variants 1+t <= 1, or itn == itn_limit.  ||A|| and
 * cond(A) are the usual bidiagonalisation estimates; ||x|| is computed
 * exactly.  x has length n (zero outside F).  Returns istop (0..7).         */
static void csr_mask_matvec(int32_t m, const int32_t* rowptr, const int32_t* colind,
                            const double* vals, const uint8_t* mask, const double* v, double* out) {
  for (int32_t i = 0; i < m; ++i) {
    double s = 0.0;
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e)
      if (mask[colind[e]]) s += vals[e] * v[colind[e]];
    out[i] = s;
  }
}
static void csr_mask_rmatvec(int32_t m, int32_t n, const int32_t* rowptr, const int32_t* colind,
                             const double* vals, const uint8_t* mask, const double* u, double* out) {
  for (int32_t j = 0; j < n; ++j) out[j] = 0.0;
  for (int32_t i = 0; i < m; ++i)
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e)
      if (mask[colind[e]]) out[colind[e]] += vals[e] * u[i];
}
static double nrm2(int32_t len, const double* v) {
  double s = 0.0;
  for (int32_t i = 0; i < len; ++i) s += v[i] * v[i];
  return sqrt(s);
}

int32_t or_lsqr(int32_t m, int32_t n, const int32_t* rowptr, const int32_t* colind,
                const double* vals, const uint8_t* mask, const double* rhs,
                double atol, double btol, double conlim, int32_t itn_limit,
                double* x, int32_t* itn_out, double* rnorm_out, double* arnorm_out,
                double* rnorm_hist, int32_t hist_cap) {
  double* u = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  double* v = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double* w = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double* t = (double*)malloc(sizeof(double) * (size_t)((m > n ? m : n) + 1));
  for (int32_t j = 0; j < n; ++j) x[j] = 0.0;
  int32_t istop = 0, itn = 0;
  double ctol = conlim > 0 ? 1.0 / conlim : 0.0;
  for (int32_t i = 0; i < m; ++i) u[i] = rhs[i];
  double beta = nrm2(m, u), alpha = 0.0;
  double bnorm = beta;
  if (beta > 0) for (int32_t i = 0; i < m; ++i) u[i] /= beta;
  csr_mask_rmatvec(m, n, rowptr, colind, vals, mask, u, v);
  if (beta > 0) alpha = nrm2(n, v);
  if (alpha > 0) for (int32_t j = 0; j < n; ++j) v[j] /= alpha;
  for (int32_t j = 0; j < n; ++j) w[j] = v[j];
  double rhobar = alpha, phibar = beta, anorm = 0.0, ddnorm = 0.0, acond = 0.0;
  double rnorm = beta, arnorm = alpha * beta, xnorm = 0.0;
  if (arnorm == 0.0) {  /* x = 0 is the solution */
    *itn_out = 0; *rnorm_out = rnorm; *arnorm_out = arnorm;
    free(u); free(v); free(w); free(t);
    return 0;
  }
  while (itn < itn_limit) {
    itn += 1;
    /* beta u = A v - alpha u */
    csr_mask_matvec(m, rowptr, colind, vals, mask, v, t);
    for (int32_t i = 0; i < m; ++i) u[i] = t[i] - alpha * u[i];
    beta = nrm2(m, u);
    if (beta > 0) {
      for (int32_t i = 0; i < m; ++i) u[i] /= beta;
      anorm = sqrt(anorm * anorm + alpha * alpha + beta * beta);
      /* alpha v = A^T u - beta v */
      csr_mask_rmatvec(m, n, rowptr, colind, vals, mask, u, t);
      for (int32_t j = 0; j < n; ++j) v[j] = t[j] - beta * v[j];
      alpha = nrm2(n, v);
      if (alpha > 0) for (int32_t j = 0; j < n; ++j) v[j] /= alpha;
    }
    /* plane rotation eliminating beta */
    double rho = sqrt(rhobar * rhobar + beta * beta);
    double cs = rhobar / rho, sn = beta / rho;
    double theta = sn * alpha;
    rhobar = -cs * alpha;
    double phi = cs * phibar;
    phibar = sn * phibar;
    double t1 = phi / rho, t2 = -theta / rho;
    double dk2 = 0.0;
    for (int32_t j = 0; j < n; ++j) {
      double dj = w[j] / rho;
      dk2 += dj * dj;
      x[j] = x[j] + t1 * w[j];
      w[j] = v[j] + t2 * w[j];
    }
    ddnorm += dk2;
    xnorm = nrm2(n, x);
    acond = anorm * sqrt(ddnorm);
    rnorm = phibar;
    arnorm = alpha * fabs(sn * phi);   /* = phibar*alpha*|cs| */
    if (rnorm_hist && itn - 1 < hist_cap) rnorm_hist[itn - 1] = rnorm;
    double test1 = bnorm > 0 ? rnorm / bnorm : 0.0;
    double test2 = (anorm * rnorm) > 0 ? arnorm / (anorm * rnorm) : 0.0;
    double test3 = acond > 0 ? 1.0 / acond : 0.0;
    double tt1 = bnorm > 0 ? test1 / (1.0 + anorm * xnorm / bnorm) : 0.0;
    double rtol = btol + (bnorm > 0 ? atol * anorm * xnorm / bnorm : 0.0);
    if (itn >= itn_limit) istop = 7;
    if (1.0 + test3 <= 1.0) istop = 6;
    if (1.0 + test2 <= 1.0) istop = 5;
    if (1.0 + tt1 <= 1.0) istop = 4;
    if (test3 <= ctol) istop = 3;
    if (test2 <= atol) istop = 2;
    if (test1 <= rtol) istop = 1;
    if (istop != 0) break;
  }
  *itn_out = itn; *rnorm_out = rnorm; *arnorm_out = arnorm;
  free(u); free(v); free(w); free(t);
  return istop;
}

/* KKT of Eq. 3 with an independent dual y' = A^T (A x - b).          */
void or_kkt(int32_t m, int32_t n, const int32_t* rowptr, const int32_t* colind,
            const double* vals, const double* b, const double* x, or_info* info) {
  double* r = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
  double* yp = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  double obj = 0.0;
  for (int32_t i = 0; i < m; ++i) {
    double s = 0.0;
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) s += vals[e] * x[colind[e]];
    r[i] = s - b[i];
    obj += r[i] * r[i];
  }
  for (int32_t j = 0; j < n; ++j) yp[j] = 0.0;
  for (int32_t i = 0; i < m; ++i)
    for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e) yp[colind[e]] += vals[e] * r[i];
  double mx = INFINITY, my = INFINITY, mc = 0.0, dot = 0.0;
  for (int32_t j = 0; j < n; ++j) {
    if (x[j] < mx) mx = x[j];
    if (yp[j] < my) my = yp[j];
    if (fabs(x[j] * yp[j]) > mc) mc = fabs(x[j] * yp[j]);
    dot += x[j] * yp[j];
  }
  info->objective = 0.5 * obj;
  info->kkt_min_x = n ? mx : 0.0;
  info->kkt_min_y = n ? my : 0.0;
  info->kkt_max_comp = mc;
  info->kkt_dot = dot;
  free(r); free(yp);
}

/* ------------------------------------------------------------------------ */
/* The block principal pivoting algorithm, step for step.
 * Inputs: CSR A (m x n), b.  Outputs (caller-allocated, length n): x (final,
 * after the optional LSQR recompute), x_ne (the last normal-equations x, may
 * be NULL), mask (1 = F), y (algorithm's own y: y_G, y_F = 0; may be NULL).
 * trace: one record per iteration (may be NULL).                            */
static void trace_extremes(int32_t n, const uint8_t* mask, const double* x, const double* y,
                           double tol, double* below, double* above) {
  double lo = 0.0, hi = INFINITY;
  for (int32_t i = 0; i < n; ++i) {
    double v = fabs(mask[i] ? x[i] : y[i]);
    if (v < tol) { if (v > lo) lo = v; }
    else if (v < hi) hi = v;
  }
  *below = lo; *above = hi;
}

int32_t or_bpp_solve(int32_t m, int32_t n, const int32_t* rowptr, const int32_t* colind,
                     const double* vals, const double* b, const or_params* prm,
                     double* x_out, double* x_ne_out, uint8_t* mask_out, double* y_out,
                     or_info* info, or_trace_rec* trace, int32_t trace_cap) {
  memset(info, 0, sizeof(*info));
  const double tol = prm->zero_tol;
  const int32_t max_iter = prm->max_iter > 0 ? prm->max_iter : 10 * n;
  double* G = (double*)malloc(sizeof(double) * (size_t)n * n);
  double* c = (double*)malloc(sizeof(double) * (size_t)n);
  double* x = (double*)calloc((size_t)n, sizeof(double));
  double* y = (double*)calloc((size_t)n, sizeof(double));
  uint8_t* mask = (uint8_t*)calloc((size_t)n, 1);
  int32_t* Fidx = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  double* M = (double*)malloc(sizeof(double) * (size_t)n * n);
  double* L = (double*)malloc(sizeof(double) * (size_t)n * n);
  double* rhs = (double*)malloc(sizeof(double) * (size_t)n);
  double* xf = (double*)malloc(sizeof(double) * (size_t)n);
  double* xfb = (double*)malloc(sizeof(double) * (size_t)n);
  int32_t last_factored = 0;  /* the last update solved the normal equations (L, M hold its factor) */
  if (!G || !c || !x || !y || !mask || !Fidx || !M || !L || !rhs || !xf || !xfb) {
    info->status = OR_OOM;
    free(G); free(c); free(x); free(y); free(mask); free(Fidx); free(M); free(L); free(rhs); free(xf); free(xfb);
    return OR_OOM;
  }
  /* Gram caching: A^T A and A^T b formed once. */
  or_gram(m, n, rowptr, colind, vals, b, G, c);
  /* F = {}, G = {1..n}, x = 0, y = -A^T b, p = 3, N = inf (c8: n+1) */
  for (int32_t j = 0; j < n; ++j) { x[j] = 0.0; y[j] = -c[j]; }
  or_clamp(n, y, tol);                         /* reading c2 */
  int32_t N = n + 1, p = prm->p_max, iter = 0, singles = 0, status = OR_OK;
  for (;;) {
    /* k = number of negative entries of x_F and y_G */
    int32_t branch = -1;
    int32_t k = 0;
    for (int32_t i = 0; i < n; ++i) k += mask[i] ? (x[i] < 0.0) : (y[i] < 0.0);
    if (k == 0) break;
    if (iter >= max_iter) { status = OR_ITERATION_LIMIT; break; }      /* c12 */
    k = or_exchange(n, mask, x, y, &N, &p, prm->p_max, &branch);
    if (branch == 2) singles += 1;
    /* P:102 Update x_F by Eq. 4 through the normal equations */
    int32_t f = 0;
    for (int32_t i = 0; i < n; ++i) if (mask[i]) Fidx[f++] = i;
    for (int32_t j = 0; j < n; ++j) x[j] = 0.0;
    last_factored = 0;
    if (f > 0) {
      or_gather(n, G, f, Fidx, M);
      int32_t rc = or_cholesky(f, M, L);
      if (rc != 0 && !prm->notpd_fallback) { status = OR_NOT_PD; break; }   /* iterations = completed solves */
      if (rc != 0) {
        /* S:366 reading c13b: the normal equations failed ("may fail
         * entirely when kappa^2 eps >= 1"), so x_F for this iteration comes
         * from LSQR on A_F (cold start, the final step's tolerances) */
        int32_t itn_fb = 0, lim = prm->lsqr_itn_limit > 0 ? prm->lsqr_itn_limit : 4 * f;
        double rn_fb, arn_fb;
        or_lsqr(m, n, rowptr, colind, vals, mask, b, prm->lsqr_atol, prm->lsqr_btol, prm->lsqr_conlim, lim,
                xfb, &itn_fb, &rn_fb, &arn_fb, NULL, 0);
        for (int32_t a = 0; a < f; ++a) x[Fidx[a]] = xfb[Fidx[a]];
        info->lsqr_fallbacks += 1;
      } else {
        for (int32_t a = 0; a < f; ++a) rhs[a] = c[Fidx[a]];
        or_chol_solve(f, L, rhs, xf);
        for (int32_t a = 0; a < f; ++a) x[Fidx[a]] = xf[a];
        last_factored = 1;
      }
    }
    /* ... and y_G by Eq. 5 (Gram form), from the unclamped x_F (c3) */
    or_dual_gram(n, G, c, mask, x, y);
    /* zero entries within tol of zero (c1), both x_F and y_G.  The
     * trace records the values nearest tol on each side BEFORE zeroing. */
    double tr_lo = 0.0, tr_hi = INFINITY;
    trace_extremes(n, mask, x, y, tol, &tr_lo, &tr_hi);
    for (int32_t i = 0; i < n; ++i) {
      if (mask[i]) { if (fabs(x[i]) < tol) x[i] = 0.0; }
      else { if (fabs(y[i]) < tol) y[i] = 0.0; }
    }
    iter += 1;
    if (trace && iter - 1 < trace_cap) {
      or_trace_rec* t = &trace[iter - 1];
      t->iter = iter; t->k = k; t->branch = branch; t->f = f;
      t->below_tol = tr_lo; t->above_tol = tr_hi;
    }
  }
  int32_t fcount = 0;
  for (int32_t i = 0; i < n; ++i) fcount += mask[i];
  if (x_ne_out) for (int32_t j = 0; j < n; ++j) x_ne_out[j] = x[j];
  /* lsqr_mode 3 (reading c23): the condition estimate of the final
   * (A^T A)_FF decides whether the final LSQR is needed: predicted relative
   * error kappa * 2^-52 ("c kappa^2 eps") above the threshold.
   * A final F solved by the LSQR fallback has no factor: kappa = inf. */
  int32_t do_lsqr = prm->lsqr_mode == 1 || prm->lsqr_mode == 2;
  if (status == OR_OK && prm->lsqr_mode == 3 && fcount > 0) {
    info->kappa = last_factored ? or_condest(fcount, L, or_norm1(fcount, M)) : INFINITY;
    do_lsqr = info->kappa * ldexp(1.0, -52) > prm->adaptive_threshold;
  }
  /* recompute the final solution on the final F with LSQR (c15, c16) */
  if (status == OR_OK && do_lsqr && fcount > 0) {
    info->refined = 1;
    int32_t itn_lim = prm->lsqr_itn_limit > 0 ? prm->lsqr_itn_limit : 4 * fcount;
    double* rhs_m = (double*)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    double* dx = (double*)malloc(sizeof(double) * (size_t)n);
    double rn, arn;
    int32_t itn = 0, istop;
    if (prm->lsqr_mode != 2) {                 /* cold start: rhs = b (modes 1, 3) */
      for (int32_t i = 0; i < m; ++i) rhs_m[i] = b[i];
      istop = or_lsqr(m, n, rowptr, colind, vals, mask, rhs_m, prm->lsqr_atol, prm->lsqr_btol,
                      prm->lsqr_conlim, itn_lim, dx, &itn, &rn, &arn, NULL, 0);
      for (int32_t j = 0; j < n; ++j) x[j] = mask[j] ? dx[j] : 0.0;
    } else {                                   /* warm correction: rhs = b - A_F x_NE */
      for (int32_t i = 0; i < m; ++i) {
        double s = 0.0;
        for (int32_t e = rowptr[i]; e < rowptr[i + 1]; ++e)
          if (mask[colind[e]]) s += vals[e] * x[colind[e]];
        rhs_m[i] = b[i] - s;
      }
      istop = or_lsqr(m, n, rowptr, colind, vals, mask, rhs_m, prm->lsqr_atol, prm->lsqr_btol,
                      prm->lsqr_conlim, itn_lim, dx, &itn, &rn, &arn, NULL, 0);
      for (int32_t j = 0; j < n; ++j) x[j] = mask[j] ? x[j] + dx[j] : 0.0;
    }
    info->lsqr_iterations = itn;
    info->lsqr_stop = istop;
    int32_t bad = 0;
    for (int32_t j = 0; j < n; ++j) {
      if (mask[j] && fabs(x[j]) < tol) x[j] = 0.0;     /* c16: re-clamp */
      if (mask[j] && x[j] < 0.0) bad = 1;
    }
    info->infeasible_after_lsqr = bad;
    free(rhs_m); free(dx);
  }
  /* outputs; y recomputed for the report only (c16) */
  or_dual_gram(n, G, c, mask, x, y);
  for (int32_t j = 0; j < n; ++j) {
    x_out[j] = x[j];
    if (mask_out) mask_out[j] = mask[j];
    if (y_out) y_out[j] = y[j];
  }
  info->status = status;
  info->iterations = iter;
  info->single_exchanges = singles;
  info->free_count = fcount;
  or_kkt(m, n, rowptr, colind, vals, b, x, info);
  free(G); free(c); free(x); free(y); free(mask); free(Fidx); free(M); free(L); free(rhs); free(xf); free(xfb);
  return status;
}

/* Batched driver: `count` independent problems with per-problem CSR blocks
 * (rowptr local, nnz_off offsets).  Problems are independent, so they are
 * spread over `threads` OpenMP threads (threads <= 0: all cores).  Returns
 * the number of threads used.                                               */
int32_t or_bpp_solve_batched(int32_t count, int32_t m, int32_t n, const int64_t* nnz_off,
                             const int32_t* rowptr, const int32_t* colind, const double* vals,
                             const double* b, const or_params* prm, double* x_out,
                             uint8_t* mask_out, or_info* info, int32_t threads) {
  int32_t used = 1;
#ifdef _OPENMP
  if (threads <= 0) threads = omp_get_num_procs();
  omp_set_num_threads(threads);
#pragma omp parallel
  {
#pragma omp single
    used = omp_get_num_threads();
#pragma omp for schedule(dynamic, 16)
    for (int32_t q = 0; q < count; ++q) {
      or_bpp_solve(m, n, rowptr + (size_t)q * (m + 1), colind + nnz_off[q], vals + nnz_off[q],
                   b + (size_t)q * m, prm, x_out + (size_t)q * n, NULL,
                   mask_out ? mask_out + (size_t)q * n : NULL, NULL, info + q, NULL, 0);
    }
  }
#else
  (void)threads;
  for (int32_t q = 0; q < count; ++q)
    or_bpp_solve(m, n, rowptr + (size_t)q * (m + 1), colind + nnz_off[q], vals + nnz_off[q],
                 b + (size_t)q * m, prm, x_out + (size_t)q * n, NULL,
                 mask_out ? mask_out + (size_t)q * n : NULL, NULL, info + q, NULL, 0);
#endif
  return used;
}

/* Brute force over all 2^n complementary partitions (n <= 20): for each F,
 * dense normal equations on F (or_cholesky), y_G by Eq. 5 (Gram form), the
 * same clamp; F is feasible when x_F >= 0 and y_G >= 0.  Writes the masks of
 * all feasible F (as bit sets) into `feasible` (cap entries); returns count,
 * or -1 if n > 20.  SURVEY §8(c) step 8 / SPEC S:344-352.                    */
int32_t or_brute_force(int32_t m, int32_t n, const int32_t* rowptr, const int32_t* colind,
                       const double* vals, const double* b, double tol,
                       uint32_t* feasible, double* x_first, int32_t cap) {
  if (n > 20) return -1;
  double* G = (double*)malloc(sizeof(double) * (size_t)n * n);
  double* c = (double*)malloc(sizeof(double) * (size_t)n);
  double* x = (double*)malloc(sizeof(double) * (size_t)n);
  double* y = (double*)malloc(sizeof(double) * (size_t)n);
  uint8_t* mask = (uint8_t*)malloc((size_t)n + 1);
  int32_t* Fidx = (int32_t*)malloc(sizeof(int32_t) * (size_t)n + 4);
  double* M = (double*)malloc(sizeof(double) * (size_t)n * n + 8);
  double* L = (double*)malloc(sizeof(double) * (size_t)n * n + 8);
  double* rhs = (double*)malloc(sizeof(double) * (size_t)n + 8);
  double* xf = (double*)malloc(sizeof(double) * (size_t)n + 8);
  or_gram(m, n, rowptr, colind, vals, b, G, c);
  int32_t found = 0;
  for (uint32_t s = 0; s < (1u << n); ++s) {
    int32_t f = 0;
    for (int32_t i = 0; i < n; ++i) {
      mask[i] = (uint8_t)((s >> i) & 1u);
      x[i] = 0.0;
      if (mask[i]) Fidx[f++] = i;
    }
    if (f > 0) {
      or_gather(n, G, f, Fidx, M);
      if (or_cholesky(f, M, L) != 0) continue;
      for (int32_t a = 0; a < f; ++a) rhs[a] = c[Fidx[a]];
      or_chol_solve(f, L, rhs, xf);
      for (int32_t a = 0; a < f; ++a) x[Fidx[a]] = xf[a];
    }
    or_dual_gram(n, G, c, mask, x, y);
    int32_t ok = 1;
    for (int32_t i = 0; i < n; ++i) {
      double v = mask[i] ? x[i] : y[i];
      if (fabs(v) < tol) v = 0.0;
      if (v < 0.0) { ok = 0; break; }
    }
    if (ok) {
      if (found < cap) {
        feasible[found] = s;
        if (found == 0 && x_first)
          for (int32_t i = 0; i < n; ++i) x_first[i] = (mask[i] && fabs(x[i]) >= tol) ? x[i] : 0.0;
      }
      ++found;
    }
  }
  free(G); free(c); free(x); free(y); free(mask); free(Fidx); free(M); free(L); free(rhs); free(xf);
  return found;
}
