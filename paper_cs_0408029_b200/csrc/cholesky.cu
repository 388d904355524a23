// cholesky.cu -- a5/a6: the normal-equations solve on the free set F
// ("solves A^T A x = A^T b using a Cholesky factorization
// of the symmetric matrix A^T A"), on the principal submatrix (A^T A)_FF of
// the cached Gram.
//
// B200 design
//   * Bordered system: the factorization runs on the (f+1) x (f+1) matrix
//     [[G_FF, .], [c_F^T, .]], whose last row of L is z^T = (L^-1 c_F)^T, so
//     the forward substitution L z = c_F comes out of the factorization and
//     only L^T x_F = z remains (one triangular solve instead of two).
//   * Gather fused into the factorization: each tile task reads
//     G[Fidx[r], Fidx[c]] directly -- (A^T A)_FF is never materialised.
//   * Tiled left-looking Cholesky, T = 64, as a dependency DAG executed by a
//     persistent kernel: tasks (i, j) are claimed in column-major order from
//     an atomic counter and wait on per-tile "ready" flags (release/acquire),
//     so there is no grid-wide barrier; a task only waits for the tiles it
//     reads.  Since tasks are claimed in topological order by running CTAs,
//     the DAG cannot deadlock.
//   * Every O(T^3) step runs on the FP64 tensor pipe, mma.sync.m8n8k4.f64
//     (SASS DMMA.8x8x4 -- the only FP64 tensor path on sm_100a, tcgen05 has no
//     f64 kind): the left-looking update C_ij -= L_ik L_jk^T, and the
//     triangular solve of the off-diagonal tiles, done as a product with the
//     explicit inverse of the diagonal tile, X = C_ij L_jj^-T.
//   * The diagonal tiles are factored by ONE CTA walking the diagonal (the
//     chain, see chol_factor_kernel): POTRF in 8-column register panels with
//     the previous column's last update folded in, TRTRI of the diagonal
//     block by doubling levels on DMMA, and the sub-diagonal tile as a
//     triangular product with that inverse; helpers compute every other tile.
//     Column-sequential work is confined to the chain's diagonal tile.
//     Pivot <= 0, < 1e-300 or non-finite -> NOT_PD (reading c13).
//   * Factor reuse: tile columns kept from the previous pivot iteration (same
//     order prefix, st->reuse_cols) are not recomputed; the rows below them
//     are (one product per column, task W(j)).
//   * L^T x = z by a second kernel: a chain CTA (x_J = a_J - N_J^T x_{J+1}
//     - P_J^T x_{J+2}) fed by helper tasks through mailboxes.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"

namespace nnls {

namespace {
constexpr int T = kTile;
constexpr int LDS = T + 4;  // smem row stride (doubles): conflict-free 8x4 fragment reads
constexpr int kThreads = 256;
constexpr int TS = T * LDS;  // a tile in global memory has the smem layout too (one bulk copy)
constexpr int kSmemDoubles = 6 * TS;

__host__ __device__ inline int tidx(int i, int j) { return i * (i + 1) / 2 + j; }
// Barrier of the CTA's 8 warps as named barrier 1 (barrier 2 is the 7-warp
// barrier of the chain's POTRF, see wsync).
__device__ __forceinline__ void csync() { asm volatile("bar.sync 1, 256;\n" ::: "memory"); }
// "empty" pattern of the back-substitution mailboxes (see backsolve_chain)
__device__ __forceinline__ unsigned long long box_empty(int epoch) {
  return 0x7FF4000000000000ull | (unsigned)epoch;
}
inline int tri_tiles(int n) {
  const int ntr = (n + 1 + T - 1) / T;
  return ntr * (ntr + 1) / 2;
}
}  // namespace

// Debug hook (not part of the ABI): per-task %globaltimer stamps of the
// factorization DAG, enabled by nnls_debug_chol_profile(ptr).
__device__ unsigned long long* g_chol_prof = nullptr;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PROF_STAMP(task, slot)                                                                  \
  do {                                                                                          \
    if (g_chol_prof != nullptr && threadIdx.x == 0) g_chol_prof[(task) * 8 + (slot)] = gtimer(); \
  } while (0)

// DAG flags: full[tri], part[tri], inv[ntr], back-solve x[ntr], a[ntr], N[ntr], half1[tri].
size_t chol_flag_count(int n) {
  const int ntr = (n + 1 + T - 1) / T;
  return 3 * (size_t)tri_tiles(n) + 4 * (size_t)ntr + 4;
}

// Lower tiles L(i,j), one inverse tile Linv_JJ and two back-solve tiles N_J,
// P_J per tile column (each T rows of stride LDS: the smem layout, so a tile
// moves as one bulk copy), then the back-solve mailboxes [parity][x | a]
// (T per tile column each).
size_t chol_tile_doubles(int n) {
  const int ntr = (n + 1 + T - 1) / T;
  return ((size_t)tri_tiles(n) + 3 * (size_t)ntr) * TS + 4 * (size_t)ntr * T;
}

// load a tile (global, T rows of stride LDS) into smem (same layout)
__device__ __forceinline__ void load_tile(double* __restrict__ dst, const double* __restrict__ src) {
  for (int e = threadIdx.x; e < T * T / 2; e += kThreads) {
    const int o = ((2 * e) / T) * LDS + (2 * e) % T;
    const double2 v = __ldcg(reinterpret_cast<const double2*>(src + o));  // other CTAs' data: bypass L1
    *reinterpret_cast<double2*>(dst + o) = v;
  }
}

__device__ __forceinline__ void store_tile(double* __restrict__ dst, const double* __restrict__ src) {
  for (int e = threadIdx.x; e < T * T / 2; e += kThreads) {
    const int o = ((2 * e) / T) * LDS + (2 * e) % T;
    *reinterpret_cast<double2*>(dst + o) = *reinterpret_cast<const double2*>(src + o);
  }
}

// asynchronous 16-byte copies global -> shared (cp.async.cg: L2 only)
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void tile_async(double* __restrict__ dst, const double* __restrict__ src) {
  for (int e = threadIdx.x; e < T * T / 2; e += kThreads) {
    const int o = ((2 * e) / T) * LDS + (2 * e) % T;
    cp_async16(dst + o, src + o);
  }
}

// acc (16 x 32 per warp) += sign * A B^T for 64 x 64 tiles in smem (B given
// by rows: C[m][n] += sum_k A[m][k] B[n][k]), on DMMA 8x8x4.
template <bool kNegate>
__device__ __forceinline__ void dmma_tile(double (&acc)[2][4][2], const double* __restrict__ A,
                                          const double* __restrict__ B, int lane, int rb0, int cb0) {
#pragma unroll 4
  for (int kk = 0; kk < T; kk += 4) {
    double av[2], bv[4];
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const double v = A[(rb0 + 8 * a + (lane >> 2)) * LDS + kk + (lane & 3)];
      av[a] = kNegate ? -v : v;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) bv[q] = B[(cb0 + 8 * q + (lane >> 2)) * LDS + kk + (lane & 3)];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int q = 0; q < 4; ++q) dmma8x8x4(acc[a][q][0], acc[a][q][1], av[a], bv[q]);
  }
}
// acc += A Bm for 64 x 64 smem tiles, Bm row-major by k (C[m][n] += sum_k
// A[m][k] Bm[k][n]: the B fragments are read transposed).
__device__ __forceinline__ void dmma_tile_nn(double (&acc)[2][4][2], const double* __restrict__ A,
                                             const double* __restrict__ Bm, int lane, int rb0, int cb0) {
#pragma unroll 4
  for (int kk = 0; kk < T; kk += 4) {
    double av[2], bv[4];
#pragma unroll
    for (int a = 0; a < 2; ++a) av[a] = A[(rb0 + 8 * a + (lane >> 2)) * LDS + kk + (lane & 3)];
#pragma unroll
    for (int q = 0; q < 4; ++q) bv[q] = Bm[(kk + (lane & 3)) * LDS + cb0 + 8 * q + (lane >> 2)];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int q = 0; q < 4; ++q) dmma8x8x4(acc[a][q][0], acc[a][q][1], av[a], bv[q]);
  }
}
// 32 x 64 products (a half tile): warp w owns rows rb0 = (w>>2)*16 .. +16,
// columns cb0 = (w&3)*16 .. +16 (2 x 2 blocks of 8x8); acc -= A B^T, K = 64.
__device__ __forceinline__ void dmma_half_sub(double (&acc)[2][2][2], const double* __restrict__ A,
                                              const double* __restrict__ B, int lane, int rb0, int cb0) {
#pragma unroll 4
  for (int kk = 0; kk < T; kk += 4) {
    double av[2], bv[2];
#pragma unroll
    for (int a = 0; a < 2; ++a) av[a] = -A[(rb0 + 8 * a + (lane >> 2)) * LDS + kk + (lane & 3)];
#pragma unroll
    for (int q = 0; q < 2; ++q) bv[q] = B[(cb0 + 8 * q + (lane >> 2)) * LDS + kk + (lane & 3)];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int q = 0; q < 2; ++q) dmma8x8x4(acc[a][q][0], acc[a][q][1], av[a], bv[q]);
  }
}
__device__ __forceinline__ void acc_half_ls(double (&acc)[2][2][2], double* S, int lane, int rb0, int cb0,
                                            bool store) {
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        double* p = S + (rb0 + 8 * a + (lane >> 2)) * LDS + cb0 + 8 * q + 2 * (lane & 3) + v;
        if (store) *p = acc[a][q][v];
        else acc[a][q][v] = *p;
      }
}
// rows [r0, r0+32) of a global tile <-> rows [0, 32) of a smem buffer
__device__ __forceinline__ void half_async(double* __restrict__ dst, const double* __restrict__ src, int r0) {
  for (int e = threadIdx.x; e < 32 * T / 2; e += kThreads) {
    const int o = ((2 * e) / T) * LDS + (2 * e) % T;
    cp_async16(dst + o, src + r0 * LDS + o);
  }
}
__device__ __forceinline__ void acc_load(double (&acc)[2][4][2], const double* S, int lane, int rb0,
                                         int cb0) {
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int v = 0; v < 2; ++v)
        acc[a][q][v] = S[(rb0 + 8 * a + (lane >> 2)) * LDS + cb0 + 8 * q + 2 * (lane & 3) + v];
}
__device__ __forceinline__ void acc_store(const double (&acc)[2][4][2], double* S, int lane, int rb0,
                                          int cb0) {
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int v = 0; v < 2; ++v)
        S[(rb0 + 8 * a + (lane >> 2)) * LDS + cb0 + 8 * q + 2 * (lane & 3) + v] = acc[a][q][v];
}

// Cholesky of the diagonal 64 x 64 tile S (smem; rows < rv, pivot columns
// < cv; a row >= cv is the bordered row c_F^T and is only eliminated), by
// panels of 8 columns: warp 0 factors the 8-wide panel in registers (lane l
// holds rows 8p+l and 8p+l+32; 8 shuffle-broadcast columns), then all 8
// warps apply the rank-8 trailing update with DMMA.  Column-sequential work
// per lane is 8 wide instead of 32/64 (the column chain is latency-bound).
// Writes L into S (lower; the strict upper part is cleared by the caller),
// 1/l_cc into rinv; returns the first bad pivot column or -1.
__device__ __forceinline__ void panel8_update_block(double* __restrict__ S, int c0, int r0, int k0,
                                                    int lane) {
  // S[r0..r0+8)[k0..k0+8) -= S[r0..][c0..c0+8) S[k0..][c0..c0+8)^T  (one DMMA block, K = 8)
  double* Cp = S + (r0 + (lane >> 2)) * LDS + k0 + 2 * (lane & 3);
  double c0v = Cp[0], c1v = Cp[1];
#pragma unroll
  for (int kk = 0; kk < 8; kk += 4) {
    const double av = -S[(r0 + (lane >> 2)) * LDS + c0 + kk + (lane & 3)];
    const double bv = S[(k0 + (lane >> 2)) * LDS + c0 + kk + (lane & 3)];
    dmma8x8x4(c0v, c1v, av, bv);
  }
  Cp[0] = c0v;
  Cp[1] = c1v;
}

// C(rows r0..r0+7, column blocks J in [j0, j1)) -= A(r0.., panel c0) B(8J.., panel c0)^T
// (rank-8 DMMA strip, j1 > j0).  Blocks go in groups of 4; inside a group
// the DMMAs are unconditional (a block index past j1 is clamped to j1 - 1
// and its result dropped) so the compiler emits no branch + warp-sync per
// block around the mma.sync.
__device__ __forceinline__ void strip8_gemm(double* __restrict__ C, const double* __restrict__ A,
                                           const double* __restrict__ B, int c0, int r0, int j0, int j1,
                                           int lane) {
  const int rr = r0 + (lane >> 2), kq = lane & 3, rq = lane >> 2;
  const double a0 = -A[rr * LDS + c0 + kq], a1 = -A[rr * LDS + c0 + 4 + kq];
#pragma unroll
  for (int h = 0; h < 8; h += 4) {
    if (j0 + h < j1) {
      double cv0[4], cv1[4];
      int Jq[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) Jq[q] = min(j0 + h + q, j1 - 1);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double* Cp = C + rr * LDS + 8 * Jq[q] + 2 * kq;
        cv0[q] = Cp[0];
        cv1[q] = Cp[1];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double b0 = B[(8 * Jq[q] + rq) * LDS + c0 + kq];
        const double b1 = B[(8 * Jq[q] + rq) * LDS + c0 + 4 + kq];
        dmma8x8x4(cv0[q], cv1[q], a0, b0);
        dmma8x8x4(cv0[q], cv1[q], a1, b1);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (j0 + h + q < j1) {
          double* Cp = C + rr * LDS + 8 * Jq[q] + 2 * kq;
          Cp[0] = cv0[q];
          Cp[1] = cv1[q];
        }
      }
    }
  }
}

// Warp 0's share of one potrf_r8 panel [c0, c0+8): see potrf_r8.  FULL: all
// 8 columns valid (no per-column bound checks, so the column chain is one
// straight-line block).  Returns the first bad pivot column or -1.
template <int NR, bool FULL>
__device__ __forceinline__ int panel_factor8(double* __restrict__ S, int c0, int r0, int rv, int cv,
                                             double* __restrict__ rinv, int lane, bool wr_rinv) {
  double D[8][8];
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c <= r; ++c) D[r][c] = S[(c0 + r) * LDS + c0 + c];
  double a[NR][8];
#pragma unroll
  for (int k = 0; k < NR; ++k) {
    const int R = r0 + lane + 32 * k;
#pragma unroll
    for (int c = 0; c < 8; ++c) a[k][c] = (R < rv) ? S[R * LDS + c0 + c] : 0.0;
  }
  int bad = -1;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    if (FULL || c0 + c < cv) {
      double d = D[c][c];
      const bool ok = (d >= 1e-300) && (d <= 1.7976931348623157e308);  // false for NaN
      bad = (!ok && bad < 0) ? c0 + c : bad;
      d = ok ? d : 1.0;  // keep the chain finite; the status reports the failure
      const double inv = rsqrt(d);
      if (lane == 0) rinv[c0 + c] = inv;
#pragma unroll
      for (int c2 = c + 1; c2 < 8; ++c2) D[c2][c] *= inv;
#pragma unroll
      for (int k = 0; k < NR; ++k) a[k][c] *= inv;
#pragma unroll
      for (int c2 = c + 1; c2 < 8; ++c2) {
        if (FULL || c0 + c2 < cv) {
#pragma unroll
          for (int c3 = c + 1; c3 <= c2; ++c3) D[c2][c3] = fma(-D[c2][c], D[c3][c], D[c2][c3]);
#pragma unroll
          for (int k = 0; k < NR; ++k) a[k][c2] = fma(-a[k][c], D[c2][c], a[k][c2]);
        }
      }
    } else {
#pragma unroll
      for (int k = 0; k < NR; ++k) a[k][c] = 0.0;
    }
  }
#pragma unroll
  for (int k = 0; k < NR; ++k) {
    const int R = r0 + lane + 32 * k;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if (R < rv && R - c0 >= c) S[R * LDS + c0 + c] = a[k][c];
  }
  return bad;
}

// Cholesky of the leading cv columns of an rv-row smem tile (rv <= 32*NR+c,
// NR = 2 covers 64 rows), in 8-column panels.  Per panel p:
//  (a) all warps apply panel p-1 to column block p (the lookahead block);
//  (b) warp 0 factors panel p: every lane factors the 8x8 diagonal block
//      REDUNDANTLY in registers (no shuffles on the rsqrt -> scale -> FMA
//      column chain) and carries the rows c0+lane+32k, k < NR, of the
//      panel (lanes 0..7, k = 0 are the diagonal-block rows themselves, with
//      the same arithmetic, so their stored values equal the redundant copy);
//  (c) meanwhile warps 1..7 apply panel p-1 to the column blocks > p.
// Returns the first non-positive pivot column or -1; 1/l_cc goes to rinv.
// Barrier of the first NW warps: NW = 8 -> csync (barrier 1); NW = 7 ->
// barrier 2 over warps 0..6 (the chain's POTRF, while warp 7 runs its
// prefetch / publish loop).
template <int NW>
__device__ __forceinline__ void wsync() {
  if (NW == 8) csync();
  else asm volatile("bar.sync 2, %0;\n" ::"n"(NW * 32) : "memory");
}

// S block (I,J) -= X(I rows) X(J rows)^T, K = 64 (the deferred last update
// of a diagonal tile, one 8x8 block); two blocks interleaved when J2 >= 0.
__device__ __forceinline__ void syrk_blocks(double* __restrict__ S, const double* __restrict__ X, int I, int J,
                                            int I2, int J2, int lane) {
  const int rq = lane >> 2, kq = lane & 3;
  double* C1 = S + (8 * I + rq) * LDS + 8 * J + 2 * kq;
  double* C2 = S + (8 * max(I2, 0) + rq) * LDS + 8 * max(J2, 0) + 2 * kq;
  const double* a1 = X + (8 * I + rq) * LDS + kq;
  const double* b1 = X + (8 * J + rq) * LDS + kq;
  const double* a2 = X + (8 * max(I2, 0) + rq) * LDS + kq;
  const double* b2 = X + (8 * max(J2, 0) + rq) * LDS + kq;
  // four independent accumulator pairs per block (k steps 4q mod 16): a
  // 4-deep DMMA dependency chain instead of 16 on the chain's POTRF
  double c[4][2], d[4][2];
  c[0][0] = C1[0];
  c[0][1] = C1[1];
  d[0][0] = C2[0];
  d[0][1] = C2[1];
#pragma unroll
  for (int q = 1; q < 4; ++q) c[q][0] = c[q][1] = d[q][0] = d[q][1] = 0.0;
#pragma unroll
  for (int kk = 0; kk < T; kk += 4) {
    const int q = (kk >> 2) & 3;
    dmma8x8x4(c[q][0], c[q][1], -a1[kk], b1[kk]);
    dmma8x8x4(d[q][0], d[q][1], -a2[kk], b2[kk]);  // (a dummy copy of block 1 when J2 < 0)
  }
  C1[0] = (c[0][0] + c[1][0]) + (c[2][0] + c[3][0]);
  C1[1] = (c[0][1] + c[1][1]) + (c[2][1] + c[3][1]);
  if (J2 >= 0) {
    C2[0] = (d[0][0] + d[1][0]) + (d[2][0] + d[3][0]);
    C2[1] = (d[0][1] + d[1][1]) + (d[2][1] + d[3][1]);
  }
}

template <int NR, int NW = 8, bool SPLIT = false>
__device__ __forceinline__ int potrf_r8(double* __restrict__ S, int rv, int cv,
                                        double* __restrict__ rinv, int* s_bad,
                                        const double* __restrict__ X = nullptr) {
  static_assert(NW == 7 || NW == 8, "potrf_r8 runs on 7 or 8 warps");
  static_assert(!SPLIT || NR == 1, "SPLIT: two panel warps with 32 rows each");
  // SPLIT: the panel rows are shared by warps 0 (rows c0..c0+31) and 1
  // (c0+32..c0+63), each also factoring the 8x8 block redundantly, which
  // halves the FP64 instructions on the column chain's warp; warps 2.. do (c).
  constexpr int NPW = SPLIT ? 2 : 1;  // panel warps
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) *s_bad = -1;
  const int np = (cv + 7) >> 3;
  const int nbr = (rv + 7) >> 3;
  // X != nullptr: the tile's last update S -= X X^T (X = the previous
  // column's sub-diagonal tile) is still pending; it is applied column block
  // by column block just ahead of the panel that needs it: block 0 here,
  // block p+1 by the strip warps during panel p.
  if (X != nullptr && w < nbr) {
    const int I2 = w + NW < nbr ? w + NW : -1;
    syrk_blocks(S, X, w, 0, I2 < 0 ? w : I2, I2 < 0 ? -1 : 0, lane);
  }
  wsync<NW>();
#pragma unroll 1
  for (int p = 0; p < np; ++p) {
    const int c0 = 8 * p;
    if (p > 0) {  // (a) the lookahead column block: at most 7 row blocks for p >= 1
      for (int I = p + w; I < nbr; I += NW) panel8_update_block(S, c0 - 8, 8 * I, c0, lane);
      wsync<NW>();
    }
    if (w < NPW) {
      const int r0 = c0 + 32 * w;
      const int bad = (c0 + 8 <= cv) ? panel_factor8<NR, true>(S, c0, r0, rv, cv, rinv, lane, w == 0)
                                     : panel_factor8<NR, false>(S, c0, r0, rv, cv, rinv, lane, w == 0);
      if (w == 0 && lane == 0 && bad >= 0 && *s_bad < 0) *s_bad = bad;
    } else {
      // (c) row strips I in [p+1, nbr) x column blocks [p+1, min(I, ncb-1)]
      // (panel p-1), then the pending last update of block (I, p+1)
      const int ncb = (cv + 7) >> 3;
      for (int I = p + 1 + (w - NPW); I < nbr; I += NW - NPW) {
        const int j1 = min(I + 1, ncb);
        if (p > 0 && p + 1 < j1) strip8_gemm(S, S, S, c0 - 8, 8 * I, p + 1, j1, lane);
        if (X != nullptr && p + 1 < ncb) syrk_blocks(S, X, I, p + 1, I, -1, lane);
      }
    }
    wsync<NW>();
  }
  return *s_bad;
}

// smem writes of this thread -> visible to the async proxy (bulk copies)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// One doubling level of trtri64: for each pair of b x b diagonal blocks
// (X11 at (o,o), X22 at (o+b,o+b), L21 at (o+b,o)), Linv21 = -X22 (L21 X11).
// Output 8x8 blocks are spread over the 8 warps (b = 8: 4 blocks, b = 16: 8,
// b = 32: 16 -> two per warp); Tm (scratch) holds L21 X11 transposed.
template <int B, int NW>
__device__ __forceinline__ void trtri_level(double* __restrict__ X, const double* __restrict__ L,
                                            double* __restrict__ Tm, int w, int lane) {
  constexpr int NB = B / 8;                         // 8x8 blocks per side
  constexpr int NT = (32 / B) * NB * NB;            // output blocks in the level
  constexpr int PER = (NT + NW - 1) / NW;           // blocks per warp (the last ones clamped)
  const int rq = lane >> 2, kq = lane & 3;
  if (w >= NT) {  // b = 8: warps 4.. idle in both steps
    wsync<NW>();
    wsync<NW>();
    return;
  }
  int o[PER], bi[PER], bj[PER], pr[PER];
  bool ok[PER];
#pragma unroll
  for (int s = 0; s < PER; ++s) {
    ok[s] = w + NW * s < NT;
    const int t = ok[s] ? w + NW * s : NT - 1;  // (a clamped duplicate: computed, not stored)
    pr[s] = t / (NB * NB);
    o[s] = 2 * B * pr[s];
    bi[s] = (t % (NB * NB)) / NB;
    bj[s] = t % NB;
  }
  double c0[PER], c1[PER];
#pragma unroll
  for (int s = 0; s < PER; ++s) c0[s] = c1[s] = 0.0;
#pragma unroll
  for (int kk = 0; kk < B; kk += 4) {  // Tm = L21 X11: A[m][k] = L21[m][k], B[n][k] = X11[k][n]
#pragma unroll
    for (int s = 0; s < PER; ++s) {
      const double av = L[(o[s] + B + 8 * bi[s] + rq) * LDS + o[s] + kk + kq];
      const double bv = X[(o[s] + kk + kq) * LDS + o[s] + 8 * bj[s] + rq];
      dmma8x8x4(c0[s], c1[s], av, bv);
    }
  }
#pragma unroll
  for (int s = 0; s < PER; ++s) {  // Tmt[pair*B + n][m]
    if (!ok[s]) continue;
    double* t = Tm + (B * pr[s] + 8 * bj[s] + 2 * kq) * LDS + 8 * bi[s] + rq;
    t[0] = c0[s];
    t[LDS] = c1[s];
  }
  wsync<NW>();
#pragma unroll
  for (int s = 0; s < PER; ++s) c0[s] = c1[s] = 0.0;
#pragma unroll
  for (int kk = 0; kk < B; kk += 4) {  // Linv21 = -X22 Tm: A = X22, B[n][k] = Tmt[n][k]
#pragma unroll
    for (int s = 0; s < PER; ++s) {
      const double av = -X[(o[s] + B + 8 * bi[s] + rq) * LDS + o[s] + B + kk + kq];
      const double bv = Tm[(B * pr[s] + 8 * bj[s] + rq) * LDS + kk + kq];
      dmma8x8x4(c0[s], c1[s], av, bv);
    }
  }
#pragma unroll
  for (int s = 0; s < PER; ++s) {
    if (!ok[s]) continue;
    double* x = X + (o[s] + B + 8 * bi[s] + rq) * LDS + o[s] + 8 * bj[s] + 2 * kq;
    x[0] = c0[s];
    x[1] = c1[s];
  }
  if (B == 32) fence_proxy_async_smem();  // X complete -> its bulk store
  wsync<NW>();
}

// X = L^-1 for the lower 64 x 64 smem tile L with cv pivots (rows / columns
// >= cv of X are zero), 1/l_cc in rinv (c < cv).  Blocked so that no step is
// a 64-long column chain: the 8x8 diagonal blocks are inverted by
// substitution (8 lanes = the block's columns, 28 dependent FMAs; warp w
// takes blocks w and w + NW), then three doubling levels b = 8, 16, 32 form
// Linv21 = -Linv22 L21 Linv11 on DMMA.  The strict upper blocks of X must be
// zero on entry (they are never written).  Runs on warps 0..NW-1 (NW = 7: the
// chain's warp 7 is still waiting for the helpers' partials meanwhile).
template <int NW>
__device__ __forceinline__ void trtri64(double* __restrict__ X, const double* __restrict__ L,
                                        const double* __restrict__ rinv, int cv, double* __restrict__ Tm,
                                        int pj) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int blk = w + NW * (lane >> 3);
  if (lane < 16 && blk < 8) {
    const int c0 = 8 * blk, col = lane & 7;
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double s = (i == col) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < i; ++k) s = fma(-L[(c0 + i) * LDS + c0 + k], x[k], s);
      x[i] = (c0 + i < cv) ? s * rinv[c0 + i] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) X[(c0 + i) * LDS + c0 + col] = x[i];
  }
  wsync<NW>();
  trtri_level<8, NW>(X, L, Tm, w, lane);
  trtri_level<16, NW>(X, L, Tm, w, lane);
  if (pj >= 0) PROF_STAMP(pj, 7);
  trtri_level<32, NW>(X, L, Tm, w, lane);
}

// acc (rows 8w..8w+7 of X, all 64 columns) = A Linv^T for 64 x 64 smem
// tiles, Linv lower triangular: column block q only needs k < 8q+8, which
// halves the DMMAs (72 per warp, 8 independent accumulators).
__device__ __forceinline__ void gemm_linvT(double (&acc)[8][2], const double* __restrict__ A,
                                           const double* __restrict__ Linv, int w, int lane) {
  const int rq = lane >> 2, kq = lane & 3;
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q][0] = acc[q][1] = 0.0;
#pragma unroll
  for (int kb = 0; kb < T / 4; ++kb) {
    const double av = A[(8 * w + rq) * LDS + 4 * kb + kq];
#pragma unroll
    for (int q = kb / 2; q < 8; ++q) dmma8x8x4(acc[q][0], acc[q][1], av, Linv[(8 * q + rq) * LDS + 4 * kb + kq]);
  }
}
__device__ __forceinline__ void store_rows8(const double (&acc)[8][2], double* __restrict__ X, int w, int lane) {
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    double* x = X + (8 * w + (lane >> 2)) * LDS + 8 * q + 2 * (lane & 3);
    x[0] = acc[q][0];
    x[1] = acc[q][1];
  }
}

// Bulk (async-proxy) store of a smem tile to its global copy (same layout):
// ONE cp.async.bulk of T*LDS doubles issued by one thread, completed later by
// bulk_store_release() of the same thread, so the chain never waits on it.
// The smem rows must have been made visible to the async proxy
// (fence_proxy_async_smem() by the writers, then a barrier).
__device__ __forceinline__ void bulk_store_tile(double* __restrict__ dst, const double* __restrict__ src) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(src);
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(sa),
               "n"(TS * 8)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
// wait for this thread's bulk stores, then release the flag(s)
__device__ __forceinline__ void bulk_store_release(int* flag, int epoch, int* flag2 = nullptr) {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
  st_release(flag, epoch);
  if (flag2 != nullptr) st_release(flag2, epoch);
}

// ---------------------------------------------------------------------------
// Factorization DAG with a diagonal CHAIN.  CTA 0 walks the diagonal:
//   for column j:  L_jj = chol(A_jj - L(j,j-1) L(j,j-1)^T)  (the previous
//                  column's last update folded into the POTRF panels);
//                  Linv_jj by blocked TRTRI;  L(j+1,j) = A(j+1,j) Linv_jj^T
// so the per-column critical path has no tile hand-off between CTAs; warp 7
// prefetches the helpers' partial tiles and raises the flags of the chain's
// bulk-stored tiles in its idle phases.  CTAs 1.. claim helper tasks from a
// queue ordered by column (see the queue comment below):
//   P(j+1,j+1): tile (j+1,j+1) with its updates k < j      -> "partial" flag
//   P(j+1,j)  : tile (j+1,j)   with its updates k < j      -> "partial" flag
//   T(i,j), i >= j+2: updates k < j, then A(i,j) Linv_jj^T -> "full" flag
// (plus W(j) / D(jq) after a kept prefix).  Every wait is on a task queued
// earlier or on the chain, and the chain only waits on queued tasks, so the
// DAG cannot deadlock.
namespace {
struct FlagSet {
  int* full;   // [tri]   L(i,j) final
  int* part;   // [tri]   partial tile (helper -> chain); rows 0-31 of a restart row-chain tile
  int* inv;    // [ntr]   Linv_jj
  int* half1;  // [tri]   rows 32-63 of a restart row-chain tile
};
// all threads' stores -> barrier -> one st.release (cumulative over what the
// barrier ordered before it) makes the tile visible with the flag
__device__ __forceinline__ void publish_flag(int* f, int epoch) {
  csync();
  if (threadIdx.x == 0) st_release(f, epoch);
}
}  // namespace

// gather tile (i,jj) of [G_FF; c_F^T] into S (lower part only on the diagonal)
__device__ __forceinline__ void gather_tile(double* __restrict__ S, const double* __restrict__ G,
                                            int ldg, const double* __restrict__ cvec,
                                            const int32_t* __restrict__ Fidx, int f, int i, int jj) {
  const int rv = min(T, f + 1 - i * T), cv = min(T, f - jj * T);
  for (int e = threadIdx.x; e < T * T; e += kThreads) {
    const int r = e / T, cc = e % T;
    const int gi = i * T + r, gj = jj * T + cc;
    double v = 0.0;
    if (r < rv && cc < cv && (i != jj || cc <= r))
      v = (gi < f) ? G[(size_t)Fidx[gi] * ldg + Fidx[gj]] : cvec[Fidx[gj]];
    S[r * LDS + cc] = v;
  }
}

// ---------------------------------------------------------------------------
// Helper operand pipeline (warp-specialized).  A helper CTA is 8 consumer
// warps (the DMMA updates, 256 threads as everywhere in this file) plus one
// PRODUCER warp: per left-looking update k of the task's tile (i, jj) it polls
// the release flags of L(i,k) and L(jj,k), then moves both tiles into a ring
// stage with ONE bulk copy each (cp.async.bulk, completion on the stage's
// "full" mbarrier); the consumers wait on that mbarrier, run the 64x64x64
// DMMA update with the accumulator in registers, and release the stage on
// its "empty" mbarrier.  No CTA-wide barrier per update; up to kStages
// updates' operands are in flight while one is computed.  Linv_jj (T tasks)
// is one more stage.
constexpr int kStages = 3;              // ring stages of two tile slots (6 tiles = the whole smem)
constexpr int kHelperThreads = kThreads + 32;
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void ring_mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void ring_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void ring_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void ring_wait(unsigned long long* b, unsigned parity) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_addr(b)), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void ring_load_tile(double* dst, const double* src, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_addr(dst)),
               "l"(src), "n"(TS * 8), "r"(smem_addr(b))
               : "memory");
}
// the 9-warp barrier of a helper CTA (task hand-off)
__device__ __forceinline__ void hsync() { asm volatile("bar.sync 3, %0;\n" ::"n"(kHelperThreads) : "memory"); }

struct HelperRing {
  unsigned long long full[kStages], empty[kStages];
};

// producer (lane 0 of warp 8): stage `cnt` of the running sequence <- L(i,k),
// L(jj,k) for k < kmax (flags waited only for rows >= jq: kept rows need
// none), then (linv_j >= 0) Linv_{linv_j} alone.  cnt advances by the stages used.
__device__ __forceinline__ void ring_produce(HelperRing& R, double* ring, const double* __restrict__ Lt,
                                             const double* __restrict__ Linv, const FlagSet& F, int epoch, int i,
                                             int jj, int kmax, int jq, int linv_j, unsigned& cnt) {
  for (int k = 0; k < kmax + (linv_j >= 0 ? 1 : 0); ++k, ++cnt) {
    const int sidx = (int)(cnt % kStages);
    const unsigned use = cnt / kStages;
    if (use > 0) ring_wait(&R.empty[sidx], (use - 1) & 1);
    double* slot = ring + (size_t)(2 * sidx) * TS;
    if (k < kmax) {
      if (i >= jq) wait_flag(&F.full[tidx(i, k)], epoch);
      if (jj >= jq) wait_flag(&F.full[tidx(jj, k)], epoch);
      asm volatile("fence.proxy.async.global;\n" ::: "memory");  // (acquired data -> async-proxy reads)
      ring_expect(&R.full[sidx], 2u * TS * 8);
      ring_load_tile(slot, Lt + (size_t)tidx(i, k) * TS, &R.full[sidx]);
      ring_load_tile(slot + TS, Lt + (size_t)tidx(jj, k) * TS, &R.full[sidx]);
    } else {
      if (linv_j >= jq) wait_flag(&F.inv[linv_j], epoch);
      asm volatile("fence.proxy.async.global;\n" ::: "memory");
      ring_expect(&R.full[sidx], 1u * TS * 8);
      ring_load_tile(slot, Linv + (size_t)linv_j * TS, &R.full[sidx]);
    }
  }
}

// [G_FF; c_F^T] tile (i, jj) gathered straight into this warp's accumulator
// fragment (rows rb0.., columns cb0.., as acc_load would read them from S)
__device__ __forceinline__ void gather_acc(double (&acc)[2][4][2], const double* __restrict__ G, int ldg,
                                           const double* __restrict__ cvec, const int32_t* __restrict__ Fidx,
                                           int f, int i, int jj, int lane, int rb0, int cb0) {
  const int rv = min(T, f + 1 - i * T), cv = min(T, f - jj * T);
  int gr[2], gc[8];
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int r = rb0 + 8 * a + (lane >> 2);
    gr[a] = (r < rv) ? ((i * T + r < f) ? Fidx[i * T + r] : -1) : -2;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int cc = cb0 + 8 * q + 2 * (lane & 3) + v;
      gc[2 * q + v] = (cc < cv) ? Fidx[jj * T + cc] : -1;
    }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int r = rb0 + 8 * a + (lane >> 2), cc = cb0 + 8 * q + 2 * (lane & 3) + v;
        const int gcv = gc[2 * q + v];
        double x = 0.0;
        if (gr[a] != -2 && gcv >= 0 && (i != jj || cc <= r))
          x = (gr[a] >= 0) ? G[(size_t)gr[a] * ldg + gcv] : cvec[gcv];
        acc[a][q][v] = x;
      }
}

// consumers: the kmax updates acc -= L(i,k) L(jj,k)^T from the ring
__device__ __forceinline__ void ring_consume_updates(HelperRing& R, const double* ring, double (&acc)[2][4][2],
                                                     int kmax, unsigned& cnt, int lane, int rb0, int cb0) {
  for (int k = 0; k < kmax; ++k, ++cnt) {
    const int sidx = (int)(cnt % kStages);
    ring_wait(&R.full[sidx], (cnt / kStages) & 1);
    const double* slot = ring + (size_t)(2 * sidx) * TS;
    dmma_tile<true>(acc, slot, slot + TS, lane, rb0, cb0);
    __syncwarp();
    if (lane == 0) ring_arrive(&R.empty[sidx]);
  }
}

// Split-K consumer layout of the piped helper tasks: warp w (0..7) owns the
// 32 x 32 quadrant (w & 3) of the tile and the k-half (w >> 2) of every
// update -- 16 independent 8x8 accumulators per warp and half the fragment
// loads per DMMA of the 16 x 32 layout; the two k-halves are summed once at
// the end of the task (q32_reduce).
__device__ __forceinline__ void q32_origin(int w, int& rb0, int& cb0, int& k0) {
  rb0 = ((w & 3) >> 1) * 32;
  cb0 = (w & 1) * 32;
  k0 = (w >> 2) * 32;
}
__device__ __forceinline__ void gather_acc32(double (&acc)[4][4][2], const double* __restrict__ G, int ldg,
                                             const double* __restrict__ cvec, const int32_t* __restrict__ Fidx,
                                             int f, int i, int jj, int lane, int rb0, int cb0) {
  const int rv = min(T, f + 1 - i * T), cv = min(T, f - jj * T);
  int gr[4], gc[8];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int r = rb0 + 8 * a + (lane >> 2);
    gr[a] = (r < rv) ? ((i * T + r < f) ? Fidx[i * T + r] : -1) : -2;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int cc = cb0 + 8 * q + 2 * (lane & 3) + v;
      gc[2 * q + v] = (cc < cv) ? Fidx[jj * T + cc] : -1;
    }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int r = rb0 + 8 * a + (lane >> 2), cc = cb0 + 8 * q + 2 * (lane & 3) + v;
        const int gcv = gc[2 * q + v];
        double x = 0.0;
        if (gr[a] != -2 && gcv >= 0 && (i != jj || cc <= r))
          x = (gr[a] >= 0) ? G[(size_t)gr[a] * ldg + gcv] : cvec[gcv];
        acc[a][q][v] = x;
      }
}
__device__ __forceinline__ void acc32_io(double (&acc)[4][4][2], double* S, int lane, int rb0, int cb0, int mode) {
  // mode 0: store, 1: load, 2: add
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        double* p = S + (rb0 + 8 * a + (lane >> 2)) * LDS + cb0 + 8 * q + 2 * (lane & 3) + v;
        if (mode == 0) *p = acc[a][q][v];
        else if (mode == 1) acc[a][q][v] = *p;
        else acc[a][q][v] += *p;
      }
}
// acc -= A B^T over k in [k0, k0+32) for the warp's 32 x 32 quadrant
__device__ __forceinline__ void dmma_q32_sub(double (&acc)[4][4][2], const double* __restrict__ A,
                                             const double* __restrict__ B, int lane, int rb0, int cb0, int k0) {
#pragma unroll 2
  for (int kk = k0; kk < k0 + 32; kk += 4) {
    double av[4], bv[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) av[a] = -A[(rb0 + 8 * a + (lane >> 2)) * LDS + kk + (lane & 3)];
#pragma unroll
    for (int q = 0; q < 4; ++q) bv[q] = B[(cb0 + 8 * q + (lane >> 2)) * LDS + kk + (lane & 3)];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int q = 0; q < 4; ++q) dmma8x8x4(acc[a][q][0], acc[a][q][1], av[a], bv[q]);
  }
}
__device__ __forceinline__ void ring_consume_updates32(HelperRing& R, const double* ring, double (&acc)[4][4][2],
                                                       int kmax, unsigned& cnt, int lane, int rb0, int cb0, int k0) {
  for (int k = 0; k < kmax; ++k, ++cnt) {
    const int sidx = (int)(cnt % kStages);
    ring_wait(&R.full[sidx], (cnt / kStages) & 1);
    const double* slot = ring + (size_t)(2 * sidx) * TS;
    dmma_q32_sub(acc, slot, slot + TS, lane, rb0, cb0, k0);
    __syncwarp();
    if (lane == 0) ring_arrive(&R.empty[sidx]);
  }
}

__global__ void __launch_bounds__(kHelperThreads, 1) chol_factor_kernel(
    const double* __restrict__ G, int ldg, const double* __restrict__ cvec,
    const int32_t* __restrict__ Fidx, double* __restrict__ Lt, double* __restrict__ Linv,
    int* __restrict__ flags, int tri, DevState* st, unsigned long long* __restrict__ box, int boxlen,
    int halves_mode) {
  extern __shared__ double smem[];
  pdl_wait();
  // helpers: BUF(0) = S, BUF(1..4) = operand double-buffers.
  // chain: BUF(0)/BUF(1) = diagonal tile of column j (alternating), BUF(5) = A/L(j+1,j)
  __shared__ double rinv[T];
  __shared__ int s_task, s_bad, s_role;
  const int f = st->f;
  const int epoch = st->epoch;
  if (f <= 0 || st->done || st->status != 0) return;  // (graph loop: nothing to solve)
  // Role by arrival, not by blockIdx: the first CTA that runs walks the
  // diagonal (helpers spin on its flags, so it must be a CTA that is already
  // resident -- a CTA with a fixed index might not be, under MPS or beside
  // other kernels); the second empties the back-substitution mailboxes.
  if (threadIdx.x == 0) s_role = atomicAdd(&st->role_factor, 1);
  __syncthreads();
  const int role = s_role;
  const int ntc = (f + T - 1) / T;      // tile columns to factor
  // tile columns [0, jq) of rows [0, jq) are kept from the previous pivot
  // iteration (same order prefix, see order_free_set in pivot.cu)
  const int jq = (st->reuse_cols > 0 && st->reuse_cols < ntc) ? st->reuse_cols : 0;
  // W_j tiles of a restart (task W(j)) live in the back-solve's N_J region,
  // which the back substitution only writes after the factorization
  double* Wbuf = Linv + (size_t)(boxlen / T) * TS;
  const int ntr = (f + 1 + T - 1) / T;  // tile rows (incl. the rhs row f)
  FlagSet F{flags, flags + tri, flags + 2 * tri, flags + 2 * tri + 4 * (boxlen / T)};
  const int tid = threadIdx.x;
  double* S = smem;
  if (role == 1 && tid < kThreads) {  // empty this epoch's back-substitution mailboxes (see box_empty)
    unsigned long long* xb = box + (size_t)(2 * (epoch & 1)) * boxlen;
    for (int e = tid; e < ntc * T; e += kThreads) {
      xb[e] = box_empty(epoch);
      xb[boxlen + e] = box_empty(epoch);
    }
  }

  if (role == 0) {
    if (tid >= kThreads) return;  // (the chain runs on 8 warps; its named barriers count 256 / 224 threads)
    PROF_STAMP(1198, 0);
    // ============================== the diagonal chain
    // BUF(0)/BUF(1): diagonal tile of column j (alternating), BUF(2): Linv_jj,
    // BUF(3): TRTRI scratch, BUF(4)/BUF(5): A/L(j+1,j) (alternating).
    // Per column: POTRF + TRTRI on warps 0-6 while warp 7 releases the
    // previous sub-diagonal tile and prefetches (cp.async) the helpers'
    // partials A(j+1,j) and A(j+1,j+1); then the product L(j+1,j) =
    // A(j+1,j) Linv_jj^T on all warps (warp 7 releases L_jj and Linv_jj).
    double* Xinv = smem + 2 * (T * LDS);  // Linv_jj
    double* Tm = smem + 3 * (T * LDS);    // trtri scratch
    int first_bad = -1;
    int* pending = nullptr;  // (tid 224) flag of the last stored sub tile, not yet released
    int* pending2 = nullptr; // (tid 224) the last L_jj's flag, not yet released
    for (int e = tid; e < T * T; e += kThreads)  // Linv's strict upper part, never written
      if ((e % T) > (e / T)) Xinv[(e / T) * LDS + (e % T)] = 0.0;
    for (int j = jq; j < ntc; ++j) {
      double* Sd = smem + (j & 1) * (T * LDS);
      double* Snext = smem + ((j + 1) & 1) * (T * LDS);
      // A/L(j+1,j) in BUF(4)/BUF(5) by column parity: L(j,j-1) stays put
      // while column j's POTRF applies it (the deferred SYRK)
      double* Lnext = smem + (4 + (j & 1)) * (T * LDS);
      const double* Lprev = (j > jq) ? smem + (4 + ((j - 1) & 1)) * (T * LDS) : nullptr;
      const int cv = min(T, f - j * T), rv = min(T, f + 1 - j * T);
      const bool has_sub = j + 1 < ntr, has_next = j + 1 < ntc;
      int* const fl_sub = &F.part[tidx(j + 1, j)];
      int* const fl_next = &F.part[tidx(j + 1, j + 1)];
      PROF_STAMP(j, 0);
      if (j == 0) {
        gather_tile(Sd, G, ldg, cvec, Fidx, f, 0, 0);
        csync();
      } else if (j == jq) {  // restart after a kept prefix: A_jj fully updated by a helper
        if (tid == 0) wait_flag(&F.part[tidx(j, j)], epoch);
        csync();
        load_tile(Sd, Lt + (size_t)tidx(j, j) * TS);
        csync();
      }
      // (j > 0: Sd holds A_jj fully updated at the end of the previous column)
      if ((tid >> 5) == 7) {
        // ---- warp 7: release the pending flag, then prefetch both partials
        const int lane = tid & 31;
        if (pending != nullptr && lane == 0) bulk_store_release(pending, epoch, pending2);
        pending = nullptr;
        pending2 = nullptr;
        int want = (has_sub ? 1 : 0) | (has_next ? 2 : 0);
        while (want) {
          int ok = 0;
          if (lane == 0) {
            if ((want & 1) && ld_acquire(fl_sub) == epoch) ok |= 1;
            if ((want & 2) && ld_acquire(fl_next) == epoch) ok |= 2;
          }
          ok = __shfl_sync(kFull, ok, 0);
          if (ok & 1) {
            const double* src = Lt + (size_t)tidx(j + 1, j) * TS;
            for (int e = lane; e < T * T / 2; e += 32) {
              const int o = ((2 * e) / T) * LDS + (2 * e) % T;
              cp_async16(Lnext + o, src + o);
            }
          }
          if (ok & 2) {
            const double* src = Lt + (size_t)tidx(j + 1, j + 1) * TS;
            for (int e = lane; e < T * T / 2; e += 32) {
              const int o = ((2 * e) / T) * LDS + (2 * e) % T;
              cp_async16(Snext + o, src + o);
            }
          }
          if (ok) cp_async_commit();
          want &= ~ok;
          if (want) __nanosleep(64);
        }
        cp_async_wait<0>();
      } else {
        // ---- warps 0..6: L_jj = chol(A_jj), then Linv_jj (while warp 7 may
        // still be waiting for the helpers' partials)
        const int bad = potrf_r8<1, 7, true>(Sd, rv, cv, rinv, &s_bad, Lprev);
        for (int e = tid; e < T * T; e += kThreads - 32)  // strict upper part
          if ((e % T) > (e / T)) Sd[(e / T) * LDS + (e % T)] = 0.0;
        if (bad >= 0 && first_bad < 0) first_bad = j * T + bad;
        wsync<7>();
        PROF_STAMP(j, 1);
        fence_proxy_async_smem();  // L_jj (Sd) -> the bulk store below
        // Linv_jj: the sub-diagonal TRSMs become products, and the back
        // substitution uses it (trtri64 fences Xinv for its bulk store)
        trtri64<7>(Xinv, Sd, rinv, cv, Tm, j);
        // Linv_jj out with plain stores (the helpers' T(i,j) tasks wait for it:
        // released right after the barrier below, no bulk-store drain on the path)
        for (int e = tid; e < T * T / 2; e += kThreads - 32) {
          const int o = ((2 * e) / T) * LDS + (2 * e) % T;
          *reinterpret_cast<double2*>(Linv + (size_t)j * TS + o) = *reinterpret_cast<const double2*>(Xinv + o);
        }
        PROF_STAMP(j, 3);
      }
      csync();  // L_jj, Linv_jj done (Linv_jj stored); partials in smem
      const int lane = tid & 31, w = tid >> 5;
      PROF_STAMP(j, 2);
      if (tid == kThreads - 32) {
        st_release(&F.inv[j], epoch);
        bulk_store_tile(Lt + (size_t)tidx(j, j) * TS, Sd);  // (released late: only the back substitution reads L_jj)
      }
      if (!has_sub) {  // last column without a sub-diagonal tile
        if (tid == kThreads - 32) bulk_store_release(&F.full[tidx(j, j)], epoch);
        break;
      }
      {  // L(j+1,j) = A(j+1,j) L_jj^-T = A(j+1,j) Linv_jj^T
        double acc[8][2];
        gemm_linvT(acc, Lnext, Xinv, w, lane);
        csync();
        store_rows8(acc, Lnext, w, lane);
      }
      PROF_STAMP(j, 4);
      fence_proxy_async_smem();  // L(j+1,j) (Lnext) -> the bulk store
      csync();
      if (tid == kThreads - 32) bulk_store_tile(Lt + (size_t)tidx(j + 1, j) * TS, Lnext);
      // (A(j+1,j+1) -= L(j+1,j) L(j+1,j)^T is applied inside the next POTRF)
      pending = &F.full[tidx(j + 1, j)];  // released by warp 7 in the next POTRF (or below)
      pending2 = &F.full[tidx(j, j)];     // (L_jj: its bulk store drains meanwhile)
      PROF_STAMP(j, 5);
    }
    if (pending != nullptr && tid == kThreads - 32) bulk_store_release(pending, epoch, pending2);  // last sub tile
    // NOT_PD is raised only after the whole chain ran: helpers read the status
    // at entry, and a helper that left early must not strand the chain
    if (tid == 0 && first_bad >= 0) {
      if (atomicCAS(&st->status, 0, 7) == 0) st->not_pd_col = first_bad;
    }
    return;
  }

  // ============================== helpers
  // queue: with a kept prefix (jq > 0) first the rows below it in the kept
  // columns, [T(jq..ntr-1, j) for j < jq], then D(jq) = tile (jq,jq) with
  // all its updates k < jq (the chain starts there); then per column j >= jq:
  // [P(j+1,j+1)?, P(j+1,j)?, T(j+2..ntr-1, j)]
  const int lane = tid & 31, w = tid >> 5;
  __shared__ HelperRing R;
  if (tid == 0) {
    for (int k = 0; k < kStages; ++k) {
      ring_mbar_init(&R.full[k], 1);
      ring_mbar_init(&R.empty[k], kThreads / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  unsigned rcnt = 0;  // ring stages used so far (identical sequence on both sides)
  for (;;) {
    // (this thread's generic smem accesses of the last task -> before the
    // bulk copies the producer issues into the same memory after the barrier)
    fence_proxy_async_smem();
    if (tid == 0) s_task = atomicAdd(&st->tile_counter, 1);
    hsync();
    int t = s_task;
    hsync();
    int j = jq, kind = -1, i = 0, half = 0;
    if (jq > 0) {
      // [W(1..jq-1)] [T(jq..ntr-1, 0)] [row-chain tasks for 0 < j < jq] [D(jq)]; the
      // row chain runs by half tiles (Th, kind 6) when all its tasks fit on the
      // helpers at once, else by whole tiles (kind 2): a waiting task holds its CTA
      const int nr = ntr - jq;
      // (measured at config 2: with 2 new tile rows the half-tile chains win even
      // when they cannot all be resident, 340 -> 255 us; with 7 they lose)
      const bool halves = halves_mode >= 0 ? halves_mode != 0 : (2 * nr * (jq - 1) <= (int)gridDim.x - 2 || nr <= 2);
      const int per = halves ? 2 : 1;
      const int nh = (jq - 1) * nr * per;
      const int u = t - (jq - 1);
      if (t < jq - 1) {
        kind = 5;
        j = t + 1;
      } else if (u < nr) {
        kind = 2;
        j = 0;
        i = jq + u;
      } else if (u - nr < nh) {
        const int v = u - nr;
        kind = halves ? 6 : 2;
        j = 1 + v / (per * nr);
        i = jq + (v % (per * nr)) / per;
        half = v % per;
      } else if (u - nr == nh) {
        kind = 3;
      }
      t -= (jq - 1) + nr + nh + 1;
    }
    while (kind < 0 && j < ntc) {
      const int np1 = (j + 1 < ntc) ? 1 : 0;          // P(j+1,j+1)
      const int np2 = (j + 1 < ntr) ? 1 : 0;          // P(j+1,j)
      const int nT = max(0, ntr - (j + 2));           // T(i,j)
      const int cnt = np1 + np2 + nT;
      if (t < cnt) {
        if (t < np1) { kind = 0; i = j + 1; }
        else if (t < np1 + np2) { kind = 1; i = j + 1; }
        else { kind = 2; i = j + 2 + (t - np1 - np2); }
        break;
      }
      t -= cnt;
      ++j;
    }
    if (kind < 0) break;
    // ---- pipelined kinds: P(j+1,j+1), P(j+1,j), T(i,j) outside a restart row chain, D(jq)
    const bool piped = kind == 0 || kind == 1 || kind == 3 || kind == 2;
    if (piped) {
      const int ti = kind == 3 ? jq : (kind == 2 ? i : j + 1);
      const int tj = kind == 3 ? jq : (kind == 0 ? j + 1 : j);
      // restart row chain (whole tiles): L(i,j) = B - L(i,j-1) W_j with
      // B = (A(i,j) - sum_{k<j-1} L(i,k) L(j,k)^T) Linv_jj^T: the ring carries
      // the j-1 updates, Linv_jj, then {L(i,j-1), W_j} as one more stage
      const bool rchain = kind == 2 && j < jq && j > 0;
      const int kmax = kind == 3 ? jq : (rchain ? j - 1 : j);
      const bool trsm = kind == 2;
      double* ring = smem;
      if (w == kThreads / 32) {  // ---- producer warp
        if (lane == 0) {
          ring_produce(R, ring, Lt, Linv, F, epoch, ti, tj, kmax, jq, trsm ? tj : -1, rcnt);
          if (rchain) {
            const int sidx = (int)(rcnt % kStages);
            const unsigned use = rcnt / kStages;
            if (use > 0) ring_wait(&R.empty[sidx], (use - 1) & 1);
            double* slot = ring + (size_t)(2 * sidx) * TS;
            wait_flag(&F.part[tidx(tj, tj - 1)], epoch);  // W_j (task W(j)): in flight first
            asm volatile("fence.proxy.async.global;\n" ::: "memory");
            ring_expect(&R.full[sidx], 2u * TS * 8);
            ring_load_tile(slot + TS, Wbuf + (size_t)tj * TS, &R.full[sidx]);
            wait_flag(&F.full[tidx(ti, tj - 1)], epoch);  // L(i,j-1): the row chain's previous step
            asm volatile("fence.proxy.async.global;\n" ::: "memory");
            ring_load_tile(slot, Lt + (size_t)tidx(ti, tj - 1) * TS, &R.full[sidx]);
            ++rcnt;
          }
        } else {
          rcnt += kmax + (trsm ? 1 : 0) + (rchain ? 1 : 0);
        }
        continue;
      }
      // ---- consumer warps 0..7: split-K 32 x 32 quadrants (q32_origin)
      int rb0, cb0, k0;
      q32_origin(w, rb0, cb0, k0);
      double acc[4][4][2];
      if (k0 == 0) {
        gather_acc32(acc, G, ldg, cvec, Fidx, f, ti, tj, lane, rb0, cb0);
      } else {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[a][q][0] = acc[a][q][1] = 0.0;
      }
      ring_consume_updates32(R, ring, acc, kmax, rcnt, lane, rb0, cb0, k0);
      // S: slot B of the next stage (free: the producer waits for the next task)
      double* Sx = ring + (size_t)(2 * (rcnt % kStages) + 1) * TS;
      csync();  // every warp is past its updates (a fast warp runs up to kStages ahead): Sx is free
      if (k0 != 0) acc32_io(acc, Sx, lane, rb0, cb0, 0);  // the second k-half's sums
      csync();
      if (k0 == 0) acc32_io(acc, Sx, lane, rb0, cb0, 2);
      if (trsm) {
        const int sidx = (int)(rcnt % kStages);
        if (k0 == 0) acc32_io(acc, Sx, lane, rb0, cb0, 0);
        ring_wait(&R.full[sidx], (rcnt / kStages) & 1);  // Linv_jj in slot A
        csync();
        double acc8[8][2];
        gemm_linvT(acc8, Sx, ring + (size_t)(2 * sidx) * TS, w, lane);
        csync();
        store_rows8(acc8, Sx, w, lane);
        csync();
        if (rchain) {  // Sx = B; the last step L(i,j) = B - L(i,j-1) W_j (split-K, the tail stage)
          __syncwarp();
          if (lane == 0) ring_arrive(&R.empty[sidx]);
          ++rcnt;
          const int s2 = (int)(rcnt % kStages);
          if (k0 == 0) {
            acc32_io(acc, Sx, lane, rb0, cb0, 1);
          } else {
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
              for (int q = 0; q < 4; ++q) acc[a][q][0] = acc[a][q][1] = 0.0;
          }
          ring_wait(&R.full[s2], (rcnt / kStages) & 1);
          const double* slot = ring + (size_t)(2 * s2) * TS;
          dmma_q32_sub(acc, slot, slot + TS, lane, rb0, cb0, k0);
          __syncwarp();
          if (lane == 0) ring_arrive(&R.empty[s2]);
          ++rcnt;
          csync();  // B read by every warp
          if (k0 != 0) acc32_io(acc, Sx, lane, rb0, cb0, 0);
          csync();
          if (k0 == 0) {
            acc32_io(acc, Sx, lane, rb0, cb0, 2);
            acc32_io(acc, Sx, lane, rb0, cb0, 0);
          }
          csync();
          store_tile(Lt + (size_t)tidx(ti, tj) * TS, Sx);
          publish_flag(&F.full[tidx(ti, tj)], epoch);
          continue;
        }
        store_tile(Lt + (size_t)tidx(ti, tj) * TS, Sx);
        __syncwarp();
        if (lane == 0) ring_arrive(&R.empty[sidx]);
        ++rcnt;
        publish_flag(&F.full[tidx(ti, tj)], epoch);
        if (jq > 0 && tj == 0 && ti >= jq && tid == 0) {  // (the restart's half-tile chain starts here)
          st_release(&F.part[tidx(ti, tj)], epoch);
          st_release(&F.half1[tidx(ti, tj)], epoch);
        }
        if (ti == tj + 2) PROF_STAMP(1000 + tj + 1, 1);
      } else {
        // partial tiles go out in the global tile layout straight from the fragments
        double* dst = Lt + (size_t)tidx(ti, tj) * TS;
        if (k0 == 0) acc32_io(acc, dst, lane, rb0, cb0, 0);
        publish_flag(&F.part[tidx(ti, tj)], epoch);
        if (kind == 0) PROF_STAMP(1000 + ti, 2);
        else if (kind == 1) PROF_STAMP(1000 + tj, 0);
      }
      continue;
    }
    if (w >= kThreads / 32) continue;  // the producer warp idles through the restart kinds
    if (kind == 6) {                 // Th(i, j, half): rows 32*half.. of L(i,j) below a kept prefix
      // the restart row chain by half tiles: each step is a 32 x 64 x 64
      // product on its own CTA (half the DMMA time of a full tile), the two
      // halves of a row chain run independently.
      // L(i,j)_h = B_h - L(i,j-1)_h W_j,  B_h = (A(i,j)_h - sum_{k<j-1} L(i,k)_h L(j,k)^T) Linv_jj^T
      const int r0 = 32 * half;
      const int rb0 = (w >> 2) * 16, cb0 = (w & 3) * 16;
      int* const hflag = half ? F.half1 : F.part;
      double* Lv = smem + 5 * T * LDS;   // Linv_jj
      double* LB = smem + 1 * T * LDS;   // L(j, k) (kept)
      double* Wt = smem + 2 * T * LDS;   // W_j^T
      double* Xp = smem + 3 * T * LDS;   // rows of L(i, j-1) / L(i, k)
      tile_async(Lv, Linv + (size_t)j * TS);
      cp_async_commit();
      {  // gather rows r0.. of A(i,j) (tile row i >= jq: never the chain's)
        const int rv = min(T, f + 1 - i * T), cv = min(T, f - j * T);
        for (int e = tid; e < 32 * T; e += kThreads) {
          const int r = r0 + e / T, cc = e % T;
          const int gi = i * T + r, gj = j * T + cc;
          double v = 0.0;
          if (r < rv && cc < cv) v = (gi < f) ? G[(size_t)Fidx[gi] * ldg + Fidx[gj]] : cvec[Fidx[gj]];
          S[(e / T) * LDS + cc] = v;
        }
      }
      csync();
      double acc[2][2][2];
      acc_half_ls(acc, S, lane, rb0, cb0, false);
      for (int k = 0; k < j - 1; ++k) {  // (off the critical path: these rows arrived a step earlier)
        if (tid == 0) wait_flag(&hflag[tidx(i, k)], epoch);
        csync();
        half_async(Xp, Lt + (size_t)tidx(i, k) * TS, r0);
        tile_async(LB, Lt + (size_t)tidx(j, k) * TS);
        cp_async_commit();
        cp_async_wait<0>();
        csync();
        dmma_half_sub(acc, Xp, LB, lane, rb0, cb0);
        csync();
      }
      acc_half_ls(acc, S, lane, rb0, cb0, true);
      cp_async_wait<0>();
      if (tid == 0) wait_flag(&F.part[tidx(j, j - 1)], epoch);  // W_j
      csync();
      tile_async(Wt, Wbuf + (size_t)j * TS);
      cp_async_commit();
      {
        double acc8[8][2];
        if (w < 4) gemm_linvT(acc8, S, Lv, w, lane);  // rows 8w.. of the half
        csync();
        if (w < 4) store_rows8(acc8, S, w, lane);  // S = B_h
      }
      if (tid == 0) wait_flag(&hflag[tidx(i, j - 1)], epoch);
      csync();
      half_async(Xp, Lt + (size_t)tidx(i, j - 1) * TS, r0);
      cp_async_commit();
      cp_async_wait<0>();
      csync();
      acc_half_ls(acc, S, lane, rb0, cb0, false);
      dmma_half_sub(acc, Xp, Wt, lane, rb0, cb0);  // -= L(i,j-1)_h W_j
      acc_half_ls(acc, S, lane, rb0, cb0, true);
      csync();
      double* dst = Lt + (size_t)tidx(i, j) * TS + r0 * LDS;
      for (int e = threadIdx.x; e < 32 * T / 2; e += kThreads) {
        const int o = ((2 * e) / T) * LDS + (2 * e) % T;
        *reinterpret_cast<double2*>(dst + o) = *reinterpret_cast<const double2*>(S + o);
      }
      publish_flag(&hflag[tidx(i, j)], epoch);
      if (half == 1 && tid == 0) {  // the whole tile: after the other half too
        wait_flag(&F.part[tidx(i, j)], epoch);
        st_release(&F.full[tidx(i, j)], epoch);
      }
      continue;
    }
    if (kind == 5) {                 // W(j) = (L(j,j-1)^T Linv_jj^T)^T = Linv_jj L(j,j-1) (kept tiles)
      const int rb0 = (w >> 1) * 16, cb0 = (w & 1) * 32;
      double* Lv = smem + 5 * T * LDS;
      double* Ls = smem + 1 * T * LDS;
      tile_async(Lv, Linv + (size_t)j * TS);
      tile_async(Ls, Lt + (size_t)tidx(j, j - 1) * TS);
      cp_async_commit();
      cp_async_wait<0>();
      csync();
      double acc[2][4][2] = {};
      dmma_tile_nn(acc, Lv, Ls, lane, rb0, cb0);
      acc_store(acc, S, lane, rb0, cb0);
      csync();
      store_tile(Wbuf + (size_t)j * TS, S);
      publish_flag(&F.part[tidx(j, j - 1)], epoch);  // (a kept tile's part flag: W_j ready)
      continue;
    }
    // (every other kind runs on the helper operand pipeline above)
  }
}

cudaError_t chol_debug_set_profile(unsigned long long* p) {
  return cudaMemcpyToSymbol(g_chol_prof, &p, sizeof(p));
}

// ---------------------------------------------------------------------------
// L^T x = z (z = row f of the bordered factor), column tiles J from the last
// to the first, as a CHAIN fed by helper tasks:
//   x_J = Linv_JJ^T (s'_J - L(J+1,J)^T x_{J+1}) = a_J - N_J^T x_{J+1},
//   s'_J = z_J - sum_{I >= J+2} L(I,J)^T x_I,   a_J = Linv_JJ^T s'_J,
//   N_J  = L(J+1,J) Linv_JJ.
// Helper task J (CTAs 1..) forms N_J first (DMMA; it needs no x) and
// publishes it, then accumulates s'_J as the x_I arrive and publishes a_J.
// The chain (CTA 0) only does x_J = a_J - N_J^T x_{J+1}: one 64x64 GEMV per
// tile column with x kept on chip and N_J streamed in ahead by bulk copies;
// warp 6 feeds it (flags, bulk copies, a_J), warp 7 publishes x_J for the
// helpers, warps 0-5 compute.  The per-column critical path has no global
// round trip (the previous design paid ~2 us of flag + fence per column).
namespace {
constexpr int kBsStages = 3;  // chain ring stages, each {N_J, P_J}
constexpr size_t kBsSmem = sizeof(double) * 6 * (size_t)TS;  // chain: 3 x 2 tiles; helper: 5 tiles

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
// arrive with the expected byte count; one bulk copy of a whole tile
__device__ __forceinline__ void mbar_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_tile_to_smem(double* dst, const double* src, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "n"(TS * 8), "r"(smem_u32(b))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned phase) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ int vld(const int* p) { return *(const volatile int*)p; }
// Mailboxes: x_J and a_J pass between CTAs as 64 doubles written with plain
// (8-byte, single-copy atomic) stores into slots that held an "empty"
// pattern -- a signalling NaN carrying the epoch, which no arithmetic result
// can equal -- and consumers poll the values themselves: no fence and no flag
// on the critical path.  The factorization kernel empties the slots of the
// epoch's parity before the back substitution starts.
__device__ __forceinline__ unsigned long long ld_box(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_box(unsigned long long* p, double v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;\n" ::"l"(p), "l"((unsigned long long)__double_as_longlong(v))
               : "memory");
}
__device__ __forceinline__ void vst(int* p, int v) { *(volatile int*)p = v; }
__device__ __forceinline__ void bar_compute() { asm volatile("bar.sync 1, 192;\n" ::: "memory"); }
}  // namespace

// acc (rows 8w..8w+7, all 64 columns) = A Linv for 64 x 64 smem tiles, Linv
// lower triangular: column block q only needs k >= 8q (72 DMMAs per warp).
__device__ __forceinline__ void gemm_linv(double (&acc)[8][2], const double* __restrict__ A,
                                          const double* __restrict__ Linv, int w, int lane) {
  const int rq = lane >> 2, kq = lane & 3;
#pragma unroll
  for (int q = 0; q < 8; ++q) acc[q][0] = acc[q][1] = 0.0;
#pragma unroll
  for (int kb = 0; kb < T / 4; ++kb) {
    const double av = A[(8 * w + rq) * LDS + 4 * kb + kq];
#pragma unroll
    for (int q = 0; q <= kb / 2 && q < 8; ++q)
      dmma8x8x4(acc[q][0], acc[q][1], av, Linv[(4 * kb + kq) * LDS + 8 * q + rq]);
  }
}

struct BsArgs {
  const double* Lt;
  const double* Linv;
  double* Nt;    // N_J = L(J+1,J) Linv_JJ tiles
  double* Pt;    // P_J = L(J+2,J) Linv_JJ tiles
  unsigned long long* box;   // mailboxes [epoch parity][x | a][boxlen]
  int boxlen;                // T * tile rows of the allocation
  unsigned long long* xbox;  // (set in the kernel: this epoch's x_J mailboxes, T per tile column)
  unsigned long long* abox;  // (a_J mailboxes)
  int* nflags;
  double* xF;
  const int32_t* Fidx;
  double* xs;
};

__device__ void backsolve_chain(const BsArgs& a, int f, int epoch, double* ring) {
  __shared__ double abuf[kBsStages][T];
  __shared__ double xbuf[3][T];
  __shared__ double part[3 * T];
  __shared__ __align__(8) unsigned long long mbar[kBsStages];
  __shared__ int s_consumed, s_xready, s_pub;
  const int ntc = (f + T - 1) / T;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int k = 0; k < kBsStages; ++k) mbar_init(&mbar[k], 2);  // tiles (or plain) + a_J
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    s_consumed = 0;
    s_xready = 0;
    s_pub = 0;
  }
  __syncthreads();
  if (w == 6) {
    // ---- feeder: arm the stage of step tN with N_J, P_J (bulk copies) as
    // soon as they are published, deliver a_J of step tA into abuf
    int tN = 0, tA = 0;
    const unsigned long long empty = box_empty(epoch);
    while (tA < ntc) {
      bool moved = false;
      if (tN < ntc && tN - vld(&s_consumed) < kBsStages) {
        const int J = ntc - 1 - tN, stage = tN % kBsStages;
        int ok = 1;
        if (lane == 0 && J < ntc - 1) ok = ld_acquire(&a.nflags[J]) == epoch;
        ok = __shfl_sync(kFull, ok, 0);
        if (ok) {
          if (lane == 0) {
            double* dst = ring + (size_t)stage * 2 * TS;
            const int nt = (J + 2 < ntc) ? 2 : (J + 1 < ntc ? 1 : 0);
            if (nt > 0) {
              mbar_expect(&mbar[stage], (unsigned)(nt * TS * 8));
              bulk_tile_to_smem(dst, a.Nt + (size_t)J * TS, &mbar[stage]);
              if (nt > 1) bulk_tile_to_smem(dst + TS, a.Pt + (size_t)J * TS, &mbar[stage]);
            } else {
              mbar_arrive(&mbar[stage]);  // the last column has neither
            }
          }
          ++tN;
          moved = true;
        }
      }
      if (tA < tN) {
        const int J = ntc - 1 - tA, stage = tA % kBsStages;
        const unsigned long long v0 = ld_box(&a.abox[J * T + lane]), v1 = ld_box(&a.abox[J * T + lane + 32]);
        if (__all_sync(kFull, v0 != empty && v1 != empty)) {
          abuf[stage][lane] = __longlong_as_double((long long)v0);
          abuf[stage][lane + 32] = __longlong_as_double((long long)v1);
          __syncwarp();
          if (lane == 0) mbar_arrive(&mbar[stage]);  // (release: abuf visible to the waiters)
          ++tA;
          moved = true;
        }
      }
      if (!moved) __nanosleep(32);
    }
  } else if (w == 7) {
    // ---- publisher: x_J -> mailbox, x_F (and xs), off the chain's path
    for (int t = 0; t < ntc; ++t) {
      while (vld(&s_xready) <= t) __nanosleep(20);
      const int J = ntc - 1 - t, cv = min(T, f - J * T);
      for (int e = lane; e < T; e += 32) {
        const double v = xbuf[t % 3][e];  // (0 beyond cv)
        st_box(&a.xbox[J * T + e], v);
        if (e < cv) {
          a.xF[J * T + e] = v;
          if (a.xs != nullptr) a.xs[a.Fidx[J * T + e]] = v;
        }
      }
      __syncwarp();
      if (lane == 0) vst(&s_pub, t + 1);
    }
  } else {
    // ---- compute warps 0-5: x_J = a_J - N_J^T x_{J+1} - P_J^T x_{J+2}
    const int c = tid & (T - 1), rg = tid >> 6;  // 3 row groups
    for (int t = 0; t < ntc; ++t) {
      const int J = ntc - 1 - t, stage = t % kBsStages;
      mbar_wait(&mbar[stage], (unsigned)((t / kBsStages) & 1));
      double p = 0.0, p2 = 0.0;
      const double* Nl = ring + (size_t)stage * 2 * TS;
      if (t > 0) {
        const double* xp = xbuf[(t - 1) % 3];
#pragma unroll 4
        for (int r = rg; r < T; r += 3) p = fma(Nl[r * LDS + c], xp[r], p);
      }
      if (t > 1) {
        const double* xp = xbuf[(t - 2) % 3];
#pragma unroll 4
        for (int r = rg; r < T; r += 3) p2 = fma(Nl[TS + r * LDS + c], xp[r], p2);
      }
      part[rg * T + c] = p + p2;
      bar_compute();
      if (tid < T) {
        if (t >= 3)
          while (vld(&s_pub) < t - 2) __nanosleep(20);  // warp 7 has read xbuf[t % 3] (step t-3)
        const int cv = min(T, f - J * T);
        const double sum = (part[tid] + part[T + tid]) + part[2 * T + tid];
        xbuf[t % 3][tid] = (tid < cv) ? abuf[stage][tid] - sum : 0.0;
      }
      bar_compute();
      if (tid == 0) {
        __threadfence_block();
        vst(&s_consumed, t + 1);  // stage (tiles, abuf) free
        vst(&s_xready, t + 1);
      }
      PROF_STAMP(900 + J, 0);
    }
  }
}

// helper task J: N_J and P_J, then s'_J and a_J
__device__ void backsolve_task(const BsArgs& a, int f, int epoch, int J, double* bsm) {
  __shared__ double part[4 * T];
  __shared__ double s_rhs[T];
  __shared__ double s_x[T];
  double* Xi = bsm;            // Linv_JJ
  double* Ls = bsm + TS;       // L(J+1, J), L(J+2, J)
  double* ring = bsm + 3 * TS; // L(I, J), double-buffered
  const int ntc = (f + T - 1) / T;
  const int Rf = f / T, rf = f % T;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int c = tid & (T - 1), rg = tid >> 6;
  const int cv = min(T, f - J * T);
  const int nI = max(0, ntc - 1 - (J + 2));  // I = ntc-1 .. J+3 (the chain applies J+1, J+2)
  const unsigned long long empty = box_empty(epoch);
  tile_async(Xi, a.Linv + (size_t)J * TS);
  if (J + 1 < ntc) tile_async(Ls, a.Lt + (size_t)tidx(J + 1, J) * TS);
  if (J + 2 < ntc) tile_async(Ls + TS, a.Lt + (size_t)tidx(J + 2, J) * TS);
  cp_async_commit();
  if (nI > 0) {
    tile_async(ring, a.Lt + (size_t)tidx(ntc - 1, J) * TS);
    cp_async_commit();
  }
  if (tid < T) s_rhs[tid] = (tid < cv) ? __ldcg(&a.Lt[(size_t)tidx(Rf, J) * TS + rf * LDS + tid]) : 0.0;
  if (nI > 0) cp_async_wait<1>();
  else cp_async_wait<0>();
  __syncthreads();
  // N_J = L(J+1,J) Linv_JJ and P_J = L(J+2,J) Linv_JJ, straight from the fragments to global
  for (int b = 1; b <= 2 && J + b < ntc; ++b) {
    double acc[8][2];
    gemm_linv(acc, Ls + (size_t)(b - 1) * TS, Xi, w, lane);
    double* Ng = (b == 1 ? a.Nt : a.Pt) + (size_t)J * TS;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      *reinterpret_cast<double2*>(Ng + (8 * w + (lane >> 2)) * LDS + 8 * q + 2 * (lane & 3)) =
          make_double2(acc[q][0], acc[q][1]);
  }
  if (J + 1 < ntc) {
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release(&a.nflags[J], epoch);
  }
  for (int k = 0; k < nI; ++k) {  // s'_J -= L(I,J)^T x_I, tiles prefetched one ahead
    const int I = ntc - 1 - k;
    double* Tl = ring + (size_t)(k & 1) * TS;
    if (k + 1 < nI) {
      tile_async(ring + (size_t)((k + 1) & 1) * TS, a.Lt + (size_t)tidx(I - 1, J) * TS);
      cp_async_commit();
    }
    if (tid < T) {  // x_I from its mailbox (0 beyond its valid rows)
      unsigned long long v;
      while ((v = ld_box(&a.xbox[I * T + tid])) == empty) __nanosleep(20);
      s_x[tid] = __longlong_as_double((long long)v);
    }
    if (k + 1 < nI) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    double p = 0.0;
#pragma unroll 4
    for (int r = rg; r < T; r += 4) p = fma(Tl[r * LDS + c], s_x[r], p);
    part[rg * T + c] = p;
    __syncthreads();
    if (tid < T) s_rhs[tid] -= (part[tid] + part[T + tid]) + (part[2 * T + tid] + part[3 * T + tid]);
    __syncthreads();
  }
  // a_J = Linv_JJ^T s'_J
  double p = 0.0;
#pragma unroll 4
  for (int r = rg; r < T; r += 4) p = fma(Xi[r * LDS + c], s_rhs[r], p);
  part[rg * T + c] = p;
  __syncthreads();
  if (tid < T) st_box(&a.abox[J * T + tid], (part[tid] + part[T + tid]) + (part[2 * T + tid] + part[3 * T + tid]));
  __syncthreads();  // (smem reused by the next task)
}

constexpr int kDualPrefetch = 1024;  // early release while the dual prefetches a good part of its G rows (PF * 32 = 512 entries, pivot.cu)
__global__ void __launch_bounds__(kThreads) chol_backsolve_kernel(BsArgs a, DevState* st) {
  extern __shared__ __align__(128) double bsm[];
  pdl_wait();
  // small F: let the dual kernel start now -- it gathers its whole G rows
  // into registers while this runs (and reads nothing of ours before its own
  // griddepcontrol.wait).  Large F: its CTAs would only compete with this
  // kernel for the SMs and the memory system, so it starts at our exit.
  if (st->f <= kDualPrefetch) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  __shared__ int s_task, s_role;
  const int f = st->f;
  const int epoch = st->epoch;
  if (f <= 0 || st->done || st->status != 0) return;  // (graph loop: nothing to solve)
  const int ntc = (f + T - 1) / T;
  a.xbox = a.box + (size_t)(2 * (epoch & 1)) * a.boxlen;
  a.abox = a.xbox + a.boxlen;
  if (threadIdx.x == 0) s_role = atomicAdd(&st->role_solve, 1);  // first CTA to run: the chain
  __syncthreads();
  if (s_role == 0) {
    backsolve_chain(a, f, epoch, bsm);
    return;
  }
  for (;;) {
    if (threadIdx.x == 0) s_task = atomicAdd(&st->solve_counter, 1);
    __syncthreads();
    const int t = s_task;
    __syncthreads();
    if (t >= ntc) break;
    backsolve_task(a, f, epoch, ntc - 1 - t, bsm);
  }
}

static cudaError_t set_attrs() {
  static DeviceOnce once;  // (per device: attributes are per device)
  cudaError_t err = cudaSuccess;
  const int ok = device_once(once, [&]() {
    err = cudaFuncSetAttribute(chol_factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)(sizeof(double) * kSmemDoubles));
    if (err == cudaSuccess)
      err = cudaFuncSetAttribute(chol_backsolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBsSmem);
    return err == cudaSuccess ? 1 : 0;
  });
  return ok ? cudaSuccess : err;
}

cudaError_t launch_chol_factor(int n, const double* G, int ldg, const double* c, const int32_t* Fidx,
                               double* Lt, int* flags, DevState* st, int sm_count, cudaStream_t s) {
  cudaError_t e = set_attrs();
  if (e != cudaSuccess) return e;
  // grid sized for the largest possible DAG; tasks are claimed dynamically
  const int tasks = tri_tiles(n) + (n + 1 + T - 1) / T + 1;  // helper tasks + the chain
  int grid = sm_count;  // ~204 KB smem per CTA: one persistent CTA per SM
  if (grid > tasks) grid = tasks;
  if (grid < 2) grid = 2;
  double* Linv = Lt + (size_t)tri_tiles(n) * TS;
  const int ntr = (n + 1 + T - 1) / T;
  // restart row chains by half tiles: -1 when all fit on the helpers (default), 0 never, 1 always
  static const int halves_mode = [] {
    const char* v = getenv("NNLS_RESTART_HALVES");
    return (v != nullptr && v[0] != 0) ? atoi(v) : -1;
  }();
  unsigned long long* box = reinterpret_cast<unsigned long long*>(Lt + ((size_t)tri_tiles(n) + 3 * (size_t)ntr) * TS);
  return launch_pdl(chol_factor_kernel, dim3(grid), dim3(kHelperThreads), sizeof(double) * kSmemDoubles, s, G, ldg, c,
                    Fidx, Lt, Linv, flags, tri_tiles(n), st, box, ntr * T, halves_mode);
}

cudaError_t launch_chol_backsolve(int n, const double* Lt, int* flags, double* xF, DevState* st,
                                  int sm_count, cudaStream_t s, const int32_t* Fidx, double* xs) {
  const int ntr = (n + 1 + T - 1) / T;
  const int tri = tri_tiles(n);
  BsArgs a;
  a.Lt = Lt;
  a.Linv = Lt + (size_t)tri * TS;
  a.Nt = const_cast<double*>(Lt) + (size_t)(tri + ntr) * TS;
  a.nflags = flags + 2 * tri + 3 * ntr;
  a.Pt = a.Nt + (size_t)ntr * TS;
  a.box = reinterpret_cast<unsigned long long*>(a.Pt + (size_t)ntr * TS);
  a.boxlen = ntr * T;
  a.xF = xF;
  a.Fidx = Fidx;
  a.xs = xs;
  int grid = ntr + 1;  // the chain + one helper per tile column
  if (grid > sm_count) grid = sm_count;
  if (grid < 2) grid = 2;
  cudaError_t e = set_attrs();
  if (e != cudaSuccess) return e;
  return launch_pdl(chol_backsolve_kernel, dim3(grid), dim3(kThreads), kBsSmem, s, a, st);
}

cudaError_t launch_cholesky_solve(int n, const double* G, int ldg, const double* c,
                                  const int32_t* Fidx, double* Lt, int* flags, double* xF,
                                  DevState* st, int sm_count, cudaStream_t s) {
  cudaError_t e = launch_chol_factor(n, G, ldg, c, Fidx, Lt, flags, st, sm_count, s);
  if (e != cudaSuccess) return e;
  return launch_chol_backsolve(n, Lt, flags, xF, st, sm_count, s);
}

}  // namespace nnls
