// ingest_gram.cu -- a0 (CSR validation, CSC build) and a1 (Gram + A^T b).
//
// a1 follows PAPER.md P:126: "A^T A_ij is just the dot product of the i-th and
// j-th columns of A ... we can precompute the full A^T A" -- formed once per
// problem and cached.  B200 design: one warp owns one row i of G and
// accumulates  G[i,:] = sum_{r in col i} a_ri * A[r,:]  (Gustavson row-by-row
// SpGEMM of A^T A) into a dense FP64 accumulator in shared memory; lanes
// scatter the entries of sparse row r (distinct columns, no conflicts), rows r
// are taken in increasing order, products and sums are rounded separately
// (no FMA).  Every G_ij is therefore the sum of the same terms in the same
// order as the dense definition -> bit-identical to the CPU oracle, exactly
// symmetric, deterministic.  The finished row is streamed to HBM once
// (coalesced), so HBM traffic is the n^2 output write plus L2-resident CSR
// reads.
#include <cuda_runtime.h>
#include <math.h>

#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "kernels.cuh"

namespace nnls {

// ---------------------------------------------------------------- validate
// Exponent statistics of the nonzero values: H = exponent of the leading bit,
// L = exponent of the lowest set bit; kept biased so that 0 means "none":
// h = max(h, H + 2048), l = max(l, 2048 - L).  Non-normal values (subnormal)
// make L tiny, i.e. "not exact".  Used by gram_is_exact().
__device__ __forceinline__ void exact_bits(double v, int& h, int& l) {
  if (v == 0.0) return;
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  const int ex = (int)((u >> 52) & 0x7FF);
  if (ex == 0) {  // subnormal
    l = max(l, 4095);
    return;
  }
  const int H = ex - 1023;
  const unsigned long long mant = (u & ((1ull << 52) - 1)) | (1ull << 52);
  const int L = H - 52 + (__ffsll((long long)mant) - 1);
  h = max(h, H + 2048);
  l = max(l, 2048 - L);
}

__global__ void validate_kernel(int m, int n, int64_t nnz, const int32_t* __restrict__ rowptr,
                                const int32_t* __restrict__ colind,
                                const double* __restrict__ vals, const double* __restrict__ b,
                                int* err) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  __shared__ int s_st[4];
  if (threadIdx.x < 4) s_st[threadIdx.x] = 0;
  __syncthreads();
  int e_local = 0, maxlen = 0;
  int hA = 0, lA = 0, hb = 0, lb = 0;  // biased exponent statistics (0: none), see exact_bits
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < m; r += warps) {
    int64_t lo = rowptr[r], hi = rowptr[r + 1];
    if (hi - lo > maxlen) maxlen = (int)min((int64_t)0x7fffffff, hi - lo);
    if (lane == 0) {
      if (r == 0 && lo != 0) e_local |= 1;
      if (r == m - 1 && hi != nnz) e_local |= 1;
      if (!isfinite(b[r])) e_local |= 4;
      exact_bits(b[r], hb, lb);
    }
    if (hi < lo || lo < 0 || hi > nnz) {
      e_local |= 1;
      continue;
    }
    for (int64_t t = lo + lane; t < hi; t += 32) {
      int cidx = colind[t];
      if (cidx < 0 || cidx >= n) e_local |= 2;
      if (t > lo && colind[t - 1] >= cidx) e_local |= 2;
      if (!isfinite(vals[t])) e_local |= 4;
      exact_bits(vals[t], hA, lA);
    }
  }
  if (e_local) atomicOr(err, e_local);
  if (lane == 0 && maxlen > 0) atomicMax(err + 1, maxlen);  // longest row (LSQR planning)
  hA = warp_max_i(hA);
  lA = warp_max_i(lA);
  hb = warp_max_i(hb);
  lb = warp_max_i(lb);
  if (lane == 0) {  // block first, then one global atomic per statistic per block
    if (hA) atomicMax(&s_st[0], hA);
    if (lA) atomicMax(&s_st[1], lA);
    if (hb) atomicMax(&s_st[2], hb);
    if (lb) atomicMax(&s_st[3], lb);
  }
  __syncthreads();
  if (threadIdx.x < 4 && s_st[threadIdx.x]) atomicMax(err + kErrExp + threadIdx.x, s_st[threadIdx.x]);
}

// Flat variant for large inputs: the entries are checked by a coalesced
// pass (range, finiteness, exponent statistics) that also counts every
// descent colind[t] <= colind[t-1]; the rows are checked by a thread each,
// which counts the descents that sit at the first entry of a non-empty row
// (allowed: a new row starts).  Any other descent is an out-of-order or
// repeated column: the last CTA to finish compares the two counts (err[60],
// err[61], zeroed with the rest of err) and raises bit 2.
__global__ void __launch_bounds__(256) validate_flat_kernel(int m, int n, int64_t nnz,
                                                             const int32_t* __restrict__ rowptr,
                                                             const int32_t* __restrict__ colind,
                                                             const double* __restrict__ vals,
                                                             const double* __restrict__ b, int* err) {
  __shared__ int s_st[4];
  __shared__ unsigned long long s_d[2];
  __shared__ bool s_last;
  if (threadIdx.x < 4) s_st[threadIdx.x] = 0;
  if (threadIdx.x < 2) s_d[threadIdx.x] = 0ull;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  int e_local = 0, maxlen = 0;
  int hA = 0, lA = 0, hb = 0, lb = 0;
  unsigned long long dall = 0, dstart = 0;
  for (int64_t t = tid; t < nnz; t += nth) {  // entries: coalesced
    const int cidx = colind[t];
    const double v = vals[t];
    if (cidx < 0 || cidx >= n) e_local |= 2;
    if (!isfinite(v)) e_local |= 4;
    exact_bits(v, hA, lA);
    if (t > 0 && colind[t - 1] >= cidx) ++dall;
  }
  for (int64_t r = tid; r < m; r += nth) {  // rows: a thread each
    const int64_t lo = rowptr[r], hi = rowptr[r + 1];
    if (r == 0 && lo != 0) e_local |= 1;
    if (r == m - 1 && hi != nnz) e_local |= 1;
    if (hi < lo || lo < 0 || hi > nnz) e_local |= 1;
    else {
      if (hi - lo > maxlen) maxlen = (int)min((int64_t)0x7fffffff, hi - lo);
      if (hi > lo && lo > 0 && colind[lo - 1] >= colind[lo]) ++dstart;
    }
    const double bv = b[r];
    if (!isfinite(bv)) e_local |= 4;
    exact_bits(bv, hb, lb);
  }
  if (e_local) atomicOr(err, e_local);
  maxlen = warp_max_i(maxlen);
  if (lane == 0 && maxlen > 0) atomicMax(err + 1, maxlen);  // longest row (LSQR planning)
  hA = warp_max_i(hA);
  lA = warp_max_i(lA);
  hb = warp_max_i(hb);
  lb = warp_max_i(lb);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    dall += __shfl_xor_sync(kFull, dall, o);
    dstart += __shfl_xor_sync(kFull, dstart, o);
  }
  if (lane == 0) {
    if (hA) atomicMax(&s_st[0], hA);
    if (lA) atomicMax(&s_st[1], lA);
    if (hb) atomicMax(&s_st[2], hb);
    if (lb) atomicMax(&s_st[3], lb);
    if (dall) atomicAdd(&s_d[0], dall);
    if (dstart) atomicAdd(&s_d[1], dstart);
  }
  __syncthreads();
  if (threadIdx.x < 4 && s_st[threadIdx.x]) atomicMax(err + kErrExp + threadIdx.x, s_st[threadIdx.x]);
  if (threadIdx.x == 0) {
    unsigned long long* d = reinterpret_cast<unsigned long long*>(err + 60);  // err[60..63]
    if (s_d[0]) atomicAdd(&d[0], s_d[0]);
    if (s_d[1]) atomicAdd(&d[1], s_d[1]);
    __threadfence();
    s_last = atomicAdd(reinterpret_cast<unsigned*>(err + 59), 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    const unsigned long long* d = reinterpret_cast<const unsigned long long*>(err + 60);
    if (atomicAdd(const_cast<unsigned long long*>(&d[0]), 0ull) != atomicAdd(const_cast<unsigned long long*>(&d[1]), 0ull))
      atomicOr(err, 2);
  }
}

cudaError_t launch_validate(int m, int n, int64_t nnz, const int32_t* rowptr, const int32_t* colind,
                            const double* vals, const double* b, int* err, cudaStream_t s) {
  if (nnz >= (1 << 20)) {  // (large inputs: the flat, coalesced variant)
    int blocks = (int)((nnz + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    validate_flat_kernel<<<blocks, 256, 0, s>>>(m, n, nnz, rowptr, colind, vals, b, err);
    return cudaGetLastError();
  }
  int blocks = (int)((((int64_t)m * 32) + 255) / 256);
  if (blocks > 4096) blocks = 4096;
  if (blocks < 1) blocks = 1;
  validate_kernel<<<blocks, 256, 0, s>>>(m, n, nnz, rowptr, colind, vals, b, err);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- CSR->CSC
// Column counts: a shared-memory histogram per CTA (when n fits), flushed
// with one global atomic per non-empty bin; few CTAs, so the flush stays
// small next to the nnz shared-memory atomics.
constexpr int kHistMax = 12288;
__global__ void colcount_kernel(int64_t nnz, int n, const int32_t* __restrict__ colind, int32_t* cnt) {
  extern __shared__ int hist[];
  const bool sm = n <= kHistMax;
  if (sm) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) hist[i] = 0;
    __syncthreads();
  }
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int c = colind[e];
    if (c >= 0 && c < n) {  // (runs before validation completes)
      if (sm) atomicAdd(&hist[c], 1);
      else atomicAdd(&cnt[c + 1], 1);
    }
  }
  if (sm) {
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      if (hist[i] != 0) atomicAdd(&cnt[i + 1], hist[i]);
  }
}
static void launch_colcount(int64_t nnz, int n, const int32_t* colind, int32_t* colptr, cudaStream_t s) {
  // ~8 entries per bin per CTA, but at least ~16K entries per CTA up to one
  // CTA per SM (config 2: 25 -> 98 CTAs; the flush adds one atomic per
  // non-empty bin per CTA)
  long long b = nnz / (8LL * (n > 0 ? n : 1));
  const long long bmin = nnz / 16384;
  if (b < bmin) b = bmin;
  if (b > 148) b = 148;
  if (b < 1) b = 1;
  const size_t smem = n <= kHistMax ? sizeof(int) * (size_t)n : 0;
  colcount_kernel<<<(int)b, 1024, smem, s>>>(nnz, n, colind, colptr);
}

// In-place inclusive scan of cnt[0..len) (cnt[0] = 0 on entry) -> colptr; one CTA.
__global__ void scan_kernel(int len, int32_t* cnt, int32_t* cursor, int* maxcnt) {
  __shared__ int32_t wsum[32];
  pdl_wait();
  __shared__ int32_t carry;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  int vmax = 0;
  for (int base = 0; base < len; base += blockDim.x) {
    int i = base + tid;
    int v = i < len ? cnt[i] : 0;
    vmax = max(vmax, v);
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(kFull, w, o);
        if (lane >= o) w += y;
      }
      wsum[lane] = w;
    }
    __syncthreads();
    int incl = x + (wid > 0 ? wsum[wid - 1] : 0) + carry;
    if (i < len) {
      cnt[i] = incl;
      cursor[i] = incl;
    }
    __syncthreads();
    if (tid == blockDim.x - 1) carry = incl;
    __syncthreads();
  }
  vmax = warp_max_i(vmax);
  if (lane == 0 && maxcnt != nullptr) atomicMax(maxcnt, vmax);  // longest column
}

__global__ void csc_scatter_kernel(int m, const int32_t* __restrict__ rowptr,
                                   const int32_t* __restrict__ colind,
                                   const double* __restrict__ vals, int32_t* cursor,
                                   int32_t* tmp_row, double* tmp_val) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < m; r += warps) {
    for (int t = rowptr[r] + lane; t < rowptr[r + 1]; t += 32) {
      int pos = atomicAdd(&cursor[colind[t]], 1);
      tmp_row[pos] = r;
      tmp_val[pos] = vals[t];
    }
  }
}

// Rows within a column arrive in arbitrary order; place each entry at its rank
// (number of smaller row indices in the column) -> sorted, deterministic.
__global__ void csc_sort_kernel(int n, const int32_t* __restrict__ colptr,
                                const int32_t* __restrict__ tmp_row,
                                const double* __restrict__ tmp_val, int32_t* rowind,
                                double* cvals) {
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < n; c += warps) {
    const int lo = colptr[c], len = colptr[c + 1] - lo;
    for (int i = lane; i < len; i += 32) {
      const int ri = tmp_row[lo + i];
      int rank = 0;
      for (int j = 0; j < len; ++j) rank += tmp_row[lo + j] < ri;
      rowind[lo + rank] = ri;
      cvals[lo + rank] = tmp_val[lo + i];
    }
  }
}

// Same ranking with the column's row indices staged in shared memory (one
// warp per column, rank by broadcast compares): columns of up to `cap` rows.
__global__ void csc_sort_smem_kernel(int n, const int32_t* __restrict__ colptr,
                                     const int32_t* __restrict__ tmp_row,
                                     const double* __restrict__ tmp_val, int32_t* rowind, double* cvals,
                                     int cap) {
  extern __shared__ int srow[];
  pdl_wait();
  const int lane = threadIdx.x & 31;
  int* my = srow + (threadIdx.x >> 5) * cap;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < n; c += warps) {
    const int lo = colptr[c], len = colptr[c + 1] - lo;
    for (int i = lane; i < len; i += 32) my[i] = tmp_row[lo + i];
    __syncwarp();
    for (int i = lane; i < len; i += 32) {
      const int ri = my[i];
      int rank = 0;
#pragma unroll 8
      for (int j = 0; j < len; ++j) rank += my[j] < ri;
      rowind[lo + rank] = ri;
      cvals[lo + rank] = tmp_val[lo + i];
    }
    __syncwarp();
  }
}

cudaError_t launch_csr_to_csc(int m, int n, int64_t nnz, const int32_t* rowptr,
                              const int32_t* colind, const double* vals, int32_t* colptr,
                              int32_t* rowind, double* cvals, int32_t* cursor, int32_t* tmp_row,
                              double* tmp_val, cudaStream_t s, int* maxcnt) {
  cudaError_t e = cudaMemsetAsync(colptr, 0, sizeof(int32_t) * (size_t)(n + 1), s);
  if (e != cudaSuccess) return e;
  if (nnz > 0) launch_colcount(nnz, n, colind, colptr, s);
  scan_kernel<<<1, 1024, 0, s>>>(n + 1, colptr, cursor, maxcnt);
  int rb = (int)(((int64_t)m * 32 + 255) / 256);
  if (rb > 4096) rb = 4096;
  if (rb < 1) rb = 1;
  csc_scatter_kernel<<<rb, 256, 0, s>>>(m, rowptr, colind, vals, cursor, tmp_row, tmp_val);
  int cb = (int)(((int64_t)n * 32 + 255) / 256);
  if (cb > 4096) cb = 4096;
  csc_sort_kernel<<<cb, 256, 0, s>>>(n, colptr, tmp_row, tmp_val, rowind, cvals);
  return cudaGetLastError();
}

cudaError_t launch_csc_count(int m, int n, int64_t nnz, const int32_t* colind, int32_t* colptr,
                             int32_t* cursor, cudaStream_t s, int* maxcnt) {
  (void)m;
  cudaError_t e = cudaMemsetAsync(colptr, 0, sizeof(int32_t) * (size_t)(n + 1), s);
  if (e != cudaSuccess) return e;
  if (nnz > 0) launch_colcount(nnz, n, colind, colptr, s);
  return launch_pdl(scan_kernel, dim3(1), dim3(1024), 0, s, n + 1, colptr, cursor, maxcnt);
}

cudaError_t launch_csc_fill(int m, int n, const int32_t* rowptr, const int32_t* colind,
                            const double* vals, const int32_t* colptr, int32_t* rowind,
                            double* cvals, int32_t* cursor, int32_t* tmp_row, double* tmp_val,
                            cudaStream_t s, int maxcnt) {
  int rb = (int)(((int64_t)m * 32 + 255) / 256);
  if (rb > 4096) rb = 4096;
  if (rb < 1) rb = 1;
  cudaError_t e = launch_pdl(csc_scatter_kernel, dim3(rb), dim3(256), 0, s, m, rowptr, colind, vals, cursor,
                             tmp_row, tmp_val);
  if (e != cudaSuccess) return e;
  int cb = (int)(((int64_t)n * 32 + 255) / 256);
  if (cb > 4096) cb = 4096;
  if (cb < 1) cb = 1;
  if (maxcnt >= 0 && maxcnt <= 1536) {  // 8 warps x maxcnt rows in shared memory (<= 48 KB)
    const int cap = maxcnt > 0 ? maxcnt : 1;
    return launch_pdl(csc_sort_smem_kernel, dim3(cb), dim3(256), sizeof(int) * 8 * (size_t)cap, s, n, colptr,
                      tmp_row, tmp_val, rowind, cvals, cap);
  } else {
    csc_sort_kernel<<<cb, 256, 0, s>>>(n, colptr, tmp_row, tmp_val, rowind, cvals);
  }
  return cudaGetLastError();
}

// Device-to-device input upload in ONE launch (rowptr, colind, vals, b as
// four segments of a grid-stride copy, 16-byte moves where both sides are
// aligned) instead of four cudaMemcpyAsync calls.
struct CopySeg {
  const char* src;
  char* dst;
  size_t bytes;
};
__global__ void __launch_bounds__(256) upload_copy_kernel(CopySeg s0, CopySeg s1, CopySeg s2, CopySeg s3) {
  const CopySeg sg[4] = {s0, s1, s2, s3};
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x, nth = (size_t)gridDim.x * blockDim.x;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const CopySeg c = sg[q];
    if (c.bytes == 0) continue;
    const bool al = ((reinterpret_cast<uintptr_t>(c.src) | reinterpret_cast<uintptr_t>(c.dst)) & 15) == 0;
    size_t done = 0;
    if (al) {
      const size_t n16 = c.bytes / 16;
      const uint4* sv = reinterpret_cast<const uint4*>(c.src);
      uint4* dv = reinterpret_cast<uint4*>(c.dst);
      for (size_t i = tid; i < n16; i += nth) dv[i] = __ldcs(&sv[i]);
      done = n16 * 16;
    }
    for (size_t i = done + tid; i < c.bytes; i += nth) c.dst[i] = c.src[i];
  }
}
cudaError_t launch_upload_copy(const void* const* src, void* const* dst, const size_t* bytes, int sm_count,
                               cudaStream_t s) {
  CopySeg g[4];
  size_t tot = 0;
  for (int q = 0; q < 4; ++q) {
    g[q].src = static_cast<const char*>(src[q]);
    g[q].dst = static_cast<char*>(dst[q]);
    g[q].bytes = bytes[q];
    tot += bytes[q];
  }
  long long blocks = (long long)((tot / 16 + 255) / 256);
  if (blocks > (long long)sm_count * 8) blocks = (long long)sm_count * 8;
  if (blocks < 1) blocks = 1;
  upload_copy_kernel<<<(int)blocks, 256, 0, s>>>(g[0], g[1], g[2], g[3]);
  return cudaGetLastError();
}

// CSR -> CSC as a stable radix sort of the entries by column: the CSR lists
// them in increasing row order, so a stable sort on the column index leaves
// each column's rows sorted (the same CSC as the scatter + rank path, in a
// few streaming passes instead of atomics and O(len^2) ranking).  The value
// sorted along is (row << 32 | entry index); one gather then writes rowind
// and cvals.
__global__ void csc_expand_kernel(int m, const int32_t* __restrict__ rowptr, unsigned long long* __restrict__ pk) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int warps = (gridDim.x * blockDim.x) >> 5;
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < m; r += warps) {
    const int t1 = rowptr[r + 1];
    for (int t = rowptr[r] + lane; t < t1; t += 32) pk[t] = ((unsigned long long)(unsigned)r << 32) | (unsigned)t;
  }
}
__global__ void csc_gather_kernel(int64_t nnz, const double* __restrict__ vals, int32_t* __restrict__ rowind,
                                  double* cvals) {
  pdl_wait();
  const unsigned long long* pk = reinterpret_cast<const unsigned long long*>(cvals);  // sorted (row, t), in place
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long v = pk[p];
    rowind[p] = (int32_t)(v >> 32);
    cvals[p] = vals[(unsigned)(v & 0xffffffffu)];
  }
}
static int csc_key_bits(int n) {
  int b = 1;
  while (b < 31 && (1 << b) < n) ++b;
  return b;
}
size_t csc_sort_temp_bytes(int64_t nnz, int n) {
  if (nnz <= 0 || nnz >= ((int64_t)1 << 31)) return 0;
  size_t bytes = 0;
  if (cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                      (const unsigned long long*)nullptr, (unsigned long long*)nullptr, (int)nnz, 0,
                                      csc_key_bits(n)) != cudaSuccess)
    return 0;
  return bytes;
}
cudaError_t launch_csc_fill_sorted(int m, int n, int64_t nnz, const int32_t* rowptr, const int32_t* colind,
                                   const double* vals, int32_t* rowind, double* cvals, int32_t* tmp_row,
                                   double* tmp_val, void* temp, size_t temp_bytes, cudaStream_t s) {
  if (nnz <= 0) return cudaSuccess;
  unsigned long long* pin = reinterpret_cast<unsigned long long*>(tmp_val);
  unsigned long long* pout = reinterpret_cast<unsigned long long*>(cvals);
  int rb = (int)(((int64_t)m * 32 + 255) / 256);
  if (rb > 4096) rb = 4096;
  if (rb < 1) rb = 1;
  cudaError_t e = launch_pdl(csc_expand_kernel, dim3(rb), dim3(256), 0, s, m, rowptr, pin);
  if (e != cudaSuccess) return e;
  size_t tb = temp_bytes;
  e = cub::DeviceRadixSort::SortPairs(temp, tb, colind, tmp_row, pin, pout, (int)nnz, 0, csc_key_bits(n), s);
  if (e != cudaSuccess) return e;
  int gb = (int)((nnz + 255) / 256);
  if (gb > 8192) gb = 8192;
  return launch_pdl(csc_gather_kernel, dim3(gb), dim3(256), 0, s, nnz, vals, rowind, cvals);
}

// ---------------------------------------------------------------- Gram
__global__ void __launch_bounds__(256) gram_kernel(
    int n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
    const double* __restrict__ vals, const int32_t* __restrict__ colptr,
    const int32_t* __restrict__ rowind, const double* __restrict__ cvals,
    const double* __restrict__ b, int row_begin, int row_end, double* __restrict__ G, int ldg,
    double* __restrict__ c, int chunk) {
  // work item = (G row i, column chunk [j0, j0 + chunk)); the chunk width
  // bounds the per-warp smem accumulator so that many warps per SM hide the
  // L2 latency of the A-row gathers.  Each entry still sums its products in
  // increasing row order r.
  extern __shared__ double acc_all[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  double* acc = acc_all + (size_t)wid * chunk;
  for (int j = lane; j < chunk; j += 32) acc[j] = 0.0;
  __syncwarp();
  const int total_warps = gridDim.x * wpb;
  const int nchunk = (n + chunk - 1) / chunk;
  constexpr int U = 8;  // A rows whose (j, a_rj) are in flight together (hides the L2 latency)
  for (int item = blockIdx.x * wpb + wid; item < n * nchunk; item += total_warps) {
    const int i = item / nchunk, j0 = (item % nchunk) * chunk;
    const int jw = min(chunk, n - j0);
    const int e0 = colptr[i], e1 = colptr[i + 1];
    double ci = 0.0;
    for (int eb = e0; eb < e1; eb += 32) {
      // prefetch 32 (row, value, row extent, b_r) tuples of column i
      int my_r = 0, my_lo = 0, my_hi = 0;
      double my_a = 0.0, my_b = 0.0;
      if (eb + lane < e1) {
        my_r = rowind[eb + lane];
        my_a = cvals[eb + lane];
        if (my_r >= row_begin && my_r < row_end) {
          my_lo = rowptr[my_r];
          my_hi = rowptr[my_r + 1];
          my_b = b[my_r];
        }
      }
      const int cnt = min(32, e1 - eb);
      for (int q0 = 0; q0 < cnt; q0 += U) {
        // gather: the first 64 entries of U rows (2 per lane), all loads in flight
        int jj[U][2];
        double av[U], vv[U][2];
        int lo_[U], hi_[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int q = min(q0 + u, cnt - 1);
          lo_[u] = __shfl_sync(kFull, my_lo, q);
          hi_[u] = (q0 + u < cnt) ? __shfl_sync(kFull, my_hi, q) : lo_[u];
          av[u] = __shfl_sync(kFull, my_a, q);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int t = lo_[u] + lane + 32 * h;
            jj[u][h] = -1;
            vv[u][h] = 0.0;
            if (t < hi_[u]) {
              jj[u][h] = colind[t];
              vv[u][h] = vals[t];
            }
          }
        }
        // apply in increasing row order (bit-identical to the sequential sum)
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (q0 + u < cnt) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const unsigned jl = (unsigned)(jj[u][h] - j0);  // -1 (empty) wraps and is skipped
              if (jl < (unsigned)jw) acc[jl] = __dadd_rn(acc[jl], __dmul_rn(av[u], vv[u][h]));
            }
            for (int t = lo_[u] + 64 + lane; t < hi_[u]; t += 32) {  // rows longer than 64
              const unsigned jl = (unsigned)(colind[t] - j0);
              if (jl < (unsigned)jw) acc[jl] = __dadd_rn(acc[jl], __dmul_rn(av[u], vals[t]));
            }
            __syncwarp();
          }
        }
      }
      // c_i = sum_r a_ri b_r in increasing r (lane 0, values already in registers)
      for (int q = 0; q < cnt && j0 == 0; ++q) {
        const double a = __shfl_sync(kFull, my_a, q);
        const double bb = __shfl_sync(kFull, my_b, q);
        const int lo = __shfl_sync(kFull, my_lo, q), hi = __shfl_sync(kFull, my_hi, q);
        if (lane == 0 && hi > lo) ci = __dadd_rn(ci, __dmul_rn(a, bb));
      }
    }
    if (lane == 0 && j0 == 0) c[i] = ci;
    // ldg > 0: full row i (stride ldg); ldg <= 0: packed lower triangle, row
    // i = entries j <= i at offset i(i+1)/2 (the row-shard all-reduce buffer)
    double* Gi = (ldg > 0 ? G + (size_t)i * ldg : G + (size_t)i * (i + 1) / 2) + j0;
    const int jst = ldg > 0 ? jw : max(0, min(jw, i + 1 - j0));
    for (int j = lane; j < jw; j += 32) {
      if (j < jst) Gi[j] = acc[j];
      acc[j] = 0.0;
    }
    __syncwarp();
  }
}

// Exact-arithmetic Gram: when every product a_ri a_rj and every partial sum
// of a column is exactly representable (gram_is_exact: the inputs' exponent
// range and the longest column bound the bits; BASELINE's 2^-12-quantized
// inputs qualify), the sum order cannot change a single bit, so a CTA per G
// row scatters ALL contributing A rows at once (flat over their entries, all
// loads in flight) with shared-memory atomics.  Bit-identical to the ordered
// kernel above and to the oracle, without its per-row dependent chain.
constexpr int kExactTuples = 512;  // longest column handled by gram_exact_kernel
__global__ void __launch_bounds__(512) gram_exact_kernel(
    int n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
    const double* __restrict__ vals, const int32_t* __restrict__ colptr,
    const int32_t* __restrict__ rowind, const double* __restrict__ cvals,
    const double* __restrict__ b, int row_begin, int row_end, double* __restrict__ G, int ldg,
    double* __restrict__ c, double scale, double inv_scale) {
  pdl_wait();
  // Every product a_ri a_rj is an integer multiple of 2^(2 L_A) (L_A: the
  // lowest set bit over A) and every column sum stays below 2^53 units, so
  // the accumulator holds exact 64-bit integers (product * scale), kept as
  // two 32-bit words updated with the native shared-memory 32-bit atomics
  // (FP64 and 64-bit ones are CAS loops on sm_100): the low word's add
  // returns the old value, and the thread whose add wrapped carries into the
  // high word -- exact two's-complement arithmetic mod 2^64.
  // Warp w scatters the contributing rows q = w, w+16, ... (lanes = the row's
  // entries); the (a_ri, row start, length) tuples of the CTA's NEXT G row are
  // loaded into registers while the current one is scattered.
  extern __shared__ unsigned acc_w[];  // [lo words n][hi words n]
  __shared__ double s_a[kExactTuples];
  __shared__ int s_lo[kExactTuples], s_len[kExactTuples];
  __shared__ double s_c[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nt = blockDim.x, nw = nt >> 5;
  unsigned* acc_lo = acc_w;
  int* acc_hi = reinterpret_cast<int*>(acc_w + n);
  // tuple of entry tid of column i -> registers (len 0: outside the shard / none)
  auto load_tuple = [&](int i, double& a, int& lo, int& len, double& cp) {
    a = 0.0;
    lo = 0;
    len = 0;
    cp = 0.0;
    if (i >= n) return;
    const int e0 = colptr[i], cnt = colptr[i + 1] - e0;  // cnt <= kExactTuples (host-checked)
    if (tid < cnt) {
      const int r = rowind[e0 + tid];
      a = cvals[e0 + tid];
      if (r >= row_begin && r < row_end) {
        lo = rowptr[r];
        len = rowptr[r + 1] - lo;
        cp = a * b[r];
      }
    }
  };
  double ta, tcp;
  int tlo, tlen;
  load_tuple(blockIdx.x, ta, tlo, tlen, tcp);
  for (int i = blockIdx.x; i < n; i += gridDim.x) {
    for (int j = tid; j < n; j += nt) {
      acc_lo[j] = 0u;
      acc_hi[j] = 0;
    }
    if (tid < kExactTuples) {
      s_a[tid] = ta;
      s_lo[tid] = tlo;
      s_len[tid] = tlen;
    }
    const int cnt = colptr[i + 1] - colptr[i];
    double cp = warp_sum(tcp);  // c_i (exact: any order)
    if (lane == 0) s_c[wid] = cp;
    __syncthreads();
    if (wid == 0) {
      double cv = lane < nw ? s_c[lane] : 0.0;
      cv = warp_sum(cv);
      if (lane == 0) c[i] = cv;
    }
    load_tuple(i + gridDim.x, ta, tlo, tlen, tcp);  // next G row's tuples, in flight meanwhile
    // scatter: warp per contributing row, two rows per pass (loads in flight together)
    for (int q = wid; q < cnt; q += 2 * nw) {
      const int q2 = q + nw;
      const double a1 = s_a[q], a2 = q2 < cnt ? s_a[q2] : 0.0;
      const int lo1 = s_lo[q], len1 = s_len[q];
      const int lo2 = q2 < cnt ? s_lo[q2] : 0, len2 = q2 < cnt ? s_len[q2] : 0;
      const int mx = max(len1, len2);
      for (int t = lane; t < mx; t += 32) {
        int j1 = -1, j2 = -1;
        double v1 = 0.0, v2 = 0.0;
        if (t < len1) {
          j1 = colind[lo1 + t];
          v1 = vals[lo1 + t];
        }
        if (t < len2) {
          j2 = colind[lo2 + t];
          v2 = vals[lo2 + t];
        }
        if (j1 >= 0) {
          const long long v = __double2ll_rn((a1 * v1) * scale);  // exact integer
          const unsigned vlo = (unsigned)v;
          const unsigned old = atomicAdd(&acc_lo[j1], vlo);
          const int vhi = (int)(v >> 32) + ((old + vlo < old) ? 1 : 0);
          if (vhi != 0) atomicAdd(&acc_hi[j1], vhi);
        }
        if (j2 >= 0) {
          const long long v = __double2ll_rn((a2 * v2) * scale);
          const unsigned vlo = (unsigned)v;
          const unsigned old = atomicAdd(&acc_lo[j2], vlo);
          const int vhi = (int)(v >> 32) + ((old + vlo < old) ? 1 : 0);
          if (vhi != 0) atomicAdd(&acc_hi[j2], vhi);
        }
      }
    }
    __syncthreads();
    double* Gi = ldg > 0 ? G + (size_t)i * ldg : G + (size_t)i * (i + 1) / 2;  // (packed: j <= i)
    const int jn = ldg > 0 ? n : i + 1;
    for (int j = tid; j < jn; j += nt)
      Gi[j] = (double)(long long)(((unsigned long long)(unsigned)acc_hi[j] << 32) | acc_lo[j]) * inv_scale;
    __syncthreads();
  }
}

// Row-ordered Gram for general (inexact) values with the whole CTA on one G
// row: the ordered kernel above keeps ONE warp per G row (its accumulator row
// is n doubles of shared memory), so at n = 8000 three warps per SM wait on
// the A-row gathers.  Here a CTA owns G row i; its 16 warps take 16
// consecutive contributing A rows r (a batch, in increasing r), one row per
// warp, all gathers in flight together and the next batch's issued before
// this one is applied.  The oracle's order only matters between products
// that land on the SAME j, so the batch's (j, a_ri a_rj) tuples -- tuple
// index = (row slot, entry), the oracle's order -- are applied in passes:
// every pending tuple claims tag[j] with a 32-bit shared-memory atomicMax of
// (epoch, -index); after a barrier the claim's winner (the earliest pending
// tuple of that j) adds its product, the others stay pending for the next
// pass.  Distinct j's proceed in parallel, equal j's in increasing row order:
// every G_ij sees the oracle's terms, order and roundings (separate multiply
// and add), bit for bit.  At config 2 a batch holds ~640 tuples over 8000
// accumulators: ~4 % of them wait a pass (the diagonal j = i, present in
// every contributing row, is summed apart by one thread).  Host-selected when the longest row
// fits a warp's two to four entries per lane (128); a column longer than the
// tuple stage (kExactTuples) is taken in segments; c_i is summed in increasing r by the last thread,
// 16 terms per batch.
constexpr int kClaimRowMax = 128;
#ifndef NNLS_CLAIM_EPOCH_MAX  // (a small value exercises the restart in tests: NNLS_EXTRA_NVCC_FLAGS)
#define NNLS_CLAIM_EPOCH_MAX ((1 << 20) - 1024)
#endif
constexpr int kClaimEpochMax = NNLS_CLAIM_EPOCH_MAX;
template <int H>  // entries per lane: rows of up to 32 H entries
__global__ void __launch_bounds__(512) gram_claim_kernel(
    int n, const int32_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
    const double* __restrict__ vals, const int32_t* __restrict__ colptr,
    const int32_t* __restrict__ rowind, const double* __restrict__ cvals,
    const double* __restrict__ b, int row_begin, int row_end, double* __restrict__ G, int ldg,
    double* __restrict__ c) {
  pdl_wait();
  extern __shared__ double acc[];  // [n] accumulators, then [n] int tags
  int* tag = reinterpret_cast<int*>(acc + n);
  __shared__ double s_a[kExactTuples], s_cp[kExactTuples];
  __shared__ int s_lo[kExactTuples], s_len[kExactTuples];
  __shared__ double s_dg[16];  // the batch's diagonal products a_ri^2, by row slot
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nt = blockDim.x, nw = nt >> 5;
  for (int j = tid; j < n; j += nt) tag[j] = 0;
  int epoch = 0;
  // tuple of entry sb + tid of column i (a column longer than the stage is
  // taken in segments of kExactTuples entries: sb = the segment's start)
  auto load_tuple = [&](int i, int sb, double& a, int& lo, int& len, double& cp) {
    a = 0.0;
    lo = 0;
    len = 0;
    cp = 0.0;
    if (i >= n) return;
    const int e0 = colptr[i] + sb, cnt = colptr[i + 1] - e0;
    if (tid < cnt && tid < kExactTuples) {
      const int r = rowind[e0 + tid];
      a = cvals[e0 + tid];
      if (r >= row_begin && r < row_end) {
        lo = rowptr[r];
        len = rowptr[r + 1] - lo;  // <= 32 H (host-checked)
        cp = __dmul_rn(a, b[r]);
      }
    }
  };
  double ta, tcp;
  int tlo, tlen;
  load_tuple(blockIdx.x, 0, ta, tlo, tlen, tcp);
  double ci = 0.0, di = 0.0;
  for (int i = blockIdx.x, sb = 0; i < n;) {
    if (sb == 0) {
      for (int j = tid; j < n; j += nt) acc[j] = 0.0;
      ci = 0.0;
      di = 0.0;
    }
    // a stage takes at most 32 batches x 16 passes = 512 epochs: restart them
    // (uniform; the staging barrier below orders it) before the keys' epoch
    // field (20 bits at H >= 3) could overflow on very long columns
    if (epoch > kClaimEpochMax) {
      for (int j = tid; j < n; j += nt) tag[j] = 0;
      epoch = 0;
    }
    if (tid < kExactTuples) {
      s_a[tid] = ta;
      s_lo[tid] = tlo;
      s_len[tid] = tlen;
      s_cp[tid] = tcp;
    }
    const int cnt_all = colptr[i + 1] - colptr[i];
    const int cnt = min(kExactTuples, cnt_all - sb);
    const bool last_seg = sb + kExactTuples >= cnt_all;
    const int i_next = last_seg ? i + (int)gridDim.x : i, sb_next = last_seg ? 0 : sb + kExactTuples;
    __syncthreads();
    load_tuple(i_next, sb_next, ta, tlo, tlen, tcp);  // the next stage's tuples, in flight meanwhile
    // the warp's row of a batch: entries lane + 32 h -> (j, a_ri a_rj)
    auto load_row = [&](int q, int (&j)[H], double (&p)[H], double& a) {
#pragma unroll
      for (int h = 0; h < H; ++h) {
        j[h] = -1;
        p[h] = 0.0;
      }
      a = 0.0;
      if (q >= cnt) return;
      a = s_a[q];
      const int lo = s_lo[q], len = s_len[q];
#pragma unroll
      for (int h = 0; h < H; ++h) {
        const int t = lane + 32 * h;
        if (t < len) {
          j[h] = colind[lo + t];
          p[h] = vals[lo + t];  // (multiplied by a_ri at use: the gathers stay in flight over a batch)
        }
      }
    };
    int jn[H];
    double pn[H];
    double an;
    load_row(wid, jn, pn, an);
    for (int q0 = 0; q0 < cnt; q0 += nw) {
      int jc[H];
      double pc[H];
      bool pend[H];
#pragma unroll
      for (int h = 0; h < H; ++h) {
        jc[h] = jn[h];
        pc[h] = __dmul_rn(an, pn[h]);
        pend[h] = jc[h] >= 0;
        // j = i: EVERY contributing row has it (G_ii = sum a_ri^2), so the
        // claims would serialise the whole batch; summed by one thread instead
        if (jc[h] == i) {
          s_dg[wid] = pc[h];
          pend[h] = false;
        }
      }
      if (lane == 0 && jc[0] < 0) s_dg[wid] = 0.0;  // no row in this slot (or outside the shard)
      load_row(q0 + nw + wid, jn, pn, an);
      // c_i = sum_r a_ri b_r in increasing r: the batch's 16 terms loaded together,
      // then the dependent adds (slots past the column's end and rows outside
      // the shard hold +0.0: x + 0.0 = x, a running sum from +0.0 is never -0.0)
      if (tid == nt - 1) {
        double t[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) t[u] = s_cp[min(q0 + u, kExactTuples - 1)];
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (q0 + u < kExactTuples) ci = __dadd_rn(ci, t[u]);
      }
      // tuple index (row slot, entry) = wid * 32 H + 32 h + lane; earlier tuple -> larger key
      const int low = (16 * 32 * H - 1) - (wid * 32 * H + lane);
      constexpr int kShift = H <= 2 ? 10 : 11;  // 16 * 32 * H keys
      int any;
      bool first = true;
      do {
        ++epoch;
        const int kb = (epoch << kShift) | low;
#pragma unroll
        for (int h = 0; h < H; ++h)
          if (pend[h]) atomicMax(&tag[jc[h]], kb - 32 * h);
        __syncthreads();
        if (first && tid == nt - 33) {  // G_ii in increasing r (row slots without the column: +0.0)
          double t[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) t[u] = s_dg[u];
#pragma unroll
          for (int u = 0; u < 16; ++u) di = __dadd_rn(di, t[u]);
        }
        first = false;
        bool left = false;
#pragma unroll
        for (int h = 0; h < H; ++h) {
          if (pend[h] && tag[jc[h]] == kb - 32 * h) {
            acc[jc[h]] = __dadd_rn(acc[jc[h]], pc[h]);
            pend[h] = false;
          }
          left |= pend[h];
        }
        any = __syncthreads_or(left);
      } while (any);
    }
    if (last_seg) {
      if (tid == nt - 1) c[i] = ci;
      double* Gi = ldg > 0 ? G + (size_t)i * ldg : G + (size_t)i * (i + 1) / 2;  // (packed: j <= i)
      const int jn_ = ldg > 0 ? n : i + 1;
      for (int j = tid; j < jn_; j += nt)
        if (j != i) Gi[j] = acc[j];
      if (tid == nt - 33) Gi[i] = di;
    }
    __syncthreads();
    i = i_next;
    sb = sb_next;
  }
}

// Packed lower triangle (row i at offset i(i+1)/2, j <= i) -> full symmetric
// n x ldg matrix.  32 x 32 blocks (bi >= bj) through shared memory so both the
// lower block (row copy) and its mirror (transposed) are written coalesced.
__global__ void __launch_bounds__(256) gram_unpack_kernel(int n, const double* __restrict__ P,
                                                          double* __restrict__ G, int ldg) {
  __shared__ double t[32][33];
  const int nb = (n + 31) / 32;
  const long long nblk = (long long)nb * (nb + 1) / 2;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 row groups
  for (long long blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    // blk -> (bi, bj), bj <= bi, row-major over the lower block triangle
    int bi = (int)((sqrt(8.0 * (double)blk + 1.0) - 1.0) * 0.5);
    while ((long long)bi * (bi + 1) / 2 > blk) --bi;
    while ((long long)(bi + 1) * (bi + 2) / 2 <= blk) ++bi;
    const int bj = (int)(blk - (long long)bi * (bi + 1) / 2);
    for (int r = ty; r < 32; r += 8) {
      const int i = 32 * bi + r, j = 32 * bj + tx;
      double v = 0.0;
      if (i < n && j <= i) v = P[(size_t)i * (i + 1) / 2 + j];
      t[r][tx] = v;
      if (i < n && j < n && (bi != bj || j <= i)) G[(size_t)i * ldg + j] = v;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {  // mirror: G[j][i] = P(i, j) for the block's j rows
      const int j = 32 * bj + r, i = 32 * bi + tx;
      if (j < n && i < n && (bi != bj || i > j)) G[(size_t)j * ldg + i] = t[tx][r];
    }
    __syncthreads();
  }
}

cudaError_t launch_gram_unpack(int n, const double* P, double* G, int ldg, int sm_count, cudaStream_t s) {
  const int nb = (n + 31) / 32;
  long long blocks = (long long)nb * (nb + 1) / 2;
  if (blocks > (long long)sm_count * 8) blocks = (long long)sm_count * 8;
  if (blocks < 1) blocks = 1;
  gram_unpack_kernel<<<(int)blocks, 256, 0, s>>>(n, P, G, ldg);
  return cudaGetLastError();
}

bool gram_is_exact(const int* err) { return err[2] <= kExactTuples && gram_bits_exact(err); }

// every product a_ri a_rj and every column partial sum exact in FP64 (the
// bit budget alone, any kernel / summation order)
bool gram_bits_exact(const int* err) { return gram_A_exact(err) && gram_c_exact(err); }

// A^T A alone: every product a_ri a_rj and every column partial sum exact
bool gram_A_exact(const int* err) {
  const int K = err[2];  // longest column
  const int hA = err[kErrExp], lA = err[kErrExp + 1];
  if (lA >= 4095) return false;
  if (hA == 0) return true;  // A == 0
  int lgK = 0;
  while ((1 << lgK) < K + 1) ++lgK;
  const int HA = hA - 2048, LA = 2048 - lA;
  // sum of K products |a a'| < 2^(2HA+2+lgK) must stay below 2^(53 + 2LA)
  if (2 * HA + 2 + lgK > 53 + 2 * LA) return false;
  if (2 * LA < -1000 || 2 * HA > 1000) return false;  // (the integer scale must stay a normal double)
  return true;
}

// A^T b: every product a_ri b_r and partial sum exact
bool gram_c_exact(const int* err) {
  const int K = err[2];
  const int hA = err[kErrExp], lA = err[kErrExp + 1], hb = err[kErrExp + 2], lb = err[kErrExp + 3];
  if (lA >= 4095 || lb >= 4095) return false;
  if (hA == 0 || hb == 0) return true;  // A == 0 or b == 0
  int lgK = 0;
  while ((1 << lgK) < K + 1) ++lgK;
  const int HA = hA - 2048, LA = 2048 - lA, Hb = hb - 2048, Lb = 2048 - lb;
  return HA + Hb + 2 + lgK <= 53 + LA + Lb;
}

cudaError_t launch_gram(int m, int n, const int32_t* rowptr, const int32_t* colind,
                        const double* vals, const int32_t* colptr, const int32_t* rowind,
                        const double* cvals, const double* b, int row_begin, int row_end,
                        double* G, int ldg, double* c, int sm_count, cudaStream_t s, bool exact,
                        int exact_lmin, int max_row, int max_col) {
  (void)m;
  if (exact && (size_t)n * sizeof(double) <= 160 * 1024) {
    static DeviceOnce attr_x;
    cudaError_t ea = cudaSuccess;
    if (!device_once(attr_x, [&]() {
          ea = cudaFuncSetAttribute(gram_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(160 * 1024));
          return ea == cudaSuccess ? 1 : 0;
        }))
      return ea;
    const size_t smem = sizeof(double) * (size_t)n;
    int per_sm = (int)((224 * 1024) / (smem + 9 * 1024));  // (8.3 KB static per CTA)
    if (per_sm > 4) per_sm = 4;
    if (per_sm < 1) per_sm = 1;
    long long blocks = (long long)sm_count * per_sm;
    if (blocks > n) blocks = n;
    const double sc = ldexp(1.0, -2 * exact_lmin);
    return launch_pdl(gram_exact_kernel, dim3((int)blocks), dim3(512), smem, s, n, rowptr, colind, vals, colptr,
                      rowind, cvals, b, row_begin, row_end, G, ldg, c, sc, 1.0 / sc);
  }
  // general values: a CTA per G row with claim-ordered batches when the rows
  // and columns fit its stages (max_row / max_col = 0: unknown -> not taken)
  if (!exact && max_row > 0 && max_row <= kClaimRowMax && max_col > 0 &&
      (size_t)n * 12 <= 200 * 1024) {
    const int H = max_row <= 64 ? 2 : (max_row <= 96 ? 3 : 4);
    auto kern = H == 2 ? gram_claim_kernel<2> : (H == 3 ? gram_claim_kernel<3> : gram_claim_kernel<4>);
    static DeviceOnce attr_c[3];
    cudaError_t ea = cudaSuccess;
    if (!device_once(attr_c[H - 2], [&]() {
          ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(200 * 1024));
          return ea == cudaSuccess ? 1 : 0;
        }))
      return ea;
    const size_t smem = 12 * (size_t)n;
    int per_sm = (int)((224 * 1024) / (smem + 13 * 1024));  // (12.3 KB static per CTA)
    if (per_sm > 4) per_sm = 4;
    if (per_sm < 1) per_sm = 1;
    long long blocks = (long long)sm_count * per_sm;
    if (blocks > n) blocks = n;
    return launch_pdl(kern, dim3((int)blocks), dim3(512), smem, s, n, rowptr, colind, vals, colptr, rowind, cvals,
                      b, row_begin, row_end, G, ldg, c);
  }
  // One chunk = the whole row when it fits (measured: splitting a row into
  // column chunks multiplies the A-row gathers and is slower at config 2).
  const int chunk = n < 1 ? 1 : (n <= 25600 ? n : 25600);
  int wpb = (int)((200 * 1024) / (sizeof(double) * (size_t)chunk));
  if (wpb > 8) wpb = 8;
  if (wpb < 1) wpb = 1;
  const size_t smem = sizeof(double) * (size_t)chunk * wpb;
  static DeviceOnce attr;  // once per device, at the maximum (a driver round trip per call otherwise)
  cudaError_t ea = cudaSuccess;
  if (!device_once(attr, [&]() {
        ea = cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(200 * 1024));
        return ea == cudaSuccess ? 1 : 0;
      }))
    return ea;
  int per_sm = (int)(220 * 1024 / (smem + 1024));
  if (per_sm < 1) per_sm = 1;
  if (per_sm * wpb > 16) per_sm = 16 / wpb;  // ~126 registers: at most 16 warps per SM
  if (per_sm < 1) per_sm = 1;
  const long long items = (long long)n * ((n + chunk - 1) / chunk);
  long long blocks = (items + wpb - 1) / wpb;
  if (blocks > (long long)sm_count * per_sm) blocks = (long long)sm_count * per_sm;
  if (blocks < 1) blocks = 1;
  gram_kernel<<<(int)blocks, wpb * 32, smem, s>>>(n, rowptr, colind, vals, colptr, rowind, cvals, b,
                                                 row_begin, row_end, G, ldg, c, chunk);
  return cudaGetLastError();
}

}  // namespace nnls
