// kernels.cu — sm_100a kernels of libsexpm (fp64 CUDA cores; no tensor cores: the
// work is a sparse Gustavson product, not a dense contraction).
//
// PAPER.md citations: P:<line>.  Kernel ids follow SURVEY.md §2.3 / DESIGN.md:
//   K8 norms/validation (plan, P:392 needs ||H||), K1 symbolic row bound (Lemma 3.1,
//   P:96-128), K2 binning, K3 numeric SpGEMM + fused 2T add + filter classification
//   (Eq. 2.7, Eq. 4.15, Eq. 4.11), K6 Algorithm 4.1 pass,
//   K4 compaction ("A~ = A - b_n"), merge T^_0 += S^_i and I + T.
#include <math.h>
#include <algorithm>
#include <stdint.h>

#include <cub/cub.cuh>

#include "kernels.cuh"

namespace sx {

std::atomic<long long> g_kernel_launches{0};  // kernels enqueued (reported as gpu_launches)
#define KL (++g_kernel_launches)

#define FULL_MASK 0xffffffffu

static inline int grid_for(int64_t items, int per_block, int cap = 1 << 30) {
  int64_t g = (items + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (int)g;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(FULL_MASK, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_down_sync(FULL_MASK, v, o);
    v = w > v ? w : v;
  }
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_min(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    T w = __shfl_down_sync(FULL_MASK, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// ------------------------------------------------------------------------------------
// K8: validation and transpose-based norm / symmetry (plan time)
// ------------------------------------------------------------------------------------
// flags[0] bits: 1 bad rowptr, 2 column out of range, 4 columns not strictly increasing,
// 8 non-finite value.
__global__ void k_validate(CsrView A, int64_t n, int *flags) {
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (w >= A.nrows) return;
  int64_t p0 = A.rp[w], p1 = A.rp[w + 1];
  int f = 0;
  if (p1 < p0 || p0 < 0 || p1 > A.nnz) f |= 1;
  else {
    for (int64_t p = p0 + lane; p < p1; p += 32) {
      int32_t c = A.col[p];
      if (c < 0 || c >= n) f |= 2;
      if (p > p0 && A.col[p - 1] >= c) f |= 4;
      if (!isfinite(A.val[p])) f |= 8;
    }
  }
  f = __reduce_or_sync(FULL_MASK, f);
  if (lane == 0 && f) atomicOr(flags, f);
}
void launch_validate(const CsrView &A, int64_t n, int *flags, cudaStream_t st) {
  if (A.nrows == 0) return;
  KL;
  k_validate<<<grid_for(A.nrows * 32, kThreads), kThreads, 0, st>>>(A, n, flags);
}

__global__ void k_col_count(CsrView A, int32_t *cnt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < A.nnz; i += stride) atomicAdd(&cnt[A.col[i]], 1);
}
void launch_col_count(const CsrView &A, int32_t *cnt, cudaStream_t st) {
  if (A.nnz == 0) return;
  KL;
  k_col_count<<<grid_for(A.nnz, kThreads, 148 * 16), kThreads, 0, st>>>(A, cnt);
}

__global__ void k_transpose_fill(CsrView A, unsigned long long *cursor, int32_t *trow,
                                 double *tval) {
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (w >= A.nrows) return;
  for (int64_t p = A.rp[w] + lane; p < A.rp[w + 1]; p += 32) {
    unsigned long long pos = atomicAdd(&cursor[A.col[p]], 1ull);
    trow[pos] = (int32_t)(A.row0 + w);
    tval[pos] = A.val[p];
  }
}
void launch_transpose_fill(const CsrView &A, int64_t *cursor, int32_t *trow, double *tval,
                           cudaStream_t st) {
  if (A.nrows == 0) return;
  KL;
  k_transpose_fill<<<grid_for(A.nrows * 32, kThreads), kThreads, 0, st>>>(
      A, reinterpret_cast<unsigned long long *>(cursor), trow, tval);
}

// insertion sort of each column segment by row (columns of sparse H are short)
__global__ void k_sort_columns(int64_t ncols, const int64_t *cp, int32_t *trow, double *tval) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ncols) return;
  int64_t a = cp[j], b = cp[j + 1];
  for (int64_t p = a + 1; p < b; p++) {
    int32_t r = trow[p];
    double v = tval[p];
    int64_t q = p - 1;
    while (q >= a && trow[q] > r) {
      trow[q + 1] = trow[q];
      tval[q + 1] = tval[q];
      q--;
    }
    trow[q + 1] = r;
    tval[q + 1] = v;
  }
}
void launch_sort_columns(int64_t ncols, const int64_t *cp, int32_t *trow, double *tval,
                         cudaStream_t st) {
  if (ncols == 0) return;
  KL;
  k_sort_columns<<<grid_for(ncols, kThreads), kThreads, 0, st>>>(ncols, cp, trow, tval);
}

// column j: sum_i |h_ij| in ascending row order (the row-major order of the definition)
__global__ void k_col_abs_sum(int64_t ncols, const int64_t *cp, const double *tval,
                              double *out) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= ncols) return;
  double s = 0.0;
  for (int64_t p = cp[j]; p < cp[j + 1]; p++) s = s + fabs(tval[p]);
  out[j] = s;
}
void launch_col_abs_sum(int64_t ncols, const int64_t *cp, const double *tval, double *out,
                        cudaStream_t st) {
  if (ncols == 0) return;
  KL;
  k_col_abs_sum<<<grid_for(ncols, kThreads), kThreads, 0, st>>>(ncols, cp, tval, out);
}

// flags bit 1: H != H^T, bit 2: H != -H^T (bit-exact; A must hold all rows)
__global__ void k_compare_transpose(CsrView A, const int64_t *cp, const int32_t *trow,
                                    const double *tval, int *flags) {
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (w >= A.nrows) return;
  int64_t r = A.row0 + w;
  int64_t p0 = A.rp[w], p1 = A.rp[w + 1];
  int64_t q0 = cp[r], q1 = cp[r + 1];
  int f = 0;
  if (p1 - p0 != q1 - q0) f = 3;
  else {
    for (int64_t t = lane; t < p1 - p0; t += 32) {
      if (A.col[p0 + t] != trow[q0 + t]) f |= 3;
      if (A.val[p0 + t] != tval[q0 + t]) f |= 1;
      if (A.val[p0 + t] != -tval[q0 + t]) f |= 2;
    }
  }
  f = __reduce_or_sync(FULL_MASK, f);
  if (lane == 0 && f) atomicOr(flags, f);
}
void launch_compare_transpose(const CsrView &A, const int64_t *cp, const int32_t *trow,
                              const double *tval, int *flags, cudaStream_t st) {
  if (A.nrows == 0) return;
  KL;
  k_compare_transpose<<<grid_for(A.nrows * 32, kThreads), kThreads, 0, st>>>(A, cp, trow,
                                                                             tval, flags);
}

// ------------------------------------------------------------------------------------
// Deterministic reductions: fixed grid of kRedBlocks CTAs over contiguous chunks, a
// fixed thread-stride order inside each chunk, a fixed tree, then one CTA over partials.
// ------------------------------------------------------------------------------------
constexpr int kRedBlocks = 592;  // 4 x 148 SMs

enum RedOp { RED_SUM = 0, RED_SUMSQ = 1, RED_MAX = 2, RED_SUMSQ_LE = 3 };

template <int OP>
__device__ __forceinline__ double red_map(double x, double tau) {
  if (OP == RED_SUMSQ) return x * x;
  if (OP == RED_SUMSQ_LE) return fabs(x) <= tau ? x * x : 0.0;
  return x;
}
template <int OP>
__device__ __forceinline__ double red_comb(double a, double b) {
  return OP == RED_MAX ? (a > b ? a : b) : a + b;
}

template <int OP>
__device__ double block_reduce(double v) {
  __shared__ double s[kWarps];
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = red_comb<OP>(v, __shfl_down_sync(FULL_MASK, v, o));
  if (lane == 0) s[warp] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x == 0) {
    r = s[0];
    for (int w = 1; w < kWarps; w++) r = red_comb<OP>(r, s[w]);
  }
  __syncthreads();
  return r;
}

template <int OP>
__global__ void k_reduce_partial(const double *x, int64_t cnt, double tau, double *partial) {
  int64_t chunk = (cnt + gridDim.x - 1) / gridDim.x;
  int64_t a = (int64_t)blockIdx.x * chunk;
  int64_t b = a + chunk < cnt ? a + chunk : cnt;
  double v = OP == RED_MAX ? -INFINITY : 0.0;
  for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x)
    v = red_comb<OP>(v, red_map<OP>(x[i], tau));
  double r = block_reduce<OP>(v);
  if (threadIdx.x == 0) partial[blockIdx.x] = r;
}
template <int OP>
__global__ void k_reduce_final(const double *partial, int np, double *out) {
  double v = OP == RED_MAX ? -INFINITY : 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) v = red_comb<OP>(v, partial[i]);
  double r = block_reduce<OP == RED_MAX ? RED_MAX : RED_SUM>(v);
  if (threadIdx.x == 0) out[0] = (OP == RED_MAX && np == 0) ? 0.0 : r;
}
template <int OP>
static void reduce_impl(const double *x, int64_t cnt, double tau, double *partial, double *out,
                        cudaStream_t st) {
  KL;
  k_reduce_partial<OP><<<kRedBlocks, kThreads, 0, st>>>(x, cnt, tau, partial);
  KL;
  k_reduce_final<OP><<<1, kThreads, 0, st>>>(partial, kRedBlocks, out);
}
void launch_reduce_max(const double *x, int64_t cnt, double *partial, double *out,
                       cudaStream_t st) {
  reduce_impl<RED_MAX>(x, cnt, 0.0, partial, out, st);
}
void launch_reduce_sumsq(const double *x, int64_t cnt, double *partial, double *out,
                         cudaStream_t st) {
  reduce_impl<RED_SUMSQ>(x, cnt, 0.0, partial, out, st);
}
void launch_reduce_sum(const double *x, int64_t cnt, double *partial, double *out,
                       cudaStream_t st) {
  reduce_impl<RED_SUM>(x, cnt, 0.0, partial, out, st);
}
// K6: one pass of Algorithm 4.1 over the staged values: sum of x^2 with |x| <= tau
void launch_alg41_pass(const double *x, int64_t cnt, double tau, double *partial, double *out,
                       cudaStream_t st) {
  reduce_impl<RED_SUMSQ_LE>(x, cnt, tau, partial, out, st);
}

// integer sum / max (max over non-negative values, 0 for an empty range): grid-stride,
// one 64-bit atomic per CTA (integer arithmetic: exact in any order)
// K6 by rows: per-row sum of x^2 over the row's staged values with |x| <= tau (lanes in a
// fixed stride, fixed warp tree), then a fixed-order reduction over rows.  The staged
// rows are in column order whatever order the product kernel processed them in, so the
// pass sums -- and Algorithm 4.1's thresholds -- are identical from run to run.
__global__ void k_alg41_rows(int64_t nrows, const int64_t *row_off, const int64_t *row_cnt,
                             const double *pool_val, double tau, double *out) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nrows) return;
  const int64_t o = row_off[w], c = row_cnt[w];
  double s = 0.0;
  for (int64_t t = lane; t < c; t += 32) {
    const double x = pool_val[o + t];
    if (fabs(x) <= tau) s += x * x;
  }
  s = warp_sum(s);
  if (lane == 0) out[w] = s;
}
void launch_alg41_pass_rows(int64_t nrows, const int64_t *row_off, const int64_t *row_cnt,
                            const double *pool_val, double tau, double *rowsum, double *partial,
                            double *out, cudaStream_t st) {
  if (nrows == 0) {
    cudaMemsetAsync(out, 0, sizeof(double), st);
    return;
  }
  KL;
  k_alg41_rows<<<grid_for(nrows * 32, kThreads), kThreads, 0, st>>>(nrows, row_off, row_cnt,
                                                                     pool_val, tau, rowsum);
  reduce_impl<RED_SUM>(rowsum, nrows, 0.0, partial, out, st);
}

__global__ void k_reduce_i64(const int64_t *x, int64_t cnt, int64_t *out, int is_max) {
  __shared__ long long s[kWarps];
  long long v = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    long long y = x[i];
    v = is_max ? (y > v ? y : v) : v + y;
  }
  v = is_max ? warp_max(v) : warp_sum(v);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long r = 0;
    for (int w = 0; w < kWarps; w++) r = is_max ? (s[w] > r ? s[w] : r) : r + s[w];
    if (is_max) atomicMax(reinterpret_cast<unsigned long long *>(out), (unsigned long long)r);
    else atomicAdd(reinterpret_cast<unsigned long long *>(out), (unsigned long long)r);
  }
}
static void reduce_i64(const int64_t *x, int64_t cnt, int64_t *out, int is_max, cudaStream_t st) {
  cudaMemsetAsync(out, 0, sizeof(int64_t), st);
  if (cnt <= 0) return;
  KL;
  k_reduce_i64<<<grid_for(cnt, kThreads * 8, kRedBlocks), kThreads, 0, st>>>(x, cnt, out, is_max);
}
void launch_reduce_max_i64(const int64_t *x, int64_t cnt, int64_t *out, cudaStream_t st) {
  reduce_i64(x, cnt, out, 1, st);
}
void launch_reduce_sum_i64(const int64_t *x, int64_t cnt, int64_t *out, cudaStream_t st) {
  reduce_i64(x, cnt, out, 0, st);
}

__global__ void k_scale_pow2(double *v, int64_t cnt, int e) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < cnt; i += stride) v[i] = ldexp(v[i], e);
}
void launch_scale_pow2(double *v, int64_t cnt, int e, cudaStream_t st) {
  if (cnt == 0 || e == 0) return;
  KL;
  k_scale_pow2<<<grid_for(cnt, kThreads, 148 * 16), kThreads, 0, st>>>(v, cnt, e);
}

__global__ void k_rowlen_sq(const int64_t *rp, int64_t nrows, int64_t *out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < nrows) {
    const int64_t l = rp[r + 1] - rp[r];
    out[r] = l * l;
  }
}
void launch_rowlen_sq(const int64_t *rp, int64_t nrows, int64_t *out, cudaStream_t st) {
  if (nrows == 0) return;
  KL;
  k_rowlen_sq<<<grid_for(nrows, kThreads), kThreads, 0, st>>>(rp, nrows, out);
}
__global__ void k_row_lengths(const int64_t *rp, int64_t nrows, int64_t *out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nrows) out[i] = rp[i + 1] - rp[i];
}
void launch_row_lengths(const int64_t *rp, int64_t nrows, int64_t *out, cudaStream_t st) {
  if (nrows == 0) return;
  KL;
  k_row_lengths<<<grid_for(nrows, kThreads), kThreads, 0, st>>>(rp, nrows, out);
}

__global__ void k_i32_to_i64(const int32_t *in, int64_t cnt, int64_t *out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) out[i] = in[i];
}
__global__ void k_copy_i64_offset(const int64_t *src, int64_t cnt, int64_t off, int64_t *dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < cnt) dst[i] = src[i] + off;
}
void launch_copy_i64_offset(const int64_t *src, int64_t cnt, int64_t off, int64_t *dst,
                            cudaStream_t st) {
  if (cnt == 0) return;
  KL;
  k_copy_i64_offset<<<grid_for(cnt, kThreads), kThreads, 0, st>>>(src, cnt, off, dst);
}

// ------------------------------------------------------------------------------------
// Exclusive scan (reduce-then-scan, 3 kernels)
// ------------------------------------------------------------------------------------
constexpr int kScanItems = 8;
constexpr int kScanTile = kThreads * kScanItems;

int64_t scan_tmp_elems(int64_t cnt) { return (cnt + kScanTile - 1) / kScanTile + 1; }

__device__ long long block_excl_scan(long long v, long long *total) {
  __shared__ long long s[kWarps];
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long y = __shfl_up_sync(FULL_MASK, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s[warp] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long acc = 0;
    for (int w = 0; w < kWarps; w++) {
      long long t = s[w];
      s[w] = acc;
      acc += t;
    }
    *total = acc;
  }
  __syncthreads();
  long long r = x - v + s[warp];
  __syncthreads();
  return r;
}

__global__ void k_scan_tiles(const int64_t *in, int64_t cnt, int64_t *tile_sum) {
  int64_t base = (int64_t)blockIdx.x * kScanTile;
  long long v = 0;
  for (int k = 0; k < kScanItems; k++) {
    int64_t i = base + (int64_t)k * kThreads + threadIdx.x;
    if (i < cnt) v += in[i];
  }
  v = warp_sum(v);
  __shared__ long long s[kWarps];
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long t = 0;
    for (int w = 0; w < kWarps; w++) t += s[w];
    tile_sum[blockIdx.x] = t;
  }
}
__global__ void k_scan_tile_sums(int64_t *tile_sum, int64_t ntiles) {
  __shared__ long long total;
  long long carry = 0;
  for (int64_t b = 0; b < ntiles; b += kThreads) {
    int64_t i = b + threadIdx.x;
    long long v = i < ntiles ? tile_sum[i] : 0;
    long long e = block_excl_scan(v, &total);
    if (i < ntiles) tile_sum[i] = e + carry;
    carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) tile_sum[ntiles] = carry;
}
__global__ void k_scan_apply(const int64_t *in, int64_t cnt, const int64_t *tile_sum,
                             int64_t *out) {
  __shared__ long long total;
  int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
  long long loc[kScanItems];
  long long s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    int64_t i = base + k;
    loc[k] = i < cnt ? in[i] : 0;
    s += loc[k];
  }
  long long e = block_excl_scan(s, &total) + tile_sum[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; k++) {
    int64_t i = base + k;
    if (i < cnt) out[i] = e;
    e += loc[k];
  }
}
__global__ void k_scan_total(const int64_t *tile_sum, int64_t ntiles, int64_t cnt, int64_t *out) {
  out[cnt] = tile_sum[ntiles];
}
void launch_exclusive_scan(const int64_t *in, int64_t cnt, int64_t *out, int64_t *tmp,
                           cudaStream_t st) {
  int64_t ntiles = (cnt + kScanTile - 1) / kScanTile;
  if (ntiles > 0) {
    KL;
    k_scan_tiles<<<(int)ntiles, kThreads, 0, st>>>(in, cnt, tmp);
    KL;
    k_scan_tile_sums<<<1, kThreads, 0, st>>>(tmp, ntiles);
    KL;
    k_scan_apply<<<(int)ntiles, kThreads, 0, st>>>(in, cnt, tmp, out);
    KL;
    k_scan_total<<<1, 1, 0, st>>>(tmp, ntiles, cnt, out);
  } else {
    cudaMemsetAsync(out, 0, sizeof(int64_t), st);
  }
}

// ------------------------------------------------------------------------------------
// K1 symbolic row bound (warp per output row).  Lemma 3.1: the nonzeros of
// row r of A*B lie in [min_k first(B_k), max_k last(B_k)] for k in row r of A.
// ------------------------------------------------------------------------------------
__global__ void k_symbolic(CsrView A, CsrView B, int self, int32_t *lo, int32_t *hi,
                           int64_t *prod, int64_t *bound) {
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (w >= A.nrows) return;
  int64_t p0 = A.rp[w], p1 = A.rp[w + 1];
  int32_t l = INT32_MAX, h = -1;
  long long pr = 0;
  for (int64_t p = p0 + lane; p < p1; p += 32) {
    int64_t k = (int64_t)A.col[p] - B.row0;
    if (k < 0 || k >= B.nrows) continue;  // caller guarantees coverage (halo)
    int64_t s = B.rp[k], e = B.rp[k + 1];
    if (e > s) {
      int32_t f = B.col[s], g = B.col[e - 1];
      l = f < l ? f : l;
      h = g > h ? g : h;
      pr += e - s;
    }
  }
  if (self && p1 > p0) {
    if (lane == 0) {
      int32_t f = A.col[p0], g = A.col[p1 - 1];
      l = f < l ? f : l;
      h = g > h ? g : h;
      pr += p1 - p0;
    }
  }
  l = warp_min(l);
  h = warp_max(h);
  pr = warp_sum(pr);
  if (lane == 0) {
    lo[w] = l;
    hi[w] = h;
    prod[w] = pr;
    long long span = h >= l ? (long long)h - l + 1 : 0;
    bound[w] = span < pr ? span : pr;
  }
}
void launch_symbolic(const CsrView &A, const CsrView &B, int self, int32_t *lo, int32_t *hi,
                     int64_t *prod, int64_t *bound, cudaStream_t st) {
  if (A.nrows == 0) return;
  KL;
  k_symbolic<<<grid_for(A.nrows * 32, kThreads), kThreads, 0, st>>>(A, B, self, lo, hi, prod,
                                                                    bound);
}

// ------------------------------------------------------------------------------------
// K2 binning: rows ordered by descending work class (longest-processing-time first) so
// the dynamic row scheduler of K3 ends with short rows.
// ------------------------------------------------------------------------------------
constexpr int kBins = 64;
__device__ __forceinline__ int work_bin(long long w) {
  return 63 - (w > 0 ? (63 - __clzll((unsigned long long)w)) : 0);  // heavy -> small bin id
}
__global__ void k_bin_count(int64_t nrows, const int64_t *work, int32_t *bin_cnt) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nrows) atomicAdd(&bin_cnt[work_bin(work[i])], 1);
}
__global__ void k_bin_offsets(int32_t *bin_cnt, int32_t *bin_off) {
  if (threadIdx.x == 0) {
    int32_t s = 0;
    for (int b = 0; b < kBins; b++) {
      bin_off[b] = s;
      s += bin_cnt[b];
      bin_cnt[b] = 0;
    }
  }
}
__global__ void k_bin_scatter(int64_t nrows, const int64_t *work, int32_t *bin_cnt,
                              const int32_t *bin_off, int32_t *order) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nrows) {
    int b = work_bin(work[i]);
    int32_t pos = bin_off[b] + atomicAdd(&bin_cnt[b], 1);
    order[pos] = (int32_t)i;
  }
}
void launch_bin_rows(int64_t nrows, const int64_t *work, int32_t *bin_cnt, int32_t *bin_off,
                     int32_t *order, cudaStream_t st) {
  if (nrows == 0) return;
  cudaMemsetAsync(bin_cnt, 0, kBins * sizeof(int32_t), st);
  KL;
  k_bin_count<<<grid_for(nrows, kThreads), kThreads, 0, st>>>(nrows, work, bin_cnt);
  KL;
  k_bin_offsets<<<1, 32, 0, st>>>(bin_cnt, bin_off);
  KL;
  k_bin_scatter<<<grid_for(nrows, kThreads), kThreads, 0, st>>>(nrows, work, bin_cnt, bin_off,
                                                               order);
}

// ------------------------------------------------------------------------------------
// K3 numeric filtered SpGEMM (one CTA per output row, dynamic row scheduler).
//
//   C~(r,:) = (self_coef * A(r,:) + sum_{k in row r of A} a_rk * B(k,:)) / divisor
//
// Squaring (Eq. 2.7 P:76 / Eq. 4.15): A = B = T^_{i-1}, self_coef = 2, divisor = 1.
// Taylor term (Eq. 4.11, Alg. 4.2): A = S^_{i-1}, B = H0, self 0, divisor i.
//
// Accumulator: a dense shared-memory window over the row's reachable column span
// [lo, hi] (K1), processed in chunks of `window` columns; B rows are sorted, so each
// k keeps a cursor that only moves forward across chunks.  The 2T term is stored first
// (no other writer in that phase), products are added with shared-memory atomics
// (warps work on different k), and the flush fuses the filter classification of
// Algorithm 4.1: entries with |x| <= floor_tau = eps_g / sqrt(K) can never be kept
// (every threshold the algorithm visits is >= eps_g / sqrt(K), K >= #entries; see
// DESIGN.md "floor lemma"), so only their x^2 is kept (per-row partial sums); the
// others are staged (col, val) in column order for the passes (K6) and compaction (K4).
// ------------------------------------------------------------------------------------
int numeric_smem_bytes(int window) { return window * (int)sizeof(double); }

__global__ void __launch_bounds__(kThreads) k_numeric(NumericArgs a) {
  extern __shared__ double win[];
  __shared__ int s_row;
  __shared__ long long s_wcnt[kWarps];
  __shared__ long long s_base[kWarps + 1];
  __shared__ long long s_selfcur;
  __shared__ unsigned long long s_off;
  __shared__ double s_fs[kWarps];
  __shared__ long long s_nz[kWarps];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int W = a.window;
  for (int i = tid; i < W; i += kThreads) win[i] = 0.0;
  int64_t *cur = a.cursor + (int64_t)blockIdx.x * a.cursor_cap;
  int32_t *sc = a.scr_col + (int64_t)blockIdx.x * a.scr_cap;
  double *sv = a.scr_val + (int64_t)blockIdx.x * a.scr_cap;
  const double inv_div_flag = a.divisor;  // division (not reciprocal multiply), reading R7

  for (;;) {
    __syncthreads();
    if (tid == 0) s_row = atomicAdd(a.row_counter, 1);
    __syncthreads();
    const int idx = s_row;
    if (idx >= a.nlist) break;
    const int64_t r = a.order ? (int64_t)a.order[idx] : (int64_t)idx;
    const int32_t lo = a.lo[r], hi = a.hi[r];
    const int64_t pa0 = a.A.rp[r], pa1 = a.A.rp[r + 1];
    const int64_t nk = pa1 - pa0;
    if (hi < lo) {
      if (tid == 0) {
        a.row_off[r] = 0;
        a.row_cnt[r] = 0;
        a.row_fsum[r] = 0.0;
        a.row_nnz[r] = 0;
      }
      continue;
    }
    for (int64_t q = tid; q < nk; q += kThreads) {
      int64_t k = (int64_t)a.A.col[pa0 + q] - a.B.row0;
      cur[q] = (k >= 0 && k < a.B.nrows) ? a.B.rp[k] : -1;
    }
    if (tid == 0) s_selfcur = pa0;
    long long nst = 0;
    double fs = 0.0;
    long long nnzu = 0;
    __syncthreads();
    for (int64_t c0 = lo; c0 <= hi; c0 += W) {
      const int64_t c1 = (c0 + W < (int64_t)hi + 1) ? c0 + W : (int64_t)hi + 1;
      const int wlen = (int)(c1 - c0);
      if (a.self_coef != 0.0) {
        const long long sc0 = s_selfcur;
        long long done = 0;
        for (long long p = sc0 + tid;; p += kThreads) {
          bool v = p < pa1 && (int64_t)a.A.col[p] < c1;
          if (v) win[a.A.col[p] - c0] = a.self_coef * a.A.val[p];
          int cnt = __syncthreads_count(v);
          done += cnt;
          if (cnt < kThreads) break;
        }
        if (tid == 0) s_selfcur = sc0 + done;
        __syncthreads();
      }
      for (int64_t q = warp; q < nk; q += kWarps) {
        long long pos = cur[q];
        if (pos < 0) continue;
        const int64_t k = (int64_t)a.A.col[pa0 + q] - a.B.row0;
        const long long end = a.B.rp[k + 1];
        const double av = a.A.val[pa0 + q];
        for (;;) {
          long long p = pos + lane;
          bool v = false;
          int32_t c = 0;
          if (p < end) {
            c = a.B.col[p];
            v = (int64_t)c < c1;
          }
          if (v) {
            double prod = av * a.B.val[p];
            atomicAdd(&win[c - c0], prod);
          }
          int cnt = __popc(__ballot_sync(FULL_MASK, v));
          pos += cnt;
          if (cnt < 32) break;
        }
        if (lane == 0) cur[q] = pos;
      }
      __syncthreads();
      // flush, pass 1: staged count per warp sub-range
      const int per = (((wlen + kWarps - 1) / kWarps) + 31) & ~31;
      const int w0 = warp * per;
      const int w1 = (w0 + per < wlen) ? w0 + per : wlen;
      long long wc = 0;
      for (int base = w0; base < w1; base += 32) {
        int i = base + lane;
        bool st = false;
        if (i < w1) {
          double x = win[i] / inv_div_flag;
          st = (x != 0.0) && (fabs(x) > a.floor_tau);
        }
        wc += __popc(__ballot_sync(FULL_MASK, st));
      }
      if (lane == 0) s_wcnt[warp] = wc;
      __syncthreads();
      if (tid == 0) {
        long long s = 0;
        for (int w = 0; w < kWarps; w++) {
          s_base[w] = s;
          s += s_wcnt[w];
        }
        s_base[kWarps] = s;
      }
      __syncthreads();
      // pass 2: classify, stage in column order, reset the window
      long long o = nst + s_base[warp];
      for (int base = w0; base < w1; base += 32) {
        int i = base + lane;
        bool st = false;
        double x = 0.0;
        if (i < w1) {
          x = win[i] / inv_div_flag;
          win[i] = 0.0;
          if (x != 0.0) {
            nnzu++;
            st = fabs(x) > a.floor_tau;
            if (!st) fs += x * x;
          }
        }
        unsigned m = __ballot_sync(FULL_MASK, st);
        if (st) {
          long long pp = o + __popc(m & lanemask_lt());
          if (pp < a.scr_cap) {
            sc[pp] = (int32_t)(c0 + i);
            sv[pp] = x;
          }
        }
        o += __popc(m);
      }
      nst += s_base[kWarps];
      __syncthreads();
    }
    // per-row partials (deterministic tree)
    fs = warp_sum(fs);
    nnzu = warp_sum(nnzu);
    if (lane == 0) {
      s_fs[warp] = fs;
      s_nz[warp] = nnzu;
    }
    if (tid == 0) s_off = atomicAdd(a.pool_used, (unsigned long long)nst);
    __syncthreads();
    const unsigned long long off = s_off;
    const bool ok = (long long)off + nst <= a.pool_cap && nst <= a.scr_cap;
    if (ok) {
      for (long long t = tid; t < nst; t += kThreads) {
        a.pool_col[off + t] = sc[t];
        a.pool_val[off + t] = sv[t];
      }
    }
    if (tid == 0) {
      double f = 0.0;
      long long z = 0;
      for (int w = 0; w < kWarps; w++) {
        f += s_fs[w];
        z += s_nz[w];
      }
      if (!ok) atomicOr(a.flags, nst > a.scr_cap ? 2 : 1);
      a.row_off[r] = (int64_t)off;
      a.row_cnt[r] = nst;
      a.row_fsum[r] = f;
      a.row_nnz[r] = z;
    }
  }
}

void launch_numeric(const NumericArgs &a, cudaStream_t st) {
  if (a.A.nrows == 0 || a.nlist == 0) return;
  int smem = numeric_smem_bytes(a.window);
  cudaFuncSetAttribute(k_numeric, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  KL;
  k_numeric<<<a.grid, kThreads, smem, st>>>(a);
}


// ------------------------------------------------------------------------------------
// K3p numeric filtered SpGEMM: one CTA per output row, k-synchronous, PAGED accumulator.
//
// Accumulator: the row's reachable column span [lo, hi] (K1) is cut into pages of 2^s
// columns (s chosen so the span has <= kPages pages); a page gets 2^s value slots the
// first time any product lands in it (page-table CAS, rare), so a column maps to its slot
// with one shared-memory load and a shift -- no probing.  Pages are allocated in the
// order products arrive, but the flush walks the page table in column order, so the
// staged row comes out sorted without any sort.  Like K3k, the B rows are added one k at
// a time in ascending k with a barrier between k (one writer per slot, no atomics on
// values, exact oracle order with _rn intrinsics: C~ bit-identical to the oracle).
// Rows whose span needs pages wider than 64 columns or whose pages overflow kSlots are
// handed to the block-window kernel.
// ------------------------------------------------------------------------------------
constexpr int kMaxPageShift = 6;
// two configurations: (threads, entries per thread per k held in the prefetch ring, ring
// depth in k, slots, pages).  v1: 256 threads; v2: 128 threads with 4 entries each (the
// per-k bookkeeping is amortized over twice the entries) and a smaller footprint (more
// CTAs per SM).
template <int T, int NE, int PF, int SLOTS, int PAGES, typename PT = int32_t, int MINSH = 4>
struct PagedCfg {
  static constexpr int kT = T, kW = T / 32, kNE = NE, kPF = PF, kSlots = SLOTS, kPages = PAGES;
  static constexpr int kMinShift = MINSH;
  using PageT = PT;  // page-table entry: slot base, -1 free, -2 being claimed, -3 overflow
  static constexpr int smem() {
    return SLOTS * 8 + ((PAGES * (int)sizeof(PT) + 7) / 8) * 8 + (SLOTS >> MINSH) * 4;
  }
};
using PagedV1 = PagedCfg<256, 2, 8, 4096, 4096>;
int paged_smem_bytes() { return PagedV1::smem(); }

__device__ __forceinline__ int page_slot(volatile int32_t *ptab, int pg, int psize, int *slot_count,
                                         int slot_cap) {
  int b = ptab[pg];
  if (b >= 0) return b;
  if (b == -1) {
    int old = atomicCAS((int32_t *)&ptab[pg], -1, -2);
    if (old == -1) {
      int nb = atomicAdd(slot_count, psize);
      if (nb + psize > slot_cap) nb = -3;  // overflow marker
      __threadfence_block();
      ptab[pg] = nb;
      return nb;
    }
  }
  while ((b = ptab[pg]) == -2) {
  }
  return b;  // >= 0 or -3 (overflow)
}

// 16-bit page table: the claim marks the entry through a CAS on its 32-bit word
__device__ __forceinline__ int page_slot(volatile int16_t *ptab, int pg, int psize, int *slot_count,
                                         int slot_cap) {
  int b = ptab[pg];
  if (b >= 0) return b;
  if (b == -1) {
    unsigned *word = (unsigned *)((uintptr_t)(ptab + pg) & ~(uintptr_t)3);
    const int shift = (pg & 1) ? 16 : 0;
    for (;;) {
      const unsigned old = *(volatile unsigned *)word;
      if (((old >> shift) & 0xFFFFu) != 0xFFFFu) break;  // no longer free
      const unsigned nw = (old & ~(0xFFFFu << shift)) | (0xFFFEu << shift);  // -2: claiming
      if (atomicCAS(word, old, nw) == old) {
        int nb = atomicAdd(slot_count, psize);
        if (nb + psize > slot_cap) nb = -3;  // overflow marker
        __threadfence_block();
        ptab[pg] = (int16_t)nb;
        return nb;
      }
    }
  }
  while ((b = ptab[pg]) == -2) {
  }
  return b;  // >= 0 or -3 (overflow)
}

template <class CFG>
__global__ void __launch_bounds__(CFG::kT) k_numeric_paged(NumericArgs a, int32_t *fail_rows,
                                                           int *fail_count) {
  constexpr int kThreads = CFG::kT, kWarps = CFG::kW, kSlots = CFG::kSlots, kPages = CFG::kPages;
  constexpr int kPF = CFG::kPF, NE = CFG::kNE;
  using PT = typename CFG::PageT;
  extern __shared__ double psm[];
  double *vals = psm;                                              // kSlots
  PT *ptab = reinterpret_cast<PT *>(psm + kSlots);                 // kPages
  int32_t *plist = reinterpret_cast<int32_t *>(
      reinterpret_cast<char *>(ptab) + ((kPages * (int)sizeof(PT) + 7) / 8) * 8);  // flush list
  __shared__ long long s_start[kThreads];
  __shared__ int s_len[kThreads];
  __shared__ double s_av[kThreads];
  __shared__ int s_row, s_slots, s_fail, s_npl;
  __shared__ unsigned long long s_off;
  __shared__ long long s_wsum[kWarps + 1];
  __shared__ double s_fs[kWarps], s_p1[kWarps];
  __shared__ long long s_nz[kWarps], s_c1[kWarps];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kSlots; i += kThreads) vals[i] = 0.0;
  for (int i = tid; i < kPages; i += kThreads) ptab[i] = -1;
  if (tid == 0) {
    s_slots = 0;
    s_fail = 0;
  }
  for (;;) {
    __syncthreads();
    if (tid == 0) s_row = atomicAdd(a.row_counter, 1);
    __syncthreads();
    const int idx = s_row;
    if (idx >= a.nlist) break;
    const int64_t r = a.order ? (int64_t)a.order[idx] : (int64_t)idx;
    const int64_t pa0 = a.A.rp[r], pa1 = a.A.rp[r + 1];
    const int nk = (int)(pa1 - pa0);
    const int32_t lo = a.lo[r], hi = a.hi[r];
    if (hi < lo) {
      if (tid == 0) {
        a.row_off[r] = 0;
        a.row_cnt[r] = 0;
        a.row_fsum[r] = 0.0;
        a.row_nnz[r] = 0;
        if (a.row_p1) {
          a.row_p1[r] = 0.0;
          a.row_c1[r] = 0;
        }
      }
      continue;
    }
    const int64_t span = (int64_t)hi - lo + 1;
    int sh = CFG::kMinShift;
    while ((span >> sh) >= kPages) sh++;
    if (sh > kMaxPageShift || nk > kSlots) {
      if (tid == 0) fail_rows[atomicAdd(fail_count, 1)] = (int32_t)r;
      continue;
    }
    const int psize = 1 << sh;
    const int npages = (int)((span - 1) >> sh) + 1;
    if (a.self_coef != 0.0) {  // 2T term first (Eq. 2.7)
      for (int64_t p = pa0 + tid; p < pa1; p += kThreads) {
        const int rel = a.A.col[p] - lo;
        const int b = page_slot(ptab, rel >> sh, psize, &s_slots, kSlots);
        if (b >= 0) vals[b + (rel & (psize - 1))] = __dmul_rn(a.self_coef, a.A.val[p]);
        else s_fail = 1;
      }
    }
    for (int kc = 0; kc < nk; kc += kThreads) {
      __syncthreads();
      if (s_fail) break;
      {
        const int j = kc + tid;
        long long st0 = 0;
        int ln = 0;
        double av = 0.0;
        if (j < nk) {
          const int64_t k = (int64_t)a.A.col[pa0 + j] - a.B.row0;
          if (k >= 0 && k < a.B.nrows) {
            st0 = a.B.rp[k];
            ln = (int)(a.B.rp[k + 1] - st0);
            av = a.A.val[pa0 + j];
          }
        }
        s_start[tid] = st0;
        s_len[tid] = ln;
        s_av[tid] = av;
      }
      __syncthreads();
      const int cn = nk - kc < kThreads ? nk - kc : kThreads;
      // register ring: entries tid + u * kThreads (u < NE) of the next kPF k's
      int32_t pc[kPF][NE];
      double pv[kPF][NE];
#pragma unroll
      for (int d = 0; d < kPF; d++) {
#pragma unroll
        for (int u = 0; u < NE; u++) {
          pc[d][u] = 0;
          pv[d][u] = 0.0;
          if (d < cn) {
            const int e = tid + u * kThreads;
            if (e < s_len[d]) {
              pc[d][u] = a.B.col[s_start[d] + e];
              pv[d][u] = a.B.val[s_start[d] + e];
            }
          }
        }
      }
      for (int kk0 = 0; kk0 < cn; kk0 += kPF) {
#pragma unroll
        for (int d = 0; d < kPF; d++) {
          const int kk = kk0 + d;
          if (kk < cn) {
            const long long st0 = s_start[kk];
            const int ln = s_len[kk];
            const double av = s_av[kk];
            int32_t c[NE];
            double v[NE];
#pragma unroll
            for (int u = 0; u < NE; u++) {
              c[u] = pc[d][u];
              v[u] = pv[d][u];
            }
            const int kn = kk + kPF;  // refill this ring slot
            if (kn < cn) {
              const int nl = s_len[kn];
              const long long ns = s_start[kn];
#pragma unroll
              for (int u = 0; u < NE; u++) {
                if (tid + u * kThreads < nl) {
                  pc[d][u] = a.B.col[ns + tid + u * kThreads];
                  pv[d][u] = a.B.val[ns + tid + u * kThreads];
                }
              }
            }
            // slot lookups, then the cell loads, multiply-adds and stores (the entries of
            // one B row have distinct columns)
            int o[NE];
#pragma unroll
            for (int u = 0; u < NE; u++) {
              o[u] = -1;
              if (tid + u * kThreads < ln) {
                const int rel = c[u] - lo;
                const int b = page_slot(ptab, rel >> sh, psize, &s_slots, kSlots);
                if (b >= 0) o[u] = b + (rel & (psize - 1));
                else s_fail = 1;
              }
            }
            double x[NE];
#pragma unroll
            for (int u = 0; u < NE; u++) x[u] = o[u] >= 0 ? vals[o[u]] : 0.0;
#pragma unroll
            for (int u = 0; u < NE; u++)
              if (o[u] >= 0) vals[o[u]] = __dadd_rn(x[u], __dmul_rn(av, v[u]));
            for (int e = tid + NE * kThreads; e < ln; e += kThreads) {
              const int rel = a.B.col[st0 + e] - lo;
              const double vv = a.B.val[st0 + e];
              const int b = page_slot(ptab, rel >> sh, psize, &s_slots, kSlots);
              if (b >= 0) {
                const int oo = b + (rel & (psize - 1));
                vals[oo] = __dadd_rn(vals[oo], __dmul_rn(av, vv));
              } else {
                s_fail = 1;
              }
            }
            __syncthreads();  // one writer per slot at any time (k -> k+1)
          }
        }
      }
    }
    __syncthreads();
    const bool failed = s_fail != 0;
    // ---- flush: allocated pages in column order ----
    // (a) ordered list of allocated pages
    if (tid == 0) s_npl = 0;
    __syncthreads();
    for (int t0 = 0; t0 < npages; t0 += kThreads) {
      const int i = t0 + tid;
      const bool f = !failed && i < npages && ptab[i] >= 0;
      const unsigned m = __ballot_sync(FULL_MASK, f);
      if (lane == 0) s_wsum[warp] = __popc(m);
      __syncthreads();
      if (tid == 0) {
        long long acc = s_npl;
        for (int w = 0; w < kWarps; w++) {
          long long t = s_wsum[w];
          s_wsum[w] = acc;
          acc += t;
        }
        s_npl = (int)acc;
      }
      __syncthreads();
      if (f) plist[s_wsum[warp] + __popc(m & lanemask_lt())] = i;
      __syncthreads();
    }
    const int npl = s_npl;
    // (b) per-thread contiguous range of slots in page order: thread handles list
    //     positions [q0, q1) of the concatenated (page, offset) sequence
    const int total_slots = npl * psize;
    const int per = (total_slots + kThreads - 1) / kThreads;
    const int q0 = tid * per < total_slots ? tid * per : total_slots;
    const int q1 = q0 + per < total_slots ? q0 + per : total_slots;
    int nst = 0;
    double fs = 0.0, p1 = 0.0;
    long long nnzu = 0, c1 = 0;
    for (int q = q0; q < q1; q++) {
      const int pgi = plist[q >> sh];
      const int o = ptab[pgi] + (q & (psize - 1));
      const double x = vals[o] / a.divisor;
      if (x != 0.0) {
        nnzu++;
        if (fabs(x) > a.floor_tau) {
          nst++;
          if (fabs(x) <= a.eps_g) p1 += x * x;
          else c1++;
        } else {
          fs += x * x;
        }
      }
    }
    if (a.row_p1) {  // fused first pass of Algorithm 4.1 (fixed order: threads, then warps)
      p1 = warp_sum(p1);
      c1 = warp_sum(c1);
      if (lane == 0) {
        s_p1[warp] = p1;
        s_c1[warp] = c1;
      }
    }
    // exclusive scan of nst over threads (thread order == column order)
    int v = nst;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(FULL_MASK, v, o);
      if (lane >= o) v += y;
    }
    if (lane == 31) s_wsum[warp] = v;
    fs = warp_sum(fs);
    nnzu = warp_sum(nnzu);
    if (lane == 0) {
      s_fs[warp] = fs;
      s_nz[warp] = nnzu;
    }
    __syncthreads();
    if (tid == 0) {
      long long acc = 0;
      for (int w = 0; w < kWarps; w++) {
        long long t = s_wsum[w];
        s_wsum[w] = acc;
        acc += t;
      }
      s_wsum[kWarps] = acc;
      s_off = failed ? 0ull : atomicAdd(a.pool_used, (unsigned long long)acc);
    }
    __syncthreads();
    const long long total = s_wsum[kWarps];
    const unsigned long long off = s_off;
    const bool ok = !failed && (long long)off + total <= a.pool_cap;
    if (ok) {
      long long pos = (long long)off + s_wsum[warp] + v - nst;
      for (int q = q0; q < q1; q++) {
        const int pgi = plist[q >> sh];
        const int o = ptab[pgi] + (q & (psize - 1));
        const double x = vals[o] / a.divisor;
        if (x != 0.0 && fabs(x) > a.floor_tau) {
          a.pool_col[pos] = lo + (pgi << sh) + (q & (psize - 1));
          a.pool_val[pos] = x;
          pos++;
        }
      }
    }
    __syncthreads();
    // (c) reset the touched pages
    if (failed) {
      for (int i = tid; i < kSlots; i += kThreads) vals[i] = 0.0;
      for (int i = tid; i < npages; i += kThreads) ptab[i] = -1;
    } else {
      for (int q = tid; q < total_slots; q += kThreads) {
        const int pgi = plist[q >> sh];
        vals[ptab[pgi] + (q & (psize - 1))] = 0.0;
      }
      __syncthreads();
      for (int i = tid; i < npl; i += kThreads) ptab[plist[i]] = -1;
    }
    if (tid == 0) {
      if (failed) {
        fail_rows[atomicAdd(fail_count, 1)] = (int32_t)r;
      } else {
        double f = 0.0;
        long long z = 0;
        for (int w = 0; w < kWarps; w++) {
          f += s_fs[w];
          z += s_nz[w];
        }
        if (!ok) atomicOr(a.flags, 1);
        a.row_off[r] = (int64_t)off;
        a.row_cnt[r] = total;
        a.row_fsum[r] = f;
        a.row_nnz[r] = z;
        if (a.row_p1) {
          double pp = 0.0;
          long long cc = 0;
          for (int w = 0; w < kWarps; w++) {
            pp += s_p1[w];
            cc += s_c1[w];
          }
          a.row_p1[r] = pp;
          a.row_c1[r] = cc;
        }
      }
      s_slots = 0;
      s_fail = 0;
    }
  }
}

template <class CFG>
static void launch_paged_cfg(const NumericArgs &a, int32_t *fail_rows, int *fail_count,
                             cudaStream_t st) {
  if (a.A.nrows == 0 || a.nlist == 0) return;
  const int smem = CFG::smem();
  cudaFuncSetAttribute(k_numeric_paged<CFG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  KL;
  k_numeric_paged<CFG><<<a.grid, CFG::kT, smem, st>>>(a, fail_rows, fail_count);
}
void launch_numeric_paged(const NumericArgs &a, int32_t *fail_rows, int *fail_count,
                          cudaStream_t st) {
  launch_paged_cfg<PagedV1>(a, fail_rows, fail_count, st);
}

// ------------------------------------------------------------------------------------
// K5p Taylor term by PULL: S~(r, j) = (sum_{k} s_rk h0_kj) / i  (Eq. 4.11).
//
// H0 rows are short (a few entries), so pushing them through an accumulator leaves most
// lanes idle.  Instead the CTA (1) maps row r of S^ into a paged shared-memory table
// (k -> s_rk), marking in a bitmap every column j reachable through H0's rows; (2) reads
// the bitmap in column order to list the candidate columns (sorted, no sort needed);
// (3) gives each candidate to one thread, which walks column j of H0 (the CSC copy H0^T
// built at plan time, ascending k) and accumulates acc = acc + (s_rk * h0_kj) over the k
// present in row r -- exactly the oracle's order, with _rn intrinsics: S~ is bit-identical
// to the oracle's, and no two threads ever write the same value.  Rows that do not fit
// the tables go to the push kernels (fail list).
// ------------------------------------------------------------------------------------
constexpr int kTPages = 4096;
constexpr int kTSlots = 2048;
constexpr int kTBitWords = 4096;
constexpr int kTCand = 2048;

int taylor_pull_smem_bytes() {
  return kTSlots * 8 + kTCand * 8 + kTPages * 4 + kTBitWords * 4 + kTCand * 4;
}

__global__ void __launch_bounds__(kThreads) k_taylor_pull(NumericArgs a, CsrView BT,
                                                          int32_t *fail_rows, int *fail_count) {
  extern __shared__ double tsm[];
  double *vals = tsm;                                                   // kTSlots
  double *xval = vals + kTSlots;                                        // kTCand
  int32_t *ptab = reinterpret_cast<int32_t *>(xval + kTCand);           // kTPages
  unsigned *bits = reinterpret_cast<unsigned *>(ptab + kTPages);        // kTBitWords
  int32_t *cand = reinterpret_cast<int32_t *>(bits + kTBitWords);       // kTCand
  __shared__ int s_row, s_slots, s_fail;
  __shared__ unsigned long long s_off;
  __shared__ long long s_wsum[kWarps + 1];
  __shared__ double s_fs[kWarps];
  __shared__ long long s_nz[kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kTSlots; i += kThreads) vals[i] = 0.0;
  for (int i = tid; i < kTPages; i += kThreads) ptab[i] = -1;
  for (int i = tid; i < kTBitWords; i += kThreads) bits[i] = 0u;
  if (tid == 0) {
    s_slots = 0;
    s_fail = 0;
  }
  for (;;) {
    __syncthreads();
    if (tid == 0) s_row = atomicAdd(a.row_counter, 1);
    __syncthreads();
    const int idx = s_row;
    if (idx >= a.nlist) break;
    const int64_t r = a.order ? (int64_t)a.order[idx] : (int64_t)idx;
    const int64_t pa0 = a.A.rp[r], pa1 = a.A.rp[r + 1];
    const int32_t lo = a.lo[r], hi = a.hi[r];
    if (hi < lo) {
      if (tid == 0) {
        a.row_off[r] = 0;
        a.row_cnt[r] = 0;
        a.row_fsum[r] = 0.0;
        a.row_nnz[r] = 0;
      }
      continue;
    }
    const int32_t alo = a.A.col[pa0], ahi = a.A.col[pa1 - 1];
    int sh = 4;
    while ((((int64_t)ahi - alo) >> sh) >= kTPages) sh++;
    const int nw = (int)(((int64_t)hi - lo) >> 5) + 1;
    if (sh > kMaxPageShift || nw > kTBitWords) {
      if (tid == 0) fail_rows[atomicAdd(fail_count, 1)] = (int32_t)r;
      continue;
    }
    const int psize = 1 << sh;
    // (1) row r of S^ into the paged table; mark reachable columns
    for (int64_t p = pa0 + tid; p < pa1; p += kThreads) {
      const int32_t k = a.A.col[p];
      const int rel = k - alo;
      const int b = page_slot(ptab, rel >> sh, psize, &s_slots, kTSlots);
      if (b >= 0 && b + psize <= kTSlots) vals[b + (rel & (psize - 1))] = a.A.val[p];
      else s_fail = 1;
      const int64_t kb = (int64_t)k - a.B.row0;
      if (kb >= 0 && kb < a.B.nrows) {
        for (int64_t q = a.B.rp[kb]; q < a.B.rp[kb + 1]; q++) {
          const int jr = a.B.col[q] - lo;
          atomicOr(&bits[jr >> 5], 1u << (jr & 31));
        }
      }
    }
    __syncthreads();
    bool failed = s_fail != 0;
    // (2) candidates in column order (contiguous word range per thread)
    const int per = (nw + kThreads - 1) / kThreads;
    const int w0 = tid * per < nw ? tid * per : nw;
    const int w1 = w0 + per < nw ? w0 + per : nw;
    int cnt = 0;
    for (int i = w0; i < w1; i++) cnt += __popc(bits[i]);
    int v = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(FULL_MASK, v, o);
      if (lane >= o) v += y;
    }
    if (lane == 31) s_wsum[warp] = v;
    __syncthreads();
    if (tid == 0) {
      long long acc = 0;
      for (int w = 0; w < kWarps; w++) {
        long long t = s_wsum[w];
        s_wsum[w] = acc;
        acc += t;
      }
      s_wsum[kWarps] = acc;
    }
    __syncthreads();
    const int ncand = (int)s_wsum[kWarps];
    if (ncand > kTCand) failed = true;
    {
      int pos = (int)s_wsum[warp] + v - cnt;
      for (int i = w0; i < w1; i++) {
        unsigned m = bits[i];
        bits[i] = 0u;
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1;
          if (!failed) cand[pos] = (i << 5) + b;
          pos++;
        }
      }
    }
    __syncthreads();
    // (3) pull: one thread per candidate column, ascending k along column j of H0
    int nst_t = 0;
    double fs = 0.0;
    long long nnzu = 0;
    if (!failed) {
      for (int c = tid; c < ncand; c += kThreads) {
        const int64_t j = (int64_t)lo + cand[c];
        double acc = 0.0;
        for (int64_t q = BT.rp[j]; q < BT.rp[j + 1]; q++) {
          const int32_t k = BT.col[q];
          if (k < alo || k > ahi) continue;
          const int rel = k - alo;
          const int b = ptab[rel >> sh];
          if (b < 0) continue;
          const double sv = vals[b + (rel & (psize - 1))];
          if (sv == 0.0) continue;  // k not in row r: the oracle has no such product
          acc = __dadd_rn(acc, __dmul_rn(sv, BT.val[q]));
        }
        const double x = acc / a.divisor;
        xval[c] = x;
        if (x != 0.0) {
          nnzu++;
          if (fabs(x) > a.floor_tau) nst_t++;
          else fs += x * x;
        }
      }
    }
    // staged count: candidates are strided over threads, so count per 256-chunk in order
    fs = warp_sum(fs);
    nnzu = warp_sum(nnzu);
    int nst_w = __reduce_add_sync(FULL_MASK, nst_t);
    if (lane == 0) {
      s_fs[warp] = fs;
      s_nz[warp] = nnzu;
      s_wsum[warp] = nst_w;
    }
    __syncthreads();
    if (tid == 0) {
      long long tot = 0;
      double f = 0.0;
      long long z = 0;
      for (int w = 0; w < kWarps; w++) {
        tot += s_wsum[w];
        f += s_fs[w];
        z += s_nz[w];
      }
      s_wsum[kWarps] = tot;
      s_fs[0] = f;
      s_nz[0] = z;
      s_off = failed ? 0ull : atomicAdd(a.pool_used, (unsigned long long)tot);
    }
    __syncthreads();
    const long long total = s_wsum[kWarps];
    const unsigned long long off = s_off;
    const bool ok = !failed && (long long)off + total <= a.pool_cap;
    if (ok) {  // ordered write: chunks of kThreads candidates, block-wide ballot scan
      long long base = 0;
      for (int c0 = 0; c0 < ncand; c0 += kThreads) {
        const int c = c0 + tid;
        const double x = c < ncand ? xval[c] : 0.0;
        const bool st = c < ncand && x != 0.0 && fabs(x) > a.floor_tau;
        const unsigned m = __ballot_sync(FULL_MASK, st);
        __syncthreads();
        if (lane == 0) s_wsum[warp] = __popc(m);
        __syncthreads();
        long long pre = 0, tot = 0;
        for (int w = 0; w < kWarps; w++) {
          if (w < warp) pre += s_wsum[w];
          tot += s_wsum[w];
        }
        if (st) {
          const long long q = (long long)off + base + pre + __popc(m & lanemask_lt());
          a.pool_col[q] = lo + cand[c];
          a.pool_val[q] = x;
        }
        base += tot;
      }
    }
    __syncthreads();
    // reset the paged table (slots of row r's k, then the page entries)
    for (int64_t p = pa0 + tid; p < pa1; p += kThreads) {
      const int rel = a.A.col[p] - alo;
      const int b = ptab[rel >> sh];
      if (b >= 0 && b + psize <= kTSlots) vals[b + (rel & (psize - 1))] = 0.0;
    }
    __syncthreads();
    for (int64_t p = pa0 + tid; p < pa1; p += kThreads) ptab[(a.A.col[p] - alo) >> sh] = -1;
    if (tid == 0) {
      if (failed) {
        fail_rows[atomicAdd(fail_count, 1)] = (int32_t)r;
      } else {
        if (!ok) atomicOr(a.flags, 1);
        a.row_off[r] = (int64_t)off;
        a.row_cnt[r] = total;
        a.row_fsum[r] = s_fs[0];
        a.row_nnz[r] = s_nz[0];
      }
      s_slots = 0;
      s_fail = 0;
    }
  }
}

void launch_taylor_pull(const NumericArgs &a, const CsrView &BT, int32_t *fail_rows,
                        int *fail_count, cudaStream_t st) {
  if (a.A.nrows == 0 || a.nlist == 0) return;
  int smem = taylor_pull_smem_bytes();
  cudaFuncSetAttribute(k_taylor_pull, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  KL;
  k_taylor_pull<<<a.grid, kThreads, smem, st>>>(a, BT, fail_rows, fail_count);
}


// ------------------------------------------------------------------------------------
// BSR-8 view of a CSR matrix (squarings, one GPU): block row I = rows 8I..8I+7, block
// column J = columns 8J..8J+7, dense 8x8 blocks (row-major, zeros where the CSR has no
// entry), block columns sorted.  Plus the block transpose: for every block column J the
// block rows K (ascending) holding a block (K, J) and that block's index.
// ------------------------------------------------------------------------------------
constexpr int kBsrWarps = 8;
constexpr int kBsrSpanWords = 512;  // block-column span per block row: 16384 blocks

// count pass (fill = false) and fill pass (fill = true); warp per block row
// FRAG: values in the fp64 tensor-core fragment order of K3m (kernel 13): element (r, c) of a
// block at 2 (4 r + c % 4) + c / 4, i.e. lane l = 4 r + c % 4 of a warp holds (r, c) and
// (r, c + 4) as one 16-byte pair -- the A operand of mma.m8n8k4 for k = c % 4 and c % 4 + 4
// in one load; otherwise row-major (K3b).
// map (optional): view row r is A's row rowmap[r], column c of A is column colmap[c] of the
// view -- the relabelling fused into the build (no relabelled CSR is written)
template <bool FILL, bool FRAG = false>
__global__ void __launch_bounds__(kBsrWarps * 32) k_bsr_build(CsrView A, int64_t nbr, int64_t *bcnt,
                                                              const int64_t *brp, int32_t *bcol,
                                                              double *bval, int *flags, RowColMap map) {
  __shared__ unsigned bits[kBsrWarps][kBsrSpanWords];
  __shared__ uint16_t prefs[kBsrWarps][kBsrSpanWords];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t I = (int64_t)blockIdx.x * kBsrWarps + wib;
  if (I >= nbr) return;
  unsigned *bm = bits[wib];
  uint16_t *pref = prefs[wib];
  const int64_t r0 = 8 * I, r1 = r0 + 8 < A.nrows ? r0 + 8 : A.nrows;
  auto srow = [&](int64_t r) { return map.rowmap ? map.rowmap[r] : r; };
  auto mcol = [&](int32_t c) { return map.colmap ? (int32_t)map.colmap[c] : c; };
  int32_t jmin = INT32_MAX, jmax = -1;
  if (!map.colmap) {
    for (int64_t r = r0; r < r1; r++) {
      const int64_t p0 = A.rp[srow(r)], p1 = A.rp[srow(r) + 1];
      if (p1 > p0) {
        jmin = min(jmin, A.col[p0] >> 3);
        jmax = max(jmax, A.col[p1 - 1] >> 3);
      }
    }
  } else {  // mapped columns are not monotone: all entries
    for (int64_t r = r0; r < r1; r++) {
      const int64_t sr = srow(r);
      for (int64_t p = A.rp[sr] + lane; p < A.rp[sr + 1]; p += 32) {
        const int32_t b = mcol(A.col[p]) >> 3;
        jmin = min(jmin, b);
        jmax = max(jmax, b);
      }
    }
    jmin = __shfl_sync(FULL_MASK, warp_min(jmin), 0);
    jmax = __shfl_sync(FULL_MASK, warp_max(jmax), 0);
  }
  if (jmax < jmin) {
    if (!FILL && lane == 0) bcnt[I] = 0;
    return;
  }
  const int nw = ((jmax - jmin) >> 5) + 1;
  if (nw > kBsrSpanWords) {
    if (lane == 0) {
      atomicOr(flags, 4);
      if (!FILL) bcnt[I] = 0;
    }
    return;
  }
  for (int w = lane; w < nw; w += 32) bm[w] = 0u;
  __syncwarp();
  for (int64_t r = r0; r < r1; r++) {
    const int64_t sr = srow(r);
    for (int64_t p = A.rp[sr] + lane; p < A.rp[sr + 1]; p += 32) {
      const int b = (mcol(A.col[p]) >> 3) - jmin;
      atomicOr(&bm[b >> 5], 1u << (b & 31));
    }
  }
  __syncwarp();
  if (!FILL) {
    int c = 0;
    for (int w = lane; w < nw; w += 32) c += __popc(bm[w]);
    c = __reduce_add_sync(FULL_MASK, c);
    if (lane == 0) bcnt[I] = c;
    return;
  }
  // ranks: exclusive popcount prefix over the words, 1 lane per word chunk
  const int per = (nw + 31) / 32;
  const int w0 = min(lane * per, nw), w1 = min(w0 + per, nw);
  int cnt = 0;
  for (int w = w0; w < w1; w++) cnt += __popc(bm[w]);
  int v = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL_MASK, v, o);
    if (lane >= o) v += y;
  }
  const int64_t base = brp[I];
  int run = v - cnt;
  for (int w = w0; w < w1; w++) {
    pref[w] = (uint16_t)run;
    unsigned m = bm[w];
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      bcol[base + run] = jmin + w * 32 + b;
      run++;
    }
  }
  const int64_t nb = brp[I + 1] - base;
  for (int64_t t = lane; t < nb * 64; t += 32) bval[base * 64 + t] = 0.0;
  __syncwarp();
  // ranks of each word for the scatter: recompute the prefix in place (word -> rank)
  // (bm[w] keeps its bits; the rank of block b = popc of the words before + bits below)
  // scatter: 4 entries' loads in flight per lane before their stores (bval does not alias A,
  // which the compiler cannot know)
  for (int64_t r = r0; r < r1; r++) {
    const int ri = (int)(r - r0);
    const int64_t sr = srow(r);
    const int64_t pe = A.rp[sr + 1];
    for (int64_t p0 = A.rp[sr] + lane; p0 < pe; p0 += 128) {
      int cc[4];
      double vv[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const int64_t p = p0 + 32 * u;
        cc[u] = p < pe ? mcol(__ldg(A.col + p)) : -1;
        vv[u] = p < pe ? __ldg(A.val + p) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (cc[u] >= 0) {
          const int c = cc[u];
          const int b = (c >> 3) - jmin;
          const int rank = pref[b >> 5] + __popc(bm[b >> 5] & ((1u << (b & 31)) - 1u));
          const int e = FRAG ? 2 * (4 * ri + (c & 3)) + ((c & 7) >> 2) : ri * 8 + (c & 7);
          bval[(base + rank) * 64 + e] = vv[u];
        }
    }
  }
}
void launch_bsr_count(const CsrView &A, int64_t nbr, int64_t *bcnt, int *flags, cudaStream_t st,
                      RowColMap map) {
  if (nbr == 0) return;
  KL;
  k_bsr_build<false><<<grid_for(nbr, kBsrWarps), kBsrWarps * 32, 0, st>>>(A, nbr, bcnt, nullptr,
                                                                           nullptr, nullptr, flags, map);
}
void launch_bsr_fill(const CsrView &A, int64_t nbr, const int64_t *brp, int32_t *bcol,
                     double *bval, int *flags, cudaStream_t st, bool frag, RowColMap map) {
  if (nbr == 0) return;
  KL;
  if (frag)
    k_bsr_build<true, true><<<grid_for(nbr, kBsrWarps), kBsrWarps * 32, 0, st>>>(A, nbr, nullptr, brp,
                                                                                bcol, bval, flags, map);
  else
    k_bsr_build<true, false><<<grid_for(nbr, kBsrWarps), kBsrWarps * 32, 0, st>>>(A, nbr, nullptr, brp,
                                                                                 bcol, bval, flags, map);
}

// block transpose: a stable radix sort of the blocks (enumerated block row by block row,
// i.e. K ascending) by block column J keeps K ascending inside every column; column
// pointers by a count and a scan.
__global__ void k_bsr_rows_of_blocks(int64_t nbr, const int64_t *brp, int32_t *brow, int64_t *bidx) {
  const int64_t K = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (K >= nbr) return;
  for (int64_t b = brp[K] + lane; b < brp[K + 1]; b += 32) {
    brow[b] = (int32_t)K;
    bidx[b] = b;
  }
}
__global__ void k_bsrT_count(int64_t nb, const int32_t *bcol, int32_t *tcnt) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&tcnt[bcol[b]], 1);
}
__global__ void k_gather_i32(const int32_t *src, const int64_t *idx, int64_t cnt, int32_t *dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}
// block transpose without a library sort: blocks scattered to their column's segment with
// an atomic cursor (any order), then every column's block indices sorted ascending (block
// indices enumerate block rows in order, so ascending index = ascending K): one CTA per column,
// bitonic network in shared memory over <= kTSortCap entries
constexpr int kTSortCap = 2048;
__global__ void k_bsrT_scatter(int64_t nbr, const int64_t *brp, const int32_t *bcol, const int64_t *tp,
                               int32_t *cur, int64_t *tb) {
  const int64_t K = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (K >= nbr) return;
  for (int64_t b = brp[K] + lane; b < brp[K + 1]; b += 32) {
    const int J = bcol[b];
    tb[tp[J] + atomicAdd(&cur[J], 1)] = b;
  }
}
__global__ void __launch_bounds__(256) k_sort_segments_i64(const int64_t *sp, int64_t nseg, int64_t *x,
                                                             int *too_long) {
  __shared__ int64_t key[kTSortCap];
  for (int64_t sgm = blockIdx.x; sgm < nseg; sgm += gridDim.x) {
    const int64_t a = sp[sgm];
    const int len = (int)(sp[sgm + 1] - a);
    if (len <= 1) continue;
    if (len > kTSortCap) {
      if (threadIdx.x == 0) atomicOr(too_long, 1);
      continue;
    }
    int m = 2;
    while (m < len) m <<= 1;
    for (int i = threadIdx.x; i < m; i += blockDim.x) key[i] = i < len ? x[a + i] : INT64_MAX;
    __syncthreads();
    for (int k = 2; k <= m; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
          const int p = i ^ j;
          if (p > i) {
            const bool up = (i & k) == 0;
            const int64_t u = key[i], v = key[p];
            if ((u > v) == up) {
              key[i] = v;
              key[p] = u;
            }
          }
        }
        __syncthreads();
      }
    for (int i = threadIdx.x; i < len; i += blockDim.x) x[a + i] = key[i];
    __syncthreads();
  }
}

size_t bsr_transpose_temp_bytes(int64_t nb) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int32_t *)nullptr, (int32_t *)nullptr,
                                  (const int64_t *)nullptr, (int64_t *)nullptr, (int)std::max<int64_t>(nb, 1));
  return bytes;
}
void launch_bsr_transpose(int64_t nbr, int64_t nbc, int64_t nb, const int64_t *brp,
                          const int32_t *bcol, int32_t *tcnt, int64_t *tp, int32_t *tk_tmp,
                          int64_t *tb_tmp, int32_t *tk, int64_t *tb, int64_t *scan_tmp,
                          int64_t *cnt64, void *sort_tmp, size_t sort_tmp_bytes, int32_t *keys_out,
                          cudaStream_t st) {
  cudaMemsetAsync(tcnt, 0, (size_t)std::max<int64_t>(nbc, 1) * sizeof(int32_t), st);
  if (nb > 0) {
    KL;
    k_bsrT_count<<<grid_for(nb, kThreads, 148 * 16), kThreads, 0, st>>>(nb, bcol, tcnt);
  }
  KL;
  k_i32_to_i64<<<grid_for(nbc, kThreads), kThreads, 0, st>>>(tcnt, nbc, cnt64);
  launch_exclusive_scan(cnt64, nbc, tp, scan_tmp, st);
  if (nb == 0) return;
  KL;
  k_bsr_rows_of_blocks<<<grid_for(nbr * 32, kThreads), kThreads, 0, st>>>(nbr, brp, tk_tmp, tb_tmp);
  // in-house: scatter by column, sort each column's block indices (tcnt reused as cursors,
  // keys_out's first word as the overflow flag)
  cudaMemsetAsync(tcnt, 0, (size_t)std::max<int64_t>(nbc, 1) * sizeof(int32_t), st);
  cudaMemsetAsync(keys_out, 0, sizeof(int32_t), st);
  KL;
  k_bsrT_scatter<<<grid_for(nbr * 32, kThreads), kThreads, 0, st>>>(nbr, brp, bcol, tp, tcnt, tb);
  KL;
  k_sort_segments_i64<<<(int)std::max<int64_t>(1, std::min<int64_t>(nbc, 148 * 8)), 256, 0, st>>>(tp, nbc, tb, keys_out);
  int too_long = 0;
  cudaMemcpyAsync(&too_long, keys_out, sizeof(int), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  if (too_long) {  // a column with more than kTSortCap blocks: stable radix sort by column
    int bits = 1;
    while (bits < 31 && (int64_t(1) << bits) <= nbc) bits++;
    KL;
    cub::DeviceRadixSort::SortPairs(sort_tmp, sort_tmp_bytes, bcol, keys_out, tb_tmp, tb, (int)nb, 0,
                                    bits, st);
  }
  KL;
  k_gather_i32<<<grid_for(nb, kThreads, 148 * 16), kThreads, 0, st>>>(tk_tmp, tb, nb, tk);
}

// ------------------------------------------------------------------------------------
// K3b numeric filtered SpGEMM on the BSR-8 view (squarings, one GPU):
//
//   C~_IJ = self * A_IJ + sum_K A_IK B_KJ      (8x8 blocks; Eq. 2.7, Eq. 4.15)
//
// One CTA per block row I (8 rows).  A's blocks of row I sit in shared memory (value rows
// and a bitmap of their block columns K); the candidate output blocks J are the union of the
// block rows B_K, K in row I (bitmap).  A warp computes whole output blocks: lane l holds
// C[i][j] for i = l/8 and l/8 + 4, j = l%8, in registers, starting from the self term, then
// for every K common to row I of A and column J of B (the block transpose lists K
// ascending) it adds a[i][k] * b[k][j] for k = 0..7 with _rn products and sums.  Every
// element therefore sees the self term and then ascending k -- a k outside the row's or the
// column's pattern contributes 0 * b or a * 0, which leaves the value bit-identical -- so C~
// is bit-identical to the oracle's.  The dense blocks go to this CTA's scratch (L2), the
// kept counts per (J, row) to shared memory; then each row's entries above the floor are
// staged contiguously in column order (block columns ascending).  The redundant products on
// the zeros of partly filled blocks (~3.6x at config 5) are paid in registers, not in
// shared-memory read-modify-writes.
// ------------------------------------------------------------------------------------
constexpr int kBThreads = 256;
constexpr int kBWarps = kBThreads / 32;
constexpr int kBACap = kBsrMaxRowBlocks;  // blocks of a row of A held in shared memory
constexpr int kBML = 64;         // matches (K) of one output block listed at a time per warp
constexpr int kBPF = 4;          // B blocks in flight per warp
constexpr int kBKWords = 256;    // K bitmap: block-column span of A's row <= 8192
constexpr int kBJWords = 512;    // J bitmap: output block-column span <= 16384
constexpr int kBJCap = kBsrScratchPerCta / 64;  // output blocks per block row

int bsr_numeric_smem_bytes() {
  return kBACap * 64 * 8 + kBWarps * kBPF * 64 * 8 + kBWarps * kBML * 8 + kBWarps * kBML * 4 +
         kBACap * 4 + kBKWords * 4 + kBKWords * 2 + kBJWords * 4 + kBJCap * 4 + kBJCap * 8 * 2 + 64;
}

// BsrView (kernels.cuh): brp / bcol / bval = block rows, sorted block columns, 64 values
// per block row-major; tp / tk / tb = block transpose: column J's block rows K (ascending)
// and block indices.

// x0 += sum_k a[i0][k] b[k][lj], x1 likewise for row i1: k ascending, _rn products and sums
__device__ __forceinline__ void bsr_block_fma(const double *bs, const double *as, int i0, int i1,
                                              int lj, double &x0, double &x1) {
  const double *bq = bs + lj, *ap0 = as + i0 * 8, *ap1 = as + i1 * 8;
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const double b = bq[k * 8];
    x0 = __dadd_rn(x0, __dmul_rn(ap0[k], b));
    x1 = __dadd_rn(x1, __dmul_rn(ap1[k], b));
  }
}

__global__ void __launch_bounds__(kBThreads, 2) k_numeric_bsr(NumericArgs a, BsrView Bv, int64_t nrows,
                                                              double *scratch, int32_t *fail_rows,
                                                              int *fail_count) {
  extern __shared__ double bsm[];
  double *aval = bsm;                                                  // kBACap * 64
  double *wstage = aval + kBACap * 64;                                 // kBWarps * kBPF * 64
  int64_t *mlb = reinterpret_cast<int64_t *>(wstage + kBWarps * kBPF * 64);  // kBWarps * kBML
  int32_t *mlk = reinterpret_cast<int32_t *>(mlb + kBWarps * kBML);    // kBWarps * kBML
  int32_t *aK = mlk + kBWarps * kBML;                                  // kBACap
  unsigned *kbits = reinterpret_cast<unsigned *>(aK + kBACap);         // kBKWords
  uint16_t *kpref = reinterpret_cast<uint16_t *>(kbits + kBKWords);    // kBKWords
  unsigned *jbits = reinterpret_cast<unsigned *>(kpref + kBKWords);    // kBJWords
  int32_t *jlist = reinterpret_cast<int32_t *>(jbits + kBJWords);      // kBJCap
  uint16_t *jcnt = reinterpret_cast<uint16_t *>(jlist + kBJCap);       // kBJCap * 8
  __shared__ int s_I, s_fail, s_na, s_nj, s_kmin, s_jmin, s_nkw, s_njw;
  __shared__ double s_fs[kBWarps][8], s_p1[kBWarps][8];
  __shared__ long long s_nz[kBWarps][8], s_c1[kBWarps][8];
  __shared__ unsigned long long s_off[8];
  __shared__ long long s_tot[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double *scr = scratch + (size_t)blockIdx.x * kBJCap * 64;
  for (int i = tid; i < kBKWords; i += kBThreads) kbits[i] = 0u;
  for (int i = tid; i < kBJWords; i += kBThreads) jbits[i] = 0u;
  const int li = lane >> 3, lj = lane & 7;  // lane holds C[li][lj] and C[li + 4][lj]
  for (;;) {
    __syncthreads();
    if (tid == 0) s_I = atomicAdd(a.row_counter, 1);
    __syncthreads();
    if (s_I >= Bv.nbr_a) break;
    const int64_t I = Bv.border ? (int64_t)Bv.border[s_I] : (int64_t)s_I;
    const int64_t r0 = 8 * I;
    const int nr = (int)(nrows - r0 < 8 ? nrows - r0 : 8);
    const int64_t ab0 = Bv.brp[I + Bv.ib0], ab1 = Bv.brp[I + Bv.ib0 + 1];
    const int na = (int)(ab1 - ab0);
    if (tid == 0) {
      int fail = na > kBACap;
      int jmin = INT32_MAX, jmax = -1;
      for (int i = 0; i < nr; i++) {
        const int64_t r = r0 + i;
        if (a.hi[r] >= a.lo[r]) {
          jmin = min(jmin, a.lo[r] >> 3);
          jmax = max(jmax, a.hi[r] >> 3);
        }
      }
      const int kmin = na > 0 ? Bv.bcol[ab0] : 0, kmax = na > 0 ? Bv.bcol[ab1 - 1] : -1;
      if (na > 0 && ((kmax - kmin) >> 5) + 1 > kBKWords) fail = 1;
      if (jmax >= jmin && ((jmax - jmin) >> 5) + 1 > kBJWords) fail = 1;
      s_fail = fail;
      s_na = na;
      s_kmin = kmin;
      s_jmin = jmin;
      s_nkw = na > 0 ? ((kmax - kmin) >> 5) + 1 : 0;
      s_njw = jmax >= jmin ? ((jmax - jmin) >> 5) + 1 : 0;
    }
    __syncthreads();
    if (s_fail || na == 0 || s_njw == 0) {
      if (tid < nr) {
        const int64_t r = r0 + tid;
        if (s_fail) {
          fail_rows[atomicAdd(fail_count, 1)] = (int32_t)r;
        } else {
          a.row_off[r] = 0;
          a.row_cnt[r] = 0;
          a.row_fsum[r] = 0.0;
          a.row_nnz[r] = 0;
          if (a.row_p1) {
            a.row_p1[r] = 0.0;
            a.row_c1[r] = 0;
          }
        }
      }
      continue;
    }
    const int kmin = s_kmin, jmin = s_jmin, nkw = s_nkw, njw = s_njw;
    // (1) row I of A: block columns, values, K bitmap
    for (int t = tid; t < na; t += kBThreads) {
      const int K = Bv.bcol[ab0 + t];
      aK[t] = K;
      atomicOr(&kbits[(K - kmin) >> 5], 1u << ((K - kmin) & 31));
    }
    for (int t = tid; t < na * 64; t += kBThreads) aval[t] = Bv.bval[ab0 * 64 + t];
    __syncthreads();
    if (tid < 32) {  // word prefix of the K bitmap
      const int per = (nkw + 31) / 32;
      const int w0 = min(lane * per, nkw), w1 = min(w0 + per, nkw);
      int c = 0;
      for (int w = w0; w < w1; w++) c += __popc(kbits[w]);
      int v = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL_MASK, v, o);
        if (lane >= o) v += y;
      }
      int run = v - c;
      for (int w = w0; w < w1; w++) {
        kpref[w] = (uint16_t)run;
        run += __popc(kbits[w]);
      }
    }
    // (2) candidate output blocks: union of the block rows of B at A's block columns
    for (int t = warp; t < na; t += kBWarps) {
      const int64_t K = aK[t] - Bv.kb0;  // the view's block row of block column aK[t]
      if (K >= 0 && K < Bv.nbr) {
        for (int64_t b = Bv.brp[K] + lane; b < Bv.brp[K + 1]; b += 32) {
          const int jb = Bv.bcol[b] - jmin;
          if (jb >= 0 && jb < njw * 32) atomicOr(&jbits[jb >> 5], 1u << (jb & 31));
        }
      }
    }
    // the self term 2 A_IJ reaches the block columns of row I itself, also where no B_K of
    // the row has block J (e.g. an empty diagonal block)
    if (a.self_coef != 0.0)
      for (int t = tid; t < na; t += kBThreads) {
        const int jb = aK[t] - jmin;
        if (jb >= 0 && jb < njw * 32) atomicOr(&jbits[jb >> 5], 1u << (jb & 31));
      }
    __syncthreads();
    if (tid < 32) {
      const int per = (njw + 31) / 32;
      const int w0 = min(lane * per, njw), w1 = min(w0 + per, njw);
      int c = 0;
      for (int w = w0; w < w1; w++) c += __popc(jbits[w]);
      int v = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL_MASK, v, o);
        if (lane >= o) v += y;
      }
      const int tot = __shfl_sync(FULL_MASK, v, 31);
      if (lane == 0) s_nj = tot;
      if (tot <= kBJCap) {
        int run = v - c;
        for (int w = w0; w < w1; w++) {
          unsigned m = jbits[w];
          while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            jlist[run++] = jmin + w * 32 + b;
          }
        }
      }
    }
    __syncthreads();
    const int nj = s_nj;
    const bool over = nj > kBJCap;
    // (3) output blocks, one warp each
    double fs0 = 0.0, fs1 = 0.0, q10 = 0.0, q11 = 0.0;
    long long nz0 = 0, nz1 = 0, c10 = 0, c11 = 0;
    unsigned long long nbp = 0;  // block products of this warp (uniform over its lanes)
    const int i0 = li, i1 = li + 4;
    if (!over) {
      for (int q = warp; q < nj; q += kBWarps) {
        const int J = jlist[q];
        double x0 = 0.0, x1 = 0.0;
        {  // self term: A_IJ, if row I of A has block J
          const int kb = J - kmin;
          if (a.self_coef != 0.0 && kb >= 0 && kb < nkw * 32 && ((kbits[kb >> 5] >> (kb & 31)) & 1u)) {
            const int ra = kpref[kb >> 5] + __popc(kbits[kb >> 5] & ((1u << (kb & 31)) - 1u));
            x0 = __dmul_rn(a.self_coef, aval[ra * 64 + i0 * 8 + lj]);
            x1 = __dmul_rn(a.self_coef, aval[ra * 64 + i1 * 8 + lj]);
          }
        }
        // matches K of row I of A and column J of B, listed in ascending K (batches of kBML),
        // then the B blocks streamed kBPF ahead: one 16-byte load per lane per block
        // (coalesced 512 bytes), staged in this warp's shared buffer for the column reads
        int64_t *wb = mlb + warp * kBML;
        int32_t *wk = mlk + warp * kBML;
        double *stg = wstage + warp * kBPF * 64;
        const int64_t t0 = Bv.tp[J], t1 = Bv.tp[J + 1];
        int64_t tb0 = t0;
        while (tb0 < t1) {
          int nm = 0;
          for (; tb0 < t1 && nm <= kBML - 32; tb0 += 32) {
            const int64_t t = tb0 + lane;
            int ra = -1;
            int64_t bidx = 0;
            if (t < t1) {
              const int K = Bv.tk[t] + (int)Bv.kb0;  // global block row
              const int kb = K - kmin;
              if (kb >= 0 && kb < nkw * 32 && ((kbits[kb >> 5] >> (kb & 31)) & 1u)) {
                ra = kpref[kb >> 5] + __popc(kbits[kb >> 5] & ((1u << (kb & 31)) - 1u));
                bidx = Bv.tb[t];
              }
            }
            const unsigned m = __ballot_sync(FULL_MASK, ra >= 0);
            if (ra >= 0) {
              const int pos = nm + __popc(m & lanemask_lt());
              wk[pos] = ra;
              wb[pos] = bidx;
            }
            nm += __popc(m);
          }
          __syncwarp();
          nbp += nm;
          double2 pf[kBPF];
#pragma unroll
          for (int d = 0; d < kBPF; d++)
            if (d < nm) pf[d] = reinterpret_cast<const double2 *>(Bv.bval + wb[d] * 64)[lane];
          int t = 0;
          // full batches of kBPF blocks: stage all, one warp barrier, then the kBPF block
          // products back to back (no control flow between them, so the shared loads of the
          // next product issue while the previous one's sums run)
          for (; t + kBPF <= nm; t += kBPF) {
#pragma unroll
            for (int d = 0; d < kBPF; d++) reinterpret_cast<double2 *>(stg + d * 64)[lane] = pf[d];
            __syncwarp();
#pragma unroll
            for (int d = 0; d < kBPF; d++)
              if (t + kBPF + d < nm) pf[d] = reinterpret_cast<const double2 *>(Bv.bval + wb[t + kBPF + d] * 64)[lane];
#pragma unroll
            for (int d = 0; d < kBPF; d++) bsr_block_fma(stg + d * 64, aval + wk[t + d] * 64, i0, i1, lj, x0, x1);
            __syncwarp();
          }
          if (t < nm) {  // tail batch (< kBPF blocks)
#pragma unroll
            for (int d = 0; d < kBPF; d++)
              if (t + d < nm) reinterpret_cast<double2 *>(stg + d * 64)[lane] = pf[d];
            __syncwarp();
#pragma unroll
            for (int d = 0; d < kBPF; d++)
              if (t + d < nm) bsr_block_fma(stg + d * 64, aval + wk[t + d] * 64, i0, i1, lj, x0, x1);
            __syncwarp();
          }
        }
        // classify (Algorithm 4.1 floor), counts per (J, row), block to scratch
        const bool ok0 = i0 < nr, ok1 = i1 < nr;
        bool st0 = false, st1 = false;
        if (ok0 && x0 != 0.0) {
          nz0++;
          if (fabs(x0) > a.floor_tau) {
            st0 = true;
            if (fabs(x0) <= a.eps_g) q10 += x0 * x0;
            else c10++;
          } else {
            fs0 += x0 * x0;
          }
        }
        if (ok1 && x1 != 0.0) {
          nz1++;
          if (fabs(x1) > a.floor_tau) {
            st1 = true;
            if (fabs(x1) <= a.eps_g) q11 += x1 * x1;
            else c11++;
          } else {
            fs1 += x1 * x1;
          }
        }
        // only the staged values go to scratch, packed at the front of their (block, row)
        // slot; the row's 8-bit keep mask (shared memory) gives their columns
        const unsigned b0m = __ballot_sync(FULL_MASK, st0), b1m = __ballot_sync(FULL_MASK, st1);
        const unsigned m0 = (b0m >> (li * 8)) & 0xFFu, m1 = (b1m >> (li * 8)) & 0xFFu;
        const unsigned below = (1u << lj) - 1u;
        if (st0) scr[(size_t)q * 64 + i0 * 8 + __popc(m0 & below)] = x0;
        if (st1) scr[(size_t)q * 64 + i1 * 8 + __popc(m1 & below)] = x1;
        if (lj == 0) {
          jcnt[q * 8 + i0] = (uint16_t)m0;
          jcnt[q * 8 + i1] = (uint16_t)m1;
        }
      }
    }
    if (a.prof && lane == 0 && nbp) atomicAdd(&a.prof[0], nbp);
    // per-row sums: lanes with the same row (8 lanes) then warps, in fixed order
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      fs0 += __shfl_xor_sync(FULL_MASK, fs0, o);
      fs1 += __shfl_xor_sync(FULL_MASK, fs1, o);
      q10 += __shfl_xor_sync(FULL_MASK, q10, o);
      q11 += __shfl_xor_sync(FULL_MASK, q11, o);
      nz0 += __shfl_xor_sync(FULL_MASK, nz0, o);
      nz1 += __shfl_xor_sync(FULL_MASK, nz1, o);
      c10 += __shfl_xor_sync(FULL_MASK, c10, o);
      c11 += __shfl_xor_sync(FULL_MASK, c11, o);
    }
    if (lj == 0) {
      s_fs[warp][i0] = fs0;
      s_fs[warp][i1] = fs1;
      s_p1[warp][i0] = q10;
      s_p1[warp][i1] = q11;
      s_nz[warp][i0] = nz0;
      s_nz[warp][i1] = nz1;
      s_c1[warp][i0] = c10;
      s_c1[warp][i1] = c11;
    }
    __syncthreads();
    // (4) stage each row's kept entries contiguously (warp i: row i)
    if (over) {
      if (tid < nr) fail_rows[atomicAdd(fail_count, 1)] = (int32_t)(r0 + tid);
    } else if (warp < nr) {
      const int i = warp;
      const int64_t r = r0 + i;
      long long tot = 0;
      for (int q0 = 0; q0 < nj; q0 += 32) {
        const int c = q0 + lane < nj ? __popc(jcnt[(q0 + lane) * 8 + i]) : 0;
        tot += __reduce_add_sync(FULL_MASK, c);
      }
      unsigned long long off = 0;
      if (lane == 0) off = atomicAdd(a.pool_used, (unsigned long long)tot);
      off = __shfl_sync(FULL_MASK, off, 0);
      const bool ok = (long long)off + tot <= a.pool_cap;
      if (ok) {
        long long pos = (long long)off;
        for (int q0 = 0; q0 < nj; q0 += 32) {
          const int q = q0 + lane;
          unsigned m = q < nj ? jcnt[q * 8 + i] : 0u;
          const int c = __popc(m);
          int v = c;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL_MASK, v, o);
            if (lane >= o) v += y;
          }
          if (c > 0) {
            long long p = pos + v - c;
            const double *src = scr + (size_t)q * 64 + i * 8;
            const int J = jlist[q];
            for (int e = 0; m; e++, p++) {
              const int j = __ffs(m) - 1;
              m &= m - 1;
              a.pool_col[p] = 8 * J + j;
              a.pool_val[p] = src[e];
            }
          }
          pos += __shfl_sync(FULL_MASK, v, 31);
        }
      }
      if (lane == 0) {
        double f = 0.0, p1 = 0.0;
        long long z = 0, c1 = 0;
        for (int w = 0; w < kBWarps; w++) {
          f += s_fs[w][i];
          p1 += s_p1[w][i];
          z += s_nz[w][i];
          c1 += s_c1[w][i];
        }
        if (!ok) atomicOr(a.flags, 1);
        a.row_off[r] = (int64_t)off;
        a.row_cnt[r] = tot;
        a.row_fsum[r] = f;
        a.row_nnz[r] = z;
        if (a.row_p1) {
          a.row_p1[r] = p1;
          a.row_c1[r] = c1;
        }
      }
    }
    __syncthreads();
    for (int i = tid; i < nkw; i += kBThreads) kbits[i] = 0u;
    for (int i = tid; i < njw; i += kBThreads) jbits[i] = 0u;
  }
}

void launch_numeric_bsr(const NumericArgs &a, const BsrView &Bv, int64_t nrows, double *scratch,
                        int32_t *fail_rows, int *fail_count, cudaStream_t st) {
  if (Bv.nbr_a == 0) return;
  const int smem = bsr_numeric_smem_bytes();
  cudaFuncSetAttribute(k_numeric_bsr, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  KL;
  k_numeric_bsr<<<a.grid, kBThreads, smem, st>>>(a, Bv, nrows, scratch, fail_rows, fail_count);
}

// ------------------------------------------------------------------------------------
// K3m numeric filtered SpGEMM on the BSR-8 view with the fp64 tensor-core instruction
// (squarings; default):
//
//   C~_IJ = self * A_IJ + sum_K A_IK B_KJ      (8x8 blocks; Eq. 2.7, Eq. 4.15)
//
// The same block decomposition as K3b, but every 8x8x8 block product is two
// mma.sync.m8n8k4.f64 instructions (DMMA: 8x8x4 fused multiply-adds each) whose operands
// come straight from the block store in fragment order (k_bsr_build<FRAG>): lane l
// (g = l / 4, t = l % 4) loads A_IK[g][t] and A_IK[g][t+4] as one 16-byte pair and B_KJ[t][g],
// B_KJ[t+4][g] as two 8-byte words (each warp-wide load one contiguous 256 or 512 bytes), and
// accumulates C_IJ[g][2t], C_IJ[g][2t+1] in registers.  Four operand loads per lane per block
// product instead of K3b's 24 shared-memory loads: the L1 wavefront bound of K3b is gone
// and the kernel is bound by the DMMA pipe (37.2 TF/s measured, profiles/r02_fp64_peak) and
// the L2 -> SM operand stream.  A's blocks are read through L1 like B's (no shared-memory
// copy of row I), so a block row of any width is handled (config 4's 3D rows); only the
// spans of the K and J bitmaps and the J count per block row are capped.
//
// Rounding: DMMA fuses each product into the running sum (one rounding per FMA), so C~ is
// not bit-identical to the oracle's DMUL + DADD order; K3b (kernel 11) is the bit-exact
// path.  The difference is a few ulps of the partial sums, inside the north-star parity
// bound (tests/test_gpu_parity.py).
//
// One CTA per block row I (dynamic scheduler over the locality order), one warp per output
// block J: for the K common to row I of A and column J of B (block transpose, ascending)
// the operand pairs of kMPF products are loaded ahead, then multiplied.  The classified
// values (Algorithm 4.1 floor, fused first pass) go to this CTA's scratch packed per
// (block, row) with an 8-bit keep mask; then each row's kept entries are staged in column
// order (block columns ascending).
// ------------------------------------------------------------------------------------
constexpr int kMThreads = 256;
constexpr int kMWarps = kMThreads / 32;
constexpr int kMKWords = 2048;             // K bitmap: block-column span of A's row <= 65536
constexpr int kMJWords = 2048;             // J bitmap: output block-column span <= 65536
constexpr int kMJCap = kBsrMJCap;          // output blocks per block row
constexpr int kMML = 64;                   // matches listed at a time per warp

int bsrm_numeric_smem_bytes() {
  return kMKWords * 4 + kMKWords * 2 + kMJWords * 4 + kMWarps * kMML * 8 + 64;
}

__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// bit l of x to bit 2l
__device__ __forceinline__ unsigned long long spread32(unsigned x) {
  unsigned long long v = x;
  v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
  v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
  v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  return (v | (v << 1)) & 0x5555555555555555ull;
}
// spread 4 bits to the even positions of 8
__device__ __forceinline__ unsigned spread4(unsigned m) {
  m = (m | (m << 2)) & 0x33u;
  return (m | (m << 1)) & 0x55u;
}

// kMPF block products' operands per set (two sets in flight), kMinB CTAs per SM: <2, 4> for
// short match lists (2D: more warps), <4, 2> for long ones (3D: more loads per warp)
// SYM (K3s, see kernels.cuh SymOut): only the output blocks J >= I, written raw to the block
// store; cand(I) to the J store; classification and staging are left to K3a
template <int kMPF, int kMinB, bool SYM = false, bool ROWCNT = true>
__global__ void __launch_bounds__(kMThreads, kMinB) k_numeric_bsrm(NumericArgs a, BsrView Bv, int64_t nrows,
                                                              double *scratch, int32_t *fail_rows,
                                                              int *fail_count, SymOut so) {
  extern __shared__ __align__(16) unsigned char msm[];
  int32_t *mla = reinterpret_cast<int32_t *>(msm);                      // kMWarps * kMML
  int32_t *mlb = mla + kMWarps * kMML;                                  // kMWarps * kMML
  unsigned *kbits = reinterpret_cast<unsigned *>(mlb + kMWarps * kMML); // kMKWords
  unsigned *jbits = kbits + kMKWords;                                   // kMJWords
  uint16_t *kpref = reinterpret_cast<uint16_t *>(jbits + kMJWords);     // kMKWords
  __shared__ int s_I, s_fail, s_nj, s_kmin, s_jmin, s_nkw, s_njw, s_nlow, s_sok;
  __shared__ long long s_cjo, s_obo;
  __shared__ double s_fs[kMWarps][8], s_p1[kMWarps][8];
  __shared__ long long s_nz[kMWarps][8], s_c1[kMWarps][8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;  // fragment coordinates
  // per-CTA scratch (L2): kMJCap output blocks, their keep masks and the J list
  double *scr = scratch + (size_t)blockIdx.x * kMJCap * 66;
  uint8_t *jm = reinterpret_cast<uint8_t *>(scr + (size_t)kMJCap * 64);
  int32_t *jlist = reinterpret_cast<int32_t *>(scr + (size_t)kMJCap * 65);
  for (int i = tid; i < kMKWords; i += kMThreads) kbits[i] = 0u;
  for (int i = tid; i < kMJWords; i += kMThreads) jbits[i] = 0u;
  // B fragment offsets: B[t][g] and B[t + 4][g] in fragment order
  const int boff = 2 * (4 * t + (g & 3)) + (g >> 2);
  // self-term offsets: A_IJ[g][2t] and A_IJ[g][2t + 1]
  const int soff0 = 2 * (4 * g + ((2 * t) & 3)) + ((2 * t) >> 2);
  const int soff1 = 2 * (4 * g + ((2 * t + 1) & 3)) + ((2 * t + 1) >> 2);
  // A's blocks: its own BSR view (Taylor terms: A = S^_{i-1}, B = H0) or B's rows (squarings)
  const int64_t *abrp = Bv.abrp ? Bv.abrp : Bv.brp;
  const int32_t *abcol = Bv.abrp ? Bv.abcol : Bv.bcol;
  const double *abval = Bv.abrp ? Bv.abval : Bv.bval;
  const double2 *av2 = reinterpret_cast<const double2 *>(abval);
  for (;;) {
    __syncthreads();
    if (tid == 0) s_I = atomicAdd(a.row_counter, 1);
    __syncthreads();
    if (s_I >= Bv.nbr_a) break;
    const int64_t I = Bv.border ? (int64_t)Bv.border[s_I] : (int64_t)s_I;
    const int64_t r0 = 8 * I;
    const int nr = (int)(nrows - r0 < 8 ? nrows - r0 : 8);
    const int64_t ab0 = abrp[I + Bv.ib0], ab1 = abrp[I + Bv.ib0 + 1];
    const int na = (int)(ab1 - ab0);
    if (tid == 0) {
      int fail = 0;
      int jmin = INT32_MAX, jmax = -1;
      if constexpr (SYM) {  // the block union's extent (K3c): cand(I) exactly symmetric
        jmin = so.wlo[I];
        jmax = so.whi[I];
      } else {
        for (int i = 0; i < nr; i++) {
          const int64_t r = r0 + i;
          if (a.hi[r] >= a.lo[r]) {
            jmin = min(jmin, a.lo[r] >> 3);
            jmax = max(jmax, a.hi[r] >> 3);
          }
        }
      }
      const int kmin = na > 0 ? abcol[ab0] : 0, kmax = na > 0 ? abcol[ab1 - 1] : -1;
      if (na > 0 && ((kmax - kmin) >> 5) + 1 > kMKWords) fail = 1;
      if (jmax >= jmin && ((jmax - jmin) >> 5) + 1 > kMJWords) fail |= 2;
      if (fail && a.prof) atomicAdd(&a.prof[fail], 1ull);  // block rows handed on: K / J span
      s_fail = fail;
      s_kmin = kmin;
      s_jmin = jmin;
      s_nkw = na > 0 ? ((kmax - kmin) >> 5) + 1 : 0;
      s_njw = jmax >= jmin ? ((jmax - jmin) >> 5) + 1 : 0;
    }
    __syncthreads();
    if (s_fail || na == 0 || s_njw == 0) {
      if constexpr (SYM) {
        if (tid == 0) {
          if (s_fail || so.nj[I] != 0) atomicOr(so.flag, s_fail ? 1 : 2);
          so.fsI[I] = 0.0;
          so.nzI[I] = 0;

        }
        continue;
      }
      if (tid < nr) {
        const int64_t r = r0 + tid;
        if (s_fail) {
          fail_rows[atomicAdd(fail_count, 1)] = (int32_t)r;
        } else {
          a.row_off[r] = 0;
          a.row_cnt[r] = 0;
          a.row_fsum[r] = 0.0;
          a.row_nnz[r] = 0;
          if (a.row_p1) {
            a.row_p1[r] = 0.0;
            a.row_c1[r] = 0;
          }
        }
      }
      continue;
    }
    const int kmin = s_kmin, jmin = s_jmin, nkw = s_nkw, njw = s_njw;
    // (1) K bitmap of row I of A, then the word prefix (ranks)
    for (int q = tid; q < na; q += kMThreads) {
      const int K = abcol[ab0 + q];
      atomicOr(&kbits[(K - kmin) >> 5], 1u << ((K - kmin) & 31));
      // (2a) the self term reaches row I's own block columns (also where no B_K has them)
      if (a.self_coef != 0.0) {
        const int jb = K - jmin;
        if (jb >= 0 && jb < njw * 32) atomicOr(&jbits[jb >> 5], 1u << (jb & 31));
      }
    }
    // (2b) candidate output blocks: union of the block rows of B at A's block columns
    for (int q = warp; q < na; q += kMWarps) {
      const int64_t K = abcol[ab0 + q] - Bv.kb0;  // the view's block row
      if (K >= 0 && K < Bv.nbr) {
        for (int64_t b = Bv.brp[K] + lane; b < Bv.brp[K + 1]; b += 32) {
          const int jb = Bv.bcol[b] - jmin;
          if (jb >= 0 && jb < njw * 32) atomicOr(&jbits[jb >> 5], 1u << (jb & 31));
        }
      }
    }
    __syncthreads();
    if (warp == 0) {  // word prefix of the K bitmap
      const int per = (nkw + 31) / 32;
      const int w0 = min(lane * per, nkw), w1 = min(w0 + per, nkw);
      int c = 0;
      for (int w = w0; w < w1; w++) c += __popc(kbits[w]);
      int v = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL_MASK, v, o);
        if (lane >= o) v += y;
      }
      int run = v - c;
      for (int w = w0; w < w1; w++) {
        kpref[w] = (uint16_t)run;
        run += __popc(kbits[w]);
      }
    } else if (warp == 1) {  // J list in ascending order
      const int per = (njw + 31) / 32;
      const int w0 = min(lane * per, njw), w1 = min(w0 + per, njw);
      int c = 0;
      for (int w = w0; w < w1; w++) c += __popc(jbits[w]);
      int v = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL_MASK, v, o);
        if (lane >= o) v += y;
      }
      const int tot = __shfl_sync(FULL_MASK, v, 31);
      if (lane == 0) s_nj = tot;
      if (tot <= kMJCap) {
        int run = v - c;
        for (int w = w0; w < w1; w++) {
          unsigned m = jbits[w];
          while (m) {
            const int b = __ffs(m) - 1;
            m &= m - 1;
            jlist[run++] = jmin + w * 32 + b;
          }
        }
      }
    }
    __syncthreads();
    const int nj = s_nj;
    const bool over = nj > kMJCap;
    if (over && a.prof && tid == 0) atomicAdd(&a.prof[4], 1ull);  // handed on: J count
    int qbeg = 0;  // first output block computed (SYM: the first J >= I)
    long long obo = 0;
    if constexpr (SYM) {
      if (tid == 0) {
        int nlow = 0, sok = 0;
        long long cjo = 0, ob = 0;
        if (over) {
          atomicOr(so.flag, 1);
        } else {
          int lo = 0, hi = nj;  // first J >= I in the ascending list
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (jlist[mid] < (int)I) lo = mid + 1;
            else hi = mid;
          }
          nlow = lo;
          // the layout from K3c's counts (scanned): both must agree with this list
          cjo = so.cj_off[I];
          ob = so.ob_off[I];
          if (so.nj[I] != nj || so.nj[I] - so.nup[I] != nlow) atomicOr(so.flag, 2);
          else sok = 1;
        }
        s_nlow = nlow;
        s_sok = sok;
        s_cjo = cjo;
        s_obo = ob;
      }
      __syncthreads();
      if (!s_sok) {
        for (int i = tid; i < nkw; i += kMThreads) kbits[i] = 0u;
        for (int i = tid; i < njw; i += kMThreads) jbits[i] = 0u;
        continue;
      }
      for (int q = tid; q < nj; q += kMThreads) so.cj[s_cjo + q] = jlist[q];
      qbeg = s_nlow;
      obo = s_obo;
    }
    // (3) output blocks, one warp each
    double fs = 0.0, q1 = 0.0;
    long long nz = 0, c1 = 0;
    int rkept = 0;  // SYM: kept entries of row g over this lane's output blocks
    unsigned long long nbp = 0;
    if (!over) {
      int32_t *wa = mla + warp * kMML;
      int32_t *wb = mlb + warp * kMML;
      for (int q = qbeg + warp; q < nj; q += kMWarps) {
        const int J = jlist[q];
        // two independent accumulator chains (even / odd matches), summed at the end: the
        // DMMAs of one output block are not one serial dependency chain
        double x0 = 0.0, x1 = 0.0, y0 = 0.0, y1 = 0.0;
        if (a.self_coef != 0.0) {  // self term: A_IJ, if row I of A has block J
          const int kb = J - kmin;
          if (kb >= 0 && kb < nkw * 32 && ((kbits[kb >> 5] >> (kb & 31)) & 1u)) {
            const int ra = kpref[kb >> 5] + __popc(kbits[kb >> 5] & ((1u << (kb & 31)) - 1u));
            const double *ap = abval + (ab0 + ra) * 64;
            x0 = a.self_coef * __ldg(ap + soff0);
            x1 = a.self_coef * __ldg(ap + soff1);
          }
        }
        // column J's block rows K: the block transpose, or (SYM: exactly symmetric T, one
        // view) row J's own block columns, B_KJ read as the transpose of B_JK
        const int64_t t0 = SYM ? Bv.brp[J] : Bv.tp[J], t1 = SYM ? Bv.brp[J + 1] : Bv.tp[J + 1];
        int64_t tb0 = t0;
        while (tb0 < t1) {
          // matches K of row I and column J (ascending K), listed in batches (32-bit block
          // indices: the view holds < 2^31 blocks, checked by the driver)
          int nm = 0;
          for (; tb0 < t1 && nm <= kMML - 32; tb0 += 32) {
            const int64_t tt = tb0 + lane;
            int ra = -1, bidx = 0;
            if (tt < t1) {
              const int kb = (SYM ? Bv.bcol[tt] : Bv.tk[tt] + (int)Bv.kb0) - kmin;
              if (kb >= 0 && kb < nkw * 32 && ((kbits[kb >> 5] >> (kb & 31)) & 1u)) {
                ra = kpref[kb >> 5] + __popc(kbits[kb >> 5] & ((1u << (kb & 31)) - 1u));
                bidx = SYM ? (int)tt : (int)Bv.tb[tt];
              }
            }
            const unsigned m = __ballot_sync(FULL_MASK, ra >= 0);
            if (ra >= 0) {
              const int pos = nm + __popc(m & lanemask_lt());
              wa[pos] = (int)ab0 + ra;
              wb[pos] = bidx;
            }
            nm += __popc(m);
            if (SYM) {  // row J's block columns ascend: none after this chunk's last can match
              const int64_t tl = tb0 + 31 < t1 ? tb0 + 31 : t1 - 1;
              if (Bv.bcol[tl] - kmin >= nkw * 32) tb0 = t1 - 32;  // (tb0 += 32 ends the scan)
            }
          }
          __syncwarp();
          nbp += nm;
          // operands of kMPF block products per set, two sets in turn (P: u.., Q: u+kMPF..);
          // loads past the list are clamped to its last entry (their products are skipped)
          double2 pa[kMPF], qa[kMPF];
          double pl[kMPF], ph[kMPF], ql[kMPF], qh[kMPF];
          const int last = nm - 1;
#define K3M_LOAD(A_, L_, H_, base)                                              \
  _Pragma("unroll") for (int d = 0; d < kMPF; d++) {                           \
    const int e = min((base) + d, last);                                       \
    A_[d] = __ldg(av2 + (size_t)wa[e] * 32 + lane);                            \
    if (SYM) { /* B_KJ[t][g], B_KJ[t+4][g] = B_JK[g][t], B_JK[g][t+4]: A's pair */ \
      const double2 bb = __ldg(av2 + (size_t)wb[e] * 32 + lane);               \
      L_[d] = bb.x;                                                            \
      H_[d] = bb.y;                                                            \
    } else {                                                                   \
      const double *bp = Bv.bval + (size_t)wb[e] * 64 + boff;                  \
      L_[d] = __ldg(bp);                                                       \
      H_[d] = __ldg(bp + 32);                                                  \
    }                                                                          \
  }
#define K3M_MMA(A_, L_, H_)                                                     \
  _Pragma("unroll") for (int d = 0; d < kMPF; d += 2) {                        \
    dmma884(x0, x1, A_[d].x, L_[d]);                                           \
    dmma884(y0, y1, A_[d + 1].x, L_[d + 1]);                                   \
    dmma884(x0, x1, A_[d].y, H_[d]);                                           \
    dmma884(y0, y1, A_[d + 1].y, H_[d + 1]);                                   \
  }
          int u = 0;
          if (nm > 0) { K3M_LOAD(pa, pl, ph, 0) }
          for (; u + 2 * kMPF <= nm; u += 2 * kMPF) {
            K3M_LOAD(qa, ql, qh, u + kMPF)
            K3M_MMA(pa, pl, ph)
            K3M_LOAD(pa, pl, ph, u + 2 * kMPF)
            K3M_MMA(qa, ql, qh)
          }
          // tail: < 2 kMPF products; set P holds u.. (loaded)
          if (u + kMPF <= nm) {
            K3M_LOAD(qa, ql, qh, u + kMPF)
            K3M_MMA(pa, pl, ph)
            u += kMPF;
#pragma unroll
            for (int d = 0; d < kMPF; d++) {
              pa[d] = qa[d];
              pl[d] = ql[d];
              ph[d] = qh[d];
            }
          }
#pragma unroll
          for (int d = 0; d < kMPF; d++)
            if (u + d < nm) {
              dmma884(x0, x1, pa[d].x, pl[d]);
              dmma884(x0, x1, pa[d].y, ph[d]);
            }
#undef K3M_LOAD
#undef K3M_MMA
          __syncwarp();
        }
        x0 += y0;
        x1 += y1;
        if constexpr (SYM) {
          // lane l = 4g + t holds elements e = 2l, 2l + 1 = (g, 2t), (g, 2t + 1) of C_IJ.  The
          // diagonal block owns its upper triangle (K3a mirrors it).  Kept entries (|x| above
          // the floor) packed in element order at the block's slot, their 64-bit mask beside;
          // dropped nonzeros only as sum x^2 and count, each entry counted for itself and its
          // mirror (x 2 off the diagonal)
          const bool dg = J == (int)I;
          const double v0 = (!dg || 2 * t >= g) ? x0 : 0.0, v1 = (!dg || 2 * t + 1 >= g) ? x1 : 0.0;
          const bool k0 = v0 != 0.0 && fabs(v0) > a.floor_tau, k1 = v1 != 0.0 && fabs(v1) > a.floor_tau;
          const double m0 = (dg && 2 * t == g) ? 1.0 : 2.0, m1 = (dg && 2 * t + 1 == g) ? 1.0 : 2.0;
          if (v0 != 0.0) {
            nz += (long long)m0;
            if (!k0) fs += m0 * (v0 * v0);
          }
          if (v1 != 0.0) {
            nz += (long long)m1;
            if (!k1) fs += m1 * (v1 * v1);
          }
          const unsigned long long msk = spread32(__ballot_sync(FULL_MASK, k0)) |
                                         (spread32(__ballot_sync(FULL_MASK, k1)) << 1);
          const int p0 = __popcll(msk & ((1ull << (2 * lane)) - 1ull));
          const size_t blk = (size_t)(obo + q - qbeg);
          double *slot = so.bstore + blk * 64;
          if (k0) slot[p0] = v0;
          if (k1) slot[p0 + (k0 ? 1 : 0)] = v1;
          if (lane == 0) so.bmask[blk] = msk;
          // kept counts of the rows: row g of I here (summed per CTA below), column c's
          // mirrors (strictly above the diagonal of a diagonal block) to row 8J + c now
          if (ROWCNT && so.rowcnt) {  // K3a's row counts (the last squaring only)
            rkept += (k0 ? 1 : 0) + (k1 ? 1 : 0);
            int mc0 = (k0 && (!dg || 2 * t > g)) ? 1 : 0, mc1 = (k1 && (!dg || 2 * t + 1 > g)) ? 1 : 0;
#pragma unroll
            for (int o = 4; o < 32; o <<= 1) {
              mc0 += __shfl_xor_sync(FULL_MASK, mc0, o);
              mc1 += __shfl_xor_sync(FULL_MASK, mc1, o);
            }
            if (g == 0) {
              if (mc0) atomicAdd(reinterpret_cast<unsigned long long *>(so.rowcnt + 8 * (int64_t)J + 2 * t), (unsigned long long)mc0);
              if (mc1) atomicAdd(reinterpret_cast<unsigned long long *>(so.rowcnt + 8 * (int64_t)J + 2 * t + 1), (unsigned long long)mc1);
            }
          }
          continue;
        }
        if (a.divisor != 1.0) {  // Taylor term: (sum_k s_rk h_kj) / i (reading R7)
          x0 = __ddiv_rn(x0, a.divisor);
          x1 = __ddiv_rn(x1, a.divisor);
        }
        // classify (Algorithm 4.1 floor, fused first pass) and pack into scratch
        const bool ok = g < nr;
        bool st0 = false, st1 = false;
        if (ok && x0 != 0.0) {
          nz++;
          if (fabs(x0) > a.floor_tau) {
            st0 = true;
            if (fabs(x0) <= a.eps_g) q1 += x0 * x0;
            else c1++;
          } else {
            fs += x0 * x0;
          }
        }
        if (ok && x1 != 0.0) {
          nz++;
          if (fabs(x1) > a.floor_tau) {
            st1 = true;
            if (fabs(x1) <= a.eps_g) q1 += x1 * x1;
            else c1++;
          } else {
            fs += x1 * x1;
          }
        }
        const unsigned b0m = __ballot_sync(FULL_MASK, st0), b1m = __ballot_sync(FULL_MASK, st1);
        const unsigned mask = spread4((b0m >> (4 * g)) & 0xFu) | (spread4((b1m >> (4 * g)) & 0xFu) << 1);
        const int p0 = __popc(mask & ((1u << (2 * t)) - 1u));
        double *dst = scr + ((size_t)q * 8 + g) * 8;
        if (st0) dst[p0] = x0;
        if (st1) dst[p0 + (st0 ? 1 : 0)] = x1;
        if (t == 0) jm[q * 8 + g] = (uint8_t)mask;
      }
    }
    if (a.prof && lane == 0 && nbp) atomicAdd(&a.prof[0], nbp);
    if constexpr (SYM) {  // the block row's dropped sum x^2 and nonzero count (warps in order)
      fs = warp_sum(fs);
      nz = warp_sum(nz);
      if (ROWCNT) {
        rkept += __shfl_xor_sync(FULL_MASK, rkept, 1);  // row g: its 4 lanes
        rkept += __shfl_xor_sync(FULL_MASK, rkept, 2);
      }
      if (lane == 0) {
        s_fs[warp][0] = fs;
        s_nz[warp][0] = nz;
      }
      if (t == 0) s_c1[warp][g] = rkept;
      __syncthreads();
      if (ROWCNT && so.rowcnt && tid < 8 && 8 * I + tid < nrows) {
        long long c = 0;
        for (int w = 0; w < kMWarps; w++) c += s_c1[w][tid];
        if (c) atomicAdd(reinterpret_cast<unsigned long long *>(so.rowcnt + 8 * I + tid), (unsigned long long)c);
      }
      if (tid == 0) {
        double f = 0.0;
        long long z = 0;
        for (int w = 0; w < kMWarps; w++) {
          f += s_fs[w][0];
          z += s_nz[w][0];
        }
        so.fsI[I] = f;
        so.nzI[I] = z;
      }
      for (int i = tid; i < nkw; i += kMThreads) kbits[i] = 0u;
      for (int i = tid; i < njw; i += kMThreads) jbits[i] = 0u;
      continue;
    }
    // per-row sums: the 4 lanes of a row, then warps in fixed order
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
      fs += __shfl_xor_sync(FULL_MASK, fs, o);
      q1 += __shfl_xor_sync(FULL_MASK, q1, o);
      nz += __shfl_xor_sync(FULL_MASK, nz, o);
      c1 += __shfl_xor_sync(FULL_MASK, c1, o);
    }
    if (t == 0) {
      s_fs[warp][g] = fs;
      s_p1[warp][g] = q1;
      s_nz[warp][g] = nz;
      s_c1[warp][g] = c1;
    }
    __syncthreads();
    // (4) stage each row's kept entries contiguously (warp i: row i)
    if (over) {
      if (tid < nr) fail_rows[atomicAdd(fail_count, 1)] = (int32_t)(r0 + tid);
    } else if (warp < nr) {
      const int i = warp;
      const int64_t r = r0 + i;
      long long tot = 0;
      for (int q0 = 0; q0 < nj; q0 += 32) {
        const int c = q0 + lane < nj ? __popc((unsigned)jm[(q0 + lane) * 8 + i]) : 0;
        tot += __reduce_add_sync(FULL_MASK, c);
      }
      unsigned long long off = 0;
      if (lane == 0) off = atomicAdd(a.pool_used, (unsigned long long)tot);
      off = __shfl_sync(FULL_MASK, off, 0);
      const bool okp = (long long)off + tot <= a.pool_cap;
      if (okp) {
        long long pos = (long long)off;
        for (int q0 = 0; q0 < nj; q0 += 32) {
          const int q = q0 + lane;
          unsigned m = q < nj ? (unsigned)jm[q * 8 + i] : 0u;
          const int c = __popc(m);
          int v = c;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(FULL_MASK, v, o);
            if (lane >= o) v += y;
          }
          if (c > 0) {
            long long p = pos + v - c;
            const double *src = scr + ((size_t)q * 8 + i) * 8;
            const int J = jlist[q];
            for (int e = 0; m; e++, p++) {
              const int j = __ffs(m) - 1;
              m &= m - 1;
              a.pool_col[p] = 8 * J + j;
              a.pool_val[p] = src[e];
            }
          }
          pos += __shfl_sync(FULL_MASK, v, 31);
        }
      }
      if (lane == 0) {
        double f = 0.0, p1 = 0.0;
        long long z = 0, cc = 0;
        for (int w = 0; w < kMWarps; w++) {
          f += s_fs[w][i];
          p1 += s_p1[w][i];
          z += s_nz[w][i];
          cc += s_c1[w][i];
        }
        if (!okp) atomicOr(a.flags, 1);
        a.row_off[r] = (int64_t)off;
        a.row_cnt[r] = tot;
        a.row_fsum[r] = f;
        a.row_nnz[r] = z;
        if (a.row_p1) {
          a.row_p1[r] = p1;
          a.row_c1[r] = cc;
        }
      }
    }
    __syncthreads();
    for (int i = tid; i < nkw; i += kMThreads) kbits[i] = 0u;
    for (int i = tid; i < njw; i += kMThreads) jbits[i] = 0u;
  }
}

void launch_numeric_bsrm(const NumericArgs &a, const BsrView &Bv, int64_t nrows, double *scratch,
                         int32_t *fail_rows, int *fail_count, cudaStream_t st, bool long_lists) {
  if (Bv.nbr_a == 0) return;
  const int smem = bsrm_numeric_smem_bytes();
  KL;
  if (long_lists) {
    cudaFuncSetAttribute(k_numeric_bsrm<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_numeric_bsrm<4, 2><<<a.grid, kMThreads, smem, st>>>(a, Bv, nrows, scratch, fail_rows, fail_count, SymOut{});
  } else {
    cudaFuncSetAttribute(k_numeric_bsrm<2, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_numeric_bsrm<2, 4><<<a.grid, kMThreads, smem, st>>>(a, Bv, nrows, scratch, fail_rows, fail_count, SymOut{});
  }
}
void launch_numeric_bsrm_sym(const NumericArgs &a, const BsrView &Bv, int64_t nrows, double *scratch,
                             const SymOut &so, cudaStream_t st, bool long_lists) {
  if (Bv.nbr_a == 0) return;
  const int smem = bsrm_numeric_smem_bytes();
  KL;
  // (no row counts when the product is handed on in block form: a leaner epilogue)
  auto kf = long_lists ? (so.rowcnt ? k_numeric_bsrm<4, 2, true, true> : k_numeric_bsrm<4, 2, true, false>)
                       : (so.rowcnt ? k_numeric_bsrm<2, 4, true, true> : k_numeric_bsrm<2, 4, true, false>);
  cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kf<<<a.grid, kMThreads, smem, st>>>(a, Bv, nrows, scratch, nullptr, nullptr, so);
}

// K3c: per block row I of the symmetric squaring, |cand(I)| (the union of the block rows K of
// the view at row I's block columns, and row I's own blocks -- K3m's candidate list) and how
// many of them are >= I: exact sizes of K3s's stores, so its layout is a scan (no atomics).
// Warp per block row, a 65536-block-column bitmap per warp; wider unions -> flag 1.
constexpr int kSymCntWarps = 8, kSymCntWords = 2048;
__global__ void __launch_bounds__(kSymCntWarps * 32) k_sym_count(BsrView Bv, int64_t *nj, int64_t *nup,
                                                                 int32_t *wlo, int32_t *whi, int *flag, int words) {
  extern __shared__ unsigned scw[];
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  unsigned *bm = scw + wi * words;
  const int64_t I = (int64_t)blockIdx.x * kSymCntWarps + wi;
  if (I >= Bv.nbr) return;
  const int64_t a0 = Bv.brp[I], a1 = Bv.brp[I + 1];
  // the union's extent (K3s's bitmap window): row I's own blocks and B's block rows K
  int jlo = INT32_MAX, jhi = -1;
  for (int64_t q = a0 + lane; q < a1; q += 32) {
    const int K = Bv.bcol[q];
    jlo = min(jlo, K);
    jhi = max(jhi, K);
    if (K < Bv.nbr && Bv.brp[K + 1] > Bv.brp[K]) {
      jlo = min(jlo, Bv.bcol[Bv.brp[K]]);
      jhi = max(jhi, Bv.bcol[Bv.brp[K + 1] - 1]);
    }
  }
  jlo = __shfl_sync(FULL_MASK, warp_min(jlo), 0);
  jhi = __shfl_sync(FULL_MASK, warp_max(jhi), 0);
  if (lane == 0) {
    wlo[I] = jlo;
    whi[I] = jhi;
  }
  if (jhi < jlo) {
    if (lane == 0) {
      nj[I] = 0;
      nup[I] = 0;
    }
    return;
  }
  const int nw = ((jhi - jlo) >> 5) + 1;
  if (nw > words) {  // wider than this launch's bitmaps: 32 asks for a launch with the largest
    if (lane == 0) {
      atomicOr(flag, words < kSymCntWords ? 32 : 1);
      nj[I] = 0;
      nup[I] = 0;
    }
    return;
  }
  for (int w = lane; w < nw; w += 32) bm[w] = 0u;
  __syncwarp();
  // the 2T term (row I's own blocks), then the block rows K of row I, 4 at a time (their
  // extents loaded together)
  for (int64_t q = a0 + lane; q < a1; q += 32) {
    const int d = Bv.bcol[q] - jlo;
    atomicOr(&bm[d >> 5], 1u << (d & 31));
  }
  for (int64_t q0 = a0; q0 < a1; q0 += 4) {
    int64_t s0[4], s1[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int K = q0 + u < a1 ? Bv.bcol[q0 + u] : (int)Bv.nbr;
      s0[u] = K < Bv.nbr ? Bv.brp[K] : 0;
      s1[u] = K < Bv.nbr ? Bv.brp[K + 1] : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; u++)
      for (int64_t b = s0[u] + lane; b < s1[u]; b += 32) {
        const int d = Bv.bcol[b] - jlo;
        atomicOr(&bm[d >> 5], 1u << (d & 31));
      }
  }
  __syncwarp();
  const int iw = (int)I - jlo;  // bits >= iw are J >= I
  int c = 0, u = 0;
  for (int w = lane; w < nw; w += 32) {
    const unsigned m = bm[w];
    c += __popc(m);
    const int b0 = w * 32;
    if (b0 >= iw) u += __popc(m);
    else if (b0 + 32 > iw) u += __popc(m >> (iw - b0));
  }
  c = __reduce_add_sync(FULL_MASK, c);
  u = __reduce_add_sync(FULL_MASK, u);
  if (lane == 0) {
    nj[I] = c;
    nup[I] = u;
  }
}
void launch_sym_count(const BsrView &Bv, int64_t *nj, int64_t *nup, int32_t *wlo, int32_t *whi, int *flag,
                      cudaStream_t st, bool wide) {
  if (Bv.nbr == 0) return;
  // 512-word bitmaps first (16 KB per CTA: occupancy); rows wider set flag 32 and the driver
  // runs the count again with the largest
  // (test hook: SEXPM_K3C_WORDS sets the first launch's bitmap words)
  const int words = wide ? kSymCntWords
                         : (getenv("SEXPM_K3C_WORDS") ? std::max(1, std::min(kSymCntWords, atoi(getenv("SEXPM_K3C_WORDS")))) : 512);
  const int smem = kSymCntWarps * words * 4;
  cudaFuncSetAttribute(k_sym_count, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  KL;
  k_sym_count<<<(unsigned)((Bv.nbr + kSymCntWarps - 1) / kSymCntWarps), kSymCntWarps * 32, smem, st>>>(Bv, nj, nup, wlo,
                                                                                                   whi, flag, words);
}

// ------------------------------------------------------------------------------------
// K3a: rows of the symmetric squaring from K3s's upper blocks (kernels.cuh SymOut).  One CTA
// per block row I (persistent over I), warp i = row r = 8I + i.  The lower blocks C_JI (J < I)
// are located once per block row (binary search of I in J's ascending list).  A row's values
// in column order: column i of C_JI for J < I, the diagonal block C_II with (i, j < i) read as
// its mirror (j, i) (T~ exactly symmetric), row i of C_IJ for J > I.  Each value x != 0 is
// classified as in the product kernels' flush (Algorithm 4.1 floor and fused first pass);
// the row is counted, reserved in the pool, then staged in a second pass over its values.
// ------------------------------------------------------------------------------------
// K3a's lower blocks: per block row I and lower candidate J < I (position p in cand(I)), the
// global index of the upper block (J, I) -- a binary search of I in J's ascending list -- to
// lidx[cj_off[I] + p] (warp per block row; flag 4 when absent: the pattern is not symmetric)
__global__ void k_sym_lidx(SymOut so, int64_t nbr) {
  const int64_t I = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (I >= nbr) return;
  const int nlow = (int)(so.nj[I] - so.nup[I]);
  const int64_t c0 = so.cj_off[I];
  for (int p = lane; p < nlow; p += 32) {
    const int J = so.cj[c0 + p];
    const int32_t *lj = so.cj + so.cj_off[J];
    const int njJ = (int)so.nj[J], nlJ = (int)(so.nj[J] - so.nup[J]);
    int lo = nlJ, hi = njJ;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (lj[mid] < (int)I) lo = mid + 1;
      else hi = mid;
    }
    int idx = -1;
    if (lo < njJ && lj[lo] == (int)I) idx = (int)(so.ob_off[J] + (lo - nlJ));
    else atomicOr(so.flag, 4);
    so.lidx[c0 + p] = idx;
  }
}
void launch_sym_lidx(const SymOut &so, int64_t nbr, cudaStream_t st) {
  if (nbr == 0) return;
  KL;
  k_sym_lidx<<<grid_for(nbr * 32, kThreads), kThreads, 0, st>>>(so, nbr);
}
constexpr int kAsmThreads = 256;
__global__ void __launch_bounds__(kAsmThreads, 4) k_sym_assemble(NumericArgs a, SymOut so, int64_t nbr,
                                                                 int64_t nrows) {
  __shared__ int32_t s_col[kAsmThreads / 32][256];  // a chunk's entries (32 blocks x 8)
  __shared__ double s_val[kAsmThreads / 32][256];
  const int tid = threadIdx.x, lane = tid & 31, i = tid >> 5;
  const unsigned long long colm = 0x0101010101010101ull << i;  // column i of a block
  for (int64_t I = blockIdx.x; I < nbr; I += gridDim.x) {
    const int nj = (int)so.nj[I], nlow = (int)(so.nj[I] - so.nup[I]);
    const int64_t c0 = so.cj_off[I];
    const int32_t *cj = so.cj + c0;
    const int64_t obo = so.ob_off[I];
    const int64_t r = 8 * I + i;
    if (r >= nrows) continue;
    const bool hasdiag = nlow < nj && cj[nlow] == (int)I;
    // block q of row i: its global index, mask, and the bits of row i's entries j = 0..7 (the
    // element of the block: (j, i) for a lower block or j < i of the diagonal one, else (i, j))
    auto blk_of = [&](int q, unsigned long long &m, int &kind) -> int64_t {
      int64_t b;
      if (q < nlow) {
        b = so.lidx[c0 + q];  // k_sym_lidx
        kind = 0;
      } else {
        b = obo + (q - nlow);
        kind = (q == nlow && hasdiag) ? 1 : 2;
      }
      m = b >= 0 ? __ldg(so.bmask + b) : 0ull;
      return b;
    };
    auto bit_of = [&](int kind, int j) { return (kind == 0 || (kind == 1 && j < i)) ? 8 * j + i : 8 * i + j; };
    // the row's kept entries at its scanned offset (K3s counted them), in column order
    const long long tot = so.rowcnt[r];
    const int64_t off = so.rowoff[r];
    const bool okp = off + tot <= a.pool_cap;
    double q1 = 0.0;   // the fused first pass: x^2 of kept |x| <= eps_g
    long long c1 = 0;  // kept |x| > eps_g (the compaction's count when one pass sufficed)
    if (okp) {
      long long pos = (long long)off;
      // the next chunk's block index, mask and column are fetched before this chunk's stores
      int64_t nb = 0;
      unsigned long long nm = 0;
      int nk = 2, nJ = 0;
      if (lane < nj) {
        nb = blk_of(lane, nm, nk);
        nJ = cj[lane];
      }
      for (int q0 = 0; q0 < nj; q0 += 32) {
        const int q = q0 + lane;
        const unsigned long long m = nm;
        const int kind = nk, J = nJ;
        const int64_t b = nb;
        if (q0 + 32 + lane < nj) {
          nb = blk_of(q0 + 32 + lane, nm, nk);
          nJ = cj[q0 + 32 + lane];
        }
        unsigned rb = 0;  // row i's kept entries j (bits)
        if (q < nj) {
#pragma unroll
          for (int j = 0; j < 8; j++) rb |= (unsigned)((m >> bit_of(kind, j)) & 1ull) << j;
        }
        const int c = __popc(rb);
        int x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(FULL_MASK, x, o);
          if (lane >= o) x += y;
        }
        if (c > 0) {  // all of the block's loads in flight at once (predicated, unrolled)
          const double *slot = so.bstore + (size_t)b * 64;
          double v[8];
          if (kind == 2) {  // row i of an upper block: its kept values are consecutive
            const double *sv = slot + __popcll(m & ((1ull << (8 * i)) - 1ull));
#pragma unroll
            for (int k = 0; k < 8; k++) v[k] = k < c ? __ldg(sv + k) : 0.0;
          } else {
#pragma unroll
            for (int j = 0; j < 8; j++) {
              const int e = bit_of(kind, j);
              v[j] = ((rb >> j) & 1u) ? __ldg(slot + __popcll(m & ((1ull << e) - 1ull))) : 0.0;
            }
          }
          // staged in shared memory at the chunk-local position, copied out coalesced below
          int p = x - c;
          if (kind == 2) {  // the k-th value is the k-th set bit's column
            unsigned rbm = rb;
#pragma unroll
            for (int k = 0; k < 8; k++)
              if (k < c) {
                const int j = __ffs(rbm) - 1;
                rbm &= rbm - 1;
                s_col[i][p + k] = 8 * J + j;
                s_val[i][p + k] = v[k];
                if (fabs(v[k]) <= a.eps_g) q1 += v[k] * v[k];
                else c1++;
              }
          } else {
#pragma unroll
            for (int j = 0; j < 8; j++)
              if ((rb >> j) & 1u) {
                s_col[i][p] = 8 * J + j;
                s_val[i][p] = v[j];
                if (fabs(v[j]) <= a.eps_g) q1 += v[j] * v[j];
                else c1++;
                p++;
              }
          }
        }
        const int ct = __shfl_sync(FULL_MASK, x, 31);  // the chunk's entries
        __syncwarp();
        for (int k = lane; k < ct; k += 32) {
          a.pool_col[pos + k] = s_col[i][k];
          a.pool_val[pos + k] = s_val[i][k];
        }
        __syncwarp();
        pos += ct;
      }
      if (lane == 0 && pos != off + tot) atomicOr(so.flag, 16);  // K3s's count disagrees
    }
    q1 = warp_sum(q1);
    c1 = warp_sum(c1);
    if (lane == 0) {
      if (!okp) atomicOr(a.flags, 1);
      a.row_off[r] = (int64_t)off;
      a.row_cnt[r] = tot;
      // Algorithm 4.1's floor sum and the distinct count per block row (K3s), on its first row
      a.row_fsum[r] = i == 0 ? so.fsI[I] : 0.0;
      a.row_nnz[r] = i == 0 ? so.nzI[I] : 0;
      if (a.row_p1) {  // the fused first pass per block row (K3s), on its first row
        a.row_p1[r] = q1;
        a.row_c1[r] = c1;
      }
    }
  }
}
void launch_sym_assemble(const NumericArgs &a, const SymOut &so, int64_t nbr, int64_t nrows, int grid,
                         cudaStream_t st) {
  if (nbr == 0) return;
  KL;
  k_sym_assemble<<<grid, kAsmThreads, 0, st>>>(a, so, nbr, nrows);
}


// ------------------------------------------------------------------------------------
// The symmetric path between two squarings: the filtered iterate handed on in block form.
//  k_sym_pass: Algorithm 4.1's pass sum over K3s's kept values (each entry and its mirror),
//    sum x^2 over |x| <= tau, per block row (warp per block row, fixed order).
//  k_sym_fin<WRITE>: the next squaring's BSR-8 view (fragment order) straight from the block
//    store: per block row I the candidate blocks J (lower ones as the transposes of (J, I), the
//    diagonal one mirrored from its upper triangle) keeping |x| > tau; COUNT: non-empty blocks
//    per block row and the iterate's statistics (nnz, sum_r nnz_r^2 for the next product count,
//    ||I + T^||_F^2, bandwidths); WRITE: block columns and values.  Warp per block row, the
//    whole warp on one block at a time (lane l: elements 2l, 2l + 1), the next block's mask
//    fetched ahead.
//  k_bsr_to_csr<WRITE>: CSR rows of a fragment-order BSR view (the fallback when the next
//    symmetric product cannot run on the view).
// ------------------------------------------------------------------------------------
__global__ void k_sym_pass(SymOut so, int64_t nbr, double tau, double *psum) {
  const int64_t I = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (I >= nbr) return;
  const int nup = (int)so.nup[I], nlow = (int)(so.nj[I] - so.nup[I]);
  const int32_t *cj = so.cj + so.cj_off[I] + nlow;
  const int64_t obo = so.ob_off[I];
  double sacc = 0.0;
  for (int u = 0; u < nup; u++) {  // the warp on one block: lane l holds kept values l, l + 32
    const unsigned long long m = __ldg(so.bmask + obo + u);
    const int c = __popcll(m);
    const bool dg = cj[u] == (int)I;
    const double *slot = so.bstore + (size_t)(obo + u) * 64;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int e = lane + 32 * h;
      if (e < c) {
        const double x = __ldg(slot + e);
        if (fabs(x) <= tau) {
          double mult = 2.0;
          if (dg) {  // the e-th set bit's element: on the diagonal it counts once
            unsigned long long mm = m;
            for (int k = 0; k < e; k++) mm &= mm - 1;
            if ((__ffsll((long long)mm) - 1) % 9 == 0) mult = 1.0;
          }
          sacc += mult * (x * x);
        }
      }
    }
  }
  sacc = warp_sum(sacc);
  if (lane == 0) psum[I] = sacc;
}
void launch_sym_pass(const SymOut &so, int64_t nbr, double tau, double *psum, cudaStream_t st) {
  if (nbr == 0) return;
  KL;
  k_sym_pass<<<grid_for(nbr * 32, kThreads), kThreads, 0, st>>>(so, nbr, tau, psum);
}

// COUNT: warp per block row I over its upper blocks only (each entry with its mirror): the
// block's elements kept after tau, a flag per upper block (non-empty), the non-empty block
// counts of I and of J (the mirror, atomics), kept counts per row (own rows summed per warp,
// mirror rows by atomics), the block row's ||I + T^||_F^2 share (x^2 twice off the diagonal,
// (1 + x)^2 on it, 1 per row without a kept diagonal) and bandwidth
__global__ void __launch_bounds__(kThreads) k_sym_fin_count(SymOut so, int64_t nbr, int64_t nrows, double tau,
                                                            SymFin f) {
  const int64_t I = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (I >= nbr) return;
  const int nup = (int)so.nup[I], nlow = (int)(so.nj[I] - so.nup[I]);
  const int32_t *cj = so.cj + so.cj_off[I] + nlow;
  const int64_t obo = so.ob_off[I];
  const int r = lane >> 2, t = lane & 3;  // stored elements (r, 2t), (r, 2t + 1)
  int rown = 0, nblk = 0, diagk = 0;
  double s2 = 0.0;
  long long l1 = 0;
  for (int u = 0; u < nup; u++) {
    const unsigned long long m = __ldg(so.bmask + obo + u);
    if (m == 0ull) {
      if (lane == 0) f.flag[obo + u] = 0;
      continue;
    }
    const int J = cj[u];
    const bool dg = J == (int)I;
    const double *slot = so.bstore + (size_t)(obo + u) * 64;
    bool k[2];
    double v[2];
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int c = 2 * t + h, se = 8 * r + c;
      const bool present = (m >> se) & 1ull;
      v[h] = present ? __ldg(slot + __popcll(m & ((1ull << se) - 1ull))) : 0.0;
      k[h] = present && fabs(v[h]) > tau;  // (the diagonal block stores only c >= r)
    }
    const unsigned any = __ballot_sync(FULL_MASK, k[0] || k[1]);
    if (lane == 0) f.flag[obo + u] = any ? 1 : 0;
    if (!any) continue;
    nblk++;
    int mc[2] = {0, 0};
#pragma unroll
    for (int h = 0; h < 2; h++)
      if (k[h]) {
        const int c = 2 * t + h;
        rown++;
        if (dg && c == r) {
          s2 += (1.0 + v[h]) * (1.0 + v[h]);
          diagk = 1;
        } else {
          s2 += 2.0 * (v[h] * v[h]);  // the entry and its mirror
          mc[h] = 1;
          l1 = max(l1, (long long)(8 * (int64_t)J + c - (8 * I + r)));
        }
      }
    // mirrors: column c of (I, J) is row 8J + c's (the 8 lanes of a column pair summed)
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      mc[0] += __shfl_xor_sync(FULL_MASK, mc[0], o);
      mc[1] += __shfl_xor_sync(FULL_MASK, mc[1], o);
    }
    if (r == 0) {
      if (mc[0]) atomicAdd(reinterpret_cast<unsigned long long *>(f.rowcnt + 8 * (int64_t)J + 2 * t), (unsigned long long)mc[0]);
      if (mc[1]) atomicAdd(reinterpret_cast<unsigned long long *>(f.rowcnt + 8 * (int64_t)J + 2 * t + 1), (unsigned long long)mc[1]);
    }
    if (!dg && lane == 0) atomicAdd(reinterpret_cast<unsigned long long *>(f.bcnt + J), 1ull);
  }
  // own rows: the 4 lanes of each row
  rown += __shfl_xor_sync(FULL_MASK, rown, 1);
  rown += __shfl_xor_sync(FULL_MASK, rown, 2);
  diagk |= __shfl_xor_sync(FULL_MASK, diagk, 1);
  diagk |= __shfl_xor_sync(FULL_MASK, diagk, 2);
  const bool rowok = 8 * I + r < nrows;
  if (t == 0 && rowok && rown)
    atomicAdd(reinterpret_cast<unsigned long long *>(f.rowcnt + 8 * I + r), (unsigned long long)rown);
  const int nodiag = __popc(__ballot_sync(FULL_MASK, t == 0 && rowok && !diagk));
  s2 = warp_sum(s2);
  l1 = warp_max(l1);
  if (lane == 0) {
    atomicAdd(reinterpret_cast<unsigned long long *>(f.bcnt + I), (unsigned long long)nblk);
    f.rsI[I] = s2 + (double)nodiag;
    f.l1I[I] = l1;
  }
}

// WRITE: warp per block row I over its candidates in column order; the non-empty ones (the
// upper block's flag, a lower block's mirror's flag) are written, the warp on one block at a
// time: lane l writes elements (r, 2t), (r, 2t + 1) in fragment order, zeros where dropped
__global__ void __launch_bounds__(kThreads) k_sym_fin_write(SymOut so, int64_t nbr, int64_t nrows, double tau,
                                                            SymFin f) {
  const int64_t I = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (I >= nbr) return;
  const int nj = (int)so.nj[I], nlow = (int)(so.nj[I] - so.nup[I]);
  const int64_t c0 = so.cj_off[I];
  const int32_t *cj = so.cj + c0;
  const int64_t obo = so.ob_off[I];
  const bool hasdiag = nlow < nj && cj[nlow] == (int)I;
  const int r = lane >> 2, t = lane & 3;
  const bool rowok = 8 * I + r < nrows;
  const int f0 = 2 * (4 * r + ((2 * t) & 3)) + ((2 * t) >> 2);
  const int f1 = 2 * (4 * r + ((2 * t + 1) & 3)) + ((2 * t + 1) >> 2);
  int64_t pos = f.brp[I];
  for (int q0 = 0; q0 < nj; q0 += 32) {
    const int q = q0 + lane;
    int64_t b = -1;
    int fl = 0;
    if (q < nj) {
      b = q < nlow ? (int64_t)so.lidx[c0 + q] : obo + (q - nlow);
      fl = b >= 0 ? f.flag[b] : 0;
    }
    unsigned nem = __ballot_sync(FULL_MASK, fl != 0);
    while (nem) {  // the chunk's non-empty blocks, in order, the whole warp on each
      const int src = __ffs(nem) - 1;
      nem &= nem - 1;
      const int qq = q0 + src;
      const int64_t bb = __shfl_sync(FULL_MASK, b, src);
      const int kind = qq < nlow ? 0 : ((qq == nlow && hasdiag) ? 1 : 2);
      const unsigned long long m = __ldg(so.bmask + bb);
      const double *slot = so.bstore + (size_t)bb * 64;
      double v[2];
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int c = 2 * t + h;
        const int se = (kind == 0 || (kind == 1 && c < r)) ? 8 * c + r : 8 * r + c;
        const bool present = (m >> se) & 1ull;
        const double x = present ? __ldg(slot + __popcll(m & ((1ull << se) - 1ull))) : 0.0;
        v[h] = (present && rowok && fabs(x) > tau) ? x : 0.0;
      }
      double *dst = f.bval + (size_t)pos * 64;
      dst[f0] = v[0];
      dst[f1] = v[1];
      if (lane == 0) f.bcol[pos] = cj[qq];
      pos++;
    }
  }
}
void launch_sym_fin(const SymOut &so, int64_t nbr, int64_t nrows, double tau, const SymFin &f, bool write,
                    cudaStream_t st) {
  if (nbr == 0) return;
  KL;
  if (write)
    k_sym_fin_write<<<grid_for(nbr * 32, kThreads), kThreads, 0, st>>>(so, nbr, nrows, tau, f);
  else
    k_sym_fin_count<<<grid_for(nbr * 32, kThreads), kThreads, 0, st>>>(so, nbr, nrows, tau, f);
}
// sum and sum of squares of the rows' counts (the next product count)
__global__ void k_rowcnt_sums(const int64_t *rc, int64_t n, int64_t *sq) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < n) sq[r] = rc[r] * rc[r];
}
void launch_rowcnt_sq(const int64_t *rc, int64_t n, int64_t *sq, cudaStream_t st) {
  if (n == 0) return;
  KL;
  k_rowcnt_sums<<<grid_for(n, kThreads), kThreads, 0, st>>>(rc, n, sq);
}

template <bool WRITE>
__global__ void k_bsr_to_csr(BsrView V, int64_t nrows, int64_t *cnt, const int64_t *rp, int32_t *col,
                             double *val) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= nrows) return;
  const int64_t I = r >> 3;
  const int i = (int)(r & 7);
  const int64_t b0 = V.brp[I], b1 = V.brp[I + 1];
  int64_t pos = WRITE ? rp[r] : 0;
  for (int64_t bb = b0; bb < b1; bb += 32) {
    const int64_t b = bb + lane;
    double x[8];
    unsigned nzm = 0;
    if (b < b1) {
      const double *blkv = V.bval + (size_t)b * 64;
#pragma unroll
      for (int c = 0; c < 8; c++) {
        x[c] = __ldg(blkv + 2 * (4 * i + (c & 3)) + (c >> 2));
        if (x[c] != 0.0) nzm |= 1u << c;
      }
    }
    const int cntb = __popc(nzm);
    int xs = cntb;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL_MASK, xs, o);
      if (lane >= o) xs += y;
    }
    if (WRITE && cntb) {
      int64_t p = pos + xs - cntb;
      const int J = V.bcol[b];
#pragma unroll
      for (int c = 0; c < 8; c++)
        if ((nzm >> c) & 1u) {
          col[p] = 8 * J + c;
          val[p] = x[c];
          p++;
        }
    }
    pos += __shfl_sync(FULL_MASK, xs, 31);
  }
  if (!WRITE && lane == 0) cnt[r] = pos;
}
void launch_bsr_to_csr(const BsrView &V, int64_t nrows, int64_t *cnt, const int64_t *rp, int32_t *col,
                       double *val, cudaStream_t st) {
  if (nrows == 0) return;
  KL;
  if (rp)
    k_bsr_to_csr<true><<<grid_for(nrows * 32, kThreads), kThreads, 0, st>>>(V, nrows, cnt, rp, col, val);
  else
    k_bsr_to_csr<false><<<grid_for(nrows * 32, kThreads), kThreads, 0, st>>>(V, nrows, cnt, rp, col, val);
}

// symmetric part from the upper triangle (kernels.cuh launch_sym_intersect); warp per row
__device__ __forceinline__ int64_t csr_find(const CsrView &A, int64_t row, int32_t c) {
  int64_t lo = A.rp[row], hi = A.rp[row + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (A.col[mid] < c) lo = mid + 1;
    else hi = mid;
  }
  return (lo < A.rp[row + 1] && A.col[lo] == c) ? lo : -1;
}
template <bool WRITE>
__global__ void k_sym_intersect(CsrView A, int64_t *cnt, const int64_t *rp_out, int32_t *col_out,
                                double *val_out) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= A.nrows) return;
  const int64_t p0 = A.rp[r], p1 = A.rp[r + 1];
  int64_t out = WRITE ? rp_out[r] : 0;
  for (int64_t b = p0; b < p1; b += 32) {
    const int64_t p = b + lane;
    bool keep = false;
    double v = 0.0;
    if (p < p1) {
      const int32_t c = A.col[p];
      if (c >= r) {
        keep = true;
        v = A.val[p];
      } else {
        const int64_t q = csr_find(A, c, (int32_t)r);
        if (q >= 0) {
          keep = true;
          v = A.val[q];
        }
      }
    }
    const unsigned m = __ballot_sync(FULL_MASK, keep);
    if (WRITE && keep) {
      const int64_t o = out + __popc(m & lanemask_lt());
      col_out[o] = A.col[p];
      val_out[o] = v;
    }
    out += __popc(m);
  }
  if (!WRITE && lane == 0) cnt[r] = out;
}
void launch_sym_intersect(const CsrView &A, int64_t *cnt, const int64_t *rp_out, int32_t *col_out,
                          double *val_out, cudaStream_t st) {
  if (A.nrows == 0) return;
  KL;
  if (rp_out)
    k_sym_intersect<true><<<grid_for(A.nrows * 32, kThreads), kThreads, 0, st>>>(A, cnt, rp_out, col_out, val_out);
  else
    k_sym_intersect<false><<<grid_for(A.nrows * 32, kThreads), kThreads, 0, st>>>(A, cnt, rp_out, col_out, val_out);
}



// ------------------------------------------------------------------------------------
// Diagonal structure of H0 (plan time): offsets d = j - k present anywhere in H0, as a
// bitmap over [-(n-1), n-1]; then the diagonals h_d[k] = H0(k, k + d).
// ------------------------------------------------------------------------------------
__global__ void k_mark_offsets(CsrView H, unsigned *bits, int64_t n) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= H.nrows) return;
  const int64_t row = H.row0 + w;
  for (int64_t p = H.rp[w] + lane; p < H.rp[w + 1]; p += 32) {
    const int64_t b = (int64_t)H.col[p] - row + (n - 1);
    // a stencil has a handful of offsets: almost every bit is set already, so read first
    // (the atomics on those few words would serialise)
    const unsigned m = 1u << (b & 31);
    if (!(*reinterpret_cast<volatile unsigned *>(&bits[b >> 5]) & m)) atomicOr(&bits[b >> 5], m);
  }
}
void launch_mark_offsets(const CsrView &H, unsigned *bits, int64_t n, cudaStream_t st) {
  if (H.nrows == 0) return;
  KL;
  k_mark_offsets<<<grid_for(H.nrows * 32, kThreads), kThreads, 0, st>>>(H, bits, n);
}
struct DiaOffsets {
  int32_t off[kDiaMax];
  int nd;
};
__global__ void k_fill_dia(CsrView H, DiaOffsets O, double *dia, int64_t n) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= H.nrows) return;
  const int64_t row = H.row0 + w;
  for (int64_t p = H.rp[w] + lane; p < H.rp[w + 1]; p += 32) {
    const int64_t d = (int64_t)H.col[p] - row;
    for (int i = 0; i < O.nd; i++)
      if (O.off[i] == d) dia[(int64_t)i * n + row] = H.val[p];
  }
}
void launch_fill_dia(const CsrView &H, const int32_t *off_host, int nd, double *dia, int64_t n,
                     cudaStream_t st) {
  if (H.nrows == 0 || nd == 0) return;
  DiaOffsets O;
  for (int i = 0; i < kDiaMax; i++) O.off[i] = i < nd ? off_host[i] : 0;
  O.nd = nd;
  KL;
  k_fill_dia<<<grid_for(H.nrows * 32, kThreads), kThreads, 0, st>>>(H, O, dia, n);
}

// ------------------------------------------------------------------------------------
// K5d Taylor term by DIAGONAL PUSH: S~(r, j) = (sum_k s_rk h0_kj) / i  (Eq. 4.11, P:306,
// Alg. 4.2 step 3 P:412), for an H0 with few distinct diagonal offsets d = j - k (grid
// stencils: 3 in 1D, 5 in 2D, 7 in 3D).  H0 is held as diagonals h_d[k] = H0(k, k + d)
// (zero where absent), offsets sorted DESCENDING.
//
// One warp per row r of S^.  Lanes take 32 consecutive entries (k, s_rk) of the row; for
// each offset d in turn every lane adds s_rk * h_d[k] into column j = k + d.  Lanes hold
// distinct k, so within one offset they write distinct columns (no atomics, no conflicts;
// __syncwarp between offsets orders the shared-memory updates).  For a fixed column j the
// contributions arrive with k = j - d ascending (offsets descending inside a chunk, chunks
// ascending), i.e. exactly the oracle's order: acc = acc + (s_rk * h_kj) with _rn
// intrinsics, then / i -- S~ is bit-identical to the oracle's.
//
// Accumulator: pages of 2^sh columns aligned to absolute multiples of 2^sh.  A first pass
// marks the pages the row can reach in a bitmap over the row's span; a popcount scan of
// the bitmap numbers the marked pages in column order, so slot(j) = 2^sh * rank(page(j)) +
// (j mod 2^sh) with two shared-memory loads and a popc, and the flush walks the slots in
// column order (rows come out sorted).  The flush divides by i, classifies against the
// Algorithm 4.1 floor (see k_numeric) and stages (col, val) in the pool.  Rows that do not
// fit (span or slot capacity) go to the fail list (pull kernel).
// ------------------------------------------------------------------------------------
constexpr int kDWarps = 4;            // warps per CTA
constexpr int kDPageWords = 256;      // page bitmap: 8192 pages per row
constexpr int kDMaxDiag = kDiaMax;

int taylor_dia_smem_bytes(int slots) {
  return kDWarps * (slots * 8 + kDPageWords * 4 + kDPageWords * 2 + (slots >> 3) * 2 + 16);
}

template <int MAXD, bool EXACT>  // bound on the number of diagonals (EXACT: == D.ndiag)
__global__ void __launch_bounds__(kDWarps * 32) k_taylor_dia(NumericArgs a, DiaView D, int slots,
                                                             int32_t *fail_rows, int *fail_count) {
  extern __shared__ double dsm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int max_pages = slots >> 3;
  const size_t wbytes = (size_t)slots * 8 + kDPageWords * 4 + kDPageWords * 2 + (size_t)max_pages * 2 + 16;
  char *base = reinterpret_cast<char *>(dsm) + wbytes * wib;
  double *acc = reinterpret_cast<double *>(base);
  unsigned *pbits = reinterpret_cast<unsigned *>(acc + slots);
  uint16_t *pref = reinterpret_cast<uint16_t *>(pbits + kDPageWords);
  uint16_t *plist = pref + kDPageWords;
  __shared__ int32_t s_doff[kDMaxDiag];
  if (threadIdx.x < kDMaxDiag) s_doff[threadIdx.x] = threadIdx.x < D.ndiag ? D.off[threadIdx.x] : 0;
  for (int i = lane; i < slots; i += 32) acc[i] = 0.0;
  for (int i = lane; i < kDPageWords; i += 32) pbits[i] = 0u;
  __syncthreads();
  const int nd = EXACT ? MAXD : D.ndiag;
  const int32_t dmin = D.dmin, dmax = D.dmax;
  const int n = (int)D.n;  // columns are int32: every column index below fits 32 bits
  unsigned long long prods = 0;
  int need = 0;              // most slots a row of this warp needed
  constexpr int kBatch = 4;  // rows taken per scheduler atomic
  for (;;) {
    int idx0 = 0;
    if (lane == 0) idx0 = atomicAdd(a.row_counter, kBatch);
    idx0 = __shfl_sync(FULL_MASK, idx0, 0);
    if (idx0 >= a.nlist) break;
    const int idx1 = idx0 + kBatch < a.nlist ? idx0 + kBatch : (int)a.nlist;
    for (int idx = idx0; idx < idx1; idx++) {
      const int64_t r = a.order ? (int64_t)a.order[idx] : (int64_t)idx;
      const int64_t p0 = a.A.rp[r], p1 = a.A.rp[r + 1];
      const int nx = (int)(p1 - p0);
      if (nx == 0) {
        if (lane == 0) {
          a.row_off[r] = 0;
          a.row_cnt[r] = 0;
          a.row_fsum[r] = 0.0;
          a.row_nnz[r] = 0;
          if (a.row_p1) {
            a.row_p1[r] = 0.0;
            a.row_c1[r] = 0;
          }
        }
        continue;
      }
      int lo = a.A.col[p0] + dmin, hi = a.A.col[p1 - 1] + dmax;
      lo = lo < 0 ? 0 : lo;
      hi = hi > n - 1 ? n - 1 : hi;
      int sh = 3;
      while (sh < 7 && ((hi >> sh) - (lo >> sh)) >= kDPageWords * 32) sh++;
      const int pg0 = lo >> sh;
      const int npg = (int)((hi >> sh) - pg0 + 1);
      bool fail = sh >= 7;
      // (1) mark reachable pages
      // lanes hold ascending k, so equal pages are adjacent lanes: a lane marks its page only
      // if the lane below holds a different one (one atomic per page run)
      if (!fail) {
        int kn = lane < nx ? a.A.col[p0 + lane] : -1;
        for (int c0 = 0; c0 < nx; c0 += 32) {
          const int k = kn;
          kn = c0 + 32 + lane < nx ? a.A.col[p0 + c0 + 32 + lane] : -1;
#pragma unroll
          for (int di = 0; di < MAXD; di++) {
            if (di < nd) {
              const int j = k + s_doff[di];
              const bool v = k >= 0 && j >= 0 && j < n;
              const int pg = v ? (j >> sh) - pg0 : -1;
              const int pgl = __shfl_up_sync(FULL_MASK, pg, 1);
              if (v && (lane == 0 || pgl != pg)) atomicOr(&pbits[pg >> 5], 1u << (pg & 31));
            }
          }
        }
        __syncwarp();
      }
      // (2) number the marked pages in column order
      const int nwords = (npg + 31) >> 5;
      int npages = 0;
      if (!fail) {
        int cnt = 0;
        for (int w = lane * 8; w < lane * 8 + 8; w++) cnt += w < nwords ? __popc(pbits[w]) : 0;
        int v = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          int y = __shfl_up_sync(FULL_MASK, v, o);
          if (lane >= o) v += y;
        }
        npages = __shfl_sync(FULL_MASK, v, 31);
        need = max(need, npages << sh);
        if ((npages << sh) > slots) {
          fail = true;
        } else {
          int run = v - cnt;
          for (int w = lane * 8; w < lane * 8 + 8; w++) {
            if (w < nwords) {
              pref[w] = (uint16_t)run;
              unsigned m = pbits[w];
              while (m) {
                const int b = __ffs(m) - 1;
                m &= m - 1;
                plist[run++] = (uint16_t)(w * 32 + b);
              }
            }
          }
        }
        __syncwarp();
      }
      if (fail) {
        for (int w = lane; w < nwords; w += 32) pbits[w] = 0u;
        if (lane == 0) fail_rows[atomicAdd(fail_count, 1)] = (int32_t)r;
        __syncwarp();
        continue;
      }
      // (3) products, offsets descending inside each chunk of 32 entries; the next chunk's
      // entries and diagonal values are loaded while this chunk is accumulated
      const int pmask = (1 << sh) - 1;
      int kc = -1;
      double sc = 0.0, hc[MAXD];
      auto load_chunk = [&](int c0, int &k, double &sv, double (&h)[MAXD]) {
        const int t = c0 + lane;
        const bool in = t < nx;
        k = in ? a.A.col[p0 + t] : -1;
        sv = in ? a.A.val[p0 + t] : 0.0;
        const double *hk = D.val + (in ? k : 0);
#pragma unroll
        for (int di = 0; di < MAXD; di++) h[di] = (di < nd && in) ? hk[(size_t)di * (size_t)n] : 0.0;
      };
      load_chunk(0, kc, sc, hc);
      for (int c0 = 0; c0 < nx; c0 += 32) {
        int kn;
        double sn, hn[MAXD];
        if (c0 + 32 < nx) load_chunk(c0 + 32, kn, sn, hn);
#pragma unroll
        for (int di = 0; di < MAXD; di++) {
          if (di < nd) {
            if (hc[di] != 0.0) {
              const int j = kc + s_doff[di];
              const int pg = (j >> sh) - pg0;
              const unsigned wd = pbits[pg >> 5];
              const int rank = pref[pg >> 5] + __popc(wd & ((1u << (pg & 31)) - 1u));
              const int o = (rank << sh) + (int)(j & pmask);
              acc[o] = __dadd_rn(acc[o], __dmul_rn(sc, hc[di]));
              prods++;
            }
            __syncwarp();
          }
        }
        if (c0 + 32 < nx) {
          kc = kn;
          sc = sn;
#pragma unroll
          for (int di = 0; di < MAXD; di++) hc[di] = hn[di];
        }
      }
      // (4) flush in column order: divide, classify, count
      const int total = npages << sh;
      int nst = 0;
      double fs = 0.0, q1 = 0.0;
      long long nnzu = 0, c1 = 0;
      for (int s0 = lane; s0 < total; s0 += 32) {
        double x = acc[s0];
        if (x != 0.0) {
          x = x / a.divisor;
          acc[s0] = x;
          if (x != 0.0) {
            nnzu++;
            if (fabs(x) > a.floor_tau) {
              nst++;
              if (fabs(x) <= a.eps_g) q1 += x * x;
              else c1++;
            } else {
              fs += x * x;
            }
          }
        }
      }
      nst = __reduce_add_sync(FULL_MASK, nst);
      fs = warp_sum(fs);
      nnzu = warp_sum(nnzu);
      q1 = warp_sum(q1);
      c1 = warp_sum(c1);
      unsigned long long off = 0;
      if (lane == 0) off = atomicAdd(a.pool_used, (unsigned long long)nst);
      off = __shfl_sync(FULL_MASK, off, 0);
      const bool ok = (long long)off + nst <= a.pool_cap;
      long long pos = (long long)off;
      for (int b0 = 0; b0 < total; b0 += 32) {
        const int s0 = b0 + lane;
        double x = 0.0;
        if (s0 < total) {
          x = acc[s0];
          acc[s0] = 0.0;
        }
        const bool st = x != 0.0 && fabs(x) > a.floor_tau;
        const unsigned m = __ballot_sync(FULL_MASK, st);
        if (st && ok) {
          const long long q = pos + __popc(m & lanemask_lt());
          a.pool_col[q] = ((pg0 + plist[s0 >> sh]) << sh) + (s0 & pmask);
          a.pool_val[q] = x;
        }
        pos += __popc(m);
      }
      for (int w = lane; w < nwords; w += 32) pbits[w] = 0u;
      if (lane == 0) {
        if (!ok) atomicOr(a.flags, 1);
        a.row_off[r] = (int64_t)off;
        a.row_cnt[r] = nst;
        a.row_fsum[r] = fs;
        a.row_nnz[r] = nnzu;
        if (a.row_p1) {
          a.row_p1[r] = q1;
          a.row_c1[r] = c1;
        }
      }
      __syncwarp();
    }
  }
  prods = warp_sum(prods);
  if (lane == 0 && prods) atomicAdd(D.prod_count, prods);
  if (lane == 0 && D.need_max && need > 0) atomicMax(D.need_max, need);
}

void launch_taylor_dia(const NumericArgs &a, const DiaView &D, int slots, int32_t *fail_rows,
                       int *fail_count, cudaStream_t st) {
  if (a.A.nrows == 0 || a.nlist == 0) return;
  const int smem = taylor_dia_smem_bytes(slots);
  // grid stencils (3 / 5 / 7 offsets in 1D / 2D / 3D) get loops of their exact length
  auto kf = D.ndiag == 3   ? k_taylor_dia<3, true>
            : D.ndiag == 5 ? k_taylor_dia<5, true>
            : D.ndiag == 7 ? k_taylor_dia<7, true>
            : D.ndiag <= 4 ? k_taylor_dia<4, false>
            : D.ndiag <= 8 ? k_taylor_dia<8, false>
                           : k_taylor_dia<16, false>;
  cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  KL;
  kf<<<a.grid, kDWarps * 32, smem, st>>>(a, D, slots, fail_rows, fail_count);
}


// ------------------------------------------------------------------------------------
// K4 compaction: keep staged entries with |x| > tau (Alg. 4.1 step 3).
// ------------------------------------------------------------------------------------
// ident != nullptr (E = I + T^_N fused into the last compaction): per row,
// ident[w] = 0 no kept diagonal (insert 1.0), 1 kept diagonal t (write 1 + t), 2 kept
// diagonal with 1 + t == 0 (purged, reading R11); cnt counts the entries of E's row.
__global__ void __launch_bounds__(kThreads, 8) k_compact_count(int64_t nrows, int64_t row0, const int64_t *row_off,
                                const int64_t *row_cnt, const int32_t *pool_col,
                                const double *pool_val, double tau, int64_t *cnt,
                                int8_t *ident) {
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (w >= nrows) return;
  int64_t o = row_off[w], c = row_cnt[w];
  const int64_t grow = row0 + w;
  long long k = 0;
  int diag = 0;  // 1: kept diagonal, 2: kept diagonal with 1 + t == 0
  for (int64_t t = lane; t < c; t += 32) {
    const double x = pool_val[o + t];
    const bool kept = fabs(x) > tau;
    k += kept;
    if (ident && kept && pool_col[o + t] == grow) diag = (1.0 + x == 0.0) ? 2 : 1;
  }
  k = warp_sum(k);
  if (ident) diag = __reduce_max_sync(FULL_MASK, diag);
  if (lane == 0) {
    if (ident) {
      ident[w] = (int8_t)diag;
      k += diag == 0 ? 1 : (diag == 2 ? -1 : 0);
    }
    cnt[w] = k;
  }
}
void launch_compact_count(int64_t nrows, const int64_t *row_off, const int64_t *row_cnt,
                          const double *pool_val, double tau, int64_t *cnt, cudaStream_t st) {
  if (nrows == 0) return;
  KL;
  k_compact_count<<<grid_for(nrows * 32, kThreads), kThreads, 0, st>>>(
      nrows, 0, row_off, row_cnt, nullptr, pool_val, tau, cnt, nullptr);
}
void launch_compact_count_ident(int64_t nrows, int64_t row0, const int64_t *row_off,
                                const int64_t *row_cnt, const int32_t *pool_col,
                                const double *pool_val, double tau, int64_t *cnt, int8_t *ident,
                                cudaStream_t st) {
  if (nrows == 0) return;
  KL;
  k_compact_count<<<grid_for(nrows * 32, kThreads), kThreads, 0, st>>>(
      nrows, row0, row_off, row_cnt, pool_col, pool_val, tau, cnt, ident);
}

__device__ __forceinline__ void row_stat_accum(int64_t grow, int32_t c, double x, double &s,
                                               int &have_diag, long long &l1, long long &l2) {
  long long d = (long long)c - grow;
  if (d == 0) {
    double y = x + 1.0;
    s += y * y;
    have_diag = 1;
  } else {
    s += x * x;
  }
  if (d > l1) l1 = d;
  if (-d > l2) l2 = -d;
}
__device__ __forceinline__ void row_stat_finish(int lane, int64_t w, double s, int have_diag,
                                                long long l1, long long l2, double *rs,
                                                int64_t *l1r, int64_t *l2r) {
  s = warp_sum(s);
  have_diag = __reduce_or_sync(FULL_MASK, have_diag);
  l1 = warp_max(l1);
  l2 = warp_max(l2);
  if (lane == 0) {
    if (rs) rs[w] = s + (have_diag ? 0.0 : 1.0);
    if (l1r) l1r[w] = l1;
    if (l2r) l2r[w] = l2;
  }
}

__global__ void __launch_bounds__(kThreads, 4) k_compact_write(int64_t nrows, int64_t row0, const int64_t *row_off,
                                const int64_t *row_cnt, const int32_t *pool_col,
                                const double *pool_val, double tau, const int64_t *rp_out,
                                int32_t *col_out, double *val_out, double *rs, int64_t *l1r,
                                int64_t *l2r, const int8_t *ident) {
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (w >= nrows) return;
  int64_t o = row_off[w], c = row_cnt[w];
  const int64_t dst0 = rp_out[w];
  int64_t dst = dst0;
  const int64_t grow = row0 + w;
  const int idg = ident ? ident[w] : -1;  // -1: plain compaction of T^
  double s = 0.0;
  int have_diag = 0;
  long long l1 = 0, l2 = 0;
  long long nlt = 0;  // kept entries left of the diagonal (insert position, idg == 0)
  // 4 chunks' loads in flight before their stores (the outputs do not alias the pool)
  for (int64_t base0 = 0; base0 < c; base0 += 128) {
    double xb[4];
    int32_t cb[4];
#pragma unroll
    for (int v = 0; v < 4; v++) {
      const int64_t tv = base0 + 32 * v + lane;
      xb[v] = tv < c ? __ldg(pool_val + o + tv) : 0.0;
      cb[v] = tv < c ? __ldg(pool_col + o + tv) : 0;
    }
#pragma unroll
    for (int v = 0; v < 4; v++) {
      const int64_t t = base0 + 32 * v + lane;
      const double x = xb[v];
      const int32_t cc = cb[v];
      const bool k = t < c && fabs(x) > tau;
      if (k) row_stat_accum(grow, cc, x, s, have_diag, l1, l2);  // statistics of T^ itself
      const bool isd = k && cc == grow;
      const bool wr = k && !(isd && idg == 2);
      unsigned m = __ballot_sync(FULL_MASK, wr);
      if (wr) {
        int64_t q = dst + __popc(m & lanemask_lt());
        if (idg == 0 && cc > grow) q += 1;  // room for the inserted diagonal
        col_out[q] = cc;
        val_out[q] = (isd && idg == 1) ? 1.0 + x : x;
      }
      dst += __popc(m);
      if (idg == 0) nlt += __popc(__ballot_sync(FULL_MASK, k && cc < grow));
    }
  }
  if (idg == 0 && lane == 0) {
    col_out[dst0 + nlt] = (int32_t)grow;
    val_out[dst0 + nlt] = 1.0;
  }
  row_stat_finish(lane, w, s, have_diag, l1, l2, rs, l1r, l2r);
}
void launch_compact_write(int64_t nrows, int64_t row0, const int64_t *row_off,
                          const int64_t *row_cnt, const int32_t *pool_col,
                          const double *pool_val, double tau, const int64_t *rp_out,
                          int32_t *col_out, double *val_out, double *rs, int64_t *l1r,
                          int64_t *l2r, cudaStream_t st, const int8_t *ident) {
  if (nrows == 0) return;
  KL;
  k_compact_write<<<grid_for(nrows * 32, kThreads), kThreads, 0, st>>>(
      nrows, row0, row_off, row_cnt, pool_col, pool_val, tau, rp_out, col_out, val_out, rs, l1r,
      l2r, ident);
}

// out[0] += rows with ident == 0 (inserted diagonals), out[1] += rows with ident == 2
__global__ void k_count_ident(const int8_t *ident, int64_t nrows, unsigned long long *out) {
  unsigned long long a = 0, b = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrows;
       i += (int64_t)gridDim.x * blockDim.x) {
    a += ident[i] == 0;
    b += ident[i] == 2;
  }
  a = warp_sum(a);
  b = warp_sum(b);
  if ((threadIdx.x & 31) == 0) {
    if (a) atomicAdd(&out[0], a);
    if (b) atomicAdd(&out[1], b);
  }
}
void launch_count_ident(const int8_t *ident, int64_t nrows, int64_t *out2, cudaStream_t st) {
  cudaMemsetAsync(out2, 0, 2 * sizeof(int64_t), st);
  if (nrows == 0) return;
  KL;
  k_count_ident<<<grid_for(nrows, kThreads * 8, kRedBlocks), kThreads, 0, st>>>(
      ident, nrows, reinterpret_cast<unsigned long long *>(out2));
}

__global__ void k_row_stats(CsrView C, double *rs, int64_t *l1r, int64_t *l2r) {
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (w >= C.nrows) return;
  const int64_t grow = C.row0 + w;
  double s = 0.0;
  int have_diag = 0;
  long long l1 = 0, l2 = 0;
  for (int64_t p = C.rp[w] + lane; p < C.rp[w + 1]; p += 32)
    row_stat_accum(grow, C.col[p], C.val[p], s, have_diag, l1, l2);
  row_stat_finish(lane, w, s, have_diag, l1, l2, rs, l1r, l2r);
}
void launch_row_stats(const CsrView &C, double *rs, int64_t *l1r, int64_t *l2r,
                      cudaStream_t st) {
  if (C.nrows == 0) return;
  KL;
  k_row_stats<<<grid_for(C.nrows * 32, kThreads), kThreads, 0, st>>>(C, rs, l1r, l2r);
}

// ------------------------------------------------------------------------------------
// Merge C = A + B of two row-sorted CSRs over the same rows (warp per row).
// Equal columns are summed as a + b (T^_0 + S^_i; T^_N + I); sums that
// are exactly zero are purged.  Each round takes up to 32 entries of each list and
// emits every entry with column <= min(last loaded column of a side that has more).
// ------------------------------------------------------------------------------------
__device__ __forceinline__ int lower_bound32(const int32_t *s, int32_t key) {
  int lo = 0, hi = 32;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (s[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <bool WRITE>
__global__ void k_merge(CsrView A, CsrView B, const int64_t *rp_out, int64_t *cnt,
                        int32_t *col_out, double *val_out) {
  __shared__ int32_t sA[kWarps][32], sB[kWarps][32];
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  if (w >= A.nrows) return;
  int64_t a0 = A.rp[w], na = A.rp[w + 1] - a0;
  int64_t b0 = B.rp[w], nb = B.rp[w + 1] - b0;
  int64_t i = 0, j = 0, out = WRITE ? rp_out[w] : 0;
  while (i < na || j < nb) {
    bool ina = i + lane < na, inb = j + lane < nb;
    int32_t ca = ina ? A.col[a0 + i + lane] : INT32_MAX;
    int32_t cb = inb ? B.col[b0 + j + lane] : INT32_MAX;
    double va = ina ? A.val[a0 + i + lane] : 0.0;
    double vb = inb ? B.val[b0 + j + lane] : 0.0;
    int32_t limA = (na - i > 32) ? __shfl_sync(FULL_MASK, ca, 31) : INT32_MAX;
    int32_t limB = (nb - j > 32) ? __shfl_sync(FULL_MASK, cb, 31) : INT32_MAX;
    int32_t lim = limA < limB ? limA : limB;
    bool oka = ina && ca <= lim, okb = inb && cb <= lim;
    sA[wi][lane] = ca;
    sB[wi][lane] = cb;
    __syncwarp();
    int posB = lower_bound32(sB[wi], ca);
    int posA = lower_bound32(sA[wi], cb);
    bool dupA = oka && posB < 32 && sB[wi][posB] == ca;
    bool dupB = okb && posA < 32 && sA[wi][posA] == cb;
    double vbm = __shfl_sync(FULL_MASK, vb, posB & 31);
    double sum = dupA ? va + vbm : va;
    bool keepA = oka && sum != 0.0;
    bool uB = okb && !dupB && vb != 0.0;
    unsigned bKA = __ballot_sync(FULL_MASK, keepA);
    unsigned bUB = __ballot_sync(FULL_MASK, uB);
    if (WRITE) {
      unsigned mB = posB >= 32 ? FULL_MASK : ((1u << posB) - 1u);
      unsigned mA = posA >= 32 ? FULL_MASK : ((1u << posA) - 1u);
      if (keepA) {
        int64_t q = out + __popc(bKA & lanemask_lt()) + __popc(bUB & mB);
        col_out[q] = ca;
        val_out[q] = sum;
      }
      if (uB) {
        int64_t q = out + __popc(bKA & mA) + __popc(bUB & lanemask_lt());
        col_out[q] = cb;
        val_out[q] = vb;
      }
    }
    out += __popc(bKA) + __popc(bUB);
    i += __popc(__ballot_sync(FULL_MASK, oka));
    j += __popc(__ballot_sync(FULL_MASK, okb));
    __syncwarp();
  }
  if (!WRITE && lane == 0) cnt[w] = out;
}
// T^_0 + S^_i fused with the compaction of S~_i (Taylor terms, P:416 with P:380): B is
// the staged S~_i (row r at pool[row_off[r] .. + row_cnt[r]), column order) under the
// final Algorithm 4.1 threshold tau -- an entry with |x| <= tau is dropped, i.e. merges as
// a 0, which the merge already treats like an absent entry (a + 0 = a, 0-valued entries
// are not emitted).  The write pass also writes S^_i itself (the kept entries) at s_rp.
template <bool WRITE>
__global__ void __launch_bounds__(kThreads, 8) k_merge_staged(CsrView A, const int64_t *alen, const int64_t *row_off,
                               const int64_t *row_cnt, const int32_t *pcol, const double *pval,
                               double tau, const int64_t *rp_out, int64_t *cnt, int32_t *col_out,
                               double *val_out, int64_t *len_out, const int64_t *s_rp,
                               int32_t *s_col, double *s_val) {
  __shared__ int32_t sA[kWarps][32], sB[kWarps][32];
  int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  if (w >= A.nrows) return;
  int64_t a0 = A.rp[w], na = alen ? alen[w] : A.rp[w + 1] - a0;
  int64_t b0 = row_off[w], nb = row_cnt[w];
  int64_t i = 0, j = 0, out = WRITE ? rp_out[w] : 0, sout = WRITE ? s_rp[w] : 0;
  while (i < na || j < nb) {
    bool ina = i + lane < na, inb = j + lane < nb;
    int32_t ca = ina ? A.col[a0 + i + lane] : INT32_MAX;
    int32_t cb = inb ? pcol[b0 + j + lane] : INT32_MAX;
    double va = ina ? A.val[a0 + i + lane] : 0.0;
    double vb = inb ? pval[b0 + j + lane] : 0.0;
    if (!(fabs(vb) > tau)) vb = 0.0;  // dropped by Algorithm 4.1
    int32_t limA = (na - i > 32) ? __shfl_sync(FULL_MASK, ca, 31) : INT32_MAX;
    int32_t limB = (nb - j > 32) ? __shfl_sync(FULL_MASK, cb, 31) : INT32_MAX;
    int32_t lim = limA < limB ? limA : limB;
    bool oka = ina && ca <= lim, okb = inb && cb <= lim;
    sA[wi][lane] = ca;
    sB[wi][lane] = cb;
    __syncwarp();
    int posB = lower_bound32(sB[wi], ca);
    int posA = lower_bound32(sA[wi], cb);
    bool dupA = oka && posB < 32 && sB[wi][posB] == ca;
    bool dupB = okb && posA < 32 && sA[wi][posA] == cb;
    double vbm = __shfl_sync(FULL_MASK, vb, posB & 31);
    double sum = dupA ? va + vbm : va;
    bool keepA = oka && sum != 0.0;
    bool uB = okb && !dupB && vb != 0.0;
    unsigned bKA = __ballot_sync(FULL_MASK, keepA);
    unsigned bUB = __ballot_sync(FULL_MASK, uB);
    if (WRITE) {
      unsigned mB = posB >= 32 ? FULL_MASK : ((1u << posB) - 1u);
      unsigned mA = posA >= 32 ? FULL_MASK : ((1u << posA) - 1u);
      if (keepA) {
        int64_t q = out + __popc(bKA & lanemask_lt()) + __popc(bUB & mB);
        col_out[q] = ca;
        val_out[q] = sum;
      }
      if (uB) {
        int64_t q = out + __popc(bKA & mA) + __popc(bUB & lanemask_lt());
        col_out[q] = cb;
        val_out[q] = vb;
      }
      const bool ks = okb && vb != 0.0;  // kept entry of S^_i
      const unsigned bS = __ballot_sync(FULL_MASK, ks);
      if (ks) {
        const int64_t q = sout + __popc(bS & lanemask_lt());
        s_col[q] = cb;
        s_val[q] = vb;
      }
      sout += __popc(bS);
    }
    out += __popc(bKA) + __popc(bUB);
    i += __popc(__ballot_sync(FULL_MASK, oka));
    j += __popc(__ballot_sync(FULL_MASK, okb));
    __syncwarp();
  }
  if (!WRITE && lane == 0) cnt[w] = out;
  if (WRITE && lane == 0 && len_out) len_out[w] = out - rp_out[w];
}
void launch_merge_staged_count(const CsrView &A, const int64_t *alen, const int64_t *row_off,
                               const int64_t *row_cnt, const int32_t *pcol, const double *pval,
                               double tau, int64_t *cnt, cudaStream_t st) {
  if (A.nrows == 0) return;
  KL;
  k_merge_staged<false><<<grid_for(A.nrows * 32, kThreads), kThreads, 0, st>>>(
      A, alen, row_off, row_cnt, pcol, pval, tau, nullptr, cnt, nullptr, nullptr, nullptr, nullptr,
      nullptr, nullptr);
}
void launch_merge_staged_write(const CsrView &A, const int64_t *alen, const int64_t *row_off,
                               const int64_t *row_cnt, const int32_t *pcol, const double *pval,
                               double tau, const int64_t *rp_out, int32_t *col_out, double *val_out,
                               int64_t *len_out, const int64_t *s_rp, int32_t *s_col, double *s_val,
                               cudaStream_t st) {
  if (A.nrows == 0) return;
  KL;
  k_merge_staged<true><<<grid_for(A.nrows * 32, kThreads), kThreads, 0, st>>>(
      A, alen, row_off, row_cnt, pcol, pval, tau, rp_out, nullptr, col_out, val_out, len_out, s_rp,
      s_col, s_val);
}
// out[r] = (alen ? alen[r] : rp[r+1] - rp[r]) + b[r]: row capacities of T^_0 + S^_i
__global__ void k_add_rowlen(const int64_t *rp, const int64_t *alen, const int64_t *b, int64_t n,
                             int64_t *out) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    out[r] = (alen ? alen[r] : rp[r + 1] - rp[r]) + b[r];
}
void launch_add_rowlen(const int64_t *rp, const int64_t *alen, const int64_t *b, int64_t n,
                       int64_t *out, cudaStream_t st) {
  if (n == 0) return;
  KL;
  k_add_rowlen<<<grid_for(n, kThreads, 148 * 16), kThreads, 0, st>>>(rp, alen, b, n, out);
}
void launch_merge_count(const CsrView &A, const CsrView &B, int64_t *cnt, cudaStream_t st) {
  if (A.nrows == 0) return;
  KL;
  k_merge<false><<<grid_for(A.nrows * 32, kThreads), kThreads, 0, st>>>(A, B, nullptr, cnt,
                                                                        nullptr, nullptr);
}
void launch_merge_write(const CsrView &A, const CsrView &B, const int64_t *rp_out,
                        int32_t *col_out, double *val_out, cudaStream_t st) {
  if (A.nrows == 0) return;
  KL;
  k_merge<true><<<grid_for(A.nrows * 32, kThreads), kThreads, 0, st>>>(A, B, rp_out, nullptr,
                                                                       col_out, val_out);
}

__global__ void k_identity(int64_t nrows, int64_t row0, int64_t *rp, int32_t *col, double *val) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nrows) {
    rp[i] = i;
    col[i] = (int32_t)(row0 + i);
    val[i] = 1.0;
  }
  if (i == 0) rp[nrows] = nrows;
}
void launch_identity(int64_t nrows, int64_t row0, int64_t *rp, int32_t *col, double *val,
                     cudaStream_t st) {
  KL;
  k_identity<<<grid_for(nrows + 1, kThreads), kThreads, 0, st>>>(nrows, row0, rp, col, val);
}

__global__ void k_rebase(const int64_t *src, int64_t cnt, int64_t base, int64_t *dst) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= cnt) dst[i] = src[i] - src[0] + base;
}
void launch_rebase_rowptr(const int64_t *src, int64_t cnt, int64_t base, int64_t *dst,
                          cudaStream_t st) {
  KL;
  k_rebase<<<grid_for(cnt + 1, kThreads), kThreads, 0, st>>>(src, cnt, base, dst);
}

}  // namespace sx

namespace sx {
// ------------------------------------------------------------------------------------
// N1 apply: Y = A X for a CSR A and a dense row-major X (ldx >= m), the
// product that advances the discretised system by one step, u_{k+1} = e^H u_k (Eq. 2.2
// P:54).  One warp per row of A.  The warp's lanes form 32/W groups of W lanes;
// lane c of a group owns columns c, c + W, ... (CT per tile) and group g takes the row's
// entries g, g + 32/W, ...; the groups' partial sums are combined by a fixed xor tree.  With
// W = 32 (m >= 32) a lane adds its columns' products over the row's entries in ascending
// column order, y = y + a_rk x_kj (_rn, no contraction) -- the oracle's order, bit for bit.
// A row's entries are loaded 32 at a time and broadcast by shuffles; X rows are read as
// contiguous W * 8-byte segments.
// ------------------------------------------------------------------------------------
template <int W, int CT>
__global__ void __launch_bounds__(256) k_spmm(CsrView A, int64_t m, const double *X, int64_t ldx,
                                              double *Y, int64_t ldy) {
  constexpr int G = 32 / W;
  const int lane = threadIdx.x & 31, g = lane / W, c = lane % W;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < A.nrows; r += nw) {
    const int64_t p0 = A.rp[r], p1 = A.rp[r + 1];
    for (int64_t c0 = 0; c0 < m; c0 += (int64_t)W * CT) {
      double acc[CT];
#pragma unroll
      for (int t = 0; t < CT; t++) acc[t] = 0.0;
      int32_t kcn = p0 + lane < p1 ? A.col[p0 + lane] : 0;  // entries prefetched a chunk ahead
      double kvn = p0 + lane < p1 ? A.val[p0 + lane] : 0.0;
      for (int64_t pb = p0; pb < p1; pb += 32) {
        const int nb = (int)(p1 - pb < 32 ? p1 - pb : 32);
        const int32_t kc = kcn;
        const double kv = kvn;
        if (pb + 32 + lane < p1) {
          kcn = A.col[pb + 32 + lane];
          kvn = A.val[pb + 32 + lane];
        }
#pragma unroll 8
        for (int e0 = 0; e0 < nb; e0 += G) {
          const int e = e0 + g;
          const bool ok = e < nb;
          const int64_t k = __shfl_sync(FULL_MASK, kc, ok ? e : 0);
          const double a = __shfl_sync(FULL_MASK, kv, ok ? e : 0);
          if (ok) {
            const double *xr = X + k * ldx + c0 + c;
#pragma unroll
            for (int t = 0; t < CT; t++)
              if (c0 + c + (int64_t)W * t < m) acc[t] = __dadd_rn(acc[t], __dmul_rn(a, xr[W * t]));
          }
        }
      }
#pragma unroll
      for (int o = W; o < 32; o <<= 1)
#pragma unroll
        for (int t = 0; t < CT; t++) acc[t] = __dadd_rn(acc[t], __shfl_xor_sync(FULL_MASK, acc[t], o));
      if (g == 0) {
#pragma unroll
        for (int t = 0; t < CT; t++)
          if (c0 + c + (int64_t)W * t < m) Y[r * ldy + c0 + c + W * t] = acc[t];
      }
    }
  }
}

// m = 1 (SpMV): lanes take the row's entries directly (no broadcast), two chunks of 32 in
// flight per iteration with separate partial sums, then a fixed xor tree (deterministic)
__global__ void __launch_bounds__(256) k_spmv(CsrView A, const double *X, int64_t ldx, double *Y,
                                              int64_t ldy) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < A.nrows; r += nw) {
    const int64_t p0 = A.rp[r], p1 = A.rp[r + 1];
    double s0 = 0.0, s1 = 0.0;
    int64_t p = p0 + lane;
    for (; p + 32 < p1; p += 64) {
      const int32_t k0 = A.col[p], k1 = A.col[p + 32];
      const double a0 = A.val[p], a1 = A.val[p + 32];
      const double x0 = X[(int64_t)k0 * ldx], x1 = X[(int64_t)k1 * ldx];
      s0 = __dadd_rn(s0, __dmul_rn(a0, x0));
      s1 = __dadd_rn(s1, __dmul_rn(a1, x1));
    }
    if (p < p1) s0 = __dadd_rn(s0, __dmul_rn(A.val[p], X[(int64_t)A.col[p] * ldx]));
    double s = __dadd_rn(s0, s1);
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) s = __dadd_rn(s, __shfl_xor_sync(FULL_MASK, s, o));
    if (lane == 0) Y[r * ldy] = s;
  }
}

void launch_spmm(const CsrView &A, int64_t m, const double *X, int64_t ldx, double *Y, int64_t ldy,
                 cudaStream_t st) {
  if (A.nrows == 0 || m == 0) return;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((A.nrows + 7) / 8, 148 * 16));
  KL;
  if (m > 64) k_spmm<32, 4><<<grid, 256, 0, st>>>(A, m, X, ldx, Y, ldy);
  else if (m > 32) k_spmm<32, 2><<<grid, 256, 0, st>>>(A, m, X, ldx, Y, ldy);
  else if (m > 16) k_spmm<32, 1><<<grid, 256, 0, st>>>(A, m, X, ldx, Y, ldy);
  else if (m > 8) k_spmm<16, 1><<<grid, 256, 0, st>>>(A, m, X, ldx, Y, ldy);
  else if (m > 4) k_spmm<8, 1><<<grid, 256, 0, st>>>(A, m, X, ldx, Y, ldy);
  else if (m > 2) k_spmm<4, 1><<<grid, 256, 0, st>>>(A, m, X, ldx, Y, ldy);
  else if (m > 1) k_spmm<2, 1><<<grid, 256, 0, st>>>(A, m, X, ldx, Y, ldy);
  else k_spmv<<<grid, 256, 0, st>>>(A, X, ldx, Y, ldy);
}

// ------------------------------------------------------------------------------------
// Result copy-out by the SMs (sexpm_result_copy_async): a few resident CTAs stream a
// detached result to the caller's mapped pinned host (or device) memory with 16-byte stores
// over the link.  The copy engines are left alone: a small read-back of the plan running
// meanwhile was measured to wait behind a whole buffer's copy-engine transfer, however
// finely that was chunked.
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_copy_out(const uint4 *__restrict__ src, uint4 *__restrict__ dst,
                                                  size_t n16, size_t tail_bytes) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    const uint4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride),
                d = __ldcs(src + i + 3 * stride);
    __stcs(dst + i, a);
    __stcs(dst + i + stride, b);
    __stcs(dst + i + 2 * stride, c);
    __stcs(dst + i + 3 * stride, d);
  }
  for (; i < n16; i += stride) __stcs(dst + i, __ldcs(src + i));
  if (blockIdx.x == 0 && threadIdx.x < tail_bytes)
    ((unsigned char *)(dst + n16))[threadIdx.x] = ((const unsigned char *)(src + n16))[threadIdx.x];
}

bool launch_copy_out(void *dst, const void *src, size_t bytes, int ctas, cudaStream_t st) {
  if ((((uintptr_t)dst) | ((uintptr_t)src)) & 15) return false;  // caller copies another way
  if (bytes == 0) return true;
  KL;
  k_copy_out<<<std::max(1, ctas), 256, 0, st>>>((const uint4 *)src, (uint4 *)dst, bytes / 16, bytes % 16);
  return true;
}
}  // namespace sx

namespace sx {
// ------------------------------------------------------------------------------------
// N3 reordering: reverse Cuthill-McKee on the device for the real
// bandwidth of Def. 3.2a.  The host (driver.cu `compute_rcm`) runs the level
// loop; these kernels do the per-level work: BFS expansion over the symmetric pattern G,
// the (degree, index) minimum of a node set, the Cuthill-McKee key of a level (smallest
// position of a neighbour in the previous level), and the permutation of a CSR matrix.
// The tie rules are the oracle's (or_rcm).
// ------------------------------------------------------------------------------------
__global__ void k_degree_nodiag(CsrView G, int32_t *deg) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= G.nrows) return;
  int c = 0;
  for (int64_t p = G.rp[w] + lane; p < G.rp[w + 1]; p += 32) c += G.col[p] != (int32_t)w;
  c = __reduce_add_sync(FULL_MASK, c);
  if (lane == 0) deg[w] = c;
}
void launch_degree_nodiag(const CsrView &G, int32_t *deg, cudaStream_t st) {
  if (G.nrows == 0) return;
  KL;
  k_degree_nodiag<<<grid_for(G.nrows * 32, kThreads), kThreads, 0, st>>>(G, deg);
}

// frontier queue[a, b) at level L: unvisited neighbours get level L + 1 and are appended
__global__ void k_bfs_expand(CsrView G, int64_t *queue, int64_t a, int64_t b, int32_t *level,
                             int32_t L, unsigned long long *tail) {
  const int64_t w = a + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= b) return;
  const int64_t v = queue[w];
  for (int64_t p = G.rp[v] + lane; p < G.rp[v + 1]; p += 32) {
    const int32_t u = G.col[p];
    if (u != (int32_t)v && atomicCAS(&level[u], -1, L + 1) == -1)
      queue[atomicAdd(tail, 1ull)] = u;
  }
}
void launch_bfs_expand(const CsrView &G, int64_t *queue, int64_t a, int64_t b, int32_t *level,
                       int32_t L, unsigned long long *tail, cudaStream_t st) {
  if (b <= a) return;
  KL;
  k_bfs_expand<<<grid_for((b - a) * 32, kThreads), kThreads, 0, st>>>(G, queue, a, b, level, L, tail);
}

// out = min over queue[a, b) (or over all nodes with !done[v] when queue == nullptr) of
// deg << 32 | v  (out must hold ~0 before)
__global__ void k_min_deg(const int64_t *queue, int64_t a, int64_t b, const int32_t *deg,
                          const int8_t *done, unsigned long long *out) {
  unsigned long long m = ~0ull;
  for (int64_t i = a + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = queue ? queue[i] : i;
    if (!queue && done[v]) continue;
    const unsigned long long k = ((unsigned long long)(unsigned)deg[v] << 32) | (unsigned long long)v;
    m = k < m ? k : m;
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(FULL_MASK, m, o);
    m = y < m ? y : m;
  }
  if ((threadIdx.x & 31) == 0 && m != ~0ull) atomicMin(out, m);
}
void launch_min_deg(const int64_t *queue, int64_t a, int64_t b, const int32_t *deg,
                    const int8_t *done, unsigned long long *out, cudaStream_t st) {
  if (b <= a) return;
  KL;
  k_min_deg<<<grid_for(b - a, kThreads, 148 * 8), kThreads, 0, st>>>(queue, a, b, deg, done, out);
}

__global__ void k_reset_level(const int64_t *queue, int64_t a, int64_t b, int32_t *level) {
  for (int64_t i = a + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b;
       i += (int64_t)gridDim.x * blockDim.x)
    level[queue[i]] = -1;
}
void launch_reset_level(const int64_t *queue, int64_t a, int64_t b, int32_t *level, cudaStream_t st) {
  if (b <= a) return;
  KL;
  k_reset_level<<<grid_for(b - a, kThreads, 148 * 16), kThreads, 0, st>>>(queue, a, b, level);
}

// level L + 1 = queue[a, b): key = (smallest position of a neighbour in level L) << 32 | degree
__global__ void k_cm_key(CsrView G, const int64_t *queue, int64_t a, int64_t b, const int32_t *level,
                         int32_t L, const int64_t *pos, const int32_t *deg, unsigned long long *key,
                         int32_t *ids) {
  const int64_t w = a + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= b) return;
  const int64_t v = queue[w];
  long long k = LLONG_MAX;
  for (int64_t p = G.rp[v] + lane; p < G.rp[v + 1]; p += 32) {
    const int32_t u = G.col[p];
    if (u != (int32_t)v && level[u] == L) k = min(k, (long long)pos[u]);
  }
  for (int o = 16; o; o >>= 1) k = min(k, __shfl_xor_sync(FULL_MASK, k, o));
  if (lane == 0) {
    key[w - a] = ((unsigned long long)k << 32) | (unsigned long long)(unsigned)deg[v];
    ids[w - a] = (int32_t)v;
  }
}
void launch_cm_key(const CsrView &G, const int64_t *queue, int64_t a, int64_t b, const int32_t *level,
                   int32_t L, const int64_t *pos, const int32_t *deg, unsigned long long *key,
                   int32_t *ids, cudaStream_t st) {
  if (b <= a) return;
  KL;
  k_cm_key<<<grid_for((b - a) * 32, kThreads), kThreads, 0, st>>>(G, queue, a, b, level, L, pos, deg, key, ids);
}

// CUB: ids sorted ascending, then stably by key (cm order of one level)
size_t cm_sort_temp_bytes(int64_t cnt) {
  size_t b1 = 0, b2 = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, b1, (const int32_t *)nullptr, (int32_t *)nullptr, (int)cnt);
  cub::DeviceRadixSort::SortPairs(nullptr, b2, (const unsigned long long *)nullptr,
                                  (unsigned long long *)nullptr, (const int32_t *)nullptr,
                                  (int32_t *)nullptr, (int)cnt);
  return b1 > b2 ? b1 : b2;
}
// key of node: keyv[node] scattered then gathered in id order
__global__ void k_scatter_key(const unsigned long long *key, const int32_t *ids, int64_t cnt,
                              unsigned long long *keyv) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
    keyv[ids[i]] = key[i];
}
__global__ void k_gather_keyv(const unsigned long long *keyv, const int32_t *ids, int64_t cnt,
                              unsigned long long *key) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
    key[i] = keyv[ids[i]];
}
__global__ void k_place_level(const int32_t *ids, int64_t cnt, int64_t base, int64_t *pos, int64_t *cm) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
    pos[ids[i]] = base + i;
    cm[base + i] = ids[i];
  }
}
void launch_cm_sort_place(unsigned long long *key, int32_t *ids, int64_t cnt, unsigned long long *key2,
                          int32_t *ids2, unsigned long long *keyv, void *tmp, size_t tmp_bytes,
                          int64_t base, int64_t *pos, int64_t *cm, cudaStream_t st) {
  if (cnt <= 0) return;
  const int g = (int)std::min<int64_t>((cnt + kThreads - 1) / kThreads, 148 * 16);
  if (cnt > 1) {
    KL;
    k_scatter_key<<<g, kThreads, 0, st>>>(key, ids, cnt, keyv);
    size_t b = tmp_bytes;
    KL;
    cub::DeviceRadixSort::SortKeys(tmp, b, ids, ids2, (int)cnt, 0, 32, st);  // ids ascending
    KL;
    k_gather_keyv<<<g, kThreads, 0, st>>>(keyv, ids2, cnt, key2);
    b = tmp_bytes;
    KL;
    cub::DeviceRadixSort::SortPairs(tmp, b, key2, key, ids2, ids, (int)cnt, 0, 64, st);  // stable by key
  }
  KL;
  k_place_level<<<g, kThreads, 0, st>>>(ids, cnt, base, pos, cm);
}

__global__ void k_mark_done(const int64_t *cm, int64_t a, int64_t b, int8_t *done, int32_t *level) {
  for (int64_t i = a + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < b; i += (int64_t)gridDim.x * blockDim.x) {
    done[cm[i]] = 1;
    level[cm[i]] = -2;  // placed: never visited again
  }
}
void launch_mark_done(const int64_t *cm, int64_t a, int64_t b, int8_t *done, int32_t *level, cudaStream_t st) {
  if (b <= a) return;
  KL;
  k_mark_done<<<grid_for(b - a, kThreads, 148 * 16), kThreads, 0, st>>>(cm, a, b, done, level);
}
__global__ void k_reverse_perm(const int64_t *cm, int64_t n, int64_t *perm, int64_t *inv) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = cm[n - 1 - i];
    perm[i] = v;
    inv[v] = i;
  }
}
void launch_reverse_perm(const int64_t *cm, int64_t n, int64_t *perm, int64_t *inv, cudaStream_t st) {
  if (n == 0) return;
  KL;
  k_reverse_perm<<<grid_for(n, kThreads, 148 * 16), kThreads, 0, st>>>(cm, n, perm, inv);
}

// C = A permuted: C row i = A row rowmap[i] with columns colmap[c], then rows sorted (CUB)
__global__ void k_perm_count(const int64_t *arp, const int64_t *rowmap, int64_t n, int64_t *cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    cnt[i] = arp[rowmap[i] + 1] - arp[rowmap[i]];
}
__global__ void k_perm_write(CsrView A, const int64_t *rowmap, const int64_t *colmap, int64_t n,
                             const int64_t *rp_out, int32_t *col_out, double *val_out) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const int64_t r = rowmap[w], a0 = A.rp[r], len = A.rp[r + 1] - a0, o = rp_out[w];
  for (int64_t p = lane; p < len; p += 32) {
    col_out[o + p] = (int32_t)colmap[A.col[a0 + p]];
    val_out[o + p] = A.val[a0 + p];
  }
}
void launch_perm_count(const int64_t *arp, const int64_t *rowmap, int64_t n, int64_t *cnt, cudaStream_t st) {
  if (n == 0) return;
  KL;
  k_perm_count<<<grid_for(n, kThreads, 148 * 16), kThreads, 0, st>>>(arp, rowmap, n, cnt);
}
void launch_perm_write(const CsrView &A, const int64_t *rowmap, const int64_t *colmap, int64_t n,
                       const int64_t *rp_out, int32_t *col_out, double *val_out, cudaStream_t st) {
  if (n == 0) return;
  KL;
  k_perm_write<<<grid_for(n * 32, kThreads), kThreads, 0, st>>>(A, rowmap, colmap, n, rp_out, col_out, val_out);
}
// segmented sort of each row's (column, value) pairs with caller-provided double buffers
// (no O(nnz) temporary inside CUB): on return *k_cur / *v_cur point at the sorted arrays
size_t seg_sort_temp_bytes(int64_t nnz, int64_t n, const int64_t *rp) {
  size_t b = 0;
  cub::DoubleBuffer<int32_t> kb(nullptr, nullptr);
  cub::DoubleBuffer<double> vb(nullptr, nullptr);
  cub::DeviceSegmentedSort::SortPairs(nullptr, b, kb, vb, (int)nnz, (int)n, rp, rp + 1);
  return b;
}
void launch_seg_sort(int32_t **k_cur, int32_t *k_alt, double **v_cur, double *v_alt, int64_t nnz,
                     int64_t n, const int64_t *rp, void *tmp, size_t tmp_bytes, cudaStream_t st) {
  if (nnz == 0 || n == 0) return;
  size_t b = tmp_bytes;
  cub::DoubleBuffer<int32_t> kb(*k_cur, k_alt);
  cub::DoubleBuffer<double> vb(*v_cur, v_alt);
  KL;
  cub::DeviceSegmentedSort::SortPairs(tmp, b, kb, vb, (int)nnz, (int)n, rp, rp + 1, st);
  *k_cur = kb.Current();
  *v_cur = vb.Current();
}
}  // namespace sx

namespace sx {
// flag |= 1 unless A's rows are, bit for bit, B's rows A.row0 - B.row0 + r (the block kernel
// reads A's blocks from B's BSR view: allowed only when A is a slice of B)
__global__ void k_rows_equal(CsrView A, CsrView B, int *flag) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= A.nrows) return;
  const int64_t rb = w + A.row0 - B.row0;
  const int64_t a0 = A.rp[w], na = A.rp[w + 1] - a0;
  if (rb < 0 || rb >= B.nrows) {
    if (lane == 0) atomicOr(flag, 1);
    return;
  }
  const int64_t b0 = B.rp[rb], nb = B.rp[rb + 1] - b0;
  bool diff = na != nb;
  if (!diff)
    for (int64_t p = lane; p < na; p += 32)
      diff |= A.col[a0 + p] != B.col[b0 + p] ||
              __double_as_longlong(A.val[a0 + p]) != __double_as_longlong(B.val[b0 + p]);
  if (__any_sync(FULL_MASK, diff) && lane == 0) atomicOr(flag, 1);
}
void launch_rows_equal(const CsrView &A, const CsrView &B, int *flag, cudaStream_t st) {
  if (A.nrows == 0) return;
  KL;
  k_rows_equal<<<grid_for(A.nrows * 32, kThreads), kThreads, 0, st>>>(A, B, flag);
}
}  // namespace sx

namespace sx {
// Row sort for relabelled CSR rows (<= kSortCap entries), one warp per row.  The keys of a
// row are distinct columns: when their span fits a 64 Ki-bit bitmap, a key's sorted position
// is the number of set bits below it (mark, word popcount prefix, rank: O(span / 32 + len)
// per row); otherwise a bitonic network over (column << 32 | position) in shared memory.
constexpr int kSortCap = 1024, kSortWarps = 8;
constexpr int kSortWords = 2048;  // bitmap words per warp (65536 columns of span)
// PERM: output row r is input row rowmap[r] (input row pointers irp), every key mapped
// through colmap, output rows at rp -- the relabelling and the sort in one pass
template <bool PERM>
__global__ void __launch_bounds__(kSortWarps * 32) k_sort_rows(const int64_t *rp, int64_t n,
                                                               const int32_t *kin, const double *vin,
                                                               int32_t *kout, double *vout,
                                                               const int64_t *irp = nullptr,
                                                               const int64_t *rowmap = nullptr,
                                                               const int64_t *colmap = nullptr) {
  extern __shared__ unsigned long long sbuf[];
  const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
  unsigned long long *buf = sbuf + wi * kSortCap;                       // bitonic keys
  unsigned *bits = reinterpret_cast<unsigned *>(buf);                     // or: bitmap words
  uint16_t *pref = reinterpret_cast<uint16_t *>(sbuf + kSortWarps * kSortCap) + wi * kSortWords;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
    const int64_t p0 = rp[r];
    const int64_t q0 = PERM ? irp[rowmap[r]] : p0;  // the input row
    const int len = (int)(rp[r + 1] - p0);
    int kmin = INT32_MAX, kmax = -1;
    int kr[kSortCap / 32];  // the row's keys, loaded once (len <= kSortCap)
#pragma unroll
    for (int t = 0; t < kSortCap / 32; t++) {
      const int i = lane + 32 * t;
      kr[t] = i < len ? (PERM ? (int)colmap[kin[q0 + i]] : kin[p0 + i]) : 0;
      if (i < len) {
        kmin = min(kmin, kr[t]);
        kmax = max(kmax, kr[t]);
      }
    }
    kmin = __shfl_sync(FULL_MASK, warp_min(kmin), 0);  // warp_min / warp_max reduce into lane 0
    kmax = __shfl_sync(FULL_MASK, warp_max(kmax), 0);
    const int64_t span = len ? (int64_t)kmax - kmin + 1 : 0;
    if (span <= (int64_t)kSortWords * 32) {
      const int nwd = (int)((span + 31) >> 5);
      for (int i = lane; i < nwd; i += 32) bits[i] = 0u;
      __syncwarp();
#pragma unroll
      for (int t = 0; t < kSortCap / 32; t++)
        if (lane + 32 * t < len) {
          const int d = kr[t] - kmin;
          atomicOr(&bits[d >> 5], 1u << (d & 31));
        }
      __syncwarp();
      const int per = (nwd + 31) / 32, w0 = min(lane * per, nwd), w1 = min(w0 + per, nwd);
      int c = 0;
      for (int w = w0; w < w1; w++) c += __popc(bits[w]);
      int v = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL_MASK, v, o);
        if (lane >= o) v += y;
      }
      int run = v - c;
      for (int w = w0; w < w1; w++) {
        pref[w] = (uint16_t)run;
        run += __popc(bits[w]);
      }
      __syncwarp();
      // values in groups of 8 loads in flight before their stores (vin / vout do not alias,
      // but the compiler cannot know: one load -> store chain per entry otherwise)
#pragma unroll
      for (int t0 = 0; t0 < kSortCap / 32; t0 += 8) {
        if (32 * t0 >= len) break;
        double vv[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const int e = lane + 32 * (t0 + u);
          vv[u] = e < len ? __ldg(vin + q0 + e) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; u++)
          if (lane + 32 * (t0 + u) < len) {
            const int k = kr[t0 + u], d = k - kmin;
            const int pos = pref[d >> 5] + __popc(bits[d >> 5] & ((1u << (d & 31)) - 1u));
            kout[p0 + pos] = k;
            vout[p0 + pos] = vv[u];
          }
      }
      __syncwarp();
      continue;
    }
    int P = 32;
    while (P < len) P <<= 1;
    for (int i = lane; i < P; i += 32)
      buf[i] = i < len ? ((unsigned long long)(unsigned)(PERM ? (int)colmap[kin[q0 + i]] : kin[p0 + i]) << 32) | (unsigned)i : ~0ull;
    __syncwarp();
    for (int k = 2; k <= P; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = lane; i < P; i += 32) {
          const int l = i ^ j;
          if (l > i) {
            const unsigned long long a = buf[i], b = buf[l];
            if ((a > b) == ((i & k) == 0)) {
              buf[i] = b;
              buf[l] = a;
            }
          }
        }
        __syncwarp();
      }
    for (int i = lane; i < len; i += 32) {
      const unsigned long long e = buf[i];
      kout[p0 + i] = (int32_t)(e >> 32);
      vout[p0 + i] = vin[q0 + (int64_t)(e & 0xFFFFFFFFull)];
    }
    __syncwarp();
  }
}
void launch_sort_rows(const int64_t *rp, int64_t n, const int32_t *kin, const double *vin, int32_t *kout,
                      double *vout, cudaStream_t st) {
  if (n == 0) return;
  const int smem = kSortWarps * kSortCap * 8 + kSortWarps * kSortWords * 2;
  cudaFuncSetAttribute(k_sort_rows<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  KL;
  k_sort_rows<false><<<(int)std::min<int64_t>((n + kSortWarps - 1) / kSortWarps, 148 * 3), kSortWarps * 32, smem, st>>>(
      rp, n, kin, vin, kout, vout);
}
void launch_perm_sort_rows(const CsrView &A, const int64_t *rowmap, const int64_t *colmap, int64_t n,
                           const int64_t *rp_out, int32_t *col_out, double *val_out, cudaStream_t st) {
  if (n == 0) return;
  const int smem = kSortWarps * kSortCap * 8 + kSortWarps * kSortWords * 2;
  cudaFuncSetAttribute(k_sort_rows<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  KL;
  k_sort_rows<true><<<(int)std::min<int64_t>((n + kSortWarps - 1) / kSortWarps, 148 * 3), kSortWarps * 32, smem, st>>>(
      rp_out, n, A.col, A.val, col_out, val_out, A.rp, rowmap, colmap);
}
}  // namespace sx

namespace sx {
// ------------------------------------------------------------------------------------
// K5s: the Taylor product S~ = S^ H0 / i for SHORT rows (1D-like bands): one THREAD per row
// with a dense window of kShortWin slots over the row's output span [lo, hi] in shared
// memory (slot t of thread x at t * blockDim + x: consecutive threads, consecutive words).
// The thread adds, for its entries k in ascending order and the diagonals in descending
// offset order, s_rk * h_d[k] into column k + d: every column sees its products in
// ascending k -- the order of K5d and of the oracle, bit for bit.  Then / i, the Algorithm
// 4.1 floor classification (and the fused first pass), staging in column order with one
// pool reservation per warp.  Rows whose span exceeds the window go to the fail list (K5d).
// ------------------------------------------------------------------------------------
constexpr int kShortWin = 64, kShortThreads = 128;
__global__ void __launch_bounds__(kShortThreads) k_taylor_dia_short(NumericArgs a, DiaView D,
                                                                   int32_t *fail_rows, int *fail_count) {
  extern __shared__ double ssm[];
  const int tid = threadIdx.x, lane = tid & 31;
  __shared__ int32_t s_doff[kDiaMax];
  if (tid < kDiaMax) s_doff[tid] = tid < D.ndiag ? D.off[tid] : 0;
  __syncthreads();
  const int nd = D.ndiag;
  const int n = (int)D.n;
  unsigned long long prods = 0;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  // warp-uniform trip count so that the warp-wide reservation below is safe
  for (int64_t base = (int64_t)blockIdx.x * blockDim.x + (tid & ~31); base < a.nlist; base += nthr) {
    const int64_t idx = base + lane;
    const bool have = idx < a.nlist;
    const int64_t r = have ? (a.order ? (int64_t)a.order[idx] : idx) : 0;
    int64_t p0 = 0, p1 = 0;
    if (have) {
      p0 = a.A.rp[r];
      p1 = a.A.rp[r + 1];
    }
    int lo = 0, span = 0;
    bool fit = true;
    if (have && p1 > p0) {
      lo = a.A.col[p0] + D.dmin;
      int hi = a.A.col[p1 - 1] + D.dmax;
      lo = lo < 0 ? 0 : lo;
      hi = hi > n - 1 ? n - 1 : hi;
      span = hi - lo + 1;
      fit = span <= kShortWin;
    }
    const bool work = have && fit && p1 > p0;
    if (have && !fit) fail_rows[atomicAdd(fail_count, 1)] = (int32_t)r;
    if (work) {
      for (int t = 0; t < span; t++) ssm[t * kShortThreads + tid] = 0.0;
      for (int64_t p = p0; p < p1; p++) {
        const int k = a.A.col[p];
        const double s = a.A.val[p];
        for (int di = 0; di < nd; di++) {
          const double h = D.val[(size_t)di * (size_t)n + k];
          if (h != 0.0) {
            const int t = k + s_doff[di] - lo;
            ssm[t * kShortThreads + tid] = __dadd_rn(ssm[t * kShortThreads + tid], __dmul_rn(s, h));
            prods++;
          }
        }
      }
    }
    // flush pass 1: / i, classify, count
    int nst = 0;
    double fs = 0.0, q1 = 0.0;
    long long nnzu = 0, c1 = 0;
    if (work) {
      for (int t = 0; t < span; t++) {
        double x = ssm[t * kShortThreads + tid];
        if (x != 0.0) {
          x = x / a.divisor;
          ssm[t * kShortThreads + tid] = x;
          if (x != 0.0) {
            nnzu++;
            if (fabs(x) > a.floor_tau) {
              nst++;
              if (fabs(x) <= a.eps_g) q1 += x * x;
              else c1++;
            } else {
              fs += x * x;
            }
          }
        }
      }
    }
    // one pool reservation per warp
    int v = nst;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL_MASK, v, o);
      if (lane >= o) v += y;
    }
    const int tot = __shfl_sync(FULL_MASK, v, 31);
    unsigned long long off = 0;
    if (lane == 0 && tot) off = atomicAdd(a.pool_used, (unsigned long long)tot);
    off = __shfl_sync(FULL_MASK, off, 0) + (unsigned long long)(v - nst);
    const bool ok = (long long)off + nst <= a.pool_cap;
    if (work && ok) {
      long long q = (long long)off;
      for (int t = 0; t < span; t++) {
        const double x = ssm[t * kShortThreads + tid];
        if (x != 0.0 && fabs(x) > a.floor_tau) {
          a.pool_col[q] = lo + t;
          a.pool_val[q] = x;
          q++;
        }
      }
    }
    if (have && fit) {
      if (!ok) atomicOr(a.flags, 1);
      a.row_off[r] = (int64_t)off;
      a.row_cnt[r] = nst;
      a.row_fsum[r] = fs;
      a.row_nnz[r] = nnzu;
      if (a.row_p1) {
        a.row_p1[r] = q1;
        a.row_c1[r] = c1;
      }
    }
  }
  prods = warp_sum(prods);
  if (lane == 0 && prods) atomicAdd(D.prod_count, prods);
}
void launch_taylor_dia_short(const NumericArgs &a, const DiaView &D, int32_t *fail_rows, int *fail_count,
                             cudaStream_t st) {
  if (a.A.nrows == 0 || a.nlist == 0) return;
  const int smem = kShortWin * kShortThreads * 8;
  cudaFuncSetAttribute(k_taylor_dia_short, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((a.nlist + kShortThreads - 1) / kShortThreads, 148 * 3));
  KL;
  k_taylor_dia_short<<<grid, kShortThreads, smem, st>>>(a, D, fail_rows, fail_count);
}
}  // namespace sx

namespace sx {
// ------------------------------------------------------------------------------------
// K5w: Taylor terms on the dense OFFSET WINDOW (Eq. 4.10-4.11, Alg. 4.2 step 3
// P:410-418).  For an H0 with few diagonal offsets D (grid stencils), row r of S~_j is
// nonzero only at columns r + o, o in the Minkowski sum W_j = D + ... + D (j times); T^_0
// after term j only at cum_j = W_1 u ... u W_j.  The driver enumerates them once per plan
// (ascending); a term is stored POSITION-MAJOR and dense: S~_j(r, r + W_j[q]) at
// S[q * nl + l] (l = local row), T^_0 likewise over cum_j.  One thread per row: every load
// and store of a warp covers 32 consecutive rows of one position (coalesced, no column
// indices, no shared-memory rows), and the tables (uniform across the warp) sit in shared
// memory.
//
// TERM launch i (thread = row r):
//   S~_i(r, r+o) = (sum over di, offsets d DESCENDING, of S^_{i-1}(r, r+o-d) h_d(r+o-d)) / i,
//   S^_{i-1} = keep(S~_{i-1}, |x| > tau_{i-1}) applied on load (S^_1 = H0's row, unfiltered,
//   reading R9).  For a fixed output column the k = r+o-d run ascending: the oracle's
//   Gustavson order with _rn products and sums, then an IEEE division (R7) -- bit-identical.
//   When 0 is in D, T^_0^(i-1) = T^_0^(i-2) + S^_{i-1} is fused into the same loop (the d = 0
//   operand is S^_{i-1} at the output's own offset; cum_{i-1} = W_{i-1} is inside W_i).
//   Classification against the Algorithm 4.1 floor (see k_numeric): |x| <= floor dropped
//   (x^2 summed), floor < |x| <= eps_g staged per row, position-major (band[k * nl + l]), the
//   only values Algorithm 4.1's passes can still decide, |x| > eps_g kept for sure (counted).
// S~ at a column outside [0, n) is exactly zero (h_d(k) = 0 where column k + d does not
// exist); the h_d loads are guarded by 0 <= k < n because they are issued before the operand
// is known (all loads of an output in flight together).
// ------------------------------------------------------------------------------------
constexpr int kWinThreads = 128;
// per output position t of W_i one record of int32 element offsets (built at plan time for
// this rank's row count nl, read with two broadcast shared-memory loads):
//   [0, ND)  the source of each diagonal: p * nl for position p of S~_{i-1} (i = 2: the plane
//            of H0's diagonal in the padded diagonal array), or the zero plane when absent
//   ND       T^_0^(i-1) store: q * nl for o_t's position q in cum_{i-1}, or -1
//   ND + 1   T^_0^(i-2) load: its position * nl, or the zero plane
//   ND + 2   o_t
int taylor_win_rec_words(int nd) { return ((taylor_win_kernel_nd(nd) + 3) + 3) / 4 * 4; }
int taylor_win_smem_bytes(int nd, int ncnt, int ccnt) {
  (void)ccnt;
  return ncnt * taylor_win_rec_words(nd) * 4 + 16;
}
template <int ND, bool H0PREV>  // H0PREV: S~_{i-1} = H0 (i = 2)
__global__ void __launch_bounds__(kWinThreads, 7) k_taylor_win(WinArgs a) {
  extern __shared__ int4 wsm4[];
  constexpr int RW = ((ND + 3) + 3) / 4 * 4;
  const int tid = threadIdx.x;
  const int ncnt = a.ncnt;
  const int32_t *s_rec = reinterpret_cast<const int32_t *>(wsm4);
  {
    const int4 *src = reinterpret_cast<const int4 *>(a.rec);
    for (int i = tid; i < ncnt * (RW / 4); i += kWinThreads) wsm4[i] = src[i];
  }
  __syncthreads();
  const int nl = (int)a.nrows;
  const double tau_prev = a.tau_prev;
  const double div = a.divisor, floor_tau = a.floor_tau, eps_g = a.eps_g;
  const int dz = a.dzero;
  uint32_t hoff[ND];
#pragma unroll
  for (int di = 0; di < ND; di++) hoff[di] = (uint32_t)(a.hoff[di] + a.hpad);  // >= 0
  // one output's operands: ND sources, ND diagonal values, the T^_0 value; all loads of the
  // next output are issued before the current one is summed (software pipeline)
  struct Ops {
    double x[ND], h[ND], t0;
    int t0n, o;
  };
  // persistent CTAs over tiles of 128 rows
  for (int64_t tile = blockIdx.x; tile * kWinThreads < a.nrows; tile += gridDim.x) {
    const int l = (int)(tile * kWinThreads) + tid;
    if (l >= nl) break;
    const int64_t r = a.row0 + l;
    const double *hb = a.dpad - a.hpad + r;         // h_d(r + o - d) = hb[hoff[di] + o]
    const double *xb = H0PREV ? a.dpad + r : a.pS + a.padr + l;  // S~_{i-1}(r, r + o') = xb[rec]
    const double *t0ob = a.T0old + l;
    double *t0nb = a.T0new + l;
    double *nsb = a.nS + a.padr + l;
    const uint32_t pstride = (uint32_t)(a.plane ? a.plane : nl);
    auto load = [&](int t, Ops &op) {
      int rc[RW];
#pragma unroll
      for (int w = 0; w < RW; w += 4) {
        const int4 v4 = *reinterpret_cast<const int4 *>(s_rec + t * RW + w);
        rc[w] = v4.x;
        rc[w + 1] = v4.y;
        rc[w + 2] = v4.z;
        rc[w + 3] = v4.w;
      }
      op.o = rc[ND + 2];
      op.t0n = rc[ND];
#pragma unroll
      for (int di = 0; di < ND; di++) {
        op.x[di] = __ldg(xb + rc[di]);  // signed: a mirrored read is a row shift s < 0
        op.h[di] = __ldg(hb + (hoff[di] + (uint32_t)op.o));
      }
      op.t0 = t0ob[(uint32_t)rc[ND + 1]];  // plain load: T^_0 is updated in place
    };
    double fs = 0.0, q1 = 0.0;
    int nnzu = 0, c1 = 0, nb = 0;
    uint32_t nso = 0;
    Ops cur, nxt;
    if (ncnt > 0) load(0, cur);
    for (int t = 0; t < ncnt; t++) {
      if (t + 1 < ncnt) load(t + 1, nxt);
      // products k ascending (offsets descending); a zero operand adds +-0, which leaves the
      // running sum unchanged (it is never -0), exactly as the oracle's skipped product
      double acc = 0.0, v0 = 0.0;
#pragma unroll
      for (int di = 0; di < ND; di++) {
        const double v = H0PREV ? cur.x[di] : (fabs(cur.x[di]) > tau_prev ? cur.x[di] : 0.0);
        if (di == dz) v0 = v;
        acc = __dadd_rn(acc, __dmul_rn(v, cur.h[di]));
      }
      if (cur.t0n >= 0) t0nb[(uint32_t)cur.t0n] = cur.t0 + v0;  // fused T^_0 update (d = 0 operand)
      const double x = acc / div;  // acc = +0 gives +0
      nsb[nso] = x;
      nso += pstride;
      if (x != 0.0) {
        // half window: an off-diagonal value stands for itself and its mirror
        const int mult = (a.half && cur.o != 0) ? 2 : 1;
        nnzu += mult;
        const double ax = fabs(x);
        if (ax <= floor_tau) {
          fs += mult * (x * x);
        } else if (ax <= eps_g) {
          q1 += mult * (x * x);
          if (nb < a.band_cap) {
            a.band_val[(int64_t)nb * nl + l] = x;
            a.band_col[(int64_t)nb * nl + l] = (int32_t)(r + cur.o);
          }
          nb++;
        } else {
          c1 += mult;
        }
      }
      cur = nxt;
    }
    a.row_cnt[l] = nb;
    a.row_fsum[l] = fs;
    a.row_p1[l] = q1;
    a.row_nnz[l] = nnzu;
    a.row_c1[l] = c1;
    if (nb > a.band_cap) atomicMax(a.band_need, (unsigned long long)nb);
  }
}
// T^_0^(i-1) = T^_0^(i-2) + S^_{i-1} as a separate streaming pass (H0 without a main
// diagonal: cum_{i-1} is then not inside W_i, so the update cannot ride on the term's loop)
__global__ void __launch_bounds__(kWinThreads) k_taylor_win_t0(WinArgs a) {
  extern __shared__ double wsm[];
  const int ccnt = a.c1cnt;
  int16_t *s_mc = reinterpret_cast<int16_t *>(wsm);
  int16_t *s_mw = s_mc + ccnt;
  for (int i = threadIdx.x; i < ccnt; i += blockDim.x) {
    s_mc[i] = a.mapC[i];
    s_mw[i] = a.mapW[i];
  }
  __syncthreads();
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= a.nrows) return;
  const int64_t r = a.row0 + l;
  for (int q = 0; q < ccnt; q++) {
    const int pc = s_mc[q], pw = s_mw[q];
    const double t0 = pc >= 0 ? a.T0old[(size_t)pc * a.nrows + l] : 0.0;  // in place: plain load
    double sv = 0.0;
    if (pw >= 0) {
      sv = a.prev_is_h0 ? __ldg(a.dia + (size_t)(a.nd - 1 - pw) * (size_t)a.n + (size_t)r)
                        : __ldg(a.pS + (size_t)pw * a.nrows + l);
      if (!a.prev_is_h0 && !(fabs(sv) > a.tau_prev)) sv = 0.0;
    }
    a.T0new[(size_t)a.cumU[q] * a.nrows + l] = t0 + sv;
  }
}
void launch_taylor_win_t0(const WinArgs &a, cudaStream_t st) {
  if (a.nrows == 0 || a.c1cnt == 0) return;
  const int smem = a.c1cnt * 4 + 16;
  cudaFuncSetAttribute(k_taylor_win_t0, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  KL;
  k_taylor_win_t0<<<(unsigned)((a.nrows + kWinThreads - 1) / kWinThreads), kWinThreads, smem, st>>>(a);
}
template <int ND>
static void launch_win_nd(const WinArgs &a, int smem, int ctas_per_sm, int sms, cudaStream_t st) {
  auto kf = a.prev_is_h0 ? k_taylor_win<ND, true> : k_taylor_win<ND, false>;
  cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int64_t tiles = (a.nrows + kWinThreads - 1) / kWinThreads;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)sms * ctas_per_sm));
  KL;
  kf<<<grid, kWinThreads, smem, st>>>(a);
}
void launch_taylor_win(const WinArgs &a, int ctas_per_sm, int sms, cudaStream_t st) {
  if (a.nrows == 0) return;
  const int smem = taylor_win_smem_bytes(a.nd, a.ncnt, a.c1cnt);
  // the kernel is specialised on the number of diagonals (records and sums unrolled)
  switch (taylor_win_kernel_nd(a.nd)) {
    case 3: launch_win_nd<3>(a, smem, ctas_per_sm, sms, st); break;
    case 5: launch_win_nd<5>(a, smem, ctas_per_sm, sms, st); break;
    case 7: launch_win_nd<7>(a, smem, ctas_per_sm, sms, st); break;
    case 1: launch_win_nd<1>(a, smem, ctas_per_sm, sms, st); break;
    case 2: launch_win_nd<2>(a, smem, ctas_per_sm, sms, st); break;
    case 4: launch_win_nd<4>(a, smem, ctas_per_sm, sms, st); break;
    case 6: launch_win_nd<6>(a, smem, ctas_per_sm, sms, st); break;
    case 8: launch_win_nd<8>(a, smem, ctas_per_sm, sms, st); break;
    case 9: launch_win_nd<9>(a, smem, ctas_per_sm, sms, st); break;
    default: launch_win_nd<kDiaMax>(a, smem, ctas_per_sm, sms, st); break;
  }
}
// Algorithm 4.1 pass over the staged band values (position-major, row_cnt per row):
// rowsum[l] = sum over k < cnt of x^2 with |x| <= tau (k order), count[l] = |x| > tau
__global__ void k_win_band_pass(int64_t nl, const int64_t *cnt, const double *band_val, double tau,
                                double *rowsum, int64_t *rowcnt, int half, const int32_t *band_col,
                                int64_t row0) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nl) return;
  const int64_t c = cnt[l];
  double s = 0.0;
  int64_t k = 0;
  for (int64_t j = 0; j < c; j++) {
    const double x = band_val[(size_t)j * nl + l];
    const int mult = (half && band_col[(size_t)j * nl + l] != row0 + l) ? 2 : 1;
    if (fabs(x) <= tau) s += mult * (x * x);
    else k += mult;
  }
  if (rowsum) rowsum[l] = s;
  if (rowcnt) rowcnt[l] = k;
}
void launch_win_band_pass(int64_t nl, const int64_t *cnt, const double *band_val, double tau, double *rowsum,
                          int64_t *rowcnt, cudaStream_t st, int half, const int32_t *band_col, int64_t row0) {
  if (nl == 0) return;
  KL;
  k_win_band_pass<<<grid_for(nl, kThreads), kThreads, 0, st>>>(nl, cnt, band_val, tau, rowsum, rowcnt, half,
                                                               band_col, row0);
}
// FINAL: T^_0 = T^_0^(m-1) + S^_m over cum_m.  Count pass (thread per row), then the write
// pass: a CTA takes 32 rows, computes 32 positions x 32 rows per round into a shared tile
// (loads coalesced over rows) and each warp writes 4 rows' nonzeros of the round
// contiguously (columns ascending) at rp_out[l] + the row's running count.
__device__ __forceinline__ double win_prev(const WinArgs &a, int p, int64_t l, int64_t r, int nd) {
  if (a.prev_is_h0) return __ldg(a.dia + (size_t)(nd - 1 - p) * (size_t)a.n + (size_t)r);
  const double x = __ldg(a.pS + (size_t)p * (size_t)(a.plane ? a.plane : a.nrows) + (size_t)a.padr + (size_t)l);
  return fabs(x) > a.tau_prev ? x : 0.0;
}
__device__ __forceinline__ double win_t0(const WinArgs &a, const int16_t *mc, const int16_t *mw, int q,
                                         int64_t l, int64_t r, int nd) {
  const int pc = mc[q], pw = mw[q];
  const double t0 = pc >= 0 ? __ldg(a.T0old + (size_t)pc * a.nrows + l) : 0.0;
  const double sv = pw >= 0 ? win_prev(a, pw, l, r, nd) : 0.0;
  return t0 + sv;
}
// sym (one GPU, symmetric H, symmetric offset list): an entry below the diagonal (o < 0) is
// read as its mirror (r + o, -o), position ccnt - 1 - q: T^_0 exactly symmetric (K3s input)
__device__ __forceinline__ double win_t0s(const WinArgs &a, const int16_t *mc, const int16_t *mw,
                                          const int32_t *offs, int q, int64_t l, int64_t r, int nd) {
  if (a.half) {  // the maps point at |o|: an entry below the diagonal is its mirror's, row r + o
    const int32_t o = offs[q];
    if (o < 0) return l + o < 0 ? 0.0 : win_t0(a, mc, mw, q, l + o, r + o, nd);
  } else if (a.sym) {
    const int32_t o = offs[q];
    if (o < 0) return l + o < 0 ? 0.0 : win_t0(a, mc, mw, a.c1cnt - 1 - q, l + o, r + o, nd);
  }
  return win_t0(a, mc, mw, q, l, r, nd);
}
__global__ void __launch_bounds__(kWinThreads) k_taylor_win_count(WinArgs a, int64_t *cnt) {
  extern __shared__ double wsm[];
  const int ccnt = a.c1cnt;
  int32_t *s_off = reinterpret_cast<int32_t *>(wsm);
  int16_t *s_mc = reinterpret_cast<int16_t *>(s_off + ccnt);
  int16_t *s_mw = s_mc + ccnt;
  for (int i = threadIdx.x; i < ccnt; i += blockDim.x) {
    s_mc[i] = a.mapC[i];
    s_mw[i] = a.mapW[i];
    s_off[i] = a.coffs[i];
  }
  __syncthreads();
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= a.nrows) return;
  const int64_t r = a.row0 + l;
  int64_t c = 0;
#pragma unroll 4
  for (int q = 0; q < ccnt; q++) c += win_t0s(a, s_mc, s_mw, s_off, q, l, r, a.nd) != 0.0;
  cnt[l] = c;
}
constexpr int kWinWT = 256;  // write pass: 8 warps, 32 rows per CTA
__global__ void __launch_bounds__(kWinWT) k_taylor_win_write(WinArgs a, const int64_t *rp_out, int32_t *col_out,
                                                             double *val_out) {
  extern __shared__ double wsm[];
  const int ccnt = a.c1cnt;
  double *tile = wsm;  // [32][33]
  int16_t *s_mc = reinterpret_cast<int16_t *>(tile + 32 * 33);
  int16_t *s_mw = s_mc + ccnt;
  int32_t *s_off = reinterpret_cast<int32_t *>(s_mw + ccnt);  // 4 ccnt bytes after s_mc
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  for (int i = tid; i < ccnt; i += blockDim.x) {
    s_mc[i] = a.mapC[i];
    s_mw[i] = a.mapW[i];
    s_off[i] = a.coffs[i];
  }
  __syncthreads();
  const int64_t lb = (int64_t)blockIdx.x * 32;
  const int64_t lr = lb + lane;  // the row this lane loads
  const bool lok = lr < a.nrows;
  int64_t cur[4];
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const int64_t lw = lb + w * 4 + j;
    cur[j] = lw < a.nrows ? rp_out[lw] : 0;
  }
  for (int q0 = 0; q0 < ccnt; q0 += 32) {
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int q = q0 + w * 4 + j;
      tile[(w * 4 + j) * 33 + lane] = (lok && q < ccnt) ? win_t0s(a, s_mc, s_mw, s_off, q, lr, a.row0 + lr, a.nd) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int rl = w * 4 + j;
      const int64_t lw = lb + rl;
      const double v = tile[lane * 33 + rl];
      const unsigned m = __ballot_sync(FULL_MASK, v != 0.0);
      if (v != 0.0 && lw < a.nrows) {
        const int64_t p = cur[j] + __popc(m & lanemask_lt());
        col_out[p] = (int32_t)(a.row0 + lw + s_off[q0 + lane]);
        val_out[p] = v;
      }
      cur[j] += __popc(m);
    }
    __syncthreads();
  }
}
void launch_taylor_win_final(const WinArgs &a, int64_t *cnt, const int64_t *rp_out, int32_t *col_out,
                             double *val_out, cudaStream_t st) {
  if (a.nrows == 0) return;
  if (!rp_out) {
    const int smem = a.c1cnt * 8 + 16;
    cudaFuncSetAttribute(k_taylor_win_count, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    KL;
    k_taylor_win_count<<<(unsigned)((a.nrows + kWinThreads - 1) / kWinThreads), kWinThreads, smem, st>>>(a, cnt);
  } else {
    const int smem = 32 * 33 * 8 + a.c1cnt * 8 + 32;
    cudaFuncSetAttribute(k_taylor_win_write, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    KL;
    k_taylor_win_write<<<(unsigned)((a.nrows + 31) / 32), kWinWT, smem, st>>>(a, rp_out, col_out, val_out);
  }
}
// ------------------------------------------------------------------------------------
// Squaring order for lattice-structured H (grid stencils; plan time, on the device): the
// rows are relabelled into 8-row aggregates that tile the grid -- 2D: the diamond tiles
// {0 <= x+y-4u < 4, 0 <= x-y+D-4v < 4} (8 lattice points each, the shape of the L1 balls the
// iterates' rows cover: as few column blocks per block row as the host BFS aggregates),
// 3D: 2 x 2 x 2 cubes.  Tiles are numbered line by line (u-major / z-major), so the relabelled
// matrix keeps the bandwidth of the index order (the BSR build's per-block-row column span);
// the block kernel's PROCESSING order takes the block rows supertile by supertile (16 x 16
// diamonds / 8 x 8 x 8 cubes) for L2 locality of the block rows in flight.  Tiles cut by
// the grid's boundary hold fewer rows: new index = (rows of earlier tiles) + (rank of the
// row's cell among its tile's occupied cells) -- a mask pass, a count + scan, a placement.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void lattice_tile(const LatticeDesc &L, int64_t r, int64_t &tile, int &c,
                                             int64_t &super) {
  if (L.dims == 2) {
    const int64_t x = r % L.G, y = r / L.G;
    const int64_t sx = x + y, dx = x - y + L.Dp;
    const int64_t u = sx >> 2, v = dx >> 2;
    c = (int)((sx & 3) * 2 + ((dx & 3) >> 1));
    tile = u * L.nv + v;
    super = (u >> 4) * L.nv16 + (v >> 4);
  } else {
    const int64_t x = r % L.G, y = (r / L.G) % L.Gy, z = r / L.GH;
    const int64_t tx = x >> 1, ty = y >> 1, tz = z >> 1;
    c = (int)(((z & 1) << 2) | ((y & 1) << 1) | (x & 1));
    tile = (tz * L.nty + ty) * L.ntx + tx;
    super = ((tz >> 3) * L.ny8 + (ty >> 3)) * L.nx8 + (tx >> 3);
  }
}
__global__ void k_lattice_mask(LatticeDesc L, unsigned *mask) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= L.n) return;
  int64_t t, sp;
  int c;
  lattice_tile(L, r, t, c, sp);
  atomicOr(&mask[t], 1u << c);
}
// per tile: 1 if full (8 rows) / the row count if partial, for the two scans below
__global__ void k_lattice_counts(int64_t ntiles, const unsigned *mask, int64_t *full, int64_t *part) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntiles) return;
  const int c = __popc(mask[t]);
  full[t] = c == 8;
  part[t] = c == 8 ? 0 : c;
}
// New index of row r.  Every 8-row group of the new numbering is one full tile, or 8 rows of
// partial (boundary-cut) tiles taken in tile order and placed where the 8th of them appears:
// groups before tile t = F_t (full tiles before t) + floor(P_t / 8) (completed partial groups,
// P_t = partial rows before t).  So the block rows of the BSR view stay tile-aligned across
// the boundary.
__global__ void k_lattice_place(LatticeDesc L, const unsigned *mask, const int64_t *F, const int64_t *P,
                                int64_t ntiles, int64_t *perm, int64_t *inv) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= L.n) return;
  int64_t t, sp;
  int c;
  lattice_tile(L, r, t, c, sp);
  const unsigned m = mask[t];
  const int k = __popc(m & ((1u << c) - 1u));
  int64_t ni;
  if (__popc(m) == 8) {
    ni = 8 * (F[t] + (P[t] >> 3)) + k;
  } else {
    const int64_t q = P[t] + k, g = q >> 3, last = 8 * g + 7;
    // the tile holding the group's 8th row: the first j with P[j] > last, minus one
    // (P has ntiles + 1 entries; none: the final, incomplete group goes after every tile)
    int64_t lo = 0, hi = ntiles + 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (P[mid] > last) hi = mid;
      else lo = mid + 1;
    }
    const int64_t istar = lo - 1;  // in [t, ntiles]
    ni = 8 * (F[istar] + g) + (q & 7);
  }
  inv[r] = ni;
  perm[ni] = r;
}
// processing order of the block rows: counting sort by the supertile of each block row's
// first row, then each supertile's block rows sorted ascending (deterministic)
__global__ void k_lattice_block_keys(LatticeDesc L, const int64_t *perm, int64_t nbt, int32_t *key,
                                     int32_t *scnt) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbt) return;
  int64_t t, sp;
  int c;
  lattice_tile(L, perm[8 * b], t, c, sp);
  key[b] = (int32_t)sp;
  atomicAdd(&scnt[sp], 1);
}
__global__ void k_lattice_block_scatter(int64_t nbt, const int32_t *key, const int64_t *start, int32_t *cur,
                                        int64_t *x) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nbt) return;
  const int32_t k = key[b];
  x[start[k] + atomicAdd(&cur[k], 1)] = b;
}
__global__ void k_i64_to_i32(const int64_t *in, int64_t n, int32_t *out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (int32_t)in[i];
}
__global__ void k_iota_i32(int64_t n, int32_t *x) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = (int32_t)i;
}
// scratch: mask ntiles u32; cnt and off 2 (ntiles + 1) i64 each (reused for the nsuper
// supertiles and the block rows: sized >= max(2 (ntiles + 1), nsuper + 1, nbt)), key nbt i32,
// scnt / cur nsuper i32, flag 1 int
void launch_lattice_order(const LatticeDesc &L, unsigned *mask, int64_t *cnt, int64_t *off, int64_t *scan_tmp,
                          int32_t *key, int32_t *scnt, int32_t *cur, int *flag, int64_t *perm, int64_t *inv,
                          int32_t *border, cudaStream_t st) {
  // cnt / off hold two arrays of ntiles + 1 each: [full | part] and their scans [F | P]
  const int64_t nt1 = L.ntiles + 1;
  cudaMemsetAsync(mask, 0, (size_t)L.ntiles * sizeof(unsigned), st);
  KL;
  k_lattice_mask<<<grid_for(L.n, kThreads), kThreads, 0, st>>>(L, mask);
  KL;
  k_lattice_counts<<<grid_for(L.ntiles, kThreads), kThreads, 0, st>>>(L.ntiles, mask, cnt, cnt + nt1);
  launch_exclusive_scan(cnt, L.ntiles, off, scan_tmp, st);
  launch_exclusive_scan(cnt + nt1, L.ntiles, off + nt1, scan_tmp, st);
  KL;
  k_lattice_place<<<grid_for(L.n, kThreads), kThreads, 0, st>>>(L, mask, off, off + nt1, L.ntiles, perm, inv);
  const int64_t nbt = (L.n + 7) / 8;
  cudaMemsetAsync(scnt, 0, (size_t)L.nsuper * sizeof(int32_t), st);
  cudaMemsetAsync(cur, 0, (size_t)L.nsuper * sizeof(int32_t), st);
  cudaMemsetAsync(flag, 0, sizeof(int), st);
  KL;
  k_lattice_block_keys<<<grid_for(nbt, kThreads), kThreads, 0, st>>>(L, perm, nbt, key, scnt);
  KL;
  k_i32_to_i64<<<grid_for(L.nsuper, kThreads), kThreads, 0, st>>>(scnt, L.nsuper, cnt);
  launch_exclusive_scan(cnt, L.nsuper, off, scan_tmp, st);
  KL;
  k_lattice_block_scatter<<<grid_for(nbt, kThreads), kThreads, 0, st>>>(nbt, key, off, cur, cnt);
  KL;
  k_sort_segments_i64<<<(int)std::max<int64_t>(1, std::min<int64_t>(L.nsuper, 148 * 8)), 256, 0, st>>>(off, L.nsuper, cnt, flag);
  KL;
  k_i64_to_i32<<<grid_for(nbt, kThreads), kThreads, 0, st>>>(cnt, nbt, border);
}
void launch_iota_i32(int64_t n, int32_t *x, cudaStream_t st) {
  if (n == 0) return;
  KL;
  k_iota_i32<<<grid_for(n, kThreads), kThreads, 0, st>>>(n, x);
}
// count of x[0..cnt) with |x| > tau (nnz of a term's kept band values)
__global__ void k_count_above(const double *x, int64_t cnt, double tau, unsigned long long *out) {
  unsigned long long c = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x)
    c += fabs(x[i]) > tau;
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}
void launch_count_above(const double *x, int64_t cnt, double tau, unsigned long long *out, cudaStream_t st) {
  cudaMemsetAsync(out, 0, sizeof(unsigned long long), st);
  if (cnt == 0) return;
  KL;
  k_count_above<<<grid_for(cnt, kThreads, 148 * 8), kThreads, 0, st>>>(x, cnt, tau, out);
}

// out64[i] = in32[i] (plan-time helper, no host round trip)
void launch_i32_to_i64(const int32_t *in, int64_t n, int64_t *out, cudaStream_t st) {
  if (n == 0) return;
  KL;
  k_i32_to_i64<<<grid_for(n, kThreads), kThreads, 0, st>>>(in, n, out);
}
// ------------------------------------------------------------------------------------
// fp64 throughput of this GPU (the roofline denominator of the squaring kernels, measured
// where the bench runs): 8 independent DFMA chains per thread, or 8 independent DMMA
// (mma.m8n8k4.f64) accumulators per warp, over a grid of 8 CTAs x 256 threads per SM.
// ------------------------------------------------------------------------------------
constexpr int kPeakIters = 4096, kPeakChains = 8;
__global__ void __launch_bounds__(256) k_peak_dfma(double *out, double a, double b) {
  double x[kPeakChains];
#pragma unroll
  for (int c = 0; c < kPeakChains; c++) x[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < kPeakIters; it++) {
#pragma unroll
    for (int c = 0; c < kPeakChains; c++) x[c] = fma(x[c], a, b);
  }
  double t = 0.0;
#pragma unroll
  for (int c = 0; c < kPeakChains; c++) t += x[c];
  out[(size_t)blockIdx.x * blockDim.x + threadIdx.x] = t;
}
__global__ void __launch_bounds__(256) k_peak_dmma(double *out, double a, double b) {
  double d0[kPeakChains], d1[kPeakChains];
#pragma unroll
  for (int c = 0; c < kPeakChains; c++) d0[c] = d1[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < kPeakIters; it++) {
#pragma unroll
    for (int c = 0; c < kPeakChains; c++) dmma884(d0[c], d1[c], a, b);
  }
  double t = 0.0;
#pragma unroll
  for (int c = 0; c < kPeakChains; c++) t += d0[c] + d1[c];
  out[(size_t)blockIdx.x * blockDim.x + threadIdx.x] = t;
}
double fp64_peak_flops_per_launch(int which, int sms) {
  const double threads = (double)sms * 8 * 256;
  return which == 0 ? threads * kPeakIters * kPeakChains * 2.0                  // 2 per DFMA
                    : threads / 32 * kPeakIters * kPeakChains * 512.0;        // 8x8x4 x 2 per DMMA
}
void launch_fp64_peak(int which, int sms, double *out, cudaStream_t st) {
  KL;
  if (which == 0)
    k_peak_dfma<<<sms * 8, 256, 0, st>>>(out, 0.999, 1e-3);
  else
    k_peak_dmma<<<sms * 8, 256, 0, st>>>(out, 0.999, 1e-3);
}

}  // namespace sx
