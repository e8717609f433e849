// Tall-skinny dense kernels (l >> n, n <= 64) on sm_100a, FP64.
//
// X lives column-major on the device (X[j*ld + i]) so that one thread per
// instance reads its row with fully coalesced warp loads (32 consecutive
// instances of a column = 256 contiguous bytes per load instruction).
// Each thread accumulates n partial sums in registers over its grid-stride
// rows; a fixed-shape warp/block tree produces one n-vector per block and a
// fixed-order second stage finishes it.  The per-row dot x_i.v is the
// sequential j = 0..n-1 loop of FeatureMatrix::row_dot (linalg.cpp:75-86)
// compiled without FMA contraction, so margins z -- and therefore the
// L2-SVM active set I (loss.cpp:94-122) -- are bit-identical to the
// reference's.
#include "common.cuh"
#include "kernels.h"

namespace tb {

namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ double log1p_exp_neg(double t) {  // loss.hpp:99-102
  if (t >= 0.0) return log1p(exp(-t));
  return -t + log1p(exp(t));
}

template <int NMAX, int LOSS>
__global__ void __launch_bounds__(kBlock) dense_forward_kernel(
    long long l, int n, long long ld, const double* __restrict__ X, const double* __restrict__ w,
    const double* __restrict__ y, double C, double* __restrict__ z, double* __restrict__ zhat,
    double* __restrict__ dvec, uint8_t* __restrict__ mask, ObjScalars* obj, Scratch sc) {
  __shared__ double s_w[NMAX];
  __shared__ double sh[kBlock / kWarp + 1];
  for (int j = threadIdx.x; j < NMAX; j += kBlock) s_w[j] = j < n ? w[j] : 0.0;
  __syncthreads();
  double term_acc = 0.0, cnt_acc = 0.0;
  for (long long i = blockIdx.x * (long long)kBlock + threadIdx.x; i < l;
       i += (long long)gridDim.x * kBlock) {
    double x[NMAX];
#pragma unroll
    for (int j = 0; j < NMAX; ++j) x[j] = j < n ? X[(long long)j * ld + i] : 0.0;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < NMAX; ++j)
      if (j < n) s += x[j] * s_w[j];
    const double yi = y[i];
    z[i] = s;
    if (LOSS == kLossLogistic) {
      const double t = yi * s;
      const double sig = 1.0 / (1.0 + exp(t));
      zhat[i] = -yi * sig;
      dvec[i] = (1.0 - sig) * sig;
      term_acc += log1p_exp_neg(t);
    } else {
      const double margin = 1.0 - yi * s;
      if (margin > 0.0) {
        mask[i] = 1;
        term_acc += margin * margin;
        cnt_acc += 1.0;
      } else {
        mask[i] = 0;
      }
    }
  }
  const double bt = block_sum<kBlock>(term_acc, sh, true);
  const double bc = block_sum<kBlock>(cnt_acc, sh, true);
  if (threadIdx.x == 0) {
    sc.partials[2 * blockIdx.x] = bt;
    sc.partials[2 * blockIdx.x + 1] = bc;
  }
  if (last_block_arrive(sc.tickets + T_FUN)) {
    const double tot = reduce_partials<kBlock>(sc.partials, gridDim.x, 2, 0, sh);
    const double cnt = reduce_partials<kBlock>(sc.partials, gridDim.x, 2, 1, sh);
    // ww of a short vector is done here, serially, like dot() (linalg.cpp:267-272)
    if (threadIdx.x == 0) {
      double ww = 0.0;
      for (int j = 0; j < n; ++j) ww += w[j] * w[j];
      obj->ww = ww;
      obj->f = 0.5 * ww + C * tot;
      obj->nact = (long long)cnt;
      obj->red[0] = tot;
      obj->red[1] = cnt;
    }
  }
}

// Per-block n-vector partials; block tree over warps then a fixed warp order.
template <int NMAX>
__device__ __forceinline__ void store_block_vector(const double (&acc)[NMAX], int n,
                                                   double* out_block) {
  __shared__ double s_red[kBlock / kWarp][NMAX];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NMAX; ++j) {
    if (j < n) {
      const double v = warp_sum(acc[j]);
      if (lane == 0) s_red[wid][j] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x < n) {
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kBlock / kWarp; ++w) t += s_red[w][threadIdx.x];
    out_block[threadIdx.x] = t;
  }
}

template <int NMAX, int KIND, int LOSS>
__global__ void __launch_bounds__(kBlock) dense_accum_kernel(
    long long l, int n, long long ld, const double* __restrict__ X, const double* __restrict__ v,
    const double* __restrict__ zhat, const double* __restrict__ dvec,
    const uint8_t* __restrict__ mask, const double* __restrict__ z, const double* __restrict__ y,
    double* __restrict__ partials) {
  __shared__ double s_v[NMAX];
  if (KIND == DA_HV) {
    for (int j = threadIdx.x; j < NMAX; j += kBlock) s_v[j] = j < n ? v[j] : 0.0;
    __syncthreads();
  }
  double acc[NMAX];
#pragma unroll
  for (int j = 0; j < NMAX; ++j) acc[j] = 0.0;
  for (long long i = blockIdx.x * (long long)kBlock + threadIdx.x; i < l;
       i += (long long)gridDim.x * kBlock) {
    if (LOSS == kLossSvm && mask != nullptr && !mask[i]) continue;  // i not in I
    if (KIND == DA_HV) {
      double x[NMAX];
#pragma unroll
      for (int j = 0; j < NMAX; ++j) x[j] = j < n ? X[(long long)j * ld + i] : 0.0;
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < NMAX; ++j)
        if (j < n) s += x[j] * s_v[j];
      // LR: a0_i = (x_i.v) * dvec_i (loss.cpp:85-89); SVM: row_axpy(i, row_dot(i,v)) (:455)
      const double c = LOSS == kLossLogistic ? s * dvec[i] : s;
#pragma unroll
      for (int j = 0; j < NMAX; ++j) acc[j] += c * x[j];
    } else if (KIND == DA_GRAD) {
      const double c = LOSS == kLossLogistic ? zhat[i] : z[i] - y[i];
#pragma unroll
      for (int j = 0; j < NMAX; ++j)
        if (j < n) acc[j] += c * X[(long long)j * ld + i];
    } else {  // DA_PRECOND: row_axpy_squared, out += a*v*v
      const double c = LOSS == kLossLogistic ? dvec[i] : 1.0;
#pragma unroll
      for (int j = 0; j < NMAX; ++j) {
        if (j < n) {
          const double xv = X[(long long)j * ld + i];
          acc[j] += (c * xv) * xv;
        }
      }
    }
  }
  store_block_vector<NMAX>(acc, n, partials + (long long)blockIdx.x * n);
}

__global__ void __launch_bounds__(1024) dense_finalize_kernel(int n, const double* partials,
                                                             int nparts, EpiView E, double* out) {
  // thread t: coordinate j = t % 64, part group t / 64 (16 groups)
  __shared__ double s_part[1024];
  const int j = threadIdx.x & 63, grp = threadIdx.x >> 6;
  double acc = 0.0;
  if (j < n)
    for (int b = grp; b < nparts; b += 16) acc += __ldcg(partials + (long long)b * n + j);
  s_part[threadIdx.x] = acc;
  __syncthreads();
  if (grp == 0 && j < n) {
    double t = 0.0;
    for (int g = 0; g < 16; ++g) t += s_part[g * 64 + j];
    out[j] = E.kind == EPI_VEC ? E.base[j] + E.scale * t
                               : (E.kind == EPI_CONST ? E.cbase + E.scale * t : t);
  }
}

__global__ void transpose_kernel(const double* __restrict__ rm, long long rows, int n,
                                 double* __restrict__ X, long long ld, long long row0) {
  __shared__ double tile[32][33];
  const long long rb = blockIdx.x * 32LL;
  const int cb = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const long long r = rb + k;
    const int c = cb + threadIdx.x;
    if (r < rows && c < n) tile[k][threadIdx.x] = rm[r * n + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = cb + k;
    const long long r = rb + threadIdx.x;
    if (r < rows && c < n) X[(long long)c * ld + row0 + r] = tile[threadIdx.x][k];
  }
}

// Active-set compaction, ascending (the IndexSet invariant, linalg.hpp:65-86).
constexpr int kChunk = 1024;  // mask entries per block (256 threads x 4)

__global__ void count_kernel(long long l, const uint8_t* mask, int32_t* counts) {
  __shared__ double sh[kBlock / kWarp + 1];
  const long long base = blockIdx.x * (long long)kChunk + threadIdx.x * 4;
  int c = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (base + k < l) c += mask[base + k] != 0;
  const double tot = block_sum<kBlock>((double)c, sh, true);
  if (threadIdx.x == 0) counts[blockIdx.x] = (int32_t)tot;
}

// exclusive scan of counts (single block, sequential per thread chunk)
__global__ void scan_kernel(int32_t* counts, int nb, long long* total) {
  __shared__ long long s_sum[1024];
  const int per = (nb + 1023) / 1024;
  const int b0 = threadIdx.x * per;
  long long s = 0;
  for (int k = 0; k < per; ++k)
    if (b0 + k < nb) s += counts[b0 + k];
  s_sum[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long run = 0;
    for (int t = 0; t < 1024; ++t) {
      const long long v = s_sum[t];
      s_sum[t] = run;
      run += v;
    }
    *total = run;
  }
  __syncthreads();
  long long run = s_sum[threadIdx.x];
  for (int k = 0; k < per; ++k) {
    if (b0 + k < nb) {
      const long long v = counts[b0 + k];
      counts[b0 + k] = (int32_t)run;
      run += v;
    }
  }
}

__global__ void scatter_kernel(long long l, const uint8_t* mask, const int32_t* offsets,
                               int32_t* idx) {
  __shared__ int s_warp[kBlock / kWarp];
  const long long base = blockIdx.x * (long long)kChunk + threadIdx.x * 4;
  int flags[4], c = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    flags[k] = (base + k < l) ? mask[base + k] != 0 : 0;
    c += flags[k];
  }
  // exclusive block scan of c (ballot-free warp scan on small ints)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int incl = c;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += t;
  }
  if (lane == 31) s_warp[wid] = incl;
  __syncthreads();
  int woff = 0;
  for (int w = 0; w < wid; ++w) woff += s_warp[w];
  int pos = offsets[blockIdx.x] + woff + incl - c;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (flags[k]) idx[pos++] = (int32_t)(base + k);
}

__global__ void gather_kernel(long long nI, int n, const double* __restrict__ X, long long ld,
                              const int32_t* __restrict__ idx, double* __restrict__ Xg,
                              long long ldg) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nI;
       k += (long long)gridDim.x * blockDim.x) {
    const long long i = idx[k];
    for (int j = 0; j < n; ++j) Xg[(long long)j * ldg + k] = X[(long long)j * ld + i];
  }
}

template <int NMAX>
void launch_forward(long long l, int n, long long ld, const double* X, int loss, const double* w,
                    const double* y, double C, double* z, double* zhat, double* dvec,
                    uint8_t* mask, ObjScalars* obj, Scratch sc, cudaStream_t s) {
  const int grid = dense_grid(l);
  if (loss == kLossLogistic)
    dense_forward_kernel<NMAX, kLossLogistic><<<grid, kBlock, 0, s>>>(l, n, ld, X, w, y, C, z, zhat,
                                                                      dvec, mask, obj, sc);
  else
    dense_forward_kernel<NMAX, kLossSvm><<<grid, kBlock, 0, s>>>(l, n, ld, X, w, y, C, z, zhat,
                                                                 dvec, mask, obj, sc);
}

template <int NMAX, int KIND>
void launch_accum_kind(long long l, int n, long long ld, const double* X, int loss, const double* v,
                       const double* zhat, const double* dvec, const uint8_t* mask,
                       const double* z, const double* y, double* partials, cudaStream_t s) {
  const int grid = dense_grid(l);
  if (loss == kLossLogistic)
    dense_accum_kernel<NMAX, KIND, kLossLogistic><<<grid, kBlock, 0, s>>>(l, n, ld, X, v, zhat,
                                                                          dvec, mask, z, y, partials);
  else
    dense_accum_kernel<NMAX, KIND, kLossSvm><<<grid, kBlock, 0, s>>>(l, n, ld, X, v, zhat, dvec,
                                                                     mask, z, y, partials);
}

template <int NMAX>
void launch_accum(int kind, long long l, int n, long long ld, const double* X, int loss,
                  const double* v, const double* zhat, const double* dvec, const uint8_t* mask,
                  const double* z, const double* y, double* partials, cudaStream_t s) {
  if (kind == DA_HV)
    launch_accum_kind<NMAX, DA_HV>(l, n, ld, X, loss, v, zhat, dvec, mask, z, y, partials, s);
  else if (kind == DA_GRAD)
    launch_accum_kind<NMAX, DA_GRAD>(l, n, ld, X, loss, v, zhat, dvec, mask, z, y, partials, s);
  else
    launch_accum_kind<NMAX, DA_PRECOND>(l, n, ld, X, loss, v, zhat, dvec, mask, z, y, partials, s);
}

}  // namespace

int dense_grid(int64_t l) {
  int64_t g = (l + kBlock - 1) / kBlock;
  int64_t cap = (int64_t)device_sm_count() * 4;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

#define TB_NMAX_DISPATCH(n, CALL)                      \
  if ((n) <= 8) { CALL(8); }                           \
  else if ((n) <= 16) { CALL(16); }                    \
  else if ((n) <= 24) { CALL(24); }                    \
  else if ((n) <= 32) { CALL(32); }                    \
  else if ((n) <= 40) { CALL(40); }                    \
  else if ((n) <= 48) { CALL(48); }                    \
  else { CALL(64); }

void dense_forward(int64_t l, int64_t n, int64_t ld, const double* X, int loss, const double* w,
                   const double* y, double C, double* z, double* zhat, double* dvec, uint8_t* mask,
                   ObjScalars* obj, Scratch sc, cudaStream_t s) {
#define TB_CALL(NM) launch_forward<NM>(l, (int)n, ld, X, loss, w, y, C, z, zhat, dvec, mask, obj, sc, s)
  TB_NMAX_DISPATCH(n, TB_CALL)
#undef TB_CALL
}

void dense_accum(int kind, int64_t l, int64_t n, int64_t ld, const double* X, int loss,
                 const double* v, const double* zhat, const double* dvec, const uint8_t* mask,
                 const double* z, const double* y, double* partials, cudaStream_t s) {
#define TB_CALL(NM) launch_accum<NM>(kind, l, (int)n, ld, X, loss, v, zhat, dvec, mask, z, y, partials, s)
  TB_NMAX_DISPATCH(n, TB_CALL)
#undef TB_CALL
}

void dense_finalize(int64_t n, const double* partials, int nparts, const EpiView& epi, double* out,
                    cudaStream_t s) {
  dense_finalize_kernel<<<1, 1024, 0, s>>>((int)n, partials, nparts, epi, out);
}

void dense_transpose_chunk(const double* rm, int64_t rows, int64_t n, double* X, int64_t ld,
                           int64_t row0, cudaStream_t s) {
  dim3 grid((unsigned)((rows + 31) / 32), (unsigned)((n + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(rm, rows, (int)n, X, ld, row0);
}

void compact_mask(int64_t l, const uint8_t* mask, int32_t* idx, int32_t* tmp, long long* count_out,
                  cudaStream_t s) {
  const int nb = (int)((l + kChunk - 1) / kChunk);
  if (nb == 0) {
    cudaMemsetAsync(count_out, 0, sizeof(long long), s);
    return;
  }
  count_kernel<<<nb, kBlock, 0, s>>>(l, mask, tmp);
  scan_kernel<<<1, 1024, 0, s>>>(tmp, nb, count_out);
  scatter_kernel<<<nb, kBlock, 0, s>>>(l, mask, tmp, idx);
}

void dense_gather(int64_t nI, int64_t n, const double* X, int64_t ld, const int32_t* idx,
                  double* Xg, int64_t ldg, cudaStream_t s) {
  long long g = (nI + 255) / 256;
  if (g > (long long)device_sm_count() * 16) g = (long long)device_sm_count() * 16;
  if (g < 1) g = 1;
  gather_kernel<<<(int)g, 256, 0, s>>>(nI, (int)n, X, ld, idx, Xg, ldg);
}

}  // namespace tb
