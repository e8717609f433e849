// Sparse kernels of the TRON hot path on sm_100a (FP64, HBM-bound).
//
//  * csr_forward / csr_dv: sub-warp vector-CSR row products over X
//    (matvec, linalg.cpp:154-162) fused with the per-instance epilogues of
//    logistic_fused_pass (loss.cpp:35-58), svm_fused_pass (loss.cpp:94-122)
//    and the D-scaling of logistic_hessian_vec (loss.cpp:82-92).
//  * csc_spmv: X^T u as a row product over the device-built CSC copy, i.e.
//    the reference's matvec_transpose / masked_matvec_transpose /
//    weighted_sq_col_sums (linalg.cpp:175-265) without its 64 private
//    n-length buffers and serial merge.  Work is split by merge path
//    (columns + nonzeros per 256-thread tile are constant), so Zipf-hot
//    columns do not unbalance the grid; split columns are combined by a
//    block-wide segmented scan and a fixed-order fix-up pass.  No atomics:
//    results are bit-reproducible run to run.
#include <cub/device/device_radix_sort.cuh>

#include "common.cuh"
#include "kernels.h"

namespace tb {

namespace {

constexpr int kBlock = 256;
constexpr int kIpt = 8;                 // merge items per thread
constexpr int kTile = kBlock * kIpt;    // merge items per tile

int g_sm_count = 0;

__device__ __forceinline__ double log1p_exp_neg(double t) {  // loss.hpp:99-102
  if (t >= 0.0) return log1p(exp(-t));
  return -t + log1p(exp(t));
}

// Streaming loads of matrix entries: read once per pass, keep them out of L1
// so the gathered vector (u or p) keeps the cache.
__device__ __forceinline__ int ldg_stream(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ldg_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// ---------------------------------------------------------------------------
// CSR forward pass: groups of G lanes per row.
// Lane `sub` of the group sums entries sub, sub+G, ... of the row; four
// entries are loaded before any gathered v_j is consumed (latency hiding).
template <int G>
__device__ __forceinline__ double row_dot_sub(const CsrView& X, long long row, int sub,
                                              const double* __restrict__ v) {
  const int beg = X.ptr[row], end = X.ptr[row + 1];
  double s = 0.0;
  int k = beg + sub;
  for (; k + 3 * G < end; k += 4 * G) {
    int c[4];
    double a[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      c[m] = ldg_stream(X.idx + k + m * G);
      a[m] = ldg_stream(X.val + k + m * G);
    }
    double b[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) b[m] = __ldg(v + c[m]);
#pragma unroll
    for (int m = 0; m < 4; ++m) s += a[m] * b[m];
  }
  for (; k < end; k += G) s += ldg_stream(X.val + k) * __ldg(v + ldg_stream(X.idx + k));
  return s;
}
// ---------------------------------------------------------------------------
template <int G, int LOSS>
__global__ void __launch_bounds__(kBlock) csr_forward_kernel(CsrView X, const double* __restrict__ w,
                                                            const double* __restrict__ y, double C,
                                                            double* __restrict__ z,
                                                            double* __restrict__ zhat,
                                                            double* __restrict__ dvec,
                                                            uint8_t* __restrict__ mask,
                                                            ObjScalars* obj, Scratch sc) {
  constexpr int RPW = kWarp / G;  // rows per warp
  __shared__ double sh[kBlock / kWarp + 1];
  const int lane = threadIdx.x & 31;
  const int sub = lane % G;
  const long long gwarp = (blockIdx.x * (long long)kBlock + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * kBlock) >> 5;
  double term_acc = 0.0, cnt_acc = 0.0;
  for (long long r0 = gwarp * RPW; r0 < X.rows; r0 += nwarps * RPW) {
    const long long row = r0 + lane / G;
    double s = 0.0;
    if (row < X.rows) {
      s = row_dot_sub<G>(X, row, sub, w);
    }
    s = group_sum<G>(s);
    if (sub == 0 && row < X.rows) {
      const double yi = y[row];
      z[row] = s;
      if (LOSS == kLossLogistic) {
        const double t = yi * s;
        const double sig = 1.0 / (1.0 + exp(t));  // exp overflow -> inf -> 0
        zhat[row] = -yi * sig;
        dvec[row] = (1.0 - sig) * sig;
        term_acc += log1p_exp_neg(t);
      } else {
        const double margin = 1.0 - yi * s;
        if (margin > 0.0) {
          mask[row] = 1;
          term_acc += margin * margin;
          cnt_acc += 1.0;
        } else {
          mask[row] = 0;
        }
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
    if (threadIdx.x == 0) {
      obj->f = 0.5 * obj->ww + C * tot;  // loss.cpp:57 / :121
      obj->nact = (long long)cnt;
      obj->red[0] = tot;
      obj->red[1] = cnt;
    }
  }
}

template <int G>
__global__ void __launch_bounds__(kBlock) csr_dv_kernel(CsrView X, const double* __restrict__ p,
                                                       const double* __restrict__ dvec,
                                                       const uint8_t* __restrict__ mask,
                                                       double* __restrict__ a) {
  constexpr int RPW = kWarp / G;
  const int lane = threadIdx.x & 31;
  const int sub = lane % G;
  const long long gwarp = (blockIdx.x * (long long)kBlock + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * kBlock) >> 5;
  for (long long r0 = gwarp * RPW; r0 < X.rows; r0 += nwarps * RPW) {
    const long long row = r0 + lane / G;
    bool active = row < X.rows;
    if (active && mask) active = mask[row] != 0;
    double s = 0.0;
    if (active) {
      s = row_dot_sub<G>(X, row, sub, p);
    }
    s = group_sum<G>(s);
    if (sub == 0 && row < X.rows) {
      // loss.cpp:86-89: a0_i *= dvec_i; svm indirect skips inactive rows.
      a[row] = mask ? (active ? s : 0.0) : s * dvec[row];
    }
  }
}

int forward_grid(int64_t rows, int group) {
  const int64_t rows_per_block = kBlock / group;
  int64_t want = (rows + rows_per_block - 1) / rows_per_block;
  int64_t cap = (int64_t)device_sm_count() * 8;
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return (int)want;
}

// ---------------------------------------------------------------------------
// Merge-path transposed product.
// ---------------------------------------------------------------------------
template <int UK, bool SQ>
__device__ __forceinline__ double weight(const UView& U, int r, double v) {
  double u;
  if (UK == U_VEC) {
    u = __ldg(U.u + r);
  } else if (UK == U_SVM_RESID) {
    u = U.mask[r] ? (U.z[r] - U.y[r]) : 0.0;
  } else {
    u = U.mask[r] ? 1.0 : 0.0;
  }
  // row_axpy: out += a*v ; row_axpy_squared: out += a*v*v  (linalg.cpp:88-109)
  return SQ ? (u * v) * v : u * v;
}

template <int EPI>
__device__ __forceinline__ void emit(const EpiView& E, double* out, long long j, double sum) {
  if (EPI == EPI_VEC)
    out[j] = E.base[j] + E.scale * sum;
  else if (EPI == EPI_CONST)
    out[j] = E.cbase + E.scale * sum;
  else
    out[j] = sum;
}

template <int UK, bool SQ, int EPI>
__global__ void __launch_bounds__(kBlock) merge_spmv_kernel(CsrView A, MergeView P, UView U,
                                                           EpiView E, double* __restrict__ out) {
  __shared__ double s_val[kTile];
  __shared__ int s_end[kTile];
  __shared__ double s_scan[kBlock];
  __shared__ int s_key[kBlock];
  __shared__ double s_wval[kBlock / kWarp];
  __shared__ int s_wkey[kBlock / kWarp];

  const int t = blockIdx.x;
  const int x0 = P.tile_row[t], y0 = P.tile_nz[t];
  const int nr = P.tile_row[t + 1] - x0;
  const int nz = P.tile_nz[t + 1] - y0;
  const int tid = threadIdx.x;

  // Stage the tile: all loads of a thread are issued before any is consumed
  // (kIpt coalesced idx/val loads in flight, then kIpt independent gathers).
  {
    int ridx[kIpt];
    double rval[kIpt];
#pragma unroll
    for (int m = 0; m < kIpt; ++m) {
      const int i = tid + m * kBlock;
      const bool ok = i < nz;
      ridx[m] = ok ? ldg_stream(A.idx + y0 + i) : 0;
      rval[m] = ok ? ldg_stream(A.val + y0 + i) : 0.0;
    }
#pragma unroll
    for (int m = 0; m < kIpt; ++m) {
      const int i = tid + m * kBlock;
      if (i < nr) s_end[i] = __ldg(A.ptr + x0 + 1 + i);
    }
    double w[kIpt];
#pragma unroll
    for (int m = 0; m < kIpt; ++m) w[m] = (tid + m * kBlock < nz) ? weight<UK, SQ>(U, ridx[m], rval[m]) : 0.0;
#pragma unroll
    for (int m = 0; m < kIpt; ++m) {
      const int i = tid + m * kBlock;
      if (i < nz) s_val[i] = w[m];
    }
  }
  __syncthreads();

  // Merge-path coordinate of this thread inside the tile.
  const int total = nr + nz;
  const int d = min(tid * kIpt, total);
  const int d_end = min(d + kIpt, total);
  int lo = max(d - nz, 0), hi = min(d, nr);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (s_end[mid] <= y0 + d - mid - 1)
      lo = mid + 1;
    else
      hi = mid;
  }
  int tx = lo, ty = d - lo;
  double acc = 0.0, first_val = 0.0;
  int first_col = -1;
  for (int step = d; step < d_end; ++step) {
    if (tx < nr && (ty >= nz || s_end[tx] <= y0 + ty)) {  // row (column of X) ends
      if (first_col < 0) {
        first_col = tx;
        first_val = acc;
      } else {
        emit<EPI>(E, out, (long long)x0 + tx, acc);  // wholly inside this thread
      }
      acc = 0.0;
      ++tx;
    } else {
      acc += s_val[ty];
      ++ty;
    }
  }

  // Block-wide inclusive segmented scan of the carries (keys are monotone).
  const int lane = tid & 31, wid = tid >> 5;
  int key = tx;
  double val = acc;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int k2 = __shfl_up_sync(0xffffffffu, key, off);
    const double v2 = __shfl_up_sync(0xffffffffu, val, off);
    if (lane >= off && k2 == key) val = v2 + val;
  }
  if (lane == 31) {
    s_wkey[wid] = key;
    s_wval[wid] = val;
  }
  __syncthreads();
  if (wid == 0) {
    constexpr int NW = kBlock / kWarp;
    int wk = lane < NW ? s_wkey[lane] : 0x7fffffff;
    double wv = lane < NW ? s_wval[lane] : 0.0;
#pragma unroll
    for (int off = 1; off < NW; off <<= 1) {
      const int k2 = __shfl_up_sync(0xffffffffu, wk, off);
      const double v2 = __shfl_up_sync(0xffffffffu, wv, off);
      if (lane >= off && k2 == wk) wv = v2 + wv;
    }
    if (lane < NW) {
      s_wkey[lane] = wk;
      s_wval[lane] = wv;
    }
  }
  __syncthreads();
  if (wid > 0 && s_wkey[wid - 1] == key) val = s_wval[wid - 1] + val;
  s_scan[tid] = val;
  s_key[tid] = key;
  __syncthreads();

  if (first_col >= 0) {
    double tot = first_val;
    if (tid > 0 && s_key[tid - 1] == first_col) tot = s_scan[tid - 1] + first_val;
    const long long col = (long long)x0 + first_col;
    if (first_col == 0 && A.ptr[x0] < y0)
      P.head[t] = tot;  // started in an earlier tile: finished by the fix-up pass
    else
      emit<EPI>(E, out, col, tot);
  }
  if (tid == kBlock - 1) P.carry[t] = s_scan[tid];
}

template <int EPI>
__global__ void __launch_bounds__(kBlock) merge_fixup_kernel(MergeView P, EpiView E,
                                                            double* __restrict__ out) {
  const int t = (blockIdx.x * kBlock + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= P.num_tiles) return;
  const int ts = P.fix_chain[t];
  if (ts < 0) return;
  double s = 0.0;
  for (int k = ts + lane; k < t; k += 32) s += P.carry[k];
  s = warp_sum(s);
  if (lane == 0) emit<EPI>(E, out, P.tile_row[t], s + P.head[t]);
}

__global__ void merge_plan_kernel(CsrView A, int32_t* tile_row, int32_t* tile_nz, int num_tiles) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > num_tiles) return;
  const long long total = (long long)A.rows + (long long)A.nnz;
  const long long diag = min((long long)t * kTile, total);
  long long lo = max(diag - (long long)A.nnz, 0LL), hi = min(diag, (long long)A.rows);
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if ((long long)A.ptr[mid + 1] <= diag - mid - 1)
      lo = mid + 1;
    else
      hi = mid;
  }
  tile_row[t] = (int32_t)lo;
  tile_nz[t] = (int32_t)(diag - lo);
}

__global__ void merge_chain_kernel(CsrView A, const int32_t* tile_row, const int32_t* tile_nz,
                                   int32_t* fix_chain, int num_tiles) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= num_tiles) return;
  const int x0 = tile_row[t], y0 = tile_nz[t];
  if (tile_row[t + 1] > x0 && A.ptr[x0] < y0) {
    // first tile ts whose end coordinate tile_row[ts+1] reaches x0
    int lo = 0, hi = t;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (tile_row[mid + 1] < x0)
        lo = mid + 1;
      else
        hi = mid;
    }
    fix_chain[t] = lo;
  } else {
    fix_chain[t] = -1;
  }
}

// CSC construction helpers
__global__ void expand_rows_kernel(CsrView X, int32_t* rowid) {
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = gw; r < X.rows; r += nw)
    for (int k = X.ptr[r] + lane; k < X.ptr[r + 1]; k += 32) rowid[k] = (int32_t)r;
}

__global__ void iota_kernel(int32_t* v, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

__global__ void permute_kernel(const int32_t* perm, const int32_t* rowid, const double* val,
                               int32_t* ridx, double* cval, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int32_t k = perm[i];
    ridx[i] = rowid[k];
    cval[i] = val[k];
  }
}

__global__ void col_ptr_kernel(const int32_t* sorted_cols, long long nnz, int32_t* cptr,
                               long long ncols) {
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j <= ncols;
       j += (long long)gridDim.x * blockDim.x) {
    long long lo = 0, hi = nnz;  // lower_bound(sorted_cols, j)
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (sorted_cols[mid] < j)
        lo = mid + 1;
      else
        hi = mid;
    }
    cptr[j] = (int32_t)lo;
  }
}

__global__ void narrow_kernel(const int64_t* in, int32_t* out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = (int32_t)in[i];
}

int grid_for(long long n, int block = 256) {
  long long g = (n + block - 1) / block;
  long long cap = (long long)device_sm_count() * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

int device_sm_count() {
  if (g_sm_count == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    g_sm_count = v;
  }
  return g_sm_count;
}

int choose_group(int64_t rows, int64_t nnz) {
  const double mean = rows > 0 ? (double)nnz / (double)rows : 0.0;
  if (mean >= 96) return 32;
  if (mean >= 32) return 16;
  if (mean >= 12) return 8;
  if (mean >= 4) return 4;
  return 2;
}

#define TB_GROUP_DISPATCH(G, ...)      \
  switch (G) {                         \
    case 32: { constexpr int GG = 32; __VA_ARGS__; } break; \
    case 16: { constexpr int GG = 16; __VA_ARGS__; } break; \
    case 8: { constexpr int GG = 8; __VA_ARGS__; } break;   \
    case 4: { constexpr int GG = 4; __VA_ARGS__; } break;   \
    default: { constexpr int GG = 2; __VA_ARGS__; } break;  \
  }

void csr_forward(const CsrView& X, int group, int loss, const double* w, const double* y, double C,
                 double* z, double* zhat, double* dvec, uint8_t* mask, ObjScalars* obj,
                 Scratch sc, cudaStream_t s) {
  const int grid = forward_grid(X.rows, group);
  if (loss == kLossLogistic) {
    TB_GROUP_DISPATCH(group, (csr_forward_kernel<GG, kLossLogistic><<<grid, kBlock, 0, s>>>(
                                 X, w, y, C, z, zhat, dvec, mask, obj, sc)));
  } else {
    TB_GROUP_DISPATCH(group, (csr_forward_kernel<GG, kLossSvm><<<grid, kBlock, 0, s>>>(
                                 X, w, y, C, z, zhat, dvec, mask, obj, sc)));
  }
}

void csr_dv(const CsrView& X, int group, const double* p, const double* dvec, const uint8_t* mask,
            double* a, cudaStream_t s) {
  const int grid = forward_grid(X.rows, group);
  TB_GROUP_DISPATCH(group, (csr_dv_kernel<GG><<<grid, kBlock, 0, s>>>(X, p, dvec, mask, a)));
}

int32_t merge_num_tiles(int64_t rows, int64_t nnz) {
  return (int32_t)((rows + nnz + kTile - 1) / kTile);
}

void merge_plan_build(const CsrView& A, int32_t* tile_row, int32_t* tile_nz, int32_t* fix_chain,
                      int32_t num_tiles, cudaStream_t s) {
  merge_plan_kernel<<<(num_tiles + 1 + 255) / 256, 256, 0, s>>>(A, tile_row, tile_nz, num_tiles);
  if (num_tiles > 0)
    merge_chain_kernel<<<(num_tiles + 255) / 256, 256, 0, s>>>(A, tile_row, tile_nz, fix_chain,
                                                               num_tiles);
}

template <int UK, bool SQ>
static void launch_merge(const CsrView& A, const MergeView& P, const UView& U, const EpiView& E,
                         double* out, cudaStream_t s) {
  const int fix_grid = (P.num_tiles * 32 + kBlock - 1) / kBlock;
  switch (E.kind) {
    case EPI_VEC:
      merge_spmv_kernel<UK, SQ, EPI_VEC><<<P.num_tiles, kBlock, 0, s>>>(A, P, U, E, out);
      merge_fixup_kernel<EPI_VEC><<<fix_grid, kBlock, 0, s>>>(P, E, out);
      break;
    case EPI_CONST:
      merge_spmv_kernel<UK, SQ, EPI_CONST><<<P.num_tiles, kBlock, 0, s>>>(A, P, U, E, out);
      merge_fixup_kernel<EPI_CONST><<<fix_grid, kBlock, 0, s>>>(P, E, out);
      break;
    default:
      merge_spmv_kernel<UK, SQ, EPI_RAW><<<P.num_tiles, kBlock, 0, s>>>(A, P, U, E, out);
      merge_fixup_kernel<EPI_RAW><<<fix_grid, kBlock, 0, s>>>(P, E, out);
      break;
  }
}

void csc_spmv(const CsrView& At, const MergeView& P, const UView& U, bool squared,
              const EpiView& E, double* out, cudaStream_t s) {
  if (P.num_tiles <= 0) return;
  if (U.kind == U_VEC) {
    if (squared)
      launch_merge<U_VEC, true>(At, P, U, E, out, s);
    else
      launch_merge<U_VEC, false>(At, P, U, E, out, s);
  } else if (U.kind == U_SVM_RESID) {
    launch_merge<U_SVM_RESID, false>(At, P, U, E, out, s);
  } else {
    launch_merge<U_MASK, true>(At, P, U, E, out, s);
  }
}

int build_csc(const CsrView& X, int32_t* cptr, int32_t* ridx, double* cval, cudaStream_t s) {
  const long long nnz = X.nnz;
  int32_t *rowid = nullptr, *perm_in = nullptr, *perm_out = nullptr, *keys_out = nullptr;
  void* temp = nullptr;
  size_t temp_bytes = 0;
  int end_bit = 1;
  while (end_bit < 31 && (1LL << end_bit) < X.cols) ++end_bit;
  cudaError_t e = cudaSuccess;
  if (nnz > 0) {
    e = cudaMallocAsync(&rowid, nnz * sizeof(int32_t), s);
    if (e == cudaSuccess) e = cudaMallocAsync(&perm_in, nnz * sizeof(int32_t), s);
    if (e == cudaSuccess) e = cudaMallocAsync(&perm_out, nnz * sizeof(int32_t), s);
    if (e == cudaSuccess) e = cudaMallocAsync(&keys_out, nnz * sizeof(int32_t), s);
    if (e == cudaSuccess)
      e = cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, X.idx, keys_out, perm_in, perm_out,
                                          (int)nnz, 0, end_bit, s);
    if (e == cudaSuccess) e = cudaMallocAsync(&temp, temp_bytes > 0 ? temp_bytes : 1, s);
    if (e == cudaSuccess) {
      expand_rows_kernel<<<grid_for(X.rows * 32), 256, 0, s>>>(X, rowid);
      iota_kernel<<<grid_for(nnz), 256, 0, s>>>(perm_in, nnz);
      e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, X.idx, keys_out, perm_in, perm_out,
                                          (int)nnz, 0, end_bit, s);
    }
    if (e == cudaSuccess) {
      permute_kernel<<<grid_for(nnz), 256, 0, s>>>(perm_out, rowid, X.val, ridx, cval, nnz);
      col_ptr_kernel<<<grid_for(X.cols + 1), 256, 0, s>>>(keys_out, nnz, cptr, X.cols);
    }
  } else {
    e = cudaMemsetAsync(cptr, 0, (X.cols + 1) * sizeof(int32_t), s);
  }
  if (rowid) cudaFreeAsync(rowid, s);
  if (perm_in) cudaFreeAsync(perm_in, s);
  if (perm_out) cudaFreeAsync(perm_out, s);
  if (keys_out) cudaFreeAsync(keys_out, s);
  if (temp) cudaFreeAsync(temp, s);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

void narrow_offsets(const int64_t* in, int32_t* out, int64_t count, cudaStream_t s) {
  narrow_kernel<<<grid_for(count), 256, 0, s>>>(in, out, count);
}

}  // namespace tb
