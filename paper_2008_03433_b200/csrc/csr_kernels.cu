// Sparse kernels of the TRON hot path on sm_100a (FP64, HBM-bound).
//
//  * csr_forward / csr_dv: sub-warp vector-CSR row products over X
//    (matvec, linalg.cpp:154-162) fused with the per-instance epilogues of
//    logistic_fused_pass (loss.cpp:35-58), svm_fused_pass (loss.cpp:94-122)
//    and the D-scaling of logistic_hessian_vec (loss.cpp:82-92).
//  * build_csc: the device-built CSC copy (stable in row order) that
//    csc_seg.cu streams for every X^T u.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "rowdot.cuh"

namespace tb {

namespace {

constexpr int kBlock = 256;
constexpr int kStagedBlock = 512;                  // one 16-warp block per SM
constexpr int kHotMax = 200 * 1024 / 8;            // staged prefix entries (200 KB)
constexpr long long kStageMinNnz = 1 << 20;        // stage only for big passes

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
// Lane `sub` of the group sums entries sub, sub+G, ... of the row; eight
// entries are loaded before any gathered v_j is consumed (latency hiding).
template <int G, bool STAGED>
__device__ __forceinline__ double row_dot_sub(const CsrView& X, long long row, int sub,
                                              const double* __restrict__ v, const double* sv,
                                              int hot) {
  // entries in flight per lane: one 16-warp block per SM when staged, so each
  // lane keeps twice as many loads in flight
  constexpr int U = STAGED ? 16 : 8;
  const int beg = X.ptr[row], end = X.ptr[row + 1];
  double s = 0.0;
  for (int k0 = beg + sub; k0 < end; k0 += U * G) {
    int c[U];
    double a[U];
#pragma unroll
    for (int m = 0; m < U; ++m) {
      const int k = k0 + m * G;
      c[m] = k < end ? ldg_stream(X.idx + k) : 0;
      a[m] = k < end ? ldg_stream(X.val + k) : 0.0;
    }
    double b[U];
#pragma unroll
    for (int m = 0; m < U; ++m) {
      if (STAGED)
        b[m] = (k0 + m * G < end) ? (c[m] < hot ? sv[c[m]] : __ldg(v + c[m])) : 0.0;
      else
        b[m] = (k0 + m * G < end) ? __ldg(v + c[m]) : 0.0;
    }
#pragma unroll
    for (int m = 0; m < U; ++m)
      if (k0 + m * G < end) s += a[m] * b[m];
  }
  return s;
}

// Hot-prefix staging: v[0, hot) is copied to shared memory once per block so
// that gathers of popular features are LDS, not L1 wavefronts (the limit of
// a gather-bound SpMV).  SYNTH-v1 draws columns Zipf(1) by index, so the
// first 25.6k columns carry ~70% of news20-shaped nonzeros.
template <bool STAGED, int BLK>
__device__ __forceinline__ void stage_prefix(const double* __restrict__ v, double* sv, int hot) {
  if (STAGED) bulk_stage_f64(sv, v, hot);
}

template <int G, int LOSS, bool STAGED>
__global__ void __launch_bounds__(STAGED ? kStagedBlock : kBlock)
    csr_forward_kernel(CsrView X, int hot, const double* __restrict__ w,
                                                            const double* __restrict__ y, double C,
                                                            const double* zin, double* z,
                                                            double* __restrict__ zhat,
                                                            double* __restrict__ dvec,
                                                            uint8_t* __restrict__ mask,
                                                            ObjScalars* obj, Scratch sc) {
  pdl_wait();
  pdl_trigger();
  constexpr int BLK = STAGED ? kStagedBlock : kBlock;
  constexpr int RPW = kWarp / G;  // rows per warp
  __shared__ double sh[BLK / kWarp + 1];
  extern __shared__ double sv[];
  stage_prefix<STAGED, BLK>(w, sv, hot);
  const int lane = threadIdx.x & 31;
  const int sub = lane % G;
  const long long gwarp = (blockIdx.x * (long long)BLK + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * BLK) >> 5;
  double term_acc = 0.0, cnt_acc = 0.0;
  for (long long r0 = gwarp * RPW; r0 < X.rows; r0 += nwarps * RPW) {
    const long long row = r0 + lane / G;
    double s = 0.0;
    if (row < X.rows) {
      s = STAGED ? row_dot_sub<G, STAGED>(X, row, sub, w, sv, hot) : row_dot_vec<G, false>(X, row, sub, w);
    }
    s = group_sum<G>(s);
    if (sub == 0 && row < X.rows) {
      const double yi = y[row];
      if (zin) s = zin[row] + s;  // earlier column panels
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
  const double bt = block_sum<BLK>(term_acc, sh, true);
  const double bc = block_sum<BLK>(cnt_acc, sh, true);
  if (threadIdx.x == 0) {
    sc.partials[2 * blockIdx.x] = bt;
    sc.partials[2 * blockIdx.x + 1] = bc;
  }
  if (last_block_arrive(sc.tickets + T_FUN)) {
    const double tot = reduce_partials<BLK>(sc.partials, gridDim.x, 2, 0, sh);
    const double cnt = reduce_partials<BLK>(sc.partials, gridDim.x, 2, 1, sh);
    if (threadIdx.x == 0) {
      obj->f = 0.5 * obj->ww + C * tot;  // loss.cpp:57 / :121
      obj->nact = (long long)cnt;
      obj->red[0] = tot;
      obj->red[1] = cnt;
    }
  }
}

template <int G, bool STAGED>
__global__ void __launch_bounds__(STAGED ? kStagedBlock : kBlock)
    csr_dv_kernel(CsrView X, int hot, const double* __restrict__ p,
                                                       const double* __restrict__ dvec,
                                                       const uint8_t* __restrict__ mask,
                                                       const double* ain, double* a, int final) {
  pdl_wait();
  pdl_trigger();
  constexpr int BLK = STAGED ? kStagedBlock : kBlock;
  constexpr int RPW = kWarp / G;
  extern __shared__ double sv[];
  stage_prefix<STAGED, BLK>(p, sv, hot);
  const int lane = threadIdx.x & 31;
  const int sub = lane % G;
  const long long gwarp = (blockIdx.x * (long long)BLK + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * BLK) >> 5;
  for (long long r0 = gwarp * RPW; r0 < X.rows; r0 += nwarps * RPW) {
    const long long row = r0 + lane / G;
    bool active = row < X.rows;
    if (active && mask) active = mask[row] != 0;
    double s = 0.0;
    if (active) {
      s = STAGED ? row_dot_sub<G, STAGED>(X, row, sub, p, sv, hot) : row_dot_vec<G, false>(X, row, sub, p);
    }
    s = group_sum<G>(s);
    if (sub == 0 && row < X.rows) {
      if (ain) s = ain[row] + s;  // earlier column panels
      // loss.cpp:86-89: a0_i *= dvec_i; svm indirect skips inactive rows.
      // (no mask and no dvec: the gathered rows X_I, every row active)
      a[row] = !final ? s : (mask ? (active ? s : 0.0) : (dvec ? s * dvec[row] : s));
    }
  }
}

// Rows are grid-strided, so the grid is capped at one wave of resident CTAs
// of this kernel (a partial second wave would be a tail: measured on N1, the
// forward kernel at 40 registers holds 6 CTAs per SM, not 8).
template <class Kernel>
int forward_grid(Kernel k, int64_t rows, int group) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kBlock, 0);
  if (per_sm < 1) per_sm = 1;
  const int64_t rows_per_block = kBlock / group;
  int64_t want = (rows + rows_per_block - 1) / rows_per_block;
  const int64_t cap = (int64_t)device_sm_count() * per_sm;
  if (want > cap) want = cap;
  if (want < 1) want = 1;
  return (int)want;
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
    if (ridx) ridx[i] = rowid[k];
    if (cval) cval[i] = val[k];
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

// Input screening on the device (the host re-checks the first offending row
// sequentially to report the reference's exact error): one warp per row,
// valid iff the columns ascend strictly within [0, n).
__global__ void csr_screen_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                  long long rows, long long n, unsigned long long* first_bad) {
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = gw; r < rows; r += nw) {
    const int b = ptr[r], e = ptr[r + 1];
    bool bad = false;
    for (int k = b + lane; k < e; k += 32) {
      const int c = idx[k];
      bad |= c < 0 || c >= n || (k > b && c <= idx[k - 1]);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(first_bad, (unsigned long long)r);
  }
}

__global__ void labels_screen_kernel(const double* __restrict__ y, long long l,
                                     unsigned long long* first_bad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < l;
       i += (long long)gridDim.x * blockDim.x)
    if (y[i] != 1.0 && y[i] != -1.0) atomicMin(first_bad, (unsigned long long)i);
}

int grid_for(long long n, int block = 256) {
  long long g = (n + block - 1) / block;
  long long cap = (long long)device_sm_count() * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TRON_B200_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

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
  static const int forced = [] {  // TRON_B200_CSR_G=2/4/8/16/32: A/B of the lanes per row
    const char* e = std::getenv("TRON_B200_CSR_G");
    return e ? std::atoi(e) : 0;
  }();
  if (forced == 2 || forced == 4 || forced == 8 || forced == 16 || forced == 32) return forced;
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

template <class K>
static void set_smem(K kernel) {
  ensure_max_dynamic_smem((const void*)kernel, kHotMax * 8);
}

// Opt-in (TRON_B200_STAGE=1): measured slower on N1 (occupancy drops to one
// 16-warp block per SM while the kernel is bound by streaming-load latency).
static bool stage_enabled() {
  static const int on = [] {
    const char* e = std::getenv("TRON_B200_STAGE");
    return (e && e[0] == '1') ? 1 : 0;
  }();
  return on != 0;
}
static bool stage_rows(const CsrView& X) {
  return stage_enabled() && X.nnz >= kStageMinNnz && X.cols > 4096;
}

void csr_forward(const CsrView& X, int group, int loss, const double* w, const double* y, double C,
                 double* z, double* zhat, double* dvec, uint8_t* mask, ObjScalars* obj,
                 Scratch sc, cudaStream_t s, const double* zin) {
  if (stage_rows(X) && !zin && !X.rbeg) {
    const int hot = (int)(X.cols < kHotMax ? X.cols : kHotMax);
    const int grid = device_sm_count();
    const size_t smem = (size_t)hot * 8;
    if (loss == kLossLogistic) {
      TB_GROUP_DISPATCH(group, {
        auto k = csr_forward_kernel<GG, kLossLogistic, true>;
        set_smem(k);
        launch_pdl(k, dim3(grid), dim3(kStagedBlock), smem, s, X, hot, w, y, C, zin, z, zhat, dvec,
                   mask, obj, sc);
      });
    } else {
      TB_GROUP_DISPATCH(group, {
        auto k = csr_forward_kernel<GG, kLossSvm, true>;
        set_smem(k);
        launch_pdl(k, dim3(grid), dim3(kStagedBlock), smem, s, X, hot, w, y, C, zin, z, zhat, dvec,
                   mask, obj, sc);
      });
    }
    return;
  }
  if (loss == kLossLogistic) {
    TB_GROUP_DISPATCH(group, {
      auto k = csr_forward_kernel<GG, kLossLogistic, false>;
      launch_pdl(k, dim3(forward_grid(k, X.rows, group)), dim3(kBlock), 0, s, X, 0, w, y, C, zin, z,
                 zhat, dvec, mask, obj, sc);
    });
  } else {
    TB_GROUP_DISPATCH(group, {
      auto k = csr_forward_kernel<GG, kLossSvm, false>;
      launch_pdl(k, dim3(forward_grid(k, X.rows, group)), dim3(kBlock), 0, s, X, 0, w, y, C, zin, z,
                 zhat, dvec, mask, obj, sc);
    });
  }
}

void csr_dv(const CsrView& X, int group, const double* p, const double* dvec, const uint8_t* mask,
            double* a, cudaStream_t s, const double* ain, bool final) {
  const int fin = final ? 1 : 0;
  if (stage_rows(X) && !ain && final && !X.rbeg) {
    const int hot = (int)(X.cols < kHotMax ? X.cols : kHotMax);
    TB_GROUP_DISPATCH(group, {
      auto k = csr_dv_kernel<GG, true>;
      set_smem(k);
      launch_pdl(k, dim3(device_sm_count()), dim3(kStagedBlock), (size_t)hot * 8, s, X, hot, p, dvec,
                 mask, ain, a, fin);
    });
    return;
  }
  TB_GROUP_DISPATCH(group, {
    auto k = csr_dv_kernel<GG, false>;
    launch_pdl(k, dim3(forward_grid(k, X.rows, group)), dim3(kBlock), 0, s, X, 0, p, dvec, mask, ain,
               a, fin);
  });
}

namespace {
constexpr int kMaxPanelBounds = 8;
struct PanelBounds {
  int32_t bound[kMaxPanelBounds];
  int32_t* split[kMaxPanelBounds];
  int n;
};
// split[k][i] = lower_bound of bound[k] in row i's (ascending) columns
__global__ void panel_split_kernel(CsrView X, PanelBounds B) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < X.rows;
       i += (long long)gridDim.x * blockDim.x) {
    const int beg = X.ptr[i], end = X.ptr[i + 1];
    for (int k = 0; k < B.n; ++k) {
      int lo = beg, hi = end;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (X.idx[mid] < B.bound[k])
          lo = mid + 1;
        else
          hi = mid;
      }
      B.split[k][i] = lo;
    }
  }
}
}  // namespace

static __global__ void panel_count_kernel(CsrView X, PanelBounds B, unsigned long long* counts) {
  unsigned long long local[kMaxPanelBounds + 1] = {};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < X.rows;
       i += (long long)gridDim.x * blockDim.x) {
    int lo = X.ptr[i];
    for (int k = 0; k <= B.n; ++k) {
      const int hi = k < B.n ? B.split[k][i] : X.ptr[i + 1];
      local[k] += (unsigned long long)(hi - lo);
      lo = hi;
    }
  }
  for (int k = 0; k <= B.n; ++k) atomicAdd(counts + k, local[k]);
}

int csr_panel_splits(const CsrView& X, const int32_t* bounds, int nbounds, int32_t* const* split,
                     unsigned long long* counts, cudaStream_t s) {
  PanelBounds B{};
  B.n = nbounds < kMaxPanelBounds ? nbounds : kMaxPanelBounds;
  for (int k = 0; k < B.n; ++k) {
    B.bound[k] = bounds[k];
    B.split[k] = split[k];
  }
  unsigned long long* dc = nullptr;
  cudaError_t e = cudaMallocAsync(&dc, (kMaxPanelBounds + 1) * sizeof(unsigned long long), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(dc, 0, (kMaxPanelBounds + 1) * sizeof(unsigned long long), s);
  if (e == cudaSuccess && X.rows > 0) {
    const int grid = (int)std::min<long long>((X.rows + 255) / 256, 148LL * 16);
    panel_split_kernel<<<grid, 256, 0, s>>>(X, B);
    panel_count_kernel<<<grid, 256, 0, s>>>(X, B, dc);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(counts, dc, (B.n + 1) * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (dc) cudaFreeAsync(dc, s);
  return e == cudaSuccess ? 0 : (int)e;
}

// Structure of the CSC copy: a stable radix sort of the column indices (row
// order kept inside a column), the row ids and the column pointers.  Needs
// only X.ptr / X.idx, so the values can still be in flight on another stream;
// *perm (nnz entries, freed by build_csc_values) maps CSC slots to CSR entries.
int build_csc_structure(const CsrView& X, int32_t* cptr, int32_t* ridx, int32_t** perm,
                        cudaStream_t s) {
  const long long nnz = X.nnz;
  int32_t *rowid = nullptr, *perm_in = nullptr, *perm_out = nullptr, *keys_out = nullptr;
  void* temp = nullptr;
  size_t temp_bytes = 0;
  int end_bit = 1;
  while (end_bit < 31 && (1LL << end_bit) < X.cols) ++end_bit;
  cudaError_t e = cudaSuccess;
  *perm = nullptr;
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
      permute_kernel<<<grid_for(nnz), 256, 0, s>>>(perm_out, rowid, nullptr, ridx, nullptr, nnz);
      col_ptr_kernel<<<grid_for(X.cols + 1), 256, 0, s>>>(keys_out, nnz, cptr, X.cols);
    }
  } else {
    e = cudaMemsetAsync(cptr, 0, (X.cols + 1) * sizeof(int32_t), s);
  }
  if (rowid) cudaFreeAsync(rowid, s);
  if (perm_in) cudaFreeAsync(perm_in, s);
  if (keys_out) cudaFreeAsync(keys_out, s);
  if (temp) cudaFreeAsync(temp, s);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess)
    *perm = perm_out;
  else if (perm_out)
    cudaFreeAsync(perm_out, s);
  return e == cudaSuccess ? 0 : (int)e;
}

// ---------------------------------------------------------------------------
// gather_rows on a CSR (linalg.cpp:197-229): X_I = rows idx[0..nI) of X, in
// order.  Offsets: row lengths then an exclusive scan; entries: one warp per
// gathered row copies its indices and values (coalesced).
namespace {
__global__ void gather_len_kernel(CsrView X, const int32_t* __restrict__ idx, long long nI,
                                  int32_t* __restrict__ gptr) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k <= nI;
       k += (long long)gridDim.x * blockDim.x)
    gptr[k] = k < nI ? X.ptr[idx[k] + 1] - X.ptr[idx[k]] : 0;
}
__global__ void gather_rows_kernel(CsrView X, const int32_t* __restrict__ idx, long long nI,
                                   const int32_t* __restrict__ gptr, int32_t* __restrict__ gidx,
                                   double* __restrict__ gval) {
  const int lane = threadIdx.x & 31;
  const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long k = w0; k < nI; k += nw) {
    const int src = X.ptr[idx[k]], len = X.ptr[idx[k] + 1] - src, dst = gptr[k];
    for (int t = lane; t < len; t += 32) {
      gidx[dst + t] = X.idx[src + t];
      gval[dst + t] = X.val[src + t];
    }
  }
}
}  // namespace

int csr_gather_offsets(const CsrView& X, const int32_t* idx, int64_t nI, int32_t* gptr,
                       long long* nnz_out, cudaStream_t s) {
  gather_len_kernel<<<grid_for(nI + 1), 256, 0, s>>>(X, idx, nI, gptr);
  size_t temp_bytes = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, gptr, gptr, (int)(nI + 1), s);
  void* temp = nullptr;
  if (e == cudaSuccess) e = cudaMallocAsync(&temp, temp_bytes > 0 ? temp_bytes : 1, s);
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, gptr, gptr, (int)(nI + 1), s);
  if (temp) cudaFreeAsync(temp, s);
  int32_t last = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&last, gptr + nI, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess) e = cudaGetLastError();
  *nnz_out = last;
  return e == cudaSuccess ? 0 : (int)e;
}

void csr_gather_rows(const CsrView& X, const int32_t* idx, int64_t nI, const int32_t* gptr,
                     int32_t* gidx, double* gval, cudaStream_t s) {
  if (nI == 0) return;
  gather_rows_kernel<<<grid_for(nI * 32), 256, 0, s>>>(X, idx, nI, gptr, gidx, gval);
  TB_LAUNCH_CHECK();
}

// Values of the CSC copy: cval[i] = val[perm[i]]; frees perm.
int build_csc_values(int32_t* perm, const double* val, double* cval, int64_t nnz, cudaStream_t s) {
  if (nnz > 0 && perm)
    permute_kernel<<<grid_for(nnz), 256, 0, s>>>(perm, nullptr, val, nullptr, cval, nnz);
  if (perm) cudaFreeAsync(perm, s);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

void screen_inputs(const int32_t* ptr, const int32_t* idx, int64_t rows, int64_t n,
                   const double* y, int64_t l, unsigned long long* first_bad2, cudaStream_t s) {
  cudaMemsetAsync(first_bad2, 0xff, 2 * sizeof(unsigned long long), s);
  if (ptr && rows > 0)
    csr_screen_kernel<<<grid_for(rows * 32), 256, 0, s>>>(ptr, idx, rows, n, first_bad2);
  if (l > 0) labels_screen_kernel<<<grid_for(l), 256, 0, s>>>(y, l, first_bad2 + 1);
  TB_LAUNCH_CHECK();
}

void narrow_offsets(const int64_t* in, int32_t* out, int64_t count, cudaStream_t s) {
  narrow_kernel<<<grid_for(count), 256, 0, s>>>(in, out, count);
  TB_LAUNCH_CHECK();
}

}  // namespace tb
