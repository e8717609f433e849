// Hessian of the dense problems as an n x n matrix (n <= 64).
//
// svm_hessian_vec (loss.cpp:139-174) is out = v + 2C sum_{i in I} (x_i . v) x_i
// and logistic_hessian_vec (loss.cpp:82-92) out = v + C sum_i D_i (x_i . v) x_i:
// both are v + s G v with G = sum_i c_i x_i x_i^T (c = the active-set mask or D)
// fixed between commits.  For the tall-skinny dense problems (P1 / Q1: n = 40,
// l = 2.3e7 / 2.15e8) G is formed once per commit on the FP64 tensor cores,
// and every Hessian product of the truncated CG becomes a 40 x 40
// matrix-vector product inside the CG kernel (cg_small_gram_loop): the 29
// passes over X of a P1 solve become 4.  For the L2-SVM the margin passes keep
// G current themselves (dense_kernels.cu FWDG / FWDD + gram_delta_finalize
// below); gram_kernel serves LR, n > 40 and stale references.  The
// preconditioner diagonal (loss.cpp:176-188) is 1 + s G_jj.
//
// gram_kernel: CTAs stride over 128-row tiles of the column-major X, staged in
// shared memory (weights applied); the FP64 tensor cores (DMMA m8n8k4) form
// the tile's G blocks, 8 warps splitting the tile's 32 k-steps; the warps'
// partials are added in warp order, the CTA writes its n x n partial, and
// gram_finalize sums the CTA partials in index order: deterministic.  (DMMA
// fuses multiply and add: G is not a reference quantity, so the rounding costs
// no parity.)
#include "common.cuh"
#include "kernels.h"

namespace tb {

namespace {

// Tile of 128 rows staged column-major with a padded stride (132 = 4 mod 16
// doubles: the DMMA fragment loads below hit distinct banks in each half-warp).
#ifndef TB_GRAM_ROWS
#define TB_GRAM_ROWS 128
#endif
#ifndef TB_GRAM_THREADS
#define TB_GRAM_THREADS 256
#endif
#ifndef TB_GRAM_CTAS
#define TB_GRAM_CTAS 2  // resident CTAs per SM (n <= 40)
#endif
constexpr int kGramRows = TB_GRAM_ROWS;
constexpr int kGramStride = kGramRows + 4;  // = 4 (mod 16) doubles
constexpr int kGramThreads = TB_GRAM_THREADS;  // warp w takes the k-steps w, w + warps, ... of a tile

// mma.sync m8n8k4 f64 (DMMA): D(8x8) += A(8x4) B(4x8); per lane one A and one
// B element and two accumulators (row g = lane/4, columns 2t, 2t+1, t = lane%4).
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// G = T^T C T over the tiles T (rows of X) with C = diag(c): the n columns in
// NB groups of 8; for a k-step of four rows one fragment per group serves as
// B (block column) and, times the row weight c_r, as A (block row) -- NB
// loads feed NB (NB+1)/2 DMMAs.  Tiles are double-buffered with cp.async: the
// next tile's rows and weights are in flight while this one is multiplied.
template <int NB, bool MASK>
__global__ void __launch_bounds__(kGramThreads, NB <= 5 ? TB_GRAM_CTAS : 1) gram_kernel(long long l, int n, long long ld,
                                                              const double* __restrict__ X,
                                                              const uint8_t* __restrict__ mask,
                                                              const double* __restrict__ dvec,
                                                              double* __restrict__ partials,
                                                              const int* __restrict__ stale) {
  pdl_wait();
  pdl_trigger();
  if (stale && *stale == 0) return;  // G of this iterate is current
  constexpr int NC = NB * 8;
  constexpr int NP = NB * (NB + 1) / 2;
  constexpr int TILE = NC * kGramStride;  // doubles per staged tile
  extern __shared__ __align__(16) double gs[];
  // buffer b: the tile at gs + b * TILE, its row weights (MASK: 128 bytes of the
  // 0/1 mask, else 128 doubles of D) at gs + 2 * TILE + b * kGramRows
  auto Tb = [&](int b) { return gs + b * TILE; };
  auto Wb = [&](int b) { return reinterpret_cast<unsigned char*>(gs + 2 * TILE + b * kGramRows); };
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  double acc[NP][2];
#pragma unroll
  for (int p = 0; p < NP; ++p) acc[p][0] = acc[p][1] = 0.0;
  // columns past n read column 0 (their rows of G are never written out)
  auto stage = [&](long long tile, int b) {
    const long long r0 = tile * kGramRows;
    for (int e = tid; e < NC * (kGramRows / 2); e += kGramThreads) {
      const int j = e / (kGramRows / 2), r = 2 * (e % (kGramRows / 2));
      cp16(Tb(b) + j * kGramStride + r, X + (long long)(j < n ? j : 0) * ld + r0 + r);
    }
    if (MASK) {
      if (tid < kGramRows / 16) cp16(Wb(b) + 16 * tid, mask + r0 + 16 * tid);
    } else {
      if (tid < kGramRows / 2) cp16(Wb(b) + 16 * tid, dvec + r0 + 2 * tid);
    }
  };
  // X, mask and D are padded with zeros to whole 256-row tiles, so the
  // 128-row tiles need no row guard
  const long long ntiles = (l + kGramRows - 1) / kGramRows;
  long long tile = blockIdx.x;
  if (tile < ntiles) stage(tile, 0);
  cp_commit();
  for (int it = 0; tile < ntiles; tile += gridDim.x, ++it) {
    const int b = it & 1;
    if (tile + gridDim.x < ntiles) stage(tile + gridDim.x, b ^ 1);
    cp_commit();
    cp_wait<1>();     // this tile's copies (this thread's) have landed
    __syncthreads();  // ... and every thread's
    const double* T = Tb(b);
    for (int ks = warp; ks < kGramRows / 4; ks += kGramThreads / 32) {
      const int rr = ks * 4 + t;
      const double c = MASK ? (Wb(b)[rr] ? 1.0 : 0.0) : reinterpret_cast<const double*>(Wb(b))[rr];
      double fb[NB], fa[NB];
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        fb[q] = T[(q * 8 + g) * kGramStride + rr];
        fa[q] = c * fb[q];
      }
      int p = 0;
#pragma unroll
      for (int c1 = 0; c1 < NB; ++c1)
#pragma unroll
        for (int c2 = c1; c2 < NB; ++c2) dmma(acc[p++], fa[c1], fb[c2]);
    }
    __syncthreads();  // the buffer is restaged two tiles later
  }
  cp_wait<0>();
  // the 8 warps' partial blocks, added in warp order
  __syncthreads();
  double* red = gs;  // [NP][64]
  for (int w = 0; w < kGramThreads / 32; ++w) {
    if (warp == w) {
#pragma unroll
      for (int p = 0; p < NP; ++p)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int idx = p * 64 + g * 8 + 2 * t + h;
          red[idx] = w == 0 ? acc[p][h] : red[idx] + acc[p][h];
        }
    }
    __syncthreads();
  }
  double* out = partials + (size_t)blockIdx.x * n * n;
  for (int e = tid; e < NP * 64; e += kGramThreads) {
    const int p = e / 64, gi = (e % 64) / 8, ci = e % 8;
    int c1 = 0, rem = p;
    while (rem >= NB - c1) {
      rem -= NB - c1;
      ++c1;
    }
    const int c2 = c1 + rem;
    const int j = c1 * 8 + gi, k = c2 * 8 + ci;
    if (j < n && k < n) {
      out[j * n + k] = red[e];
      if (c1 != c2) out[k * n + j] = red[e];  // the lower triangle mirrors the upper
    }
  }
}

// G = sum of the per-CTA partials: one warp per element, its lanes striding
// over the partials in index order, then the fixed butterfly (deterministic).
// flags (nullable; gram_flags layout): every CTA reads flags[0] first and
// returns when G is current; the last CTA to finish clears it (a ticket in
// flags[2]), so no CTA can see the flag cleared before reading it.
__global__ void __launch_bounds__(256) gram_finalize_kernel(int n, const double* __restrict__ partials,
                                                           int nparts, double* __restrict__ G, int* flags) {
  if (flags && flags[0] == 0) return;
  const int nn = n * n;
  const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (e < nn) {
    double s = 0.0;
    for (int b = lane; b < nparts; b += 32) s += partials[(size_t)b * nn + e];
    s = warp_sum(s);
    if (lane == 0) G[e] = s;
  }
  if (flags) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(flags + 2, 1) == (int)gridDim.x - 1) {
        flags[0] = 0;  // G matches the slot's mask
        flags[1] = 0;  // ... and was formed from scratch
        flags[2] = 0;
      }
    }
  }
}

// G_out = G_ref + sum of the per-CTA Delta partials of the margin pass
// (dense_pass PM_FWDD) when the reference can be updated; otherwise (the pass
// skipped the Delta) G_out is flagged stale.
__global__ void __launch_bounds__(256) gram_delta_finalize_kernel(int n, const double* __restrict__ parts,
                                                                 int nparts, const double* __restrict__ Gref,
                                                                 const int* __restrict__ ref_flags,
                                                                 double* __restrict__ Gout, int* out_flags) {
  pdl_wait();
  pdl_trigger();
  const bool ok = !gram_ref_is_empty(ref_flags);
  const int nn = n * n;
  const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (ok && e < nn) {
    double s = 0.0;
    for (int b = lane; b < nparts; b += 32) s += parts[(size_t)b * nn + e];
    s = warp_sum(s);
    if (lane == 0) Gout[e] = Gref[e] + s;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out_flags[0] = ok ? 0 : 1;
    out_flags[1] = ok ? ref_flags[1] + 1 : 0;
  }
}

int finalize_grid(int64_t n) { return (int)((n * n * 32 + 255) / 256); }

__global__ void gram_hv_kernel(int n, const double* __restrict__ G, const double* __restrict__ v,
                               double scale, double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < n; ++k) s += G[j * n + k] * v[k];
    out[j] = v[j] + scale * s;
  }
}

__global__ void gram_precond_kernel(int n, const double* __restrict__ G, double scale,
                                    double* __restrict__ M) {
  for (int j = threadIdx.x; j < n; j += blockDim.x) M[j] = 1.0 + scale * G[j * n + j];
}

}  // namespace

void gram_finalize(int64_t n, const double* partials, int nparts, double* G, cudaStream_t s, int* flags) {
  gram_finalize_kernel<<<finalize_grid(n), 256, 0, s>>>((int)n, partials, nparts, G, flags);
  TB_LAUNCH_CHECK();
}

void gram_delta_finalize(int64_t n, const double* parts, int nparts, const double* Gref, const int* ref_flags,
                         double* Gout, int* out_flags, cudaStream_t s) {
  launch_pdl(gram_delta_finalize_kernel, dim3(finalize_grid(n)), dim3(256), 0, s, (int)n, parts, nparts, Gref,
             ref_flags, Gout, out_flags);
}

void gram_hv(int64_t n, const double* G, const double* v, double scale, double* out, cudaStream_t s) {
  launch_pdl(gram_hv_kernel, dim3(1), dim3(64), 0, s, (int)n, G, v, scale, out);
}

void gram_precond(int64_t n, const double* G, double scale, double* M, cudaStream_t s) {
  gram_precond_kernel<<<1, 64, 0, s>>>((int)n, G, scale, M);
  TB_LAUNCH_CHECK();
}

int gram_grid(int64_t l, int64_t n) {
  const int64_t tiles = (l + kGramRows - 1) / kGramRows;
  int64_t g = (int64_t)device_sm_count() * (n <= 40 ? TB_GRAM_CTAS : 1);  // resident CTAs per SM
  if (g > tiles) g = tiles;
  return (int)(g > 0 ? g : 1);
}

namespace {
template <int NB, bool W>
void launch_gram(int64_t l, int64_t n, int64_t ld, const double* X, const uint8_t* mask,
                 const double* dvec, double* partials, const int* stale, int grid, cudaStream_t s) {
  const size_t tile = ((size_t)2 * NB * 8 * kGramStride + 2 * kGramRows) * sizeof(double);
  const size_t red = (size_t)(NB * (NB + 1) / 2) * 64 * sizeof(double);
  const size_t bytes = tile > red ? tile : red;
  ensure_max_dynamic_smem((const void*)gram_kernel<NB, W>, (int)bytes);
  launch_pdl(gram_kernel<NB, W>, dim3(grid), dim3(kGramThreads), bytes, s, (long long)l, (int)n,
             (long long)ld, X, mask, dvec, partials, stale);
}
template <bool W>
void dispatch_gram(int64_t l, int64_t n, int64_t ld, const double* X, const uint8_t* mask,
                   const double* dvec, double* partials, const int* stale, int grid, cudaStream_t s) {
  switch ((n + 7) / 8) {
    case 1: launch_gram<1, W>(l, n, ld, X, mask, dvec, partials, stale, grid, s); break;
    case 2: launch_gram<2, W>(l, n, ld, X, mask, dvec, partials, stale, grid, s); break;
    case 3: launch_gram<3, W>(l, n, ld, X, mask, dvec, partials, stale, grid, s); break;
    case 4: launch_gram<4, W>(l, n, ld, X, mask, dvec, partials, stale, grid, s); break;
    case 5: launch_gram<5, W>(l, n, ld, X, mask, dvec, partials, stale, grid, s); break;
    case 6: launch_gram<6, W>(l, n, ld, X, mask, dvec, partials, stale, grid, s); break;
    case 7: launch_gram<7, W>(l, n, ld, X, mask, dvec, partials, stale, grid, s); break;
    default: launch_gram<8, W>(l, n, ld, X, mask, dvec, partials, stale, grid, s); break;
  }
}
}  // namespace

void dense_gram(int64_t l, int64_t n, int64_t ld, const double* X, const uint8_t* mask,
                const double* dvec, double* partials, double* G, cudaStream_t s, int* stale) {
  const int grid = gram_grid(l, n);
  if (mask)
    dispatch_gram<true>(l, n, ld, X, mask, dvec, partials, stale, grid, s);
  else
    dispatch_gram<false>(l, n, ld, X, mask, dvec, partials, stale, grid, s);
  gram_finalize_kernel<<<finalize_grid(n), 256, 0, s>>>((int)n, partials, grid, G, stale);
  TB_LAUNCH_CHECK();
}

}  // namespace tb
