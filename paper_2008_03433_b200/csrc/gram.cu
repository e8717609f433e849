// Hessian of the dense problems as an n x n matrix (n <= 64).
//
// svm_hessian_vec (loss.cpp:139-174) is out = v + 2C sum_{i in I} (x_i . v) x_i
// and logistic_hessian_vec (loss.cpp:82-92) out = v + C sum_i D_i (x_i . v) x_i:
// both are v + s G v with G = sum_i c_i x_i x_i^T (c = the active-set mask or D)
// fixed between commits.  For the tall-skinny dense problems (P1 / Q1: n = 40,
// l = 2.3e7 / 2.15e8) G is formed once per commit -- one pass over X, on the
// FP64 FMA pipes -- and every Hessian product of the truncated CG becomes a
// 40 x 40 matrix-vector product inside the CG step kernel: the 25 passes over
// X of a P1 solve become 4.  The preconditioner diagonal (loss.cpp:176-188) is
// 1 + s G_jj.
//
// gram_kernel: CTAs stride over 128-row tiles of the column-major X.  A tile
// and its row weights are staged in shared memory; thread (b, ph) owns the 4x4
// block b of the upper triangle (NB (NB+1) / 2 blocks, NB = ceil(n/4)) over the
// rows r = ph (mod P) of the tile, 16 register accumulators, 8 shared loads per
// 16 FMAs (explicit __fma_rn: the build's -fmad=false would split them; G is not
// a reference quantity, so the fused rounding costs no parity).  The P row phases are combined in a fixed order, the CTA writes its
// full n x n partial (mirrored), and gram_finalize sums the CTA partials in
// index order: deterministic.
#include "common.cuh"
#include "kernels.h"

namespace tb {

namespace {

constexpr int kGramRows = 128;
constexpr int kGramStride = kGramRows + 1;  // padded columns: spreads the blocks over the banks
constexpr int kGramThreads = 256;

__global__ void __launch_bounds__(kGramThreads) gram_kernel(long long l, int n, long long ld,
                                                           const double* __restrict__ X,
                                                           const uint8_t* __restrict__ mask,
                                                           const double* __restrict__ dvec,
                                                           double* __restrict__ partials) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) double gs[];  // [NB*4][kGramStride] tile, then [kGramRows] weights
  const int NB = (n + 3) >> 2;
  const int NC = NB * 4;
  double* cs = gs + (size_t)NC * kGramStride;
  const int nblk = NB * (NB + 1) / 2;
  const int P = kGramThreads / nblk;  // row phases per block (>= 1 for n <= 64)
  const int tid = threadIdx.x;
  const bool worker = tid < nblk * P;
  const int b = worker ? tid / P : 0, ph = worker ? tid % P : 0;
  // block b -> (bj, bk), bj <= bk, row-major over the upper triangle
  int bj = 0, rem = b;
  while (rem >= NB - bj) {
    rem -= NB - bj;
    ++bj;
  }
  const int bk = bj + rem;
  double acc[4][4];
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[p][q] = 0.0;

  const long long ntiles = (l + kGramRows - 1) / kGramRows;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const long long r0 = t * kGramRows;
    __syncthreads();  // the previous tile is consumed
    for (int e = tid; e < NC * kGramRows; e += kGramThreads) {
      const int j = e / kGramRows, r = e % kGramRows;
      const long long i = r0 + r;
      gs[j * kGramStride + r] = (j < n && i < l) ? __ldg(X + (long long)j * ld + i) : 0.0;
    }
    for (int r = tid; r < kGramRows; r += kGramThreads) {
      const long long i = r0 + r;
      cs[r] = i < l ? (mask ? (mask[i] ? 1.0 : 0.0) : dvec[i]) : 0.0;
    }
    __syncthreads();
    if (worker) {
      const double* A = gs + (size_t)(4 * bj) * kGramStride;
      const double* B = gs + (size_t)(4 * bk) * kGramStride;
      for (int r = ph; r < kGramRows; r += P) {
        const double c = cs[r];
        double a[4], bb[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) a[p] = c * A[p * kGramStride + r];
#pragma unroll
        for (int q = 0; q < 4; ++q) bb[q] = B[q * kGramStride + r];
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[p][q] = __fma_rn(a[p], bb[q], acc[p][q]);  // (no -fmad here)
      }
    }
  }
  // phases of each block, in order (reuse the tile's shared memory)
  __syncthreads();
  double* red = gs;  // [nblk*P][16]
  if (worker)
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int q = 0; q < 4; ++q) red[(size_t)tid * 16 + p * 4 + q] = acc[p][q];
  __syncthreads();
  double* out = partials + (size_t)blockIdx.x * n * n;
  for (int e = tid; e < nblk * 16; e += kGramThreads) {
    const int bb = e / 16, pq = e % 16, p = pq / 4, q = pq % 4;
    double s = 0.0;
    for (int h = 0; h < P; ++h) s += red[(size_t)(bb * P + h) * 16 + pq];
    int jj = 0, rr = bb;
    while (rr >= NB - jj) {
      rr -= NB - jj;
      ++jj;
    }
    const int kk = jj + rr;
    const int j = 4 * jj + p, k = 4 * kk + q;
    if (j < n && k < n) {
      out[j * n + k] = s;
      out[k * n + j] = s;  // diagonal blocks write each entry twice, with the same bits
    }
  }
}

__global__ void gram_finalize_kernel(int n, const double* __restrict__ partials, int nparts,
                                     double* __restrict__ G) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nparts; ++b) s += partials[(size_t)b * n * n + e];
    G[e] = s;
  }
}

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

void gram_hv(int64_t n, const double* G, const double* v, double scale, double* out, cudaStream_t s) {
  launch_pdl(gram_hv_kernel, dim3(1), dim3(64), 0, s, (int)n, G, v, scale, out);
}

void gram_precond(int64_t n, const double* G, double scale, double* M, cudaStream_t s) {
  gram_precond_kernel<<<1, 64, 0, s>>>((int)n, G, scale, M);
  TB_LAUNCH_CHECK();
}

int gram_grid(int64_t l) {
  const int64_t tiles = (l + kGramRows - 1) / kGramRows;
  int64_t g = (int64_t)device_sm_count() * 3;
  if (g > tiles) g = tiles;
  return (int)(g > 0 ? g : 1);
}

void dense_gram(int64_t l, int64_t n, int64_t ld, const double* X, const uint8_t* mask,
                const double* dvec, double* partials, double* G, cudaStream_t s) {
  const int NB = (int)((n + 3) / 4);
  const size_t smem = ((size_t)NB * 4 * kGramStride + kGramRows) * sizeof(double);
  const size_t red = (size_t)kGramThreads * 16 * sizeof(double);
  const size_t bytes = smem > red ? smem : red;
  ensure_max_dynamic_smem((const void*)gram_kernel, (int)bytes);
  const int grid = gram_grid(l);
  launch_pdl(gram_kernel, dim3(grid), dim3(kGramThreads), bytes, s, (long long)l, (int)n, (long long)ld,
             X, mask, dvec, partials);
  gram_finalize_kernel<<<(int)((n * n + 255) / 256), 256, 0, s>>>((int)n, partials, grid, G);
  TB_LAUNCH_CHECK();
}

}  // namespace tb
