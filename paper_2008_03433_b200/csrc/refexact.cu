// Reference-order reductions for the dense L2-SVM (opt-in: the context option
// `reference_order`).  With them a GPU solve is bit-for-bit the reference's
// (objective, w, every CG count, the active set, predictions).
//
// The reference fixes every reduction's order (proj/include/tron/parallel.hpp:
// 14-34): an l- or |I|-length sum is cut into kReductionBlocks = 64 blocks
// [len*b/64, len*(b+1)/64), each summed SEQUENTIALLY from 0.0, and the 64
// partials merged by a pairwise tree (stride 1, 2, 4, ...); n-length dot
// products are serial left to right (linalg.cpp:267-286).  Margins are
// already bit-exact on the device (sequential row dot, no FMA); what remains
// are the sequential block sums.  They are dependency chains -- one add per
// row, |I|/64 rows long -- so each of the 64 blocks runs on its own SM:
//
//  * ro_accum (svm_gradient / svm_hessian_vec Indirect / masked_sq_col_sums,
//    loss.cpp:129-188, linalg.cpp:231-265): CTA b streams the rows of its
//    block I[|I|b/64 .. |I|(b+1)/64) -- a contiguous row range of the
//    column-major X, 128-row TMA boxes -- and
//      - 4 "term" warps form each row's coefficient (the sequential row dot
//        x_i.v for Hv, z_i - y_i for the gradient, 1 for the preconditioner)
//        and the products c_i*x_ij (row_axpy's a*row[j], one rounding) into a
//        padded row-major term tile;
//      - 2 "chain" warps (one lane per feature j) add the tile's terms in row
//        order: acc_j += t_ij.  Inactive rows and rows outside the block carry
//        t = 0: adding +-0 to an accumulator that started at +0.0 never changes
//        it (round-to-nearest cannot produce -0 from +0 + x unless x = -0, and
//        then the sum is +0), so the chain equals the reference's loop over I.
//    The last CTA merges the 64 partial vectors with the reference's tree and
//    applies the epilogue (w + 2C g, v + 2C Hv, 1 + 2C M); the gradient pass
//    also forms norm2(g) serially and the finiteness flag.
//  * ro_hinge (svm_fused_pass's f, loss.cpp:94-122): 64 chains over the rows
//    of max(1 - y z, 0)^2 (reduce_sum, parallel.cpp:91-100), the scalar tree,
//    and f = 0.5*dot(w,w) + C*sum with a serial dot.
#include "common.cuh"
#include "kernels.h"

namespace tb {

namespace {

constexpr int kBlocks = 64;        // kReductionBlocks (parallel.hpp:24)
constexpr int kRoRows = 128;       // rows per TMA box
constexpr int kTermWarps = 4;      // one row per thread
constexpr int kChainWarps = 2;     // one feature per lane (n <= 64)
constexpr int kRoThreads = (1 + kTermWarps + kChainWarps) * kWarp;

struct RoArgs {
  int mode;  // RO_HV, RO_GRAD, RO_PRECOND
  long long l;
  int n;
  const long long* count;  // |I| (device)
  const int32_t* idx;      // I, ascending
  const uint8_t* mask;     // [ld] active flags
  const double* v;         // HV: v
  const double* z;         // GRAD: margins
  const double* y;         // GRAD: labels
  double* partials;        // [64][n]
  unsigned* ticket;
  EpiView epi;             // base + scale*s or cbase + scale*s
  double* out;             // [n]
  ObjScalars* obj;         // GRAD: gnorm, grad_nonfinite
  int nstages;
};

__device__ __forceinline__ void range_of(long long len, int b, long long& lo, long long& hi) {
  lo = len * b / kBlocks;  // reduction_block (parallel.hpp:29-31)
  hi = len * (b + 1) / kBlocks;
}

__global__ void __launch_bounds__(kRoThreads, 1)
    ro_accum_kernel(const __grid_constant__ CUtensorMap xmap, RoArgs a) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) unsigned long long full[3], empty[3], tfull[2], tempty[2];
  __shared__ double s_v[64];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int n = a.n;
  const int tstride = n + 1;  // padded term rows: conflict-free for both roles
  const size_t xbytes = (size_t)kRoRows * n * 8;
  const size_t sbytes = (xbytes + kRoRows + 127) & ~(size_t)127;  // box + mask bytes
  double* terms = reinterpret_cast<double*>(smem + (size_t)a.nstages * sbytes);

  const long long cnt = *a.count;
  long long klo, khi;
  range_of(cnt, blockIdx.x, klo, khi);
  long long rlo = 0, rhi = -1;  // row range of this block's active rows
  if (khi > klo) {
    rlo = a.idx[klo];
    rhi = a.idx[khi - 1];
  }
  const long long t0 = rlo / kRoRows;
  const long long ntiles = khi > klo ? rhi / kRoRows - t0 + 1 : 0;

  if (tid == 0) {
    for (int s = 0; s < a.nstages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kTermWarps);
    }
    for (int u = 0; u < 2; ++u) {
      mbar_init(&tfull[u], kTermWarps);
      mbar_init(&tempty[u], kChainWarps);
    }
    mbar_fence_init();
  }
  for (int j = tid; j < 64; j += kRoThreads) s_v[j] = (a.mode == RO_HV && j < n) ? a.v[j] : 0.0;
  __syncwarp();
  __syncthreads();

  if (wid == 0) {
    // ---- producer: one {128 rows x n} box of X plus the tile's mask bytes
    if (lane == 0) {
      for (long long k = 0; k < ntiles; ++k) {
        const int s = (int)(k % a.nstages);
        if (k >= a.nstages) mbar_wait_parity(&empty[s], (unsigned)(((k / a.nstages) - 1) & 1));
        unsigned char* base = smem + (size_t)s * sbytes;
        const long long row0 = (t0 + k) * kRoRows;
        mbar_arrive_expect_tx(&full[s], (unsigned)(xbytes + kRoRows));
        tma_load_2d(base, &xmap, (int)row0, 0, &full[s]);
        bulk_g2s(base + xbytes, a.mask + row0, kRoRows, &full[s]);
      }
    }
  } else if (wid <= kTermWarps) {
    // ---- term warps: thread r owns row row0 + r of the tile
    const int r = tid - kWarp;
    for (long long k = 0; k < ntiles; ++k) {
      const int s = (int)(k % a.nstages);
      const int u = (int)(k & 1);
      mbar_wait_parity(&full[s], (unsigned)((k / a.nstages) & 1));
      const double* xs = reinterpret_cast<const double*>(smem + (size_t)s * sbytes);
      const uint8_t* ms = reinterpret_cast<const uint8_t*>(xs) + xbytes;
      const long long i = (t0 + k) * kRoRows + r;
      const bool act = i >= rlo && i <= rhi && ms[r] != 0;
      double c = 0.0;
      if (act) {
        if (a.mode == RO_HV) {  // row_dot(i, v): sequential over j (linalg.cpp:75-86)
          double sdot = 0.0;
          for (int j = 0; j < n; ++j) sdot += xs[j * kRoRows + r] * s_v[j];
          c = sdot;
        } else if (a.mode == RO_GRAD) {
          c = a.z[i] - a.y[i];  // residual (loss.cpp:132)
        } else {
          c = 1.0;  // masked_sq_col_sums: row_axpy_squared(i, 1.0) (linalg.cpp:257-265)
        }
      }
      if (k >= 2) mbar_wait_parity(&tempty[u], (unsigned)(((k >> 1) - 1) & 1));
      double* T = terms + (size_t)u * kRoRows * tstride + (size_t)r * tstride;
      if (a.mode == RO_PRECOND) {
        for (int j = 0; j < n; ++j) {
          const double x = xs[j * kRoRows + r];
          T[j] = act ? (c * x) * x : 0.0;  // a * row[j] * row[j]
        }
      } else {
        for (int j = 0; j < n; ++j) T[j] = c * xs[j * kRoRows + r];  // a * row[j]; c = 0 off I
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&empty[s]);
        mbar_arrive(&tfull[u]);
      }
    }
  } else {
    // ---- chain warps: lane j adds column j of each term tile in row order
    const int j = tid - (1 + kTermWarps) * kWarp;
    double acc = 0.0;  // KernelScratch::acquire_zeroed
    for (long long k = 0; k < ntiles; ++k) {
      const int u = (int)(k & 1);
      mbar_wait_parity(&tfull[u], (unsigned)((k >> 1) & 1));
      if (j < n) {
        const double* T = terms + (size_t)u * kRoRows * tstride + j;
#pragma unroll 16
        for (int r = 0; r < kRoRows; ++r) acc += T[(size_t)r * tstride];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[u]);
    }
    if (j < n) a.partials[(size_t)blockIdx.x * n + j] = acc;
  }

  // ---- the last CTA: merge_vector_tree (parallel.hpp:101-109) + epilogue
  if (last_block_arrive(a.ticket)) {
    if (tid < n) {
      double* P = a.partials;
      for (int stride = 1; stride < kBlocks; stride *= 2)
        for (int i = 0; i + stride < kBlocks; i += 2 * stride)
          P[(size_t)i * n + tid] = __ldcg(P + (size_t)i * n + tid) + __ldcg(P + (size_t)(i + stride) * n + tid);
      const double sj = __ldcg(P + tid);
      const EpiView& E = a.epi;
      a.out[tid] = E.kind == EPI_VEC ? E.base[tid] + E.scale * sj : E.cbase + E.scale * sj;
    }
    if (a.mode == RO_GRAD) {
      __syncthreads();
      if (tid == 0) {  // all_finite(g), then norm2(g) = sqrt(serial dot) (tron.cpp:147-152)
        double gg = 0.0;
        int bad = 0;
        for (int j = 0; j < n; ++j) {
          const double g = a.out[j];
          bad |= !isfinite(g);
          gg += g * g;
        }
        a.obj->gnorm = sqrt(gg);
        a.obj->grad_nonfinite = bad;
      }
    }
  }
}

// hinge-sum chains: CTA b sums max(1 - y_i z_i, 0)^2 over rows [l b/64, l(b+1)/64)
constexpr int kHingeThreads = 256;
constexpr int kHingeTile = 2048;

__global__ void __launch_bounds__(kHingeThreads, 1)
    ro_hinge_kernel(long long l, int n, const double* __restrict__ z, const double* __restrict__ y,
                    const double* __restrict__ w, double C, double* partials, unsigned* ticket,
                    ObjScalars* obj) {
  pdl_wait();
  pdl_trigger();
  __shared__ double h[2][kHingeTile];
  const int tid = threadIdx.x;
  long long lo, hi;
  range_of(l, blockIdx.x, lo, hi);
  const long long ntiles = (hi - lo + kHingeTile - 1) / kHingeTile;
  auto fill = [&](long long k) {  // hinge_sq[i] (loss.cpp:107-113), 0 past the block
    double* H = h[k & 1];
    for (int r = tid - kWarp; r >= 0 && r < kHingeTile; r += kHingeThreads - kWarp) {
      const long long i = lo + k * kHingeTile + r;
      double v = 0.0;
      if (i < hi) {
        const double margin = 1.0 - y[i] * z[i];
        v = margin > 0.0 ? margin * margin : 0.0;
      }
      H[r] = v;
    }
  };
  double acc = 0.0;  // reduce_sum's per-block accumulator (parallel.cpp:95-97)
  if (tid >= kWarp && ntiles > 0) fill(0);
  __syncthreads();
  for (long long k = 0; k < ntiles; ++k) {
    if (tid >= kWarp) {
      if (k + 1 < ntiles) fill(k + 1);
    } else if (tid == 0) {
      const double* H = h[k & 1];
      const int rows = (int)min((long long)kHingeTile, hi - lo - k * kHingeTile);
      for (int r = 0; r < rows; ++r) acc += H[r];
    }
    __syncthreads();
  }
  if (tid == 0) partials[blockIdx.x] = acc;
  if (last_block_arrive(ticket) && tid == 0) {
    double s[kBlocks];
    for (int b = 0; b < kBlocks; ++b) s[b] = __ldcg(partials + b);
    for (int stride = 1; stride < kBlocks; stride *= 2)  // merge_scalar_tree (parallel.hpp:91-99)
      for (int i = 0; i + stride < kBlocks; i += 2 * stride) s[i] += s[i + stride];
    double ww = 0.0;  // dot(w, w) (linalg.cpp:267-272)
    for (int j = 0; j < n; ++j) ww += w[j] * w[j];
    obj->ww = ww;
    obj->f = 0.5 * ww + C * s[0];  // loss.cpp:119
    obj->red[0] = s[0];
  }
}

}  // namespace

int ro_accum_smem(int64_t n) {
  const size_t xbytes = (size_t)kRoRows * n * 8;
  const size_t sbytes = (xbytes + kRoRows + 127) & ~(size_t)127;
  const size_t tbytes = 2 * (size_t)kRoRows * (n + 1) * 8;
  const int stages = (3 * sbytes + tbytes <= 220 * 1024) ? 3 : 2;
  return (int)(stages * sbytes + tbytes);
}

void ro_accum(int mode, int64_t l, int64_t n, const CUtensorMap& xmap128, const long long* count,
              const int32_t* idx, const uint8_t* mask, const double* v, const double* z,
              const double* y, double* partials, unsigned* ticket, const EpiView& epi, double* out,
              ObjScalars* obj, cudaStream_t s) {
  RoArgs a{};
  a.mode = mode;
  a.l = l;
  a.n = (int)n;
  a.count = count;
  a.idx = idx;
  a.mask = mask;
  a.v = v;
  a.z = z;
  a.y = y;
  a.partials = partials;
  a.ticket = ticket;
  a.epi = epi;
  a.out = out;
  a.obj = obj;
  const size_t xbytes = (size_t)kRoRows * n * 8;
  const size_t sbytes = (xbytes + kRoRows + 127) & ~(size_t)127;
  const size_t tbytes = 2 * (size_t)kRoRows * (n + 1) * 8;
  a.nstages = (3 * sbytes + tbytes <= 220 * 1024) ? 3 : 2;
  const int smem = ro_accum_smem(n);
  ensure_max_dynamic_smem((const void*)ro_accum_kernel, smem);
  launch_pdl(ro_accum_kernel, dim3(kBlocks), dim3(kRoThreads), (size_t)smem, s, xmap128, a);
}

void ro_hinge(int64_t l, int64_t n, const double* z, const double* y, const double* w, double C,
              double* partials, unsigned* ticket, ObjScalars* obj, cudaStream_t s) {
  launch_pdl(ro_hinge_kernel, dim3(kBlocks), dim3(kHingeThreads), 0, s, (long long)l, (int)n, z, y,
             w, C, partials, ticket, obj);
}

}  // namespace tb

// ---------------------------------------------------------------------------
// truncated_cg (tron.cpp:37-108) for n <= 64 in the reference's arithmetic
// order: serial dot products, the same element-wise updates.  One thread does
// everything (a few hundred flops per iteration); hp comes finished from
// ro_accum.
// ---------------------------------------------------------------------------
namespace tb {
namespace {

__device__ __forceinline__ void ro_set_cond(Cond c, int v) {
  if (c.on) cudaGraphSetConditional((cudaGraphConditionalHandle)c.h, v ? 1u : 0u);
}

__device__ __forceinline__ double sdot(const double* a, const double* b, long long n) {
  double acc = 0.0;  // dot (linalg.cpp:267-272)
  for (long long j = 0; j < n; ++j) acc += a[j] * b[j];
  return acc;
}

__device__ __forceinline__ double zj(const double* r, const double* M, long long j) {
  return M ? r[j] / M[j] : r[j];  // apply_precond (tron.cpp:46-53)
}

__device__ void ro_cg_finish(const CgVectors& v, CgState* st) {  // tron.cpp:99-106
  if (st->iters >= st->max_iters && st->exit_kind != kCgBoundary && st->rnorm > st->stop)
    st->exit_kind = kCgMaxIters;
  else if (st->exit_kind != kCgBoundary)
    st->exit_kind = kCgConverged;
  st->q = 0.5 * (sdot(v.d, v.g, v.n) - sdot(v.d, v.r0, v.n));
  st->dnorm = sqrt(sdot(v.d, v.d, v.n));
}

__global__ void ro_cg_init_kernel(CgVectors v, CgState* st, Cond cond) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x != 0) return;
  const long long n = v.n;
  for (long long j = 0; j < n; ++j) {
    v.d[j] = 0.0;
    v.r0[j] = -v.g[j];
    v.p[j] = zj(v.r0, v.M, j);
  }
  st->rz = sdot(v.r0, v.p, n);  // p = z here
  st->rnorm = sqrt(sdot(v.r0, v.r0, n));
  st->rpar = 0;
  st->iters = 0;
  st->boundary = 0;
  st->fail = 0;
  st->exit_kind = kCgConverged;
  const int cont = (0 < st->max_iters) && !(st->rnorm <= st->stop);
  st->cont = cont;
  ro_set_cond(cond, cont);
  if (!cont) ro_cg_finish(v, st);
}

__global__ void ro_cg_step_kernel(CgVectors v, CgState* st, Cond cond) {
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x != 0) return;
  const long long n = v.n;
  st->iters += 1;
  const double php = sdot(v.p, v.hp, n);
  st->php = php;
  if (!(php > 0.0)) {
    st->fail = 1;
    st->cont = 0;
    ro_set_cond(cond, 0);
    return;
  }
  const double alpha = st->rz / php;
  st->alpha = alpha;
  for (long long j = 0; j < n; ++j) v.d[j] += alpha * v.p[j];
  const double delta = st->delta;
  if (sqrt(sdot(v.d, v.d, n)) > delta) {
    for (long long j = 0; j < n; ++j) v.d[j] += -alpha * v.p[j];
    const double dp = sdot(v.d, v.p, n);
    const double dd = sdot(v.d, v.d, n);
    const double pp = sdot(v.p, v.p, n);
    const double rad = sqrt(dp * dp + pp * (delta * delta - dd));
    const double tau = dp >= 0.0 ? (delta * delta - dd) / (dp + rad) : (rad - dp) / pp;
    for (long long j = 0; j < n; ++j) v.d[j] += tau * v.p[j];
    for (long long j = 0; j < n; ++j) v.r0[j] += -tau * v.hp[j];
    st->tau = tau;
    st->boundary = 1;
    st->exit_kind = kCgBoundary;
    st->cont = 0;
    ro_set_cond(cond, 0);
    ro_cg_finish(v, st);
    return;
  }
  for (long long j = 0; j < n; ++j) v.r0[j] += -alpha * v.hp[j];
  double rz_next = 0.0;
  for (long long j = 0; j < n; ++j) rz_next += v.r0[j] * zj(v.r0, v.M, j);
  const double beta = rz_next / st->rz;
  for (long long j = 0; j < n; ++j) v.p[j] = zj(v.r0, v.M, j) + beta * v.p[j];
  st->beta = beta;
  st->rz = rz_next;
  st->rnorm = sqrt(sdot(v.r0, v.r0, n));
  st->exit_kind = kCgMaxIters;
  const int cont = (st->iters < st->max_iters) && !(st->rnorm <= st->stop);
  st->cont = cont;
  ro_set_cond(cond, cont);
  if (!cont) ro_cg_finish(v, st);
}

}  // namespace

void ro_cg_init(const CgVectors& v, CgState* st, Cond cond, cudaStream_t s) {
  launch_pdl(ro_cg_init_kernel, dim3(1), dim3(32), 0, s, v, st, cond);
}
void ro_cg_step(const CgVectors& v, CgState* st, Cond cond, cudaStream_t s) {
  launch_pdl(ro_cg_step_kernel, dim3(1), dim3(32), 0, s, v, st, cond);
}

}  // namespace tb
