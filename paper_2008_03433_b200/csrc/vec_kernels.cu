// Device-resident truncated CG (tron.cpp:37-108) and the n-vector helpers
// of the outer loop (tron.cpp:127-217).  Only scalars ever need to leave
// the device: every dot/norm of the reference's serial vector ops
// (linalg.cpp:267-286) becomes a two-stage block reduction whose second
// stage runs in the last block to finish (fixed order => deterministic).
//
// Two engines:
//  * large-n: one grid-stride kernel per CG phase (php, update, direction),
//    used for the high-dimensional sparse problems (n up to 2e7);
//  * small-n: the whole iteration in one single-block kernel (n <= 4096),
//    used for the tall-skinny dense problems (n = 40) where launch count,
//    not bandwidth, is the cost.
// Both can run under a CUDA-graph while node: the kernel that decides
// whether CG continues sets the conditional handle.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

#include <cooperative_groups.h>

namespace tb {

namespace {

constexpr int kBlock = 256;

int vec_grid(int64_t n) {
  int64_t g = (n + kBlock * 4 - 1) / (kBlock * 4);
  int64_t cap = (int64_t)device_sm_count() * 4;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

__device__ __forceinline__ void set_cond(Cond c, int v) {
  if (c.on) cudaGraphSetConditional((cudaGraphConditionalHandle)c.h, v ? 1u : 0u);
}

// (uses are unrolled by four: a thread keeps four iterations' loads in
// flight; the per-thread summation order is unchanged)
#define GRID_STRIDE(j, n)                                                       \
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < (n); \
       j += (long long)gridDim.x * blockDim.x)

__global__ void __launch_bounds__(kBlock) axpy_dot_kernel(long long n, const double* w,
                                                         const double* d, double* wc,
                                                         ObjScalars* obj, Scratch sc) {
  pdl_wait();
  pdl_trigger();
  __shared__ double sh[kBlock / kWarp + 1];
  double acc = 0.0;
#pragma unroll 4
  GRID_STRIDE(j, n) {
    const double v = d ? w[j] + d[j] : w[j];  // axpy_inplace(1.0, d, w_cand), tron.cpp:176-177
    wc[j] = v;
    acc += v * v;
  }
  const double b = block_sum<kBlock>(acc, sh, true);
  if (threadIdx.x == 0) sc.partials[blockIdx.x] = b;
  if (last_block_arrive(sc.tickets + T_AXPY)) {
    const double tot = reduce_partials<kBlock>(sc.partials, gridDim.x, 1, 0, sh);
    if (threadIdx.x == 0) obj->ww = tot;
  }
}

__global__ void __launch_bounds__(kBlock) norm_check_kernel(long long n, const double* g,
                                                           ObjScalars* obj, Scratch sc) {
  pdl_wait();
  pdl_trigger();
  __shared__ double sh[kBlock / kWarp + 1];
  double acc = 0.0, bad = 0.0;
#pragma unroll 4
  GRID_STRIDE(j, n) {
    const double v = g[j];
    acc += v * v;
    if (!isfinite(v)) bad = 1.0;
  }
  const double b = block_sum<kBlock>(acc, sh, true);
  const double bb = block_sum<kBlock>(bad, sh, true);
  if (threadIdx.x == 0) {
    sc.partials[2 * blockIdx.x] = b;
    sc.partials[2 * blockIdx.x + 1] = bb;
  }
  if (last_block_arrive(sc.tickets + T_NORM)) {
    const double tot = reduce_partials<kBlock>(sc.partials, gridDim.x, 2, 0, sh);
    const double nb = reduce_partials<kBlock>(sc.partials, gridDim.x, 2, 1, sh);
    if (threadIdx.x == 0) {
      obj->gnorm = sqrt(tot);
      obj->grad_nonfinite = nb > 0.0;
    }
  }
}

__global__ void __launch_bounds__(kBlock) dot2_kernel(long long n, const double* a, const double* b,
                                                     const double* c, const double* d, double* out2,
                                                     Scratch sc) {
  pdl_wait();
  pdl_trigger();
  __shared__ double sh[kBlock / kWarp + 1];
  double x = 0.0, y = 0.0;
#pragma unroll 4
  GRID_STRIDE(j, n) {
    x += a[j] * b[j];
    y += c[j] * d[j];
  }
  const double bx = block_sum<kBlock>(x, sh, true);
  const double by = block_sum<kBlock>(y, sh, true);
  if (threadIdx.x == 0) {
    sc.partials[2 * blockIdx.x] = bx;
    sc.partials[2 * blockIdx.x + 1] = by;
  }
  if (last_block_arrive(sc.tickets + T_DOT2)) {
    const double tx = reduce_partials<kBlock>(sc.partials, gridDim.x, 2, 0, sh);
    const double ty = reduce_partials<kBlock>(sc.partials, gridDim.x, 2, 1, sh);
    if (threadIdx.x == 0) {
      out2[0] = tx;
      out2[1] = ty;
    }
  }
}

__global__ void __launch_bounds__(kBlock) epilogue_kernel(long long n, const double* raw, EpiView E,
                                                         double* out) {
  pdl_wait();
  pdl_trigger();
  // EPI_VEC with dot_parts: the emission's reduction (EpiView::dot_*), as the
  // segmented kernels do it unsharded -- so p.Hp and ||g|| survive sharding
  // (raw is the allreduced sum: every rank reduces the same bits)
  const bool dot = E.kind == EPI_VEC && E.dot_parts != nullptr;
  double acc = 0.0, bad = 0.0;
#pragma unroll 4
  GRID_STRIDE(j, n) {
    const double s = raw ? raw[j] : 0.0;
    const double o = E.kind == EPI_VEC ? E.base[j] + E.scale * s
                                       : (E.kind == EPI_CONST ? E.cbase + E.scale * s : s);
    out[j] = o;
    if (dot) {
      if (E.dot_mode == 0) {
        acc += E.base[j] * o;
      } else {
        acc += o * o;
        if (!isfinite(o)) bad = 1.0;
      }
    }
  }
  if (!dot) return;
  __shared__ double sh[kBlock / kWarp + 1];
  const double b = block_sum<kBlock>(acc, sh, true);
  const double bb = block_sum<kBlock>(bad, sh, true);
  if (threadIdx.x == 0) {
    E.dot_parts[2 * blockIdx.x] = b;
    E.dot_parts[2 * blockIdx.x + 1] = bb;
  }
  if (last_block_arrive(E.dot_ticket)) {
    const double tot = reduce_partials<kBlock>(E.dot_parts, gridDim.x, 2, 0, sh);
    const double nb = reduce_partials<kBlock>(E.dot_parts, gridDim.x, 2, 1, sh);
    if (threadIdx.x == 0) {
      if (E.dot_mode == 0) {
        *E.dot_out = tot;
      } else {
        E.dot_obj->gnorm = sqrt(tot);
        E.dot_obj->grad_nonfinite = nb > 0.0;
      }
    }
  }
}

// ---------------- large-n CG ----------------

__device__ __forceinline__ double zval(const double* r, const double* M, long long j) {
  return M ? r[j] / M[j] : r[j];  // apply_precond, tron.cpp:46-53
}

__global__ void __launch_bounds__(kBlock) cg_init_kernel(CgVectors v, CgState* st, Scratch sc,
                                                        Cond cond) {
  pdl_wait();
  pdl_trigger();
  __shared__ double sh[kBlock / kWarp + 1];
  double rz = 0.0, rr = 0.0;
#pragma unroll 4
  GRID_STRIDE(j, v.n) {
    v.d[j] = 0.0;
    const double r = -v.g[j];
    v.r0[j] = r;
    const double z = v.M ? r / v.M[j] : r;
    v.p[j] = z;
    rz += r * z;
    rr += r * r;
  }
  const double a = block_sum<kBlock>(rz, sh, true);
  const double b = block_sum<kBlock>(rr, sh, true);
  if (threadIdx.x == 0) {
    sc.partials[2 * blockIdx.x] = a;
    sc.partials[2 * blockIdx.x + 1] = b;
  }
  if (last_block_arrive(sc.tickets + T_CG_INIT)) {
    const double trz = reduce_partials<kBlock>(sc.partials, gridDim.x, 2, 0, sh);
    const double trr = reduce_partials<kBlock>(sc.partials, gridDim.x, 2, 1, sh);
    if (threadIdx.x == 0) {
      st->rz = trz;
      st->rnorm = sqrt(trr);
      st->rpar = 0;
      st->iters = 0;
      st->boundary = 0;
      st->fail = 0;
      st->exit_kind = 0;
      const int cont = (st->iters < st->max_iters) && !(st->rnorm <= st->stop);
      st->cont = cont;
      if (!cont) {  // no iteration: d = 0 (tron.cpp:99-106 with q(0) = 0, ||0|| = 0)
        st->exit_kind = (st->iters >= st->max_iters && st->rnorm > st->stop) ? kCgMaxIters
                                                                             : kCgConverged;
        st->q = 0.0;
        st->dnorm = 0.0;
      }
      set_cond(cond, cont);
    }
  }
}

// ---------------- mid-n CG: one cluster of 8 CTAs per iteration ----------------
// For n up to kClusterCgMaxN the CG vector work of an iteration (tron.cpp:70-97:
// p.Hp, alpha, d, the boundary test and tau, r, z, beta, p) is one kernel on a
// cluster of 8 CTAs: each CTA owns a contiguous slice of the n-vectors, the
// dot products are block sums exchanged through distributed shared memory and
// added in rank order (every CTA holds the identical total), and cluster
// barriers replace the three kernel boundaries of the large-n engine.
namespace cgc = cooperative_groups;
constexpr int kClusterCtas = 8;
constexpr int kClusterBlock = 1024;

// Sums K values over the whole cluster; identical result in every thread.
template <int K>
__device__ __forceinline__ void cluster_sum(double (&v)[K], double* sh, double (*slot)[4]) {
  cgc::cluster_group cl = cgc::this_cluster();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const double b = block_sum<kClusterBlock>(v[k], sh, true);
    if (threadIdx.x == 0) (*slot)[k] = b;
  }
  cl.sync();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double t = 0.0;
    for (int r = 0; r < kClusterCtas; ++r) t += (*cl.map_shared_rank(slot, r))[k];
    v[k] = t;
  }
  cl.sync();  // the slots may be rewritten by the next sum
}

__global__ void __cluster_dims__(kClusterCtas, 1, 1) __launch_bounds__(kClusterBlock)
    cg_cluster_step_kernel(CgVectors v, CgState* st, Cond cond) {
  pdl_wait();
  pdl_trigger();
  __shared__ double sh[kClusterBlock / kWarp + 1];
  __shared__ double slot[4];
  const long long n = v.n;
  const int rank = (int)cgc::this_cluster().block_rank();
  const long long j0 = n * rank / kClusterCtas, j1 = n * (rank + 1) / kClusterCtas;
  const double rz_old = st->rz, delta = st->delta;
  const long long iters = st->iters + 1, max_iters = st->max_iters;
  const double stop = st->stop;
  const int rpar = st->rpar;
  const bool lead = rank == 0 && threadIdx.x == 0;
  double* r = rpar ? v.r1 : v.r0;
  // p.Hp (tron.cpp:71-75)
  double a1[1] = {0.0};
  for (long long j = j0 + threadIdx.x; j < j1; j += kClusterBlock) a1[0] += v.p[j] * v.hp[j];
  cluster_sum<1>(a1, sh, &slot);
  const double php = a1[0];
  if (!(php > 0.0)) {
    if (lead) {
      st->iters = iters;
      st->php = php;
      st->fail = 1;
      st->cont = 0;
      set_cond(cond, 0);
    }
    return;
  }
  const double alpha = rz_old / php;
  // d += alpha p, ||d|| (tron.cpp:76-78)
  double a2[1] = {0.0};
  for (long long j = j0 + threadIdx.x; j < j1; j += kClusterBlock) {
    const double dj = v.d[j] + alpha * v.p[j];
    v.d[j] = dj;
    a2[0] += dj * dj;
  }
  cluster_sum<1>(a2, sh, &slot);
  if (sqrt(a2[0]) > delta) {
    // boundary: retreat, then tau on ||d + tau p|| = delta (tron.cpp:78-90)
    double a3[3] = {0.0, 0.0, 0.0};
    for (long long j = j0 + threadIdx.x; j < j1; j += kClusterBlock) {
      const double pj = v.p[j];
      const double dj = v.d[j] + (-alpha) * pj;
      v.d[j] = dj;
      a3[0] += dj * pj;
      a3[1] += dj * dj;
      a3[2] += pj * pj;
    }
    cluster_sum<3>(a3, sh, &slot);
    const double dp = a3[0], dd = a3[1], pp = a3[2];
    const double rad = sqrt(dp * dp + pp * (delta * delta - dd));
    const double tau = dp >= 0.0 ? (delta * delta - dd) / (dp + rad) : (rad - dp) / pp;
    double a4[3] = {0.0, 0.0, 0.0};  // q(d) and ||d|| of the final step (tron.cpp:99-106)
    for (long long j = j0 + threadIdx.x; j < j1; j += kClusterBlock) {
      const double dj = v.d[j] + tau * v.p[j];
      const double rj = r[j] + (-tau) * v.hp[j];
      v.d[j] = dj;
      r[j] = rj;
      a4[0] += dj * v.g[j];
      a4[1] += dj * rj;
      a4[2] += dj * dj;
    }
    cluster_sum<3>(a4, sh, &slot);
    if (lead) {
      st->iters = iters;
      st->php = php;
      st->alpha = alpha;
      st->tau = tau;
      st->boundary = 1;
      st->exit_kind = kCgBoundary;
      st->q = 0.5 * (a4[0] - a4[1]);
      st->dnorm = sqrt(a4[2]);
      st->cont = 0;
      set_cond(cond, 0);
    }
    return;
  }
  // r -= alpha Hp, z = M^-1 r (tron.cpp:91-95)
  double* rn = rpar ? v.r0 : v.r1;
  double a5[2] = {0.0, 0.0};
  for (long long j = j0 + threadIdx.x; j < j1; j += kClusterBlock) {
    const double rj = r[j] + (-alpha) * v.hp[j];
    rn[j] = rj;
    const double z = v.M ? rj / v.M[j] : rj;
    a5[0] += rj * z;
    a5[1] += rj * rj;
  }
  cluster_sum<2>(a5, sh, &slot);
  const double rz = a5[0], rnorm = sqrt(a5[1]);
  const double beta = rz / rz_old;
  for (long long j = j0 + threadIdx.x; j < j1; j += kClusterBlock)
    v.p[j] = zval(rn, v.M, j) + beta * v.p[j];  // tron.cpp:96
  const int cont = (iters < max_iters) && !(rnorm <= stop);
  if (!cont) {
    // exit classification, q(d) = (d.g - d.r)/2, ||d|| (tron.cpp:97-106)
    double a6[3] = {0.0, 0.0, 0.0};
    for (long long j = j0 + threadIdx.x; j < j1; j += kClusterBlock) {
      const double dj = v.d[j];
      a6[0] += dj * v.g[j];
      a6[1] += dj * rn[j];
      a6[2] += dj * dj;
    }
    cluster_sum<3>(a6, sh, &slot);
    if (lead) {
      st->exit_kind = (iters >= max_iters && rnorm > stop) ? kCgMaxIters : kCgConverged;
      st->q = 0.5 * (a6[0] - a6[1]);
      st->dnorm = sqrt(a6[2]);
    }
  }
  if (lead) {
    st->iters = iters;
    st->php = php;
    st->alpha = alpha;
    st->beta = beta;
    st->rz = rz;
    st->rpar = rpar ^ 1;
    st->rnorm = rnorm;
    st->cont = cont;
    set_cond(cond, cont);
  }
}

// ---------------- small-n CG (single block) ----------------

constexpr int kSmallBlock = 512;

__device__ __forceinline__ double sblock_sum(double v, double* sh) {
  return block_sum<kSmallBlock>(v, sh, true);
}

__device__ void small_finish(const CgVectors& v, CgState* st, double* sh) {
  // exit classification + q(d) + ||d|| (tron.cpp:99-106)
  const double* r = st->rpar ? v.r1 : v.r0;
  double dg = 0.0, dr = 0.0, dd = 0.0;
  for (long long j = threadIdx.x; j < v.n; j += kSmallBlock) {
    dg += v.d[j] * v.g[j];
    dr += v.d[j] * r[j];
    dd += v.d[j] * v.d[j];
  }
  dg = sblock_sum(dg, sh);
  dr = sblock_sum(dr, sh);
  dd = sblock_sum(dd, sh);
  if (threadIdx.x == 0) {
    if (st->iters >= st->max_iters && st->exit_kind != kCgBoundary && st->rnorm > st->stop)
      st->exit_kind = kCgMaxIters;
    else if (st->exit_kind != kCgBoundary)
      st->exit_kind = kCgConverged;
    st->q = 0.5 * (dg - dr);
    st->dnorm = sqrt(dd);
  }
}

__global__ void __launch_bounds__(kSmallBlock) cg_small_init_kernel(CgVectors v, CgState* st,
                                                                    Cond cond) {
  pdl_wait();
  pdl_trigger();
  __shared__ double sh[kSmallBlock / kWarp + 1];
  double rz = 0.0, rr = 0.0;
  for (long long j = threadIdx.x; j < v.n; j += kSmallBlock) {
    v.d[j] = 0.0;
    const double r = -v.g[j];
    v.r0[j] = r;
    const double z = v.M ? r / v.M[j] : r;
    v.p[j] = z;
    rz += r * z;
    rr += r * r;
  }
  rz = sblock_sum(rz, sh);
  rr = sblock_sum(rr, sh);
  __shared__ int s_cont;
  if (threadIdx.x == 0) {
    st->rz = rz;
    st->rnorm = sqrt(rr);
    st->rpar = 0;
    st->iters = 0;
    st->boundary = 0;
    st->fail = 0;
    st->exit_kind = kCgConverged;
    s_cont = (0 < st->max_iters) && !(st->rnorm <= st->stop);
    st->cont = s_cont;
    set_cond(cond, s_cont);
  }
  __syncthreads();
  if (!s_cont) small_finish(v, st, sh);
}

// One CG iteration of the small engine (tron.cpp:64-106) on one block:
// hp (from G, or the per-CTA Hv partials), p.Hp, the step, the boundary case,
// r, beta, p; returns whether the CG continues.
template <int SPLIT>
__device__ __forceinline__ bool small_step(CgVectors v, const double* partials, int nparts, double scale,
                                           CgState* st, Cond cond, const double* gram, double* sh,
                                           double* s_part, int* s_flag) {
  const long long n = v.n;
  if (gram) {
    // hp = p + scale * G p (gram.cu: the dense Hessian of the committed iterate)
    for (long long j = threadIdx.x; j < n; j += kSmallBlock) {
      double t = 0.0;
      for (long long k = 0; k < n; ++k) t += gram[j * n + k] * v.p[k];
      v.hp[j] = v.p[j] + scale * t;
    }
    __syncthreads();
  } else if (partials) {
    // hp_j = p_j + scale * sum_b partials[b*n + j], fixed order (SPLIT lanes per j)
    const int per = kSmallBlock / SPLIT;  // coordinates handled per pass
    for (long long j0 = 0; j0 < n; j0 += per) {
      const int jj = threadIdx.x % per, grp = threadIdx.x / per;
      const long long j = j0 + jj;
      double acc = 0.0;
      if (j < n)
        for (int b = grp; b < nparts; b += SPLIT) acc += __ldcg(partials + (long long)b * n + j);
      s_part[threadIdx.x] = acc;
      __syncthreads();
      if (grp == 0 && j < n) {
        double t = 0.0;
        for (int g2 = 0; g2 < SPLIT; ++g2) t += s_part[g2 * per + jj];
        v.hp[j] = v.p[j] + scale * t;
      }
      __syncthreads();
    }
  }
  // php (tron.cpp:70-76)
  double php = 0.0;
  for (long long j = threadIdx.x; j < n; j += kSmallBlock) php += v.p[j] * v.hp[j];
  php = sblock_sum(php, sh);
  if (threadIdx.x == 0) {
    st->iters += 1;
    st->php = php;
    (*s_flag) = !(php > 0.0);
    if ((*s_flag)) {
      st->fail = 1;
      st->cont = 0;
      set_cond(cond, 0);
    } else {
      st->alpha = st->rz / php;
    }
  }
  __syncthreads();
  if ((*s_flag)) return false;
  const double alpha = st->alpha;
  double dd = 0.0;
  for (long long j = threadIdx.x; j < n; j += kSmallBlock) {
    const double dj = v.d[j] + alpha * v.p[j];
    v.d[j] = dj;
    dd += dj * dj;
  }
  dd = sblock_sum(dd, sh);
  const bool boundary = sqrt(dd) > st->delta;  // uniform
  double* r = st->rpar ? v.r1 : v.r0;
  if (boundary) {
    double dp = 0.0, d2 = 0.0, pp = 0.0;
    for (long long j = threadIdx.x; j < n; j += kSmallBlock) {
      const double pj = v.p[j];
      const double dj = v.d[j] + (-alpha) * pj;
      v.d[j] = dj;
      dp += dj * pj;
      d2 += dj * dj;
      pp += pj * pj;
    }
    dp = sblock_sum(dp, sh);
    d2 = sblock_sum(d2, sh);
    pp = sblock_sum(pp, sh);
    const double delta = st->delta;
    const double rad = sqrt(dp * dp + pp * (delta * delta - d2));
    const double tau = dp >= 0.0 ? (delta * delta - d2) / (dp + rad) : (rad - dp) / pp;
    for (long long j = threadIdx.x; j < n; j += kSmallBlock) {
      v.d[j] = v.d[j] + tau * v.p[j];
      r[j] = r[j] + (-tau) * v.hp[j];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      st->tau = tau;
      st->boundary = 1;
      st->exit_kind = kCgBoundary;
      st->cont = 0;
      set_cond(cond, 0);
    }
    __syncthreads();
    small_finish(v, st, sh);
    return false;
  }
  double rz = 0.0, rr = 0.0;
  for (long long j = threadIdx.x; j < n; j += kSmallBlock) {
    const double rj = r[j] + (-alpha) * v.hp[j];
    r[j] = rj;
    const double z = v.M ? rj / v.M[j] : rj;
    rz += rj * z;
    rr += rj * rj;
  }
  rz = sblock_sum(rz, sh);
  rr = sblock_sum(rr, sh);
  const double beta = rz / st->rz;
  for (long long j = threadIdx.x; j < n; j += kSmallBlock)
    v.p[j] = zval(r, v.M, j) + beta * v.p[j];
  __syncthreads();
  if (threadIdx.x == 0) {
    st->beta = beta;
    st->rz = rz;
    st->rnorm = sqrt(rr);
    st->exit_kind = kCgMaxIters;
    (*s_flag) = (st->iters < st->max_iters) && !(st->rnorm <= st->stop);
    st->cont = (*s_flag);
    set_cond(cond, (*s_flag));
  }
  __syncthreads();
  if (!(*s_flag)) small_finish(v, st, sh);
  return (*s_flag) != 0;
}

template <int SPLIT>
__global__ void __launch_bounds__(kSmallBlock) cg_small_step_kernel(CgVectors v,
                                                                    const double* partials,
                                                                    int nparts, double scale,
                                                                    CgState* st, Cond cond,
                                                                    const double* gram) {
  pdl_wait();
  pdl_trigger();
  __shared__ double sh[kSmallBlock / kWarp + 1];
  __shared__ double s_part[kSmallBlock];
  __shared__ int s_flag;
  small_step<SPLIT>(v, partials, nparts, scale, st, cond, gram, sh, s_part, &s_flag);
}

// Gram mode (n <= 64): the whole CG loop in one launch -- G staged in shared
// memory once, then iterations until the step says stop (the WHILE node
// around it then runs once); the iterations are those of cg_small_step_kernel.
__global__ void __launch_bounds__(kSmallBlock) cg_small_gram_loop_kernel(CgVectors v, double scale,
                                                                         CgState* st, Cond cond,
                                                                         const double* gram) {
  pdl_wait();
  pdl_trigger();
  __shared__ double sh[kSmallBlock / kWarp + 1];
  __shared__ double s_part[kSmallBlock];
  __shared__ int s_flag;
  __shared__ double sG[64 * 64];
  const long long nn = v.n * v.n;
  for (long long e = threadIdx.x; e < nn; e += kSmallBlock) sG[e] = gram[e];
  __syncthreads();
  if (!st->cont) return;  // (the init found r already small enough)
  while (small_step<8>(v, nullptr, 0, scale, st, cond, sG, sh, s_part, &s_flag)) {
  }
}

}  // namespace

void vec_axpy_dot(int64_t n, const double* w, const double* d, double* wc, ObjScalars* obj,
                  Scratch sc, cudaStream_t s) {
  launch_pdl(axpy_dot_kernel, dim3(vec_grid(n)), dim3(kBlock), 0, s, (long long)n, w, d, wc, obj, sc);
}

void vec_norm_check(int64_t n, const double* g, ObjScalars* obj, Scratch sc, cudaStream_t s) {
  launch_pdl(norm_check_kernel, dim3(vec_grid(n)), dim3(kBlock), 0, s, (long long)n, g, obj, sc);
}

// ---------------- large-n CG: one cooperative kernel per iteration ----------------
// The vector work of a CG iteration (tron.cpp:70-106) for n too large for one
// cluster: p.Hp, then d += alpha p together with a speculative r -= alpha Hp
// into the other parity buffer (one barrier serves ||d||, r.z and r.r), then
// beta and p -- grid barriers instead of the three kernels and last-block
// tickets of the cg_php / cg_update / cg_direction sequence.  Per-entry
// arithmetic is theirs; totals come from grid_sums (fixed order).
namespace {
constexpr int kCoopBlock = 256;
namespace cgg = cooperative_groups;

__global__ void __launch_bounds__(kCoopBlock) cg_coop_step_kernel(CgVectors v, CgState* st,
                                                                 double* parts, Cond cond,
                                                                 const double* php_in) {
  cgg::grid_group grid = cgg::this_grid();
  __shared__ double sh[kCoopBlock / kWarp + 1];
  __shared__ double red[4];
  const long long gt = blockIdx.x * (long long)kCoopBlock + threadIdx.x;
  const long long NT = (long long)gridDim.x * kCoopBlock;
  const double rz_old = st->rz, delta = st->delta, stop = st->stop;
  const long long iters = st->iters + 1, max_iters = st->max_iters;
  const int rpar = st->rpar;
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  int buf = 0;
  // distinct buffers: restrict lets the unrolled passes issue the next
  // iterations' loads ahead of this iteration's stores
  double* __restrict__ r = rpar ? v.r1 : v.r0;
  double* __restrict__ rn = rpar ? v.r0 : v.r1;
  double* __restrict__ vd = v.d;
  double* __restrict__ vp = v.p;
  const double* __restrict__ vhp = v.hp;
  const double* __restrict__ vM = v.M;
  const double* __restrict__ vg = v.g;
  // p.Hp (tron.cpp:71-75): summed by the Hv kernels as they emitted hp
  // (php_in), else a pass over p and hp
  double php;
  if (php_in) {
    php = *php_in;
  } else {
    double x1[1] = {0.0};
#pragma unroll 4
    for (long long j = gt; j < v.n; j += NT) x1[0] += vp[j] * vhp[j];
    grid_sums<kCoopBlock, 1>(x1, parts, buf, sh, red, grid);
    php = x1[0];
  }
  if (!(php > 0.0)) {
    if (lead) {
      st->iters = iters;
      st->php = php;
      st->fail = 1;
      st->cont = 0;
      set_cond(cond, 0);
    }
    return;
  }
  const double alpha = rz_old / php;
  // d += alpha p (tron.cpp:76-78); r -= alpha Hp, z = M^-1 r (tron.cpp:91-95)
  double x2[3] = {0.0, 0.0, 0.0};
#pragma unroll 4
  for (long long j = gt; j < v.n; j += NT) {
    const double dj = vd[j] + alpha * vp[j];
    vd[j] = dj;
    x2[0] += dj * dj;
    const double rj = r[j] + (-alpha) * vhp[j];
    rn[j] = rj;
    const double z = vM ? rj / vM[j] : rj;
    x2[1] += rj * z;
    x2[2] += rj * rj;
  }
  grid_sums<kCoopBlock, 3>(x2, parts, buf, sh, red, grid);
  if (sqrt(x2[0]) > delta) {
    // boundary: retreat, then tau on ||d + tau p|| = delta (tron.cpp:78-90)
    double x3[3] = {0.0, 0.0, 0.0};
  #pragma unroll 4
  for (long long j = gt; j < v.n; j += NT) {
      const double pj = vp[j];
      const double dj = vd[j] + (-alpha) * pj;
      vd[j] = dj;
      x3[0] += dj * pj;
      x3[1] += dj * dj;
      x3[2] += pj * pj;
    }
    grid_sums<kCoopBlock, 3>(x3, parts, buf, sh, red, grid);
    const double dp = x3[0], dd = x3[1], pp = x3[2];
    const double rad = sqrt(dp * dp + pp * (delta * delta - dd));
    const double tau = dp >= 0.0 ? (delta * delta - dd) / (dp + rad) : (rad - dp) / pp;
    double x4[3] = {0.0, 0.0, 0.0};  // q(d) and ||d|| of the final step (tron.cpp:99-106)
  #pragma unroll 4
  for (long long j = gt; j < v.n; j += NT) {
      const double dj = vd[j] + tau * vp[j];
      const double rj = r[j] + (-tau) * vhp[j];
      vd[j] = dj;
      r[j] = rj;
      x4[0] += dj * vg[j];
      x4[1] += dj * rj;
      x4[2] += dj * dj;
    }
    grid_sums<kCoopBlock, 3>(x4, parts, buf, sh, red, grid);
    if (lead) {
      st->iters = iters;
      st->php = php;
      st->alpha = alpha;
      st->tau = tau;
      st->boundary = 1;
      st->exit_kind = kCgBoundary;
      st->q = 0.5 * (x4[0] - x4[1]);
      st->dnorm = sqrt(x4[2]);
      st->cont = 0;
      set_cond(cond, 0);
    }
    return;
  }
  const double rz = x2[1], rnorm = sqrt(x2[2]);
  const double beta = rz / rz_old;
#pragma unroll 4
  for (long long j = gt; j < v.n; j += NT) vp[j] = (vM ? rn[j] / vM[j] : rn[j]) + beta * vp[j];  // tron.cpp:96
  const int cont = (iters < max_iters) && !(rnorm <= stop);
  if (!cont) {
    // exit classification, q(d) = (d.g - d.r)/2, ||d|| (tron.cpp:97-106)
    double x6[3] = {0.0, 0.0, 0.0};
  #pragma unroll 4
  for (long long j = gt; j < v.n; j += NT) {
      const double dj = vd[j];
      x6[0] += dj * vg[j];
      x6[1] += dj * rn[j];
      x6[2] += dj * dj;
    }
    grid_sums<kCoopBlock, 3>(x6, parts, buf, sh, red, grid);
    if (lead) {
      st->exit_kind = (iters >= max_iters && rnorm > stop) ? kCgMaxIters : kCgConverged;
      st->q = 0.5 * (x6[0] - x6[1]);
      st->dnorm = sqrt(x6[2]);
    }
  }
  if (lead) {
    st->iters = iters;
    st->php = php;
    st->alpha = alpha;
    st->beta = beta;
    st->rz = rz;
    st->rpar = rpar ^ 1;
    st->rnorm = rnorm;
    st->cont = cont;
    set_cond(cond, cont);
  }
}
}  // namespace

#ifndef TB_COOP_PER_SM
#define TB_COOP_PER_SM 4
#endif
// 4 CTAs of 8 warps per SM: the passes stream ~10 n-vectors from HBM and need
// the loads in flight; more CTAs make each grid barrier dearer
int cg_coop_grid() {
  static const int g = [] {
    int per_sm = 0;  // a cooperative grid must be co-resident
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cg_coop_step_kernel, kCoopBlock, 0);
    return std::max(1, std::min(per_sm, TB_COOP_PER_SM)) * device_sm_count();
  }();
  return g;
}

void cg_coop_step(const CgVectors& v, CgState* st, double* parts, Cond cond, cudaStream_t s,
                  const double* php_in) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)cg_coop_grid());
  cfg.blockDim = dim3(kCoopBlock);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, cg_coop_step_kernel, v, st, parts, cond, php_in);
  if (e != cudaSuccess) launch_failed(e, "cg_coop_step (cooperative launch)");
}

__global__ void obj_combine_kernel(ObjScalars* obj, const double* red, long long nblk, double C) {
  double tot = 0.0, cnt = 0.0;
  for (long long b = 0; b < nblk; ++b) {
    tot += red[2 * b];
    cnt += red[2 * b + 1];
  }
  obj->f = 0.5 * obj->ww + C * tot;  // loss.cpp:57 / :119
  obj->nact = (long long)cnt;
  obj->red[0] = tot;
  obj->red[1] = cnt;
}

void obj_combine_blocks(ObjScalars* obj, const double* red, int64_t nblk, double C, cudaStream_t s) {
  obj_combine_kernel<<<1, 1, 0, s>>>(obj, red, (long long)nblk, C);
  TB_LAUNCH_CHECK();
}

__global__ void __launch_bounds__(kBlock) lincomb_kernel(long long n, double a, const double* x,
                                                        double b, const double* y, double* out) {
  pdl_wait();
  pdl_trigger();
  GRID_STRIDE(j, n) {
    const double xv = x ? a * x[j] : 0.0;
    out[j] = y ? (x ? xv + b * y[j] : b * y[j]) : xv;
  }
}

__global__ void __launch_bounds__(kBlock) div_kernel(long long n, const double* r, const double* M,
                                                    double* z) {
  pdl_wait();
  pdl_trigger();
  GRID_STRIDE(j, n) z[j] = M ? r[j] / M[j] : r[j];  // apply_precond, tron.cpp:46-53
}

__global__ void __launch_bounds__(kBlock) sumsq_bad_kernel(long long n, const double* g, double* out2,
                                                          Scratch sc) {
  pdl_wait();
  pdl_trigger();
  __shared__ double sh[kBlock / kWarp + 1];
  double acc = 0.0, bad = 0.0;
  GRID_STRIDE(j, n) {
    const double v = g[j];
    acc += v * v;
    if (!isfinite(v)) bad = 1.0;
  }
  const double b = block_sum<kBlock>(acc, sh, true);
  const double bb = block_sum<kBlock>(bad, sh, true);
  if (threadIdx.x == 0) {
    sc.partials[2 * blockIdx.x] = b;
    sc.partials[2 * blockIdx.x + 1] = bb;
  }
  if (last_block_arrive(sc.tickets + T_SUMSQ)) {
    const double tot = reduce_partials<kBlock>(sc.partials, gridDim.x, 2, 0, sh);
    const double nb = reduce_partials<kBlock>(sc.partials, gridDim.x, 2, 1, sh);
    if (threadIdx.x == 0) {
      out2[0] = tot;
      out2[1] = nb;
    }
  }
}

__global__ void set_gnorm_kernel(ObjScalars* obj, const double* in2) {
  obj->gnorm = sqrt(in2[0]);
  obj->grad_nonfinite = in2[1] > 0.0;
}

__global__ void __launch_bounds__(kBlock) row_scale_kernel(long long l, double* a, const double* dvec,
                                                          const uint8_t* mask) {
  pdl_wait();
  pdl_trigger();
  GRID_STRIDE(i, l) a[i] = dvec ? a[i] * dvec[i] : (mask[i] ? a[i] : 0.0);  // loss.cpp:86-89, :150-160
}

void vec_lincomb(int64_t n, double a, const double* x, double b, const double* y, double* out,
                 cudaStream_t s) {
  if (n > 0) launch_pdl(lincomb_kernel, dim3(vec_grid(n)), dim3(kBlock), 0, s, (long long)n, a, x, b, y, out);
}
void vec_div(int64_t n, const double* r, const double* M, double* z, cudaStream_t s) {
  if (n > 0) launch_pdl(div_kernel, dim3(vec_grid(n)), dim3(kBlock), 0, s, (long long)n, r, M, z);
}
void vec_sumsq_bad(int64_t n, const double* g, double* out2, Scratch sc, cudaStream_t s) {
  launch_pdl(sumsq_bad_kernel, dim3(vec_grid(n)), dim3(kBlock), 0, s, (long long)n, g, out2, sc);
}
namespace {
// Replica checksum: the wrap-around sum of the 64-bit patterns of w, f and
// delta (integer addition: the same in any order), as four 16-bit chunks and
// their squares -- exact in doubles, so after a sum over the ranks every rank
// can test "all equal" as world * sum(h^2) == sum(h)^2.
__global__ void __launch_bounds__(256) replica_checksum_kernel(long long n, const double* __restrict__ w,
                                                               double f, double delta, double* out8) {
  __shared__ unsigned long long sh[256];
  unsigned long long s = 0;
  for (long long i = threadIdx.x; i < n; i += 256) s += (unsigned long long)__double_as_longlong(w[i]);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) sh[threadIdx.x] += sh[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const unsigned long long t = sh[0] + (unsigned long long)__double_as_longlong(f) * 3ull +
                                 (unsigned long long)__double_as_longlong(delta) * 5ull;
    for (int c = 0; c < 4; ++c) {
      const double h = (double)((t >> (16 * c)) & 0xffffull);
      out8[c] = h;
      out8[4 + c] = h * h;
    }
  }
}
}  // namespace

void replica_checksum(int64_t n, const double* w, double f, double delta, double* out8, cudaStream_t s) {
  replica_checksum_kernel<<<1, 256, 0, s>>>((long long)n, w, f, delta, out8);
  TB_LAUNCH_CHECK();
}

void obj_set_gnorm(ObjScalars* obj, const double* in2, cudaStream_t s) {
  set_gnorm_kernel<<<1, 1, 0, s>>>(obj, in2);
  TB_LAUNCH_CHECK();
}
void vec_row_scale(int64_t l, double* a, const double* dvec, const uint8_t* mask, cudaStream_t s) {
  if (l > 0) launch_pdl(row_scale_kernel, dim3(vec_grid(l)), dim3(kBlock), 0, s, (long long)l, a, dvec, mask);
}

void vec_dot2(int64_t n, const double* a, const double* b, const double* c, const double* d,
              double* out2, Scratch sc, cudaStream_t s) {
  launch_pdl(dot2_kernel, dim3(vec_grid(n)), dim3(kBlock), 0, s, (long long)n, a, b, c, d, out2, sc);
}

void vec_epilogue(int64_t n, const double* raw, const EpiView& epi, double* out, cudaStream_t s) {
  launch_pdl(epilogue_kernel, dim3(vec_grid(n)), dim3(kBlock), 0, s, (long long)n, raw, epi, out);
}

void cg_cluster_step(const CgVectors& v, CgState* st, Cond cond, cudaStream_t s) {
  launch_pdl(cg_cluster_step_kernel, dim3(kClusterCtas), dim3(kClusterBlock), 0, s, v, st, cond);
}

void cg_large_init(const CgVectors& v, CgState* st, Scratch sc, Cond cond, cudaStream_t s) {
  launch_pdl(cg_init_kernel, dim3(vec_grid(v.n)), dim3(kBlock), 0, s, v, st, sc, cond);
}

void cg_small_init(const CgVectors& v, CgState* st, Cond cond, cudaStream_t s) {
  launch_pdl(cg_small_init_kernel, dim3(1), dim3(kSmallBlock), 0, s, v, st, cond);
}

void cg_small_step(const CgVectors& v, const double* partials, int nparts, double scale,
                   CgState* st, Cond cond, cudaStream_t s) {
  const double* no_gram = nullptr;
  if (v.n <= 32)
    launch_pdl(cg_small_step_kernel<16>, dim3(1), dim3(kSmallBlock), 0, s, v, partials, nparts, scale,
               st, cond, no_gram);
  else if (v.n <= 64)
    launch_pdl(cg_small_step_kernel<8>, dim3(1), dim3(kSmallBlock), 0, s, v, partials, nparts, scale,
               st, cond, no_gram);
  else
    launch_pdl(cg_small_step_kernel<1>, dim3(1), dim3(kSmallBlock), 0, s, v, partials, nparts, scale,
               st, cond, no_gram);
}

void cg_small_gram_loop(const CgVectors& v, const double* G, double scale, CgState* st, Cond cond,
                        cudaStream_t s) {
  launch_pdl(cg_small_gram_loop_kernel, dim3(1), dim3(kSmallBlock), 0, s, v, scale, st, cond, G);
}

void cg_small_step_gram(const CgVectors& v, const double* G, double scale, CgState* st, Cond cond,
                        cudaStream_t s) {
  const double* no_parts = nullptr;
  launch_pdl(cg_small_step_kernel<8>, dim3(1), dim3(kSmallBlock), 0, s, v, no_parts, 0, scale, st, cond,
             G);
}

namespace {
__global__ void read_flush_kernel(const double2* __restrict__ p, long long n2, double* sink) {
  double acc = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2;
       i += (long long)gridDim.x * blockDim.x) {
    const double2 v = __ldcg(p + i);
    acc += v.x + v.y;
  }
  if (acc == 1.2345e-300) *sink = acc;  // never taken; keeps the loads
}
}  // namespace

// Evicts the L2 by READING a buffer larger than it: the cache is left holding
// clean, unrelated lines, so a timed kernel pays neither hits on its own data
// nor write-backs of a write-based flush (kernel timing only).
void l2_read_flush(const double* buf, int64_t n, cudaStream_t s) {
  read_flush_kernel<<<device_sm_count() * 4, 512, 0, s>>>((const double2*)buf, n / 2,
                                                           const_cast<double*>(buf));
  TB_LAUNCH_CHECK();
}

}  // namespace tb
