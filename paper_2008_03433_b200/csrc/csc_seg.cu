// X^T u over the device CSC copy: warp-per-chunk segmented reduction.
//
// The reference computes X^T u (matvec_transpose / masked_matvec_transpose /
// weighted_sq_col_sums, proj/src/linalg.cpp:175-265) by scattering every row
// into one of 64 private n-length buffers and merging them serially
// (parallel.hpp:101-123) -- the dominant cost of TRON-LR at large n.  Here
// the CSC copy turns it into a segmented sum over contiguous memory:
//
//  * the nonzeros are cut into fixed chunks of 256 (one warp, 8 per lane),
//    so work is balanced regardless of column lengths (Zipf-hot columns of
//    20k+ entries cost the same as short ones);
//  * per-entry "last entry of its column" bits, the chunk -> column-rank
//    map, the table of non-empty columns and the list of empty ones are
//    built once per matrix on the device (the structure never changes
//    during a solve);
//  * a lane sums its 8 products sequentially, column pieces that cross
//    lanes are combined by one warp-level segmented scan, the pieces of
//    long columns by a fixed-order fix-up pass.  No atomics, no shared
//    memory, no block barriers: results are bit-reproducible run to run.
//  * the empty columns (27% of news20) are written from their own list in
//    the same launch, so the epilogue (base_j + scale*sum) covers every j
//    in one pass.
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"
#include "rowdot.cuh"

#include <algorithm>
#include <cstdlib>

namespace tb {

namespace {

constexpr int kBlock = 256;  // 8 warps = 8 chunks in flight per block
constexpr int kEmptyItems = 4;  // empty rows per lane per visit

// TB_LD256: the chunk's nonzeros as 256-bit loads (sm_100: one LDG.256 moves
// 32 B per lane) marked L2::evict_first, so the once-read X stream does not
// push the gathered vector out of L2.
#ifndef TB_LD256
#define TB_LD256 1  // measured: N1 Hv 91.8 -> 80.6 us, K1 3.63 -> 3.47 ms
#endif
constexpr int kSegBlocksPerSm = 2;  // 128 registers: 16 warps per SM (seg_dot_slots counts on it)
__device__ __forceinline__ void ld4d_ef(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.b64 {%0, %1, %2, %3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p));
}
__device__ __forceinline__ void ld8i_ef(const int* p, int (&x)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]),
                 "=r"(x[7])
               : "l"(p));
}
#if !TB_LD256
__device__ __forceinline__ void ld2(const double* p, double& a, double& b) {
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(a), "=d"(b)
               : "l"(p));
}
__device__ __forceinline__ void ld4(const int* p, int& a, int& b, int& c, int& d) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "l"(p));
}
#endif

// Reduction over the emitted values (EpiView::dot_*): dacc gathers
// base_j * out_j (mode 0) or out_j^2 (mode 1), bad counts non-finite out_j.
struct DotAcc {
  double acc = 0.0, bad = 0.0;
  __device__ __forceinline__ void add(const EpiView& E, double b, double o) {
    if (E.dot_mode == 0) {
      acc += b * o;
    } else {
      acc += o * o;
      if (!isfinite(o)) bad = 1.0;
    }
  }
};

// Epilogue out_j = base_j + scale*sum (VEC), cbase + scale*sum (CONST) or
// sum (RAW); base_j is requested early (epi_base) and applied at emission.
// COH (persistent CG kernel): the vector is written inside the same kernel by
// other CTAs, so it is read through L2 (ld.global.cg), never the
// non-coherent path.
#ifndef TB_COH_LOAD
#define TB_COH_LOAD 1  // 0: ld.global.cg (L2 only), 1: plain ld.global (ordered by grid.sync)
#endif
__device__ __forceinline__ double ld_coh(const double* p) {
#if TB_COH_LOAD
  return *p;
#else
  return __ldcg(p);
#endif
}
template <bool COH>
__device__ __forceinline__ double ldv(const double* p) {
  return COH ? ld_coh(p) : __ldg(p);
}
template <int EPI, bool COH = false>
__device__ __forceinline__ double epi_base(const EpiView& E, int j) {
  return (EPI == EPI_VEC && j >= 0) ? ldv<COH>(E.base + j) : 0.0;
}
template <int EPI>
__device__ __forceinline__ double epi_apply(const EpiView& E, double base, double sum) {
  if (EPI == EPI_VEC) return base + E.scale * sum;
  if (EPI == EPI_CONST) return E.cbase + E.scale * sum;
  return sum;
}

// Effective per-row weight u_r (row_axpy's a, linalg.cpp:88-109).
template <int UK, bool COH = false>
__device__ __forceinline__ double ueff(const UView& U, long long r) {
  if (UK == U_VEC) return ldv<COH>(U.u + r);
  if (UK == U_SVM_RESID) return U.mask[r] ? (U.z[r] - U.y[r]) : 0.0;
  return U.mask[r] ? 1.0 : 0.0;
}

// Operands of one chunk for one lane, moved through a three-stage software
// pipeline so that no load sits on a chunk's own dependency chain:
//   chunk rank          requested three chunks ahead,
//   nonzeros, last-entry bits, row table (col)   two ahead,
//   gathered u_r and the epilogue bases          one ahead,
//   sums, scans and emission                     now.
struct LaneChunk {
  long long base;  // the lane's first entry (multiple of kSegLaneItems)
  double v[kSegLaneItems];
  int ix[kSegLaneItems];
  double g[kSegLaneItems];  // gathered u_r (stage 2)
  double bv[2];             // epilogue bases of col[] (stage 2)
  unsigned word, cr;        // last-entry bits holding the lane's items; chunk rank
  int col[2];               // nz_col[rank + lane], nz_col[rank + 32 + lane]; -1 past the table
};

// The CSC copy is padded to whole chunks (zero entries, no last-entry bits),
// so every chunk is read in full without bounds checks.
__device__ __forceinline__ void load_chunk(const CsrView& A, const SegView& S, long long t, int lane,
                                           unsigned cr, LaneChunk& c) {
  c.base = t * kSegChunk + lane * kSegLaneItems;  // 64-B aligned (values), 32-B (indices)
#if TB_LD256
  static_assert(kSegLaneItems == 8, "two 256-bit value loads, one index load per lane");
  ld4d_ef(A.val + c.base, c.v[0], c.v[1], c.v[2], c.v[3]);
  ld4d_ef(A.val + c.base + 4, c.v[4], c.v[5], c.v[6], c.v[7]);
  ld8i_ef(A.idx + c.base, c.ix);
#else
#pragma unroll
  for (int m = 0; m < kSegLaneItems; m += 2) ld2(A.val + c.base + m, c.v[m], c.v[m + 1]);
#pragma unroll
  for (int m = 0; m < kSegLaneItems; m += 4)
    ld4(A.idx + c.base + m, c.ix[m], c.ix[m + 1], c.ix[m + 2], c.ix[m + 3]);
#endif
  // a lane's 8 items never straddle a 32-bit word (base is a multiple of 8)
  c.word = __ldg(S.lastbits + (c.base >> 5));
  c.cr = cr;
  const long long r0 = cr & 0x7fffffffu;
  c.col[0] = r0 + lane < S.nnzc ? __ldg(S.nz_col + r0 + lane) : -1;
  c.col[1] = r0 + 32 + lane < S.nnzc ? __ldg(S.nz_col + r0 + 32 + lane) : -1;
}

// Stage 2.  STAGED: the u_r are LDS reads, so the products are formed here
// and only they stay live; otherwise the gathered u_r stay in flight until
// the chunk is processed.
template <int UK, bool SQ, int EPI, bool STAGED, bool COH>
__device__ __forceinline__ void gather_chunk(const UView& U, const EpiView& E, const double* su,
                                             LaneChunk& c) {
#pragma unroll
  for (int m = 0; m < kSegLaneItems; ++m) {
    if (STAGED) {
      const double u = su[c.ix[m]];
      c.g[m] = SQ ? (u * c.v[m]) * c.v[m] : u * c.v[m];  // row_axpy(_squared)
    } else {
      c.g[m] = ueff<UK, COH>(U, c.ix[m]);
    }
  }
  c.bv[0] = epi_base<EPI, COH>(E, c.col[0]);
  c.bv[1] = epi_base<EPI, COH>(E, c.col[1]);
}

// One chunk: products, per-lane sequential sums, warp segmented scan, emission.
template <bool SQ, int EPI, bool STAGED, bool COH>
__device__ __forceinline__ void process_chunk(const CsrView& A, const SegView& S, const EpiView& E,
                                              double* __restrict__ out, long long t,
                                              const LaneChunk& cur, int lane, double* ebuf,
                                              DotAcc& dacc) {
  double w[kSegLaneItems];
#pragma unroll
  for (int m = 0; m < kSegLaneItems; ++m)  // row_axpy / row_axpy_squared
    w[m] = STAGED ? cur.g[m] : (SQ ? (cur.g[m] * cur.v[m]) * cur.v[m] : cur.g[m] * cur.v[m]);

  const unsigned bits = (cur.word >> (cur.base & 31)) & 0xffu;
  const int chunk_rank = (int)(cur.cr & 0x7fffffffu);
  const bool cont_in = (cur.cr >> 31) != 0;

  // rank of the row containing this lane's first item
  const int cnt = __popc(bits);
  int incl = cnt;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += y;
  }
  const int r0 = chunk_rank + incl - cnt;

  // sequential pass over the lane's items; the sums of the rows ending here
  // go to the warp's buffer, indexed by their order in the chunk
  // (branch-free: predicated stores and selects; the first row ending here,
  // whose sum may continue a previous lane's, is rewritten after the scan)
  double acc = 0.0;
  int k = incl - cnt;
#pragma unroll
  for (int m = 0; m < kSegLaneItems; ++m) {
    acc += w[m];
    const bool end = (bits >> m) & 1u;
    if (end) ebuf[k] = acc;
    k += end;
    acc = end ? 0.0 : acc;
  }

  // warp segmented inclusive scan of the carries, keyed by row rank
  const int key = r0 + cnt;
  double val = acc;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int k2 = __shfl_up_sync(0xffffffffu, key, off);
    const double v2 = __shfl_up_sync(0xffffffffu, val, off);
    if (lane >= off && k2 == key) val = v2 + val;
  }
  const int prev_key = __shfl_up_sync(0xffffffffu, key, 1);
  const double prev_val = __shfl_up_sync(0xffffffffu, val, 1);
  if (cnt > 0 && lane > 0 && prev_key == r0) ebuf[incl - cnt] = prev_val + ebuf[incl - cnt];
  const double tail = __shfl_sync(0xffffffffu, val, 31);  // the row open at the chunk's end
  // emission, warp-cooperative: consecutive rows to consecutive lanes
  // (coalesced stores); the first 64 use the prefetched row table and bases
  __syncwarp();
  const int nend = __shfl_sync(0xffffffffu, incl, 31);
  if (lane < nend) {
    const double v = ebuf[lane];
    if (lane == 0 && cont_in) {
      S.head[t] = v;  // row began in an earlier chunk: finished by the fix-up
    } else {
      const double o = epi_apply<EPI>(E, cur.bv[0], v);
      out[cur.col[0]] = o;
      if (EPI == EPI_VEC && E.dot_parts) dacc.add(E, cur.bv[0], o);
    }
  }
  if (lane + 32 < nend) {
    const double o = epi_apply<EPI>(E, cur.bv[1], ebuf[lane + 32]);
    out[cur.col[1]] = o;
    if (EPI == EPI_VEC && E.dot_parts) dacc.add(E, cur.bv[1], o);
  }
  for (int q = lane + 64; q < nend; q += 32) {
    const int j = __ldg(S.nz_col + chunk_rank + q);
    const double bj = epi_base<EPI, COH>(E, j);
    const double o = epi_apply<EPI>(E, bj, ebuf[q]);
    out[j] = o;
    if (EPI == EPI_VEC && E.dot_parts) dacc.add(E, bj, o);
  }
  if (lane == 0) S.carry[t] = tail;
  __syncwarp();  // the buffer is reused by the warp's next chunk
}

constexpr int kStagedBlock = 512;                  // one 16-warp block per SM
constexpr long long kStageMaxBytes = 190 * 1024;   // + 32 KB of emission buffers

// Persistent warps walk chunks t, t+W, t+2W, ... through the pipeline above.
// STAGED: u (length A.cols) is first copied to shared memory (TMA bulk copy),
// so a gather is an LDS instead of a 32-line L1 request; the L1 wavefront
// queue, not HBM, bounds the unstaged kernel on L2-resident u.
// The empty rows (out_j = epilogue of 0) are a flat list shared by all warps.
// Body shared with the persistent CG kernel (which runs it with COH and
// without STAGED); every thread of the block calls it.
template <int UK, bool SQ, int EPI, bool STAGED, bool COH, int BLK>
__device__ __forceinline__ void seg_body(const CsrView& A, const SegView& S, const UView& U,
                                         const EpiView& E, double* __restrict__ out, double* su,
                                         double* ebuf, long long gw, long long W, int lane) {
  const long long nch = S.nchunks;

  long long t = gw;
  // chunk ranks of the warp's next 32 chunks (t, t+W, ...), one per lane,
  // refilled every 32 chunks: a chunk's row-table loads never wait for its rank
  long long cr_base = t;
  unsigned crv = t + lane * W < nch ? __ldg(S.chunk_rank + t + lane * W) : 0u;
  auto rank_of = [&](long long tt) -> unsigned {
    long long k = (tt - cr_base) / W;
    if (k >= 32) {  // warp-uniform
      cr_base = tt;
      crv = tt + lane * W < nch ? __ldg(S.chunk_rank + tt + lane * W) : 0u;
      k = 0;
    }
    return __shfl_sync(0xffffffffu, crv, (int)k);
  };
  LaneChunk b0, b1;
  if (t < nch) {
    load_chunk(A, S, t, lane, rank_of(t), b0);
    if (t + W < nch) load_chunk(A, S, t + W, lane, rank_of(t + W), b1);
  }
  DotAcc dacc;  // this lane's part of the emission reduction (E.dot_parts)
  // two buffers in ping-pong (unrolled by two: a register copy of a buffer
  // whose loads are in flight would wait for them).
  // chunk t: processed; t+W: gathered; t+2W: nonzeros in flight
  auto seg_walk = [&](long long t) {
#define TB_SEG_STEP(P, G)                                                      \
  process_chunk<SQ, EPI, STAGED, COH>(A, S, E, out, t, P, lane, ebuf, dacc);   \
  if (t + W >= nch) break;                                                     \
  gather_chunk<UK, SQ, EPI, STAGED, COH>(U, E, su, G);                         \
  if (t + 2 * W < nch) load_chunk(A, S, t + 2 * W, lane, rank_of(t + 2 * W), P); \
  t += W;
    gather_chunk<UK, SQ, EPI, STAGED, COH>(U, E, su, b0);
    for (;;) {
      TB_SEG_STEP(b0, b1)
      TB_SEG_STEP(b1, b0)
    }
#undef TB_SEG_STEP
  };
  if (STAGED) {
    if (UK == U_VEC) {
      bulk_stage_f64(su, U.u, A.cols);  // TMA bulk copy (UBLKCP)
    } else {
      for (long long i = threadIdx.x; i < A.cols; i += BLK) su[i] = ueff<UK>(U, i);
      __syncthreads();
    }
  }

  for (long long b = gw * (32 * kEmptyItems); b < S.nempty; b += W * (32 * kEmptyItems)) {
    int e[kEmptyItems];
    double bb[kEmptyItems];
#pragma unroll
    for (int m = 0; m < kEmptyItems; ++m) {
      const long long i = b + m * 32 + lane;
      e[m] = i < S.nempty ? __ldg(S.empty_col + i) : -1;
    }
#pragma unroll
    for (int m = 0; m < kEmptyItems; ++m) bb[m] = epi_base<EPI, COH>(E, e[m]);
#pragma unroll
    for (int m = 0; m < kEmptyItems; ++m)
      if (e[m] >= 0) {
        const double o = epi_apply<EPI>(E, bb[m], 0.0);
        out[e[m]] = o;
        if (EPI == EPI_VEC && E.dot_parts) dacc.add(E, bb[m], o);
      }
  }
  if (t < nch) seg_walk(t);
  if (EPI == EPI_VEC && E.dot_parts) {  // warp partial, fixed order
    const double a = warp_sum(dacc.acc), b = warp_sum(dacc.bad);
    if (lane == 0) {
      E.dot_parts[2 * gw] = a;
      E.dot_parts[2 * gw + 1] = b;
    }
  }
}


template <int UK, bool SQ, int EPI, bool STAGED>
__global__ void __launch_bounds__(STAGED ? kStagedBlock : kBlock, STAGED ? 1 : kSegBlocksPerSm)
    seg_spmv_kernel(CsrView A, SegView S, UView U, EpiView E, double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  constexpr int BLK = STAGED ? kStagedBlock : kBlock;
  extern __shared__ double su[];
  __shared__ double ebuf_all[BLK / kWarp][kSegChunk];
  const int lane = threadIdx.x & 31;
  const long long W = ((long long)gridDim.x * BLK) >> 5;
  const long long gw = (blockIdx.x * (long long)BLK + threadIdx.x) >> 5;
  seg_body<UK, SQ, EPI, STAGED, false, BLK>(A, S, U, E, out, su, ebuf_all[threadIdx.x >> 5], gw, W,
                                             lane);
}

// Rows split across chunks, finished in the chunk t holding their last entry:
// the partials of chunks first[t] .. t-1 (carry) plus chunk t's own part
// (head).  Lane i of a warp takes chunk 32w + i; spans of up to 16 chunks
// are summed by the lane in order, longer ones (Zipf-hot rows) by the whole
// warp, lane-strided then as a tree.  The order depends on the structure
// only, so results are bit-reproducible.
constexpr int kFixSerial = 16;
template <int EPI, bool COH>
__device__ __forceinline__ void fixup_one(const SegView& S, const EpiView& E,
                                          double* __restrict__ out, long long t, int lane,
                                          DotAcc& dacc) {
  long long f = t < S.nchunks ? __ldg(S.chunk_first + t) : -1;
  if (f >= 0 && t - f > kFixCta) f = -1;  // a CTA of its own finishes it (seg_fixup_kernel)
  const bool longspan = f >= 0 && t - f > kFixSerial;
  if (f >= 0 && !longspan) {
    double s = COH ? ld_coh(S.carry + f) : S.carry[f];
    for (long long v = f + 1; v < t; ++v) s = s + (COH ? ld_coh(S.carry + v) : S.carry[v]);
    const int j = S.nz_col[S.chunk_rank[t] & 0x7fffffffu];
    const double bj = epi_base<EPI, COH>(E, j);
    const double o = epi_apply<EPI>(E, bj, s + (COH ? ld_coh(S.head + t) : S.head[t]));
    out[j] = o;
    if (EPI == EPI_VEC && E.dot_parts) dacc.add(E, bj, o);
  }
  unsigned todo = __ballot_sync(0xffffffffu, longspan);
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    const long long tt = __shfl_sync(0xffffffffu, t, src);
    const long long ff = __shfl_sync(0xffffffffu, f, src);
    double s = 0.0;
#pragma unroll 4
    for (long long v = ff + lane; v < tt; v += 32) s += COH ? ld_coh(S.carry + v) : S.carry[v];
    s = warp_sum(s);  // valid in lane 0
    if (lane == 0) {
      const int j = S.nz_col[S.chunk_rank[tt] & 0x7fffffffu];
      const double bj = epi_base<EPI, COH>(E, j);
      const double o = epi_apply<EPI>(E, bj, s + (COH ? ld_coh(S.head + tt) : S.head[tt]));
      out[j] = o;
      if (EPI == EPI_VEC && E.dot_parts) dacc.add(E, bj, o);
    }
  }
}

// CTAs [0, nreg) take one chunk per thread (fixup_one); CTA nreg + k finishes
// the k-th long span S.long_fix[k] with all its threads (lane-strided sums,
// then the block tree: a fixed order, so results stay bit-reproducible).
template <int EPI>
__global__ void __launch_bounds__(kBlock) seg_fixup_kernel(SegView S, EpiView E,
                                                          double* __restrict__ out, long long Wseg,
                                                          int nreg) {
  pdl_wait();
  pdl_trigger();
  DotAcc dacc;
  if ((int)blockIdx.x < nreg) {
    fixup_one<EPI, false>(S, E, out, blockIdx.x * (long long)kBlock + threadIdx.x, threadIdx.x & 31,
                          dacc);
  } else {
    __shared__ double shl[kBlock / kWarp + 1];
    const long long t = __ldg(S.long_fix + (blockIdx.x - nreg));
    const long long f = __ldg(S.chunk_first + t);
    double s = 0.0;
#pragma unroll 4
    for (long long v = f + threadIdx.x; v < t; v += kBlock) s += S.carry[v];
    s = block_sum<kBlock>(s, shl);  // valid in thread 0
    if (threadIdx.x == 0) {
      const int j = S.nz_col[S.chunk_rank[t] & 0x7fffffffu];
      const double bj = epi_base<EPI, false>(E, j);
      const double o = epi_apply<EPI>(E, bj, s + S.head[t]);
      out[j] = o;
      if (EPI == EPI_VEC && E.dot_parts) dacc.add(E, bj, o);
    }
  }
  if (EPI == EPI_VEC && E.dot_parts) {
    // this CTA's fix-ups, then the last CTA adds every partial in index order:
    // [0, Wseg) the segmented kernel's warps, then the fix-up CTAs
    __shared__ double sh[kBlock / kWarp + 1];
    const double a = block_sum<kBlock>(dacc.acc, sh);
    const double b = block_sum<kBlock>(dacc.bad, sh);
    if (threadIdx.x == 0) {
      E.dot_parts[2 * (Wseg + blockIdx.x)] = a;
      E.dot_parts[2 * (Wseg + blockIdx.x) + 1] = b;
    }
    if (last_block_arrive(E.dot_ticket)) {
      const int cnt = (int)(Wseg + gridDim.x);
      const double tot = reduce_partials<kBlock>(E.dot_parts, cnt, 2, 0, sh);
      const double nb = reduce_partials<kBlock>(E.dot_parts, cnt, 2, 1, sh);
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
}

template <int UK, bool SQ, int EPI, bool STAGED>
void launch_one(const CsrView& A, const SegView& S, const UView& U, const EpiView& E, double* out,
                cudaStream_t s) {
  constexpr int BLK = STAGED ? kStagedBlock : kBlock;
  size_t smem = 0;
  long long cap = device_sm_count();
  if (STAGED) {
    smem = (size_t)A.cols * sizeof(double);
    ensure_max_dynamic_smem((const void*)seg_spmv_kernel<UK, SQ, EPI, true>, (int)kStageMaxBytes);
  } else {
    cap *= kSegBlocksPerSm;  // persistent: blocks of 8 warps per SM (register-limited)
  }
  // never more warps than chunks or visits of the empty list
  const long long warps =
      std::max<long long>(S.nchunks, (S.nempty + 32 * kEmptyItems - 1) / (32 * kEmptyItems));
  long long grid = (warps * 32 + BLK - 1) / BLK;
  if (grid > cap) grid = cap;
  launch_pdl(seg_spmv_kernel<UK, SQ, EPI, STAGED>, dim3((int)grid), dim3(BLK), smem, s, A, S, U, E,
             out);
  // the fix-up kernel also finishes E.dot_out, so it always runs when asked to
  int nreg = (int)((S.nchunks + kBlock - 1) / kBlock);
  if (E.dot_parts && nreg == 0) nreg = 1;
  const int fgrid = nreg + (int)S.nlong;
  const long long Wseg = grid * (BLK / 32);
  if (fgrid)
    launch_pdl(seg_fixup_kernel<EPI>, dim3(fgrid), dim3(kBlock), 0, s, S, E, out, Wseg, nreg);
}

template <int UK, bool SQ, int EPI>
void launch_epi(const CsrView& A, const SegView& S, const UView& U, const EpiView& E, double* out,
                cudaStream_t s) {
  // u staged in shared memory when it fits (TRON_B200_STAGE=0 disables)
  static const bool stage_on = [] {
    const char* e = std::getenv("TRON_B200_STAGE");
    return !(e && e[0] == '0');
  }();
  // ... and when it pays: each staged u_r must serve enough nonzeros to cover
  // the per-SM copy (R1, 74 per row: no; N1, 450: yes)
  if (stage_on && (long long)A.cols * (long long)sizeof(double) <= kStageMaxBytes &&
      A.nnz >= 128 * A.cols)
    launch_one<UK, SQ, EPI, true>(A, S, U, E, out, s);
  else
    launch_one<UK, SQ, EPI, false>(A, S, U, E, out, s);
}

template <int UK, bool SQ>
void launch_seg(const CsrView& A, const SegView& S, const UView& U, const EpiView& E, double* out,
                cudaStream_t s) {
  switch (E.kind) {
    case EPI_VEC:
      launch_epi<UK, SQ, EPI_VEC>(A, S, U, E, out, s);
      break;
    case EPI_CONST:
      launch_epi<UK, SQ, EPI_CONST>(A, S, U, E, out, s);
      break;
    default:
      launch_epi<UK, SQ, EPI_RAW>(A, S, U, E, out, s);
      break;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// Device-built plan with fixed 256-entry chunks (every boundary inside a
// row becomes a fix-up): fully parallel, no host round trip of the CSC
// structure.
// ---------------------------------------------------------------------------
namespace {

__global__ void plan_cols_kernel(const int32_t* cptr, long long n, uint32_t* lastbits,
                                 int32_t* nonempty, int32_t* ids, uint8_t* empty) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    const int b = cptr[c], e = cptr[c + 1];
    ids[c] = (int32_t)c;
    nonempty[c] = e > b;
    empty[c] = e <= b;
    if (e > b) atomicOr(lastbits + ((e - 1) >> 5), 1u << ((e - 1) & 31));
  }
}

__global__ void plan_chunk_rank_kernel(const int32_t* cptr, long long n, const int32_t* colrank,
                                       long long nchunks, uint32_t* rank, int32_t* first) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nchunks;
       t += (long long)gridDim.x * blockDim.x) {
    const long long x = t * kSegChunk;
    long long lo = 0, hi = n + 1;  // upper_bound(cptr[0..n], x) - 1
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (cptr[mid] <= x)
        lo = mid + 1;
      else
        hi = mid;
    }
    const long long c = lo - 1;
    const bool cont = cptr[c] < x;
    rank[t] = (uint32_t)colrank[c] | (cont ? 0x80000000u : 0u);
    // fix-up of the row continued into chunk t when it also ends there
    first[t] = cont && cptr[c + 1] <= x + kSegChunk ? (int32_t)(cptr[c] / kSegChunk) : -1;
  }
}

__global__ void plan_long_flags_kernel(const int32_t* first, long long nchunks, uint8_t* flag) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nchunks;
       t += (long long)gridDim.x * blockDim.x)
    flag[t] = first[t] >= 0 && t - first[t] > kFixCta;
}

__global__ void plan_sentinel_kernel(int32_t* nz_col, const int32_t* colrank, long long n) {
  nz_col[colrank[n]] = (int32_t)n;
}

int pgrid(long long n) {
  long long g = (n + 255) / 256;
  const long long cap = (long long)device_sm_count() * 16;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

}  // namespace

int seg_plan_device(const int32_t* cptr, int64_t n, int64_t nnz, SegView* P, uint32_t* chunk_rank,
                    int32_t* chunk_first, uint32_t* lastbits, int32_t* nz_col, int32_t* empty_col,
                    int32_t* long_fix, cudaStream_t s) {
  const int64_t nchunks = (nnz + kSegChunk - 1) / kSegChunk;
  const size_t n1 = n > 0 ? n : 1;
  int32_t *nonempty = nullptr, *colrank = nullptr, *ids = nullptr;
  uint8_t* empty = nullptr;
  long long* cnt = nullptr;  // [0] non-empty rows, [1] empty rows, [2] long fix-ups
  uint8_t* lflag = nullptr;
  void* temp = nullptr;
  size_t tb1 = 0, tb2 = 0, tb3 = 0, tb4 = 0;
  const int64_t nch1 = nchunks > 0 ? nchunks : 1;
  cudaError_t e = cudaMallocAsync(&nonempty, (n1 + 1) * sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&colrank, (n1 + 1) * sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&ids, n1 * sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&empty, n1, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&cnt, 3 * sizeof(long long), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&lflag, nch1, s);
  thrust::counting_iterator<int32_t> chunk_ids(0);
  if (e == cudaSuccess)
    e = cub::DeviceSelect::Flagged(nullptr, tb4, chunk_ids, lflag, long_fix, cnt + 2, (int)nch1, s);
  if (e == cudaSuccess)
    e = cub::DeviceScan::ExclusiveSum(nullptr, tb1, nonempty, colrank, (int)(n + 1), s);
  if (e == cudaSuccess)
    e = cub::DeviceSelect::Flagged(nullptr, tb2, ids, nonempty, nz_col, cnt, (int)n, s);
  if (e == cudaSuccess)
    e = cub::DeviceSelect::Flagged(nullptr, tb3, ids, empty, empty_col, cnt + 1, (int)n, s);
  if (e == cudaSuccess)
    e = cudaMallocAsync(&temp, std::max<size_t>(std::max(std::max(tb1, tb4), std::max(tb2, tb3)), 1), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(nonempty, 0, (n1 + 1) * sizeof(int32_t), s);
  if (e == cudaSuccess)
    e = cudaMemsetAsync(lastbits, 0, (size_t)(nchunks * (kSegChunk / 32) + 2) * sizeof(uint32_t), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, 3 * sizeof(long long), s);
  if (e == cudaSuccess) {
    if (n > 0) plan_cols_kernel<<<pgrid(n), 256, 0, s>>>(cptr, n, lastbits, nonempty, ids, empty);
    e = cub::DeviceScan::ExclusiveSum(temp, tb1, nonempty, colrank, (int)(n + 1), s);
  }
  if (e == cudaSuccess && n > 0)
    e = cub::DeviceSelect::Flagged(temp, tb2, ids, nonempty, nz_col, cnt, (int)n, s);
  if (e == cudaSuccess && n > 0)
    e = cub::DeviceSelect::Flagged(temp, tb3, ids, empty, empty_col, cnt + 1, (int)n, s);
  if (e == cudaSuccess) {
    plan_sentinel_kernel<<<1, 1, 0, s>>>(nz_col, colrank, n);
    if (nchunks > 0) {
      plan_chunk_rank_kernel<<<pgrid(nchunks), 256, 0, s>>>(cptr, n, colrank, nchunks, chunk_rank,
                                                            chunk_first);
      plan_long_flags_kernel<<<pgrid(nchunks), 256, 0, s>>>(chunk_first, nchunks, lflag);
      e = cub::DeviceSelect::Flagged(temp, tb4, chunk_ids, lflag, long_fix, cnt + 2, (int)nchunks, s);
    }
  }
  long long counts[3] = {0, 0, 0};
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(counts, cnt, sizeof(counts), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  for (void* p : {(void*)nonempty, (void*)colrank, (void*)ids, (void*)empty, (void*)cnt, (void*)lflag, temp})
    if (p) cudaFreeAsync(p, s);
  if (e == cudaSuccess) e = cudaGetLastError();
  P->nchunks = nchunks;
  P->nnzc = counts[0];
  P->nempty = counts[1];
  P->chunk_rank = chunk_rank;
  P->chunk_first = chunk_first;
  P->lastbits = lastbits;
  P->nz_col = nz_col;
  P->empty_col = empty_col;
  P->long_fix = long_fix;
  P->nlong = counts[2];
  return e == cudaSuccess ? 0 : (int)e;
}

int64_t seg_dot_slots(int64_t nchunks) {
  // doubles: 2 per slot; segmented warps (16 per SM in either variant) + fix-up CTAs
  return 2 * ((int64_t)device_sm_count() * 16 + (nchunks + kBlock - 1) / kBlock + 1 +
              seg_long_fix_cap(nchunks));
}

void csc_spmv(const CsrView& At, const SegView& S, const UView& U, bool squared,
              const EpiView& E, double* out, cudaStream_t s) {
  if (S.nchunks <= 0) {  // no nonzeros: every column is empty
    if (At.rows > 0) vec_epilogue(At.rows, nullptr, E, out, s);
    return;
  }
  if (U.kind == U_VEC) {
    if (squared)
      launch_seg<U_VEC, true>(At, S, U, E, out, s);
    else
      launch_seg<U_VEC, false>(At, S, U, E, out, s);
  } else if (U.kind == U_SVM_RESID) {
    launch_seg<U_SVM_RESID, false>(At, S, U, E, out, s);
  } else {
    launch_seg<U_MASK, true>(At, S, U, E, out, s);
  }
}

}  // namespace tb
