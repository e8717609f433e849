// Streamed segmented SpMV over a compressed matrix (CSR: segments = rows,
// CSC: segments = columns), FP64, sm_100a.
//
// One kernel computes   out_s = epilogue_s( sum_{k in segment s} val_k * g(idx_k) )
// for every segment s, where g gathers from a dense vector (w, p, u, ...)
// and the epilogue is the fused per-row / per-column tail of the hot path:
//   * CSR forward  (logistic_fused_pass / svm_fused_pass, loss.cpp:35-122)
//   * CSR D-scaled row products of the Hessian product (loss.cpp:85-89)
//   * CSC transposed products X^T u with base + scale * sum epilogues
//     (matvec_transpose, masked_matvec_transpose, *_sq_col_sums,
//      linalg.cpp:175-265; gradient / Hv / preconditioner, loss.cpp:74-188)
//
// Layout (built once per matrix on the device, seg_stream_build):
//   * the nonzeros are cut into 2048-entry tiles of eight 256-entry pieces
//     (one warp: 32 lanes x 8 consecutive entries), stored lane-interleaved
//     inside each piece (entry (lane L, item m) at m*32 + L), so a warp's
//     shared-memory reads are conflict-free and its 8 items per lane stay in
//     logical order;
//   * one byte per lane marks which of its 8 entries end a segment;
//   * each tile is one contiguous record -- values, indices, end bytes and
//     the ids of the segments the tile ends, in order -- so a tile arrives
//     with a single bulk copy and knows its segment ids without touching the
//     offsets array.

// Kernel: a persistent CTA owns a contiguous range of tiles.  One producer
// warp streams each tile record into a 4-stage shared-memory ring with TMA
// bulk copies; 16
// compute warps (two groups of 8 alternating tiles, one piece per warp)
// gather, multiply and reduce, and one combiner warp finishes the tile:
//   * each lane sums its 8 items sequentially; a warp segmented scan joins
//     segments that cross lanes;
//   * a combiner warp joins segments that cross pieces and tiles: each
//     compute warp hands it a record per piece (head partial, trailing
//     partial, whether the piece ends a segment) through shared memory, and
//     it walks the CTA's tiles in order with a running carry (a segmented
//     scan over the 8 pieces of a tile), emitting the pieces' head segments
//     before releasing the stage to the producer;
//   * a segment that crosses into an earlier CTA's range is handed to the
//     last CTA to finish (ticket), which completes it over the per-CTA
//     records -- so one launch does the whole product.
// No atomics on floating-point data, fixed reduction orders throughout:
// repeated runs are bit-identical.
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "common.cuh"
#include "kernels.h"

#include <cstdlib>

namespace tb {

namespace {

constexpr int kPiece = 256;
constexpr int kTileEntries = kPiece * kStreamTilePieces;  // 2048
#ifndef TB_STREAM_GROUPS
#define TB_STREAM_GROUPS 2
#endif
constexpr int kGroups = TB_STREAM_GROUPS;
constexpr int kComputeWarps = kStreamTilePieces * kGroups;
constexpr int kProducerWarp = kComputeWarps;
constexpr int kCombinerWarp = kComputeWarps + 1;
constexpr int kThreads = (kComputeWarps + 2) * kWarp;
// Tile record: [val 16 KB | idx 8 KB | end bytes 256 B | ids of the segments
// the tile ends, in order (4 B each, padded to 16 B)] -- one TMA bulk copy
// per tile (copies under ~16 KB cost throughput: scripts/tma_probe.cu).
constexpr int kValBytes = kTileEntries * 8;
constexpr int kIdxBytes = kTileEntries * 4;
constexpr int kEndBytes = kStreamTilePieces * 32;
constexpr int kRecHead = kValBytes + kIdxBytes + kEndBytes;  // 24,832
constexpr int kStageBytes = kRecHead + kTileEntries * 4;      // 33,024 (a tile ends <= 2048)
constexpr int kMaxOffSmem = 1024;

__device__ __forceinline__ double log1p_exp_neg(double t) {  // loss.hpp:99-102
  if (t >= 0.0) return log1p(exp(-t));
  return -t + log1p(exp(t));
}

// ---------------------------------------------------------------------------
// epilogue / gather operators
//   gather(idx)       the dense-vector operand of one stored entry
//   product(v, x)     its contribution to the segment sum
//   aux(seg)          the segment's epilogue operand (base_j, y_i, D_i ...),
//                     loaded ahead of the sum so stores never wait on it
//   store(seg, s, a)  the epilogue
// ---------------------------------------------------------------------------
struct OpBase {
  __device__ __forceinline__ void block_finish(double*) {}
  __device__ __forceinline__ void finalize(double*) {}
};

// X^T u over the CSC stream (segments = columns)
template <int UK, bool SQ, int EPI>
struct TransOp : OpBase {
  UView U;
  EpiView E;
  double* out;
  __device__ __forceinline__ double gather(int r) const {
    if (UK == U_VEC) return __ldg(U.u + r);
    if (UK == U_SVM_RESID) return U.mask[r] ? (U.z[r] - U.y[r]) : 0.0;
    return U.mask[r] ? 1.0 : 0.0;
  }
  // row_axpy: out += a*v ; row_axpy_squared: out += a*v*v  (linalg.cpp:88-109)
  __device__ __forceinline__ double product(double v, double x) const {
    return SQ ? (x * v) * v : x * v;
  }
  __device__ __forceinline__ double aux(long long j) const {
    return EPI == EPI_VEC ? __ldg(E.base + j) : 0.0;
  }
  __device__ __forceinline__ void store(long long j, double sum, double a) {
    if (EPI == EPI_VEC)
      out[j] = a + E.scale * sum;
    else if (EPI == EPI_CONST)
      out[j] = E.cbase + E.scale * sum;
    else
      out[j] = sum;
  }
};

// D-scaled row products of the CSR stream: a_i = (x_i . p) * D_i, or
// [i in I] (x_i . p) for the SVM indirect Hessian (loss.cpp:85-89, :139-174)
struct DvOp : OpBase {
  const double* p;
  const double* dvec;
  const uint8_t* mask;
  double* a;
  __device__ __forceinline__ double gather(int j) const { return __ldg(p + j); }
  __device__ __forceinline__ double product(double v, double x) const { return v * x; }
  __device__ __forceinline__ double aux(long long i) const {
    return mask ? (double)mask[i] : __ldg(dvec + i);
  }
  __device__ __forceinline__ void store(long long i, double s, double d) {
    a[i] = mask ? (d != 0.0 ? s : 0.0) : s * d;
  }
};

// Fused margin pass over the CSR stream (logistic_fused_pass loss.cpp:35-58,
// svm_fused_pass :94-122); f = 0.5*ww + C*sum finished by the last CTA.
template <int LOSS>
struct FwdOp : OpBase {
  const double* w;
  const double* y;
  double C;
  double* z;
  double* zhat;
  double* dvec;
  uint8_t* mask;
  ObjScalars* obj;
  Scratch sc;
  double term = 0.0, cnt = 0.0;
  __device__ __forceinline__ double gather(int j) const { return __ldg(w + j); }
  __device__ __forceinline__ double product(double v, double x) const { return v * x; }
  __device__ __forceinline__ double aux(long long i) const { return __ldg(y + i); }
  __device__ __forceinline__ void store(long long i, double s, double yi) {
    z[i] = s;
    if (LOSS == kLossLogistic) {
      const double t = yi * s;
      const double sig = 1.0 / (1.0 + exp(t));  // exp overflow -> inf -> 0
      zhat[i] = -yi * sig;
      dvec[i] = (1.0 - sig) * sig;
      term += log1p_exp_neg(t);
    } else {
      const double margin = 1.0 - yi * s;
      if (margin > 0.0) {
        mask[i] = 1;
        term += margin * margin;
        cnt += 1.0;
      } else {
        mask[i] = 0;
      }
    }
  }
  __device__ __forceinline__ void block_finish(double* sh) {
    const double bt = block_sum<kThreads>(term, sh, true);
    const double bc = block_sum<kThreads>(cnt, sh, true);
    if (threadIdx.x == 0) {
      sc.partials[2 * blockIdx.x] = bt;
      sc.partials[2 * blockIdx.x + 1] = bc;
    }
    term = cnt = 0.0;  // published; the last CTA's own tail emits start from zero
  }
  __device__ __forceinline__ void finalize(double* sh) {
    const double et = block_sum<kThreads>(term, sh, true);
    const double ec = block_sum<kThreads>(cnt, sh, true);
    const double tot = reduce_partials<kThreads>(sc.partials, gridDim.x, 2, 0, sh) + et;
    const double nct = reduce_partials<kThreads>(sc.partials, gridDim.x, 2, 1, sh) + ec;
    if (threadIdx.x == 0) {
      obj->f = 0.5 * obj->ww + C * tot;  // loss.cpp:57 / :121
      obj->nact = (long long)nct;
      obj->red[0] = tot;
      obj->red[1] = nct;
    }
  }
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Per-piece hand-off from a compute warp to the combiner warp.
struct PieceRec {
  double head;      // partial of the piece's head segment (entries up to its first end)
  double trailing;  // partial after the piece's last end (the whole piece if it has none)
  double aux;       // the head segment's epilogue operand
  int seg;          // the head segment
  int has_end;
};

// DBG (profiling experiments only, TRON_B200_STREAM_DEBUG): 1 = no gathers,
// 2 = compute warps only consume the stage (results are wrong in both).
template <class Op, int DBG, int kStages>
__global__ void __launch_bounds__(kThreads, 1) seg_stream_kernel(StreamView A, Op op) {
  extern __shared__ __align__(128) unsigned char smem[];
  // full: producer -> compute (TMA bytes); empty: compute -> producer (the
  // stage is read into registers); done / rfree: compute <-> combiner (records)
  __shared__ __align__(8) unsigned long long full[kStages], empty[kStages], done[kStages],
      rfree[kStages];
  __shared__ PieceRec rec[kStages][kStreamTilePieces];
  __shared__ long long s_off[kMaxOffSmem + 1];
  __shared__ double sh[kThreads / kWarp + 1];
  __shared__ unsigned s_epoch;
  __shared__ bool s_last;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const long long t0 = A.ntiles * blockIdx.x / gridDim.x;
  const long long t1 = A.ntiles * (blockIdx.x + 1) / gridDim.x;
  const int ntl = (int)(t1 - t0);
  const bool off_in_smem = ntl <= kMaxOffSmem;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kStreamTilePieces);
      mbar_init(&done[s], kStreamTilePieces);
      mbar_init(&rfree[s], 1);
    }
    mbar_fence_init();
    s_epoch = *reinterpret_cast<volatile unsigned*>(A.epoch);
  }
  if (off_in_smem)
    for (int k = tid; k <= ntl; k += kThreads) s_off[k] = A.tile_off[t0 + k];
  __syncthreads();
  const unsigned tag = s_epoch + 1u;  // this launch's record tag
  auto off_of = [&](long long t) -> long long {
    return off_in_smem ? s_off[t - t0] : __ldg(A.tile_off + t);
  };

  if (wid == kProducerWarp) {
    // ---------------- producer: one lane streams the CTA's tiles
    if (lane == 0) {
      for (int k = 0; k < ntl; ++k) {
        const int s = k % kStages;
        if (k >= kStages) mbar_wait_parity(&empty[s], (unsigned)(((k / kStages) - 1) & 1));
        const long long t = t0 + k;
        const long long o0 = off_of(t);
        const unsigned bytes = (unsigned)(off_of(t + 1) - o0);
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(smem + (size_t)s * kStageBytes, A.rec + o0, bytes, &full[s]);
      }
    }
  } else if (wid == kCombinerWarp) {
    // ---------------- combiner: joins segments across the tile's pieces and
    // across tiles (in order), stores the pieces' head segments, frees stages
    double carry = 0.0;    // partial of the segment open at the current position
    bool any_end = false;  // a segment ended in this CTA's range so far
    int pend_seg = -1;     // the CTA's first segment end, when its segment began in an
    double pend_val = 0.0, pend_aux = 0.0;  // earlier CTA's range
    const bool mine = lane < kStreamTilePieces;
    const int q = mine ? lane : kStreamTilePieces - 1;
    for (int k = 0; k < ntl; ++k) {
      const int s = k % kStages;
      mbar_wait_parity(&done[s], (unsigned)((k / kStages) & 1));
      const PieceRec r = rec[s][q];
      const int has = mine ? r.has_end : 0;
      // inclusive segmented scan over the pieces: (sum of trailings since the
      // last piece with an end, any end so far)
      double a = mine ? r.trailing : 0.0;
      int f = has;
#pragma unroll
      for (int off = 1; off < kStreamTilePieces; off <<= 1) {
        const double a2 = __shfl_up_sync(0xffffffffu, a, off);
        const int f2 = __shfl_up_sync(0xffffffffu, f, off);
        if (lane >= off && !f) a = a2 + a;
        if (lane >= off) f |= f2;
      }
      const double cout = f ? a : carry + a;  // carry out of each piece
      double cin = __shfl_up_sync(0xffffffffu, cout, 1);
      int fin = __shfl_up_sync(0xffffffffu, f, 1);  // an end earlier in the tile
      if (lane == 0) {
        cin = carry;
        fin = 0;
      }
      const double tot = cin + r.head;
      const bool hand_off = has && !(t0 == 0 || any_end || fin);
      if (has && !hand_off) op.store(r.seg, tot, r.aux);
      const unsigned hb = __ballot_sync(0xffffffffu, hand_off);
      if (hb) {
        pend_seg = __shfl_sync(0xffffffffu, r.seg, __ffs(hb) - 1);
        pend_val = __shfl_sync(0xffffffffu, tot, __ffs(hb) - 1);
        pend_aux = __shfl_sync(0xffffffffu, r.aux, __ffs(hb) - 1);
      }
      carry = __shfl_sync(0xffffffffu, cout, kStreamTilePieces - 1);
      any_end = any_end || __shfl_sync(0xffffffffu, f, kStreamTilePieces - 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(&rfree[s]);
    }
    if (lane == 0) {
      // publish this range's record, then finish the hand-off from the
      // records of the earlier ranges (they publish before they wait)
      A.cta_tail[blockIdx.x] = carry;
      A.cta_flags[blockIdx.x] = any_end ? 1 : 0;
      st_release(A.cta_tag + blockIdx.x, tag);
      if (pend_seg >= 0) {
        double before = 0.0;  // tails of the earlier ranges back to one with an end
        for (int c = (int)blockIdx.x - 1; c >= 0; --c) {
          while (ld_acquire(A.cta_tag + c) != tag) {
          }
          before += __ldcg(A.cta_tail + c);
          if (__ldcg(A.cta_flags + c) & 1) break;
        }
        op.store(pend_seg, before + pend_val, pend_aux);
      }
    }
  } else {
    // ---------------- compute warps: group g takes tiles k = g, g+2, ...; warp q one piece
    const int g = wid / kStreamTilePieces, q = wid % kStreamTilePieces;
    // empty segments (sum 0): this CTA's share of their list, 32 per warp per
    // iteration, their loads in flight with the gathers
    const long long ne = *A.nempty;
    const long long e1 = ne * (blockIdx.x + 1) / gridDim.x;
    long long ec = ne * blockIdx.x / gridDim.x + (long long)wid * 32;
    auto empties_issue = [&](int& es, double& ea) {
      const long long ei = ec + lane;
      es = -1;
      if (ei < e1) {
        es = __ldg(A.empty_seg + ei);
        ea = op.aux(es);
      }
    };
    auto empties_store = [&](int es, double ea) {
      if (es >= 0) op.store(es, 0.0, ea);
      ec += kComputeWarps * 32;
    };
    for (int k = g; k < ntl; k += kGroups) {
      const int s = k % kStages;
      mbar_wait_parity(&full[s], (unsigned)((k / kStages) & 1));
      const unsigned char* st = smem + (size_t)s * kStageBytes;
      const double* sv = reinterpret_cast<const double*>(st) + q * kPiece;
      const int* si = reinterpret_cast<const int*>(st + kValBytes) + q * kPiece;
      const uint8_t* se = st + kValBytes + kIdxBytes;
      const int32_t* sids = reinterpret_cast<const int32_t*>(st + kRecHead);

      double v[8];
      int ix[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        v[m] = sv[m * 32 + lane];
        ix[m] = si[m * 32 + lane];
      }
      const unsigned eb = se[q * 32 + lane];
      // rank of the first end of this piece: ends in earlier pieces of the tile
      int pc = 0;
      if (lane < kStreamTilePieces) {
        const unsigned long long* e64 = reinterpret_cast<const unsigned long long*>(se + lane * 32);
        pc = __popcll(e64[0]) + __popcll(e64[1]) + __popcll(e64[2]) + __popcll(e64[3]);
      }
      int pincl = pc;
#pragma unroll
      for (int off = 1; off < kStreamTilePieces; off <<= 1) {
        const int y2 = __shfl_up_sync(0xffffffffu, pincl, off);
        if (lane >= off) pincl += y2;
      }
      // index (among the tile's ends) of this piece's first end
      const int piece_rank = __shfl_sync(0xffffffffu, pincl - pc, q);
      const int cnt = __popc(eb);
      int incl = cnt;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y2 = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y2;
      }
      const int excl = incl - cnt;
      // the segments this lane ends and their epilogue operands: issued
      // together with the gathers
      int sg[8];
      double ax[8];
      {
        int rr = piece_rank + excl;
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          if (eb & (1u << m)) {
            sg[m] = sids[rr];
            ax[m] = op.aux(sg[m]);
            ++rr;
          } else {
            sg[m] = 0;
            ax[m] = 0.0;
          }
        }
      }
      // everything this warp needs from the stage is in registers: release it,
      // so the producer refills it while the gathers are in flight
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (DBG == 2) {
        if (lane == 0) {
          if (k >= kStages) mbar_wait_parity(&rfree[s], (unsigned)(((k / kStages) - 1) & 1));
          rec[s][q].has_end = 0;
          rec[s][q].trailing = v[0] + ax[0];
          mbar_arrive(&done[s]);
        }
        continue;
      }
      double x[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) x[m] = DBG == 1 ? (double)ix[m] : op.gather(ix[m]);
      int es;
      double ea = 0.0;
      empties_issue(es, ea);

      // lane: sequential sum of its 8 items
      double acc = 0.0, head = 0.0, hax = 0.0;
      int hseg = 0;
      bool have_head = false;
#pragma unroll
      for (int m = 0; m < 8; ++m) {
        acc += op.product(v[m], x[m]);
        if (eb & (1u << m)) {
          if (!have_head) {
            head = acc;
            hseg = sg[m], hax = ax[m];
            have_head = true;
          } else {
            op.store(sg[m], acc, ax[m]);  // segment wholly inside this lane
          }
          acc = 0.0;
        }
      }
      // warp segmented inclusive scan of the lane carries, keyed by end count
      double val = acc;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int k2 = __shfl_up_sync(0xffffffffu, incl, off);
        const double v2 = __shfl_up_sync(0xffffffffu, val, off);
        if (lane >= off && k2 == incl) val = v2 + val;
      }
      const int prev_key = __shfl_up_sync(0xffffffffu, incl, 1);
      const double prev_val = __shfl_up_sync(0xffffffffu, val, 1);
      double hpart = 0.0;
      if (have_head) {
        const double tot = (lane > 0 && prev_key == excl) ? prev_val + head : head;
        if (excl > 0)
          op.store(hseg, tot, hax);
        else
          hpart = tot;  // the piece's head segment: joined by the combiner
      }
      const int tot_ends = __shfl_sync(0xffffffffu, incl, 31);
      const double trailing = __shfl_sync(0xffffffffu, val, 31);
      const unsigned hb = __ballot_sync(0xffffffffu, have_head && excl == 0);
      const int hl = hb ? __ffs(hb) - 1 : 0;
      const double hp = __shfl_sync(0xffffffffu, hpart, hl);
      const double ha = __shfl_sync(0xffffffffu, hax, hl);
      const int hs = __shfl_sync(0xffffffffu, hseg, hl);
      if (lane == 0) {
        if (k >= kStages) mbar_wait_parity(&rfree[s], (unsigned)(((k / kStages) - 1) & 1));
        PieceRec& pr = rec[s][q];
        pr.head = hp;
        pr.trailing = trailing;
        pr.aux = ha;
        pr.seg = hs;
        pr.has_end = tot_ends > 0;
        mbar_arrive(&done[s]);  // release: the combiner reads the record after its wait
      }
      empties_store(es, ea);
    }
    while (DBG != 2 && ec < e1) {
      int es;
      double ea = 0.0;
      empties_issue(es, ea);
      empties_store(es, ea);
    }
  }
  __syncthreads();
  op.block_finish(sh);
  if (tid == 0) {
    __threadfence();
    const unsigned tk = atomicAdd(A.ticket, 1u);
    s_last = tk == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // ---------------- last CTA: the op's finish
  op.finalize(sh);
  if (tid == 0) {
    *A.ticket = 0u;
    *reinterpret_cast<volatile unsigned*>(A.epoch) = tag;
  }
}

template <class Op, int DBG, int NS>
void launch_stream_dbg(const StreamView& A, const Op& op, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(seg_stream_kernel<Op, DBG, NS>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, NS * kStageBytes);
    configured = true;
  }
  seg_stream_kernel<Op, DBG, NS><<<seg_stream_grid(A.ntiles), kThreads, NS * kStageBytes, s>>>(A, op);
}

template <class Op, int NS>
void launch_stream_ns(int dbg, const StreamView& A, const Op& op, cudaStream_t s) {
  if (dbg == 1)
    launch_stream_dbg<Op, 1, NS>(A, op, s);
  else if (dbg == 2)
    launch_stream_dbg<Op, 2, NS>(A, op, s);
  else
    launch_stream_dbg<Op, 0, NS>(A, op, s);
}

template <class Op>
void launch_stream(const StreamView& A, const Op& op, cudaStream_t s) {
  static const int dbg = [] {
    const char* e = std::getenv("TRON_B200_STREAM_DEBUG");
    return e ? std::atoi(e) : 0;
  }();
  static const int stages = [] {
    const char* e = std::getenv("TRON_B200_STREAM_STAGES");
    return e ? std::atoi(e) : 4;
  }();
  if (stages >= 6)
    launch_stream_ns<Op, 6>(dbg, A, op, s);
  else
    launch_stream_ns<Op, 4>(dbg, A, op, s);
}

// ---------------------------------------------------------------------------
// layout construction (all on the device; once per matrix)
// ---------------------------------------------------------------------------
__device__ __forceinline__ long long phys_pos(long long within_tile) {
  const int p = (int)(within_tile >> 8), w = (int)(within_tile & 255), L = w >> 3, m = w & 7;
  return (long long)p * kPiece + m * 32 + L;
}

__global__ void nonempty_flags_kernel(const int32_t* ptr, long long nseg, int32_t* ne,
                                      uint8_t* empty) {
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < nseg;
       s += (long long)gridDim.x * blockDim.x) {
    const bool f = ptr[s + 1] > ptr[s];
    ne[s] = f;
    empty[s] = !f;
  }
}

__global__ void iota_kernel(int32_t* v, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

// end bit of every non-empty segment (byte = piece*32 + lane, bit = item)
__global__ void mark_ends_kernel(const int32_t* ptr, long long nseg, unsigned* ends32) {
  for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < nseg;
       s += (long long)gridDim.x * blockDim.x) {
    if (ptr[s + 1] <= ptr[s]) continue;
    const long long last = ptr[s + 1] - 1;
    const long long byte = (last >> 8) * 32 + ((last & 255) >> 3);
    atomicOr(ends32 + (byte >> 2), 1u << (8 * (byte & 3) + (last & 7)));
  }
}

// ends per tile (popcount of its 256 end bytes) and the tile's record size
__global__ void tile_count_kernel(const unsigned long long* ends64, long long ntiles, int32_t* cnt,
                                  long long* rsz) {
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long t = gw; t < ntiles; t += nw) {
    int c = __popcll(ends64[t * 32 + lane]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if (lane == 0) {
      cnt[t] = c;
      rsz[t] = kRecHead + ((c * 4 + 15) & ~15);
    }
  }
}

// one warp per segment: values and indices into their tile records (lane-
// interleaved), and the segment id into its tile's list of ended segments
__global__ void pack_kernel(const int32_t* __restrict__ ptr, long long nseg,
                            const int32_t* __restrict__ idx, const double* __restrict__ val,
                            const int32_t* __restrict__ seg_rank,
                            const int32_t* __restrict__ tile_rank,
                            const long long* __restrict__ off, unsigned char* __restrict__ rec) {
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long sgm = gw; sgm < nseg; sgm += nw) {
    const int b = ptr[sgm], e = ptr[sgm + 1];
    for (int k = b + lane; k < e; k += 32) {
      const long long t = k / kTileEntries;
      unsigned char* r = rec + off[t];
      const long long ph = phys_pos(k - t * kTileEntries);
      reinterpret_cast<double*>(r)[ph] = val[k];
      reinterpret_cast<int32_t*>(r + kValBytes)[ph] = idx[k];
    }
    if (lane == 0 && e > b) {
      const long long t = (long long)(e - 1) / kTileEntries;
      reinterpret_cast<int32_t*>(rec + off[t] + kRecHead)[seg_rank[sgm] - tile_rank[t]] =
          (int32_t)sgm;
    }
  }
}

__global__ void copy_ends_kernel(const unsigned long long* ends64, long long ntiles,
                                 const long long* off, unsigned char* rec) {
  const long long gw = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long t = gw; t < ntiles; t += nw)
    reinterpret_cast<unsigned long long*>(rec + off[t] + kValBytes + kIdxBytes)[lane] =
        ends64[t * 32 + lane];
}

int grid_for(long long n, int block = 256) {
  long long g = (n + block - 1) / block;
  const long long cap = (long long)device_sm_count() * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace

int seg_stream_grid(int64_t ntiles) {
  int64_t g = ntiles < device_sm_count() ? ntiles : device_sm_count();
  return (int)(g < 1 ? 1 : g);
}

size_t seg_stream_sizes(int64_t nseg, int64_t nnz, SegStreamSizes* z) {
  z->ntiles = (nnz + kTileEntries - 1) / kTileEntries;
  // records: fixed head per tile + the ended segments' ids (<= nseg) + padding
  z->rec_bytes = z->ntiles * (int64_t)kRecHead + 4 * nseg + 16 * z->ntiles;
  return 0;
}

int seg_stream_build(const int32_t* ptr, int64_t nseg, int64_t nnz, const int32_t* idx,
                     const double* val, const StreamView& A, cudaStream_t s) {
  const int64_t ntiles = A.ntiles;
  SegStreamSizes z;
  seg_stream_sizes(nseg, nnz, &z);
  // temporaries
  int32_t *nonempty = nullptr, *seg_rank = nullptr, *ids = nullptr, *tcount = nullptr,
          *tile_rank = nullptr;
  uint8_t* eflags = nullptr;
  unsigned long long* ends = nullptr;
  long long* rsz = nullptr;
  void* temp = nullptr;
  size_t tb1 = 0, tb2 = 0, tb3 = 0, tb4 = 0;
  const size_t ns1 = nseg > 0 ? nseg : 1;
  cudaError_t e = cudaMallocAsync(&nonempty, (ns1 + 1) * sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&seg_rank, (ns1 + 1) * sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&ids, ns1 * sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&eflags, ns1, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&ends, (ntiles > 0 ? ntiles : 1) * kEndBytes, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&tcount, (ntiles + 1) * sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&tile_rank, (ntiles + 1) * sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&rsz, (ntiles + 1) * sizeof(long long), s);
  if (e == cudaSuccess)
    e = cub::DeviceScan::ExclusiveSum(nullptr, tb1, nonempty, seg_rank, (int)(nseg + 1), s);
  if (e == cudaSuccess)
    e = cub::DeviceSelect::Flagged(nullptr, tb2, ids, eflags, const_cast<int32_t*>(A.empty_seg),
                                   A.nempty, (int)nseg, s);
  if (e == cudaSuccess)
    e = cub::DeviceScan::ExclusiveSum(nullptr, tb3, tcount, tile_rank, (int)(ntiles + 1), s);
  if (e == cudaSuccess)
    e = cub::DeviceScan::ExclusiveSum(nullptr, tb4, rsz, const_cast<long long*>(A.tile_off),
                                      (int)(ntiles + 1), s);
  if (e == cudaSuccess)
    e = cudaMallocAsync(&temp, std::max<size_t>(std::max(std::max(tb1, tb2), std::max(tb3, tb4)), 1),
                        s);
  // segments: non-empty flags, their ranks, the empty list
  if (e == cudaSuccess) e = cudaMemsetAsync(nonempty, 0, (ns1 + 1) * sizeof(int32_t), s);
  if (e == cudaSuccess && nseg > 0) {
    nonempty_flags_kernel<<<grid_for(nseg), 256, 0, s>>>(ptr, nseg, nonempty, eflags);
    iota_kernel<<<grid_for(nseg), 256, 0, s>>>(ids, nseg);
    e = cub::DeviceSelect::Flagged(temp, tb2, ids, eflags, const_cast<int32_t*>(A.empty_seg),
                                   A.nempty, (int)nseg, s);
  } else if (e == cudaSuccess) {
    e = cudaMemsetAsync(A.nempty, 0, sizeof(long long), s);
  }
  if (e == cudaSuccess)
    e = cub::DeviceScan::ExclusiveSum(temp, tb1, nonempty, seg_rank, (int)(nseg + 1), s);
  // tiles: end bits, ended-segment counts, record sizes and offsets
  if (e == cudaSuccess && ntiles > 0) e = cudaMemsetAsync(ends, 0, ntiles * kEndBytes, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(tcount, 0, (ntiles + 1) * sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(rsz, 0, (ntiles + 1) * sizeof(long long), s);
  if (e == cudaSuccess && ntiles > 0) {
    mark_ends_kernel<<<grid_for(nseg), 256, 0, s>>>(ptr, nseg, reinterpret_cast<unsigned*>(ends));
    tile_count_kernel<<<grid_for(ntiles * 32), 256, 0, s>>>(ends, ntiles, tcount, rsz);
  }
  if (e == cudaSuccess)
    e = cub::DeviceScan::ExclusiveSum(temp, tb3, tcount, tile_rank, (int)(ntiles + 1), s);
  if (e == cudaSuccess)
    e = cub::DeviceScan::ExclusiveSum(temp, tb4, rsz, const_cast<long long*>(A.tile_off),
                                      (int)(ntiles + 1), s);
  // records (padding entries: value 0, index 0, no end bit)
  if (e == cudaSuccess && ntiles > 0) e = cudaMemsetAsync(A.rec, 0, z.rec_bytes, s);
  if (e == cudaSuccess && ntiles > 0) {
    pack_kernel<<<grid_for(nseg * 32), 256, 0, s>>>(ptr, nseg, idx, val, seg_rank, tile_rank,
                                                    A.tile_off, A.rec);
    copy_ends_kernel<<<grid_for(ntiles * 32), 256, 0, s>>>(ends, ntiles, A.tile_off, A.rec);
  }
  // ticket and epoch start at 0; per-CTA record tags never match before the first launch
  if (e == cudaSuccess) e = cudaMemsetAsync(A.epoch, 0, sizeof(unsigned), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(A.cta_tag, 0, kMaxPartialBlocks * sizeof(unsigned), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(A.ticket, 0, sizeof(unsigned), s);
  for (void* p : {(void*)nonempty, (void*)seg_rank, (void*)ids, (void*)eflags, (void*)ends,
                  (void*)tcount, (void*)tile_rank, (void*)rsz, temp})
    if (p) cudaFreeAsync(p, s);
  if (e == cudaSuccess) e = cudaGetLastError();
  return e == cudaSuccess ? 0 : (int)e;
}

// ---------------------------------------------------------------------------
// public launchers
// ---------------------------------------------------------------------------
void stream_forward(const StreamView& A, int loss, const double* w, const double* y, double C,
                    double* z, double* zhat, double* dvec, uint8_t* mask, ObjScalars* obj,
                    Scratch sc, cudaStream_t s) {
  if (loss == kLossLogistic) {
    FwdOp<kLossLogistic> op;
    op.w = w, op.y = y, op.C = C, op.z = z, op.zhat = zhat, op.dvec = dvec, op.mask = mask;
    op.obj = obj, op.sc = sc;
    launch_stream(A, op, s);
  } else {
    FwdOp<kLossSvm> op;
    op.w = w, op.y = y, op.C = C, op.z = z, op.zhat = zhat, op.dvec = dvec, op.mask = mask;
    op.obj = obj, op.sc = sc;
    launch_stream(A, op, s);
  }
}

void stream_dv(const StreamView& A, const double* p, const double* dvec, const uint8_t* mask,
               double* a, cudaStream_t s) {
  DvOp op;
  op.p = p, op.dvec = dvec, op.mask = mask, op.a = a;
  launch_stream(A, op, s);
}

template <int UK, bool SQ>
static void trans_epi(const StreamView& A, const UView& U, const EpiView& E, double* out,
                      cudaStream_t s) {
  if (E.kind == EPI_VEC) {
    TransOp<UK, SQ, EPI_VEC> op;
    op.U = U, op.E = E, op.out = out;
    launch_stream(A, op, s);
  } else if (E.kind == EPI_CONST) {
    TransOp<UK, SQ, EPI_CONST> op;
    op.U = U, op.E = E, op.out = out;
    launch_stream(A, op, s);
  } else {
    TransOp<UK, SQ, EPI_RAW> op;
    op.U = U, op.E = E, op.out = out;
    launch_stream(A, op, s);
  }
}

void stream_transposed(const StreamView& At, const UView& U, bool squared, const EpiView& E,
                       double* out, cudaStream_t s) {
  if (U.kind == U_VEC) {
    if (squared)
      trans_epi<U_VEC, true>(At, U, E, out, s);
    else
      trans_epi<U_VEC, false>(At, U, E, out, s);
  } else if (U.kind == U_SVM_RESID) {
    trans_epi<U_SVM_RESID, false>(At, U, E, out, s);
  } else {
    trans_epi<U_MASK, true>(At, U, E, out, s);
  }
}

}  // namespace tb
