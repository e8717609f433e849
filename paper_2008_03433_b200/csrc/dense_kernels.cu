// Tall-skinny dense kernels (l >> n, n <= 64) on sm_100a, FP64.
//
// X lives column-major on the device (X[j*ld + i], ld = l rounded up to a
// multiple of 256 rows, padding zeroed).  Every pass is one stream over X
// through a TMA bulk-copy pipeline:
//
//  * a persistent 8-warp CTA (one per SM) walks 256-row tiles t = blockIdx.x,
//    blockIdx.x + gridDim.x, ...;
//  * thread 0 issues one 2-D tensor-map box (the tile's rows x n columns)
//    plus bulk copies of the per-row side arrays the pass needs (y, D, mask,
//    ...) into a shared-memory stage, completing on that stage's mbarrier, and
//    refills a stage as soon as every warp has released it;
//  * 2-4 stages are in flight, so the bytes outstanding per SM are set by
//    shared memory (80-160 KB), not by registers -- the limiter of the
//    register-blocked thread-per-row kernel this replaces (255 regs, 12%
//    warps active, 45% of HBM peak: profiles/round1_P1_kernels.md);
//  * one thread per row reads its row from shared memory (conflict-free:
//    consecutive rows are consecutive doubles), forms the row dot
//    sequentially over j = 0..n-1 exactly like FeatureMatrix::row_dot
//    (linalg.cpp:75-86; no FMA contraction, so margins -- and with them the
//    L2-SVM active set I (loss.cpp:94-122) -- are bit-identical to the
//    reference), and accumulates c_i * x_i into n register accumulators;
//  * a fixed-shape block tree emits one n-vector per CTA; a fixed-order
//    second stage (dense_finalize / cg_small_step) finishes it.
//
// The margin pass also accumulates the gradient partials of the candidate
// (loss.cpp:74-80 / :129-137) -- free under the HBM bound -- so commit()
// never re-reads X; in Gram mode it also forms the whole Gram matrix (FWDG,
// a solve's starting point) or adds the rows that changed side to the
// committed one (FWDD, every candidate: gram.cu).
#include "common.cuh"
#include "kernels.h"

#include <cstdlib>

namespace tb {

namespace {

constexpr int kSmemBudget = 200 * 1024;

// Per-row side arrays staged with each tile (slot offsets inside a stage).
struct StageLayout {
  int n, T;
  int nd;            // number of staged double side arrays (<= 3)
  bool has_mask;     // staged uint8 mask
  __host__ __device__ int bytes() const { return (n + nd) * T * 8 + (has_mask ? T : 0); }
};

__device__ __forceinline__ double log1p_exp_neg(double t) {  // loss.hpp:99-102
  if (t >= 0.0) return log1p(exp(-t));
  return -t + log1p(exp(t));
}

struct PassArgs {
  long long l, ld;
  int n;
  const double* X;
  const double* v;       // w (FWD) or v (HV)
  const double* y;
  const double* dvec;    // LR: D (HV, PRECOND)
  const uint8_t* mask;   // SVM: active mask (HV, PRECOND); nullptr = all rows active
  double C;
  // FWD outputs
  double* z;
  double* zhat;
  double* dvec_out;
  uint8_t* mask_out;
  ObjScalars* obj;
  Scratch sc;
  double* partials;      // [gridDim.x][n]
  double* gram_partials; // PM_FWDG: [gridDim.x][n*n] Gram partials (gram.cu's G) of the candidate;
                         // PM_FWDD: the partials of its change against the reference slot
  const int* ref_stale;  // PM_FWDD: the reference slot's Gram flag (0: its G matches a.mask)
};

// PM_FWDD (L2-SVM): the margin pass also accumulates
//   Delta = sum_i (m_i - m_ref_i) x_i x_i^T
// over the rows whose active bit differs from the reference slot's mask
// (a.mask), so that the candidate's Gram matrix is G_ref + Delta
// (gram_delta_finalize) instead of a fresh pass over X: between commits only
// 6-11% of P1's rows change sides (profiles/active_churn_P1.jsonl, scripts/active_churn.py).
// When G_ref is not current (or the chain of updates is due for a refresh)
// the pass is a plain FWD and the candidate's G is left stale (formed afresh
// by ensure_gram if a CG needs it).
enum PassMode : int { PM_FWD = 0, PM_HV = 1, PM_PRECOND = 2, PM_FWDG = 3, PM_FWDD = 4 };

// mma.sync m8n8k4 f64 (DMMA), as gram.cu
__device__ __forceinline__ void dmma8(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Side arrays of a mode: d-arrays in order, then the mask.
template <int MODE, int LOSS>
struct Side {
  static constexpr bool fwd = MODE == PM_FWD || MODE == PM_FWDG || MODE == PM_FWDD;
  static constexpr int nd = fwd ? 1 : (LOSS == kLossLogistic ? 1 : 0);
  static constexpr bool mask = (!fwd && LOSS == kLossSvm) || MODE == PM_FWDD;  // (FWDD: the reference mask)
};

// TB_DENSE_PRODUCER_WARP=1: a dedicated producer warp issues the copies.
// Default: thread 0 issues them -- the first stages up front, then each stage
// again as soon as every warp has released it -- so the CTA is 8 warps, not 9,
// and a thread may hold 255 registers instead of 168 (the register file is
// split over the four sub-partitions: 3 warps of one CTA shared one of them).
#ifndef TB_DENSE_PRODUCER_WARP
#define TB_DENSE_PRODUCER_WARP 0
#endif
constexpr int kProdWarps = TB_DENSE_PRODUCER_WARP ? 1 : 0;

// T compute threads (one row of the tile each) [+ one producer warp].
template <int NMAX, int T, int MODE, int LOSS>
__global__ void __launch_bounds__(T + kProdWarps * kWarp, 1)
    dense_pass_kernel(const __grid_constant__ CUtensorMap xmap, PassArgs a, int nstages) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) unsigned long long full[4], empty[4];
  __shared__ double s_v[NMAX];
  constexpr int BLK = T + kProdWarps * kWarp;
  constexpr int NCW = T / kWarp;  // compute warps
  __shared__ double sh[BLK / kWarp + 1];
  using SD = Side<MODE, LOSS>;
  const int n = a.n;
  const bool use_mask = SD::mask && a.mask != nullptr;
  StageLayout L{n, T, SD::nd, use_mask};
  const int sbytes = (L.bytes() + 127) & ~127;
  const long long ntiles = (a.l + T - 1) / T;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  if (tid == 0) {
    for (int s = 0; s < nstages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    mbar_fence_init();
  }
  for (int j = tid; j < NMAX; j += BLK) s_v[j] = (j < n && MODE != PM_PRECOND) ? a.v[j] : 0.0;
  __syncthreads();

  double acc[NMAX];
#pragma unroll
  for (int j = 0; j < NMAX; ++j) acc[j] = 0.0;
  double term_acc = 0.0, cnt_acc = 0.0;
  // PM_FWDG: the candidate's Gram matrix G = sum_i c_i x_i x_i^T in the same
  // pass (gram.cu's DMMA scheme on the staged tile): NB groups of 8 columns,
  // NP block pairs, two accumulators per pair and lane
  constexpr bool FG = MODE == PM_FWDG;
  constexpr bool FD = MODE == PM_FWDD;
  constexpr int NB = (FG || FD) ? (NMAX + 7) / 8 : 1;
  constexpr int NP = NB * (NB + 1) / 2;
  __shared__ double s_w[FG ? 2 : 1][FG ? T : 1];  // row weights c_i, by tile parity
  // PM_FWDD: the tile's changed rows, compacted kDR at a time into a
  // column-major block (stride kDS = 4 mod 16 doubles: conflict-free DMMA
  // fragment loads), their weights +-1, and the per-warp counts by tile parity
  constexpr int kDR = 64, kDS = kDR + 4;
  // (two blocks by tile parity: a tile's rows are multiplied during the next
  // tile, after its count barrier -- one CTA barrier per tile)
  __shared__ double s_cb[FD ? 2 : 1][FD ? NMAX * kDS : 1];
  __shared__ double s_cw[FD ? 2 : 1][FD ? kDR : 1];
  __shared__ int s_cnt[FD ? 2 : 1][FD ? NCW : 1];
  int pend = 0;  // PM_FWDD: rows (whole k-steps) of the previous tile waiting in its block
  const bool dodelta = FD && !gram_ref_is_empty(a.ref_stale);
  double gacc[FD ? 1 : NP][2];  // (FWDD: dacc below)
#pragma unroll
  for (int p = 0; p < (FD ? 1 : NP); ++p) gacc[p][0] = gacc[p][1] = 0.0;
  // PM_FWDD: warp w owns the block pairs w, w + NCW, ... of the Delta (two
  // accumulators per pair and lane, summed over every k-step of every round
  // in order: deterministic, and only NPW pairs' registers per thread)
  constexpr int NPW = FD ? (NP + NCW - 1) / NCW : 1;
  double dacc[NPW][2];
  int dc1[NPW], dc2[NPW];
  // the rows of a block (rows4: whole k-steps) times themselves: this warp's pairs
  auto delta_rows = [&](const double* cb, const double* cw, int rows4) {
    const int g = lane >> 2, tq = lane & 3;
    for (int ks = 0; ks < rows4 / 4; ++ks) {
      const int rr = ks * 4 + tq;
      const double w = cw[rr];
#pragma unroll
      for (int q = 0; q < NPW; ++q) {
        if (dc1[q] >= 0) {
          const double fa = w * cb[(dc1[q] * 8 + g) * kDS + rr];
          const double fb = cb[(dc2[q] * 8 + g) * kDS + rr];
          dmma8(dacc[q], fa, fb);
        }
      }
    }
  };
#pragma unroll
  for (int q = 0; q < NPW; ++q) {
    dacc[q][0] = dacc[q][1] = 0.0;
    int pp = wid + q * NCW, c1 = 0;
    if (pp >= NP) pp = -1;
    int rem = pp < 0 ? 0 : pp;
    while (rem >= NB - c1) {
      rem -= NB - c1;
      ++c1;
    }
    dc1[q] = pp < 0 ? -1 : c1;
    dc2[q] = c1 + rem;
  }

  // one 2-D TMA box {T rows x n columns} of X per tile plus the per-row side
  // arrays, into stage k % nstages (one thread)
  auto issue = [&](long long k) {
    const long long t = blockIdx.x + k * gridDim.x;
    const int s = (int)(k % nstages);
    unsigned char* base = smem + (size_t)s * sbytes;
    const long long row0 = t * T;
    mbar_arrive_expect_tx(&full[s], (unsigned)L.bytes());
    tma_load_2d(base, &xmap, (int)row0, 0, &full[s]);
    if (SD::nd >= 1) {
      const double* src = SD::fwd ? a.y : a.dvec;
      bulk_g2s(base + (size_t)n * T * 8, src + row0, T * 8, &full[s]);
    }
    if (use_mask) bulk_g2s(base + (size_t)(n + SD::nd) * T * 8, a.mask + row0, T, &full[s]);
  };
  if (!kProdWarps && tid == 0)
    for (long long k = 0; k < nstages && blockIdx.x + k * gridDim.x < ntiles; ++k) issue(k);
  if (kProdWarps && wid == NCW) {
    // ---- producer warp
    if (lane == 0) {
      for (long long k = 0;; ++k) {
        const long long t = blockIdx.x + k * gridDim.x;
        if (t >= ntiles) break;
        const int s = (int)(k % nstages);
        if (k >= nstages) mbar_wait_parity(&empty[s], (unsigned)(((k / nstages) - 1) & 1));
        issue(k);
      }
    }
  } else {
  long long last_k = 0;
  for (long long k = 0;; ++k) {
    const long long t = blockIdx.x + k * gridDim.x;
    if (t >= ntiles) break;
    int fd_tot_k = 0;  // PM_FWDD: this tile's changed rows
    const int s = (int)(k % nstages);
    mbar_wait_parity(&full[s], (unsigned)((k / nstages) & 1));
    const double* xs = reinterpret_cast<const double*>(smem + (size_t)s * sbytes);
    const double* side = xs + (size_t)n * T;
    const uint8_t* ms = reinterpret_cast<const uint8_t*>(side + (size_t)SD::nd * T);
    const long long i = t * T + tid;
    const bool in = i < a.l;

    // the whole row into registers first: all LDS issued back to back
    double x[NMAX];
#pragma unroll
    for (int j = 0; j < NMAX; ++j) x[j] = j < n ? xs[j * T + tid] : 0.0;
    if (MODE == PM_PRECOND) {
      // row_axpy_squared: out += c*x*x with c = D_i (LR) or [i in I] (SVM)
      double c = LOSS == kLossLogistic ? side[tid] : (use_mask ? (ms[tid] ? 1.0 : 0.0) : 1.0);
      if (!in) c = 0.0;
#pragma unroll
      for (int j = 0; j < NMAX; ++j) acc[j] += (c * x[j]) * x[j];
    } else {
      // sequential row dot (row_dot, linalg.cpp:75-86)
      double sdot = 0.0;
#pragma unroll
      for (int j = 0; j < NMAX; ++j)
        if (j < n) sdot += x[j] * s_v[j];
      double c;
      double cg = 0.0;  // PM_FWDG: this row's Gram weight (SVM: [i in I], LR: D_i)
      if (SD::fwd) {
        const double yi = side[tid];
        c = 0.0;
        if (in) {
          a.z[i] = sdot;
          if (LOSS == kLossLogistic) {  // logistic_fused_pass, loss.cpp:35-58
            const double tt = yi * sdot;
            const double sig = 1.0 / (1.0 + exp(tt));  // exp overflow -> inf -> 0
            const double zh = -yi * sig;
            a.zhat[i] = zh;
            const double di = (1.0 - sig) * sig;
            a.dvec_out[i] = di;
            cg = di;
            term_acc += log1p_exp_neg(tt);
            c = zh;  // gradient coefficient (loss.cpp:74-80)
          } else {  // svm_fused_pass, loss.cpp:94-122 (strict margin > 0)
            const double margin = 1.0 - yi * sdot;
            if (margin > 0.0) {
              a.mask_out[i] = 1;
              cg = 1.0;
              term_acc += margin * margin;
              cnt_acc += 1.0;
              c = sdot - yi;  // svm_gradient coefficient (loss.cpp:129-137)
            } else {
              a.mask_out[i] = 0;
            }
          }
        }
      } else {  // PM_HV: LR a0_i = (x_i.v) D_i (loss.cpp:85-89); SVM row_axpy(i, x_i.v) over I
        if (LOSS == kLossLogistic)
          c = sdot * side[tid];
        else
          c = use_mask ? (ms[tid] ? sdot : 0.0) : sdot;
        if (!in) c = 0.0;
      }
      // PM_FWDD, part 1: this row's change of side (+1 entered I, -1 left it,
      // 0 unchanged), its place among the tile's changed rows, and -- for the
      // first kDR of them -- the row into the block straight from the registers
      bool fd_ch = false;
      int fd_pos = 0, fd_tot = 0;
      double fd_cdel = 0.0;
      if (FD && dodelta) {
        fd_cdel = in ? cg - (ms[tid] ? 1.0 : 0.0) : 0.0;
        fd_ch = fd_cdel != 0.0;
        const unsigned bal = __ballot_sync(0xffffffffu, fd_ch);
        int* cnt = s_cnt[FD ? (k & 1) : 0];
        if (lane == 0) cnt[wid] = __popc(bal);
        asm volatile("bar.sync 1, %0;" ::"r"(T) : "memory");
        fd_pos = __popc(bal & ((1u << lane) - 1u));
        for (int w = 0; w < NCW; ++w) {
          const int c2 = cnt[w];
          fd_pos += w < wid ? c2 : 0;
          fd_tot += c2;
        }
        fd_tot_k = fd_tot;
        if (fd_tot <= kDR) {  // (else the rounds of part 2)
          double* cb = s_cb[FD ? (k & 1) : 0];
          double* cw = s_cw[FD ? (k & 1) : 0];
          if (fd_ch) {
#pragma unroll
            for (int j = 0; j < NMAX; ++j) cb[j * kDS + fd_pos] = x[j];  // (zeros beyond n)
            cw[fd_pos] = fd_cdel;
          }
          const int t4 = (fd_tot + 3) & ~3;
          if (tid < t4 - fd_tot) {  // the last k-step's padding rows: weight 0, finite values
#pragma unroll
            for (int j = 0; j < NMAX; ++j) cb[j * kDS + fd_tot + tid] = 0.0;
            cw[fd_tot + tid] = 0.0;
          }
        }
      }
#pragma unroll
      for (int j = 0; j < NMAX; ++j) acc[j] += c * x[j];  // x[j] = 0 beyond n
      if (FG) {
        // the tile's Gram blocks: every row weight first (a barrier of the
        // compute warps), then warp w takes the k-steps w, w + NCW, ... of the tile
        double* wts = s_w[FG ? (k & 1) : 0];
        wts[tid] = cg;
        asm volatile("bar.sync 1, %0;" ::"r"(T) : "memory");
        const int g = lane >> 2, tq = lane & 3;
        for (int ks = wid; ks < T / 4; ks += NCW) {
          const int rr = ks * 4 + tq;
          const double cw = wts[rr];
          double fb[NB], fa[NB];
#pragma unroll
          for (int q = 0; q < NB; ++q) {
            const int col = q * 8 + g;
            fb[q] = col < n ? xs[col * T + rr] : 0.0;
            fa[q] = cw * fb[q];
          }
          int pp = 0;
#pragma unroll
          for (int c1 = 0; c1 < NB; ++c1)
#pragma unroll
            for (int c2 = c1; c2 < NB; ++c2) dmma8(gacc[pp++], fa[c1], fb[c2]);
        }
      }
      if (FD && dodelta) {
        if (fd_tot > kDR) {
          if (pend > 0) delta_rows(s_cb[FD ? ((k + 1) & 1) : 0], s_cw[FD ? ((k + 1) & 1) : 0], pend);
          pend = 0;
          // more than kDR rows changed in this tile (rare): rounds now, from the
          // stage (the registers are gone), with barriers
          double* cb = s_cb[FD ? (k & 1) : 0];
          double* cw = s_cw[FD ? (k & 1) : 0];
          for (int r0 = 0; r0 < fd_tot; r0 += kDR) {
            const int nr = fd_tot - r0 < kDR ? fd_tot - r0 : kDR, nr4 = (nr + 3) & ~3;
            if (fd_ch && fd_pos >= r0 && fd_pos < r0 + kDR) {
              const int q = fd_pos - r0;
#pragma unroll
              for (int j = 0; j < NMAX; ++j) cb[j * kDS + q] = j < n ? xs[j * T + tid] : 0.0;
              cw[q] = fd_cdel;
            }
            if (tid < nr4 - nr) {
#pragma unroll
              for (int j = 0; j < NMAX; ++j) cb[j * kDS + nr + tid] = 0.0;
              cw[nr + tid] = 0.0;
            }
            asm volatile("bar.sync 1, %0;" ::"r"(T) : "memory");
            delta_rows(cb, cw, nr4);
            asm volatile("bar.sync 1, %0;" ::"r"(T) : "memory");  // the block is restaged next
          }
        }
      }
    }
    int pend_now = 0;  // PM_FWDD: the previous tile's rows, multiplied after this stage's release
    if (FD && dodelta) {
      pend_now = pend;
      pend = fd_tot_k <= kDR ? ((fd_tot_k + 3) & ~3) : 0;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
    if (!kProdWarps && wid == 0 && blockIdx.x + (k + nstages) * gridDim.x < ntiles) {
      // refill stage s once every warp has released it
      mbar_wait_parity(&empty[s], (unsigned)((k / nstages) & 1));
      if (lane == 0) issue(k + nstages);
      __syncwarp();
    }
    // PM_FWDD, part 2: the PREVIOUS tile's block on the FP64 tensor cores
    // (every warp wrote its rows before this tile's count barrier; the block is
    // rewritten only after the next one), off the stage
    if (pend_now > 0) delta_rows(s_cb[FD ? ((k + 1) & 1) : 0], s_cw[FD ? ((k + 1) & 1) : 0], pend_now);
    last_k = k;
  }
  if (FD && dodelta && pend > 0) {  // the last tile's rows
    asm volatile("bar.sync 1, %0;" ::"r"(T) : "memory");
    delta_rows(s_cb[FD ? (last_k & 1) : 0], s_cw[FD ? (last_k & 1) : 0], pend);
  }
  }
  __syncthreads();  // all stages consumed; the producer has no copy in flight

  // block tree: warp sums, then a fixed warp order (producer warp adds zeros)
  double* s_red = reinterpret_cast<double*>(smem);
  constexpr int NW = NCW;
#pragma unroll
  for (int j = 0; j < NMAX; ++j) {
    if (j < n) {
      const double r = warp_sum(acc[j]);
      if (lane == 0 && wid < NCW) s_red[wid * NMAX + j] = r;
    }
  }
  __syncthreads();
  if (tid < n) {
    double tsum = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) tsum += s_red[w * NMAX + tid];
    a.partials[(long long)blockIdx.x * n + tid] = tsum;
  }

  if (FG || (FD && dodelta)) {
    // the compute warps' Gram partials, added in warp order (after the
    // gradient tree's slots), then this CTA's n x n partial, mirrored
    __syncthreads();
    double* gred = s_red + NCW * NMAX;  // [NP][64]
    const int g = lane >> 2, tq = lane & 3;
    if (FD) {  // each pair has one owner warp
      if (wid < NCW) {
#pragma unroll
        for (int q = 0; q < NPW; ++q)
          if (dc1[q] >= 0)
#pragma unroll
            for (int h = 0; h < 2; ++h) gred[(wid + q * NCW) * 64 + g * 8 + 2 * tq + h] = dacc[q][h];
      }
      __syncthreads();
    } else {
      for (int w = 0; w < NCW; ++w) {
        if (wid == w) {
#pragma unroll
          for (int p = 0; p < NP; ++p)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int idx = p * 64 + g * 8 + 2 * tq + h;
              gred[idx] = w == 0 ? gacc[p][h] : gred[idx] + gacc[p][h];
            }
        }
        __syncthreads();
      }
    }
    double* gout = a.gram_partials + (size_t)blockIdx.x * n * n;
    for (int e = tid; e < NP * 64; e += BLK) {
      const int p = e / 64, gi = (e % 64) / 8, ci = e % 8;
      int c1 = 0, rem = p;
      while (rem >= NB - c1) {
        rem -= NB - c1;
        ++c1;
      }
      const int c2 = c1 + rem;
      const int j = c1 * 8 + gi, kk = c2 * 8 + ci;
      if (j < n && kk < n) {
        gout[j * n + kk] = gred[e];
        if (c1 != c2) gout[kk * n + j] = gred[e];
      }
    }
  }

  if (SD::fwd) {
    const double bt = block_sum<BLK>(term_acc, sh, true);
    const double bc = block_sum<BLK>(cnt_acc, sh, true);
    if (tid == 0) {
      a.sc.partials[2 * blockIdx.x] = bt;
      a.sc.partials[2 * blockIdx.x + 1] = bc;
    }
    if (last_block_arrive(a.sc.tickets + T_FUN)) {
      const double tot = reduce_partials<BLK>(a.sc.partials, gridDim.x, 2, 0, sh);
      const double cnt = reduce_partials<BLK>(a.sc.partials, gridDim.x, 2, 1, sh);
      // ww of a short vector, serially like dot() (linalg.cpp:267-272)
      if (tid == 0) {
        double ww = 0.0;
        for (int j = 0; j < n; ++j) ww += a.v[j] * a.v[j];
        a.obj->ww = ww;
        a.obj->f = 0.5 * ww + a.C * tot;
        a.obj->nact = (long long)cnt;
        a.obj->red[0] = tot;
        a.obj->red[1] = cnt;
      }
    }
  }
}

int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return (e && *e) ? std::atoi(e) : dflt;
}

template <int NMAX, int T, int MODE, int LOSS>
void launch_pass(const CUtensorMap& m, const PassArgs& a, cudaStream_t s) {
  using SD = Side<MODE, LOSS>;
  StageLayout L{a.n, T, SD::nd, SD::mask && a.mask != nullptr};
  const int sbytes = (L.bytes() + 127) & ~127;
  static const int max_stages = env_int("TRON_B200_DENSE_STAGES", 4);
  int ns = kSmemBudget / sbytes;
  if (ns > max_stages) ns = max_stages;
  if (ns > 4) ns = 4;
  if (ns < 2) ns = 2;
  size_t smem = (size_t)ns * sbytes;
  size_t red = (size_t)(T / kWarp) * NMAX * 8;
  if (MODE == PM_FWDG || MODE == PM_FWDD) {
    const int NB = (NMAX + 7) / 8;
    red += (size_t)(NB * (NB + 1) / 2) * 64 * 8;
  }
  if (smem < red) smem = red;
  auto k = dense_pass_kernel<NMAX, T, MODE, LOSS>;
  // (the attribute must not exceed the opt-in max minus the static shared memory)
  ensure_max_dynamic_smem((const void*)k, (int)smem);
  const int grid = dense_grid(a.l, a.n);
  launch_pdl(k, dim3(grid), dim3(T + kProdWarps * kWarp), smem, s, m, a, ns);
}

template <int NMAX, int T>
void launch_mode_t(int mode, int loss, const CUtensorMap& m, const PassArgs& a, cudaStream_t s) {
  if (loss == kLossLogistic) {
    if (mode == PM_FWD) launch_pass<NMAX, T, PM_FWD, kLossLogistic>(m, a, s);
    else if (mode == PM_HV) launch_pass<NMAX, T, PM_HV, kLossLogistic>(m, a, s);
    else if (mode == PM_FWDG) { if constexpr (NMAX <= 40) launch_pass<NMAX, T, PM_FWDG, kLossLogistic>(m, a, s); }
    else launch_pass<NMAX, T, PM_PRECOND, kLossLogistic>(m, a, s);
  } else {
    if (mode == PM_FWD) launch_pass<NMAX, T, PM_FWD, kLossSvm>(m, a, s);
    else if (mode == PM_HV) launch_pass<NMAX, T, PM_HV, kLossSvm>(m, a, s);
    else if (mode == PM_FWDG) { if constexpr (NMAX <= 40) launch_pass<NMAX, T, PM_FWDG, kLossSvm>(m, a, s); }
    else if (mode == PM_FWDD) { if constexpr (NMAX <= 40) launch_pass<NMAX, T, PM_FWDD, kLossSvm>(m, a, s); }
    else launch_pass<NMAX, T, PM_PRECOND, kLossSvm>(m, a, s);
  }
}

template <int NMAX>
void launch_mode(int mode, int loss, const CUtensorMap& m, const PassArgs& a, cudaStream_t s) {
  if (dense_tile_rows(a.n) == 128)
    launch_mode_t<NMAX, 128>(mode, loss, m, a, s);
  else if (NMAX <= 48)
    launch_mode_t<NMAX, 256>(mode, loss, m, a, s);
}

#define TB_NMAX_DISPATCH(n, CALL)                      \
  if ((n) <= 8) { CALL(8); }                           \
  else if ((n) <= 16) { CALL(16); }                    \
  else if ((n) <= 24) { CALL(24); }                    \
  else if ((n) <= 32) { CALL(32); }                    \
  else if ((n) <= 40) { CALL(40); }                    \
  else if ((n) <= 48) { CALL(48); }                    \
  else { CALL(64); }

void launch(int mode, int loss, const CUtensorMap& m, const PassArgs& a, cudaStream_t s) {
#define TB_CALL(NM) launch_mode<NM>(mode, loss, m, a, s)
  TB_NMAX_DISPATCH(a.n, TB_CALL)
#undef TB_CALL
}

__global__ void __launch_bounds__(1024) dense_finalize_kernel(int n, const double* partials,
                                                             int nparts, EpiView E, double* out) {
  pdl_wait();
  pdl_trigger();
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
constexpr int kBlock = 256;
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
  // exclusive block scan of c
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

// Gathered panel: rows idx of X, column-major with ldg rows; rows
// [nI, ldg) are zero so the tiled passes can stream whole tiles.
__global__ void gather_kernel(long long nI, int n, const double* __restrict__ X, long long ld,
                              const int32_t* __restrict__ idx, double* __restrict__ Xg,
                              long long ldg) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < ldg;
       k += (long long)gridDim.x * blockDim.x) {
    if (k < nI) {
      const long long i = idx[k];
      for (int j = 0; j < n; ++j) Xg[(long long)j * ldg + k] = X[(long long)j * ld + i];
    } else {
      for (int j = 0; j < n; ++j) Xg[(long long)j * ldg + k] = 0.0;
    }
  }
}

}  // namespace

int64_t dense_ld(int64_t l) { return (l + kDenseTile - 1) / kDenseTile * kDenseTile; }

int dense_make_map(CUtensorMap* map, const double* X, int64_t ld, int64_t rows, int64_t n) {
  return dense_make_map_box(map, X, ld, rows, n, dense_tile_rows(n));
}

int dense_make_map_box(CUtensorMap* map, const double* X, int64_t ld, int64_t rows, int64_t n,
                       int box_rows) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<EncodeFn>(fn);
  }();
  if (!encode) return -1;
  if (rows < 1) rows = 1;
  const cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)(n > 0 ? n : 1)};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)box_rows, (cuuint32_t)(n > 0 ? n : 1)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(X), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)r;
}

int dense_tile_rows(int64_t n) {
  static const int forced = env_int("TRON_B200_DENSE_TILE", 0);  // A/B experiments
  if (n > 48) return 128;
  return forced == 128 ? 128 : 256;
}

int dense_grid(int64_t l, int64_t n) {
  const int64_t T = dense_tile_rows(n);
  int64_t g = (l + T - 1) / T;
  const int64_t cap = (int64_t)device_sm_count();
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

bool dense_forward_gram_fused(int64_t n) { return n <= 40; }
bool dense_forward_gram_delta(int64_t n) { return n <= 40; }

void dense_forward(int64_t l, int64_t n, int64_t ld, const double* X, const CUtensorMap& xmap,
                   int loss, const double* w,
                   const double* y, double C, double* z, double* zhat, double* dvec, uint8_t* mask,
                   double* gparts, ObjScalars* obj, Scratch sc, cudaStream_t s,
                   double* gram_parts, const uint8_t* mask_ref, const int* ref_stale) {
  PassArgs a{};
  a.gram_partials = gram_parts;
  a.mask = mask_ref;
  a.ref_stale = ref_stale;
  a.l = l;
  a.ld = ld;
  a.n = (int)n;
  a.X = X;
  a.v = w;
  a.y = y;
  a.C = C;
  a.z = z;
  a.zhat = zhat;
  a.dvec_out = dvec;
  a.mask_out = mask;
  a.obj = obj;
  a.sc = sc;
  a.partials = gparts;
  launch(gram_parts ? (mask_ref ? PM_FWDD : PM_FWDG) : PM_FWD, loss, xmap, a, s);
}

void dense_accum(int kind, int64_t l, int64_t n, int64_t ld, const double* X,
                 const CUtensorMap& xmap, int loss,
                 const double* v, const double* dvec, const uint8_t* mask, double* partials,
                 cudaStream_t s) {
  PassArgs a{};
  a.l = l;
  a.ld = ld;
  a.n = (int)n;
  a.X = X;
  a.v = v;
  a.dvec = dvec;
  a.mask = mask;
  a.partials = partials;
  launch(kind == DA_HV ? PM_HV : PM_PRECOND, loss, xmap, a, s);
}

void dense_finalize(int64_t n, const double* partials, int nparts, const EpiView& epi, double* out,
                    cudaStream_t s) {
  launch_pdl(dense_finalize_kernel, dim3(1), dim3(1024), 0, s, (int)n, partials, nparts, epi, out);
}

void dense_transpose_chunk(const double* rm, int64_t rows, int64_t n, double* X, int64_t ld,
                           int64_t row0, cudaStream_t s) {
  dim3 grid((unsigned)((rows + 31) / 32), (unsigned)((n + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(rm, rows, (int)n, X, ld, row0);
  TB_LAUNCH_CHECK();
}

void compact_mask(int64_t l, const uint8_t* mask, int32_t* idx, int32_t* tmp, long long* count_out,
                  cudaStream_t s) {
  const int nb = (int)((l + kChunk - 1) / kChunk);
  if (nb == 0) {
    cudaMemsetAsync(count_out, 0, sizeof(long long), s);
    return;
  }
  count_kernel<<<nb, kBlock, 0, s>>>(l, mask, tmp);
  TB_LAUNCH_CHECK();
  scan_kernel<<<1, 1024, 0, s>>>(tmp, nb, count_out);
  TB_LAUNCH_CHECK();
  scatter_kernel<<<nb, kBlock, 0, s>>>(l, mask, tmp, idx);
  TB_LAUNCH_CHECK();
}

void dense_gather(int64_t nI, int64_t n, const double* X, int64_t ld, const int32_t* idx,
                  double* Xg, int64_t ldg, cudaStream_t s) {
  long long g = (ldg + 255) / 256;
  if (g > (long long)device_sm_count() * 16) g = (long long)device_sm_count() * 16;
  if (g < 1) g = 1;
  gather_kernel<<<(int)g, 256, 0, s>>>(nI, (int)n, X, ld, idx, Xg, ldg);
  TB_LAUNCH_CHECK();
}

}  // namespace tb
