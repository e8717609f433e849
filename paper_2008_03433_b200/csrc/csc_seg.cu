// X^T u over the device CSC copy: warp-per-chunk segmented reduction.
//
// The reference computes X^T u (matvec_transpose / masked_matvec_transpose /
// weighted_sq_col_sums, proj/src/linalg.cpp:175-265) by scattering every row
// into one of 64 private n-length buffers and merging them serially
// (parallel.hpp:101-123) -- the dominant cost of TRON-LR at large n.  Here
// the CSC copy turns it into a segmented sum over contiguous memory:
//
//  * the nonzeros are cut into chunks of at most 256 (one warp, 8 per
//    lane) packed greedily along column boundaries, so work is balanced
//    regardless of column lengths (Zipf-hot columns of 20k+ entries and the
//    27% empty columns of news20 cost the same) and only columns longer
//    than a chunk are split;
//  * per-entry "last entry of its column" bits, the chunk -> column-rank
//    map and the table of non-empty columns are precomputed once per
//    matrix on the host (the structure never changes during a solve);
//  * a lane sums its 8 products sequentially, column pieces that cross
//    lanes are combined by one warp-level segmented scan, the pieces of
//    long columns by a fixed-order fix-up pass.  No atomics, no shared
//    memory, no block barriers: results are bit-reproducible run to run.
//  * each emitted column also writes the empty columns that follow it, so
//    the epilogue (base_j + scale*sum) covers every j in one pass.
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <cstdlib>

namespace tb {

namespace {

constexpr int kBlock = 256;         // 8 warps = 8 chunks per block
constexpr int kStagedBlock = 512;   // one 16-warp block per SM holding u in shared memory
constexpr long long kStageMaxBytes = 190 * 1024;  // + 32 KB of static emission buffers

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
__device__ __forceinline__ double epi_value(const EpiView& E, long long j, double sum) {
  if (EPI == EPI_VEC) return E.base[j] + E.scale * sum;
  if (EPI == EPI_CONST) return E.cbase + E.scale * sum;
  return sum;
}

// Writes column nz_col[rank] and the empty columns up to the next non-empty one.
template <int EPI>
__device__ __forceinline__ void emit_rank(const SegView& S, const EpiView& E, double* out, int rank,
                                          double sum) {
  const int j = __ldg(S.nz_col + rank);
  const int j_next = __ldg(S.nz_col + rank + 1);
  out[j] = epi_value<EPI>(E, j, sum);
  for (int e = j + 1; e < j_next; ++e) out[e] = epi_value<EPI>(E, e, 0.0);
}

// Effective per-row weight u_i for the staged variant (shared memory).
template <int UK>
__device__ __forceinline__ double ueff(const UView& U, long long r) {
  if (UK == U_VEC) return U.u[r];
  if (UK == U_SVM_RESID) return U.mask[r] ? (U.z[r] - U.y[r]) : 0.0;
  return U.mask[r] ? 1.0 : 0.0;
}

// Raw operands of one chunk for one lane (loaded one chunk ahead).
struct LaneChunk {
  int cs, ce;
  long long base;
  double v[kSegLaneItems];
  int ix[kSegLaneItems];
  unsigned lo_word, hi_word, cr;
};

__device__ __forceinline__ void load_chunk(const CsrView& A, const SegView& S, long long t, int lane,
                                           LaneChunk& c) {
  if (S.fixed_chunks) {  // device-built plan: chunk t is [256t, 256t + 256), no load on the chain
    c.cs = (int)(t * kSegChunk);
    c.ce = (int)min((long long)c.cs + kSegChunk, (long long)A.nnz);
  } else {
    c.cs = __ldg(S.chunk_start + t);
    c.ce = __ldg(S.chunk_start + t + 1);
  }
  c.base = (long long)(c.cs & ~3) + lane * kSegLaneItems;  // 16-B aligned lanes
  if (c.base + kSegLaneItems <= A.nnz) {
#pragma unroll
    for (int m = 0; m < kSegLaneItems; m += 2) ld2(A.val + c.base + m, c.v[m], c.v[m + 1]);
#pragma unroll
    for (int m = 0; m < kSegLaneItems; m += 4)
      ld4(A.idx + c.base + m, c.ix[m], c.ix[m + 1], c.ix[m + 2], c.ix[m + 3]);
  } else {
#pragma unroll
    for (int m = 0; m < kSegLaneItems; ++m) {
      const long long k = c.base + m;
      c.v[m] = k < A.nnz ? A.val[k] : 0.0;
      c.ix[m] = k < A.nnz ? A.idx[k] : 0;
    }
  }
  const bool any = c.base < c.ce && c.base + kSegLaneItems > c.cs;
  c.lo_word = any ? __ldg(S.lastbits + (c.base >> 5)) : 0u;
  c.hi_word = any ? __ldg(S.lastbits + (c.base >> 5) + 1) : 0u;
  c.cr = __ldg(S.chunk_rank + t);
}

// One chunk: gathers, per-lane sequential sums, warp segmented scan, emission.
template <int UK, bool SQ, int EPI, bool STAGED>
__device__ __forceinline__ void process_chunk(const CsrView& A, const SegView& S, const UView& U,
                                              const EpiView& E, double* __restrict__ out,
                                              const double* su, long long t, const LaneChunk& cur,
                                              int lane, double* ebuf) {
  // gathers of the current chunk
  double w[kSegLaneItems];
#pragma unroll
  for (int m = 0; m < kSegLaneItems; ++m) {
    const long long k = cur.base + m;
    if (STAGED) {
      const double u = su[cur.ix[m]];
      const double p = SQ ? (u * cur.v[m]) * cur.v[m] : u * cur.v[m];
      w[m] = (k >= cur.cs && k < cur.ce) ? p : 0.0;
    } else {
      w[m] = (k >= cur.cs && k < cur.ce) ? weight<UK, SQ>(U, cur.ix[m], cur.v[m]) : 0.0;
    }
  }

  unsigned bits = 0u;
  if (cur.base < cur.ce && cur.base + kSegLaneItems > cur.cs) {
    // base is a multiple of 4: the lane's 8 bits may straddle two words
    const unsigned long long pair =
        (unsigned long long)cur.lo_word | ((unsigned long long)cur.hi_word << 32);
    bits = (unsigned)(pair >> (cur.base & 31)) & 0xffu;
    const long long lo = cur.cs - cur.base, hi = cur.ce - cur.base;  // keep [cs, ce)
    if (lo > 0) bits &= ~((1u << lo) - 1u);
    if (hi < kSegLaneItems) bits &= (1u << hi) - 1u;
  }
  const int chunk_rank = (int)(cur.cr & 0x7fffffffu);
  const bool cont_in = (cur.cr >> 31) != 0;

  // rank of the column containing this lane's first item
  const int cnt = __popc(bits);
  int incl = cnt;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += y;
  }
  const int r0 = chunk_rank + incl - cnt;

  // sequential pass over the lane's items; the sums of the columns ending
  // here go to the warp's buffer, indexed by their order in the chunk
  double acc = 0.0, head_val = 0.0;
  bool have_head = false;
  int k = incl - cnt;
#pragma unroll
  for (int m = 0; m < kSegLaneItems; ++m) {
    acc += w[m];
    if (bits & (1u << m)) {
      if (!have_head) {
        head_val = acc;
        have_head = true;
      } else {
        ebuf[k] = acc;  // column wholly inside this lane
      }
      ++k;
      acc = 0.0;
    }
  }

  // warp segmented inclusive scan of the carries, keyed by column rank
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
  if (have_head) ebuf[incl - cnt] = (lane > 0 && prev_key == r0) ? prev_val + head_val : head_val;
  if (lane == 31) S.carry[t] = val;
  // emission, warp-cooperative: consecutive columns to consecutive lanes, so
  // the nz_col / base loads and the stores of a chunk are coalesced and no
  // lane walks a chain of dependent loads
  __syncwarp();
  const int nend = __shfl_sync(0xffffffffu, incl, 31);
  for (int q = lane; q < nend; q += 32) {
    const double v = ebuf[q];
    if (q == 0 && cont_in)
      S.head[t] = v;  // column began in an earlier chunk: finished by the fix-up
    else
      emit_rank<EPI>(S, E, out, chunk_rank + q, v);
  }
  __syncwarp();  // the buffer is reused by the warp's next chunk

}

// Persistent warps walk chunks t, t+W, ...; the next chunk's operands are
// requested before the current chunk's gathers are consumed, so the
// descriptor -> data -> gather -> emission latency chain of consecutive
// chunks overlaps.
// STAGED: the gathered vector u (length A.cols = l) is first copied into
// shared memory, so the per-nonzero random gather is an LDS instead of an
// L1 wavefront (a 32-address LDG costs ~32 L1 wavefronts; measured on N1
// the gathers, not HBM, bounded this kernel).
template <int UK, bool SQ, int EPI, bool STAGED>
#ifndef TB_SEG_BLOCKS_PER_SM
#define TB_SEG_BLOCKS_PER_SM 3
#endif
#ifndef TB_SEG_PREFETCH2
#define TB_SEG_PREFETCH2 0
#endif
__global__ void __launch_bounds__(STAGED ? kStagedBlock : kBlock, STAGED ? 1 : TB_SEG_BLOCKS_PER_SM)
    seg_spmv_kernel(CsrView A, SegView S, UView U, EpiView E, double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ double su[];
  constexpr int BLK = STAGED ? kStagedBlock : kBlock;
  __shared__ double ebuf_all[BLK / kWarp][kSegChunk];
  const int lane = threadIdx.x & 31;
  double* ebuf = ebuf_all[threadIdx.x >> 5];
  if (STAGED) {
    if (UK == U_VEC) {
      bulk_stage_f64(su, U.u, A.cols);  // TMA bulk copy (UBLKCP)
    } else {
#pragma unroll 4
      for (long long i = threadIdx.x; i < A.cols; i += BLK) su[i] = ueff<UK>(U, i);
      __syncthreads();
    }
  }
  const long long W = ((long long)gridDim.x * BLK) >> 5;
  long long t = (blockIdx.x * (long long)BLK + threadIdx.x) >> 5;
  if (t >= S.nchunks) return;  // warp-uniform

  // Columns before the first non-empty one (usually none).
  if (t == 0 && lane == 0)
    for (int e = 0; e < __ldg(S.nz_col); ++e) out[e] = epi_value<EPI>(E, e, 0.0);

  LaneChunk cur;
  load_chunk(A, S, t, lane, cur);
  if (!STAGED && !TB_SEG_PREFETCH2) {
    // one chunk ahead: the next chunk's operands are requested before this
    // chunk's gathers are consumed
    for (;;) {
      const long long tn = t + W;
      LaneChunk nxt;
      if (tn < S.nchunks) load_chunk(A, S, tn, lane, nxt);
      process_chunk<UK, SQ, EPI, STAGED>(A, S, U, E, out, su, t, cur, lane, ebuf);
      if (tn >= S.nchunks) break;
      t = tn;
      cur = nxt;
    }
  } else {
    // u in shared memory makes the gathers cheap; with one 16-warp block per
    // SM, keep two chunks in flight per warp instead
    LaneChunk nxt;
    if (t + W < S.nchunks) load_chunk(A, S, t + W, lane, nxt);
    for (;;) {
      process_chunk<UK, SQ, EPI, STAGED>(A, S, U, E, out, su, t, cur, lane, ebuf);
      if (t + W >= S.nchunks) break;
      if (t + 2 * W < S.nchunks) load_chunk(A, S, t + 2 * W, lane, cur);
      process_chunk<UK, SQ, EPI, STAGED>(A, S, U, E, out, su, t + W, nxt, lane, ebuf);
      if (t + 2 * W >= S.nchunks) break;
      if (t + 3 * W < S.nchunks) load_chunk(A, S, t + 3 * W, lane, nxt);
      t += 2 * W;
    }
  }
}

template <int EPI>
__global__ void __launch_bounds__(kBlock) seg_fixup_kernel(SegView S, EpiView E,
                                                          double* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const long long f = (blockIdx.x * (long long)kBlock + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (f >= S.nfix) return;
  const int t = S.fix_chunk[f], ts = S.fix_first[f];
  double s = 0.0;
  for (int k = ts + lane; k < t; k += 32) s += S.carry[k];  // fixed order
  s = warp_sum(s);
  if (lane == 0) emit_rank<EPI>(S, E, out, (int)(S.chunk_rank[t] & 0x7fffffffu), s + S.head[t]);
}

template <int UK, bool SQ, int EPI, bool STAGED>
void launch_one(const CsrView& A, const SegView& S, const UView& U, const EpiView& E, double* out,
                cudaStream_t s) {
  if (STAGED) {
    const size_t smem = (size_t)A.cols * sizeof(double);
    static bool configured = false;  // per instantiation
    if (!configured) {
      cudaFuncSetAttribute(seg_spmv_kernel<UK, SQ, EPI, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kStageMaxBytes);
      configured = true;
    }
    long long want = (S.nchunks * 32 + kStagedBlock - 1) / kStagedBlock;
    const long long cap = device_sm_count();
    launch_pdl(seg_spmv_kernel<UK, SQ, EPI, true>, dim3((int)(want < cap ? want : cap)),
               dim3(kStagedBlock), smem, s, A, S, U, E, out);
  } else {
    // persistent: 3 blocks of 8 warps per SM (register-limited), never more than chunks
    long long want = (S.nchunks * 32 + kBlock - 1) / kBlock;
    const long long cap = (long long)device_sm_count() * TB_SEG_BLOCKS_PER_SM;
    launch_pdl(seg_spmv_kernel<UK, SQ, EPI, false>, dim3((int)(want < cap ? want : cap)),
               dim3(kBlock), 0, s, A, S, U, E, out);
  }
  const int fgrid = (int)((S.nfix * 32 + kBlock - 1) / kBlock);
  if (fgrid) launch_pdl(seg_fixup_kernel<EPI>, dim3(fgrid), dim3(kBlock), 0, s, S, E, out);
}

template <int UK, bool SQ>
void launch_seg(const CsrView& A, const SegView& S, const UView& U, const EpiView& E, double* out,
                cudaStream_t s) {
  // Opt-in (TRON_B200_STAGE=1): see csr_kernels.cu stage_enabled().
  static const bool stage_on = [] {
    const char* e = std::getenv("TRON_B200_STAGE");
    return e && e[0] == '1';
  }();
  const bool staged = stage_on && (long long)A.cols * (long long)sizeof(double) <= kStageMaxBytes;
  switch (E.kind) {
    case EPI_VEC:
      staged ? launch_one<UK, SQ, EPI_VEC, true>(A, S, U, E, out, s)
             : launch_one<UK, SQ, EPI_VEC, false>(A, S, U, E, out, s);
      break;
    case EPI_CONST:
      staged ? launch_one<UK, SQ, EPI_CONST, true>(A, S, U, E, out, s)
             : launch_one<UK, SQ, EPI_CONST, false>(A, S, U, E, out, s);
      break;
    default:
      staged ? launch_one<UK, SQ, EPI_RAW, true>(A, S, U, E, out, s)
             : launch_one<UK, SQ, EPI_RAW, false>(A, S, U, E, out, s);
      break;
  }
}

}  // namespace

// Greedy packing of whole rows (CSC: columns) into chunks of <= kSegChunk
// lane slots; a chunk's lanes start at its first entry rounded down to a
// multiple of 4 (16-byte aligned vector loads), so it holds entries
// [start, (start & ~3) + kSegChunk).  Rows that fit nowhere whole are split
// into consecutive pieces finished by the fix-up pass.
void seg_plan_host(const int32_t* ptr, int64_t rows, int64_t nnz, SegPlanHost* P) {
  P->chunk_start.clear();
  P->chunk_rank.clear();
  P->nz_col.clear();
  P->fix_chunk.clear();
  P->fix_first.clear();
  P->lastbits.assign((size_t)((nnz + 31) / 32 + 1), 0u);
  int64_t open_base = -1;  // aligned base of the chunk being filled, -1 = none
  uint32_t rank = 0;
  for (int64_t c = 0; c < rows; ++c) {
    const int64_t b = ptr[c], e = ptr[c + 1];
    if (e <= b) continue;
    P->nz_col.push_back((int32_t)c);
    P->lastbits[(size_t)((e - 1) >> 5)] |= 1u << ((e - 1) & 31);
    if (open_base >= 0 && e <= open_base + kSegChunk) {
      ++rank;  // fits in the open chunk
      continue;
    }
    if (e <= (b & ~int64_t{3}) + kSegChunk) {  // starts a new chunk
      P->chunk_start.push_back((int32_t)b);
      P->chunk_rank.push_back(rank);
      open_base = b & ~int64_t{3};
    } else {  // long row: consecutive pieces, the last one finished by the fix-up
      const int32_t first = (int32_t)P->chunk_start.size();
      for (int64_t p = b; p < e;) {
        const int64_t pe = std::min<int64_t>((p & ~int64_t{3}) + kSegChunk, e);
        P->chunk_start.push_back((int32_t)p);
        P->chunk_rank.push_back(rank | (p > b ? 0x80000000u : 0u));
        if (pe == e) {
          P->fix_chunk.push_back((int32_t)P->chunk_start.size() - 1);
          P->fix_first.push_back(first);
        }
        p = pe;
      }
      open_base = -1;
    }
    ++rank;
  }
  P->nz_col.push_back((int32_t)rows);
  P->chunk_start.push_back((int32_t)nnz);
}

// ---------------------------------------------------------------------------
// Device-built plan with fixed 256-entry chunks (every boundary inside a
// column becomes a fix-up): fully parallel, no host round trip of the CSC
// structure -- what context creation uses.
// ---------------------------------------------------------------------------
namespace {

__global__ void plan_chunk_start_kernel(int32_t* cs, long long nchunks, long long nnz) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t <= nchunks;
       t += (long long)gridDim.x * blockDim.x)
    cs[t] = (int32_t)(t * kSegChunk < nnz ? t * kSegChunk : nnz);
}

__global__ void plan_cols_kernel(const int32_t* cptr, long long n, uint32_t* lastbits,
                                 int32_t* nonempty, int32_t* ids, uint8_t* spans) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n;
       c += (long long)gridDim.x * blockDim.x) {
    const int b = cptr[c], e = cptr[c + 1];
    ids[c] = (int32_t)c;
    nonempty[c] = e > b;
    spans[c] = e > b && (b / kSegChunk) != ((e - 1) / kSegChunk);
    if (e > b) atomicOr(lastbits + ((e - 1) >> 5), 1u << ((e - 1) & 31));
  }
}

__global__ void plan_chunk_rank_kernel(const int32_t* cptr, long long n, const int32_t* colrank,
                                       long long nchunks, uint32_t* rank) {
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
    rank[t] = (uint32_t)colrank[c] | (cptr[c] < x ? 0x80000000u : 0u);
  }
}

__global__ void plan_fix_kernel(const int32_t* cptr, const int32_t* cols, const long long* count,
                                int32_t* fix_chunk, int32_t* fix_first) {
  const long long m = *count;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    const int c = cols[i];
    fix_first[i] = cptr[c] / kSegChunk;
    fix_chunk[i] = (cptr[c + 1] - 1) / kSegChunk;
  }
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

int seg_plan_device(const int32_t* cptr, int64_t n, int64_t nnz, SegView* P, int32_t* chunk_start,
                    uint32_t* chunk_rank, uint32_t* lastbits, int32_t* nz_col, int32_t* fix_chunk,
                    int32_t* fix_first, cudaStream_t s) {
  const int64_t nchunks = (nnz + kSegChunk - 1) / kSegChunk;
  const size_t n1 = n > 0 ? n : 1;
  int32_t *nonempty = nullptr, *colrank = nullptr, *ids = nullptr, *cols = nullptr;
  uint8_t* spans = nullptr;
  long long *cnt_nz = nullptr, *cnt_fix = nullptr;
  void* temp = nullptr;
  size_t tb1 = 0, tb2 = 0, tb3 = 0;
  cudaError_t e = cudaMallocAsync(&nonempty, (n1 + 1) * sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&colrank, (n1 + 1) * sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&ids, n1 * sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&cols, n1 * sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&spans, n1, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&cnt_nz, 2 * sizeof(long long), s);
  cnt_fix = cnt_nz + 1;
  if (e == cudaSuccess)
    e = cub::DeviceScan::ExclusiveSum(nullptr, tb1, nonempty, colrank, (int)(n + 1), s);
  if (e == cudaSuccess)
    e = cub::DeviceSelect::Flagged(nullptr, tb2, ids, nonempty, nz_col, cnt_nz, (int)n, s);
  if (e == cudaSuccess)
    e = cub::DeviceSelect::Flagged(nullptr, tb3, ids, spans, cols, cnt_fix, (int)n, s);
  if (e == cudaSuccess)
    e = cudaMallocAsync(&temp, std::max<size_t>(std::max(tb1, std::max(tb2, tb3)), 1), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(nonempty, 0, (n1 + 1) * sizeof(int32_t), s);
  if (e == cudaSuccess)
    e = cudaMemsetAsync(lastbits, 0, (size_t)((nnz + 31) / 32 + 1) * sizeof(uint32_t), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(cnt_nz, 0, 2 * sizeof(long long), s);
  if (e == cudaSuccess) {
    plan_chunk_start_kernel<<<pgrid(nchunks + 1), 256, 0, s>>>(chunk_start, nchunks, nnz);
    if (n > 0) plan_cols_kernel<<<pgrid(n), 256, 0, s>>>(cptr, n, lastbits, nonempty, ids, spans);
    e = cub::DeviceScan::ExclusiveSum(temp, tb1, nonempty, colrank, (int)(n + 1), s);
  }
  if (e == cudaSuccess && n > 0)
    e = cub::DeviceSelect::Flagged(temp, tb2, ids, nonempty, nz_col, cnt_nz, (int)n, s);
  if (e == cudaSuccess && n > 0)
    e = cub::DeviceSelect::Flagged(temp, tb3, ids, spans, cols, cnt_fix, (int)n, s);
  if (e == cudaSuccess) {
    plan_sentinel_kernel<<<1, 1, 0, s>>>(nz_col, colrank, n);
    if (nchunks > 0)
      plan_chunk_rank_kernel<<<pgrid(nchunks), 256, 0, s>>>(cptr, n, colrank, nchunks, chunk_rank);
    plan_fix_kernel<<<pgrid(n), 256, 0, s>>>(cptr, cols, cnt_fix, fix_chunk, fix_first);
  }
  long long nfix = 0;
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(&nfix, cnt_fix, sizeof(long long), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  for (void* p : {(void*)nonempty, (void*)colrank, (void*)ids, (void*)cols, (void*)spans,
                  (void*)cnt_nz, temp})
    if (p) cudaFreeAsync(p, s);
  if (e == cudaSuccess) e = cudaGetLastError();
  P->nchunks = nchunks;
  P->nfix = nfix;
  P->fixed_chunks = 1;
  P->chunk_start = chunk_start;
  P->chunk_rank = chunk_rank;
  P->lastbits = lastbits;
  P->nz_col = nz_col;
  P->fix_chunk = fix_chunk;
  P->fix_first = fix_first;
  return e == cudaSuccess ? 0 : (int)e;
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
