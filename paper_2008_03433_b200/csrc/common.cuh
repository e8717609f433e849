// Shared device helpers: deterministic warp/block reductions and the
// "last block finalizes" ticket used by every two-stage reduction.
//
// Determinism contract (the device analogue of the reference's fixed
// 64-block partition + pairwise tree, proj/include/tron/parallel.hpp:14-34):
// every reduction's shape depends only on the problem size and the launch
// configuration (fixed per device), never on timing, so repeated runs are
// bit-identical.  No floating-point atomics anywhere.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cooperative_groups.h>
#include <utility>

namespace tb {

constexpr int kWarp = 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;  // valid in lane 0
}

__device__ __forceinline__ double warp_allsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;  // identical in every lane (fixed butterfly order)
}

// Sum over a power-of-two lane group of width G (G <= 32), result in the
// group's first lane.
template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o, G);
  return v;
}

// Block-wide sum; result valid in thread 0 (and returned to all threads
// when `broadcast`).  `sh` needs BLOCK/32 + 1 doubles.
template <int BLOCK>
__device__ __forceinline__ double block_sum(double v, double* sh, bool broadcast = false) {
  constexpr int NW = BLOCK / kWarp;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) sh[wid] = v;
  __syncwarp();  // reconverge the warp before the block barrier
  __syncthreads();
  if (wid == 0) {
    double t = lane < NW ? sh[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) sh[NW] = t;
  }
  __syncthreads();
  double r = broadcast ? sh[NW] : (threadIdx.x == 0 ? sh[NW] : 0.0);
  if (broadcast) __syncthreads();
  return r;
}

// Grid-wide sums of K values in a cooperative kernel: block sums, one
// partial per CTA, a grid barrier, then every CTA adds all CTA partials in the
// same fixed order, so all CTAs hold identical totals.  parts: [2][grid][4]
// doubles used alternately (`buf` flips), so a CTA never overwrites a slot
// another CTA may still be reading.  sh: BLOCK/32 + 1 doubles, red: 4.
template <int BLOCK, int K>
__device__ __forceinline__ void grid_sums(double (&x)[K], double* parts, int& buf, double* sh,
                                          double* red, cooperative_groups::grid_group& grid) {
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = block_sum<BLOCK>(x[k], sh);  // thread 0
  double* P = parts + (size_t)buf * gridDim.x * 4;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) P[blockIdx.x * 4 + k] = x[k];
  }
  grid.sync();
  static_assert(BLOCK >= 32 * K, "one warp per component");
  if (threadIdx.x < 32 * K) {  // warp k adds component k; loads unrolled ahead of the adds
    const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double t = 0.0;
#pragma unroll 8
    for (int b = lane; b < (int)gridDim.x; b += 32) t += __ldcg(P + b * 4 + k);
    t = warp_allsum(t);
    if (lane == 0) red[k] = t;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = red[k];
  __syncthreads();
  buf ^= 1;
}

// Ticket: returns true in exactly one block (the last to arrive) after all
// blocks have published their partials.  The ticket is reset for reuse.
__device__ __forceinline__ bool last_block_arrive(unsigned int* ticket) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int t = atomicAdd(ticket, 1u);
    am_last = (t == gridDim.x - 1);
    if (am_last) *ticket = 0u;
  }
  __syncthreads();
  if (am_last) __threadfence();
  return am_last;
}

// Fixed-order reduction of `count` partials laid out with stride `stride`
// (component c of block b at partials[b*stride + c]).  Called by one block.
template <int BLOCK>
__device__ __forceinline__ double reduce_partials(const double* partials, int count, int stride,
                                                  int c, double* sh) {
  double acc = 0.0;
  for (int b = threadIdx.x; b < count; b += BLOCK) acc += __ldcg(partials + (size_t)b * stride + c);
  return block_sum<BLOCK>(acc, sh, true);
}

// Copies `count` doubles global -> shared with TMA bulk copies
// (cp.async.bulk ... mbarrier::complete_tx), issued by one thread; every
// thread of the block returns once the bytes have landed.  `src` must be
// 16-byte aligned (cudaMalloc'd vectors are).
__device__ __forceinline__ void bulk_stage_f64(double* dst, const double* src, long long count) {
  __shared__ __align__(8) unsigned long long mbar;
  const long long full = count & ~1LL;  // 16-byte multiple handled by TMA
  const unsigned bytes = (unsigned)(full * 8);
  const unsigned mb = (unsigned)__cvta_generic_to_shared(&mbar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(bytes)
                 : "memory");
    const unsigned d0 = (unsigned)__cvta_generic_to_shared(dst);
    constexpr unsigned kPiece = 32768;
    for (unsigned off = 0; off < bytes; off += kPiece) {
      const unsigned sz = bytes - off < kPiece ? bytes - off : kPiece;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              d0 + off),
          "l"((const char*)src + off), "r"(sz), "r"(mb)
          : "memory");
    }
    if (full < count) dst[full] = src[full];
  }
  __syncthreads();
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(mb)
        : "memory");
  }
  __syncthreads();
}

// ---- mbarrier + 1-D TMA bulk copy primitives (sm_90+/sm_100a PTX) --------
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(unsigned long long* bar, unsigned parity) {
  const unsigned mb = smem_addr(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(mb), "r"(parity)
        : "memory");
  }
}
// global -> shared bulk copy (TMA, non-tensor); bytes % 16 == 0, both ends 16-B aligned.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// 2-D TMA tensor load of the box at coordinates {c0 (innermost), c1}.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(smem_addr(bar))
      : "memory");
}

// ---- programmatic dependent launch (PDL) ------------------------------------
// Kernels of the solve sequence start with pdl_wait() (no access to a
// predecessor's output before it) and call pdl_trigger() once every CTA has
// started, so the next kernel's launch overlaps this one's tail.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();  // TRON_B200_PDL=0 turns the launch attribute off

// A failed launch raises TRON_ERR_CUDA (engine.cpp) instead of leaving the
// device scalars the host reads next at their previous values.
[[noreturn]] void launch_failed(cudaError_t e, const char* what);
// cudaFuncAttributeMaxDynamicSharedMemorySize >= bytes for `func` on the
// CURRENT device (the attribute is per device); idempotent, thread-safe.
void ensure_max_dynamic_smem(const void* func, int bytes);

// <<<>>> with the programmatic-stream-serialization attribute (when enabled).
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  if (e != cudaSuccess) launch_failed(e, "cudaLaunchKernelEx");
}

// After a <<<>>> launch: raise on a launch-configuration error.
#define TB_LAUNCH_CHECK()                                            \
  do {                                                               \
    const cudaError_t tb_e_ = cudaPeekAtLastError();                 \
    if (tb_e_ != cudaSuccess) ::tb::launch_failed(tb_e_, "launch");  \
  } while (0)

}  // namespace tb
