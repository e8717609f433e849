// Probe: streaming bandwidth of a persistent 1-CTA-per-SM consumer through a
// shared-memory ring, fed by (a) 1-D cp.async.bulk copies or (b) 2-D tensor
// TMA boxes, for several copy sizes and stage counts.  Build + run on a B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe scripts/tma_probe.cu -lcuda
//   /tmp/tma_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c));
}
__device__ __forceinline__ void mb_expect(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned par) {
  unsigned done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(sa(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned bytes, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(dst)),
               "l"(src), "r"(bytes), "r"(sa(b)) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int c0, int c1, unsigned long long* b) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(sa(dst)), "l"(reinterpret_cast<unsigned long long>(m)), "r"(c0), "r"(c1), "r"(sa(b)) : "memory");
}

// MODE 0: tile = NCOPY 1-D copies of (TILE/NCOPY) bytes; MODE 1: one 2-D box of TILE bytes
template <int MODE>
__global__ void __launch_bounds__(288, 1) stream_kernel(const __grid_constant__ CUtensorMap map, const char* src,
                                                        long long ntiles, int tile, int ncopy, int nst, double* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long full[8], empty[8];
  const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < nst; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long t0 = ntiles * blockIdx.x / gridDim.x, t1 = ntiles * (blockIdx.x + 1) / gridDim.x;
  const int n = (int)(t1 - t0);
  if (wid == 8) {
    if (lane == 0)
      for (int k = 0; k < n; ++k) {
        const int s = k % nst;
        if (k >= nst) mb_wait(&empty[s], ((k / nst) - 1) & 1);
        unsigned char* d = sm + (size_t)s * tile;
        mb_expect(&full[s], tile);
        const long long t = t0 + k;
        if (MODE == 0) {
          const int piece = tile / ncopy;
          for (int c = 0; c < ncopy; ++c) bulk(d + c * piece, src + t * tile + c * piece, piece, &full[s]);
        } else {
          tma2d(d, &map, 0, (int)(t * (tile / 2048)), &full[s]);
        }
      }
  } else {
    double acc = 0;
    for (int k = 0; k < n; ++k) {
      const int s = k % nst;
      mb_wait(&full[s], (k / nst) & 1);
      const double* d = reinterpret_cast<const double*>(sm + (size_t)s * tile);
      acc += d[tid];  // touch
      __syncwarp();
      if (lane == 0) mb_arrive(&empty[s]);
    }
    if (acc == 12345.678) sink[0] = acc;
  }
}

int main() {
  const long long bytes = 2LL << 30;
  char* src;
  double* sink;
  cudaMalloc(&src, bytes);
  cudaMemset(src, 0, bytes);
  cudaMalloc(&sink, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn encode = (EncodeFn)fn;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  struct Cfg { int mode, tile, ncopy, nst; };
  Cfg cfgs[] = {{0, 16384, 1, 4}, {0, 16384, 1, 8}, {0, 32768, 1, 4}, {0, 32768, 4, 4}, {0, 65536, 1, 3},
                {0, 8192, 1, 8},  {0, 16384, 8, 4}, {1, 16384, 1, 4}, {1, 32768, 1, 4}, {1, 65536, 1, 3},
                {1, 16384, 1, 8}, {0, 49152, 1, 4}};
  for (const Cfg& c : cfgs) {
    CUtensorMap map;
    const int rows_per_tile = c.tile / 2048;  // box {256 doubles, rows}
    cuuint64_t dims[2] = {256, (cuuint64_t)(bytes / 2048)};
    cuuint64_t str[1] = {2048};
    cuuint32_t box[2] = {256, (cuuint32_t)rows_per_tile};
    cuuint32_t es[2] = {1, 1};
    encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const long long ntiles = bytes / c.tile;
    const size_t smem = (size_t)c.tile * c.nst;
    auto k0 = stream_kernel<0>;
    auto k1 = stream_kernel<1>;
    cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      if (c.mode == 0)
        k0<<<sms, 288, smem>>>(map, src, ntiles, c.tile, c.ncopy, c.nst, sink);
      else
        k1<<<sms, 288, smem>>>(map, src, ntiles, c.tile, c.ncopy, c.nst, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("mode=%s tile=%6d copies=%d stages=%d : %7.1f GB/s  (%s)\n", c.mode ? "2d-tensor" : "1d-bulk", c.tile,
           c.ncopy, c.nst, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
