// Does compute-sanitizer synccheck flag a converged block barrier on sm_100a?
// Kernel `plain`: every thread reaches __syncthreads with no branch at all.
// Kernel `loop_sum`: the grid-stride loop + warp shuffle + block tree of
// common.cuh's block_sum.  Both are race- and divergence-free by construction;
// errors reported on them are tool artifacts.
//   nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o /tmp/probe scripts/synccheck_probe.cu
#include <cstdio>
__global__ void plain(double* out) {
  __shared__ double sh[32];
  sh[threadIdx.x & 31] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = sh[5];
}
__device__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__global__ void loop_sum(const double* x, long long n, double* out) {
  __shared__ double sh[17];
  double acc = 0.0;
  for (long long j = threadIdx.x; j < n; j += blockDim.x) acc += x[j];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
  __syncwarp();
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) out[0] = t;
  }
}
int main() {
  double *x, *o;
  cudaMalloc(&x, 40 * 8);
  cudaMalloc(&o, 8 * 8);
  cudaMemset(x, 0, 40 * 8);
  plain<<<2, 512>>>(o);
  loop_sum<<<1, 512>>>(x, 40, o);
  cudaError_t e = cudaDeviceSynchronize();
  std::printf("probe done: %s\n", cudaGetErrorString(e));
  return 0;
}
