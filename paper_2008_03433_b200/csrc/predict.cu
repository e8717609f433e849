// predict (proj/src/model.cpp:88-117) on the device: label_i = sign(x_i . w),
// ties to +1, and the number of labels equal to y_i.
//
// Each row's score is summed sequentially in storage order, one thread per
// row, with -fmad=false (DMUL + DADD): the same rounding as the reference's
// loop, so the labels are bit-for-bit the reference's for the same w.
// Dense rows are read column-major (row i of column j at X[j*ld + i]), so
// consecutive threads read consecutive addresses.  Not on the solve's hot
// path: one pass over X per call.
#include "common.cuh"
#include "kernels.h"

namespace tb {

namespace {

constexpr int kBlock = 256;

__device__ __forceinline__ void count_correct(bool ok, unsigned long long* correct) {
  const unsigned ballot = __ballot_sync(0xffffffffu, ok);
  if ((threadIdx.x & 31) == 0 && ballot) atomicAdd(correct, (unsigned long long)__popc(ballot));
}

__global__ void __launch_bounds__(kBlock) predict_csr_kernel(CsrView X, const double* __restrict__ w,
                                                             const double* __restrict__ y,
                                                             double* __restrict__ labels,
                                                             unsigned long long* correct) {
  const long long stride = (long long)gridDim.x * kBlock;
  const long long rows_up = (X.rows + 31) / 32 * 32;  // whole warps for the ballot
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < rows_up; i += stride) {
    bool ok = false;
    if (i < X.rows) {
      double score = 0.0;
      for (int k = X.ptr[i]; k < X.ptr[i + 1]; ++k) score += X.val[k] * w[X.idx[k]];
      const double label = score < 0.0 ? -1.0 : 1.0;
      labels[i] = label;
      ok = y && y[i] == label;
    }
    count_correct(ok, correct);
  }
}

__global__ void __launch_bounds__(kBlock) predict_dense_kernel(long long l, int n, long long ld,
                                                               const double* __restrict__ X,
                                                               const double* __restrict__ w,
                                                               const double* __restrict__ y,
                                                               double* __restrict__ labels,
                                                               unsigned long long* correct) {
  const long long stride = (long long)gridDim.x * kBlock;
  const long long rows_up = (l + 31) / 32 * 32;
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < rows_up; i += stride) {
    bool ok = false;
    if (i < l) {
      double score = 0.0;
      for (int j = 0; j < n; ++j) score += X[(long long)j * ld + i] * w[j];
      const double label = score < 0.0 ? -1.0 : 1.0;
      labels[i] = label;
      ok = y && y[i] == label;
    }
    count_correct(ok, correct);
  }
}

int predict_grid(long long rows) {
  long long g = (rows + kBlock - 1) / kBlock;
  const long long cap = (long long)device_sm_count() * 8;
  if (g > cap) g = cap;
  return (int)(g > 0 ? g : 1);
}

}  // namespace

void predict_csr(const CsrView& X, const double* w, const double* y, double* labels,
                 unsigned long long* correct, cudaStream_t s) {
  cudaMemsetAsync(correct, 0, sizeof(unsigned long long), s);
  if (X.rows == 0) return;
  predict_csr_kernel<<<predict_grid(X.rows), kBlock, 0, s>>>(X, w, y, labels, correct);
  TB_LAUNCH_CHECK();
}

namespace {
__global__ void __launch_bounds__(kBlock) predict_scores_kernel(long long l, const double* __restrict__ sc,
                                                                const double* __restrict__ y,
                                                                double* __restrict__ labels,
                                                                unsigned long long* correct) {
  const long long stride = (long long)gridDim.x * kBlock;
  const long long rows_up = (l + 31) / 32 * 32;
  for (long long i = (long long)blockIdx.x * kBlock + threadIdx.x; i < rows_up; i += stride) {
    bool ok = false;
    if (i < l) {
      const double label = sc[i] < 0.0 ? -1.0 : 1.0;
      labels[i] = label;
      ok = y && y[i] == label;
    }
    count_correct(ok, correct);
  }
}
}  // namespace

void predict_from_scores(int64_t l, const double* scores, const double* y, double* labels,
                         unsigned long long* correct, cudaStream_t s) {
  cudaMemsetAsync(correct, 0, sizeof(unsigned long long), s);
  if (l == 0) return;
  predict_scores_kernel<<<predict_grid(l), kBlock, 0, s>>>(l, scores, y, labels, correct);
  TB_LAUNCH_CHECK();
}

void predict_dense(int64_t l, int64_t n, int64_t ld, const double* X, const double* w,
                   const double* y, double* labels, unsigned long long* correct, cudaStream_t s) {
  cudaMemsetAsync(correct, 0, sizeof(unsigned long long), s);
  if (l == 0) return;
  predict_dense_kernel<<<predict_grid(l), kBlock, 0, s>>>(l, (int)n, ld, X, w, y, labels, correct);
  TB_LAUNCH_CHECK();
}

}  // namespace tb
