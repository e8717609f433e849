// Row products over the CSR (z_i = x_i . v), shared by csr_kernels.cu and
// the persistent CG kernel (csc_seg.cu).
#pragma once

#include "common.cuh"
#include "kernels.h"

namespace tb {

// Vectorised variant: lane `sub` owns groups of four consecutive entries
// (group q covers [base + 4q, base + 4q + 4), base = row start rounded down to
// a multiple of 4, entries outside the row masked), so the indices are one
// 16-byte load and the values two; NG groups per lane are in flight per step.
#ifndef TB_CSR_NG
#define TB_CSR_NG 1
#endif
#ifndef TB_CSR_STREAM_NA
#define TB_CSR_STREAM_NA 1
#endif
#if TB_CSR_STREAM_NA
#define TB_NA ".L1::no_allocate"
#else
#define TB_NA ""
#endif
__device__ __forceinline__ void ldv4i(const int* p, int& a, int& b, int& c, int& d) {
  asm volatile("ld.global.nc" TB_NA ".v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
               : "l"(p));
}
__device__ __forceinline__ void ldv2d(const double* p, double& a, double& b) {
  asm volatile("ld.global.nc" TB_NA ".v2.f64 {%0, %1}, [%2];"
               : "=d"(a), "=d"(b)
               : "l"(p));
}
#ifndef TB_LD256
#define TB_LD256 1
#endif
// four values (32 B, 32-B aligned) as one 256-bit load, L2::evict_first
__device__ __forceinline__ void ldv4d_ef(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.b64 {%0, %1, %2, %3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d)
               : "l"(p));
}
// COH: v is written inside the same (persistent) kernel by other CTAs, so it
// is read through L2 (ld.global.cg), never the non-coherent path.
template <int G, bool COH, int NG = TB_CSR_NG>
__device__ __forceinline__ double row_dot_vec(const CsrView& X, long long row, int sub,
                                              const double* __restrict__ v) {
  const int beg = X.rbeg ? X.rbeg[row] : X.ptr[row];
  const int end = X.rend ? X.rend[row] : X.ptr[row + 1];
  const int base = beg & ~3;
  double s = 0.0;
  for (int g0 = base + 4 * sub; g0 < end; g0 += 4 * G * NG) {
    int c[NG * 4];
    double a[NG * 4];
#pragma unroll
    for (int q = 0; q < NG; ++q) {
      const int k = g0 + 4 * G * q;
      if (k < end) {  // the group is inside the (16-B padded) arrays
        ldv4i(X.idx + k, c[4 * q], c[4 * q + 1], c[4 * q + 2], c[4 * q + 3]);
#if TB_LD256
        ldv4d_ef(X.val + k, a[4 * q], a[4 * q + 1], a[4 * q + 2], a[4 * q + 3]);
#else
        ldv2d(X.val + k, a[4 * q], a[4 * q + 1]);
        ldv2d(X.val + k + 2, a[4 * q + 2], a[4 * q + 3]);
#endif
      } else {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          c[4 * q + m] = 0;
          a[4 * q + m] = 0.0;
        }
      }
    }
    double b[NG * 4];
#pragma unroll
    for (int m = 0; m < NG * 4; ++m) {
      const int k = g0 + 4 * G * (m / 4) + (m % 4);
      // gathers allocate in L1 (measured: L1::no_allocate gathers, even of
      // the cold tail only, are 2-3x slower on N1/K1)
      b[m] = (k >= beg && k < end) ? (COH ? v[c[m]] : __ldg(v + c[m])) : 0.0;
    }
#pragma unroll
    for (int m = 0; m < NG * 4; ++m) {
      const int k = g0 + 4 * G * (m / 4) + (m % 4);
      if (k >= beg && k < end) s += a[m] * b[m];
    }
  }
  return s;
}

}  // namespace tb
