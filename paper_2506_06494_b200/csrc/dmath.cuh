// FP64 reciprocal, division, sqrt and rsqrt on the FP64 pipe only.
//
// nvcc lowers 1.0/x and sqrt(x) to MUFU.RCP64H / MUFU.RSQ64H seeds plus
// Newton steps. On sm_100 those MUFU ops keep the XU pipe busy for ~30
// cycles per warp instruction: ncu on k_element_mplus showed the XU pipe
// 82% busy (realtime) while it issued only 2.8% of its peak instruction
// rate, with the FP64 pipe at 22%. These versions seed from the IEEE bit
// pattern with an integer subtract and refine with DFMA Newton steps, so
// they run on the FP64 pipe, which has headroom.
//
// Accuracy: a few ulp (the parity tolerances are 1e-12 relative). Domain:
// finite normal inputs (x > 0 for the square roots). Zero maps to a huge
// finite reciprocal / rsqrt rather than inf, and sqrt_nr(0) = 0.
#pragma once
#include <cmath>

namespace jgs2 {

// 1/x: seed error < 5.1%, four Newton steps (e -> e^2).
__device__ __forceinline__ double rcp_nr(double x) {
  double y = __longlong_as_double(0x7FDE6238502484BALL - __double_as_longlong(x));
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    double e = fma(-x, y, 1.0);
    y = fma(y, e, y);
  }
  return y;
}

// a/b: a * (1/b) plus one residual correction.
__device__ __forceinline__ double div_nr(double a, double b) {
  double y = rcp_nr(b);
  double q = a * y;
  double r = fma(-b, q, a);
  return fma(r, y, q);
}

// 1/sqrt(x), x > 0: seed error < 3.5%, four Newton steps (e -> 1.5 e^2).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y = __longlong_as_double(0x5FE6EB50C7B537A9LL - (__double_as_longlong(x) >> 1));
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    double e = fma(-(x * y), y, 1.0);
    y = fma(0.5 * y, e, y);
  }
  return y;
}

// sqrt(x) from y = rsqrt_nr(x): x*y plus one residual correction.
__device__ __forceinline__ double sqrt_from_rsqrt(double x, double y) {
  double s = x * y;
  double r = fma(-s, s, x);
  return fma(0.5 * y, r, s);
}

__device__ __forceinline__ double sqrt_nr(double x) { return sqrt_from_rsqrt(x, rsqrt_nr(x)); }

// Host/device spellings: the Newton forms on the device, IEEE on the host.
__host__ __device__ __forceinline__ double hd_div(double a, double b) {
#ifdef __CUDA_ARCH__
  return div_nr(a, b);
#else
  return a / b;
#endif
}
__host__ __device__ __forceinline__ double hd_rcp(double x) {
#ifdef __CUDA_ARCH__
  return rcp_nr(x);
#else
  return 1.0 / x;
#endif
}
__host__ __device__ __forceinline__ double hd_sqrt(double x) {
#ifdef __CUDA_ARCH__
  return sqrt_nr(x);
#else
  return std::sqrt(x);
#endif
}
__host__ __device__ __forceinline__ double hd_rsqrt(double x) {
#ifdef __CUDA_ARCH__
  return rsqrt_nr(x);
#else
  return 1.0 / std::sqrt(x);
#endif
}

}  // namespace jgs2
