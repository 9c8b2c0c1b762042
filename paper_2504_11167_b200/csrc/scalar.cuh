// Scalar abstraction for the real (double) and complex (zc = complex<double>) kernels.
// The double overloads compile to exactly the arithmetic of the real-only kernels.
// Complex pivot magnitude follows LAPACK izamax: |Re| + |Im| (dcabs1).
#pragma once

#include <cuda_runtime.h>

namespace lrs {

struct __align__(16) zc {
  double x, y;  // real, imaginary
};

template <class S> struct IsC { static constexpr bool value = false; };
template <> struct IsC<zc> { static constexpr bool value = true; };

__host__ __device__ __forceinline__ double s_zero(double) { return 0.0; }
__host__ __device__ __forceinline__ zc s_zero(zc) { return {0.0, 0.0}; }
template <class S> __host__ __device__ __forceinline__ S s_real(double v);
template <> __host__ __device__ __forceinline__ double s_real<double>(double v) { return v; }
template <> __host__ __device__ __forceinline__ zc s_real<zc>(double v) { return {v, 0.0}; }

__host__ __device__ __forceinline__ double s_add(double a, double b) { return a + b; }
__host__ __device__ __forceinline__ zc s_add(zc a, zc b) { return {a.x + b.x, a.y + b.y}; }
__host__ __device__ __forceinline__ double s_sub(double a, double b) { return a - b; }
__host__ __device__ __forceinline__ zc s_sub(zc a, zc b) { return {a.x - b.x, a.y - b.y}; }
__host__ __device__ __forceinline__ double s_neg(double a) { return -a; }
__host__ __device__ __forceinline__ zc s_neg(zc a) { return {-a.x, -a.y}; }
__host__ __device__ __forceinline__ double s_conj(double a) { return a; }
__host__ __device__ __forceinline__ zc s_conj(zc a) { return {a.x, -a.y}; }
__host__ __device__ __forceinline__ double s_mul(double a, double b) { return a * b; }
__host__ __device__ __forceinline__ zc s_mul(zc a, zc b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
__host__ __device__ __forceinline__ double s_scale(double a, double s) { return a * s; }
__host__ __device__ __forceinline__ zc s_scale(zc a, double s) { return {a.x * s, a.y * s}; }
// c + a * b
__host__ __device__ __forceinline__ double s_fma(double a, double b, double c) { return fma(a, b, c); }
__host__ __device__ __forceinline__ zc s_fma(zc a, zc b, zc c) {
  return {fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y))};
}
// c + conj(a) * b
__host__ __device__ __forceinline__ double s_cfma(double a, double b, double c) { return fma(a, b, c); }
__host__ __device__ __forceinline__ zc s_cfma(zc a, zc b, zc c) {
  return {fma(a.x, b.x, fma(a.y, b.y, c.x)), fma(a.x, b.y, fma(-a.y, b.x, c.y))};
}
__host__ __device__ __forceinline__ double s_div(double a, double b) { return a / b; }
__host__ __device__ __forceinline__ zc s_div(zc a, zc b) {
  // Smith's algorithm
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, d = b.x + b.y * r;
    return {(a.x + a.y * r) / d, (a.y - a.x * r) / d};
  }
  const double r = b.x / b.y, d = b.x * r + b.y;
  return {(a.x * r + a.y) / d, (a.y * r - a.x) / d};
}
__host__ __device__ __forceinline__ double s_inv(double a) { return 1.0 / a; }
__host__ __device__ __forceinline__ zc s_inv(zc a) { return s_div(zc{1.0, 0.0}, a); }
// pivot magnitude (LAPACK idamax / izamax)
__host__ __device__ __forceinline__ double s_abs1(double a) { return fabs(a); }
__host__ __device__ __forceinline__ double s_abs1(zc a) { return fabs(a.x) + fabs(a.y); }
// |a| and |a|^2
__host__ __device__ __forceinline__ double s_abs(double a) { return fabs(a); }
// a / m for m = |a| > 0 without forming 1 / m (which overflows for a denormal m)
__host__ __device__ __forceinline__ double s_unit_phase(double a, double) { return copysign(1.0, a); }
__host__ __device__ __forceinline__ zc s_unit_phase(zc a, double m) { return {a.x / m, a.y / m}; }
__host__ __device__ __forceinline__ double s_abs(zc a) { return hypot(a.x, a.y); }
__host__ __device__ __forceinline__ double s_abs2(double a) { return a * a; }
__host__ __device__ __forceinline__ double s_abs2(zc a) { return a.x * a.x + a.y * a.y; }
__host__ __device__ __forceinline__ bool s_iszero(double a) { return a == 0.0; }
__host__ __device__ __forceinline__ bool s_iszero(zc a) { return a.x == 0.0 && a.y == 0.0; }

__device__ __forceinline__ zc warp_sum_z(zc v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  return v;
}

}  // namespace lrs
