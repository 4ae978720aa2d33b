// rpy_common.cuh -- device helpers shared by the RPY kernels and the near-pair list builder.
//
// The "near" predicate (r < 2 abar: the overlap branch of the RPY tensor, BASELINE.json
// configs[0]) must be evaluated with bit-identical arithmetic wherever it is used: the
// far-field kernel drops exactly the pairs the near list holds, so every pair is counted
// once.  d = x_j - x_i (IEEE subtraction is exactly antisymmetric, so the predicate is
// symmetric in i and j); r^2 by the fixed fma chain below.
#pragma once

namespace sc {

__device__ __forceinline__ double rpy_r2(const double4& pi, const double4& pj, double& dx, double& dy,
                                         double& dz) {
  dx = pj.x - pi.x;
  dy = pj.y - pi.y;
  dz = pj.z - pi.z;
  return fma(dz, dz, fma(dy, dy, dx * dx));
}

// poly: abar = w_i + w_j (stored half radii); mono: bits of (2a)^2.  r2 >= 0, so the
// integer comparison of the bit patterns is the numeric comparison.
__device__ __forceinline__ bool rpy_is_near(double r2, double abar, bool poly, long long near_bits) {
  return poly ? (r2 < 4.0 * (abar * abar)) : (__double_as_longlong(r2) < near_bits);
}

// 1/sqrt(x): MUFU.RSQ64H seed (2^-20) + one cubic correction (2^-52).
__device__ __forceinline__ double rsqrt_dp(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = x * y;
  const double e = fma(-h, y, 1.0);
  const double p = fma(0.375, e, 0.5);
  const double t = y * e;
  return fma(t, p, y);
}

__device__ __forceinline__ void two_sum_acc(double& hi, double& lo, double v) {
  const double s = hi + v;
  const double bp = s - hi;
  const double err = (hi - (s - bp)) + (v - bp);
  hi = s;
  lo += err;
}

}  // namespace sc
