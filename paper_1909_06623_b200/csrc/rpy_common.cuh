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

// Symmetric kernel: instead of dropping near pairs with a compare + select per pair, the
// pair loop evaluates the FAR formula for every pair at a clamped r^2:
//   r2c = (max(hi32(r2), hi32(tau)), lo32(r2)),  tau = (2 abar)^2
// (one integer max on the high word; r2c = r2 whenever r2 >= tau, since then
// hi32(r2) >= hi32(tau)).  For a near pair (r2 < tau, incl. the self pair r2 = 0) the value
// is bounded (r2c >= 2^-20-ish below tau), and the combine adds T_near(r) - T_far(r2c) for
// every near-list pair and the self pair -- recomputed by rpy_far_clamped_contrib below, so
// the clamped term cancels to rounding.  The near list keeps the predicate above.
__device__ __forceinline__ double rpy_clamp_r2(double r2, int tau_hi) {
  const int hi = max(__double2hiint(r2), tau_hi);
  return __hiloint2double(hi, __double2loint(r2));
}
// hi32((2 abar)^2) from abar^2: multiplying by 4 adds 2 to the exponent field.
__device__ __forceinline__ int rpy_tau_hi(double abar2) { return __double2hiint(abar2) + (2 << 20); }

// The far-formula contribution (scaled by 8 pi mu) the symmetric kernel adds for the pair
// (d = x_j - x_i, r2 = |d|^2, pair radius abar) with the clamp above:
//   c1 f + c2 (d.f) d,  c1 = y + (2/3) abar^2 y^3,  c2 = y^3 (1 - 2 abar^2 y^2),  y = 1/sqrt(r2c).
__device__ __forceinline__ void rpy_far_clamped_contrib(double dx, double dy, double dz, double r2, double abar,
                                                        const double4& f, double& ux, double& uy, double& uz) {
  const double abar2 = abar * abar;
  const double r2c = rpy_clamp_r2(r2, rpy_tau_hi(abar2));
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2c));
  double h = r2c * y;
  double e = fma(-h, y, 1.0);
  h = fma(0.375, e, 0.5);
  e = y * e;
  y = fma(e, h, y);
  h = y * y;
  e = y * h;
  const double s = abar2 * h;
  const double c1 = y * fma(s, 2.0 / 3.0, 1.0);
  const double c2 = e * fma(s, -2.0, 1.0);
  const double t = c2 * fma(dz, f.z, fma(dy, f.y, dx * f.x));
  ux = fma(t, dx, c1 * f.x);
  uy = fma(t, dy, c1 * f.y);
  uz = fma(t, dz, c1 * f.z);
}

__device__ __forceinline__ void two_sum_acc(double& hi, double& lo, double v) {
  const double s = hi + v;
  const double bp = s - hi;
  const double err = (hi - (s - bp)) + (v - bp);
  hi = s;
  lo += err;
}

}  // namespace sc
