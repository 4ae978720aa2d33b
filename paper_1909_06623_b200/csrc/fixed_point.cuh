// fixed_point.cuh -- exact, order-independent accumulation of FP64 partial sums in 128-bit fixed
// point (three int64 limbs per value, integer atomics): the symmetric RPY kernel (rpy.cu) and the
// fast summation's near field (fmm.cu).
#pragma once

#include <cstdint>

#include "sc_internal.h"

namespace sc {

// Exact, order-independent accumulation of partial sums (the symmetric RPY
// kernel and the fast summation's symmetric near field): every partial sum v (a CTA's forward sum
// for one of its target rows, or its reverse sum for one of its source rows) is rounded ONCE to the fixed-point integer X = round(v 2^s)
// (|X| < 2^100 by the choice of s, fx_shift) and added with integer atomics into three int64
// limbs per (row, component): X = x2 2^86 + x1 2^43 + x0, 0 <= x0, x1 < 2^43.  Integer addition
// is associative, so the sums -- hence U -- are bitwise independent of the CTA schedule and of
// the number of GPUs (the limbs of every rank are all-reduced exactly as int64); each limb sum
// stays below 2^63 for up to 2^20 contributions per row.  Memory: 72 B per row (O(N)), instead
// of one double slot per (partner super-block, row) (O(N^2/512)).
struct FxScale {
  unsigned long long maxf_bits;    // max_j |f_j| (components), as the bits of a non-negative double
  unsigned long long maxinva_bits; // max_j 1/a_j
  int32_t bad;                     // a non-finite partial sum was met
  int32_t pad;
};
constexpr long long kM43 = (1LL << 43) - 1;

// s such that any row sum (npad sources, each |T_ij f_j| <= 2 max|f| / a_min per component) is
// below 2^100 in magnitude after scaling by 2^s.
__device__ __forceinline__ int fx_shift(const FxScale* fs, int64_t npad) {
  const double mf = __longlong_as_double(static_cast<long long>(fs->maxf_bits));
  const double mi = __longlong_as_double(static_cast<long long>(fs->maxinva_bits));
  const double B = 2.0 * mf * mi * static_cast<double>(npad);
  if (!(B > 0.0) || !isfinite(B)) return 0;
  int sh = 100 - (ilogb(B) + 1);
  return sh < -1000 ? -1000 : (sh > 1000 ? 1000 : sh);
}
__device__ __forceinline__ double pow2(int k) {  // exact 2^k, |k| <= 1000
  const int h = k / 2;
  return __longlong_as_double(static_cast<long long>(1023 + h) << 52) *
         __longlong_as_double(static_cast<long long>(1023 + k - h) << 52);
}
// v 2^s rounded to the nearest integer (ties away from zero) in 128-bit two's complement, as limbs
__device__ __forceinline__ void fx_limbs(double v, double scale, long long& x0, long long& x1, long long& x2,
                                         bool& bad) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v * scale));
  const int e = static_cast<int>((b >> 52) & 0x7ff);
  unsigned __int128 X = 0;
  if (e == 0x7ff) {
    bad = true;  // NaN / Inf
  } else if (e != 0) {
    const unsigned long long m = (b & ((1ull << 52) - 1)) | (1ull << 52);
    const int sh = e - 1075;  // |v 2^s| = m 2^sh
    if (sh > 48) {
      bad = true;  // outside the bound of fx_shift (cannot happen for finite inputs)
    } else if (sh >= 0) {
      X = static_cast<unsigned __int128>(m) << sh;
    } else if (sh >= -53) {
      X = (m + (1ull << (-sh - 1))) >> (-sh);
    }
  }
  const __int128 Xs = (b >> 63) ? -static_cast<__int128>(X) : static_cast<__int128>(X);
  x0 = static_cast<long long>(Xs & kM43);
  x1 = static_cast<long long>((Xs >> 43) & kM43);
  x2 = static_cast<long long>(Xs >> 86);
}
__device__ __forceinline__ void fx_red3(long long* acc /* [3 comps][3 limbs] */, double vx, double vy, double vz,
                                        double scale, bool& bad) {
  SC_DCHECK(acc != nullptr);
  const double v[3] = {vx, vy, vz};
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    long long x0, x1, x2;
    fx_limbs(v[c], scale, x0, x1, x2, bad);
    unsigned long long* a = reinterpret_cast<unsigned long long*>(acc + 3 * c);
    if (x0) atomicAdd(a + 0, static_cast<unsigned long long>(x0));  // RED.E.ADD.64 (no return)
    if (x1) atomicAdd(a + 1, static_cast<unsigned long long>(x1));
    if (x2) atomicAdd(a + 2, static_cast<unsigned long long>(x2));
  }
}
// limb sums -> double (carry-normalised; one rounding), times 2^-s
__device__ __forceinline__ double fx_value(const long long* l, double inv_scale) {
  long long S0 = l[0], S1 = l[1], S2 = l[2];
  long long c = S0 >> 43;
  S0 &= kM43;
  S1 += c;
  c = S1 >> 43;
  S1 &= kM43;
  S2 += c;
  const long long hi = S2 * (1LL << 43) + S1;  // |S2| <= 2^14
  return fma(static_cast<double>(hi), 0x1p43, static_cast<double>(S0)) * inv_scale;
}


}  // namespace sc
