// rpy.cu -- all-pairs Rotne-Prager-Yamakawa mobility apply, FP64, sm_100a.
//
// U_i = F_i/(6 pi mu a_i) + sum_{j != i} T(r_ij; abar) F_j   (BASELINE.json configs[0], [1])
//   r >= 2 abar: T = (1/(8 pi mu r)) [ (1 + 2 abar^2/(3 r^2)) I + (1 - 2 abar^2/r^2) rhat rhat^T ]
//   r <  2 abar: T = (1/(6 pi mu abar)) [ (1 - 9 r/(32 abar)) I + (3 r/(32 abar)) rhat rhat^T ]
// The paper's MVOP cost is dominated by this apply.
//
// Design:
//  * FP64 CUDA-core arithmetic (not a dense contraction: no tensor cores).
//  * Per pair, with d = x_j - x_i and the global factor 1/(8 pi mu) hoisted:
//      far : c1 = 1/r + (2/3) a^2 / r^3,  c2 = (1/r^3)(1 - 2 a^2/r^2)
//      near: c1 = (4/(3 abar))(1 - 9 r/(32 abar)),  c2 = 1/(8 abar^2 r)
//      U_i += c1 f_j + c2 (d . f_j) d
//    The near formula at r = 0 (with 1/r -> 0) is exactly the self block I/(6 pi mu a_i).
//  * 1/sqrt(r^2): MUFU.RSQ64H seed (2^-20) + one cubic correction -> 2^-52.
//  * Two kernels compute the sum:
//    - rpy_sym_kernel (default for N >= 4,096): each UNORDERED pair once, feeding both
//      bodies (36 FP64 instructions per unordered pair); super-block pairs of 512 x 512, source
//      super-block by one TMA bulk copy, 4 targets per lane in registers, the source's reverse
//      accumulator carried by a warp rotation; near and self pairs by a high-word r^2 clamp
//      swapped for the overlap branch in the combine; partials per (partner, row) slot summed in
//      a fixed order (deterministic, the same for any number of GPUs up to the final all-reduce).
//    - rpy_partial_kernel (small N, or forced; the bitwise P-invariant multi-GPU unit): target
//      rows x all sources, 4 targets x 2 sources interleaved per thread, sources through two
//      TMA-fed shared-memory stages, near pairs zeroed and added from the near list by the
//      combine; the source range is split into nsplit chunks (grid.y) chosen from N only.
//  * Accuracy: plain FP64 sums inside a tile, compensated (TwoSum) across tiles / splits / slots.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <functional>
#include <vector>

#include "fixed_point.cuh"
#include "rpy_common.cuh"
#include "sc_internal.h"

namespace sc {
namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra.uni DONE_%=;\n"
      "bra.uni LAB_WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

struct Consts {
  double k23a2;   // (2/3) a^2          (mono)
  double m2a2;    // -2 a^2             (mono)
  double kn1;     // 4/(3a)             (mono, near)
  double kn2;     // -9/(32a)           (mono, near)
  double kn3;     // 1/(8 a^2)          (mono, near)
  long long near_bits;  // bits of (2a)^2  (mono)
  int tau_hi;           // high word of (2a)^2 (mono; symmetric kernel's clamp)
};

// Far-field contributions of TPT targets x SU sources, branch-free and written stage by
// stage over the KK = TPT*SU independent pair chains so the FP64 instruction stream
// interleaves them (the pipe is latency-bound on a single chain):
//   acc_t += c1 f + c2 (d.f) d  with the far coefficients, or nothing when the pair is
//   "near" (r < 2 abar, which includes the self pair r = 0).  Near pairs are in the
//   near list built with the contacts (same predicate, rpy_common.cuh); rpy_combine adds
//   their overlap-branch contribution.  c1 = c2 = 0 is selected with FSEL (not the FP64
//   pipe), which also discards the NaN that rsqrt(0) produces for the self pair.
template <bool POLY, int TPT, int SU>
__device__ __forceinline__ void rpy_far_block(const double4 (&p)[TPT], const double4* __restrict__ tp,
                                              const double4* __restrict__ tf, int q, const Consts& k,
                                              double (&ax)[TPT], double (&ay)[TPT], double (&az)[TPT]) {
  constexpr int KK = TPT * SU;
  double4 pj[SU], fj[SU];
#pragma unroll
  for (int u = 0; u < SU; ++u) {
    pj[u] = tp[q + u];
    fj[u] = tf[q + u];
  }
  double dx[KK], dy[KK], dz[KK], r2[KK], y[KK], h[KK], e[KK], c1[KK], c2[KK];
#pragma unroll
  for (int c = 0; c < KK; ++c) {
    const int t = c % TPT, u = c / TPT;
    r2[c] = rpy_r2(p[t], pj[u], dx[c], dy[c], dz[c]);
  }
#pragma unroll
  for (int c = 0; c < KK; ++c) asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y[c]) : "d"(r2[c]));
  // cubic correction e = 1 - r2 y^2, rinv = y + y e (1/2 + 3e/8): 2^-20 -> 2^-52
#pragma unroll
  for (int c = 0; c < KK; ++c) h[c] = r2[c] * y[c];
#pragma unroll
  for (int c = 0; c < KK; ++c) e[c] = fma(-h[c], y[c], 1.0);
#pragma unroll
  for (int c = 0; c < KK; ++c) {
    h[c] = fma(0.375, e[c], 0.5);
    e[c] = y[c] * e[c];
  }
#pragma unroll
  for (int c = 0; c < KK; ++c) y[c] = fma(e[c], h[c], y[c]);  // rinv
#pragma unroll
  for (int c = 0; c < KK; ++c) h[c] = y[c] * y[c];  // rinv^2
#pragma unroll
  for (int c = 0; c < KK; ++c) e[c] = y[c] * h[c];  // rinv^3
  bool nr[KK];
  if (POLY) {
#pragma unroll
    for (int c = 0; c < KK; ++c) {
      const int t = c % TPT, u = c / TPT;
      const double abar = p[t].w + pj[u].w;  // (a_i + a_j)/2 from stored half radii
      const double abar2 = abar * abar;
      const double s = abar2 * h[c];
      c1[c] = y[c] * fma(s, 2.0 / 3.0, 1.0);
      c2[c] = e[c] * fma(s, -2.0, 1.0);
      nr[c] = rpy_is_near(r2[c], abar, true, 0);
    }
  } else {
#pragma unroll
    for (int c = 0; c < KK; ++c) {
      c1[c] = fma(k.k23a2, e[c], y[c]);
      c2[c] = e[c] * fma(k.m2a2, h[c], 1.0);
      nr[c] = rpy_is_near(r2[c], 0.0, false, k.near_bits);
    }
  }
#pragma unroll
  for (int c = 0; c < KK; ++c) {
    c1[c] = nr[c] ? 0.0 : c1[c];
    c2[c] = nr[c] ? 0.0 : c2[c];
  }
#pragma unroll
  for (int c = 0; c < KK; ++c) {
    const int u = c / TPT;
    h[c] = fma(dz[c], fj[u].z, fma(dy[c], fj[u].y, dx[c] * fj[u].x));  // d.f
  }
#pragma unroll
  for (int c = 0; c < KK; ++c) c2[c] *= h[c];
#pragma unroll
  for (int c = 0; c < KK; ++c) {
    const int t = c % TPT, u = c / TPT;
    ax[t] = fma(c2[c], dx[c], fma(c1[c], fj[u].x, ax[t]));
    ay[t] = fma(c2[c], dy[c], fma(c1[c], fj[u].y, ay[t]));
    az[t] = fma(c2[c], dz[c], fma(c1[c], fj[u].z, az[t]));
  }
}

// grid: (row blocks of kRpyRows, nsplit).  block: kRpyThreads (= kRpyRows / kRpyTpt).
// dynamic smem: 2 stages x (positions, forces) x kRpyTile double4 + 2 mbarriers.
template <bool POLY>
__global__ void __launch_bounds__(kRpyThreads)
    rpy_partial_kernel(const double4* __restrict__ pos4, const double4* __restrict__ f4, int64_t npad, int64_t n,
                       int64_t src_per_split, int64_t row0, int64_t nrows, Consts k,
                       double* __restrict__ part, const int32_t* __restrict__ done, int32_t* err) {
  constexpr int TPT = kRpyTpt, NT = kRpyThreads, SU = kRpySu;
  if (done != nullptr && *done) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double4* sp = reinterpret_cast<double4*>(smem_raw);        // [2][kRpyTile] positions
  double4* sf = sp + 2 * kRpyTile;                            // [2][kRpyTile] forces
  uint64_t* bar = reinterpret_cast<uint64_t*>(sf + 2 * kRpyTile);

  const int tid = threadIdx.x;
  const int split = blockIdx.y;
  const int64_t rloc = static_cast<int64_t>(blockIdx.x) * kRpyRows;  // row offset within [row0, row0+nrows)
  const int64_t s0 = static_cast<int64_t>(split) * src_per_split;
  int64_t s1 = s0 + src_per_split;
  if (s1 > npad) s1 = npad;
  const int ntiles = s0 < s1 ? static_cast<int>((s1 - s0) / kRpyTile) : 0;

  double4 p[TPT];
#pragma unroll
  for (int t = 0; t < TPT; ++t) p[t] = pos4[row0 + rloc + tid + t * NT];
  constexpr uint32_t kTileBytes = kRpyTile * sizeof(double4);

  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (int t = 0; t < 2 && t < ntiles; ++t) {
      mbar_expect_tx(&bar[t], 2 * kTileBytes);
      tma_load_1d(sp + t * kRpyTile, pos4 + s0 + static_cast<int64_t>(t) * kRpyTile, kTileBytes, &bar[t]);
      tma_load_1d(sf + t * kRpyTile, f4 + s0 + static_cast<int64_t>(t) * kRpyTile, kTileBytes, &bar[t]);
    }
  }

  double hx[TPT], hy[TPT], hz[TPT], lx[TPT], ly[TPT], lz[TPT];
#pragma unroll
  for (int t = 0; t < TPT; ++t) hx[t] = hy[t] = hz[t] = lx[t] = ly[t] = lz[t] = 0.0;
  for (int tl = 0; tl < ntiles; ++tl) {
    const int st = tl & 1;
    mbar_wait(&bar[st], (tl >> 1) & 1);
    const double4* tp = sp + st * kRpyTile;
    const double4* tf = sf + st * kRpyTile;
    double ax[TPT], ay[TPT], az[TPT];
#pragma unroll
    for (int t = 0; t < TPT; ++t) ax[t] = ay[t] = az[t] = 0.0;
#pragma unroll 1
    for (int q = 0; q < kRpyTile; q += SU) rpy_far_block<POLY, TPT, SU>(p, tp, tf, q, k, ax, ay, az);
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      two_sum_acc(hx[t], lx[t], ax[t]);
      two_sum_acc(hy[t], ly[t], ay[t]);
      two_sum_acc(hz[t], lz[t], az[t]);
    }
    __syncthreads();  // every thread is done with stage st
    if (tid == 0 && tl + 2 < ntiles) {
      const int64_t sb = s0 + static_cast<int64_t>(tl + 2) * kRpyTile;
      mbar_expect_tx(&bar[st], 2 * kTileBytes);
      tma_load_1d(sp + st * kRpyTile, pos4 + sb, kTileBytes, &bar[st]);
      tma_load_1d(sf + st * kRpyTile, f4 + sb, kTileBytes, &bar[st]);
    }
  }
  // partial layout: [split][row][3], row relative to row0
  double* o = part + (static_cast<int64_t>(split) * nrows + rloc) * 3;
#pragma unroll
  for (int t = 0; t < TPT; ++t) {
    const int r = tid + t * NT;
    o[r * 3 + 0] = hx[t] + lx[t];
    o[r * 3 + 1] = hy[t] + ly[t];
    o[r * 3 + 2] = hz[t] + lz[t];
  }
}

// U4[row0 + r] = scale * (sum_s part[s][r]  +  self term  +  overlap-branch terms of the
// near list), summed in a fixed order with TwoSum.  Near pair (r < 2 abar):
//   T = (1/(6 pi mu abar)) [(1 - 9r/(32 abar)) I + (3/(32 abar)) d d^T / r]
// i.e. with the 1/(8 pi mu) factor hoisted, c1 = (4/(3 abar))(1 - 9r/(32 abar)),
// c2 = 1/(8 abar^2 r); the self pair (r = 0) gives c1 = 4/(3 a_i), the self mobility.
template <bool POLY>
__global__ void rpy_combine_kernel(const double* __restrict__ part, int nsplit, int64_t row0, int64_t nrows,
                                   int64_t n, double scale, const double4* __restrict__ pos4,
                                   const double4* __restrict__ f4, const int32_t* __restrict__ near_ptr,
                                   const int32_t* __restrict__ near_idx, double4* __restrict__ u4,
                                   const int32_t* __restrict__ done, int32_t* __restrict__ err) {
  if (done != nullptr && *done) return;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  double hx = 0, hy = 0, hz = 0, lx = 0, ly = 0, lz = 0;
  for (int s = 0; s < nsplit; ++s) {
    const double* p = part + (static_cast<int64_t>(s) * nrows + r) * 3;
    two_sum_acc(hx, lx, p[0]);
    two_sum_acc(hy, ly, p[1]);
    two_sum_acc(hz, lz, p[2]);
  }
  const int64_t row = row0 + r;
  if (row >= n) {
    u4[row] = make_double4(0.0, 0.0, 0.0, 0.0);
    return;
  }
  const double4 pi = pos4[row];
  const double4 fi = f4[row];
  const double cs = (2.0 / 3.0) / pi.w;  // 4/(3 a_i), w = a_i/2
  two_sum_acc(hx, lx, cs * fi.x);
  two_sum_acc(hy, ly, cs * fi.y);
  two_sum_acc(hz, lz, cs * fi.z);
  const double a_mono = 2.0 * pi.w;
  const long long near_bits = __double_as_longlong(4.0 * (a_mono * a_mono));
  for (int32_t e = near_ptr[row]; e < near_ptr[row + 1]; ++e) {
    const int32_t j = near_idx[e];
    const double4 pj = pos4[j];
    const double4 fj = f4[j];
    double dx, dy, dz;
    const double r2 = rpy_r2(pi, pj, dx, dy, dz);
    const double abar = POLY ? pi.w + pj.w : a_mono;
    if (!rpy_is_near(r2, abar, POLY, near_bits)) continue;  // (list built with the same predicate)
    double rr = 0.0, rs = 0.0;
    if (r2 > 0.0) {
      rs = rsqrt_dp(r2);
      rr = r2 * rs;
    } else {
      atomicExch(err, 1);  // coincident centres (reading A12)
    }
    const double ia = 1.0 / abar;
    const double c1 = (4.0 / 3.0) * ia * fma(-9.0 / 32.0 * ia, rr, 1.0);
    const double c2 = 0.125 * ia * ia * rs;
    const double t = c2 * fma(dz, fj.z, fma(dy, fj.y, dx * fj.x));
    two_sum_acc(hx, lx, fma(t, dx, c1 * fj.x));
    two_sum_acc(hy, ly, fma(t, dy, c1 * fj.y));
    two_sum_acc(hz, lz, fma(t, dz, c1 * fj.z));
  }
  u4[row] = make_double4(scale * (hx + lx), scale * (hy + ly), scale * (hz + lz), 0.0);
}

constexpr size_t kRpySmem = 4 * kRpyTile * sizeof(double4) + 2 * sizeof(uint64_t);

// ---------------------------------------------------------------------------------------
// Symmetric variant (1 GPU): the RPY pair block is symmetric, T_ij = T_ji (it depends on
// d d^T and |d|), so each unordered pair is evaluated ONCE and feeds both bodies:
//   U_i += c1 f_j + c2 (d.f_j) d,   U_j += c1 f_i + c2 (d.f_i) d.
// 36 FP64 instructions per unordered pair instead of 2 x 26.
//
// Work unit: a pair (SI, SJ), SI <= SJ, of super-blocks of kSymSB = 512 bodies.  A CTA of
// 4 warps holds the SI targets in registers (lane l of warp w: rows (w + 4m)*32 + l,
// m = 0..3) and the SJ sources (positions, forces) in shared memory (one TMA bulk copy).
// Phase p (16 of them): warp w pairs its 4 row sub-blocks with source sub-block
// cj = (w + p) mod 16 -- distinct across warps -- through 32 rotation steps: at step k lane l
// meets source (l + k) mod 32 and carries that source's accumulator U_j, passed to lane
// l - 1 by one warp shuffle per step; after 32 steps lane l holds source l's sum and adds it
// to the CTA's shared accumulator (no two warps touch one sub-block in a phase).
// SI == SJ: forward contributions only (every ordered pair of the super-block once).
// Near pairs (r < 2 abar) and the self pair are NOT tested in the loop: r^2 is clamped on its
// high word (one integer max, rpy_common.cuh) so they get a bounded far-formula value, which
// the combine swaps for the overlap branch (round-1 tuning harness: 82.9% vs 81.3% of the FP64
// peak for the compare + select form).
//
// Output: part[slot][row][3] with slot = the partner super-block: rows of SI get slot SJ
// (forward), rows of SJ get slot SI (reverse), so every (slot, row) is written exactly
// once per apply and rpy_combine sums the NS slots of a row in a fixed order.
constexpr int kSymSB = 512;                    // bodies per super-block
// (warps, targets per lane) variants with NW * TPT * 32 = kSymSB; ctx->sym_variant picks one
constexpr int kSymNsub = kSymSB / 32;          // 16 sub-blocks of 32
constexpr size_t kSymSmem = 2 * kSymSB * sizeof(double4) + 3 * kSymSB * sizeof(double) + 16;

template <bool POLY, int NW, int TPT, int MINB, int HS>
__global__ void __launch_bounds__(NW * 32, MINB)
    rpy_sym_kernel(const double4* __restrict__ pos4, const double4* __restrict__ f4, const int2* __restrict__ pairs,
                   int64_t npad, Consts k, long long* __restrict__ acc, FxScale* __restrict__ fs,
                   const int32_t* __restrict__ done) {
  constexpr int hs = HS;  // source parts per super-block pair (compile-time: no index math at HS = 1)
  static_assert(NW * TPT * 32 == kSymSB, "super-block size");
  constexpr int kSymThreads = NW * 32;
  if (done != nullptr && *done) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double4* sp = reinterpret_cast<double4*>(smem_raw);  // SJ positions
  double4* sf = sp + kSymSB;                           // SJ forces
  double* sacc = reinterpret_cast<double*>(sf + kSymSB);  // SJ reverse accumulators [kSymSB][3]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sacc + 3 * kSymSB);

  // hs > 1 (small N, one GPU): the CTA takes the source part h of SJ only (16/hs sub-blocks)
  const int2 pr = pairs[blockIdx.x / hs];
  const int h = static_cast<int>(blockIdx.x % hs);
  SC_DCHECK(pr.x >= 0 && pr.y >= 0 && (pr.x + 1) * int64_t(kSymSB) <= npad && (pr.y + 1) * int64_t(kSymSB) <= npad);
  constexpr int nph = kSymNsub / hs;
  // HS >= 8: fewer source sub-blocks than warps -> per-warp reverse accumulators
  // (NW x 512/HS x 3 doubles, within the 512 x 3 of the shared allocation)
  constexpr bool kPerWarp = nph < NW;
  static_assert(!kPerWarp || NW * (kSymSB / HS) <= kSymSB, "per-warp accumulators fit");
  const int64_t SI = pr.x, SJ = pr.y;
  const bool rev = SI != SJ;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  constexpr uint32_t kBytes = kSymSB / hs * sizeof(double4);
  const int src0 = h * (kSymSB / hs);  // first source of this part within SJ
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    mbar_expect_tx(bar, 2 * kBytes);
    tma_load_1d(sp + src0, pos4 + SJ * kSymSB + src0, kBytes, bar);
    tma_load_1d(sf + src0, f4 + SJ * kSymSB + src0, kBytes, bar);
  }
  double4 p[TPT];
  double fx[TPT], fy[TPT], fz[TPT], ax[TPT], ay[TPT], az[TPT];
#pragma unroll
  for (int m = 0; m < TPT; ++m) {
    const int64_t row = SI * kSymSB + (w + NW * m) * 32 + lane;
    p[m] = pos4[row];
    const double4 f = f4[row];
    fx[m] = f.x;
    fy[m] = f.y;
    fz[m] = f.z;
    ax[m] = ay[m] = az[m] = 0.0;
  }
  for (int q = tid; q < 3 * kSymSB; q += kSymThreads) sacc[q] = 0.0;
  mbar_wait(bar, 0);
  __syncthreads();

#pragma unroll 1
  for (int ph = 0; ph < nph; ++ph) {
    const int cj = h * nph + (w + ph) % nph;  // distinct across the 4 warps when nph >= 4
    const double4* tp = sp + cj * 32;
    const double4* tf = sf + cj * 32;
    double rx = 0.0, ry = 0.0, rz = 0.0;  // accumulator of the source this lane meets
#pragma unroll 1
    for (int st = 0; st < 32; ++st) {
      const int s = (lane + st) & 31;
      const double4 pj = tp[s];
      const double4 fj = tf[s];
      double dx[TPT], dy[TPT], dz[TPT], r2[TPT], y[TPT], h[TPT], e[TPT], c1[TPT], c2[TPT];
#pragma unroll
      for (int m = 0; m < TPT; ++m) r2[m] = rpy_r2(p[m], pj, dx[m], dy[m], dz[m]);
      // near pairs (incl. self): far formula at the clamped r^2 (rpy_common.cuh); the
      // combine swaps it for the overlap branch -- no compare/select in this loop
      double ab2[TPT];
#pragma unroll
      for (int m = 0; m < TPT; ++m) {
        if (POLY) {
          const double abar = p[m].w + pj.w;
          ab2[m] = abar * abar;
          r2[m] = rpy_clamp_r2(r2[m], rpy_tau_hi(ab2[m]));
        } else {
          r2[m] = rpy_clamp_r2(r2[m], k.tau_hi);
        }
      }
#pragma unroll
      for (int m = 0; m < TPT; ++m) asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y[m]) : "d"(r2[m]));
#pragma unroll
      for (int m = 0; m < TPT; ++m) h[m] = r2[m] * y[m];
#pragma unroll
      for (int m = 0; m < TPT; ++m) e[m] = fma(-h[m], y[m], 1.0);
#pragma unroll
      for (int m = 0; m < TPT; ++m) {
        h[m] = fma(0.375, e[m], 0.5);
        e[m] = y[m] * e[m];
      }
#pragma unroll
      for (int m = 0; m < TPT; ++m) y[m] = fma(e[m], h[m], y[m]);  // rinv
#pragma unroll
      for (int m = 0; m < TPT; ++m) h[m] = y[m] * y[m];  // rinv^2
#pragma unroll
      for (int m = 0; m < TPT; ++m) e[m] = y[m] * h[m];  // rinv^3
#pragma unroll
      for (int m = 0; m < TPT; ++m) {
        if (POLY) {
          const double s2 = ab2[m] * h[m];
          c1[m] = y[m] * fma(s2, 2.0 / 3.0, 1.0);
          c2[m] = e[m] * fma(s2, -2.0, 1.0);
        } else {
          c1[m] = fma(k.k23a2, e[m], y[m]);
          c2[m] = e[m] * fma(k.m2a2, h[m], 1.0);
        }
      }
      // forward: U_i += c1 f_j + c2 (d.f_j) d
#pragma unroll
      for (int m = 0; m < TPT; ++m) {
        const double t = c2[m] * fma(dz[m], fj.z, fma(dy[m], fj.y, dx[m] * fj.x));
        ax[m] = fma(t, dx[m], fma(c1[m], fj.x, ax[m]));
        ay[m] = fma(t, dy[m], fma(c1[m], fj.y, ay[m]));
        az[m] = fma(t, dz[m], fma(c1[m], fj.z, az[m]));
      }
      if (rev) {  // reverse: U_j += c1 f_i + c2 (d.f_i) d  (same T: even in d)
#pragma unroll
        for (int m = 0; m < TPT; ++m) {
          const double t = c2[m] * fma(dz[m], fz[m], fma(dy[m], fy[m], dx[m] * fx[m]));
          rx = fma(t, dx[m], fma(c1[m], fx[m], rx));
          ry = fma(t, dy[m], fma(c1[m], fy[m], ry));
          rz = fma(t, dz[m], fma(c1[m], fz[m], rz));
        }
        const int src = (lane + 1) & 31;  // next step this lane meets the source lane+1 met now
        rx = __shfl_sync(0xffffffffu, rx, src);
        ry = __shfl_sync(0xffffffffu, ry, src);
        rz = __shfl_sync(0xffffffffu, rz, src);
      }
    }
    if (rev) {  // after 32 steps lane l holds source l's sum
      if (kPerWarp) {  // small parts: every warp its own accumulators (warps may share a cj)
        double* a = sacc + ((w * nph + (cj - h * nph)) * 32 + lane) * 3;
        a[0] += rx;
        a[1] += ry;
        a[2] += rz;
      } else {
        double* a = sacc + (cj * 32 + lane) * 3;
        a[0] += rx;
        a[1] += ry;
        a[2] += rz;
        __syncthreads();
      }
    }
  }
  // forward sums (rows of SI) and reverse sums (rows of part h of SJ) -> fixed-point limbs
  const double scale = pow2(fx_shift(fs, npad));
  bool bad = false;
#pragma unroll
  for (int m = 0; m < TPT; ++m) {
    const int64_t row = SI * kSymSB + (w + NW * m) * 32 + lane;
    fx_red3(acc + row * 9, ax[m], ay[m], az[m], scale, bad);
  }
  if (rev) {
    __syncthreads();
    constexpr int kPart = kSymSB / HS;
    for (int q = tid; q < kPart; q += kSymThreads) {
      double v[3];
      if (kPerWarp) {  // fixed order over the warps' accumulators
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          double t = 0.0;
#pragma unroll
          for (int ww = 0; ww < NW; ++ww) t += sacc[ww * 3 * kPart + 3 * q + c];
          v[c] = t;
        }
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) v[c] = sacc[3 * (src0 + q) + c];
      }
      fx_red3(acc + (SJ * kSymSB + src0 + q) * 9, v[0], v[1], v[2], scale, bad);
    }
  }
  if (bad) fs->bad = 1;
}

// max_j |f_j| and max_j 1/a_j (for the fixed-point scale); fs zeroed before the launch
__global__ void fx_prep_kernel(const double4* __restrict__ pos4, const double4* __restrict__ f4, int64_t npad,
                               FxScale* __restrict__ fs, const int32_t* __restrict__ done) {
  if (done != nullptr && *done) return;
  double mf = 0.0, mi = 0.0;
  for (int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b < npad;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double4 f = f4[b];
    mf = fmax(mf, fmax(fabs(f.x), fmax(fabs(f.y), fabs(f.z))));
    mi = fmax(mi, 0.5 / pos4[b].w);  // w = a/2
  }
  if (!(mf <= 1.7e308)) mf = 1.7e308;  // NaN / Inf forces: the kernel flags them (fx_limbs)
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    mf = fmax(mf, __shfl_xor_sync(0xffffffffu, mf, o));
    mi = fmax(mi, __shfl_xor_sync(0xffffffffu, mi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&fs->maxf_bits, static_cast<unsigned long long>(__double_as_longlong(mf)));
    atomicMax(&fs->maxinva_bits, static_cast<unsigned long long>(__double_as_longlong(mi)));
  }
}

}  // namespace

bool rpy_use_sym(const sc_ctx* ctx) {
  if (ctx->rpy_mode == 1) return false;
  if (ctx->rpy_mode == 2) return true;
  // auto: enough super-blocks to fill the machine (the fixed-point accumulators are O(N): no
  // memory limit beyond the bodies themselves)
  return ctx->npad >= 8 * kSymSB;
}

// Cyclic-half assignment of super-block pairs: super-block S evaluates (S, S) and
// (S, S+d mod NS) for d in D(S) = {1 .. (NS-1)/2} (+ {NS/2} if NS is even and S < NS/2).
// Every unordered pair appears exactly once and every S carries ~NS/2 pairs, so a
// contiguous range of super-blocks per rank balances the ranks.  The orientation of a
// pair (which side is "SI") depends on NS only, so the slot contents -- and with one GPU
// or an emulated world the result -- are the same for any number of ranks.
static bool sym_in_D(int64_t S, int64_t d, int64_t NS) {
  if (d <= 0 || d >= NS) return false;
  if (d <= (NS - 1) / 2) return true;
  return NS % 2 == 0 && d == NS / 2 && S < NS / 2;
}
__device__ __forceinline__ bool sym_in_D_dev(int64_t S, int64_t d, int64_t NS) {
  if (d <= 0 || d >= NS) return false;
  if (d <= (NS - 1) / 2) return true;
  return NS % 2 == 0 && d == NS / 2 && S < NS / 2;
}
static void sym_rank_range(int64_t NS, int W, int r, int64_t* s0, int64_t* s1) {
  const int64_t spr = (NS + W - 1) / W;
  *s0 = std::min<int64_t>(NS, r * spr);
  *s1 = std::min<int64_t>(NS, (r + 1) * spr);
}

}  // namespace sc

// Host-only C ABI helper (include/stokescol.h): rank r's super-block pairs of the symmetric kernel.
extern "C" int sc_sym_pair_table(int64_t nsb, int world, int rank, int32_t* pairs, int64_t* count) {
  if (nsb < 1 || world < 1 || rank < 0 || rank >= world || count == nullptr) return SC_EINVAL;
  int64_t a0, a1, k = 0;
  sc::sym_rank_range(nsb, world, rank, &a0, &a1);
  for (int64_t S = a0; S < a1; ++S)
    for (int64_t d = 0; d < nsb; ++d) {
      if (d != 0 && !sc::sym_in_D(S, d, nsb)) continue;
      if (pairs != nullptr) {
        pairs[2 * k] = static_cast<int32_t>(S);
        pairs[2 * k + 1] = static_cast<int32_t>((S + d) % nsb);
      }
      ++k;
    }
  *count = k;
  return SC_OK;
}

namespace sc {

// Combine for the symmetric kernel: the row's exact fixed-point sum (all ranks' contributions
// after the int64 all-reduce), then the self term and the near-list swap (TwoSum), scaled by
// 1/(8 pi mu).  Reads the limbs and zeroes them for the next apply.
template <bool POLY>
__global__ void rpy_sym_combine_kernel(long long* __restrict__ acc, const FxScale* __restrict__ fs, int64_t npad,
                                       int64_t n, double scale, const double4* __restrict__ pos4,
                                       const double4* __restrict__ f4, const int32_t* __restrict__ near_ptr,
                                       const int32_t* __restrict__ near_idx, double4* __restrict__ out,
                                       const int32_t* __restrict__ done, int32_t* __restrict__ err) {
  if (done != nullptr && *done) return;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (row >= npad) return;
  long long* a = acc + row * 9;
  long long l[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) {
    l[k] = a[k];
    a[k] = 0;
  }
  const double inv = pow2(-fx_shift(fs, npad));
  double hx = fx_value(l + 0, inv), hy = fx_value(l + 3, inv), hz = fx_value(l + 6, inv);
  double lx = 0, ly = 0, lz = 0;
  if (row < n) {
    const double4 pi = pos4[row];
    const double4 fi = f4[row];
    const double cs = (2.0 / 3.0) / pi.w;  // self: 4/(3 a_i)
    {  // the pair loop added the clamped far formula for the self pair (d = 0): swap it
      double sx, sy, sz;
      rpy_far_clamped_contrib(0.0, 0.0, 0.0, 0.0, 2.0 * pi.w, fi, sx, sy, sz);
      two_sum_acc(hx, lx, fma(cs, fi.x, -sx));
      two_sum_acc(hy, ly, fma(cs, fi.y, -sy));
      two_sum_acc(hz, lz, fma(cs, fi.z, -sz));
    }
    const double a_mono = 2.0 * pi.w;
    const long long near_bits = __double_as_longlong(4.0 * (a_mono * a_mono));
    for (int32_t e = near_ptr[row]; e < near_ptr[row + 1]; ++e) {
      const int32_t j = near_idx[e];
      SC_DCHECK(j >= 0 && j < n && j != row);
      const double4 pj = pos4[j];
      const double4 fj = f4[j];
      double dx, dy, dz;
      const double r2 = rpy_r2(pi, pj, dx, dy, dz);
      const double abar = POLY ? pi.w + pj.w : a_mono;
      if (!rpy_is_near(r2, abar, POLY, near_bits)) continue;
      double rr = 0.0, rs = 0.0;
      if (r2 > 0.0) {
        rs = rsqrt_dp(r2);
        rr = r2 * rs;
      } else {
        atomicExch(err, 1);  // coincident centres (reading A12)
      }
      const double ia = 1.0 / abar;
      const double c1 = (4.0 / 3.0) * ia * fma(-9.0 / 32.0 * ia, rr, 1.0);
      const double c2 = 0.125 * ia * ia * rs;
      const double t = c2 * fma(dz, fj.z, fma(dy, fj.y, dx * fj.x));
      double fx_, fy_, fz_;  // minus what the pair loop added for this pair
      rpy_far_clamped_contrib(dx, dy, dz, r2, abar, fj, fx_, fy_, fz_);
      two_sum_acc(hx, lx, fma(t, dx, fma(c1, fj.x, -fx_)));
      two_sum_acc(hy, ly, fma(t, dy, fma(c1, fj.y, -fy_)));
      two_sum_acc(hz, lz, fma(t, dz, fma(c1, fj.z, -fz_)));
    }
  }
  const double nan = __longlong_as_double(0x7ff8000000000000LL);
  out[row] = fs->bad ? make_double4(nan, nan, nan, 0.0)  // non-finite forces: propagate (SC_ENONFINITE)
             : row < n ? make_double4(scale * (hx + lx), scale * (hy + ly), scale * (hz + lz), 0.0)
                       : make_double4(0.0, 0.0, 0.0, 0.0);
}

static Consts make_consts(double a) {
  Consts k;
  k.k23a2 = 2.0 / 3.0 * a * a;
  k.m2a2 = -2.0 * a * a;
  k.kn1 = 4.0 / (3.0 * a);
  k.kn2 = -9.0 / (32.0 * a);
  k.kn3 = 1.0 / (8.0 * a * a);
  const double n2 = 4.0 * a * a;
  k.near_bits = *reinterpret_cast<const long long*>(&n2);
  k.tau_hi = static_cast<int>(k.near_bits >> 32);
  return k;
}

int rpy_init_device(sc_ctx* ctx) {
  cudaError_t e = cudaSuccess;
#define SC_ATTR(P, NW, TPT, MINB, HS)                                                                              \
  if (e == cudaSuccess)                                                                                          \
  e = cudaFuncSetAttribute(rpy_sym_kernel<P, NW, TPT, MINB, HS>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                           kSymSmem)
  SC_ATTR(false, 4, 4, 3, 1); SC_ATTR(true, 4, 4, 3, 1); SC_ATTR(false, 4, 4, 3, 2); SC_ATTR(true, 4, 4, 3, 2);
  SC_ATTR(false, 4, 4, 3, 4); SC_ATTR(true, 4, 4, 3, 4); SC_ATTR(false, 4, 4, 3, 8); SC_ATTR(true, 4, 4, 3, 8);
  SC_ATTR(false, 8, 2, 2, 1); SC_ATTR(true, 8, 2, 2, 1); SC_ATTR(false, 16, 1, 1, 1); SC_ATTR(true, 16, 1, 1, 1);
#undef SC_ATTR
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(rpy_partial_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRpySmem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(rpy_partial_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRpySmem);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaFuncSetAttribute(rpy)");
  return 0;
}

// u4 = RPY(f4) with the symmetric kernel.  ranks: the ranks whose pairs this process
// evaluates (W = 1: everything).  mode 0: one GPU; mode 1: emulated world (every rank's pairs on
// this GPU, same accumulators); mode 2: real multi-GPU -> `reduce` all-reduces the int64 limbs
// between the pair kernel and the combine.  The result is bitwise the same in every mode.
int rpy_apply_sym(sc_ctx* ctx, const double4* f4, double mu, double4* u4, const int32_t* done, int W,
                  const std::vector<int>& ranks, int mode, const std::function<int()>& reduce) {
  const int64_t NS = ctx->npad / kSymSB;
  if (NS * kSymSB != ctx->npad) return fail(ctx, SC_EINVAL, "symmetric RPY needs npad % 512 == 0");
  if (ctx->sym_nsb != NS || ctx->sym_world != W) {  // pair tables of every rank, concatenated
    std::vector<int2> tab;
    std::vector<int64_t> off(1, 0);
    for (int r = 0; r < W; ++r) {
      int64_t a0, a1;
      sym_rank_range(NS, W, r, &a0, &a1);
      for (int64_t S = a0; S < a1; ++S) {
        tab.push_back(make_int2(static_cast<int>(S), static_cast<int>(S)));
        for (int64_t d = 1; d < NS; ++d)
          if (sym_in_D(S, d, NS)) tab.push_back(make_int2(static_cast<int>(S), static_cast<int>((S + d) % NS)));
      }
      off.push_back(static_cast<int64_t>(tab.size()));
    }
    if (int rc = ensure(ctx, ctx->sym_pairs, tab.size())) return rc;
    SC_CUDA(cudaMemcpyAsync(ctx->sym_pairs.p, tab.data(), tab.size() * sizeof(int2), cudaMemcpyHostToDevice,
                            ctx->stream));
    SC_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->sym_nsb = NS;
    ctx->sym_world = W;
    ctx->sym_off = off;
  }
  // small N: split every super-block pair's sources in hs parts so the grid fills 148 SMs x 3
  // CTAs; hs minimises the makespan ceil(units / (3 x 148 resident CTAs)) / hs, with ~2% per-unit
  // prologue cost per halving (C2: 136 pairs -> hs = 8); large N keeps hs = 1.  hs depends on N
  // only (all pairs, not this rank's), so every partial sum -- and U -- is the same for any P.
  int hs = 1;
  if (ctx->sym_hs == 1 || ctx->sym_hs == 2 || ctx->sym_hs == 4 || ctx->sym_hs == 8) {
    hs = ctx->sym_hs;
  } else if (ctx->sym_variant == 0) {
    const double units = 0.5 * static_cast<double>(NS) * static_cast<double>(NS + 1);
    const double slots = 3.0 * (ctx->num_sms > 0 ? ctx->num_sms : 148);
    double best = 1e300;
    for (int c = 1; c <= 8; c *= 2) {
      const double cost = std::ceil(units * c / slots) / c * (1.0 + 0.02 * c);
      if (cost < best) {
        best = cost;
        hs = c;
      }
    }
  }
  const int64_t npad = ctx->npad;
  const size_t nacc = static_cast<size_t>(npad) * 9;
  if (ctx->sym_acc.n < nacc || ctx->sym_acc.p == nullptr) ctx->sym_acc_dirty = true;
  if (int rc = ensure(ctx, ctx->sym_acc, nacc)) return rc;
  if (int rc = ensure(ctx, ctx->fx_scale, 4)) return rc;
  if (ctx->sym_acc_dirty)  // first use, or an apply that did not reach its combine
    SC_CUDA(cudaMemsetAsync(ctx->sym_acc.p, 0, nacc * sizeof(long long), ctx->stream));
  ctx->sym_acc_dirty = true;
  FxScale* fs = reinterpret_cast<FxScale*>(ctx->fx_scale.p);
  SC_CUDA(cudaMemsetAsync(fs, 0, sizeof(FxScale), ctx->stream));
  timer_begin(ctx, SC_K_COMBINE);
  fx_prep_kernel<<<static_cast<unsigned>(std::min<int64_t>((npad + 255) / 256, 4 * 148)), 256, 0, ctx->stream>>>(
      ctx->pos4.p, f4, npad, fs, done);
  timer_end(ctx, SC_K_COMBINE);
  if (int rc = check_launch(ctx, "fx_prep")) return rc;
  const Consts k = make_consts(ctx->a_const);
  long long* acc = ctx->sym_acc.p;
  for (int r : ranks) {
    const int64_t p0 = ctx->sym_off[r], np = ctx->sym_off[r + 1] - p0;
    if (np == 0) continue;
    const unsigned g = static_cast<unsigned>(np * hs);
    const int2* pt = ctx->sym_pairs.p + p0;
    timer_begin(ctx, SC_K_RPY);
#define SC_SYM(P, NW, TPT, MINB, HS) \
  rpy_sym_kernel<P, NW, TPT, MINB, HS><<<g, NW * 32, kSymSmem, ctx->stream>>>(ctx->pos4.p, f4, pt, npad, k, acc, fs, done)
    switch (ctx->sym_variant) {
      case 1: if (ctx->poly) SC_SYM(true, 8, 2, 2, 1); else SC_SYM(false, 8, 2, 2, 1); break;
      case 3: if (ctx->poly) SC_SYM(true, 16, 1, 1, 1); else SC_SYM(false, 16, 1, 1, 1); break;
      default:
        if (hs == 8) {
          if (ctx->poly) SC_SYM(true, 4, 4, 3, 8); else SC_SYM(false, 4, 4, 3, 8);
        } else if (hs == 4) {
          if (ctx->poly) SC_SYM(true, 4, 4, 3, 4); else SC_SYM(false, 4, 4, 3, 4);
        } else if (hs == 2) {
          if (ctx->poly) SC_SYM(true, 4, 4, 3, 2); else SC_SYM(false, 4, 4, 3, 2);
        } else {
          if (ctx->poly) SC_SYM(true, 4, 4, 3, 1); else SC_SYM(false, 4, 4, 3, 1);
        }
        break;
    }
#undef SC_SYM
    timer_end(ctx, SC_K_RPY);
    if (int rc = check_launch(ctx, "rpy_sym")) return rc;
  }
  if (mode == 2 && reduce) {
    if (int rc = reduce()) return rc;
  }
  const double scale = 1.0 / (8.0 * 3.14159265358979323846 * mu);
  const unsigned nb = static_cast<unsigned>((npad + 255) / 256);
  timer_begin(ctx, SC_K_COMBINE);
  if (ctx->poly)
    rpy_sym_combine_kernel<true><<<nb, 256, 0, ctx->stream>>>(acc, fs, npad, ctx->n, scale, ctx->pos4.p, f4,
                                                             ctx->near_ptr.p, ctx->near_idx.p, u4, done, ctx->derr);
  else
    rpy_sym_combine_kernel<false><<<nb, 256, 0, ctx->stream>>>(acc, fs, npad, ctx->n, scale, ctx->pos4.p, f4,
                                                              ctx->near_ptr.p, ctx->near_idx.p, u4, done, ctx->derr);
  timer_end(ctx, SC_K_COMBINE);
  if (int rc = check_launch(ctx, "rpy_sym_combine")) return rc;
  ctx->sym_acc_dirty = false;
  return 0;
}

namespace {
}  // namespace

int choose_nsplit(int64_t npad, int world) {
  (void)world;  // must not depend on the number of GPUs (bitwise P-invariance)
  int64_t s = npad / 128;  // >= one 128-source tile per split; small N still fills several SMs
  int ns = 1;
  while (ns * 2 <= s && ns < 32) ns *= 2;
  return ns;
}

int rpy_apply_rows(sc_ctx* ctx, const double4* f4, int64_t row0, int64_t nrows, double mu, double4* u4,
                   const int32_t* done) {
  if (nrows <= 0) return 0;
  if (nrows % kRpyRows != 0 || row0 % kRpyRows != 0) return fail(ctx, SC_EINVAL, "rpy rows not aligned");
  const int ns = ctx->nsplit;
  int64_t per = (ctx->npad + ns - 1) / ns;
  per = (per + kRpyTile - 1) / kRpyTile * kRpyTile;
  if (int rc = ensure(ctx, ctx->rpy_part, static_cast<size_t>(ns) * nrows * 3)) return rc;
  const double a = ctx->a_const;
  Consts k;
  k.k23a2 = 2.0 / 3.0 * a * a;
  k.m2a2 = -2.0 * a * a;
  k.kn1 = 4.0 / (3.0 * a);
  k.kn2 = -9.0 / (32.0 * a);
  k.kn3 = 1.0 / (8.0 * a * a);
  const double n2 = 4.0 * a * a;
  k.near_bits = *reinterpret_cast<const long long*>(&n2);
  dim3 grid(static_cast<unsigned>(nrows / kRpyRows), static_cast<unsigned>(ns));
  timer_begin(ctx, SC_K_RPY);
  if (ctx->poly)
    rpy_partial_kernel<true><<<grid, kRpyThreads, kRpySmem, ctx->stream>>>(
        ctx->pos4.p, f4, ctx->npad, ctx->n, per, row0, nrows, k, ctx->rpy_part.p, done, ctx->derr);
  else
    rpy_partial_kernel<false><<<grid, kRpyThreads, kRpySmem, ctx->stream>>>(
        ctx->pos4.p, f4, ctx->npad, ctx->n, per, row0, nrows, k, ctx->rpy_part.p, done, ctx->derr);
  timer_end(ctx, SC_K_RPY);
  if (int rc = check_launch(ctx, "rpy_partial")) return rc;
  const double scale = 1.0 / (8.0 * 3.14159265358979323846 * mu);
  timer_begin(ctx, SC_K_COMBINE);
  if (ctx->poly)
    rpy_combine_kernel<true><<<static_cast<unsigned>((nrows + 255) / 256), 256, 0, ctx->stream>>>(
        ctx->rpy_part.p, ns, row0, nrows, ctx->n, scale, ctx->pos4.p, f4, ctx->near_ptr.p, ctx->near_idx.p, u4,
        done, ctx->derr);
  else
    rpy_combine_kernel<false><<<static_cast<unsigned>((nrows + 255) / 256), 256, 0, ctx->stream>>>(
        ctx->rpy_part.p, ns, row0, nrows, ctx->n, scale, ctx->pos4.p, f4, ctx->near_ptr.p, ctx->near_idx.p, u4,
        done, ctx->derr);
  timer_end(ctx, SC_K_COMBINE);
  return check_launch(ctx, "rpy_combine");
}

}  // namespace sc
