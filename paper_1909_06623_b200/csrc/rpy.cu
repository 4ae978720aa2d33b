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
//    The near formula at r = 0 (with 1/r -> 0) is exactly the self block
//    I/(6 pi mu a_i), so the self term needs no special case.
//  * 1/sqrt(r^2): MUFU.RSQ64H seed (2^-20) + one cubic correction -> 2^-52.
//    26 DP instructions per monodisperse pair.
//  * Sources staged in shared memory by 1-D TMA bulk copies (cp.async.bulk,
//    mbarrier completion), two stages; each thread owns 2 targets.
//  * Source range split into nsplit chunks (grid.y) so the grid fills 148 SMs
//    even with few target rows per GPU; per-split partials are combined in a
//    fixed order by rpy_combine (deterministic, independent of the number of
//    GPUs).  Inside a split: plain FP64 sums over a 128-source tile, then a
//    compensated (TwoSum) add of each tile sum.
#include <cstdio>

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

__device__ __forceinline__ double rsqrt_dp(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  // cubic correction: e = 1 - x y^2, y' = y (1 + e/2 + 3 e^2/8)  (error 2^-20 -> ~2^-52)
  double h = x * y;
  double e = fma(-h, y, 1.0);
  double p = fma(0.375, e, 0.5);
  double t = y * e;
  return fma(t, p, y);
}

__device__ __forceinline__ void two_sum_acc(double& hi, double& lo, double v) {
  double s = hi + v;
  double bp = s - hi;
  double err = (hi - (s - bp)) + (v - bp);
  hi = s;
  lo += err;
}

struct Consts {
  double k23a2;   // (2/3) a^2          (mono)
  double m2a2;    // -2 a^2             (mono)
  double kn1;     // 4/(3a)             (mono, near)
  double kn2;     // -9/(32a)           (mono, near)
  double kn3;     // 1/(8 a^2)          (mono, near)
  long long near_bits;  // bits of (2a)^2  (mono)
};

// One (target, source) pair: acc += c1 f + c2 (d.f) d.
template <bool POLY>
__device__ __forceinline__ void rpy_pair(const double4& pi, const double4& pj, const double4& fj,
                                         const Consts& k, int64_t i, int64_t j, double& ax, double& ay,
                                         double& az, int32_t* err) {
  const double dx = pj.x - pi.x;
  const double dy = pj.y - pi.y;
  const double dz = pj.z - pi.z;
  const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
  const double rinv = rsqrt_dp(r2);
  const double rinv2 = rinv * rinv;
  const double rinv3 = rinv * rinv2;
  double c1, c2;
  bool near;
  double abar = 0.0, abar2 = 0.0;
  if (POLY) {
    abar = pi.w + pj.w;  // (a_i + a_j)/2 from stored half radii
    abar2 = abar * abar;
    const double s = abar2 * rinv2;
    c1 = rinv * fma(s, 2.0 / 3.0, 1.0);
    c2 = rinv3 * fma(s, -2.0, 1.0);
    near = r2 < 4.0 * abar2;
  } else {
    c1 = fma(k.k23a2, rinv3, rinv);
    c2 = rinv3 * fma(k.m2a2, rinv2, 1.0);
    near = __double_as_longlong(r2) < k.near_bits;  // r2 >= 0: integer order == numeric order
  }
  if (near) {  // overlapping pair or the self pair (rare: warp-divergent branch)
    double r, rs;
    if (r2 > 0.0) {
      r = r2 * rinv;
      rs = rinv;
    } else {
      r = 0.0;
      rs = 0.0;
      if (j != i) atomicExch(err, 1);  // coincident centres (reading A12)
    }
    if (POLY) {
      const double ia = 1.0 / abar;
      c1 = (4.0 / 3.0) * ia * fma(-9.0 / 32.0 * ia, r, 1.0);
      c2 = 0.125 * ia * ia * rs;
    } else {
      c1 = k.kn1 * fma(k.kn2, r, 1.0);
      c2 = k.kn3 * rs;
    }
  }
  const double rf = fma(dz, fj.z, fma(dy, fj.y, dx * fj.x));
  const double t = c2 * rf;
  ax = fma(t, dx, fma(c1, fj.x, ax));
  ay = fma(t, dy, fma(c1, fj.y, ay));
  az = fma(t, dz, fma(c1, fj.z, az));
}

// grid: (row blocks, nsplit).  block: kRpyThreads.  dynamic smem: 2 stages x 2 x kRpyTile double4 + bars.
template <bool POLY>
__global__ void __launch_bounds__(kRpyThreads, 3)
    rpy_partial_kernel(const double4* __restrict__ pos4, const double4* __restrict__ f4, int64_t npad,
                       int64_t src_per_split, int64_t row0, int64_t nrows, Consts k,
                       double* __restrict__ part, const int32_t* __restrict__ done, int32_t* err) {
  if (done != nullptr && *done) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double4* sp = reinterpret_cast<double4*>(smem_raw);        // [2][kRpyTile] positions
  double4* sf = sp + 2 * kRpyTile;                            // [2][kRpyTile] forces
  uint64_t* bar = reinterpret_cast<uint64_t*>(sf + 2 * kRpyTile);

  const int tid = threadIdx.x;
  const int split = blockIdx.y;
  const int64_t rloc = static_cast<int64_t>(blockIdx.x) * kRpyRows;  // row offset within [row0, row0+nrows)
  const int64_t i0 = row0 + rloc + tid;
  const int64_t i1 = i0 + kRpyThreads;
  const int64_t s0 = static_cast<int64_t>(split) * src_per_split;
  int64_t s1 = s0 + src_per_split;
  if (s1 > npad) s1 = npad;
  const int ntiles = s0 < s1 ? static_cast<int>((s1 - s0) / kRpyTile) : 0;

  const double4 p0 = pos4[i0];
  const double4 p1 = pos4[i1];
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

  double hx0 = 0, hy0 = 0, hz0 = 0, lx0 = 0, ly0 = 0, lz0 = 0;
  double hx1 = 0, hy1 = 0, hz1 = 0, lx1 = 0, ly1 = 0, lz1 = 0;
  for (int t = 0; t < ntiles; ++t) {
    const int st = t & 1;
    mbar_wait(&bar[st], (t >> 1) & 1);
    const double4* tp = sp + st * kRpyTile;
    const double4* tf = sf + st * kRpyTile;
    const int64_t jb = s0 + static_cast<int64_t>(t) * kRpyTile;
    double ax0 = 0, ay0 = 0, az0 = 0, ax1 = 0, ay1 = 0, az1 = 0;
#pragma unroll 2
    for (int q = 0; q < kRpyTile; ++q) {
      const double4 pj = tp[q];
      const double4 fj = tf[q];
      rpy_pair<POLY>(p0, pj, fj, k, i0, jb + q, ax0, ay0, az0, err);
      rpy_pair<POLY>(p1, pj, fj, k, i1, jb + q, ax1, ay1, az1, err);
    }
    two_sum_acc(hx0, lx0, ax0);
    two_sum_acc(hy0, ly0, ay0);
    two_sum_acc(hz0, lz0, az0);
    two_sum_acc(hx1, lx1, ax1);
    two_sum_acc(hy1, ly1, ay1);
    two_sum_acc(hz1, lz1, az1);
    __syncthreads();  // every thread is done with stage st
    if (tid == 0 && t + 2 < ntiles) {
      const int64_t sb = s0 + static_cast<int64_t>(t + 2) * kRpyTile;
      mbar_expect_tx(&bar[st], 2 * kTileBytes);
      tma_load_1d(sp + st * kRpyTile, pos4 + sb, kTileBytes, &bar[st]);
      tma_load_1d(sf + st * kRpyTile, f4 + sb, kTileBytes, &bar[st]);
    }
  }
  // partial layout: [split][row][3], row relative to row0
  double* o = part + (static_cast<int64_t>(split) * nrows + rloc) * 3;
  o[tid * 3 + 0] = hx0 + lx0;
  o[tid * 3 + 1] = hy0 + ly0;
  o[tid * 3 + 2] = hz0 + lz0;
  o[(tid + kRpyThreads) * 3 + 0] = hx1 + lx1;
  o[(tid + kRpyThreads) * 3 + 1] = hy1 + ly1;
  o[(tid + kRpyThreads) * 3 + 2] = hz1 + lz1;
}

// U4[row0 + r] = scale * sum_s part[s][r] in fixed split order (compensated).
__global__ void rpy_combine_kernel(const double* __restrict__ part, int nsplit, int64_t row0, int64_t nrows,
                                   int64_t n, double scale, double4* __restrict__ u4,
                                   const int32_t* __restrict__ done) {
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
  double4 u;
  if (row < n) {
    u = make_double4(scale * (hx + lx), scale * (hy + ly), scale * (hz + lz), 0.0);
  } else {
    u = make_double4(0.0, 0.0, 0.0, 0.0);
  }
  u4[row] = u;
}

constexpr size_t kRpySmem = 4 * kRpyTile * sizeof(double4) + 2 * sizeof(uint64_t);

}  // namespace

int choose_nsplit(int64_t npad, int world) {
  (void)world;  // must not depend on the number of GPUs (bitwise P-invariance)
  int64_t s = npad / 512;
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
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(rpy_partial_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRpySmem);
    cudaFuncSetAttribute(rpy_partial_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kRpySmem);
    attr_set = true;
  }
  timer_begin(ctx, SC_K_RPY);
  if (ctx->poly)
    rpy_partial_kernel<true><<<grid, kRpyThreads, kRpySmem, ctx->stream>>>(
        ctx->pos4.p, f4, ctx->npad, per, row0, nrows, k, ctx->rpy_part.p, done, ctx->derr);
  else
    rpy_partial_kernel<false><<<grid, kRpyThreads, kRpySmem, ctx->stream>>>(
        ctx->pos4.p, f4, ctx->npad, per, row0, nrows, k, ctx->rpy_part.p, done, ctx->derr);
  timer_end(ctx, SC_K_RPY);
  if (int rc = check_launch(ctx, "rpy_partial")) return rc;
  const double scale = 1.0 / (8.0 * 3.14159265358979323846 * mu);
  timer_begin(ctx, SC_K_COMBINE);
  rpy_combine_kernel<<<static_cast<unsigned>((nrows + 255) / 256), 256, 0, ctx->stream>>>(
      ctx->rpy_part.p, ns, row0, nrows, ctx->n, scale, u4, done);
  timer_end(ctx, SC_K_COMBINE);
  return check_launch(ctx, "rpy_combine");
}

}  // namespace sc
