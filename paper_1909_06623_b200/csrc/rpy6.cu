// rpy6.cu -- NEXT row f4(ii): the full 6N RPY grand mobility, FP64, sm_100a.
//
//   U_i     = sum_j M^tt_ij F_j + M^tr_ij T_j,      Omega_i = sum_j M^rt_ij F_j + M^rr_ij T_j
// with the translational blocks of BASELINE.json configs[0] (abar = (a_i + a_j)/2, configs[1])
// and the RPY coupling blocks (reading A27; oracle.c orc_rpy6_block), r = x_i - x_j:
//   tr, rt: -c(r) [rhat]x,  c = 1/(8 pi mu r^2) (r >= 2a),  (1/(16 pi mu a^2))(r/a - 3r^2/(8a^2)) (r < 2a)
//   rr: (1/(16 pi mu r^3))(3 rhat rhat - I) (r >= 2a),
//       (1/(8 pi mu a^3))[(1 - 27r/(32a) + 5r^3/(64a^3)) I + (9r/(32a) - 3r^3/(64a^3)) rhat rhat] (r < 2a)
//   self: tt I/(6 pi mu a_i), rr I/(8 pi mu a_i^3).
// The LCP's MVOP never needs the coupling blocks (sphere columns of D carry no torque,
// P:L426-L427, so D^T M D = D^T M^tt D); this apply is used for U_ext = M F_ext (torques
// enter through tr) and for U_c = M D gamma (Omega_c through rt) -- once or twice per step.
//
// Target-row kernel: one thread per target, sources staged through shared memory in tiles of
// 128, source range split over grid.y (fills 148 SMs at small N); plain FP64 sums inside a tile,
// compensated (TwoSum) across tiles and splits, fixed order -> deterministic.  Per pair the far
// branch is branch-free; overlapping pairs (r < 2 abar) take the near branch (rare).  The factor
// 1/(8 pi mu) is applied once at the end.
#include <cmath>

#include "rpy_common.cuh"
#include "sc_internal.h"

namespace sc {
namespace {

constexpr int kT6 = 128;     // threads (targets) per CTA
constexpr int kTile6 = 128;  // sources per shared-memory tile

__global__ void __launch_bounds__(kT6) rpy6_partial_kernel(const double4* __restrict__ pos4,
                                                          const double4* __restrict__ f4,
                                                          const double4* __restrict__ t4, int64_t npad,
                                                          int64_t per_split, double* __restrict__ part,
                                                          int32_t* __restrict__ err) {
  __shared__ double4 sp[kTile6], sf[kTile6], st[kTile6];
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kT6 + threadIdx.x;
  const int split = blockIdx.y;
  const int64_t s0 = static_cast<int64_t>(split) * per_split;
  const int64_t s1 = min(npad, s0 + per_split);
  const double4 pi = pos4[i];
  double hu[3] = {0, 0, 0}, lu[3] = {0, 0, 0}, hw[3] = {0, 0, 0}, lw[3] = {0, 0, 0};
  for (int64_t sb = s0; sb < s1; sb += kTile6) {
    __syncthreads();
    for (int q = threadIdx.x; q < kTile6; q += kT6) {
      sp[q] = pos4[sb + q];
      sf[q] = f4[sb + q];
      st[q] = t4[sb + q];
    }
    __syncthreads();
    double u[3] = {0, 0, 0}, w[3] = {0, 0, 0};
#pragma unroll 2
    for (int q = 0; q < kTile6; ++q) {
      if (sb + q == i) continue;  // self blocks are added by the combine
      const double4 pj = sp[q];
      const double4 F = sf[q];
      const double4 T = st[q];
      double dx, dy, dz;
      const double r2 = rpy_r2(pi, pj, dx, dy, dz);  // d = x_j - x_i = -r_ij
      if (r2 == 0.0) {
        atomicExch(err, 1);  // coincident centres (reading A12)
        continue;
      }
      const double ab = pi.w + pj.w;  // abar from stored half radii
      const double s = rsqrt_dp(r2);  // 1/r
      const double s2 = s * s, s3 = s * s2;
      const double dF = fma(dz, F.z, fma(dy, F.y, dx * F.x));
      const double dT = fma(dz, T.z, fma(dy, T.y, dx * T.x));
      // T x d and F x d (r_ij = -d, so T x r_ij = -(T x d))
      const double tdx = T.y * dz - T.z * dy, tdy = T.z * dx - T.x * dz, tdz = T.x * dy - T.y * dx;
      const double fdx = F.y * dz - F.z * dy, fdy = F.z * dx - F.x * dz, fdz = F.x * dy - F.y * dx;
      double c1, c2, cx, rI, rR;  // tt: c1 F + c2 (d.F) d; coupling: -cx (. x d); rr: rI T + rR (d.T) d
      if (r2 >= 4.0 * (ab * ab)) {
        const double a2 = ab * ab;
        c1 = fma(2.0 / 3.0 * a2, s3, s);
        c2 = s3 * fma(-2.0 * a2, s2, 1.0);
        cx = s3;
        rI = -0.5 * s3;
        rR = 1.5 * s3 * s2;
      } else {
        const double r = r2 * s, ia = 1.0 / ab, x = r * ia;
        c1 = (4.0 / 3.0) * ia * fma(-9.0 / 32.0, x, 1.0);
        c2 = 0.125 * ia * ia * s;
        cx = 0.5 * ia * ia * x * fma(-3.0 / 8.0, x, 1.0) * s;  // (1/(2 a^2))(r/a - 3r^2/(8a^2)) / r
        const double ia3 = ia * ia * ia, x3 = x * x * x;
        rI = ia3 * (1.0 - 27.0 / 32.0 * x + 5.0 / 64.0 * x3);
        rR = ia3 * (9.0 / 32.0 * x - 3.0 / 64.0 * x3) * s2;
      }
      const double tF = c2 * dF, tT = rR * dT;
      u[0] = fma(c1, F.x, fma(tF, dx, fma(-cx, tdx, u[0])));
      u[1] = fma(c1, F.y, fma(tF, dy, fma(-cx, tdy, u[1])));
      u[2] = fma(c1, F.z, fma(tF, dz, fma(-cx, tdz, u[2])));
      w[0] = fma(rI, T.x, fma(tT, dx, fma(-cx, fdx, w[0])));
      w[1] = fma(rI, T.y, fma(tT, dy, fma(-cx, fdy, w[1])));
      w[2] = fma(rI, T.z, fma(tT, dz, fma(-cx, fdz, w[2])));
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      two_sum_acc(hu[k], lu[k], u[k]);
      two_sum_acc(hw[k], lw[k], w[k]);
    }
  }
  double* o = part + (static_cast<int64_t>(split) * npad + i) * 6;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    o[k] = hu[k] + lu[k];
    o[3 + k] = hw[k] + lw[k];
  }
}

// UW[i] = (1/(8 pi mu)) (sum over splits in order + self blocks), user layout n x 6.
__global__ void rpy6_combine_kernel(const double* __restrict__ part, int nsplit, int64_t npad, int64_t n,
                                    double scale, const double4* __restrict__ pos4, const double4* __restrict__ f4,
                                    const double4* __restrict__ t4, double* __restrict__ UW) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double h[6] = {0, 0, 0, 0, 0, 0}, l[6] = {0, 0, 0, 0, 0, 0};
  for (int s = 0; s < nsplit; ++s) {
    const double* p = part + (static_cast<int64_t>(s) * npad + i) * 6;
#pragma unroll
    for (int k = 0; k < 6; ++k) two_sum_acc(h[k], l[k], p[k]);
  }
  const double a = 2.0 * pos4[i].w;
  const double ct = (4.0 / 3.0) / a, cr = 1.0 / (a * a * a);  // x 1/(8 pi mu): 1/(6 pi mu a), 1/(8 pi mu a^3)
  const double4 F = f4[i], T = t4[i];
  two_sum_acc(h[0], l[0], ct * F.x);
  two_sum_acc(h[1], l[1], ct * F.y);
  two_sum_acc(h[2], l[2], ct * F.z);
  two_sum_acc(h[3], l[3], cr * T.x);
  two_sum_acc(h[4], l[4], cr * T.y);
  two_sum_acc(h[5], l[5], cr * T.z);
  double* o = UW + 6 * i;
#pragma unroll
  for (int k = 0; k < 6; ++k) o[k] = scale * (h[k] + l[k]);
}

}  // namespace

// UW (n x 6, device) = full RPY grand mobility applied to (f4, t4) (packed, [npad]).
int rpy6_apply(sc_ctx* ctx, const double4* f4, const double4* t4, double mu, double* UW) {
  const int64_t npad = ctx->npad, n = ctx->n;
  if (n == 0) return 0;
  int ns = 1;
  while (ns * 2 <= npad / kTile6 && ns < 16 && (npad / kT6) * ns < 4 * 148) ns *= 2;
  int64_t per = (npad + ns - 1) / ns;
  per = (per + kTile6 - 1) / kTile6 * kTile6;
  if (int rc = ensure(ctx, ctx->rpy6_part, static_cast<size_t>(ns) * npad * 6)) return rc;
  const dim3 grid(static_cast<unsigned>(npad / kT6), static_cast<unsigned>(ns));
  timer_begin(ctx, SC_K_RPY);
  rpy6_partial_kernel<<<grid, kT6, 0, ctx->stream>>>(ctx->pos4.p, f4, t4, npad, per, ctx->rpy6_part.p, ctx->derr);
  timer_end(ctx, SC_K_RPY);
  if (int rc = check_launch(ctx, "rpy6_partial")) return rc;
  const double scale = 1.0 / (8.0 * 3.14159265358979323846 * mu);
  timer_begin(ctx, SC_K_COMBINE);
  rpy6_combine_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(
      ctx->rpy6_part.p, ns, npad, n, scale, ctx->pos4.p, f4, t4, UW);
  timer_end(ctx, SC_K_COMBINE);
  return check_launch(ctx, "rpy6_combine");
}

}  // namespace sc
