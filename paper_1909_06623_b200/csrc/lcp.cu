// lcp.cu -- (a3) projection + D-gather, (a5) D^T + fused BB reductions, and the
// small kernels around the BBPGD loop (Alg. 1).
//
// K-GATHER (a3): per body b, F_b = sum_{l ∋ b} sigma_bl D_l,b gamma_l with
//   gamma_l = max(0, gamma_l^old - alpha g_l^old)   (Steps 8-9)
// recomputed identically by both incident bodies; the first body (owner)
// writes gamma_l.  For rods the 6x6 drag mobility is applied in the same
// thread (U = M_b F_b), so the rods MVOP is one gather + one D^T pass; the
// gather also writes the half rates h_e = (sigma n, sigma r x n)_e . (U, W)_b of
// the body's incidences.
// K-DT (a5): per constraint g_l = n.(U_i - U_j) + q_l (spheres) or
//   h_{e_i(l)} + h_{e_j(l)} + q_l (rods: n.(U_i - U_j) + (r_i x n).W_i - (r_j x n).W_j)
//   (Step 10), fused with the partial sums of s.s, s.y, y.y and min(gamma, g)^2
//   (Steps 11, 14-15) over a FIXED chunking: spheres, chunk c = constraints
//   whose first body lies in [256c, 256c+256); rods, 256 consecutive constraints
//   (chunk_bounds, lcp_common.cuh).  One CTA per chunk, fixed-order tree -> the sums are
//   independent of the launch shape (spheres: and of the number of GPUs).
// K-FINALIZE: one CTA sums the chunk partials in fixed order and applies the
//   BB1/BB2 update, the convergence test and the breakdown rule (reading A5).
#include <cmath>

#include "lcp_common.cuh"
#include "sc_internal.h"

namespace sc {
namespace {

#ifndef SC_RODS_PEEL
#define SC_RODS_PEEL 2  // rods half rates: a lane's first PEEL incidences issued straight-line (loads in flight)
#endif

constexpr int kT = 256;
inline unsigned nblk(int64_t n) { return static_cast<unsigned>((n + kT - 1) / kT); }

enum GatherMode { kProj = 0, kRaw = 1 };
constexpr int kLpbS = 2;  // lanes per body in the D-gather: spheres (~2.7 incidences per body)
#ifndef SC_RODS_LPB
#define SC_RODS_LPB 4
#endif
constexpr int kLpbR = SC_RODS_LPB;  // rods (~4.5 incidences per body)
enum GatherOut { kOutF4 = 0, kOutRodU = 1, kOutFT = 2 };

// LPB lanes cooperate on one body (incidences e0+k, e0+k+LPB, ...), then an xor-butterfly
// combines them (every lane ends with the same bits: a+b == b+a) -- more loads in flight
// than one serial chain per body.
template <int KIND, int MODE, int OUT, int LPB>
__global__ void __launch_bounds__(kT) gather_kernel(
    const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ inc, const double4* __restrict__ icol4,
    const double* __restrict__ a, int astride,
    const double2* __restrict__ st_old, double2* __restrict__ st_new, const DevScalars* __restrict__ dsc, int64_t n,
    int64_t nout,
    const double4* __restrict__ dir4, const double4* __restrict__ mob4, double4* __restrict__ out4,
    double* __restrict__ outFT, const int32_t* __restrict__ done, int64_t nc_chk, double* __restrict__ hout) {
  if (done != nullptr && *done) return;
  const int64_t gt = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t b = gt / LPB;
  const int k = static_cast<int>(gt % LPB);
  const bool real = b < n;
  const double alpha = MODE == kProj ? dsc->alpha : 0.0;
  double fx = 0, fy = 0, fz = 0, tx = 0, ty = 0, tz = 0;
  const int32_t e0 = real ? row_ptr[b] : 0, e1 = real ? row_ptr[b + 1] : 0;
  SC_DCHECK(e0 >= 0 && e0 <= e1 && e1 <= 2 * nc_chk);
  // rods: the body's axis and drag coefficients are independent of the incidence chain -- issue
  // their loads first so they overlap it
  double4 tb = make_double4(0, 0, 0, 0), mb = make_double4(0, 0, 0, 0);
  if (OUT == kOutRodU && real && k == 0) {
    tb = dir4[b];
    mb = mob4[b];
  }
  if (KIND == kRods && OUT == kOutRodU) {
    // the lane's first SC_RODS_PEEL incidences straight-line: their loads in flight together
    // (measured faster than an unrolled loop; keeping their columns in registers for the h pass
    // below cost occupancy: 64 -> 70 / 90 registers, slower)
    double f[6] = {0, 0, 0, 0, 0, 0};
    const double2* icr = reinterpret_cast<const double2*>(icol4);
    auto one = [&](int32_t e, double2* c) {
      const int32_t v = inc[e];
      const int32_t l = v >> 1;
      double gm;
      if (MODE == kProj) {
        const double2 s = st_old[l];
        const double x = __dsub_rn(s.x, __dmul_rn(alpha, s.y));  // Step 8
        gm = x > 0.0 ? x : 0.0;                                  // Step 9
        if ((v & 1) == 0) st_new[l].x = gm;                      // owner = first body
      } else {
        gm = a[static_cast<int64_t>(l) * astride];
      }
      c[0] = icr[3 * e];
      c[1] = icr[3 * e + 1];
      c[2] = icr[3 * e + 2];
      f[0] = fma(gm, c[0].x, f[0]);
      f[1] = fma(gm, c[0].y, f[1]);
      f[2] = fma(gm, c[1].x, f[2]);
      f[3] = fma(gm, c[1].y, f[3]);
      f[4] = fma(gm, c[2].x, f[4]);
      f[5] = fma(gm, c[2].y, f[5]);
    };
    double2 ct[3];
#pragma unroll
    for (int p = 0; p < SC_RODS_PEEL; ++p)
      if (e0 + k + p * LPB < e1) one(e0 + k + p * LPB, ct);
    for (int32_t e = e0 + k + SC_RODS_PEEL * LPB; e < e1; e += LPB) one(e, ct);
    fx = f[0]; fy = f[1]; fz = f[2]; tx = f[3]; ty = f[4]; tz = f[5];
  } else if (KIND == kRods) {  // (F, T) out: the signed columns of the incidences, streamed (assemble.cu)
    double f[6] = {0, 0, 0, 0, 0, 0};
    rods_gather_lane<LPB, MODE == kProj>(e0, e1, k, alpha, inc, a, astride, st_old, st_new,
                                         reinterpret_cast<const double2*>(icol4), f);
    fx = f[0]; fy = f[1]; fz = f[2]; tx = f[3]; ty = f[4]; tz = f[5];
  } else {
#pragma unroll 2
    for (int32_t e = e0 + k; e < e1; e += LPB) {
      const int32_t v = inc[e];
      const int32_t l = v >> 1;
      SC_DCHECK(l >= 0 && l < nc_chk);
      double gm;
      if (MODE == kProj) {
        const double2 st = st_old[l];                              // (gamma_l, g_l)
        const double x = __dsub_rn(st.x, __dmul_rn(alpha, st.y));  // gamma - alpha g (Step 8)
        gm = x > 0.0 ? x : 0.0;                                    // projection (Step 9)
        if ((v & 1) == 0) st_new[l].x = gm;                         // owner = first body
      } else {
        gm = a[static_cast<int64_t>(l) * astride];
      }
      // incidence column (signed D_l block of this body, stored in incidence order: streamed)
      const double4 nv = icol4[e];
      fx = fma(gm, nv.x, fx);
      fy = fma(gm, nv.y, fy);
      fz = fma(gm, nv.z, fz);
    }
  }
#pragma unroll
  for (int o = LPB / 2; o >= 1; o >>= 1) {
    fx += __shfl_xor_sync(0xffffffffu, fx, o);
    fy += __shfl_xor_sync(0xffffffffu, fy, o);
    fz += __shfl_xor_sync(0xffffffffu, fz, o);
    if (KIND == kRods) {
      tx += __shfl_xor_sync(0xffffffffu, tx, o);
      ty += __shfl_xor_sync(0xffffffffu, ty, o);
      tz += __shfl_xor_sync(0xffffffffu, tz, o);
    }
  }
  if (KIND == kRods && OUT == kOutRodU) {
    // the body's (U, W) from its lane 0 to every lane, then each lane writes the half rate
    // h_e = (signed column of e) . (U, W) of its incidences: D_l^T (U, W) = h_{e_i(l)} + h_{e_j(l)}
    // (the D^T pass reads 2 x 8 B per constraint instead of the columns and 2 body velocities)
    double4 U = make_double4(0, 0, 0, 0), W = U;
    if (k == 0 && real) {
      const double f[6] = {fx, fy, fz, tx, ty, tz};
      rods_drag(tb, mb, f, U, W);
    }
    const int src = static_cast<int>(threadIdx.x & 31) & ~(LPB - 1);
    U.x = __shfl_sync(0xffffffffu, U.x, src);
    U.y = __shfl_sync(0xffffffffu, U.y, src);
    U.z = __shfl_sync(0xffffffffu, U.z, src);
    W.x = __shfl_sync(0xffffffffu, W.x, src);
    W.y = __shfl_sync(0xffffffffu, W.y, src);
    W.z = __shfl_sync(0xffffffffu, W.z, src);
    const double2* icr = reinterpret_cast<const double2*>(icol4);
    auto half_rate = [&](const double2* c) {
      const double un = fma(c[1].x, U.z, fma(c[0].y, U.y, c[0].x * U.x));
      const double wr = fma(c[2].y, W.z, fma(c[2].x, W.y, c[1].y * W.x));
      return un + wr;
    };
    for (int32_t e = e0 + k; e < e1; e += LPB) {
      const double2 c[3] = {icr[3 * e], icr[3 * e + 1], icr[3 * e + 2]};
      hout[e] = half_rate(c);
    }
    // (U, W) themselves only from the raw gathers (the solve recomputes U_c from the final gamma;
    // the iteration's D^T needs only the half rates)
    if (MODE == kProj || k != 0 || b >= nout) return;
    rods_store_uw(out4, b, U, W);  // (zero for padded rows)
    return;
  }
  if (k != 0 || b >= nout) return;
  if (!real) {  // padded source rows: zero force
    if (OUT == kOutF4) out4[b] = make_double4(0, 0, 0, 0);
    return;
  }
  if (OUT == kOutF4) {
    out4[b] = make_double4(fx, fy, fz, 0.0);
  } else if (OUT == kOutFT) {
    double* o = outFT + 6 * b;
    o[0] = fx; o[1] = fy; o[2] = fz; o[3] = tx; o[4] = ty; o[5] = tz;
  }
}

__global__ void __launch_bounds__(kR) finalize_kernel(const double* __restrict__ part, int64_t nchunks, int mode,
                                                      DevScalars* __restrict__ s) {
  if (s->done) return;
  __shared__ double red[4 * kR];
  finalize_block(part, nchunks, mode, s, red);
}

// BBPGD modes on the packed state st = (gamma, g): kDtIter, kDtAlpha0, kDtG0 (warm start),
// kDtInitSt (g_0 = q); APGD modes on plain vectors: kDtInitQ, kDtGrad.
enum DtMode { kDtIter = 0, kDtAlpha0 = 1, kDtG0 = 2, kDtInitQ = 3, kDtGrad = 4, kDtInitSt = 5 };

// One CTA per chunk c in [c0, c0 + gridDim.x).  FUSE (1 GPU): the last CTA to finish
// (threadfence + counter) also runs K-FINALIZE, saving a launch per iteration; the sums are
// the same fixed-order sums as the separate finalize kernel.
template <int KIND, int MODE, bool FUSE>
__global__ void __launch_bounds__(kR) dt_kernel(
    const int32_t* __restrict__ first_ptr, int64_t n, int64_t nc, int64_t c0, const int32_t* __restrict__ ci,
    const int32_t* __restrict__ cj, const double4* __restrict__ nrm4, const double4* __restrict__ u4,
    const double* __restrict__ q, const double* __restrict__ gam_new, double* __restrict__ g_out, double2* __restrict__ st_old, double2* __restrict__ st_new,
    double* __restrict__ part, const int32_t* __restrict__ done, int64_t nchunks, DevScalars* __restrict__ sc,
    unsigned int* __restrict__ counter, const int2* __restrict__ einc, const double* __restrict__ hinc) {
  if (done != nullptr && *done) return;
  __shared__ double red[4 * kR];
  const int64_t c = c0 + blockIdx.x;
  int32_t l0, l1;
  chunk_bounds(first_ptr, n, nc, c, l0, l1);
  double p[4] = {0, 0, 0, 0};
  SC_DCHECK(l0 >= 0 && l0 <= l1 && l1 <= nc);
  for (int32_t l = l0 + threadIdx.x; l < l1; l += kR) {
    double v = 0.0;
    if (MODE != kDtInitQ && MODE != kDtInitSt) {
      if (KIND == kSpheres) {
        const int32_t i = ci[l], j = cj[l];
        SC_DCHECK(i >= 0 && i < n && j > i && j < n + SC_MAX_WALLS);
        const bool wall = j >= n;  // a wall (NEXT row f2): static, not in the mobility
        const double4 nv = nrm4[l];
        const double4 z4 = make_double4(0.0, 0.0, 0.0, 0.0);
        const double4 ui = u4[i], uj = wall ? z4 : u4[j];
        v = fma(nv.z, ui.z - uj.z, fma(nv.y, ui.y - uj.y, nv.x * (ui.x - uj.x)));
      } else {  // rods: the two half rates of the gather (e_j = -1: a wall at rest)
        const int2 ep = einc[l];
        SC_DCHECK(ep.x >= 0 && ep.x < 2 * nc && ep.y < 2 * nc);
        const double hj = ep.y >= 0 ? hinc[ep.y] : 0.0;
        v = hinc[ep.x] + hj;
      }
    }
    if (MODE == kDtIter) {
      dt_iter_terms<false>(l, v, q, st_old, st_new, p);
    } else if (MODE == kDtAlpha0) {
      const double g0 = st_old[l].y;
      p[0] = fma(g0, g0, p[0]);
      p[1] = fma(g0, v, p[1]);
    } else if (MODE == kDtG0 || MODE == kDtInitSt) {  // g0 = D^T U + q (warm start) / = q (gamma0 = 0)
      const double g = (MODE == kDtG0 ? v : 0.0) + q[l];
      st_old[l].y = g;
      const double gn = st_old[l].x;
      const double m = gn < g ? gn : g;
      p[3] = fma(m, m, p[3]);
    } else if (MODE == kDtGrad) {  // g = M x + q for x = gam_new; x.Mx, q.x, phi(x)^2 (APGD)
      const double x = gam_new[l];
      const double g = v + q[l];
      g_out[l] = g;
      const double m = x < g ? x : g;
      p[0] = fma(x, v, p[0]);
      p[1] = fma(q[l], x, p[1]);
      p[2] = fma(m, m, p[2]);
    } else {  // kDtInitQ (APGD, gamma0 = 0: g0 = q)
      const double g = q[l];
      g_out[l] = g;
      const double gn = gam_new[l];
      const double m = gn < g ? gn : g;
      p[3] = fma(m, m, p[3]);
    }
  }
  cta_reduce4_shfl(p, red);  // fixed order, one barrier; the sums in thread 0
  if (!FUSE) {
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < 4; ++k) part[c * 4 + k] = p[k];
    }
    return;
  }
  // last-CTA K-FINALIZE: only thread 0's partial stores must be ordered before its counter
  // increment (the g stores of the other threads need no fence: the next kernel sees them),
  // so one thread writes the 4 partials and fences instead of a membar in every thread
  __shared__ bool last;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) part[c * 4 + k] = p[k];
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  finalize_block(part, nchunks, MODE == kDtIter ? 0 : (MODE == kDtAlpha0 ? 1 : 2), sc, red);
  if (threadIdx.x == 0) *counter = 0u;
}

__global__ void proj_own_kernel(const double2* __restrict__ st_old, double2* __restrict__ st_new,
                                const DevScalars* __restrict__ dsc, int64_t l0, int64_t l1) {
  if (dsc->done) return;
  const int64_t l = l0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l >= l1) return;
  const double2 s = st_old[l];
  const double x = __dsub_rn(s.x, __dmul_rn(dsc->alpha, s.y));
  st_new[l].x = x > 0.0 ? x : 0.0;
}

// st = (max(0, gamma_0), 0): the projected initial guess (Step 1) into the packed state
__global__ void pack_gamma0_kernel(const double* __restrict__ gam0, int64_t nc, double2* __restrict__ st) {
  const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l >= nc) return;
  const double x = gam0[l];
  st[l] = make_double2(x > 0.0 ? x : 0.0, 0.0);
}
__global__ void unpack_state_kernel(const double2* __restrict__ st, int64_t nc, double* __restrict__ gam,
                                    double* __restrict__ g) {
  const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l >= nc) return;
  const double2 s = st[l];
  gam[l] = s.x;
  g[l] = s.y;
}

__global__ void pack_ft_kernel(const double* __restrict__ FT, int64_t n, int64_t npad, double4* __restrict__ f4,
                               double4* __restrict__ t4) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= npad) return;
  if (b < n) {
    const double* f = FT + 6 * b;
    f4[b] = make_double4(f[0], f[1], f[2], 0.0);
    t4[b] = make_double4(f[3], f[4], f[5], 0.0);
  } else {
    f4[b] = make_double4(0, 0, 0, 0);
    t4[b] = make_double4(0, 0, 0, 0);
  }
}

__global__ void unpack_spheres_kernel(const double4* __restrict__ u4, const double4* __restrict__ t4,
                                      const double4* __restrict__ pos4, double rot_scale, int64_t n,
                                      double* __restrict__ UW) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= n) return;
  const double4 u = u4[b];
  const double a = 2.0 * pos4[b].w;
  const double r = rot_scale / (a * a * a);  // W = T / (8 pi mu a^3)
  double* o = UW + 6 * b;
  o[0] = u.x; o[1] = u.y; o[2] = u.z;
  if (t4 != nullptr) {
    const double4 t = t4[b];
    o[3] = r * t.x; o[4] = r * t.y; o[5] = r * t.z;
  } else {
    o[3] = 0.0; o[4] = 0.0; o[5] = 0.0;
  }
}

__global__ void rod_drag_user_kernel(const double* __restrict__ FT, const double4* __restrict__ dir4,
                                     const double4* __restrict__ mob4, int64_t n, double* __restrict__ UW) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= n) return;
  const double* f = FT + 6 * b;
  const double4 t = dir4[b];
  const double4 m = mob4[b];
  const double tf = fma(t.z, f[2], fma(t.y, f[1], t.x * f[0]));
  const double cpar = (m.x - m.y) * tf;
  double* o = UW + 6 * b;
  o[0] = fma(m.y, f[0], cpar * t.x);
  o[1] = fma(m.y, f[1], cpar * t.y);
  o[2] = fma(m.y, f[2], cpar * t.z);
  o[3] = m.z * f[3];
  o[4] = m.z * f[4];
  o[5] = m.z * f[5];
}

__global__ void rod_unpack_kernel(const double4* __restrict__ u4, int64_t n, double* __restrict__ UW) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= n) return;
  double4 u, w;
  rods_load_uw<false>(u4, b, u, w);
  double* o = UW + 6 * b;
  o[0] = u.x; o[1] = u.y; o[2] = u.z; o[3] = w.x; o[4] = w.y; o[5] = w.z;
}

// out_l = D_l^T UW (+ gap_l * qscale if addq; minus n_k . V_k for a constraint with moving wall k)
template <int KIND>
__global__ void dt_user_kernel(const int32_t* __restrict__ ci, const int32_t* __restrict__ cj,
                               const double4* __restrict__ nrm4, const double4* __restrict__ rxn4,
                               const double* __restrict__ UW, int64_t nc, int64_t n, int addgap, double inv_dt,
                               WallRates wr, double* __restrict__ out) {
  const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l >= nc) return;
  const double zero6[6] = {0, 0, 0, 0, 0, 0};
  const double* ui = UW + 6 * static_cast<int64_t>(ci[l]);
  const double* uj = cj[l] < n ? UW + 6 * static_cast<int64_t>(cj[l]) : zero6;  // cj >= n: a wall
  const double4 nv = nrm4[l];
  double v = nv.x * (ui[0] - uj[0]) + nv.y * (ui[1] - uj[1]) + nv.z * (ui[2] - uj[2]);
  if (KIND == kRods) {
    const double4 ra = rxn4[2 * l], rb = rxn4[2 * l + 1];
    v += (ra.x * ui[3] + ra.y * ui[4] + ra.z * ui[5]) - (rb.x * uj[3] + rb.y * uj[4] + rb.z * uj[5]);
  }
  if (addgap && cj[l] >= n) v -= wr.r[cj[l] - n];  // moving boundary
  out[l] = addgap ? nv.w * inv_dt + v : v;  // q = Phi/dt + D^T U_nc
}

// The loop condition of the device-side BBPGD loop (a CUDA-graph conditional WHILE node): run the
// body again unless K-FINALIZE has set `done`.
__global__ void loop_continue_kernel(cudaGraphConditionalHandle cond, const int32_t* __restrict__ done) {
  cudaGraphSetConditional(cond, *done ? 0u : 1u);
}

__global__ void count_active_kernel(const double* __restrict__ gam, int64_t nc, int32_t* __restrict__ out) {
  __shared__ int32_t s;
  if (threadIdx.x == 0) s = 0;
  __syncthreads();
  int32_t c = 0;
  for (int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; l < nc;
       l += static_cast<int64_t>(gridDim.x) * blockDim.x)
    c += gam[l] > 0.0 ? 1 : 0;
  atomicAdd(&s, c);
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(out, s);
}

// phi = || min(gamma, g) ||_2, one CTA, fixed order: thread t sums l = t, t + 1024,
// ..., then a fixed tree.
__global__ void __launch_bounds__(1024) minmap_kernel(const double* __restrict__ gam, const double* __restrict__ g,
                                                      int64_t nc, double* __restrict__ out) {
  __shared__ double red[1024];
  double acc = 0.0;
  for (int64_t l = threadIdx.x; l < nc; l += 1024) {
    const double m = gam[l] < g[l] ? gam[l] : g[l];
    acc = fma(m, m, acc);
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 512; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sqrt(red[0]);
}

}  // namespace

// ------------------------------------------------------------------ launchers
// Steps 8-9 + F = D gamma on the packed state: st[pp] -> st[pp ^ 1].x (owner)
int launch_gather_proj(sc_ctx* ctx, int pp, double mu) {
  (void)mu;
  const int32_t* done = &ctx->dsc->done;
  const double2* so = ctx->st[pp].p;
  double2* sn = ctx->st[pp ^ 1].p;
  timer_begin(ctx, SC_K_GATHER);
  if (ctx->kind == kSpheres)
    gather_kernel<kSpheres, kProj, kOutF4, kLpbS><<<nblk(ctx->npad * kLpbS), kT, 0, ctx->stream>>>(
        ctx->row_ptr.p, ctx->inc.p, ctx->icol4.p, nullptr, 1, so, sn, ctx->dsc, ctx->n,
        ctx->npad, nullptr, nullptr, ctx->f4.p, nullptr, done, ctx->nc, nullptr);
  else
    gather_kernel<kRods, kProj, kOutRodU, kLpbR><<<nblk(ctx->npad * kLpbR), kT, 0, ctx->stream>>>(
        ctx->row_ptr.p, ctx->inc.p, ctx->icol4.p, nullptr, 1, so, sn, ctx->dsc, ctx->n,
        ctx->npad, ctx->dir4.p, ctx->rodmob4.p, ctx->u4.p, nullptr, done, ctx->nc, ctx->hinc.p);
  timer_end(ctx, SC_K_GATHER);
  return check_launch(ctx, "gather_proj");
}

// F = D v for v[l * vstride] (vstride 2: a component of the packed state)
int launch_gather_raw(sc_ctx* ctx, const double* v, int vstride, double mu, double* FT_user, bool gated) {
  (void)mu;
  timer_begin(ctx, SC_K_GATHER);
  if (FT_user != nullptr) {
    if (ctx->kind == kSpheres)
      gather_kernel<kSpheres, kRaw, kOutFT, kLpbS><<<nblk(ctx->n * kLpbS), kT, 0, ctx->stream>>>(
          ctx->row_ptr.p, ctx->inc.p, ctx->icol4.p, v, vstride, nullptr, nullptr, ctx->dsc,
          ctx->n, ctx->n, nullptr, nullptr, nullptr, FT_user, nullptr, ctx->nc, nullptr);
    else
      gather_kernel<kRods, kRaw, kOutFT, kLpbR><<<nblk(ctx->n * kLpbR), kT, 0, ctx->stream>>>(
          ctx->row_ptr.p, ctx->inc.p, ctx->icol4.p, v, vstride, nullptr, nullptr, ctx->dsc,
          ctx->n, ctx->n, nullptr, nullptr, nullptr, FT_user, nullptr, ctx->nc, nullptr);
  } else {
    const int32_t* done = gated ? &ctx->dsc->done : nullptr;
    if (ctx->kind == kSpheres)
      gather_kernel<kSpheres, kRaw, kOutF4, kLpbS><<<nblk(ctx->npad * kLpbS), kT, 0, ctx->stream>>>(
          ctx->row_ptr.p, ctx->inc.p, ctx->icol4.p, v, vstride, nullptr, nullptr, ctx->dsc,
          ctx->n, ctx->npad, nullptr, nullptr, ctx->f4.p, nullptr, done, ctx->nc, nullptr);
    else
      gather_kernel<kRods, kRaw, kOutRodU, kLpbR><<<nblk(ctx->npad * kLpbR), kT, 0, ctx->stream>>>(
          ctx->row_ptr.p, ctx->inc.p, ctx->icol4.p, v, vstride, nullptr, nullptr, ctx->dsc,
          ctx->n, ctx->npad, ctx->dir4.p, ctx->rodmob4.p, ctx->u4.p, nullptr, done, ctx->nc, ctx->hinc.p);
  }
  timer_end(ctx, SC_K_GATHER);
  return check_launch(ctx, "gather_raw");
}

int launch_proj_own(sc_ctx* ctx, int pp, int64_t l0, int64_t l1) {
  if (l1 <= l0) return 0;
  timer_begin(ctx, SC_K_GATHER);
  proj_own_kernel<<<nblk(l1 - l0), kT, 0, ctx->stream>>>(ctx->st[pp].p, ctx->st[pp ^ 1].p, ctx->dsc, l0, l1);
  timer_end(ctx, SC_K_GATHER);
  return check_launch(ctx, "proj_own");
}

int launch_pack_gamma0(sc_ctx* ctx, const double* gam0) {
  if (ctx->nc == 0) return 0;
  timer_begin(ctx, SC_K_MISC);
  pack_gamma0_kernel<<<nblk(ctx->nc), kT, 0, ctx->stream>>>(gam0, ctx->nc, ctx->st[0].p);
  timer_end(ctx, SC_K_MISC);
  return check_launch(ctx, "pack_gamma0");
}

int launch_unpack_state(sc_ctx* ctx, int pp, double* gam, double* g) {
  if (ctx->nc == 0) return 0;
  timer_begin(ctx, SC_K_MISC);
  unpack_state_kernel<<<nblk(ctx->nc), kT, 0, ctx->stream>>>(ctx->st[pp].p, ctx->nc, gam, g);
  timer_end(ctx, SC_K_MISC);
  return check_launch(ctx, "unpack_state");
}

// D^T over chunks [c0, c1).  BBPGD modes (0 iteration, 1 alpha_0, 2 warm g_0, 5 g_0 = q) on the packed
// state st[pp] (-> st[pp ^ 1]); APGD modes (3 g = q, 4 gradient) on plain vectors x / g_out.
int launch_dt(sc_ctx* ctx, int mode, int pp, const double* x, double* g_out, int64_t c0, int64_t c1, bool fuse) {
  if (c1 <= c0) return 0;
  if (fuse && (c0 != 0 || c1 != ctx->nchunks)) return fail(ctx, SC_EINVAL, "fused finalize needs all chunks");
  const unsigned grid = static_cast<unsigned>(c1 - c0);
  const int32_t* done = &ctx->dsc->done;
  const double4* u4 = ctx->u4.p;
  double* part = ctx->chunk_part.p;
  const double* q = ctx->q.p;
  double2* so = ctx->st[pp].p;
  double2* sn = ctx->st[pp ^ 1].p;
  const int32_t* fp = ctx->kind == kRods ? nullptr : ctx->first_ptr.p;  // rods: constraint tiles
#define SC_DT(KIND, MODE)                                                                                       \
  do {                                                                                                          \
    if (fuse)                                                                                                   \
      dt_kernel<KIND, MODE, true><<<grid, kR, 0, ctx->stream>>>(fp, ctx->n, ctx->nc, c0, ctx->ci.p, ctx->cj.p,    \
                                                                ctx->nrm4.p, u4, q, x, g_out, so, sn, \
                                                                part, done, ctx->nchunks, ctx->dsc, ctx->dcount,   \
                                                                ctx->einc.p, ctx->hinc.p);                         \
    else                                                                                                        \
      dt_kernel<KIND, MODE, false><<<grid, kR, 0, ctx->stream>>>(fp, ctx->n, ctx->nc, c0, ctx->ci.p, ctx->cj.p,   \
                                                                 ctx->nrm4.p, u4, q, x, g_out, so,   \
                                                                 sn, part, done, ctx->nchunks, ctx->dsc,          \
                                                                 ctx->dcount, ctx->einc.p, ctx->hinc.p);          \
  } while (0)
#define SC_DT_ALL(KIND)                                \
  switch (mode) {                                      \
    case kDtIter: SC_DT(KIND, kDtIter); break;         \
    case kDtAlpha0: SC_DT(KIND, kDtAlpha0); break;     \
    case kDtG0: SC_DT(KIND, kDtG0); break;             \
    case kDtGrad: SC_DT(KIND, kDtGrad); break;         \
    case kDtInitSt: SC_DT(KIND, kDtInitSt); break;     \
    default: SC_DT(KIND, kDtInitQ); break;             \
  }
  timer_begin(ctx, SC_K_DT);
  if (ctx->kind == kSpheres) {
    SC_DT_ALL(kSpheres)
  } else {
    SC_DT_ALL(kRods)
  }
#undef SC_DT_ALL
#undef SC_DT
  timer_end(ctx, SC_K_DT);
  return check_launch(ctx, "dt");
}

int launch_finalize(sc_ctx* ctx, int mode, const double* part) {
  timer_begin(ctx, SC_K_FINALIZE);
  finalize_kernel<<<1, kR, 0, ctx->stream>>>(part, ctx->nchunks, mode, ctx->dsc);
  timer_end(ctx, SC_K_FINALIZE);
  return check_launch(ctx, "finalize");
}

int launch_pack_ft(sc_ctx* ctx, const double* FT, double4* f4, double4* t4) {
  timer_begin(ctx, SC_K_MISC);
  pack_ft_kernel<<<nblk(ctx->npad), kT, 0, ctx->stream>>>(FT, ctx->n, ctx->npad, f4, t4);
  timer_end(ctx, SC_K_MISC);
  return check_launch(ctx, "pack_ft");
}

int launch_unpack_uw_spheres(sc_ctx* ctx, const double4* u4, const double4* t4, double mu, double* UW) {
  if (ctx->n == 0) return 0;
  const double rot = 1.0 / (8.0 * 3.14159265358979323846 * mu);
  timer_begin(ctx, SC_K_MISC);
  unpack_spheres_kernel<<<nblk(ctx->n), kT, 0, ctx->stream>>>(u4, t4, ctx->pos4.p, rot, ctx->n, UW);
  timer_end(ctx, SC_K_MISC);
  return check_launch(ctx, "unpack_spheres");
}

int launch_rod_drag_user(sc_ctx* ctx, const double* FT, double mu, double* UW) {
  (void)mu;
  if (ctx->n == 0) return 0;
  timer_begin(ctx, SC_K_MISC);
  rod_drag_user_kernel<<<nblk(ctx->n), kT, 0, ctx->stream>>>(FT, ctx->dir4.p, ctx->rodmob4.p, ctx->n, UW);
  timer_end(ctx, SC_K_MISC);
  return check_launch(ctx, "rod_drag_user");
}

int launch_rod_unpack(sc_ctx* ctx, const double4* u4, double* UW) {
  if (ctx->n == 0) return 0;
  timer_begin(ctx, SC_K_MISC);
  rod_unpack_kernel<<<nblk(ctx->n), kT, 0, ctx->stream>>>(u4, ctx->n, UW);
  timer_end(ctx, SC_K_MISC);
  return check_launch(ctx, "rod_unpack");
}

int launch_dt_user(sc_ctx* ctx, const double* UW, double* out, const double* addq, double qscale) {
  if (ctx->nc == 0) return 0;
  const int addgap = addq != nullptr ? 1 : 0;
  WallRates wr;
  for (int k = 0; k < SC_MAX_WALLS; ++k) {  // n_k . V_k (q only; D^T itself never sees the walls)
    const double4 w = ctx->walls[k];
    const double* v = ctx->wall_vel[k];
    wr.r[k] = addgap ? (w.x * v[0] + w.y * v[1]) + w.z * v[2] : 0.0;
  }
  timer_begin(ctx, SC_K_DT);
  if (ctx->kind == kSpheres)
    dt_user_kernel<kSpheres><<<nblk(ctx->nc), kT, 0, ctx->stream>>>(ctx->ci.p, ctx->cj.p, ctx->nrm4.p, nullptr,
                                                                     UW, ctx->nc, ctx->n, addgap, qscale, wr, out);
  else
    dt_user_kernel<kRods><<<nblk(ctx->nc), kT, 0, ctx->stream>>>(ctx->ci.p, ctx->cj.p, ctx->nrm4.p,
                                                                  ctx->rxn4.p, UW, ctx->nc, ctx->n, addgap, qscale, wr,
                                                                  out);
  timer_end(ctx, SC_K_DT);
  return check_launch(ctx, "dt_user");
}

int launch_minmap(sc_ctx* ctx, const double* gam, const double* g, int64_t nc, double* out) {
  timer_begin(ctx, SC_K_MISC);
  minmap_kernel<<<1, 1024, 0, ctx->stream>>>(gam, g, nc, out);
  timer_end(ctx, SC_K_MISC);
  return check_launch(ctx, "minmap");
}

int launch_loop_continue(sc_ctx* ctx, cudaGraphConditionalHandle cond) {
  loop_continue_kernel<<<1, 1, 0, ctx->stream>>>(cond, &ctx->dsc->done);
  return check_launch(ctx, "loop_continue");
}

int launch_count_active(sc_ctx* ctx, const double* gam, int32_t* out) {
  if (ctx->nc == 0) return 0;
  timer_begin(ctx, SC_K_MISC);
  count_active_kernel<<<148, kT, 0, ctx->stream>>>(gam, ctx->nc, out);
  timer_end(ctx, SC_K_MISC);
  return check_launch(ctx, "count_active");
}

}  // namespace sc
