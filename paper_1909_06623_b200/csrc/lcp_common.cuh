// lcp_common.cuh -- fixed-order reductions shared by the LCP kernels (lcp.cu) and the
// persistent small-problem solver (persist.cu): per-CTA tree and K-FINALIZE (the BBPGD scalar
// update of Alg. 1 Steps 11-15, with reading A5's breakdown rule).
#pragma once

#include "sc_internal.h"

namespace sc {

constexpr int kR = 256;  // threads of the reduction kernels (D^T per chunk, finalize); 512 measured slower
constexpr int kChunkTile = 256;  // rods: a reduction chunk is a tile of 256 consecutive constraints

// Constraint range [l0, l1) of reduction chunk c.  Spheres (first_ptr != NULL): the constraints
// whose first body lies in [256c, 256c + 256) -- body-aligned, so a chunk belongs to exactly one
// rank of a multi-GPU context.  Rods (first_ptr == NULL; one GPU): 256 consecutive constraints,
// one per thread of the chunk's CTA (rods average ~2.2 constraints per body, so body chunks
// left most threads with 2-3 serial constraints and the grid with a 1.06-wave tail).
__device__ __forceinline__ void chunk_bounds(const int32_t* __restrict__ first_ptr, int64_t n, int64_t nc,
                                             int64_t c, int32_t& l0, int32_t& l1) {
  if (first_ptr == nullptr) {
    const int64_t a = c * kChunkTile, b = a + kChunkTile;
    l0 = static_cast<int32_t>(a < nc ? a : nc);
    l1 = static_cast<int32_t>(b < nc ? b : nc);
    return;
  }
  int64_t blo = c * kChunkBodies, bhi = blo + kChunkBodies;
  if (blo > n) blo = n;
  if (bhi > n) bhi = n;
  l0 = first_ptr[blo];
  l1 = first_ptr[bhi];
}

__device__ __forceinline__ void block_reduce4(double v[4], double* red /* [4][kR] smem */) {
  const int t = threadIdx.x;
#pragma unroll
  for (int k = 0; k < 4; ++k) red[k * kR + t] = v[k];
  __syncthreads();
  for (int w = kR / 2; w > 0; w >>= 1) {
    if (t < w) {
#pragma unroll
      for (int k = 0; k < 4; ++k) red[k * kR + t] += red[k * kR + t + w];
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = red[k * kR];
}

// Loads of data another CTA of the same launch may have written (persistent kernels: L1 is not
// coherent across SMs, so those go through L2 with ld.cg); plain loads elsewhere.  Same values.
template <bool CG>
__device__ __forceinline__ double ldv(const double* p) {
  return CG ? __ldcg(p) : *p;
}
template <bool CG>
__device__ __forceinline__ double4 ldv4(const double4* p) {
  if (!CG) return *p;
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = __ldcg(q), b = __ldcg(q + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

// Rods body velocities (U, W) in the velocity buffer u4 (64 B per body), packed as 3 double2
// (48 B: D^T reads 3 vector loads per body instead of 4).
__device__ __forceinline__ void rods_store_uw(double4* u4, int64_t b, const double4& U, const double4& W) {
  double2* q = reinterpret_cast<double2*>(u4) + 3 * b;
  q[0] = make_double2(U.x, U.y);
  q[1] = make_double2(U.z, W.x);
  q[2] = make_double2(W.y, W.z);
}
template <bool CG>
__device__ __forceinline__ void rods_load_uw(const double4* u4, int64_t b, double4& U, double4& W) {
  const double2* q = reinterpret_cast<const double2*>(u4) + 3 * b;
  const double2 a = CG ? __ldcg(q) : q[0], c = CG ? __ldcg(q + 1) : q[1], d = CG ? __ldcg(q + 2) : q[2];
  U = make_double4(a.x, a.y, c.x, 0.0);
  W = make_double4(c.y, d.x, d.y, 0.0);
}

// Rods, one lane of the D-gather (Steps 8-9 with PROJ): lane k of body b sums the
// incidences e0+k, e0+k+LPB, ... of gamma_l = max(0, gamma_l - alpha g_l) (PROJ; the first body
// writes gamma_l) or gamma_l = a_l (raw) times the signed column (sigma n, sigma r x n) of the
// incidence, streamed in incidence order (assemble.cu rod_incidence_columns, 3 double2 each).
template <int LPB, bool PROJ>
__device__ __forceinline__ void rods_gather_lane(int32_t e0, int32_t e1, int k, double alpha,
                                                 const int32_t* __restrict__ inc, const double* a, int astride,
                                                 const double2* st_old, double2* st_new,
                                                 const double2* __restrict__ icolr, double f[6]) {
#pragma unroll 2
  for (int32_t e = e0 + k; e < e1; e += LPB) {
    const int32_t v = inc[e];
    const int32_t l = v >> 1;
    SC_DCHECK(l >= 0);
    double gm;
    if (PROJ) {
      const double2 s = st_old[l];                                // (gamma_l, g_l): one 16-B load
      const double x = __dsub_rn(s.x, __dmul_rn(alpha, s.y));     // Step 8
      gm = x > 0.0 ? x : 0.0;                                     // Step 9
      if ((v & 1) == 0) st_new[l].x = gm;                         // owner = first body
    } else {
      gm = a[static_cast<int64_t>(l) * astride];
    }
    const double2 c0 = icolr[3 * e], c1 = icolr[3 * e + 1], c2 = icolr[3 * e + 2];
    f[0] = fma(gm, c0.x, f[0]);
    f[1] = fma(gm, c0.y, f[1]);
    f[2] = fma(gm, c1.x, f[2]);
    f[3] = fma(gm, c1.y, f[3]);
    f[4] = fma(gm, c2.x, f[4]);
    f[5] = fma(gm, c2.y, f[5]);
  }
}

// Rods drag (configs[3]): U = (1/zeta_par) t t^T F + (1/zeta_perp)(I - t t^T) F, W = T / zeta_rot;
// m = (1/zeta_par, 1/zeta_perp, 1/zeta_rot).
__device__ __forceinline__ void rods_drag(const double4& t, const double4& m, const double f[6], double4& U,
                                          double4& W) {
  const double tf = fma(t.z, f[2], fma(t.y, f[1], t.x * f[0]));
  const double cpar = (m.x - m.y) * tf;
  U = make_double4(fma(m.y, f[0], cpar * t.x), fma(m.y, f[1], cpar * t.y), fma(m.y, f[2], cpar * t.z), 0.0);
  W = make_double4(m.z * f[3], m.z * f[4], m.z * f[5], 0.0);
}
// Step 10 (g = D^T U + q, written) and the partial sums of Steps 11, 14-15 for constraint l:
// s.s, s.y, y.y, min(gamma, g)^2 with s = gamma_new - gamma_old, y = g - g_old.  The BBPGD state
// is packed per constraint, st = (gamma_l, g_l) (one 16-B access in the gathers).
template <bool CG>
__device__ __forceinline__ void dt_iter_terms(int64_t l, double v, const double* __restrict__ q,
                                              const double2* st_old, double2* st_new, double p[4]) {
  const double g = v + q[l];
  const double2 snw = CG ? __ldcg(st_new + l) : st_new[l];  // (gamma_new, -): full 16-B accesses,
  st_new[l] = make_double2(snw.x, g);                         // coalesced, instead of 8-B halves
  const double gn = snw.x;
  const double2 so = CG ? __ldcg(st_old + l) : st_old[l];
  const double s = gn - so.x;
  const double y = g - so.y;
  const double m = gn < g ? gn : g;
  p[0] = fma(s, s, p[0]);
  p[1] = fma(s, y, p[1]);
  p[2] = fma(y, y, p[2]);
  p[3] = fma(m, m, p[3]);
}

// Fixed-order CTA reduction with one barrier: shuffle-down tree in each warp, then warp 0 sums
// the warp results in order (result valid in thread 0).  red: >= 4 * (kR / 32) doubles.
__device__ __forceinline__ void cta_reduce4_shfl(double v[4], double* red) {
  constexpr int kW = kR / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) red[k * kW + w] = v[k];
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = lane < kW ? red[k * kW + lane] : 0.0;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
#pragma unroll
      for (int k = 0; k < 4; ++k) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
    }
  }
}

// Sums chunk partials in fixed order (thread t: chunks t, t+256, ...; then a fixed tree)
// and advances the BBPGD scalars.  mode 0: after Step 10 of iteration j; mode 1: alpha_0
// (Step 6); mode 2: phi_0 (Step 3).  Called by one whole CTA of kR threads.
// The scalar update of K-FINALIZE from the reduced sums p (one thread).
__device__ __forceinline__ void finalize_scalars(const double p[4], int mode, DevScalars* s, bool writer = true);

__device__ __forceinline__ void finalize_block(const double* part, int64_t nchunks, int mode, DevScalars* s, double* red,
                                               bool writer = true) {
  double p[4] = {0, 0, 0, 0};
#pragma unroll 4
  for (int64_t c = threadIdx.x; c < nchunks; c += kR) {  // (loads of several chunks in flight)
    const double2* q = reinterpret_cast<const double2*>(part + c * 4);
    const double2 a = __ldcg(q), b = __ldcg(q + 1);
    p[0] += a.x;
    p[1] += a.y;
    p[2] += b.x;
    p[3] += b.y;
  }
  block_reduce4(p, red);
  if (threadIdx.x != 0) return;
  finalize_scalars(p, mode, s, writer);
}

// writer: this copy of the scalars records the residual trace (the persistent loop runs the
// finalize redundantly in every CTA; only CTA 0 writes the trace).
__device__ __forceinline__ void finalize_scalars(const double p[4], int mode, DevScalars* s, bool writer) {
  for (int k = 0; k < 4; ++k) s->p[k] = p[k];
  if (mode == 1) {
    const double a = p[0] / p[1];  // alpha_0 = g0.g0 / g0.M g0
    if (!(isfinite(a) && a > 0.0)) {
      s->nonfinite = 1;
      s->done = 1;
    } else {
      s->alpha = a;
    }
    return;
  }
  const double phi = sqrt(p[3]);
  s->phi = phi;
  if (writer && s->trace != nullptr) {  // trace[0] = phi_0 (Step 3), trace[j] = phi_j (Step 11)
    const int k = mode == 2 ? 0 : s->iter + 1;
    if (k < s->trace_cap) s->trace[k] = phi;
  }
  if (!isfinite(phi)) {
    s->nonfinite = 1;
    s->done = 1;
    return;
  }
  s->conv = phi < s->tol ? 1 : 0;
  if (mode == 2) {
    if (s->conv) s->done = 1;
    return;
  }
  const int j = s->iter + 1;
  s->iter = j;
  if (!s->fixed && s->conv) {  // Steps 11-12: stop, gamma_j is the solution
    s->done = 1;
    return;
  }
  // Steps 14-15 (inside the loop body of Alg. 1, so also at j = j_max)
  const bool bb2 = s->bb_mode == 1 || (s->bb_mode == 2 && (j % 2 == 0));
  const double a_new = bb2 ? p[1] / p[2] : p[0] / p[1];
  if (p[1] > 0.0 && isfinite(a_new) && a_new > 0.0) {
    s->alpha = a_new;
  } else {
    s->breakdowns += 1;  // reading A5: keep the previous alpha
  }
  if (j >= s->max_iter) s->done = 1;
}

}  // namespace sc
