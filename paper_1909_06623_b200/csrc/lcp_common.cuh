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

__device__ __forceinline__ void finalize_block(const double* part, int64_t nchunks, int mode, DevScalars* s, double* red) {
  double p[4] = {0, 0, 0, 0};
  for (int64_t c = threadIdx.x; c < nchunks; c += kR) {
#pragma unroll
    for (int k = 0; k < 4; ++k) p[k] += __ldcg(part + c * 4 + k);
  }
  block_reduce4(p, red);
  if (threadIdx.x != 0) return;
  finalize_scalars(p, mode, s);
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
