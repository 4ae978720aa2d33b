// lcp_common.cuh -- fixed-order reductions shared by the LCP kernels (lcp.cu) and the
// persistent small-problem solver (persist.cu): per-CTA tree and K-FINALIZE (the BBPGD scalar
// update of Alg. 1 Steps 11-15, with reading A5's breakdown rule).
#pragma once

#include "sc_internal.h"

namespace sc {

constexpr int kR = 256;  // threads of the reduction kernels (D^T per chunk, finalize); 512 measured slower

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
__device__ __forceinline__ void finalize_scalars(const double p[4], int mode, DevScalars* s);

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

__device__ __forceinline__ void finalize_scalars(const double p[4], int mode, DevScalars* s) {
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
  if (s->fixed) {
    if (j >= s->max_iter) {
      s->done = 1;
      return;
    }
  } else if (s->conv || j >= s->max_iter) {
    s->done = 1;
    return;
  }
  const bool bb2 = s->bb_mode == 1 || (s->bb_mode == 2 && (j % 2 == 0));
  const double a_new = bb2 ? p[1] / p[2] : p[0] / p[1];
  if (p[1] > 0.0 && isfinite(a_new) && a_new > 0.0) {
    s->alpha = a_new;
  } else {
    s->breakdowns += 1;  // reading A5: keep the previous alpha
  }
}

}  // namespace sc
