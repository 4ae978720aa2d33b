// apgd.cu -- vector kernels of the APGD comparison solver (NEXT row f3).
//
// The paper compares BBPGD with the Accelerated Projected Gradient Descent of Mazhar et
// al. 2015: Nesterov momentum with an adaptive
// Lipschitz estimate L_k (back-tracking) and a gradient restart.  The MVOP is the same as
// BBPGD's (D-gather, mobility, D^T); these kernels are the per-constraint vector steps and
// the fixed-order reductions around it.  One GPU (replicas under a multi-GPU context).
#include "lcp_common.cuh"
#include "sc_internal.h"

namespace sc {
namespace {

constexpr int kA = 256;

__device__ __forceinline__ void reduce4(double v[4], double* red) {
  const int t = threadIdx.x;
#pragma unroll
  for (int k = 0; k < 4; ++k) red[k * kA + t] = v[k];
  __syncthreads();
  for (int w = kA / 2; w > 0; w >>= 1) {
    if (t < w) {
#pragma unroll
      for (int k = 0; k < 4; ++k) red[k * kA + t] += red[k * kA + t + w];
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) v[k] = red[k * kA];
}

// gamma_new = max(0, y - t g) (projected gradient step from the extrapolated point y);
// chunk partials: g.(gamma_new - y), |gamma_new - y|^2, g.(gamma_new - gamma), 0.
__global__ void __launch_bounds__(kA) apgd_step_kernel(const int32_t* __restrict__ first_ptr, int64_t n, int64_t nc,
                                                       const double* __restrict__ y, const double* __restrict__ g,
                                                       const double* __restrict__ gam, double t,
                                                       double* __restrict__ gam_new, double* __restrict__ part) {
  __shared__ double red[4 * kA];
  const int64_t c = blockIdx.x;
  int32_t l0, l1;
  chunk_bounds(first_ptr, n, nc, c, l0, l1);  // the chunking of the D^T kernels
  double p[4] = {0, 0, 0, 0};
  for (int32_t l = l0 + threadIdx.x; l < l1; l += kA) {
    const double x = y[l] - t * g[l];
    const double gn = x > 0.0 ? x : 0.0;
    gam_new[l] = gn;
    const double d = gn - y[l];
    p[0] = fma(g[l], d, p[0]);
    p[1] = fma(d, d, p[1]);
    p[2] = fma(g[l], gn - gam[l], p[2]);
  }
  reduce4(p, red);
  if (threadIdx.x < 4) part[c * 4 + threadIdx.x] = p[threadIdx.x];
}

// y = gamma_new + beta (gamma_new - gamma)  (Nesterov extrapolation)
__global__ void apgd_momentum_kernel(const double* __restrict__ gam_new, const double* __restrict__ gam, double beta,
                                     int64_t nc, double* __restrict__ y) {
  const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l >= nc) return;
  const double gn = gam_new[l];
  y[l] = fma(beta, gn - gam[l], gn);
}

// fixed-order sum of the chunk partials -> out[4]
__global__ void __launch_bounds__(kA) sum_chunks_kernel(const double* __restrict__ part, int64_t nchunks,
                                                        double* __restrict__ out) {
  __shared__ double red[4 * kA];
  double p[4] = {0, 0, 0, 0};
  for (int64_t c = threadIdx.x; c < nchunks; c += kA) {
#pragma unroll
    for (int k = 0; k < 4; ++k) p[k] += part[c * 4 + k];
  }
  reduce4(p, red);
  if (threadIdx.x < 4) out[threadIdx.x] = p[threadIdx.x];
}

}  // namespace

int apgd_launch_step(sc_ctx* ctx, const double* y, const double* g, const double* gam, double t, double* gam_new) {
  timer_begin(ctx, SC_K_MISC);
  const int32_t* fp = ctx->kind == kRods ? nullptr : ctx->first_ptr.p;
  apgd_step_kernel<<<static_cast<unsigned>(ctx->nchunks), kA, 0, ctx->stream>>>(fp, ctx->n, ctx->nc, y, g, gam, t,
                                                                                gam_new, ctx->chunk_part.p);
  timer_end(ctx, SC_K_MISC);
  return check_launch(ctx, "apgd_step");
}

int apgd_launch_momentum(sc_ctx* ctx, const double* gam_new, const double* gam, double beta, double* y) {
  if (ctx->nc == 0) return 0;
  timer_begin(ctx, SC_K_MISC);
  apgd_momentum_kernel<<<static_cast<unsigned>((ctx->nc + 255) / 256), 256, 0, ctx->stream>>>(gam_new, gam, beta,
                                                                                             ctx->nc, y);
  timer_end(ctx, SC_K_MISC);
  return check_launch(ctx, "apgd_momentum");
}

int launch_sum_chunks(sc_ctx* ctx, double* out4) {
  timer_begin(ctx, SC_K_FINALIZE);
  sum_chunks_kernel<<<1, kA, 0, ctx->stream>>>(ctx->chunk_part.p, ctx->nchunks, out4);
  timer_end(ctx, SC_K_FINALIZE);
  return check_launch(ctx, "sum_chunks");
}

}  // namespace sc
