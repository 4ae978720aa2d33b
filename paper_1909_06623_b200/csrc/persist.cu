// persist.cu -- persistent BBPGD iteration loop for small sphere problems (one GPU).
//
// For N up to a few thousand (BASELINE configs[0], C1: 512 spheres) every kernel of an
// iteration is latency-bound: the graph-replayed sequence gather -> RPY -> combine -> D^T is
// ~45 us per iteration of which the arithmetic is a few us.  Here ONE cooperative launch runs
// Steps 7-16 of Alg. 1 until convergence or j_max, the phases separated by
// grid-wide barriers instead of kernel boundaries:
//   A  projection + F = D gamma (Steps 8-9)      per body, the D-gather of lcp.cu (same order)
//   B  U = RPY(F)                                one warp per target row, lanes over sources,
//                                                overlap branch evaluated in place, self term
//   C  g = D^T U + q and the chunk partials      one CTA per 256-body chunk (same order as lcp.cu)
//   D  K-FINALIZE (alpha, phi, convergence)      every CTA, redundantly, on its own shared copy
//                                                of the scalars (identical arithmetic), so no
//                                                fourth barrier is needed
// The chunk partial sums and the finalize are the fixed-order sums of lcp.cu, so the iteration
// is deterministic; the RPY sum order differs from the tiled kernels (tolerance parity).
#include <cooperative_groups.h>

#include <algorithm>

#include "lcp_common.cuh"
#include "rpy_common.cuh"
#include "sc_internal.h"

namespace cg = cooperative_groups;

namespace sc {
namespace {

// L2 load of a double4 written by another CTA in this launch (L1 is not coherent across SMs)
__device__ __forceinline__ double4 ldcg4(const double4* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = __ldcg(q), b = __ldcg(q + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

constexpr int kPT = 256;  // threads per CTA (= kR: finalize_block and the chunk tree)
static_assert(kPT == kR, "persistent CTA size");

struct PersistArgs {
  int64_t n, npad, nc, nchunks;
  const double4* pos4;
  double4* f4;
  double4* u4;
  const int32_t* row_ptr;
  const int32_t* inc;
  const double4* icol4;
  const int32_t* first_ptr;
  const int32_t* ci;
  const int32_t* cj;
  const double4* nrm4;
  const double* q;
  double2* st0;  // packed (gamma, g) ping-pong: iteration j reads [j & 1], writes [(j & 1) ^ 1]
  double2* st1;
  double* part;
  DevScalars* sc;
  int32_t* err;
  double scale;  // 1/(8 pi mu): u4 holds U in the units of rpy.cu's combine output
};

__global__ void __launch_bounds__(kPT) bbpgd_persistent_kernel(PersistArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ DevScalars s;
  __shared__ double red[4 * kR];
  extern __shared__ double4 dyn[];  // [npad] positions, [npad] forces (phase B)
  if (threadIdx.x == 0) s = *a.sc;
  __syncthreads();
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * kPT + threadIdx.x;
  const int64_t nthreads = static_cast<int64_t>(gridDim.x) * kPT;
  const int lane = threadIdx.x & 31;
  const int64_t warp = tid >> 5, nwarps = nthreads >> 5;
  while (!s.done) {
    const int pp = s.iter & 1;
    const double2* so = pp ? a.st1 : a.st0;
    double2* sn = pp ? a.st0 : a.st1;
    const double alpha = s.alpha;
    // ---- A: projection + D-gather, 2 lanes per body (lcp.cu gather_kernel<kSpheres, kProj, kOutF4, 2>)
    for (int64_t t = tid; t < 2 * a.npad; t += nthreads) {
      const int64_t b = t >> 1;
      const int k = static_cast<int>(t & 1);
      const bool real = b < a.n;
      double fx = 0, fy = 0, fz = 0;
      const int32_t e0 = real ? a.row_ptr[b] : 0, e1 = real ? a.row_ptr[b + 1] : 0;
      for (int32_t e = e0 + k; e < e1; e += 2) {
        const int32_t v = a.inc[e];
        const int32_t l = v >> 1;
        SC_DCHECK(l >= 0 && l < a.nc);
        const double2 st = __ldcg(so + l);
        const double x = __dsub_rn(st.x, __dmul_rn(alpha, st.y));
        const double gm = x > 0.0 ? x : 0.0;
        if ((v & 1) == 0) sn[l].x = gm;
        const double4 nv = a.icol4[e];
        fx = fma(gm, nv.x, fx);
        fy = fma(gm, nv.y, fy);
        fz = fma(gm, nv.z, fz);
      }
      // (the 2 lanes of a body are adjacent threads of one warp: t and t ^ 1)
      fx += __shfl_xor_sync(0xffffffffu, fx, 1);
      fy += __shfl_xor_sync(0xffffffffu, fy, 1);
      fz += __shfl_xor_sync(0xffffffffu, fz, 1);
      if (k == 0) a.f4[b] = real ? make_double4(fx, fy, fz, 0.0) : make_double4(0, 0, 0, 0);
    }
    grid.sync();
    // ---- B: U = RPY(F), one warp per row (sums scaled by 8 pi mu, written as U).  Every CTA
    //      first stages all N sources (positions, forces: 64 B each, <= 64 KB) in shared memory
    //      with coalesced loads in flight together, so the pair loop reads shared memory.
    {
      double4* sp = dyn;
      double4* sf = dyn + a.npad;
      const bool rows_here = static_cast<int64_t>(blockIdx.x) * (kPT / 32) < a.n;  // (CTA has a row)
      if (rows_here)
        for (int64_t j = threadIdx.x; j < a.n; j += kPT) {
          sp[j] = a.pos4[j];
          sf[j] = ldcg4(&a.f4[j]);
        }
      __syncthreads();
    }
    for (int64_t i = warp; i < a.n; i += nwarps) {
      const double4* sp = dyn;
      const double4* sf = dyn + a.npad;
      const double4 pi = sp[i];
      double ux = 0, uy = 0, uz = 0;
#pragma unroll 4
      for (int64_t j = lane; j < a.n; j += 32) {
        if (j == i) continue;
        const double4 pj = sp[j];
        const double4 fj = sf[j];
        double dx, dy, dz;
        const double r2 = rpy_r2(pi, pj, dx, dy, dz);
        if (r2 == 0.0) {
          atomicExch(a.err, 1);  // coincident centres (reading A12)
          continue;
        }
        const double abar = pi.w + pj.w;  // (a_i + a_j)/2 from stored half radii
        const double rs = rsqrt_dp(r2);
        double c1, c2;
        if (r2 >= 4.0 * (abar * abar)) {  // far: 1/r + (2/3) a^2/r^3, (1/r^3)(1 - 2 a^2/r^2)
          const double h = rs * rs, e = rs * h, a2 = abar * abar;
          c1 = fma(2.0 / 3.0 * a2, e, rs);
          c2 = e * fma(-2.0 * a2, h, 1.0);
        } else {  // overlap: (4/(3a))(1 - 9r/(32a)), 1/(8 a^2 r)
          const double ia = 1.0 / abar;
          c1 = (4.0 / 3.0) * ia * fma(-9.0 / 32.0 * ia, r2 * rs, 1.0);
          c2 = 0.125 * ia * ia * rs;
        }
        const double tt = c2 * fma(dz, fj.z, fma(dy, fj.y, dx * fj.x));
        ux = fma(tt, dx, fma(c1, fj.x, ux));
        uy = fma(tt, dy, fma(c1, fj.y, uy));
        uz = fma(tt, dz, fma(c1, fj.z, uz));
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) {
        ux += __shfl_xor_sync(0xffffffffu, ux, o);
        uy += __shfl_xor_sync(0xffffffffu, uy, o);
        uz += __shfl_xor_sync(0xffffffffu, uz, o);
      }
      if (lane == 0) {
        const double4 fi = dyn[a.npad + i];
        const double cs = (2.0 / 3.0) / pi.w;  // self: 4/(3 a_i)
        a.u4[i] = make_double4(a.scale * fma(cs, fi.x, ux), a.scale * fma(cs, fi.y, uy),
                               a.scale * fma(cs, fi.z, uz), 0.0);
      }
    }
    grid.sync();
    // ---- C: g = D^T U + q and the chunk partials (lcp.cu dt_kernel<kSpheres, kDtIter>)
    for (int64_t c = blockIdx.x; c < a.nchunks; c += gridDim.x) {
      int64_t blo = c * kChunkBodies, bhi = blo + kChunkBodies;
      if (blo > a.n) blo = a.n;
      if (bhi > a.n) bhi = a.n;
      const int32_t l0 = a.first_ptr[blo], l1 = a.first_ptr[bhi];
      double p[4] = {0, 0, 0, 0};
      for (int32_t l = l0 + threadIdx.x; l < l1; l += kR) {
        const int32_t i = a.ci[l], j = a.cj[l];
        SC_DCHECK(l < a.nc && i >= 0 && i < a.n && j > i && j < a.n + SC_MAX_WALLS);
        const double4 nv = a.nrm4[l];
        const double4 ui = ldcg4(&a.u4[i]);
        const double4 uj = j < a.n ? ldcg4(&a.u4[j]) : make_double4(0, 0, 0, 0);  // j >= n: a wall
        const double v = fma(nv.z, ui.z - uj.z, fma(nv.y, ui.y - uj.y, nv.x * (ui.x - uj.x)));
        const double g = v + a.q[l];
        const double gnw = __ldcg(&sn[l].x);
        sn[l] = make_double2(gnw, g);
        const double2 sto = __ldcg(so + l);
        const double sd = gnw - sto.x;
        const double y = g - sto.y;
        const double m = gnw < g ? gnw : g;
        p[0] = fma(sd, sd, p[0]);
        p[1] = fma(sd, y, p[1]);
        p[2] = fma(y, y, p[2]);
        p[3] = fma(m, m, p[3]);
      }
      cta_reduce4_shfl(p, red);
      if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) a.part[c * 4 + k] = p[k];
      }
      __syncthreads();
    }
    grid.sync();
    // ---- D: K-FINALIZE on every CTA's own copy: thread 0 sums the few chunk partials
    //      (npad <= 2048: <= 8 chunks) in chunk order -> the same scalars on every CTA
    if (threadIdx.x == 0) {
      double p[4] = {0, 0, 0, 0};
      for (int64_t c = 0; c < a.nchunks; ++c) {
#pragma unroll
        for (int k = 0; k < 4; ++k) p[k] += __ldcg(a.part + c * 4 + k);
      }
      finalize_scalars(p, 0, &s, blockIdx.x == 0);
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.sc = s;
}

}  // namespace

bool persist_eligible(const sc_ctx* ctx) {
  // (a forced RPY kernel choice, sc_set_rpy_kernel, keeps the launch-per-kernel path)
  return ctx->use_persist && ctx->rpy_mode == 0 && ctx->kind == kSpheres && ctx->world == 1 && ctx->comm == nullptr &&
         ctx->mobility_model != 2 &&
         ctx->emul_world == 1 && ctx->npad <= kPersistMaxBodies && ctx->nc > 0 && ctx->persist_grid > 0;
}

// Per-device setup (sc_create): the kernel's shared-memory attribute and its grid (one CTA per SM
// of this context's device, if it can be resident).
int persist_init_device(sc_ctx* ctx) {
  const size_t smem_max = 2 * sizeof(double4) * kPersistMaxBodies;
  cudaError_t e = cudaFuncSetAttribute(bbpgd_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem_max));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaFuncSetAttribute(bbpgd_persistent)");
  int occ = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bbpgd_persistent_kernel, kPT, smem_max);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "occupancy(bbpgd_persistent)");
  ctx->persist_grid = occ >= 1 ? ctx->num_sms : 0;  // one CTA per SM: cheapest grid barrier
  return 0;
}

// Steps 7-16 of Alg. 1 in one cooperative launch (the scalars in ctx->dsc after Step 6).
int bbpgd_persistent(sc_ctx* ctx, double mu) {
  int grid = ctx->persist_grid;
  if (grid <= 0) return fail(ctx, SC_ECUDA, "persistent BBPGD kernel cannot be resident");
  if (ctx->persist_grid_cap > 0 && ctx->persist_grid_cap < grid) grid = ctx->persist_grid_cap;
  PersistArgs a;
  a.n = ctx->n;
  a.npad = ctx->npad;
  a.nc = ctx->nc;
  a.nchunks = ctx->nchunks;
  a.pos4 = ctx->pos4.p;
  a.f4 = ctx->f4.p;
  a.u4 = ctx->u4.p;
  a.row_ptr = ctx->row_ptr.p;
  a.inc = ctx->inc.p;
  a.icol4 = ctx->icol4.p;
  a.first_ptr = ctx->first_ptr.p;
  a.ci = ctx->ci.p;
  a.cj = ctx->cj.p;
  a.nrm4 = ctx->nrm4.p;
  a.q = ctx->q.p;
  a.st0 = ctx->st[0].p;
  a.st1 = ctx->st[1].p;
  a.part = ctx->chunk_part.p;
  a.sc = ctx->dsc;
  a.err = ctx->derr;
  a.scale = 1.0 / (8.0 * 3.14159265358979323846 * mu);
  void* args[] = {&a};
  timer_begin(ctx, SC_K_MISC);
  const size_t smem = 2 * sizeof(double4) * static_cast<size_t>(ctx->npad);
  cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(bbpgd_persistent_kernel), dim3(grid),
                                              dim3(kPT), args, smem, ctx->stream);
  timer_end(ctx, SC_K_MISC);
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaLaunchCooperativeKernel(bbpgd_persistent)");
  return check_launch(ctx, "bbpgd_persistent");
}

}  // namespace sc
