// assemble.cu -- (a2) assemble_D: column form of D and the body -> constraint incidence.
//
// D = [D_0 D_1 ...]: column l has +n on body i and -n on body j
// (spheres, 6 nnz) plus the torques r_i x n and -(r_j x n) for rods (12 nnz).
// The paper stores D^T in CRS with rows partitioned over ranks;
// here the column data lives per constraint (nrm4, rxn4) and the incidence
// row_ptr/inc lists, per body, the constraints touching it in ascending
// constraint order with the side in bit 0, so F = D gamma is an atomic-free,
// deterministic per-body gather.
#include <algorithm>

#include "sc_internal.h"

namespace sc {
namespace {

constexpr int kT = 256;
inline unsigned nblk(int64_t n) { return static_cast<unsigned>((n + kT - 1) / kT); }

__global__ void degree_count(const int32_t* __restrict__ ci, const int32_t* __restrict__ cj, int64_t nc,
                             int64_t n, int32_t* __restrict__ deg) {
  const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l >= nc) return;
  atomicAdd(&deg[ci[l]], 1);
  if (cj[l] < n) atomicAdd(&deg[cj[l]], 1);  // cj >= n: a wall (no column entries, NEXT row f2)
}

__global__ void incidence_fill(const int32_t* __restrict__ ci, const int32_t* __restrict__ cj, int64_t nc,
                               int64_t n, int32_t* __restrict__ cursor, int32_t* __restrict__ inc) {
  const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l >= nc) return;
  inc[atomicAdd(&cursor[ci[l]], 1)] = static_cast<int32_t>(l << 1);
  if (cj[l] < n) inc[atomicAdd(&cursor[cj[l]], 1)] = static_cast<int32_t>((l << 1) | 1);
}

__global__ void incidence_sort(const int32_t* __restrict__ row_ptr, int64_t n, int32_t* __restrict__ inc) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= n) return;
  const int32_t a = row_ptr[b], e = row_ptr[b + 1];
  for (int32_t k = a + 1; k < e; ++k) {
    const int32_t v = inc[k];
    int32_t m = k - 1;
    while (m >= a && inc[m] > v) {
      inc[m + 1] = inc[m];
      --m;
    }
    inc[m + 1] = v;
  }
}

// Signed D_l block of every incidence, in incidence (per-body) order, so the spheres'
// D-gather streams it: sigma n, sigma = +1 on i, -1 on j.
template <int KIND>
__global__ void incidence_columns(const int32_t* __restrict__ inc, const int32_t* __restrict__ ninc_dev, int64_t ninc,
                                  const double4* __restrict__ nrm4,
                                  const double4* __restrict__ /*rxn4*/, double4* __restrict__ icol4) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= ninc || e >= *ninc_dev) return;  // row_ptr[n] = 2 n_c - (wall constraints)
  const int32_t v = inc[e];
  const int32_t l = v >> 1;
  const int side = v & 1;
  const double sg = side ? -1.0 : 1.0;
  const double4 n = nrm4[l];
  if (KIND == kSpheres) {
    icol4[e] = make_double4(sg * n.x, sg * n.y, sg * n.z, 0.0);
  }
}

// Rods (SC_ROD_ICOL): the signed 6-vector column (sigma n, sigma r_side x n) of every incidence,
// 3 double2 per incidence, streamed by the D-gather in incidence order.
__global__ void rod_incidence_columns(const int32_t* __restrict__ inc, const int32_t* __restrict__ ninc_dev,
                                      int64_t ninc, const double4* __restrict__ nrm4,
                                      const double4* __restrict__ rxn4, double2* __restrict__ icolr) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= ninc || e >= *ninc_dev) return;
  const int32_t v = inc[e];
  const int32_t l = v >> 1;
  const int side = v & 1;
  const double sg = side ? -1.0 : 1.0;
  const double4 n = nrm4[l], r = rxn4[2 * l + side];
  icolr[3 * e] = make_double2(sg * n.x, sg * n.y);
  icolr[3 * e + 1] = make_double2(sg * n.z, sg * r.x);
  icolr[3 * e + 2] = make_double2(sg * r.y, sg * r.z);
}

// einc[l] = (e_i, e_j): where constraint l's two incidences sit in the body-sorted incidence
// list (the rods D^T reads the per-incidence half rates h_e there); e_j = -1 for a wall.
__global__ void rod_incidence_positions(const int32_t* __restrict__ inc, const int32_t* __restrict__ ninc_dev,
                                        int64_t ninc, int32_t* __restrict__ epos) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= ninc || e >= *ninc_dev) return;
  epos[inc[e]] = static_cast<int32_t>(e);  // inc[e] = 2 l + side
}

__global__ void rod_columns(const double4* __restrict__ nrm4, const double4* __restrict__ lev4, int64_t nc,
                            double4* __restrict__ rxn4) {
  const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l >= nc) return;
  const double4 n = nrm4[l];
  const double4 ri = lev4[2 * l], rj = lev4[2 * l + 1];
  rxn4[2 * l] = make_double4(ri.y * n.z - ri.z * n.y, ri.z * n.x - ri.x * n.z, ri.x * n.y - ri.y * n.x, 0.0);
  rxn4[2 * l + 1] = make_double4(rj.y * n.z - rj.z * n.y, rj.z * n.x - rj.x * n.z, rj.x * n.y - rj.y * n.x, 0.0);
}

}  // namespace

int assemble(sc_ctx* ctx) {
  const int64_t n = ctx->n, nc = ctx->nc;
  if (int rc = ensure(ctx, ctx->row_ptr, n + 1)) return rc;
  if (int rc = ensure(ctx, ctx->inc, 2 * nc)) return rc;
  if (int rc = ensure(ctx, ctx->pair_cnt, n + 1)) return rc;
  if (int rc = ensure(ctx, ctx->cell_cnt, n + 1)) return rc;
  if (int rc = ensure(ctx, ctx->scan_tmp, scan_tmp_size(n + 1) + 1)) return rc;
  int32_t* deg = ctx->pair_cnt.p;
  SC_CUDA(cudaMemsetAsync(deg, 0, sizeof(int32_t) * (n + 1), ctx->stream));
  if (nc > 0) {
    timer_begin(ctx, SC_K_ASSEMBLE);
    degree_count<<<nblk(nc), kT, 0, ctx->stream>>>(ctx->ci.p, ctx->cj.p, nc, n, deg);
    timer_end(ctx, SC_K_ASSEMBLE);
    if (int rc = check_launch(ctx, "degree_count")) return rc;
  }
  if (int rc = exclusive_scan_i32(ctx, deg, ctx->row_ptr.p, n, ctx->scan_tmp.p)) return rc;
  if (nc > 0) {
    int32_t* cursor = ctx->cell_cnt.p;
    SC_CUDA(cudaMemcpyAsync(cursor, ctx->row_ptr.p, sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, ctx->stream));
    timer_begin(ctx, SC_K_ASSEMBLE);
    incidence_fill<<<nblk(nc), kT, 0, ctx->stream>>>(ctx->ci.p, ctx->cj.p, nc, n, cursor, ctx->inc.p);
    timer_end(ctx, SC_K_ASSEMBLE);
    if (int rc = check_launch(ctx, "incidence_fill")) return rc;
    timer_begin(ctx, SC_K_ASSEMBLE);
    incidence_sort<<<nblk(n), kT, 0, ctx->stream>>>(ctx->row_ptr.p, n, ctx->inc.p);
    timer_end(ctx, SC_K_ASSEMBLE);
    if (int rc = check_launch(ctx, "incidence_sort")) return rc;
    if (ctx->kind == kRods) {
      if (int rc = ensure(ctx, ctx->rxn4, 2 * nc)) return rc;
      timer_begin(ctx, SC_K_ASSEMBLE);
      rod_columns<<<nblk(nc), kT, 0, ctx->stream>>>(ctx->nrm4.p, ctx->lev4.p, nc, ctx->rxn4.p);
      timer_end(ctx, SC_K_ASSEMBLE);
      if (int rc = check_launch(ctx, "rod_columns")) return rc;
      // signed 6-vector columns in incidence order (the rods gathers stream them)
      if (int rc = ensure(ctx, ctx->icol4, 3 * nc + 1)) return rc;  // 3 double2 per incidence
      timer_begin(ctx, SC_K_ASSEMBLE);
      rod_incidence_columns<<<nblk(2 * nc), kT, 0, ctx->stream>>>(ctx->inc.p, ctx->row_ptr.p + n, 2 * nc, ctx->nrm4.p,
                                                                  ctx->rxn4.p,
                                                                  reinterpret_cast<double2*>(ctx->icol4.p));
      timer_end(ctx, SC_K_ASSEMBLE);
      if (int rc = check_launch(ctx, "rod_incidence_columns")) return rc;
      if (int rc = ensure(ctx, ctx->einc, nc)) return rc;
      if (int rc = ensure(ctx, ctx->hinc, 2 * nc + 1)) return rc;
      SC_CUDA(cudaMemsetAsync(ctx->einc.p, 0xFF, sizeof(int2) * nc, ctx->stream));  // -1: no incidence (wall)
      timer_begin(ctx, SC_K_ASSEMBLE);
      rod_incidence_positions<<<nblk(2 * nc), kT, 0, ctx->stream>>>(ctx->inc.p, ctx->row_ptr.p + n, 2 * nc,
                                                                    reinterpret_cast<int32_t*>(ctx->einc.p));
      timer_end(ctx, SC_K_ASSEMBLE);
      if (int rc = check_launch(ctx, "rod_incidence_positions")) return rc;

    }
    if (ctx->kind == kSpheres) {  // (rods gather from the per-constraint columns)
      const int64_t ninc = 2 * nc;
      if (int rc = ensure(ctx, ctx->icol4, ninc)) return rc;
      timer_begin(ctx, SC_K_ASSEMBLE);
      incidence_columns<kSpheres><<<nblk(ninc), kT, 0, ctx->stream>>>(ctx->inc.p, ctx->row_ptr.p + n, ninc, ctx->nrm4.p, nullptr,
                                                                      ctx->icol4.p);
      timer_end(ctx, SC_K_ASSEMBLE);
      if (int rc = check_launch(ctx, "incidence_columns")) return rc;
    }
  }
  // reduction chunks (lcp_common.cuh chunk_bounds): spheres 256-body blocks (multi-GPU ownership),
  // rods 256-constraint tiles
  ctx->nchunks = ctx->kind == kRods ? std::max<int64_t>(1, (nc + 255) / 256) : ctx->npad / kChunkBodies;
  ctx->assembled = true;
  return 0;
}

}  // namespace sc
