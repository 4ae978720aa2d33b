// contacts.cu -- (a1) build_contacts: cell-list near-pair detection on the GPU.
//
// Near set A(C, delta) = { l : Phi_l(C) < delta_l } (strict '<' and
// delta from BASELINE.json, reading A1).  Output sorted by (i, j), i < j.
//
// Pipeline (all device kernels; the host reads two scalars: the bounding box and n_c):
//   bbox reduce -> cell id per body -> counting sort by cell (count, scan, scatter)
//   -> per body i: test j > i in the 27 neighbouring cells, count
//   -> exclusive scan of counts (first_ptr) -> emit j's -> sort each i's j's
//   -> per constraint: gap, normal (and rod lever arms) with the exact expression.
// The gap/normal expressions use explicit round-to-nearest intrinsics (no FMA
// contraction), in the same association as the definition, so the constraint
// set and its values are bit-identical to the plain CPU definition (reading A20).
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "rpy_common.cuh"
#include "sc_internal.h"

namespace sc {
namespace {

constexpr int kBboxBlocks = 296;  // 2 x 148 SMs
constexpr int kT = 256;

// bbox partials: [blk][7] = min xyz, max xyz, max of w-derived size
__global__ void bbox_partial(const double4* __restrict__ p, int64_t n, int size_mode, double* __restrict__ out) {
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY}, sz = 0.0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double4 v = p[i];
    mn[0] = fmin(mn[0], v.x); mn[1] = fmin(mn[1], v.y); mn[2] = fmin(mn[2], v.z);
    mx[0] = fmax(mx[0], v.x); mx[1] = fmax(mx[1], v.y); mx[2] = fmax(mx[2], v.z);
    sz = fmax(sz, size_mode == 0 ? 2.0 * v.w : v.w);  // spheres: radius = 2 * (a/2); rods: L
  }
  __shared__ double s[7][kT];
  for (int d = 0; d < 3; ++d) { s[d][threadIdx.x] = mn[d]; s[3 + d][threadIdx.x] = mx[d]; }
  s[6][threadIdx.x] = sz;
  __syncthreads();
  for (int w = kT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      for (int d = 0; d < 3; ++d) {
        s[d][threadIdx.x] = fmin(s[d][threadIdx.x], s[d][threadIdx.x + w]);
        s[3 + d][threadIdx.x] = fmax(s[3 + d][threadIdx.x], s[3 + d][threadIdx.x + w]);
      }
      s[6][threadIdx.x] = fmax(s[6][threadIdx.x], s[6][threadIdx.x + w]);
    }
    __syncthreads();
  }
  if (threadIdx.x < 7) out[blockIdx.x * 7 + threadIdx.x] = s[threadIdx.x][0];
}

// one warp per component: min of the 3 lower bounds, max of the 3 upper bounds and the size
__global__ void bbox_final(double* __restrict__ part, int nb) {
  const int d = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (d >= 7) return;
  const bool is_min = d < 3;
  double r = is_min ? INFINITY : -INFINITY;
  for (int b = lane; b < nb; b += 32) r = is_min ? fmin(r, part[b * 7 + d]) : fmax(r, part[b * 7 + d]);
  for (int o = 16; o > 0; o >>= 1) {
    const double v = __shfl_xor_sync(0xffffffffu, r, o);
    r = is_min ? fmin(r, v) : fmax(r, v);
  }
  __syncthreads();  // every warp has read its column before lane 0 overwrites row 0
  if (lane == 0) part[d] = r;
}

struct Grid {
  double lo[3];
  double inv_h;
  int m[3];
};

__device__ __forceinline__ int cell_coord(double x, double lo, double inv_h, int m) {
  int k = static_cast<int>(floor((x - lo) * inv_h));
  return k < 0 ? 0 : (k >= m ? m - 1 : k);
}

__global__ void cell_assign(const double4* __restrict__ p, int64_t n, Grid g, int32_t* __restrict__ cell_of,
                            int32_t* __restrict__ cnt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double4 v = p[i];
  const int kx = cell_coord(v.x, g.lo[0], g.inv_h, g.m[0]);
  const int ky = cell_coord(v.y, g.lo[1], g.inv_h, g.m[1]);
  const int kz = cell_coord(v.z, g.lo[2], g.inv_h, g.m[2]);
  const int c = (kz * g.m[1] + ky) * g.m[0] + kx;
  cell_of[i] = c;
  atomicAdd(&cnt[c], 1);
}

__global__ void cell_scatter(const double4* __restrict__ p, const double4* __restrict__ d, int64_t n,
                             const int32_t* __restrict__ cell_of, int32_t* __restrict__ cursor,
                             int32_t* __restrict__ sorted_idx, double4* __restrict__ sorted4,
                             double4* __restrict__ sorted_d4) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t slot = atomicAdd(&cursor[cell_of[i]], 1);
  sorted_idx[slot] = static_cast<int32_t>(i);
  sorted4[slot] = p[i];
  if (d != nullptr) sorted_d4[slot] = d[i];
}

// ---------------------------------------------------------------- spheres
// Exact sphere test, same association as the definition:
//   dx = x_i - x_j; r = sqrt((dx*dx + dy*dy) + dz*dz); gap = r - (a_i + a_j);
//   contact iff gap < gap_abs + gap_rel * min(a_i, a_j).
struct SphereTest {
  double gap_abs, gap_rel;
  __device__ __forceinline__ bool operator()(const double4& pi, const double4& pj, double& dx, double& dy,
                                             double& dz, double& r, double& gap) const {
    dx = __dsub_rn(pi.x, pj.x);
    dy = __dsub_rn(pi.y, pj.y);
    dz = __dsub_rn(pi.z, pj.z);
    r = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    const double ai = 2.0 * pi.w, aj = 2.0 * pj.w;  // exact: w = a/2
    gap = __dsub_rn(r, __dadd_rn(ai, aj));
    const double amin = ai < aj ? ai : aj;
    const double thr = __dadd_rn(gap_abs, __dmul_rn(gap_rel, amin));
    return gap < thr;
  }
};

// ------------------------------------------------------------------ rods
// Closest points of two axis segments (clamped parametric method), evaluated
// with the same association as the definition (reading A15).
struct RodPair {
  double P1[3], P2[3];
};

__device__ __forceinline__ double dot3_rn(const double* a, const double* b) {
  return __dadd_rn(__dadd_rn(__dmul_rn(a[0], b[0]), __dmul_rn(a[1], b[1])), __dmul_rn(a[2], b[2]));
}

__device__ void segment_closest_rn(const double4& ci, const double4& ti, const double4& cj, const double4& tj,
                                   RodPair& o) {
  const double L1 = ci.w, L2 = cj.w;
  const double c1[3] = {ci.x, ci.y, ci.z}, t1[3] = {ti.x, ti.y, ti.z};
  const double c2[3] = {cj.x, cj.y, cj.z}, t2[3] = {tj.x, tj.y, tj.z};
  double p1[3], p2[3], d1[3], d2[3], r[3];
  const double h1 = __dmul_rn(0.5, L1), h2 = __dmul_rn(0.5, L2);
  for (int k = 0; k < 3; ++k) {
    p1[k] = __dsub_rn(c1[k], __dmul_rn(h1, t1[k]));
    p2[k] = __dsub_rn(c2[k], __dmul_rn(h2, t2[k]));
    d1[k] = __dmul_rn(L1, t1[k]);
    d2[k] = __dmul_rn(L2, t2[k]);
    r[k] = __dsub_rn(p1[k], p2[k]);
  }
  const double a = dot3_rn(d1, d1);
  const double e = dot3_rn(d2, d2);
  const double f = dot3_rn(d2, r);
  const double c = dot3_rn(d1, r);
  const double bb = dot3_rn(d1, d2);
  const double ae = __dmul_rn(a, e);
  const double denom = __dsub_rn(ae, __dmul_rn(bb, bb));
  double s;
  if (denom > __dmul_rn(1e-14, ae)) {
    s = __ddiv_rn(__dsub_rn(__dmul_rn(bb, f), __dmul_rn(c, e)), denom);
    if (s < 0.0) s = 0.0;
    if (s > 1.0) s = 1.0;
  } else {
    s = 0.0;
  }
  double t = __ddiv_rn(__dadd_rn(__dmul_rn(bb, s), f), e);
  if (t < 0.0) {
    t = 0.0;
    s = __ddiv_rn(-c, a);
    if (s < 0.0) s = 0.0;
    if (s > 1.0) s = 1.0;
  } else if (t > 1.0) {
    t = 1.0;
    s = __ddiv_rn(__dsub_rn(bb, c), a);
    if (s < 0.0) s = 0.0;
    if (s > 1.0) s = 1.0;
  }
  for (int k = 0; k < 3; ++k) {
    o.P1[k] = __dadd_rn(p1[k], __dmul_rn(d1[k], s));
    o.P2[k] = __dadd_rn(p2[k], __dmul_rn(d2[k], t));
  }
}

struct RodTest {
  double b2;        // 2b
  double thresh;    // gap threshold
  double prefilter; // 2b + |thresh|, loosened
  // returns contact decision; fills closest points, distance and gap
  __device__ __forceinline__ bool operator()(const double4& ci, const double4& ti, const double4& cj,
                                             const double4& tj, RodPair& rp, double& dist, double& gap) const {
    const double ox = ci.x - cj.x, oy = ci.y - cj.y, oz = ci.z - cj.z;
    const double cd2 = ox * ox + oy * oy + oz * oz;
    const double lim = (0.5 * (ci.w + cj.w) + prefilter) * (1.0 + 1e-9) + 1e-12;
    if (cd2 > lim * lim) return false;  // exact superset: closest points lie within L/2 of the centres
    segment_closest_rn(ci, ti, cj, tj, rp);
    const double dx = __dsub_rn(rp.P1[0], rp.P2[0]);
    const double dy = __dsub_rn(rp.P1[1], rp.P2[1]);
    const double dz = __dsub_rn(rp.P1[2], rp.P2[2]);
    dist = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
    gap = __dsub_rn(dist, b2);
    return gap < thresh;
  }
};

// ------------------------------------------------------------------ walls
// NEXT row f2: particle-boundary collisions.  A wall is the static plane
// {x : n.x = h} (unit n pointing into the fluid); it is not in the mobility matrix, so its
// constraint column has entries on the particle only.  Constraint (i, n + k) for wall k:
//   spheres: Phi = (n.c_i - h) - a_i,  contact iff Phi < gap_abs + gap_rel * a_i
//   rods:    the axis point closest to the wall, P = c + s t with s = -L/2 (n.t > 0),
//            +L/2 (n.t < 0), 0 (n.t = 0: parallel, the centre); Phi = (n.P - h) - b,
//            contact iff Phi < gap_thresh; lever arm r_i = P - c_i
// with the normal n (from the wall to the particle), evaluated without FMA contraction
// (fixed association, like the pair tests: bit-identical to the oracle).
struct WallSet {
  int nw;
  double4 w[SC_MAX_WALLS];  // (nx, ny, nz, h)
};

__device__ __forceinline__ double wall_dot_rn(const double4& w, double x, double y, double z) {
  return __dadd_rn(__dadd_rn(__dmul_rn(w.x, x), __dmul_rn(w.y, y)), __dmul_rn(w.z, z));
}

// returns the contact decision; gap and (rods) the closest axis point P
template <int KIND>
__device__ __forceinline__ bool wall_test(const double4& c, const double4& t, const double4& w, const SphereTest& st,
                                          const RodTest& rt, double& gap, double (&P)[3]) {
  if (KIND == kSpheres) {
    const double a = 2.0 * c.w;  // exact: w = a/2
    gap = __dsub_rn(__dsub_rn(wall_dot_rn(w, c.x, c.y, c.z), w.w), a);
    P[0] = c.x; P[1] = c.y; P[2] = c.z;
    return gap < __dadd_rn(st.gap_abs, __dmul_rn(st.gap_rel, a));
  } else {
    const double nt = wall_dot_rn(w, t.x, t.y, t.z);
    const double hl = 0.5 * c.w;  // exact
    const double s = nt > 0.0 ? -hl : (nt < 0.0 ? hl : 0.0);
    P[0] = __dadd_rn(c.x, __dmul_rn(s, t.x));
    P[1] = __dadd_rn(c.y, __dmul_rn(s, t.y));
    P[2] = __dadd_rn(c.z, __dmul_rn(s, t.z));
    gap = __dsub_rn(__dsub_rn(wall_dot_rn(w, P[0], P[1], P[2]), w.w), 0.5 * rt.b2);
    return gap < rt.thresh;
  }
}

// Pass 1 (count) / pass 2 (emit j's), one thread per cell-sorted body.
template <int KIND, bool EMIT>
__global__ void pair_search(const double4* __restrict__ s4, const double4* __restrict__ sd4,
                            const int32_t* __restrict__ sidx, const int32_t* __restrict__ cell_start,
                            int64_t n, Grid g, SphereTest st, RodTest rt, WallSet walls,
                            int32_t* __restrict__ cnt, const int32_t* __restrict__ off, int32_t* __restrict__ ci,
                            int32_t* __restrict__ cj) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const double4 pi = s4[s];
  const double4 ti = KIND == kRods ? sd4[s] : make_double4(0, 0, 0, 0);
  const int32_t i = sidx[s];
  const int kx = cell_coord(pi.x, g.lo[0], g.inv_h, g.m[0]);
  const int ky = cell_coord(pi.y, g.lo[1], g.inv_h, g.m[1]);
  const int kz = cell_coord(pi.z, g.lo[2], g.inv_h, g.m[2]);
  int32_t count = 0;
  int32_t o = EMIT ? off[i] : 0;
  for (int z = max(kz - 1, 0); z <= min(kz + 1, g.m[2] - 1); ++z)
    for (int y = max(ky - 1, 0); y <= min(ky + 1, g.m[1] - 1); ++y) {
      const int crow = (z * g.m[1] + y) * g.m[0];
      const int c0 = crow + max(kx - 1, 0), c1 = crow + min(kx + 1, g.m[0] - 1);
      const int t0 = cell_start[c0], t1 = cell_start[c1 + 1];  // x-adjacent cells are contiguous
      for (int t = t0; t < t1; ++t) {
        const int32_t j = sidx[t];
        if (j <= i) continue;
        bool hit;
        if (KIND == kSpheres) {
          double dx, dy, dz, r, gap;
          hit = st(pi, s4[t], dx, dy, dz, r, gap);
        } else {
          RodPair rp;
          double dist, gap;
          hit = rt(pi, ti, s4[t], sd4[t], rp, dist, gap);
        }
        if (hit) {
          if (EMIT) {
            SC_DCHECK(o < off[i + 1]);
            ci[o] = i;
            cj[o] = j;
            ++o;
          } else {
            ++count;
          }
        }
      }
    }
  for (int k = 0; k < walls.nw; ++k) {  // wall k is "body" n + k (sorts after every particle)
    double gap, P[3];
    if (wall_test<KIND>(pi, ti, walls.w[k], st, rt, gap, P)) {
      if (EMIT) {
        SC_DCHECK(o < off[i + 1]);
        ci[o] = i;
        cj[o] = static_cast<int32_t>(n + k);
        ++o;
      } else {
        ++count;
      }
    }
  }
  if (!EMIT) cnt[i] = count;
}

// Near list for the RPY overlap branch: every j != i with r_ij < 2 abar (the predicate of
// rpy_common.cuh, bit-identical to the far-field kernel's).  Pass 1 counts, pass 2 emits;
// one thread per cell-sorted body, output indexed by the body's own index.
template <bool EMIT>
__global__ void near_search(const double4* __restrict__ s4, const int32_t* __restrict__ sidx,
                            const int32_t* __restrict__ cell_start, int64_t n, Grid g, bool poly,
                            long long near_bits, int32_t* __restrict__ cnt, const int32_t* __restrict__ off,
                            int32_t* __restrict__ out) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= n) return;
  const double4 pi = s4[s];
  const int32_t i = sidx[s];
  const int kx = cell_coord(pi.x, g.lo[0], g.inv_h, g.m[0]);
  const int ky = cell_coord(pi.y, g.lo[1], g.inv_h, g.m[1]);
  const int kz = cell_coord(pi.z, g.lo[2], g.inv_h, g.m[2]);
  int32_t count = 0;
  int32_t o = EMIT ? off[i] : 0;
  for (int z = max(kz - 1, 0); z <= min(kz + 1, g.m[2] - 1); ++z)
    for (int y = max(ky - 1, 0); y <= min(ky + 1, g.m[1] - 1); ++y) {
      const int crow = (z * g.m[1] + y) * g.m[0];
      const int t0 = cell_start[crow + max(kx - 1, 0)], t1 = cell_start[crow + min(kx + 1, g.m[0] - 1) + 1];
      for (int t = t0; t < t1; ++t) {
        const int32_t j = sidx[t];
        if (j == i) continue;
        const double4 pj = s4[t];
        double dx, dy, dz;
        const double r2 = rpy_r2(pi, pj, dx, dy, dz);
        if (!rpy_is_near(r2, pi.w + pj.w, poly, near_bits)) continue;
        if (EMIT)
          out[o++] = j;
        else
          ++count;
      }
    }
  if (!EMIT) cnt[i] = count;
}

// Sort each body's partner list by j (lists are short: insertion sort in place).
__global__ void sort_partners(const int32_t* __restrict__ off, int64_t n, int32_t* __restrict__ cj) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t a = off[i], b = off[i + 1];
  for (int32_t k = a + 1; k < b; ++k) {
    const int32_t v = cj[k];
    int32_t m = k - 1;
    while (m >= a && cj[m] > v) {
      cj[m + 1] = cj[m];
      --m;
    }
    cj[m + 1] = v;
  }
}

__global__ void sphere_geometry(const int32_t* __restrict__ ci, const int32_t* __restrict__ cj, int64_t nc,
                                int64_t n, const double4* __restrict__ p, SphereTest st, WallSet walls,
                                double4* __restrict__ nrm4, int32_t* __restrict__ err) {
  const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l >= nc) return;
  if (cj[l] >= n) {  // wall constraint: the wall normal
    const double4 w = walls.w[cj[l] - n];
    double gap, P[3];
    RodTest rt{0, 0, 0};
    wall_test<kSpheres>(p[ci[l]], make_double4(0, 0, 0, 0), w, st, rt, gap, P);
    nrm4[l] = make_double4(w.x, w.y, w.z, gap);
    return;
  }
  double dx, dy, dz, r, gap;
  st(p[ci[l]], p[cj[l]], dx, dy, dz, r, gap);
  if (r == 0.0) {
    atomicExch(err, 2);  // coincident centres (reading A12)
    nrm4[l] = make_double4(0, 0, 0, gap);
    return;
  }
  nrm4[l] = make_double4(__ddiv_rn(dx, r), __ddiv_rn(dy, r), __ddiv_rn(dz, r), gap);
}

__global__ void rod_geometry(const int32_t* __restrict__ ci, const int32_t* __restrict__ cj, int64_t nc, int64_t n,
                             const double4* __restrict__ c4, const double4* __restrict__ d4, RodTest rt,
                             WallSet walls, double4* __restrict__ nrm4, double4* __restrict__ lev4,
                             int32_t* __restrict__ err) {
  const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l >= nc) return;
  const int32_t i = ci[l], j = cj[l];
  if (j >= n) {  // wall constraint: normal n_w, lever arm P - c_i on the rod, none on the wall
    const double4 w = walls.w[j - n], pi = c4[i];
    double gap, P[3];
    SphereTest st{0, 0};
    wall_test<kRods>(pi, d4[i], w, st, rt, gap, P);
    nrm4[l] = make_double4(w.x, w.y, w.z, gap);
    lev4[2 * l] = make_double4(__dsub_rn(P[0], pi.x), __dsub_rn(P[1], pi.y), __dsub_rn(P[2], pi.z), 0.0);
    lev4[2 * l + 1] = make_double4(0.0, 0.0, 0.0, 0.0);
    return;
  }
  const double4 pi = c4[i], pj = c4[j], ti = d4[i], tj = d4[j];
  RodPair rp;
  double dist, gap;
  RodTest nofilter = rt;
  nofilter.prefilter = INFINITY;
  nofilter(pi, ti, pj, tj, rp, dist, gap);
  double nx, ny, nz;
  if (dist < 1e-300) {
    // crossing axes: n = +-(t_i x t_j), oriented so that n . (c_i - c_j) >= 0
    const double cx = __dsub_rn(__dmul_rn(ti.y, tj.z), __dmul_rn(ti.z, tj.y));
    const double cy = __dsub_rn(__dmul_rn(ti.z, tj.x), __dmul_rn(ti.x, tj.z));
    const double cz = __dsub_rn(__dmul_rn(ti.x, tj.y), __dmul_rn(ti.y, tj.x));
    const double cn = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(cx, cx), __dmul_rn(cy, cy)), __dmul_rn(cz, cz)));
    if (cn == 0.0) {
      atomicExch(err, 2);
      nx = ny = nz = 0.0;
    } else {
      const double ox = __dsub_rn(pi.x, pj.x), oy = __dsub_rn(pi.y, pj.y), oz = __dsub_rn(pi.z, pj.z);
      const double sg =
          __dadd_rn(__dadd_rn(__dmul_rn(cx, ox), __dmul_rn(cy, oy)), __dmul_rn(cz, oz)) >= 0.0 ? 1.0 : -1.0;
      nx = __ddiv_rn(__dmul_rn(sg, cx), cn);
      ny = __ddiv_rn(__dmul_rn(sg, cy), cn);
      nz = __ddiv_rn(__dmul_rn(sg, cz), cn);
    }
  } else {
    nx = __ddiv_rn(__dsub_rn(rp.P1[0], rp.P2[0]), dist);
    ny = __ddiv_rn(__dsub_rn(rp.P1[1], rp.P2[1]), dist);
    nz = __ddiv_rn(__dsub_rn(rp.P1[2], rp.P2[2]), dist);
  }
  nrm4[l] = make_double4(nx, ny, nz, gap);
  lev4[2 * l] = make_double4(__dsub_rn(rp.P1[0], pi.x), __dsub_rn(rp.P1[1], pi.y), __dsub_rn(rp.P1[2], pi.z), 0.0);
  lev4[2 * l + 1] =
      make_double4(__dsub_rn(rp.P2[0], pj.x), __dsub_rn(rp.P2[1], pj.y), __dsub_rn(rp.P2[2], pj.z), 0.0);
}

inline unsigned nblk(int64_t n, int t = kT) { return static_cast<unsigned>((n + t - 1) / t); }

int build_common(sc_ctx* ctx, SphereTest st, RodTest rt) {
  WallSet walls;
  walls.nw = ctx->nwalls;
  for (int k = 0; k < SC_MAX_WALLS; ++k) walls.w[k] = ctx->walls[k];
  const int64_t n = ctx->n;
  const int kind = ctx->kind;
  ctx->nc = 0;
  ctx->assembled = false;
  ctx->have_q = false;
  if (int rc = ensure(ctx, ctx->first_ptr, n + 1)) return rc;
  if (n == 0) {
    SC_CUDA(cudaMemsetAsync(ctx->first_ptr.p, 0, sizeof(int32_t), ctx->stream));
    ctx->h_first_ptr.assign(1, 0);
    return 0;
  }
  // 1. bounding box and the largest body size (sphere radius / rod length)
  if (int rc = ensure(ctx, ctx->bbox_part, kBboxBlocks * 7)) return rc;
  timer_begin(ctx, SC_K_CONTACTS);
  bbox_partial<<<kBboxBlocks, kT, 0, ctx->stream>>>(ctx->pos4.p, n, kind == kSpheres ? 0 : 1, ctx->bbox_part.p);
  timer_end(ctx, SC_K_CONTACTS);
  if (int rc = check_launch(ctx, "bbox_partial")) return rc;
  timer_begin(ctx, SC_K_CONTACTS);
  bbox_final<<<1, 224, 0, ctx->stream>>>(ctx->bbox_part.p, kBboxBlocks);
  timer_end(ctx, SC_K_CONTACTS);
  if (int rc = check_launch(ctx, "bbox_final")) return rc;
  double bb[7];
  SC_CUDA(cudaMemcpyAsync(bb, ctx->bbox_part.p, sizeof(bb), cudaMemcpyDeviceToHost, ctx->stream));
  SC_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int d = 0; d < 7; ++d)
    if (!std::isfinite(bb[d])) return fail(ctx, SC_ENONFINITE, "non-finite body coordinates");
  // 2. cell edge >= the largest possible contact centre distance (x(1+1e-6) against rounding)
  const double smax = bb[6];
  double cutoff;
  if (kind == kSpheres)
    cutoff = 2.0 * smax + std::max(st.gap_abs, 0.0) + st.gap_rel * smax;
  else
    cutoff = smax + rt.b2 + std::fabs(rt.thresh);
  double h = cutoff * (1.0 + 1e-6) + 1e-12;
  Grid g;
  int64_t m[3];
  for (;;) {
    for (int d = 0; d < 3; ++d) m[d] = static_cast<int64_t>(std::floor((bb[3 + d] - bb[d]) / h)) + 1;
    if (m[0] * m[1] * m[2] <= 4 * n + 1024 && m[0] * m[1] * m[2] < (int64_t(1) << 30)) break;
    h *= 1.25;
  }
  for (int d = 0; d < 3; ++d) {
    g.lo[d] = bb[d];
    g.m[d] = static_cast<int>(m[d]);
  }
  g.inv_h = 1.0 / h;
  const int64_t ncell = m[0] * m[1] * m[2];
  // 3. counting sort of bodies by cell
  if (int rc = ensure(ctx, ctx->cell_of, n)) return rc;
  if (int rc = ensure(ctx, ctx->cell_cnt, ncell + 1)) return rc;
  if (int rc = ensure(ctx, ctx->cell_start, ncell + 1)) return rc;
  if (int rc = ensure(ctx, ctx->sorted_idx, n)) return rc;
  if (int rc = ensure(ctx, ctx->sorted4, n)) return rc;
  if (kind == kRods) {
    if (int rc = ensure(ctx, ctx->sorted_dir4, n)) return rc;
  }
  if (int rc = ensure(ctx, ctx->pair_cnt, n + 1)) return rc;
  const int64_t scan_n = std::max<int64_t>(ncell + 1, n + 1);
  if (int rc = ensure(ctx, ctx->scan_tmp, scan_tmp_size(scan_n) + 1)) return rc;
  SC_CUDA(cudaMemsetAsync(ctx->cell_cnt.p, 0, sizeof(int32_t) * (ncell + 1), ctx->stream));
  timer_begin(ctx, SC_K_CONTACTS);
  cell_assign<<<nblk(n), kT, 0, ctx->stream>>>(ctx->pos4.p, n, g, ctx->cell_of.p, ctx->cell_cnt.p);
  timer_end(ctx, SC_K_CONTACTS);
  if (int rc = check_launch(ctx, "cell_assign")) return rc;
  if (int rc = exclusive_scan_i32(ctx, ctx->cell_cnt.p, ctx->cell_start.p, ncell, ctx->scan_tmp.p)) return rc;
  // cursor = copy of cell_start (reuse cell_cnt)
  SC_CUDA(cudaMemcpyAsync(ctx->cell_cnt.p, ctx->cell_start.p, sizeof(int32_t) * ncell, cudaMemcpyDeviceToDevice,
                          ctx->stream));
  timer_begin(ctx, SC_K_CONTACTS);
  cell_scatter<<<nblk(n), kT, 0, ctx->stream>>>(ctx->pos4.p, kind == kRods ? ctx->dir4.p : nullptr, n,
                                                 ctx->cell_of.p, ctx->cell_cnt.p, ctx->sorted_idx.p,
                                                 ctx->sorted4.p, ctx->sorted_dir4.p);
  timer_end(ctx, SC_K_CONTACTS);
  if (int rc = check_launch(ctx, "cell_scatter")) return rc;
  // 4. count partners j > i
  timer_begin(ctx, SC_K_CONTACTS);
  if (kind == kSpheres)
    pair_search<kSpheres, false><<<nblk(n), kT, 0, ctx->stream>>>(
        ctx->sorted4.p, nullptr, ctx->sorted_idx.p, ctx->cell_start.p, n, g, st, rt, walls, ctx->pair_cnt.p, nullptr,
        nullptr, nullptr);
  else
    pair_search<kRods, false><<<nblk(n), kT, 0, ctx->stream>>>(
        ctx->sorted4.p, ctx->sorted_dir4.p, ctx->sorted_idx.p, ctx->cell_start.p, n, g, st, rt, walls,
        ctx->pair_cnt.p, nullptr, nullptr, nullptr);
  timer_end(ctx, SC_K_CONTACTS);
  if (int rc = check_launch(ctx, "pair_count")) return rc;
  // 5. first_ptr = exclusive scan of counts; n_c = first_ptr[n]
  if (int rc = exclusive_scan_i32(ctx, ctx->pair_cnt.p, ctx->first_ptr.p, n, ctx->scan_tmp.p)) return rc;
  // spheres: count the RPY near list too before the one host read of both totals
  const double a0 = ctx->a_const;
  const double n2 = 4.0 * (a0 * a0);
  const long long nb = *reinterpret_cast<const long long*>(&n2);
  if (kind == kSpheres) {
    if (int rc = ensure(ctx, ctx->near_ptr, n + 1)) return rc;
    if (int rc = ensure(ctx, ctx->pair_off, n + 1)) return rc;
    timer_begin(ctx, SC_K_CONTACTS);
    near_search<false><<<nblk(n), kT, 0, ctx->stream>>>(ctx->sorted4.p, ctx->sorted_idx.p, ctx->cell_start.p, n,
                                                        g, ctx->poly != 0, nb, ctx->pair_off.p, nullptr, nullptr);
    timer_end(ctx, SC_K_CONTACTS);
    if (int rc = check_launch(ctx, "near_count")) return rc;
    if (int rc = exclusive_scan_i32(ctx, ctx->pair_off.p, ctx->near_ptr.p, n, ctx->scan_tmp.p)) return rc;
  }
  int32_t nc32 = 0, nn = 0;
  SC_CUDA(cudaMemcpyAsync(&nc32, ctx->first_ptr.p + n, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  if (kind == kSpheres)
    SC_CUDA(cudaMemcpyAsync(&nn, ctx->near_ptr.p + n, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  SC_CUDA(cudaStreamSynchronize(ctx->stream));
  if (nc32 < 0) return fail(ctx, SC_ENOMEM, "constraint count overflows int32");
  const int64_t nc = nc32;
  ctx->nc = nc;
  if (int rc = ensure(ctx, ctx->ci, nc)) return rc;
  if (int rc = ensure(ctx, ctx->cj, nc)) return rc;
  if (int rc = ensure(ctx, ctx->nrm4, nc)) return rc;
  if (kind == kRods) {
    if (int rc = ensure(ctx, ctx->lev4, 2 * nc)) return rc;
  }
  if (nc > 0) {
    // 6. emit, sort partners per i, geometry per constraint
    timer_begin(ctx, SC_K_CONTACTS);
    if (kind == kSpheres)
      pair_search<kSpheres, true><<<nblk(n), kT, 0, ctx->stream>>>(
          ctx->sorted4.p, nullptr, ctx->sorted_idx.p, ctx->cell_start.p, n, g, st, rt, walls, nullptr,
          ctx->first_ptr.p, ctx->ci.p, ctx->cj.p);
    else
      pair_search<kRods, true><<<nblk(n), kT, 0, ctx->stream>>>(
          ctx->sorted4.p, ctx->sorted_dir4.p, ctx->sorted_idx.p, ctx->cell_start.p, n, g, st, rt, walls, nullptr,
          ctx->first_ptr.p, ctx->ci.p, ctx->cj.p);
    timer_end(ctx, SC_K_CONTACTS);
    if (int rc = check_launch(ctx, "pair_emit")) return rc;
    timer_begin(ctx, SC_K_CONTACTS);
    sort_partners<<<nblk(n), kT, 0, ctx->stream>>>(ctx->first_ptr.p, n, ctx->cj.p);
    timer_end(ctx, SC_K_CONTACTS);
    if (int rc = check_launch(ctx, "sort_partners")) return rc;
    timer_begin(ctx, SC_K_CONTACTS);
    if (kind == kSpheres)
      sphere_geometry<<<nblk(nc), kT, 0, ctx->stream>>>(ctx->ci.p, ctx->cj.p, nc, n, ctx->pos4.p, st, walls,
                                                         ctx->nrm4.p, ctx->derr);
    else
      rod_geometry<<<nblk(nc), kT, 0, ctx->stream>>>(ctx->ci.p, ctx->cj.p, nc, n, ctx->pos4.p, ctx->dir4.p, rt,
                                                      walls, ctx->nrm4.p, ctx->lev4.p, ctx->derr);
    timer_end(ctx, SC_K_CONTACTS);
    if (int rc = check_launch(ctx, "geometry")) return rc;
  }
  if (kind == kSpheres) {
    // near list (pairs in the RPY overlap branch), both directions, sorted per body (counted above)
    if (int rc = ensure(ctx, ctx->near_idx, nn)) return rc;
    if (nn > 0) {
      timer_begin(ctx, SC_K_CONTACTS);
      near_search<true><<<nblk(n), kT, 0, ctx->stream>>>(ctx->sorted4.p, ctx->sorted_idx.p, ctx->cell_start.p, n,
                                                         g, ctx->poly != 0, nb, nullptr, ctx->near_ptr.p,
                                                         ctx->near_idx.p);
      timer_end(ctx, SC_K_CONTACTS);
      if (int rc = check_launch(ctx, "near_emit")) return rc;
      timer_begin(ctx, SC_K_CONTACTS);
      sort_partners<<<nblk(n), kT, 0, ctx->stream>>>(ctx->near_ptr.p, n, ctx->near_idx.p);
      timer_end(ctx, SC_K_CONTACTS);
      if (int rc = check_launch(ctx, "near_sort")) return rc;
    }
  }
  ctx->h_first_ptr.resize(n + 1);
  SC_CUDA(cudaMemcpyAsync(ctx->h_first_ptr.data(), ctx->first_ptr.p, sizeof(int32_t) * (n + 1),
                          cudaMemcpyDeviceToHost, ctx->stream));
  SC_CUDA(cudaMemcpyAsync(ctx->herr, ctx->derr, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  SC_CUDA(cudaStreamSynchronize(ctx->stream));
  if (*ctx->herr != 0) {
    SC_CUDA(cudaMemsetAsync(ctx->derr, 0, sizeof(int32_t), ctx->stream));
    return fail(ctx, SC_EDEGENERATE, "coincident centres (zero-length contact normal)");
  }
  return 0;
}

}  // namespace

int build_contacts_spheres(sc_ctx* ctx, double gap_abs, double gap_rel) {
  SphereTest st{gap_abs, gap_rel};
  RodTest rt{0, 0, 0};
  return build_common(ctx, st, rt);
}

int build_contacts_rods(sc_ctx* ctx, double gap_thresh) {
  SphereTest st{0, 0};
  RodTest rt{2.0 * ctx->rod_b, gap_thresh, 2.0 * ctx->rod_b + std::fabs(gap_thresh)};
  return build_common(ctx, st, rt);
}

}  // namespace sc
