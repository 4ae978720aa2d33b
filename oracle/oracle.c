/* oracle.c -- plain CPU FP64 oracle for the per-time-step collision
 * resolution solve of arXiv 1909.06623 (Yan et al. 2020), Sec. 3.
 *
 * TEST INFRASTRUCTURE: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / reference leg may load this.  Shares no code with the CUDA
 * product.  Compiled with  gcc -O2 -fopenmp -ffp-contract=off  (no FMA
 * contraction: the contact gap/normal expressions below are the definition
 * the GPU must reproduce bit for bit, reading A20).
 *
 * Each function cites the passage it follows ("P:Lnnn" = PAPER.md line).
 * Everything is written as the direct definition: no blocking, no fusion.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORC_PI 3.14159265358979323846

/* ------------------------------------------------------------------------ */
/* Contacts: near set A(C, delta) = { l : Phi_l(C) <= delta }  */
/* with BASELINE's strict threshold "gap < 0.1a" (reading A1).              */
/* ------------------------------------------------------------------------ */

/* Sphere-sphere minimal separation Phi = |c_i - c_j| - a_i - a_j and the
 * unit normal from j to i (reading A13).  Fixed association, no FMA. */
static int sphere_pair(const double* pos, const double* radius, int64_t i, int64_t j,
                       double gap_abs, double gap_rel, double* gap, double* nrm) {
  double dx = pos[3 * i + 0] - pos[3 * j + 0];
  double dy = pos[3 * i + 1] - pos[3 * j + 1];
  double dz = pos[3 * i + 2] - pos[3 * j + 2];
  double r = sqrt((dx * dx + dy * dy) + dz * dz);
  double ai = radius[i], aj = radius[j];
  double g = r - (ai + aj);
  double amin = ai < aj ? ai : aj;
  double thresh = gap_abs + gap_rel * amin;
  if (!(g < thresh)) return 0;
  if (r == 0.0) return -2; /* coincident centres: degenerate normal (reading A12) */
  *gap = g;
  nrm[0] = dx / r;
  nrm[1] = dy / r;
  nrm[2] = dz / r;
  return 1;
}

int64_t orc_contacts_spheres_brute(int64_t n, const double* pos, const double* radius,
                                   double gap_abs, double gap_rel, int64_t cap,
                                   int32_t* ci, int32_t* cj, double* gap, double* normal) {
  if (n < 0 || !pos || !radius) return -1;
  /* pass 1: count per i (all j > i) */
  int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 16) reduction(| : bad)
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = 0;
    for (int64_t j = i + 1; j < n; ++j) {
      double g, nr[3];
      int s = sphere_pair(pos, radius, i, j, gap_abs, gap_rel, &g, nr);
      if (s < 0) bad = 1;
      if (s > 0) ++c;
    }
    cnt[i + 1] = c;
  }
  if (bad) { free(cnt); return -2; }
  for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  int64_t total = cnt[n];
  if (total > cap) { free(cnt); return total; }
  /* pass 2: emit in (i, j) order */
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = 0; i < n; ++i) {
    int64_t o = cnt[i];
    for (int64_t j = i + 1; j < n; ++j) {
      double g, nr[3];
      if (sphere_pair(pos, radius, i, j, gap_abs, gap_rel, &g, nr) > 0) {
        ci[o] = (int32_t)i; cj[o] = (int32_t)j; gap[o] = g;
        normal[3 * o + 0] = nr[0]; normal[3 * o + 1] = nr[1]; normal[3 * o + 2] = nr[2];
        ++o;
      }
    }
  }
  free(cnt);
  return total;
}

/* Uniform grid (independent of the GPU's cell list): bucket bodies by
 * floor((x - xmin)/h) with h >= the largest possible contact distance, test
 * the 27 surrounding buckets, keep j > i, sort each i's partners by j. */
static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

int64_t orc_contacts_spheres_grid(int64_t n, const double* pos, const double* radius,
                                  double gap_abs, double gap_rel, int64_t cap,
                                  int32_t* ci, int32_t* cj, double* gap, double* normal) {
  if (n < 0 || !pos || !radius) return -1;
  if (n == 0) return 0;
  double lo[3] = {pos[0], pos[1], pos[2]}, hi[3] = {pos[0], pos[1], pos[2]};
  double amax = radius[0];
  for (int64_t i = 0; i < n; ++i) {
    for (int d = 0; d < 3; ++d) {
      if (pos[3 * i + d] < lo[d]) lo[d] = pos[3 * i + d];
      if (pos[3 * i + d] > hi[d]) hi[d] = pos[3 * i + d];
    }
    if (radius[i] > amax) amax = radius[i];
  }
  double h = (2.0 * amax + fabs(gap_abs) + fabs(gap_rel) * amax) * 1.001 + 1e-9;
  int64_t m[3];
  for (int d = 0; d < 3; ++d) {
    m[d] = (int64_t)floor((hi[d] - lo[d]) / h) + 1;
    if (m[d] < 1) m[d] = 1;
  }
  while (m[0] * m[1] * m[2] > 8 * n + 64) { /* keep the table O(n) */
    h *= 1.5;
    for (int d = 0; d < 3; ++d) m[d] = (int64_t)floor((hi[d] - lo[d]) / h) + 1;
  }
  int64_t ncell = m[0] * m[1] * m[2];
  int64_t* head = (int64_t*)calloc((size_t)ncell + 1, sizeof(int64_t));
  int64_t* cell = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t* fill = (int64_t*)calloc((size_t)ncell, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) {
    int64_t k[3];
    for (int d = 0; d < 3; ++d) {
      k[d] = (int64_t)floor((pos[3 * i + d] - lo[d]) / h);
      if (k[d] >= m[d]) k[d] = m[d] - 1;
      if (k[d] < 0) k[d] = 0;
    }
    cell[i] = (k[2] * m[1] + k[1]) * m[0] + k[0];
    head[cell[i] + 1]++;
  }
  for (int64_t c = 0; c < ncell; ++c) head[c + 1] += head[c];
  for (int64_t i = 0; i < n; ++i) order[head[cell[i]] + fill[cell[i]]++] = i;
  free(fill);

  int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  int bad = 0;
  for (int pass = 0; pass < 2; ++pass) {
#pragma omp parallel for schedule(dynamic, 64) reduction(| : bad)
    for (int64_t i = 0; i < n; ++i) {
      int32_t partners[4096];
      int np = 0;
      int64_t ki = cell[i];
      int64_t kx = ki % m[0], ky = (ki / m[0]) % m[1], kz = ki / (m[0] * m[1]);
      for (int64_t z = kz - 1; z <= kz + 1; ++z)
        for (int64_t y = ky - 1; y <= ky + 1; ++y)
          for (int64_t x = kx - 1; x <= kx + 1; ++x) {
            if (x < 0 || y < 0 || z < 0 || x >= m[0] || y >= m[1] || z >= m[2]) continue;
            int64_t c = (z * m[1] + y) * m[0] + x;
            for (int64_t p = head[c]; p < head[c + 1]; ++p) {
              int64_t j = order[p];
              if (j <= i) continue;
              double g, nr[3];
              int s = sphere_pair(pos, radius, i, j, gap_abs, gap_rel, &g, nr);
              if (s < 0) bad = 1;
              if (s > 0 && np < 4096) partners[np++] = (int32_t)j;
            }
          }
      if (pass == 0) {
        cnt[i + 1] = np;
      } else {
        qsort(partners, (size_t)np, sizeof(int32_t), cmp_i32);
        int64_t o = cnt[i];
        for (int q = 0; q < np; ++q) {
          double g, nr[3];
          sphere_pair(pos, radius, i, partners[q], gap_abs, gap_rel, &g, nr);
          ci[o] = (int32_t)i; cj[o] = partners[q]; gap[o] = g;
          normal[3 * o + 0] = nr[0]; normal[3 * o + 1] = nr[1]; normal[3 * o + 2] = nr[2];
          ++o;
        }
      }
    }
    if (bad) break;
    if (pass == 0) {
      for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
      if (cnt[n] > cap) break;
    }
  }
  int64_t total = cnt[n];
  free(cnt); free(head); free(cell); free(order);
  if (bad) return -2;
  return total;
}

/* Spherocylinder minimal separation: closest points of the two axis segments
 * (textbook clamped parametric method; reading A15), segment of body k from
 * p = c - (L/2) t to p + L t. */
void orc_segment_closest(const double* c1, const double* t1, double L1,
                         const double* c2, const double* t2, double L2,
                         double* P1, double* P2) {
  double p1[3], p2[3], d1[3], d2[3], r[3];
  for (int k = 0; k < 3; ++k) {
    p1[k] = c1[k] - (0.5 * L1) * t1[k];
    p2[k] = c2[k] - (0.5 * L2) * t2[k];
    d1[k] = L1 * t1[k];
    d2[k] = L2 * t2[k];
    r[k] = p1[k] - p2[k];
  }
  double a = (d1[0] * d1[0] + d1[1] * d1[1]) + d1[2] * d1[2];
  double e = (d2[0] * d2[0] + d2[1] * d2[1]) + d2[2] * d2[2];
  double f = (d2[0] * r[0] + d2[1] * r[1]) + d2[2] * r[2];
  double c = (d1[0] * r[0] + d1[1] * r[1]) + d1[2] * r[2];
  double bb = (d1[0] * d2[0] + d1[1] * d2[1]) + d1[2] * d2[2];
  double denom = a * e - bb * bb;
  double s;
  if (denom > 1e-14 * (a * e)) {
    s = (bb * f - c * e) / denom;
    if (s < 0.0) s = 0.0;
    if (s > 1.0) s = 1.0;
  } else {
    s = 0.0; /* (near-)parallel: pick s = 0, then t from s */
  }
  double t = (bb * s + f) / e;
  if (t < 0.0) {
    t = 0.0;
    s = -c / a;
    if (s < 0.0) s = 0.0;
    if (s > 1.0) s = 1.0;
  } else if (t > 1.0) {
    t = 1.0;
    s = (bb - c) / a;
    if (s < 0.0) s = 0.0;
    if (s > 1.0) s = 1.0;
  }
  for (int k = 0; k < 3; ++k) {
    P1[k] = p1[k] + d1[k] * s;
    P2[k] = p2[k] + d2[k] * t;
  }
}

static int rod_pair(const double* center, const double* dir, const double* length, double b,
                    double gap_thresh, int64_t i, int64_t j, double* gap, double* nrm, double* lev) {
  double Pi[3], Pj[3];
  orc_segment_closest(center + 3 * i, dir + 3 * i, length[i], center + 3 * j, dir + 3 * j,
                      length[j], Pi, Pj);
  double dx = Pi[0] - Pj[0], dy = Pi[1] - Pj[1], dz = Pi[2] - Pj[2];
  double dist = sqrt((dx * dx + dy * dy) + dz * dz);
  double g = dist - 2.0 * b;
  if (!(g < gap_thresh)) return 0;
  if (dist < 1e-300) {
    /* axes intersect: normal along t_i x t_j, oriented from j to i */
    const double* a1 = dir + 3 * i;
    const double* a2 = dir + 3 * j;
    double cx = a1[1] * a2[2] - a1[2] * a2[1];
    double cy = a1[2] * a2[0] - a1[0] * a2[2];
    double cz = a1[0] * a2[1] - a1[1] * a2[0];
    double cn = sqrt((cx * cx + cy * cy) + cz * cz);
    if (cn == 0.0) return -2;
    double ox = center[3 * i] - center[3 * j], oy = center[3 * i + 1] - center[3 * j + 1],
           oz = center[3 * i + 2] - center[3 * j + 2];
    double sg = ((cx * ox + cy * oy) + cz * oz) >= 0.0 ? 1.0 : -1.0;
    nrm[0] = sg * cx / cn; nrm[1] = sg * cy / cn; nrm[2] = sg * cz / cn;
  } else {
    nrm[0] = dx / dist; nrm[1] = dy / dist; nrm[2] = dz / dist;
  }
  *gap = g;
  for (int k = 0; k < 3; ++k) {
    lev[k] = Pi[k] - center[3 * i + k];
    lev[3 + k] = Pj[k] - center[3 * j + k];
  }
  return 1;
}

int64_t orc_contacts_rods(int64_t n, const double* center, const double* dir, const double* length,
                          double b, double gap_thresh, int brute, int64_t cap,
                          int32_t* ci, int32_t* cj, double* gap, double* normal, double* lever) {
  if (n < 0 || !center || !dir || !length) return -1;
  double Lmax = 0.0;
  for (int64_t i = 0; i < n; ++i) if (length[i] > Lmax) Lmax = length[i];
  /* Exact prefilter: each closest point lies within L/2 of its centre, so a
   * contact needs |c_i - c_j| <= (L_i + L_j)/2 + 2b + gap_thresh. */
  int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  /* Sort bodies by x to prune: only j with |x_j - x_i| <= Lmax + 2b + thresh. */
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  double* xs = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  /* simple insertion-free approach: counting sort by integer slab index */
  double reach = Lmax + 2.0 * b + fabs(gap_thresh);
  double xmin = n ? center[0] : 0.0;
  for (int64_t i = 0; i < n; ++i) if (center[3 * i] < xmin) xmin = center[3 * i];
  int64_t nslab = 1;
  for (int64_t i = 0; i < n; ++i) {
    int64_t s = (int64_t)floor((center[3 * i] - xmin) / reach);
    if (s + 1 > nslab) nslab = s + 1;
  }
  int64_t* sh = (int64_t*)calloc((size_t)nslab + 1, sizeof(int64_t));
  int64_t* slab = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    slab[i] = (int64_t)floor((center[3 * i] - xmin) / reach);
    sh[slab[i] + 1]++;
  }
  for (int64_t s = 0; s < nslab; ++s) sh[s + 1] += sh[s];
  int64_t* sf = (int64_t*)calloc((size_t)nslab, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) order[sh[slab[i]] + sf[slab[i]]++] = i;
  free(sf);
  (void)xs;
  int bad = 0;
  for (int pass = 0; pass < 2; ++pass) {
#pragma omp parallel for schedule(dynamic, 64) reduction(| : bad)
    for (int64_t i = 0; i < n; ++i) {
      int32_t partners[4096];
      int np = 0;
      int64_t s0 = brute ? 0 : slab[i] - 1, s1 = brute ? nslab - 1 : slab[i] + 1;
      if (s0 < 0) s0 = 0;
      if (s1 > nslab - 1) s1 = nslab - 1;
      for (int64_t p = sh[s0]; p < sh[s1 + 1]; ++p) {
        int64_t j = order[p];
        if (j <= i) continue;
        if (!brute) {
          double ox = center[3 * i] - center[3 * j], oy = center[3 * i + 1] - center[3 * j + 1],
                 oz = center[3 * i + 2] - center[3 * j + 2];
          double cd = sqrt((ox * ox + oy * oy) + oz * oz);
          if (cd > 0.5 * (length[i] + length[j]) + 2.0 * b + fabs(gap_thresh)) continue;
        }
        double g, nr[3], lv[6];
        int st = rod_pair(center, dir, length, b, gap_thresh, i, j, &g, nr, lv);
        if (st < 0) bad = 1;
        if (st > 0 && np < 4096) partners[np++] = (int32_t)j;
      }
      if (pass == 0) {
        cnt[i + 1] = np;
      } else {
        qsort(partners, (size_t)np, sizeof(int32_t), cmp_i32);
        int64_t o = cnt[i];
        for (int q = 0; q < np; ++q) {
          double g, nr[3], lv[6];
          rod_pair(center, dir, length, b, gap_thresh, i, partners[q], &g, nr, lv);
          ci[o] = (int32_t)i; cj[o] = partners[q]; gap[o] = g;
          for (int k = 0; k < 3; ++k) normal[3 * o + k] = nr[k];
          for (int k = 0; k < 6; ++k) lever[6 * o + k] = lv[k];
          ++o;
        }
      }
    }
    if (bad) break;
    if (pass == 0) {
      for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
      if (cnt[n] > cap) break;
    }
  }
  int64_t total = cnt[n];
  free(cnt); free(order); free(xs); free(sh); free(slab);
  if (bad) return -2;
  return total;
}

/* ------------------------------------------------------------------------ */
/* Particle-boundary collisions (NEXT row f2): "for each       */
/* collision pair l between a particle and a boundary, a vector D_l can be  */
/* added to D ... these D_l column vectors have 6 non-zero entries          */
/* corresponding to the degrees of freedom of the particle only"; a         */
/* boundary "does not appear in the mobility matrix".  Boundaries here are  */
/* static planes n_k . x = h_k (unit n_k into the fluid).  Constraint       */
/* (i, n + k); normal n_k (from the wall to the particle, reading A13's     */
/* "from j to i").  Minimal separation of the particle and plane:  */
/*   sphere: Phi = (n . c - h) - a;                                         */
/*   rod: the axis segment's signed distance n.(c + s t) - h is linear in s */
/*        on [-L/2, L/2], so its minimum is at s = -L/2 (n.t > 0), +L/2     */
/*        (n.t < 0), anywhere for n.t = 0 (take s = 0, the centre);         */
/*        Phi = (n . P - h) - b with P = c + s t, lever r = P - c.          */
/* Thresholds as for pairs (reading A1): spheres gap_abs + gap_rel * a,     */
/* rods gap_abs.  Output in body order (i ascending, then k).               */
/* ------------------------------------------------------------------------ */
int64_t orc_contacts_walls(int kind, int64_t n, const double* pos, const double* radius, const double* dir,
                           const double* length, double b, int nw, const double* walls, double gap_abs,
                           double gap_rel, int64_t cap, int32_t* ci, int32_t* cj, double* gap, double* normal,
                           double* lever) {
  if (n < 0 || nw < 0 || (nw > 0 && !walls) || !pos) return -1;
  if (kind == 1 && (!dir || !length)) return -1;
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double* c = pos + 3 * i;
    for (int k = 0; k < nw; ++k) {
      const double* w = walls + 4 * k;
      double P[3] = {c[0], c[1], c[2]};
      double g, thr;
      if (kind == 0) {
        double a = radius ? radius[i] : 1.0;
        g = (((w[0] * c[0] + w[1] * c[1]) + w[2] * c[2]) - w[3]) - a;
        thr = gap_abs + gap_rel * a;
      } else {
        const double* t = dir + 3 * i;
        double nt = (w[0] * t[0] + w[1] * t[1]) + w[2] * t[2];
        double hl = 0.5 * length[i];
        double sv = nt > 0.0 ? -hl : (nt < 0.0 ? hl : 0.0);
        for (int d = 0; d < 3; ++d) P[d] = c[d] + sv * t[d];
        g = (((w[0] * P[0] + w[1] * P[1]) + w[2] * P[2]) - w[3]) - b;
        thr = gap_abs;
      }
      if (!(g < thr)) continue;
      if (m < cap) {
        ci[m] = (int32_t)i;
        cj[m] = (int32_t)(n + k);
        gap[m] = g;
        for (int d = 0; d < 3; ++d) normal[3 * m + d] = w[d];
        if (lever) {
          for (int d = 0; d < 3; ++d) {
            lever[6 * m + d] = P[d] - c[d];
            lever[6 * m + 3 + d] = 0.0;
          }
        }
      }
      ++m;
    }
  }
  return m;
}

/* ------------------------------------------------------------------------ */
/* D and D^T.  Column l: on body i (+n, r_i x n), on body j   */
/* (-n, -(r_j x n)); spheres carry no torque.                 */
/* ------------------------------------------------------------------------ */
static void column_blocks(const double* normal, const double* lever, int64_t l, double Di[6],
                          double Dj[6]) {
  const double* nv = normal + 3 * l;
  for (int k = 0; k < 3; ++k) { Di[k] = nv[k]; Dj[k] = -nv[k]; }
  if (lever) {
    const double* ri = lever + 6 * l;
    const double* rj = lever + 6 * l + 3;
    Di[3] = ri[1] * nv[2] - ri[2] * nv[1];
    Di[4] = ri[2] * nv[0] - ri[0] * nv[2];
    Di[5] = ri[0] * nv[1] - ri[1] * nv[0];
    Dj[3] = -(rj[1] * nv[2] - rj[2] * nv[1]);
    Dj[4] = -(rj[2] * nv[0] - rj[0] * nv[2]);
    Dj[5] = -(rj[0] * nv[1] - rj[1] * nv[0]);
  } else {
    for (int k = 3; k < 6; ++k) { Di[k] = 0.0; Dj[k] = 0.0; }
  }
}

int orc_apply_D(int64_t n, int64_t nc, const int32_t* ci, const int32_t* cj, const double* normal,
                const double* lever, const double* gamma, double* FT) {
  if (n < 0 || nc < 0) return -1;
  memset(FT, 0, sizeof(double) * 6 * (size_t)n);
  /* F_c = D gamma, accumulated in ascending constraint order.
   * cj >= n: a wall (entries on the particle only). */
  for (int64_t l = 0; l < nc; ++l) {
    if (ci[l] < 0 || cj[l] < 0 || ci[l] >= n || cj[l] >= n + ORC_MAX_WALLS) return -1;
    double Di[6], Dj[6];
    column_blocks(normal, lever, l, Di, Dj);
    for (int k = 0; k < 6; ++k) {
      FT[6 * (int64_t)ci[l] + k] += Di[k] * gamma[l];
      if (cj[l] < n) FT[6 * (int64_t)cj[l] + k] += Dj[k] * gamma[l];
    }
  }
  return 0;
}

int orc_apply_DT(int64_t n, int64_t nc, const int32_t* ci, const int32_t* cj, const double* normal,
                 const double* lever, const double* UW, double* out) {
  if (n < 0 || nc < 0) return -1;
  for (int64_t l = 0; l < nc; ++l) {
    if (ci[l] < 0 || cj[l] < 0 || ci[l] >= n || cj[l] >= n + ORC_MAX_WALLS) return -1;
    double Di[6], Dj[6];
    column_blocks(normal, lever, l, Di, Dj);
    double s = 0.0;
    for (int k = 0; k < 6; ++k) s += Di[k] * UW[6 * (int64_t)ci[l] + k];
    if (cj[l] < n)  /* a wall is at rest */
      for (int k = 0; k < 6; ++k) s += Dj[k] * UW[6 * (int64_t)cj[l] + k];
    out[l] = s;
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Mobility.  RPY translational blocks exactly as printed in B:configs[0]:  */
/*  r >= 2a: (1/(8 pi mu r)) [ (I + r r^T / r^2) + (2a^2/(3r^2)) (I - 3 r r^T/r^2) ] */
/*  r <  2a: (1/(6 pi mu a)) [ (1 - 9r/(32a)) I + (3/(32a)) r r^T / r ]       */
/* with a -> (a_i + a_j)/2 for unequal radii (B:configs[1], reading A11);   */
/* self block I/(6 pi mu a_i); self rotation I/(8 pi mu a_i^3) (reading A10). */
/* ------------------------------------------------------------------------ */
void orc_rpy_block(const double* xi, double ai, const double* xj, double aj, double mu, int self,
                   double* M) {
  if (self) {
    double s = 1.0 / (6.0 * ORC_PI * mu * ai);
    for (int p = 0; p < 3; ++p)
      for (int q = 0; q < 3; ++q) M[3 * p + q] = (p == q) ? s : 0.0;
    return;
  }
  double rv[3] = {xj[0] - xi[0], xj[1] - xi[1], xj[2] - xi[2]};
  double r2 = rv[0] * rv[0] + rv[1] * rv[1] + rv[2] * rv[2];
  double r = sqrt(r2);
  double a = 0.5 * (ai + aj);
  for (int p = 0; p < 3; ++p) {
    for (int q = 0; q < 3; ++q) {
      double I = (p == q) ? 1.0 : 0.0;
      double rr = rv[p] * rv[q];
      double v;
      if (r >= 2.0 * a) {
        v = (1.0 / (8.0 * ORC_PI * mu * r)) *
            ((I + rr / r2) + (2.0 * a * a / (3.0 * r2)) * (I - 3.0 * rr / r2));
      } else {
        v = (1.0 / (6.0 * ORC_PI * mu * a)) * ((1.0 - 9.0 * r / (32.0 * a)) * I + (3.0 / (32.0 * a)) * rr / r);
      }
      M[3 * p + q] = v;
    }
  }
}

static int rpy_row(int64_t n, const double* pos, const double* radius, double mu, const double* FT,
                   int64_t i, double* out6) {
  long double acc[3] = {0.0L, 0.0L, 0.0L};
  double M[9];
  for (int64_t j = 0; j < n; ++j) {
    if (j != i) {
      if (pos[3 * i] == pos[3 * j] && pos[3 * i + 1] == pos[3 * j + 1] && pos[3 * i + 2] == pos[3 * j + 2])
        return -2; /* coincident centres (reading A12) */
    }
    orc_rpy_block(pos + 3 * i, radius[i], pos + 3 * j, radius[j], mu, j == i, M);
    for (int p = 0; p < 3; ++p)
      for (int q = 0; q < 3; ++q) acc[p] += (long double)M[3 * p + q] * (long double)FT[6 * j + q];
  }
  for (int p = 0; p < 3; ++p) out6[p] = (double)acc[p];
  double rot = 1.0 / (8.0 * ORC_PI * mu * radius[i] * radius[i] * radius[i]);
  for (int p = 0; p < 3; ++p) out6[3 + p] = rot * FT[6 * i + 3 + p];
  return 0;
}

int orc_rpy_apply_rows(int64_t n, const double* pos, const double* radius, double mu,
                       const double* FT, int64_t row0, int64_t row1, double* UW_rows) {
  if (n < 0 || row0 < 0 || row1 > n || row0 > row1 || !(mu > 0)) return -1;
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(| : bad)
  for (int64_t i = row0; i < row1; ++i) {
    if (rpy_row(n, pos, radius, mu, FT, i, UW_rows + 6 * (i - row0)) != 0) bad = 1;
  }
  return bad ? -2 : 0;
}

int orc_rpy_apply(int64_t n, const double* pos, const double* radius, double mu,
                  const double* FT, double* UW) {
  return orc_rpy_apply_rows(n, pos, radius, mu, FT, 0, n, UW);
}

/* ------------------------------------------------------------------------ */
/* NEXT row f4(ii): the full 6N RPY grand mobility (reading A27).  The      */
/* paper cites RPY only and BASELINE specifies the              */
/* translational blocks; the coupling blocks below restate the RPY          */
/* literature's expressions for equal spheres (radius a -> abar, reading    */
/* A11), with r = x_i - x_j, rhat = r / |r|, [v]x w = v x w:                */
/*   rt (Omega_i from F_j) and tr (U_i from T_j):  -c(r) [rhat]x,           */
/*     c = 1/(8 pi mu r^2)                             r >= 2a              */
/*     c = (1/(16 pi mu a^2)) (r/a - 3 r^2/(8 a^2))    r <  2a              */
/*   rr (Omega_i from T_j):                                                 */
/*     (1/(16 pi mu r^3)) (3 rhat rhat^T - I)          r >= 2a              */
/*     (1/(8 pi mu a^3)) [(1 - 27r/(32a) + 5r^3/(64a^3)) I                  */
/*                        + (9r/(32a) - 3r^3/(64a^3)) rhat rhat^T]   r < 2a */
/* Far field: rt = 1/2 curl of the translational (Stokeslet + degenerate    */
/* quadrupole) field, rr = 1/2 curl of the rotlet; the branches join C^1 at */
/* r = 2a and reduce to the self blocks (0 and I/(8 pi mu a^3)) at r = 0.   */
/* Self: tt I/(6 pi mu a_i), rr I/(8 pi mu a_i^3), tr = rt = 0.             */
/* M66 row-major: [[tt, tr], [rt, rr]] maps (F_j, T_j) to (U_i, Omega_i).   */
/* ------------------------------------------------------------------------ */
void orc_rpy6_block(const double* xi, double ai, const double* xj, double aj, double mu, int self,
                    double* M66) {
  double tt[9];
  orc_rpy_block(xi, ai, xj, aj, mu, self, tt);
  for (int k = 0; k < 36; ++k) M66[k] = 0.0;
  for (int p = 0; p < 3; ++p)
    for (int q = 0; q < 3; ++q) M66[6 * p + q] = tt[3 * p + q];
  if (self) {
    double s = 1.0 / (8.0 * ORC_PI * mu * ai * ai * ai);
    for (int p = 0; p < 3; ++p) M66[6 * (3 + p) + 3 + p] = s;
    return;
  }
  double rv[3] = {xi[0] - xj[0], xi[1] - xj[1], xi[2] - xj[2]};
  double r = sqrt(rv[0] * rv[0] + rv[1] * rv[1] + rv[2] * rv[2]);
  double e[3] = {rv[0] / r, rv[1] / r, rv[2] / r};
  double a = 0.5 * (ai + aj);
  double c, cI, cR;
  if (r >= 2.0 * a) {
    c = 1.0 / (8.0 * ORC_PI * mu * r * r);
    cI = -1.0 / (16.0 * ORC_PI * mu * r * r * r);
    cR = 3.0 / (16.0 * ORC_PI * mu * r * r * r);
  } else {
    c = (1.0 / (16.0 * ORC_PI * mu * a * a)) * (r / a - 3.0 * r * r / (8.0 * a * a));
    cI = (1.0 / (8.0 * ORC_PI * mu * a * a * a)) * (1.0 - 27.0 * r / (32.0 * a) + 5.0 * r * r * r / (64.0 * a * a * a));
    cR = (1.0 / (8.0 * ORC_PI * mu * a * a * a)) * (9.0 * r / (32.0 * a) - 3.0 * r * r * r / (64.0 * a * a * a));
  }
  /* [e]x as a matrix: [[0,-e2,e1],[e2,0,-e0],[-e1,e0,0]]; the blocks are -c [e]x */
  double X[9] = {0.0, -e[2], e[1], e[2], 0.0, -e[0], -e[1], e[0], 0.0};
  for (int p = 0; p < 3; ++p)
    for (int q = 0; q < 3; ++q) {
      M66[6 * p + 3 + q] = -c * X[3 * p + q];        /* tr */
      M66[6 * (3 + p) + q] = -c * X[3 * p + q];      /* rt */
      M66[6 * (3 + p) + 3 + q] = cI * (p == q ? 1.0 : 0.0) + cR * e[p] * e[q];  /* rr */
    }
}

static int rpy6_row(int64_t n, const double* pos, const double* radius, double mu, const double* FT,
                    int64_t i, double* out6) {
  long double acc[6] = {0.0L, 0.0L, 0.0L, 0.0L, 0.0L, 0.0L};
  double M[36];
  for (int64_t j = 0; j < n; ++j) {
    if (j != i && pos[3 * i] == pos[3 * j] && pos[3 * i + 1] == pos[3 * j + 1] && pos[3 * i + 2] == pos[3 * j + 2])
      return -2; /* coincident centres (reading A12) */
    orc_rpy6_block(pos + 3 * i, radius[i], pos + 3 * j, radius[j], mu, j == i, M);
    for (int p = 0; p < 6; ++p)
      for (int q = 0; q < 6; ++q) acc[p] += (long double)M[6 * p + q] * (long double)FT[6 * j + q];
  }
  for (int p = 0; p < 6; ++p) out6[p] = (double)acc[p];
  return 0;
}

int orc_rpy6_apply_rows(int64_t n, const double* pos, const double* radius, double mu, const double* FT,
                        int64_t row0, int64_t row1, double* UW_rows) {
  if (n < 0 || row0 < 0 || row1 > n || row0 > row1 || !(mu > 0)) return -1;
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(| : bad)
  for (int64_t i = row0; i < row1; ++i) {
    if (rpy6_row(n, pos, radius, mu, FT, i, UW_rows + 6 * (i - row0)) != 0) bad = 1;
  }
  return bad ? -2 : 0;
}

/* Spherocylinder drag, B:configs[3]:
 *   U = (1/zeta_par) t t^T F + (1/zeta_perp) (I - t t^T) F,
 *   zeta_perp = 2 zeta_par = 4 pi mu L / ln(L/(2b)),
 *   Omega = T / zeta_rot,  zeta_rot = pi mu L^3 / (3 ln(L/(2b))). */
int orc_rod_drag_apply(int64_t n, const double* dir, const double* length, double b, double mu,
                       const double* FT, double* UW) {
  if (n < 0 || !(b > 0) || !(mu > 0)) return -1;
#pragma omp parallel for
  for (int64_t i = 0; i < n; ++i) {
    double L = length[i];
    double lg = log(L / (2.0 * b));
    double zperp = 4.0 * ORC_PI * mu * L / lg;
    double zpar = 0.5 * zperp;
    double zrot = ORC_PI * mu * L * L * L / (3.0 * lg);
    const double* t = dir + 3 * i;
    const double* F = FT + 6 * i;
    for (int p = 0; p < 3; ++p) {
      double v = 0.0;
      for (int q = 0; q < 3; ++q) {
        double tt = t[p] * t[q];
        double I = (p == q) ? 1.0 : 0.0;
        v += ((1.0 / zpar) * tt + (1.0 / zperp) * (I - tt)) * F[q];
      }
      UW[6 * i + p] = v;
      UW[6 * i + 3 + p] = F[3 + p] / zrot;
    }
  }
  return 0;
}

static int mobility(const orc_system* s, const double* FT, double* UW) {
  if (s->kind == 0) return orc_rpy_apply(s->n, s->pos, s->radius, s->mu, FT, UW);
  if (s->kind == 2) return orc_rpy6_apply_rows(s->n, s->pos, s->radius, s->mu, FT, 0, s->n, UW);
  return orc_rod_drag_apply(s->n, s->dir, s->length, s->b, s->mu, FT, UW);
}

/* One evaluation of M x = D^T Mobility D x: one MVOP. */
int orc_mvop(const orc_system* s, const double* x, double* w) {
  double* FT = (double*)malloc(sizeof(double) * 6 * (size_t)(s->n > 0 ? s->n : 1));
  double* UW = (double*)malloc(sizeof(double) * 6 * (size_t)(s->n > 0 ? s->n : 1));
  int st = orc_apply_D(s->n, s->nc, s->ci, s->cj, s->normal, s->lever, x, FT);
  if (st == 0) st = mobility(s, FT, UW);
  if (st == 0) st = orc_apply_DT(s->n, s->nc, s->ci, s->cj, s->normal, s->lever, UW, w);
  free(FT);
  free(UW);
  return st;
}

/* q = Phi/dt + D^T U_nc. */
int orc_lcp_q(const orc_system* s, const double* gap, double dt, const double* U_nc, double* q) {
  if (!(dt > 0)) return -1;
  int st = orc_apply_DT(s->n, s->nc, s->ci, s->cj, s->normal, s->lever, U_nc, q);
  if (st) return st;
  for (int64_t l = 0; l < s->nc; ++l) q[l] = gap[l] / dt + q[l];
  return 0;
}

/* Moving boundaries (NEXT row f2: "a boundary refers to any object either static
 * or moving with a prescribed velocity"; it "does not appear in the mobility matrix").  Wall k
 * moves with the prescribed velocity V_k, so the gap rate of a particle-wall constraint l = (i, k)
 * is n_k . (U_i + Omega_i x r_i) - n_k . V_k: D is unchanged and the wall's motion
 * enters only the constant part of the LCP,
 *   q_l = gap_l/dt + D_l^T U_nc - n_l . V_k   (cj[l] = n + k; n_l = n_k for a wall constraint). */
int orc_lcp_q_moving_walls(const orc_system* s, const double* gap, double dt, const double* U_nc, int nw,
                           const double* wall_vel, double* q) {
  int st = orc_lcp_q(s, gap, dt, U_nc, q);
  if (st) return st;
  for (int64_t l = 0; l < s->nc; ++l) {
    int64_t k = (int64_t)s->cj[l] - s->n;
    if (k < 0) continue;
    if (k >= nw) return -1;
    const double* nl = s->normal + 3 * l;
    const double* v = wall_vel + 3 * k;
    q[l] = q[l] - (nl[0] * v[0] + nl[1] * v[1] + nl[2] * v[2]);
  }
  return 0;
}

/* phi(gamma, g) = || min(gamma, g) ||_2, long double sum. */
double orc_minmap_residual(int64_t n, const double* gamma, const double* g) {
  long double s = 0.0L;
  for (int64_t l = 0; l < n; ++l) {
    double m = gamma[l] < g[l] ? gamma[l] : g[l];
    s += (long double)m * (long double)m;
  }
  return sqrt((double)s);
}

static double dot(int64_t n, const double* a, const double* b) {
  long double s = 0.0L;
  for (int64_t l = 0; l < n; ++l) s += (long double)a[l] * (long double)b[l];
  return (double)s;
}

/* ------------------------------------------------------------------------ */
/* BBPGD, Alg. 1, step numbers in the comments.  Readings:    */
/* A3 gamma_0 given (zero in parity runs); A5 on breakdown (s^T y <= 0 or a */
/* non-finite step) reuse the previous alpha and count it; A6 strict '<';  */
/* A7 return the last iterate when j_max is reached; A8 MVOPs = 2 + iters. */
/* ------------------------------------------------------------------------ */
typedef int (*mvop_fn)(const void* ctx, const double* x, double* w);

static int bbpgd_core(int64_t n, mvop_fn mv, const void* ctx, const double* q, double tol,
                      int32_t max_iter, int32_t bb_mode, int32_t fixed_iters, double* gamma,
                      double* g_out, orc_stats* st) {
  memset(st, 0, sizeof(*st));
  size_t bytes = sizeof(double) * (size_t)(n > 0 ? n : 1);
  double* g = (double*)malloc(bytes);
  double* gprev = (double*)malloc(bytes);
  double* gam_prev = (double*)malloc(bytes);
  double* w = (double*)malloc(bytes);
  int status = 0;
  /* Step 1: initial guess gamma_0 (projected: the CQP is over gamma >= 0). */
  for (int64_t l = 0; l < n; ++l) if (!(gamma[l] > 0.0)) gamma[l] = 0.0;
  /* Step 2: g_0 = M gamma_0 + q  (one MVOP, even when gamma_0 = 0: A8). */
  int st_mv = mv(ctx, gamma, w);
  if (st_mv) { status = st_mv; goto done; }
  st->mvops = 1;
  for (int64_t l = 0; l < n; ++l) g[l] = w[l] + q[l];
  /* Step 3-5: converged already? */
  st->residual = orc_minmap_residual(n, gamma, g);
  if (!isfinite(st->residual)) { status = -3; goto done; }
  if (st->residual < tol) { st->converged = 1; goto done; }
  /* Step 6: alpha_0 = g0^T g0 / g0^T M g0  (second MVOP). */
  st_mv = mv(ctx, g, w);
  if (st_mv) { status = st_mv; goto done; }
  st->mvops = 2;
  double alpha = dot(n, g, g) / dot(n, g, w);
  if (!isfinite(alpha) || !(alpha > 0.0)) { status = -3; goto done; }
  /* Steps 7-16 */
  for (int32_t j = 1; j <= max_iter; ++j) {
    memcpy(gam_prev, gamma, bytes);
    memcpy(gprev, g, bytes);
    /* Step 8: descent step; Step 9: projection max(0, .) (reading A23) */
    for (int64_t l = 0; l < n; ++l) {
      double v = gam_prev[l] - alpha * gprev[l];
      gamma[l] = v > 0.0 ? v : 0.0;
    }
    /* Step 10: gradient g_j = M gamma_j + q */
    st_mv = mv(ctx, gamma, w);
    if (st_mv) { status = st_mv; goto done; }
    st->mvops += 1;
    for (int64_t l = 0; l < n; ++l) g[l] = w[l] + q[l];
    st->iters = j;
    /* Step 11: convergence test */
    st->residual = orc_minmap_residual(n, gamma, g);
    if (!isfinite(st->residual)) { status = -3; goto done; }
    if (st->residual < tol) {
      st->converged = 1;
      if (!fixed_iters) break;
    }
    /* Steps 14-15 also run at j = j_max: Alg. 1 has them inside the loop body */
    /* Step 14: s = gamma_j - gamma_{j-1}, y = g_j - g_{j-1} */
    long double ss = 0.0L, sy = 0.0L, yy = 0.0L;
    for (int64_t l = 0; l < n; ++l) {
      double s = gamma[l] - gam_prev[l];
      double y = g[l] - gprev[l];
      ss += (long double)s * s;
      sy += (long double)s * y;
      yy += (long double)y * y;
    }
    /* Step 15: BB1 = s^T s / s^T y, BB2 = s^T y / y^T y */
    int use_bb2 = (bb_mode == 1) || (bb_mode == 2 && (j % 2 == 0));
    double a_new = use_bb2 ? (double)(sy / yy) : (double)(ss / sy);
    if (sy > 0.0L && isfinite(a_new) && a_new > 0.0) {
      alpha = a_new;
    } else {
      st->bb_breakdowns += 1; /* reading A5: keep the previous alpha */
    }
  }
  if (fixed_iters) {
    st->converged = st->residual < tol; /* reading A22: report the final residual */
    status = 0;
  } else if (!st->converged) {
    status = 1;
  }
done:
  if (g_out && status >= 0) memcpy(g_out, g, bytes);
  {
    int32_t act = 0;
    for (int64_t l = 0; l < n; ++l) if (gamma[l] > 0.0) ++act;
    st->active = act; /* |A_c| = #{gamma_l > 0} */
  }
  free(g); free(gprev); free(gam_prev); free(w);
  return status;
}

static int sys_mv(const void* ctx, const double* x, double* w) {
  return orc_mvop((const orc_system*)ctx, x, w);
}

int orc_bbpgd(const orc_system* s, const double* q, double tol, int32_t max_iter, int32_t bb_mode,
              int32_t fixed_iters, double* gamma, double* g_out, double* Fc_out, double* Uc_out,
              orc_stats* st) {
  int status = bbpgd_core(s->nc, sys_mv, s, q, tol, max_iter, bb_mode, fixed_iters, gamma, g_out, st);
  if (status < 0) return status;
  /* U_c and F_c for the returned gamma. */
  if (Fc_out || Uc_out) {
    double* FT = (double*)malloc(sizeof(double) * 6 * (size_t)(s->n > 0 ? s->n : 1));
    orc_apply_D(s->n, s->nc, s->ci, s->cj, s->normal, s->lever, gamma, FT);
    if (Fc_out) memcpy(Fc_out, FT, sizeof(double) * 6 * (size_t)s->n);
    if (Uc_out) mobility(s, FT, Uc_out);
    free(FT);
  }
  return status;
}

typedef struct { int64_t n; const double* M; } dense_ctx;
static int dense_mv(const void* ctx, const double* x, double* w) {
  const dense_ctx* d = (const dense_ctx*)ctx;
  for (int64_t r = 0; r < d->n; ++r) {
    long double s = 0.0L;
    for (int64_t c = 0; c < d->n; ++c) s += (long double)d->M[r * d->n + c] * x[c];
    w[r] = (double)s;
  }
  return 0;
}

int orc_bbpgd_dense(int64_t n, const double* M, const double* q, double tol, int32_t max_iter,
                    int32_t bb_mode, double* gamma, double* g_out, orc_stats* st) {
  dense_ctx d = {n, M};
  return bbpgd_core(n, dense_mv, &d, q, tol, max_iter, bb_mode, 0, gamma, g_out, st);
}

/* ------------------------------------------------------------------------ */
/* Step 4 of the time step: C^{k+1} = C^k + G U dt (Eq. time-step,  */
/* P:L468) with the quaternion kinematics theta' = Psi(theta) Omega          */
/* and renormalisation of the quaternion.                     */
/* ------------------------------------------------------------------------ */
int orc_euler_update(int64_t n, double dt, const double* UW, double* pos, double* quat, double* dir) {
  if (n < 0 || !(dt > 0)) return -1;
  for (int64_t i = 0; i < n; ++i) {
    const double* U = UW + 6 * i;
    const double* W = U + 3;
    for (int k = 0; k < 3; ++k) pos[3 * i + k] = pos[3 * i + k] + dt * U[k];
    if (quat) {
      double* th = quat + 4 * i;
      double s = th[0], px = th[1], py = th[2], pz = th[3];
      /* Psi Omega = 1/2 [ -p.W ; s W - p x W ] */
      double ds = -0.5 * (px * W[0] + py * W[1] + pz * W[2]);
      double cx = py * W[2] - pz * W[1];
      double cy = pz * W[0] - px * W[2];
      double cz = px * W[1] - py * W[0];
      double dx = 0.5 * (s * W[0] - cx);
      double dy = 0.5 * (s * W[1] - cy);
      double dz = 0.5 * (s * W[2] - cz);
      s += dt * ds; px += dt * dx; py += dt * dy; pz += dt * dz;
      double nn = sqrt(s * s + px * px + py * py + pz * pz);
      th[0] = s / nn; th[1] = px / nn; th[2] = py / nn; th[3] = pz / nn;
    }
    if (dir) {
      double* t = dir + 3 * i;
      double wx = W[1] * t[2] - W[2] * t[1];
      double wy = W[2] * t[0] - W[0] * t[2];
      double wz = W[0] * t[1] - W[1] * t[0];
      double ax = t[0] + dt * wx, ay = t[1] + dt * wy, az = t[2] + dt * wz;
      double nn = sqrt(ax * ax + ay * ay + az * az);
      t[0] = ax / nn; t[1] = ay / nn; t[2] = az / nn;
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------ */
/* APGD (NEXT row f3): accelerated projected gradient descent of Mazhar et   */
/* al. 2015, the comparison solver the paper cites.  Readings  */
/* (A24): gamma_0 = 0, L_0 = g0.M g0 / g0.g0, back-tracking L <- 2L */
/* until f(x') <= f(y) + g.(x' - y) + L/2 |x' - y|^2, Nesterov theta / beta, */
/* gradient restart when g.(x' - x) > 0, L <- 0.9 L after each step, stop on */
/* phi(x', M x' + q) < tol.  stats->bb_breakdowns = restarts.                 */
/* ------------------------------------------------------------------------ */
static int apgd_core(int64_t n, mvop_fn mv, const void* ctx, const double* q, double tol, int32_t max_iter,
                     double* gamma, double* g_out, orc_stats* st) {
  memset(st, 0, sizeof(*st));
  size_t bytes = sizeof(double) * (size_t)(n > 0 ? n : 1);
  double* x = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  double* xn = (double*)malloc(bytes);
  double* y = (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double));
  double* gy = (double*)malloc(bytes);
  double* gn = (double*)malloc(bytes);
  double* w = (double*)malloc(bytes);
  int status = 0;
  /* gamma_0 = 0, g_0 = M 0 + q = q (one counted MVOP, as Step 2 of Alg. 1) */
  for (int64_t l = 0; l < n; ++l) gy[l] = q[l];
  st->mvops = 1;
  st->residual = orc_minmap_residual(n, x, gy);
  if (st->residual < tol) { st->converged = 1; memcpy(gn, gy, bytes); goto done; }
  if (mv(ctx, gy, w)) { status = -1; goto done; }
  st->mvops = 2;
  double L = dot(n, gy, w) / dot(n, gy, gy);
  if (!(isfinite(L) && L > 0.0)) { status = -3; goto done; }
  double t = 1.0 / L, theta = 1.0, fy = 0.0;
  int restarts = 0;
  for (int32_t k = 1; k <= max_iter; ++k) {
    double fxn = 0.0, s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int bt = 0;; ++bt) {
      long double a0 = 0.0L, a1 = 0.0L, a2 = 0.0L;
      for (int64_t l = 0; l < n; ++l) {
        double v = y[l] - t * gy[l];
        xn[l] = v > 0.0 ? v : 0.0;
        double d = xn[l] - y[l];
        a0 += (long double)gy[l] * d;
        a1 += (long double)d * d;
        a2 += (long double)gy[l] * (xn[l] - x[l]);
      }
      s0 = (double)a0; s1 = (double)a1; s2 = (double)a2;
      if (mv(ctx, xn, w)) { status = -1; goto done; }
      st->mvops += 1;
      for (int64_t l = 0; l < n; ++l) gn[l] = w[l] + q[l];
      fxn = 0.5 * dot(n, xn, w) + dot(n, q, xn);
      double rhs = fy + s0 + 0.5 * L * s1;
      if (fxn <= rhs + 1e-12 * (fabs(fxn) + fabs(rhs)) || bt >= 60) break;
      L *= 2.0;
      t = 1.0 / L;
    }
    st->iters = k;
    st->residual = orc_minmap_residual(n, xn, gn);
    if (!isfinite(st->residual)) { status = -3; goto done; }
    double theta_n = 0.5 * (-theta * theta + theta * sqrt(theta * theta + 4.0));
    double beta = theta * (1.0 - theta) / (theta * theta + theta_n);
    int restart = s2 > 0.0;
    for (int64_t l = 0; l < n; ++l) {
      double xo = x[l];
      x[l] = xn[l];
      xn[l] = xo; /* xn now holds gamma_k */
    }
    if (st->residual < tol) { st->converged = 1; break; }
    if (restart) {
      ++restarts;
      memcpy(y, x, bytes);
      memcpy(gy, gn, bytes);
      fy = fxn;
      theta = 1.0;
    } else {
      for (int64_t l = 0; l < n; ++l) y[l] = x[l] + beta * (x[l] - xn[l]);
      if (mv(ctx, y, w)) { status = -1; goto done; }
      st->mvops += 1;
      for (int64_t l = 0; l < n; ++l) gy[l] = w[l] + q[l];
      fy = 0.5 * dot(n, y, w) + dot(n, q, y);
      theta = theta_n;
    }
    L *= 0.9;
    t = 1.0 / L;
  }
  st->bb_breakdowns = restarts;
  if (!st->converged) status = 1;
done:
  memcpy(gamma, x, bytes);
  if (g_out && status >= 0) {
    /* gradient at the returned iterate */
    if (mv(ctx, x, w) == 0)
      for (int64_t l = 0; l < n; ++l) g_out[l] = w[l] + q[l];
  }
  {
    int32_t act = 0;
    for (int64_t l = 0; l < n; ++l) if (gamma[l] > 0.0) ++act;
    st->active = act;
  }
  free(x); free(xn); free(y); free(gy); free(gn); free(w);
  return status;
}

int orc_apgd(const orc_system* s, const double* q, double tol, int32_t max_iter, double* gamma, double* g_out,
             orc_stats* st) {
  return apgd_core(s->nc, sys_mv, s, q, tol, max_iter, gamma, g_out, st);
}

int orc_apgd_dense(int64_t n, const double* M, const double* q, double tol, int32_t max_iter, double* gamma,
                   double* g_out, orc_stats* st) {
  dense_ctx d = {n, M};
  return apgd_core(n, dense_mv, &d, q, tol, max_iter, gamma, g_out, st);
}
