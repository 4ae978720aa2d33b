/* oracle.h -- plain, slow, obviously-correct CPU FP64 oracle.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA product under
 * paper_1909_06623_b200/ and include/ (and neither side includes the other).
 *
 * Citations: "P:Lnnn" = line of /root/reference/PAPER.md (arXiv 1909.06623),
 * "B:configs[k]" = /root/repo/BASELINE.json.  Readings A1..A23 are listed in
 * DESIGN.md ("Readings of the paper").
 *
 * Layouts: vectors of bodies are row-major double[N][k]; 6-vectors per body
 * are (Fx,Fy,Fz,Tx,Ty,Tz) / (Ux,Uy,Uz,Wx,Wy,Wz).
 * Constraint lists are sorted by (i, j) with i < j; the unit normal points
 * from j to i (reading A13), +n acts on i and -n on j.
 *
 * Status codes: 0 ok, 1 not converged, -1 bad argument, -2 degenerate
 * (coincident centres), -3 non-finite value, -4 capacity exceeded.
 */
#ifndef STOKESCOL_ORACLE_H
#define STOKESCOL_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* ---- contacts (P:L449-L463 near set A(C, delta); threshold reading A1) ---- */
/* Spheres: include pair i<j iff  gap < gap_abs + gap_rel*min(a_i,a_j),
 * gap = |c_i - c_j| - (a_i + a_j).  Brute force over all pairs.  Returns n_c
 * (or a negative status); writes at most cap entries. */
int64_t orc_contacts_spheres_brute(int64_t n, const double* pos, const double* radius,
                                   double gap_abs, double gap_rel, int64_t cap,
                                   int32_t* ci, int32_t* cj, double* gap, double* normal);
/* Same set by an independent uniform grid search (large N). */
int64_t orc_contacts_spheres_grid(int64_t n, const double* pos, const double* radius,
                                  double gap_abs, double gap_rel, int64_t cap,
                                  int32_t* ci, int32_t* cj, double* gap, double* normal);
/* Spherocylinders: segment-segment minimal distance, gap = dist - 2b < gap_thresh.
 * lever[l][0][:] = P_i - c_i, lever[l][1][:] = P_j - c_j.  brute != 0: all pairs
 * without the centre-distance prefilter (for verifying the prefilter). */
int64_t orc_contacts_rods(int64_t n, const double* center, const double* dir, const double* length,
                          double b, double gap_thresh, int brute, int64_t cap,
                          int32_t* ci, int32_t* cj, double* gap, double* normal, double* lever);
/* Closest points between two segments (exposed for tests). */
void orc_segment_closest(const double* c1, const double* t1, double L1,
                         const double* c2, const double* t2, double L2,
                         double* P1, double* P2);

/* ---- particle-boundary constraints (NEXT row f2) ---- */
/* Static planes n_k . x = h_k (walls: nw x 4 = (nx, ny, nz, h), unit n into the fluid).
 * kind 0 spheres (radius may be NULL: 1), 1 rods (dir, length, radius b).  Emits
 * (i, n + k) in body order with gap, normal n_k and (rods, lever != NULL) r_i = P - c_i,
 * r_j = 0.  Thresholds: spheres gap_abs + gap_rel * a_i, rods gap_abs (strict '<'). */
#define ORC_MAX_WALLS 8
int64_t orc_contacts_walls(int kind, int64_t n, const double* pos, const double* radius, const double* dir,
                           const double* length, double b, int nw, const double* walls, double gap_abs,
                           double gap_rel, int64_t cap, int32_t* ci, int32_t* cj, double* gap, double* normal,
                           double* lever);

/* ---- collision matrix D and its transpose ---- */
/* cj >= n marks a wall constraint (entries on body ci only). */
/* lever == NULL: sphere columns (6 nnz); else rod columns (12 nnz). */
int orc_apply_D(int64_t n, int64_t nc, const int32_t* ci, const int32_t* cj, const double* normal,
                const double* lever, const double* gamma, double* FT /* n x 6 */);
int orc_apply_DT(int64_t n, int64_t nc, const int32_t* ci, const int32_t* cj, const double* normal,
                 const double* lever, const double* UW /* n x 6 */, double* out /* nc */);

/* ---- mobility U = M F (formulas B:configs[0], [1], [3]) ---- */
/* RPY translational pair blocks + self translation 1/(6 pi mu a_i) + self rotation
 * 1/(8 pi mu a_i^3); pair radius (a_i+a_j)/2 (reading A11).  Sums in long double. */
int orc_rpy_apply(int64_t n, const double* pos, const double* radius, double mu,
                  const double* FT, double* UW);
/* Rows [row0, row1) only (sampled parity at full size). */
int orc_rpy_apply_rows(int64_t n, const double* pos, const double* radius, double mu,
                       const double* FT, int64_t row0, int64_t row1, double* UW_rows);
/* The 3x3 translational block M_ij (i != j) or M_ii, as printed in B:configs[0]. */
void orc_rpy_block(const double* xi, double ai, const double* xj, double aj, double mu, int self,
                   double* M33);
/* NEXT row f4(ii): the full 6N RPY grand mobility (reading A27): translation-rotation and
 * rotation-rotation pair blocks added to orc_rpy_block's; M66 row-major [[tt, tr], [rt, rr]]
 * maps (F_j, T_j) to (U_i, Omega_i).  Sums in long double. */
void orc_rpy6_block(const double* xi, double ai, const double* xj, double aj, double mu, int self,
                    double* M66);
int orc_rpy6_apply_rows(int64_t n, const double* pos, const double* radius, double mu, const double* FT,
                        int64_t row0, int64_t row1, double* UW_rows);
/* Block-diagonal spherocylinder drag (B:configs[3]). */
int orc_rod_drag_apply(int64_t n, const double* dir, const double* length, double b, double mu,
                       const double* FT, double* UW);

/* ---- LCP setup and BBPGD (Alg. 1) ---- */
typedef struct {
  int kind;               /* 0 spheres RPY, 1 rods drag, 2 spheres full 6N RPY (f4(ii)) */
  int64_t n;
  const double* pos;      /* spheres */
  const double* radius;   /* spheres */
  const double* dir;      /* rods */
  const double* length;   /* rods */
  double b, mu;
  int64_t nc;
  const int32_t* ci; const int32_t* cj;
  const double* normal; const double* lever;
} orc_system;

/* q = gap/dt + D^T U_nc. */
int orc_lcp_q(const orc_system* s, const double* gap, double dt, const double* U_nc, double* q);
/* q with moving walls: q_l -= n_l . V_k for wall constraints (cj = n + k); wall_vel: nw x 3. */
int orc_lcp_q_moving_walls(const orc_system* s, const double* gap, double dt, const double* U_nc, int nw,
                           const double* wall_vel, double* q);
/* One MVOP  w = M x = D^T (Mobility (D x)). */
int orc_mvop(const orc_system* s, const double* x, double* w);

typedef struct {
  int32_t iters, mvops, converged, bb_breakdowns, active;
  double residual;
} orc_stats;
/* bb_mode: 0 BB1, 1 BB2, 2 alternate.  fixed_iters != 0: no early
 * exit inside the loop (reading A22).  gamma in: gamma_0 >= 0 (zero: reading A3),
 * out: solution.  g_out / Fc_out (n x 6) / Uc_out (n x 6) may be NULL. */
int orc_bbpgd(const orc_system* s, const double* q, double tol, int32_t max_iter, int32_t bb_mode,
              int32_t fixed_iters, double* gamma, double* g_out, double* Fc_out, double* Uc_out,
              orc_stats* st);
/* Same algorithm on a dense n x n matrix (row-major), for enumeration tests. */
int orc_bbpgd_dense(int64_t n, const double* M, const double* q, double tol, int32_t max_iter,
                    int32_t bb_mode, double* gamma, double* g_out, orc_stats* st);
/* phi = || min(gamma, g) ||_2. */
double orc_minmap_residual(int64_t n, const double* gamma, const double* g);

/* APGD comparison solver (Mazhar et al. 2015, cited at P:L546-L558; readings A24):
 * gamma_0 = 0; stats->mvops counts every MVOP incl. back-tracking; bb_breakdowns = restarts. */
int orc_apgd(const orc_system* s, const double* q, double tol, int32_t max_iter, double* gamma, double* g_out,
             orc_stats* st);
int orc_apgd_dense(int64_t n, const double* M, const double* q, double tol, int32_t max_iter, double* gamma,
                   double* g_out, orc_stats* st);

/* Explicit Euler update of the configuration, step 4 of the
 * four-step procedure: c' = c + dt U, theta' = normalize(theta + dt Psi(theta) Omega)
 * with Psi = 1/2 [-p^T ; s I - [p]x] for theta = (s, p); rod axes t' = normalize(t + dt Omega x t).
 * UW: n x 6 total velocity (U_nc + U_c).  quat (n x 4, (s, px, py, pz)) and dir (n x 3) may be
 * NULL; updated in place. */
int orc_euler_update(int64_t n, double dt, const double* UW, double* pos, double* quat, double* dir);

#ifdef __cplusplus
}
#endif
#endif
