/* stokescol.h -- C ABI of the B200 collision-resolution library (libstokescol.so).
 *
 * The per-time-step collision solve of Yan et al., "A scalable computational
 * platform for particulate Stokes suspensions" (arXiv 1909.06623), Sec. 3:
 *   LCP   0 <= gamma  _|_  Phi/dt + D^T (U_ext + M D gamma) >= 0
 *   CQP   min 1/2 gamma^T (D^T M D) gamma + q^T gamma,  gamma >= 0
 *   BBPGD Alg. 1
 * with an all-pairs Rotne-Prager-Yamakawa mobility for spheres
 * (BASELINE.json configs[0], [1]) or a block-diagonal slender-body drag for
 * spherocylinders (configs[3]).  "P:Lnnn" = line of /root/reference/PAPER.md.
 *
 * Conventions (all entry points):
 *  - extern "C", no exceptions cross the boundary; every call returns an
 *    sc_status (>= 0 success, < 0 error; sc_last_error() explains).
 *  - Pointers may be HOST or DEVICE memory: the library inspects each with
 *    cudaPointerGetAttributes; host buffers are staged through the context's
 *    stream (synchronously).  Device buffers are used in place.  The caller
 *    owns every buffer it passes; the context owns its internal workspaces.
 *  - All arrays are contiguous, row-major, FP64 unless stated (int32 for
 *    indices).  Per-body 6-vectors are (Fx,Fy,Fz,Tx,Ty,Tz) /
 *    (Ux,Uy,Uz,Wx,Wy,Wz).
 *  - Constraint lists are sorted by (i, j) with i < j in the caller's body
 *    indices.  The unit normal n points from body j to body i; column l of D
 *    carries +n (and r_i x n for rods) on i and -n (and -(r_j x n)) on j
 *    (reading A13).
 *  - Work is ordered on the context's CUDA stream.  Calls that return host
 *    scalars (n_c, stats) synchronise that stream.
 *  - Multi-GPU contexts (sc_create_dist) are collective: every rank makes
 *    the same sequence of calls with the same full inputs; results are
 *    bitwise identical to a 1-GPU context (both RPY
 *    kernels).  The fast summation (mobility model 2) is 1-GPU only.
 */
#ifndef STOKESCOL_H
#define STOKESCOL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct sc_ctx sc_ctx;

typedef enum {
  SC_OK = 0,
  SC_NOT_CONVERGED = 1, /* soft: outputs valid, the last iterate is returned (reading A7) */
  SC_EINVAL = -1,       /* NULL/bad sizes, call out of order */
  SC_EDEGENERATE = -2,  /* coincident centres / zero-length normal (reading A12) */
  SC_ENONFINITE = -3,   /* NaN/Inf met in a gradient or step (SPEC hard error) */
  SC_ENOMEM = -4,
  SC_ECUDA = -5,
  SC_ENCCL = -6
} sc_status;

/* Library version (major*10000 + minor*100 + patch). */
int sc_version(void);
/* Build flags: bit 0 = checked build (device-side bounds asserts, build.py -DSC_CHECKS=1). */
int sc_build_flags(void);

/* ---------------------------------------------------------------- context */
/* One context per GPU.  device: CUDA ordinal.  stream: a cudaStream_t to
 * order all work on, or NULL for a context-owned non-blocking stream. */
int sc_create(sc_ctx** out, int device, void* stream);
/* Multi-GPU (one process per GPU, NCCL over NVLink): nccl_id is the 128-byte
 * ncclUniqueId that rank 0 obtained from sc_nccl_unique_id and broadcast to
 * every rank (e.g. via torch.distributed).  world = 1 builds a one-rank
 * communicator: the context runs the multi-GPU code path (partition, NCCL
 * broadcast / all-reduce) with results bitwise equal to sc_create's. */
int sc_nccl_unique_id(void* out128);
int sc_create_dist(sc_ctx** out, int device, void* stream, const void* nccl_id, int rank, int world);
void sc_destroy(sc_ctx* ctx);
const char* sc_last_error(const sc_ctx* ctx);
/* The stream the context orders its work on (a cudaStream_t). */
void* sc_stream(const sc_ctx* ctx);

/* ------------------------------- NEXT row f2: particle-boundary collisions */
/* Static planar walls ("a vector D_l can be added to D ... with
 * non-zero entries corresponding to the degrees of freedom of the particle
 * only"; a boundary does not appear in the mobility matrix).  Wall k is the
 * plane {x : n_k . x = h_k}, n_k a unit vector pointing into the fluid.
 * walls: HOST array n_walls x 4 = (nx, ny, nz, h); n_walls <= SC_MAX_WALLS
 * (0 removes them).  Applies to every later build_contacts / collision_step /
 * time_step call on this context.  Wall-particle constraint l has
 * cj[l] = n + k (sorted after the particle pairs of body ci[l]), normal n_k
 * (from the wall to the particle), and
 *   spheres: gap = (n_k . c_i - h_k) - a_i, contact iff gap < gap_abs + gap_rel * a_i;
 *   rods:    P = c_i + s t_i, s = -L/2 if n_k.t_i > 0, +L/2 if < 0, 0 if = 0 (the
 *            axis point nearest the wall); gap = (n_k . P - h_k) - b, contact iff
 *            gap < gap_thresh; lever r_i = P - c_i, r_j = 0.
 * Evaluated without FMA contraction (bit-identical to the plain definition).
 * The D column carries +n_k (and r_i x n_k) on body i only; the wall is at rest unless
 * sc_set_wall_velocities gives it a velocity.
 * Errors: SC_EINVAL (n_walls out of range, NULL walls, |n_k| != 1 beyond 1e-12). */
#define SC_MAX_WALLS 8
int sc_set_walls(sc_ctx* ctx, int n_walls, const double* walls);
/* Moving boundaries (a boundary is "any object either static or moving with a
 * prescribed velocity"; reading A28).  vel: HOST array n_walls x 3, the velocity V_k of
 * wall k (n_walls must equal the count of the last sc_set_walls, which resets every V_k to 0).
 * D is unchanged; the wall's motion enters the constant term of the LCP only:
 *   q_l = gap_l/dt + D_l^T U_nc - n_k . V_k  for a particle-wall constraint l with wall k
 * (sc_lcp_q, sc_collision_step, sc_time_step).  sc_time_step then advances each plane with its
 * velocity, h_k <- h_k + dt n_k . V_k (tangential motion leaves the plane in place).
 * Errors: SC_EINVAL (count mismatch, NULL, non-finite). */
int sc_set_wall_velocities(sc_ctx* ctx, int n_walls, const double* vel);
/* The current planes (HOST n_walls x 4 = (nx, ny, nz, h)), e.g. after sc_time_step moved them. */
int sc_get_walls(const sc_ctx* ctx, double* walls);

/* ---------------------------------------------------- (a1) build_contacts */
/* Spheres.  Stores the bodies in the context and computes the near set
 * A(C, delta) = { (i,j) : Phi_ij < delta_ij } with
 *   Phi_ij   = |c_i - c_j| - (a_i + a_j)  (may be negative: overlaps allowed)
 *   delta_ij = gap_abs + gap_rel * min(a_i, a_j)   (reading A1; strict '<').
 * pos: n x 3, radius: n (radius == NULL: all radii = 1).  n_c: out, number of
 * constraints.  The gap and normal are evaluated without FMA contraction so
 * the set and the values are bit-identical to the plain definition (reading
 * A20).  Errors: SC_EINVAL (n < 0, NULL pos, gap_rel < 0), SC_EDEGENERATE
 * (two centres coincide). */
int sc_build_contacts_spheres(sc_ctx* ctx, int64_t n, const double* pos, const double* radius,
                              double gap_abs, double gap_rel, int64_t* n_c);
/* Spherocylinders of radius b: centre, unit axis dir (n x 3), cylinder
 * length (n).  Phi_ij = (minimal distance of the axis segments) - 2b,
 * contact iff Phi_ij < gap_thresh.  Also stores the lever arms
 * r_i = P_i - c_i, r_j = P_j - c_j of the closest points. */
int sc_build_contacts_rods(sc_ctx* ctx, int64_t n, const double* center, const double* dir,
                           const double* length, double b, double gap_thresh, int64_t* n_c);
/* Copy the constraint list out (any pointer may be NULL):
 * ci, cj: n_c int32; gap: n_c; normal: n_c x 3; lever: n_c x 2 x 3 (rods). */
int sc_get_contacts(sc_ctx* ctx, int32_t* ci, int32_t* cj, double* gap, double* normal, double* lever);

/* ------------------------------------------------------- (a2) assemble_D */
/* Builds the column form of D and the body -> constraint
 * incidence (CSR, sorted by constraint id) used by the atomic-free gather
 * F = D gamma, plus the fixed chunking of constraints for deterministic
 * reductions.  Must follow a build_contacts call. */
int sc_assemble_D(sc_ctx* ctx);
/* F = D gamma (gamma: n_c; FT: n x 6). */
int sc_apply_D(sc_ctx* ctx, const double* gamma, double* FT);
/* out = D^T UW (UW: n x 6; out: n_c) -- the linearised gap rate. */
int sc_apply_DT(sc_ctx* ctx, const double* UW, double* out);

/* ---------------------------------------------------- (a4) mobility_apply */
/* UW = Mobility(FT) for the bodies of the last build_contacts call, viscosity mu.
 * Spheres: U_i = F_i/(6 pi mu a_i) + sum_{j != i} T(r_ij; abar) F_j with the RPY
 * tensor of BASELINE.json configs[0] (abar = (a_i+a_j)/2, configs[1]), and
 * W_i = T_i/(8 pi mu a_i^3).  Rods: the 6x6 drag block per body (configs[3]).
 * FT, UW: n x 6. */
int sc_mobility_apply(sc_ctx* ctx, double mu, const double* FT, double* UW);

/* -------------------------------------------------- LCP right-hand side q */
/* q = gap/dt + D^T U_nc.  U_nc: n x 6.  The context keeps q for
 * sc_bbpgd_solve; q_out (n_c) may be NULL. */
int sc_lcp_q(sc_ctx* ctx, double dt, const double* U_nc, double* q_out);

/* ------------------------------- NEXT row f4(ii): the full 6N RPY mobility */
/* model 0 (default): the mobility of BASELINE.json configs[0]/[1] -- translational RPY pair
 * blocks plus the self rotation T/(8 pi mu a^3).  model 1: the full RPY grand mobility, adding
 * the translation-rotation and rotation-rotation pair blocks (reading A27; r = x_i - x_j,
 * rhat = r/|r|, abar = (a_i + a_j)/2):
 *   Omega_i from F_j and U_i from T_j: -c [rhat]x,
 *     c = 1/(8 pi mu r^2) (r >= 2 abar), (1/(16 pi mu abar^2))(r/abar - 3 r^2/(8 abar^2)) (r < 2 abar);
 *   Omega_i from T_j: (1/(16 pi mu r^3))(3 rhat rhat^T - I) (r >= 2 abar),
 *     (1/(8 pi mu abar^3))[(1 - 27r/(32 abar) + 5r^3/(64 abar^3)) I
 *                          + (9r/(32 abar) - 3r^3/(64 abar^3)) rhat rhat^T] (r < 2 abar).
 * Spheres only (rods keep their drag).  With model 1, sc_mobility_apply (hence U_ext in
 * sc_collision_step / sc_time_step) and the U_c output of sc_bbpgd_solve use the full
 * mobility; the LCP iteration itself is unchanged (sphere columns of D carry no torque, so
 * D^T M D only involves the translational blocks).  On a multi-GPU context every rank
 * evaluates all rows of this apply.  Errors: SC_EINVAL for another model. */
int sc_set_mobility_model(sc_ctx* ctx, int model);
/* ---------------------------- NEXT row f4(i): fast O(N) summation of the RPY apply */
/* model 2 (sc_set_mobility_model): the BASELINE RPY mobility (model 0's operator) evaluated by a
 * Chebyshev-interpolation ("black-box") FMM on a uniform octree, the O(N) route the paper takes
 * with KIFMM: far field = the RPY far branch between the Chebyshev nodes of
 * well-separated boxes (n^3 nodes per box, n = order), near field (the 27 leaves around a body,
 * every overlapping pair included) = the exact pair sum.  Approximate: the relative error of the
 * apply falls with the order (measured rel. L2 errors); every sum is in a
 * fixed order (deterministic).  Mono- or polydisperse spheres (polydisperse: the far branch is split
 * into radius-free kernels of the densities F, (a/2) F, (a/2)^2 F, reading A29) on a 1-GPU context
 * (rods keep their drag mobility under every model); used
 * by sc_mobility_apply, sc_lcp_q's U_ext and every BBPGD MVOP.  leaf_level 0 = chosen from N and the
 * order (leaf side >= 2 a_max).  Errors: SC_EINVAL (order not 4/6/8, leaf_level outside 0..8; model 2 on
 * a multi-GPU context, at the first apply). */
int sc_set_fmm_params(sc_ctx* ctx, int order, int leaf_level);
/* The lowest order whose stated relative L2 bar of the apply (2e-3 / 6e-5 / 3e-6 for orders
 * 4 / 6 / 8) meets rel_err, with the automatic leaf level; order_out
 * (nullable) receives it.  Errors: SC_EINVAL (rel_err below 3e-6 or not finite: the direct kernel
 * is the exact operator). */
int sc_set_fmm_tolerance(sc_ctx* ctx, double rel_err, int* order_out);
/* Compressed M2L of the fast summation.  Per level l, the 316 M2L operators
 * K_o (3n^3 x 3n^3: the RPY far branch between the Chebyshev nodes of a box and of the box at
 * offset o) share one orthonormal basis U_l, the dominant eigenvectors of sum_o K_o K_o^T (K_o^T =
 * K_-o, so one basis serves both sides), kept while lambda >= eps^2 lambda_max with eps a fixed
 * fraction of the order's stated error; M2L becomes
 * L = U_l sum_o C_o (U_l^T M), C_o = U_l^T K_o U_l (k_l x k_l).  The bases are computed once per
 * tree geometry (root side, leaf level, order, radius) and cached.  Polydisperse: one basis for the
 * two radius-free parts O and D of the split far branch, four compressed products per offset.
 * mode 0: direct M2L; mode 1: compressed at every order; mode 2 (default): compressed where it
 * measured faster -- monodisperse order 8 from N = 2^15, order 6 from 2^18, order 4 from 2^21;
 * polydisperse order 8
 * from 2^17, order 6 from 2^20 (the root side is then rounded up to 8 a_max 2^(i/8) so the cached
 * bases survive small changes of the bounding box).
 * Errors: SC_EINVAL (mode not 0/1/2). */
int sc_set_fmm_compression(sc_ctx* ctx, int mode);
/* out4 = {mode (0/1/2), compressed M2L active for the current bodies and order (0/1), rank of the
 * cached bases at their leaf level (0: none built yet), that leaf level} */
int sc_get_fmm_compression_info(const sc_ctx* ctx, int32_t* out4);
/* out3 = {order, leaf level of the current tree (0: not built yet), tree built (0/1)} */
int sc_get_fmm_info(const sc_ctx* ctx, int32_t* out3);

/* ------------------------------------------------------- residual (SPEC) */
/* phi = || min(gamma, g) ||_2, the min-map complementarity residual of the LCP (
 * BBPGD's convergence measure).  gamma, g: n_c values (host or device); phi: one double
 * (host or device).  Fixed-order reduction (deterministic).  Errors: SC_EINVAL (NULL, n_c < 0). */
int sc_minmap_residual(sc_ctx* ctx, int64_t n_c, const double* gamma, const double* g, double* phi);

/* ------------------------------------------------------ (a6) bbpgd_solve */
typedef struct {
  double mu;            /* viscosity used by every MVOP */
  double tol;           /* absolute tolerance on phi = ||min(gamma, g)||_2 */
  int32_t max_iter;     /* j_max */
  int32_t bb_mode;      /* 0 = BB1 (paper default), 1 = BB2, 2 = alternate */
  int32_t fixed_iters;  /* 1: run exactly max_iter iterations, no early exit (reading A22) */
  int32_t warm_start;   /* 0: gamma_0 = 0 (reading A3); 1: gamma holds gamma_0 on entry;
                           2: gamma_0 = the previous solve's gamma of the same body pair (i, j),
                              0 for new pairs -- the warm start of a time-stepping run (Step 1,
                              P:L586); needs the same body count, else falls back to 0 */
} sc_bbpgd_opts;

typedef struct {
  int32_t iters;        /* GD steps j taken */
  int32_t mvops;        /* evaluations of M x = 2 + iters, 1 if gamma_0 solves */
  int32_t converged;    /* phi < tol at the returned iterate */
  int32_t bb_breakdowns;/* steps where s^T y <= 0: previous alpha reused (reading A5) */
  int32_t active;       /* |A_c| = #{gamma_l > 0} */
  int32_t reserved;
  double residual;      /* phi at the returned iterate */
  double alpha;         /* last BB step length */
} sc_bbpgd_stats;

/* Solve the CQP for the context's q (from sc_lcp_q).  gamma (n_c): out (in
 * too if warm_start).  g_out (n_c), Fc_out = D gamma (n x 6) and
 * Uc_out = Mobility(Fc) (n x 6) may be NULL.  Returns SC_OK, SC_NOT_CONVERGED
 * or an error; stats may be NULL. */
int sc_bbpgd_solve(sc_ctx* ctx, const sc_bbpgd_opts* opts, double* gamma, double* g_out,
                   double* Fc_out, double* Uc_out, sc_bbpgd_stats* stats);

/* ------------------------------------------------- the whole time-step path */
/* One call = the four steps of P:L480-L489 minus the position update:
 * build_contacts, assemble_D, U_ext = Mobility(F_ext), q, bbpgd_solve.
 * kind 0: spheres (pos, radius, gap_abs, gap_rel); kind 1: rods (pos = centres,
 * dir, length, b, gap_abs = threshold).  F_ext: n x 6.  Fc_out/Uc_out: n x 6,
 * may be NULL.  n_c: out. */
typedef struct {
  int32_t kind;
  int32_t reserved;
  int64_t n;
  const double* pos;
  const double* radius;
  const double* dir;
  const double* length;
  double b;
  double gap_abs, gap_rel;
  double mu, dt;
  const double* F_ext;
} sc_problem;
int sc_collision_step(sc_ctx* ctx, const sc_problem* prob, const sc_bbpgd_opts* opts,
                      double* Fc_out, double* Uc_out, int64_t* n_c, sc_bbpgd_stats* stats);

/* ------------------------------------- NEXT row f3: APGD comparison solver */
/* Accelerated projected gradient descent (Mazhar et al. 2015) on
 * the same CQP and MVOP as sc_bbpgd_solve, for the paper's BBPGD-vs-APGD MVOP
 * comparison.  Uses opts->mu, tol, max_iter (gamma_0 = 0);
 * stats->mvops counts every mobility solve (back-tracking trials included),
 * stats->bb_breakdowns counts gradient restarts.  One GPU (SC_EINVAL on a
 * multi-GPU or emulated context). */
int sc_apgd_solve(sc_ctx* ctx, const sc_bbpgd_opts* opts, double* gamma, double* g_out, sc_bbpgd_stats* stats);

/* --------------------------------------------- NEXT row f1: one time step */
/* The four steps of P:L480-L489: U_nc = Mobility(F_ext), contacts + D, the LCP
 * (BBPGD) -> U_c, and the explicit Euler update of the configuration
 * (P:L465-L470):
 *   c' = c + dt (U_nc + U_c),
 *   theta' = normalize(theta + dt Psi(theta) Omega), Psi = 1/2 [-p^T ; s I - [p]x],
 *   rods: t' = normalize(t + dt Omega x t).
 * pos_out: n x 3 (required); dir_out: n x 3 (rods, required for rods);
 * quat: n x 4 quaternions (s, px, py, pz) updated in place (may be NULL);
 * U_out: n x 6 total velocity U_nc + U_c (may be NULL).  Returns like
 * sc_bbpgd_solve (SC_NOT_CONVERGED still updates the configuration). */
int sc_time_step(sc_ctx* ctx, const sc_problem* prob, const sc_bbpgd_opts* opts, double* pos_out, double* dir_out,
                 double* quat, double* U_out, int64_t* n_c, sc_bbpgd_stats* stats);

/* ----------------------------------------------------------- measurement */
/* Kernel families for timing/launch accounting. */
enum {
  SC_K_CONTACTS = 0, SC_K_ASSEMBLE = 1, SC_K_GATHER = 2, SC_K_RPY = 3, SC_K_COMBINE = 4,
  SC_K_DT = 5, SC_K_FINALIZE = 6, SC_K_MISC = 7, SC_K_COUNT = 8
};
/* enable != 0: bracket every launch with CUDA events on the context stream. */
int sc_set_timing(sc_ctx* ctx, int enable);
/* Sum of event-timed launch durations (ms) and launch count for a family
 * since the last reset (synchronises the stream). */
int sc_get_timing(sc_ctx* ctx, int family, double* total_ms, int64_t* launches);
int sc_reset_timing(sc_ctx* ctx);
/* Total number of kernels this context launched since creation. */
int64_t sc_launch_count(const sc_ctx* ctx);

/* Residual trace of the next solves (Alg. 1 Steps 3 and 11): with capacity > 0
 * every sc_bbpgd_solve records phi_0 (the residual at gamma_0) and phi_j after each GD step j,
 * up to `capacity` values, in a context-owned device buffer (one store per iteration; no host
 * synchronisation).  capacity = 0 turns it off.  Errors: SC_EINVAL (capacity < 0). */
int sc_set_residual_trace(sc_ctx* ctx, int32_t capacity);
/* Copy the trace of the last solve: *count = number of values recorded (min(capacity set,
 * iterations + 1)); the first min(capacity, *count) go to out (host or device).  Synchronises.
 * Errors: SC_EINVAL (NULL count, capacity < 0, NULL out with capacity > 0). */
int sc_get_residual_trace(sc_ctx* ctx, double* out, int32_t capacity, int32_t* count);
/* Communicator of the context: out4 = {nranks, rank, CUDA device, NCCL version code}; a 1-GPU
 * context reports {1, 0, device, version}.  Errors: SC_EINVAL (NULL), SC_ENCCL. */
int sc_comm_info(const sc_ctx* ctx, int32_t* out4);

/* Host-only helper (no GPU needed): the row/chunk partition a world-sized
 * context uses for n bodies.  out7 = {npad,
 * rows_per_rank, row_lo, row_hi, chunk_lo, chunk_hi, nsplit}: rank owns RPY
 * target rows [row_lo, row_hi) and the constraints whose first body lies there
 * (the paper's smaller-index rule); chunk c = bodies
 * [256c, 256c+256). */
int sc_plan_partition(int64_t n, int world, int rank, int64_t* out7);

/* Host-only helper (no GPU needed): the super-block pairs (SI, SJ) of the symmetric RPY kernel
 * that rank `rank` of `world` evaluates for nsb super-blocks of 512 bodies (DESIGN.md "K-RPY":
 * super-block S takes (S, S) and (S, S + d mod nsb) for d = 1 .. (nsb-1)/2, plus d = nsb/2 when
 * nsb is even and S < nsb/2; rank r takes the contiguous super-block range [r s, (r+1) s),
 * s = ceil(nsb/world)).  pairs: 2 x count int32 (may be NULL to query count).  Rows of SI receive
 * the sources of SJ ("forward") and, for SI != SJ, rows of SJ the sources of SI ("reverse").
 * Errors: SC_EINVAL. */
int sc_sym_pair_table(int64_t nsb, int world, int rank, int32_t* pairs, int64_t* count);

/* Testing hook: make a 1-GPU context run the multi-GPU decomposition of `world`
 * ranks (every rank's share of every step in turn, on this GPU).  The NCCL
 * collectives become their shared-memory equivalents (broadcast and all-gather
 * are in place already; the all-reduce of the zero-padded chunk partials is a
 * copy), so results must be bitwise identical to world = 1.  world = 1 turns it
 * off.  Errors: SC_EINVAL on a multi-GPU context or world < 1. */
int sc_set_emulated_world(sc_ctx* ctx, int world);

/* Choice of the RPY apply kernel: 0 = automatic (the
 * symmetric pair-tile kernel for N >= 4096 -- on one GPU and on a multi-GPU
 * context, where every rank evaluates its share of the super-block pairs and the
 * exact fixed-point row sums are all-reduced as int64 -- else the target-row
 * kernel), 1 = target-row kernel (rows sharded over the ranks), 2 = symmetric
 * pair-tile kernel (each unordered pair evaluated once).  Both kernels give
 * results that are bitwise independent of the number of ranks; they differ from
 * each other in rounding only.  Mode 0 on one GPU also runs the BBPGD loop of small
 * sphere problems (padded N <= 2048) as one persistent cooperative kernel
 * (DESIGN.md); modes 1 and 2 keep the kernel-per-step path.  Errors: SC_EINVAL for
 * another mode. */
int sc_set_rpy_kernel(sc_ctx* ctx, int mode);

#ifdef __cplusplus
}
#endif
#endif /* STOKESCOL_H */
