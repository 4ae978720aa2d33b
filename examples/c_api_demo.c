/* c_api_demo.c -- the C ABI used from plain C (no Python, no torch): a small suspension of
 * spheres pushed together, one collision-resolution solve with HOST buffers
 * (sc_collision_step stages them), then the stats and a check of the solution.
 *
 *   gcc -O2 -I include examples/c_api_demo.c -L paper_1909_06623_b200 -lstokescol \
 *       -Wl,-rpath,paper_1909_06623_b200 -lm -o examples/c_api_demo && ./examples/c_api_demo
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "stokescol.h"

#define CHECK(call)                                                                   \
  do {                                                                                \
    int rc_ = (call);                                                                 \
    if (rc_ < 0) {                                                                    \
      fprintf(stderr, "%s failed: %d (%s)\n", #call, rc_, sc_last_error(ctx));        \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

int main(void) {
  /* a 8 x 8 x 8 lattice of unit spheres, spacing 2.05 (gap 0.05 < 0.1 a: every neighbour pair
   * is a constraint), every sphere pushed towards the lattice centre */
  const int m = 8;
  const int64_t n = (int64_t)m * m * m;
  double* pos = (double*)malloc(sizeof(double) * 3 * n);
  double* F = (double*)calloc(6 * n, sizeof(double));
  double* Fc = (double*)malloc(sizeof(double) * 6 * n);
  double* Uc = (double*)malloc(sizeof(double) * 6 * n);
  const double h = 2.05, c = 0.5 * (m - 1) * h;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j)
      for (int k = 0; k < m; ++k) {
        const int64_t b = ((int64_t)i * m + j) * m + k;
        pos[3 * b] = i * h;
        pos[3 * b + 1] = j * h;
        pos[3 * b + 2] = k * h;
        F[6 * b] = -(pos[3 * b] - c);
        F[6 * b + 1] = -(pos[3 * b + 1] - c);
        F[6 * b + 2] = -(pos[3 * b + 2] - c);
      }
  sc_ctx* ctx = NULL;
  if (sc_create(&ctx, 0, NULL) != SC_OK) {
    fprintf(stderr, "sc_create failed (no GPU?)\n");
    return 2;
  }
  sc_problem prob = {0};
  prob.kind = 0;
  prob.n = n;
  prob.pos = pos;
  prob.radius = NULL; /* all radii 1 */
  prob.gap_abs = 0.0;
  prob.gap_rel = 0.1;
  prob.mu = 1.0;
  prob.dt = 0.01;
  prob.F_ext = F;
  sc_bbpgd_opts opts = {0};
  opts.mu = 1.0;
  opts.tol = 1e-8;
  opts.max_iter = 2000;
  int64_t nc = 0;
  sc_bbpgd_stats st;
  CHECK(sc_collision_step(ctx, &prob, &opts, Fc, Uc, &nc, &st));
  /* contact forces are internal: they sum to zero (Newton's third law) */
  double sx = 0, sy = 0, sz = 0, fmax = 0;
  for (int64_t b = 0; b < n; ++b) {
    sx += Fc[6 * b];
    sy += Fc[6 * b + 1];
    sz += Fc[6 * b + 2];
    fmax = fmax > fabs(Fc[6 * b]) ? fmax : fabs(Fc[6 * b]);
  }
  printf("n = %lld, n_c = %lld, iterations = %d, MVOPs = %d, residual = %.3e, converged = %d, active = %d\n",
         (long long)n, (long long)nc, st.iters, st.mvops, st.residual, st.converged, st.active);
  printf("sum of contact forces = (%.2e, %.2e, %.2e), max |F_c,x| = %.3f\n", sx, sy, sz, fmax);
  const int ok = st.converged == 1 && nc == 3 * (int64_t)m * m * (m - 1) &&
                 fabs(sx) + fabs(sy) + fabs(sz) < 1e-9 * (1 + fmax);
  sc_destroy(ctx);
  free(pos); free(F); free(Fc); free(Uc);
  printf(ok ? "c_api_demo: ok\n" : "c_api_demo: FAILED\n");
  return ok ? 0 : 1;
}
