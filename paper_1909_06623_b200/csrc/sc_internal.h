// sc_internal.h -- internal declarations of libstokescol (B200, sm_100a, FP64).
// Not part of the C ABI (see include/stokescol.h).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <functional>
#include <string>
#include <vector>

#include "stokescol.h"

// Checked build (-DSC_CHECKS=1, build.py): device-side bounds asserts on the indexed accesses of the
// hot kernels (compute-sanitizer is not available on this pool; tests run against this build too).
#ifndef SC_CHECKS
#define SC_CHECKS 0
#endif
#if SC_CHECKS
#include <cassert>
#define SC_DCHECK(cond) assert(cond)
#else
#define SC_DCHECK(cond) ((void)0)
#endif

namespace sc {

constexpr int kRpyThreads = 64;         // threads per RPY CTA
constexpr int kRpyTpt = 4;              // targets per thread
constexpr int kRpySu = 2;               // sources interleaved per step (ILP: TPT*SU pair chains)
constexpr int kRpyRows = kRpyThreads * kRpyTpt;  // 256 target rows per CTA
constexpr int kRpyTile = 128;           // sources per shared-memory tile
constexpr int kNpadQuantum = 512;       // npad = N rounded up to this (RPY row blocks and super-blocks)
constexpr int kChunkBodies = 256;       // B_c: bodies per reduction chunk
constexpr int kPartials = 4;            // doubles per chunk partial
constexpr int kPersistMaxBodies = 2048; // persistent single-launch BBPGD loop up to this npad (persist.cu)

enum BodyKind { kNone = -1, kSpheres = 0, kRods = 1 };

// Device-side solver scalars (one struct in device memory; mirrored to pinned host).
struct DevScalars {
  double alpha;      // current BB step alpha_{j}
  double phi;        // last residual
  double p[4];       // last reduced partials
  double tol;
  int32_t iter;      // GD steps done
  int32_t done;      // 1: stop (converged, j_max or error)
  int32_t conv;      // phi < tol at the last evaluation
  int32_t breakdowns;
  int32_t nonfinite;
  int32_t max_iter;
  int32_t bb_mode;
  int32_t fixed;
  int32_t err;       // contact degeneracy etc.
  int32_t trace_cap; // residual trace: phi_0, phi_1, ... of the solve (sc_set_residual_trace)
  double* trace;     // device buffer of trace_cap doubles (NULL: off)
};

struct KernelTimer {
  bool enabled = false;
  std::vector<cudaEvent_t> ev[SC_K_COUNT];  // pairs (start, stop)
  double total_ms[SC_K_COUNT] = {};
  int64_t launches[SC_K_COUNT] = {};
  std::vector<cudaEvent_t> pool;
};

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;  // capacity in elements
};

}  // namespace sc

struct sc_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  int64_t launch_count = 0;
  sc::KernelTimer timer;

  // multi-GPU
  int rank = 0, world = 1;
  int emul_world = 1;           // testing: run the multi-GPU decomposition of this many ranks on one GPU
  ncclComm_t comm = nullptr;

  // bodies
  int kind = sc::kNone;
  int64_t n = 0, npad = 0;      // npad: multiple of kRpyRows * world
  int poly = 0;                 // spheres: radii not all equal
  double a_const = 1.0;
  double rod_b = 0.5;
  int nwalls = 0;               // NEXT row f2: static planar walls (sc_set_walls)
  double4 walls[SC_MAX_WALLS] = {};  // (nx, ny, nz, h): plane n.x = h, unit n into the fluid
  double wall_vel[SC_MAX_WALLS][3] = {};  // prescribed wall velocities V_k (moving boundaries)
  sc::DBuf<double4> pos4;       // spheres: (x,y,z,a/2); rods: (x,y,z,L)
  sc::DBuf<double4> dir4;       // rods: (tx,ty,tz,0)
  sc::DBuf<double4> rodmob4;    // rods: (1/zeta_par, 1/zeta_perp, 1/zeta_rot, mu) for rod_mu
  double rod_mu = -1.0;

  // contacts (sorted by (i,j))
  int64_t nc = 0;
  sc::DBuf<int32_t> ci, cj;
  sc::DBuf<double4> nrm4;       // (nx,ny,nz,gap)
  sc::DBuf<double4> lev4;       // rods: [2*l] = r_i, [2*l+1] = r_j (w = 0)
  sc::DBuf<double4> rxn4;       // rods: [2*l] = r_i x n, [2*l+1] = r_j x n
  bool assembled = false;
  sc::DBuf<int32_t> row_ptr;    // n+1
  sc::DBuf<int32_t> inc;        // 2*nc: (l << 1) | side
  sc::DBuf<double4> icol4;      // signed D columns per incidence (spheres: 1 double4; rods: 3 double2)
  sc::DBuf<int2> einc;          // rods: incidence positions (e_i, e_j) of constraint l (e_j = -1: wall)
  sc::DBuf<double> hinc;        // rods: h_e = (signed column of e) . (U, W) of its body, per incidence
  sc::DBuf<int32_t> first_ptr;  // n+1: constraints with first body < b start at first_ptr[b]
  sc::DBuf<int32_t> near_ptr, near_idx;  // spheres: RPY overlap-branch partners per body (CSR)
  int64_t nchunks = 0;
  std::vector<int32_t> h_first_ptr;  // host copy (chunk bounds, ownership)

  // LCP state
  bool have_q = false;
  sc::DBuf<double> q;
  sc::DBuf<double> gam[2], g[2], w, gam_user, uc;  // w: U_ext (n x 6); uc: U_c for time stepping
  sc::DBuf<double2> st[2];      // BBPGD state (gamma_l, g_l), ping-pong
  sc::DBuf<double> apgd_y, apgd_sums;  // APGD: extrapolated point, reduced sums
  sc::DBuf<int64_t> prev_key;   // warm start: (i*n + j) keys of the previous solve (sorted)
  sc::DBuf<double> prev_gam;    // ... and its gamma
  int64_t prev_nc = 0, prev_n = -1;
  sc::DBuf<double> chunk_part;  // nchunks * 4
  sc::DBuf<double> chunk_red;   // reduced (allreduce output)
  sc::DBuf<double4> f4;         // sources: (Fx,Fy,Fz,0) [npad]
  sc::DBuf<double4> t4;         // torques for the public mobility apply [npad]
  sc::DBuf<double4> u4;         // velocities (Ux,Uy,Uz,0) [npad] (spheres) or [2*npad] (rods: U, W)
  sc::DBuf<double> rpy_part;    // nsplit * rows * 3
  int mobility_model = 0;       // 0: BASELINE RPY (tt + self rotation); 1: full 6N RPY (NEXT row f4(ii));
                                // 2: BASELINE RPY by the fast summation (NEXT row f4(i), fmm.cu)
  // fast RPY summation (fmm.cu): Chebyshev order, leaf level (0: automatic), the tree of the bodies
  int fmm_order = 6, fmm_leaf_level = 0, fmm_L_used = 0, fmm_poly = 0;
  int64_t fmm_maxleaf = 0;      // bodies in the fullest leaf
  bool fmm_ready = false;       // tree built for the current bodies
  double fmm_geom[4] = {};      // root cube corner (x, y, z) and side
  sc::DBuf<uint32_t> fmm_key;
  sc::DBuf<int32_t> fmm_idx0, fmm_sidx, fmm_cnt, fmm_lstart;
  sc::DBuf<char> fmm_cubtmp;
  sc::DBuf<double4> fmm_spos4, fmm_sf4;
  sc::DBuf<double> fmm_M, fmm_L;
  sc::DBuf<long long> fmm_acc;              // symmetric near field: fixed-point limbs, 9 per (sorted) body
  sc::DBuf<unsigned long long> fmm_fx;      // ... and its scale block (FxScale)
  std::vector<int64_t> fmm_lev_off;
  sc::DBuf<int64_t> fmm_lev_off_dev;
  // compressed M2L (sc_set_fmm_compression): per level l the basis U_l (3n^3 x k_l) of the M2L
  // operators and the 316 compressed operators C_o = U^T K_o U (k_l x k_l), cached for a geometry key
  int fmm_compress = 2;           // 0 off, 1 on, 2 auto (orders 6 and 8)
  double fmm_svd_key[5] = {};     // (root side, leaf level, order, a, valid)
  std::vector<int> fmm_svd_k;     // k_l per level (index l)
  std::vector<int64_t> fmm_svd_uoff, fmm_svd_coff;  // offsets of U_l, C_l in the buffers below
  sc::DBuf<double> fmm_svd_U, fmm_svd_C, fmm_Mc, fmm_Lc, fmm_svd_work;
  sc::DBuf<int32_t> fmm_svd_li;   // offset index (7^3 grid) -> operator index (-1: adjacent)
  std::vector<int32_t> fmm_svd_lih;  // (host copy)
  sc::DBuf<uint64_t> fmm_svd_ptrs;   // batched-GEMM pointer tables
  void* cublas = nullptr;         // cublasHandle_t / cusolverDnHandle_t (fmm.cu)
  void* cusolver = nullptr;
  sc::DBuf<double> rpy6_part;   // full RPY: nsplit * npad * 6 partials
  sc::DBuf<double> ft_tmp;      // n x 6 scratch (F_c for the full-RPY U_c)
  int nsplit = 1;
  int rpy_mode = 0;             // 0 auto, 1 target-row kernel, 2 symmetric pair-tile kernel
  bool use_persist = true;      // persistent BBPGD loop for small sphere problems (env SC_NO_PERSIST=1: off)
  int batch_override = 0;       // tuning: iterations enqueued between host reads (env SC_BATCH)
  bool use_graphs = true;       // CUDA-graph replay of small-problem iteration batches (env SC_NO_GRAPHS=1: off)
  int sym_variant = 0;          // tuning: (warps, targets/lane) of the symmetric kernel (env SC_SYM_VARIANT)
  int sym_hs = 0;
  int persist_grid_cap = 0;     // tuning: CTAs of the persistent loop (env SC_PERSIST_GRID; 0 = one per SM)               // tuning: source parts per super-block pair (env SC_SYM_HS; 0 = cost model)
  int64_t sym_nsb = -1;         // super-blocks the pair tables were built for
  int sym_world = -1;           // ... and the number of ranks
  sc::DBuf<int2> sym_pairs;     // (SI, SJ) of every rank, concatenated (cyclic-half assignment)
  std::vector<int64_t> sym_off; // rank r's pairs: [sym_off[r], sym_off[r+1])
  sc::DBuf<long long> sym_acc;  // symmetric kernel: fixed-point limbs [npad][3 comps][3 limbs] (rpy.cu)
  sc::DBuf<unsigned long long> fx_scale;  // ... and its per-apply scale (FxScale)
  bool sym_acc_dirty = true;    // limbs not known to be zero (first use / interrupted apply)
  sc::DBuf<double> trace;          // residual trace (phi per iteration) of the last solve
  int32_t trace_cap = 0, trace_count = 0;
  // per-device setup, done in sc_create on this context's device (kernel attributes, sizes)
  size_t total_mem = 0;            // device memory (bytes)
  int num_sms = 0;
  int persist_grid = 0;            // persistent BBPGD kernel: CTAs (one per SM; 0 = not resident)
  sc::DevScalars* dsc = nullptr;   // device scalars
  sc::DevScalars* hsc = nullptr;   // pinned mirror
  int32_t* derr = nullptr;         // device error flag
  unsigned int* dcount = nullptr;  // last-CTA counter of the fused D^T + finalize
  int32_t* herr = nullptr;         // pinned mirror

  // scratch for contacts
  sc::DBuf<double> bbox_part;
  sc::DBuf<int32_t> cell_of, cell_cnt, cell_start, sorted_idx, pair_cnt, pair_off, scan_tmp;
  sc::DBuf<double4> sorted4, sorted_dir4;

  // staging for host pointers: a pool of device buffers kept across calls (a cudaMalloc /
  // cudaFree pair per staged array per call measured 0.1-0.7 s of stalls on the e2e path)
  sc::DBuf<char> stage;
  std::vector<sc::DBuf<char>> stage_pool;
  std::vector<bool> stage_busy;
};

namespace sc {

// ---- error helpers -------------------------------------------------------
int fail(sc_ctx* c, int code, const std::string& msg);
int cuda_fail(sc_ctx* c, cudaError_t e, const char* what);
#define SC_CUDA(call)                                        \
  do {                                                       \
    cudaError_t e_ = (call);                                 \
    if (e_ != cudaSuccess) return sc::cuda_fail(ctx, e_, #call); \
  } while (0)

template <typename T>
int ensure(sc_ctx* ctx, DBuf<T>& b, size_t n) {
  if (b.n >= n && b.p) return 0;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.n = 0;
  size_t want = n > 0 ? n : 1;
  cudaError_t e = cudaMalloc(&b.p, want * sizeof(T));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaMalloc");
  b.n = want;
  return 0;
}
template <typename T>
void release(DBuf<T>& b) {
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.n = 0;
}

// ---- launch accounting ---------------------------------------------------
void timer_begin(sc_ctx* ctx, int family);
void timer_end(sc_ctx* ctx, int family);
int check_launch(sc_ctx* ctx, const char* what);

// ---- scans (scan.cu) -------------------------------------------------------
// exclusive scan of n int32 into out (out[n] = total); tmp sized by scan_tmp_size(n).
size_t scan_tmp_size(int64_t n);
int exclusive_scan_i32(sc_ctx* ctx, const int32_t* in, int32_t* out, int64_t n, int32_t* tmp);

// ---- contacts (contacts.cu) ----------------------------------------------
int build_contacts_spheres(sc_ctx* ctx, double gap_abs, double gap_rel);
int build_contacts_rods(sc_ctx* ctx, double gap_thresh);

// ---- assemble (assemble.cu) ----------------------------------------------
int assemble(sc_ctx* ctx);

// ---- mobility (rpy.cu) ----------------------------------------------------
// U4[rows row0 .. row0+nrows) = scale * sum_j T_ij f4_j (+ self), from packed
// sources f4 [npad]; nrows multiple of kRpyRows.  done: optional device flag.
int rpy_apply_rows(sc_ctx* ctx, const double4* f4, int64_t row0, int64_t nrows, double mu,
                   double4* u4, const int32_t* done);
int choose_nsplit(int64_t npad, int world);
// NEXT row f4(i): u4 = RPY(f4) by the Chebyshev-interpolation FMM (builds the tree on first use)
int fmm_init_device(sc_ctx* ctx);  // interpolation tables into constant memory (sc_create)
int fmm_setup(sc_ctx* ctx);
int fmm_apply(sc_ctx* ctx, const double4* f4, double mu, double4* u4, const int32_t* done);
void fmm_destroy_handles(sc_ctx* ctx);
bool fmm_uses_library_calls(const sc_ctx* ctx);  // the compressed M2L (cuBLAS) is active
// per-device kernel attributes (max dynamic shared memory); called by sc_create
int rpy_init_device(sc_ctx* ctx);
int persist_init_device(sc_ctx* ctx);
// NEXT row f4(ii): UW (n x 6, device) = full 6N RPY grand mobility of the packed (f4, t4).
int rpy6_apply(sc_ctx* ctx, const double4* f4, const double4* t4, double mu, double* UW);
bool rpy_use_sym(const sc_ctx* ctx);
int rpy_apply_sym(sc_ctx* ctx, const double4* f4, double mu, double4* u4, const int32_t* done, int W,
                  const std::vector<int>& ranks, int mode, const std::function<int()>& reduce);

// ---- LCP kernels (lcp.cu) -------------------------------------------------
// gather F = D v (mode raw) or F = D max(0, gam_old - alpha g_old) with the owner
// writing gam_new (mode proj).  Output: f4 (spheres) or u4 after the drag (rods, fused)
// or a user FT (n x 6).
// The BBPGD state is packed per constraint: st[k][l] = (gamma_l, g_l), ping-pong k = 0, 1.
int launch_gather_proj(sc_ctx* ctx, int pp, double mu);  // st[pp] -> st[pp ^ 1].x, F
// gated: skip when the solve's done flag is set (inside the BBPGD loop); false after the loop
int launch_gather_raw(sc_ctx* ctx, const double* v, int vstride, double mu, double* FT_user /*nullable*/,
                      bool gated = true);
int launch_proj_own(sc_ctx* ctx, int pp, int64_t l0, int64_t l1);
int launch_pack_gamma0(sc_ctx* ctx, const double* gam0);  // st[0] = (max(0, gamma_0), 0)
int launch_unpack_state(sc_ctx* ctx, int pp, double* gam, double* g);
// D^T: mode 0 iteration (g_new = D^T U + q, partials ss,sy,yy,mm), mode 1 alpha0
// (partials g.g, g.M g), mode 2 warm g_0 = D^T U + q, mode 5 g_0 = q (both: partial mm) -- on the
// packed state st[pp]; APGD: mode 3 (g_out = q), mode 4 (g_out = M x + q; x.Mx, q.x, mm); chunks [c0,c1)
int launch_dt(sc_ctx* ctx, int mode, int pp, const double* x, double* g_out, int64_t c0, int64_t c1, bool fuse);
int launch_dt_user(sc_ctx* ctx, const double* UW, double* out, const double* addq, double qscale);
// q = gap/dt + D^T U_nc - n_k . V_k on the constraints with moving walls
int launch_lcp_q(sc_ctx* ctx, const double* U_nc, double inv_dt, double* q);
int launch_finalize(sc_ctx* ctx, int mode, const double* part);
int launch_init_g0(sc_ctx* ctx, const double* q, double* g0, int64_t c0, int64_t c1);
int launch_pack_ft(sc_ctx* ctx, const double* FT, double4* f4, double4* t4);
int launch_unpack_uw_spheres(sc_ctx* ctx, const double4* u4, const double4* t4, double mu, double* UW);
int launch_rod_drag_user(sc_ctx* ctx, const double* FT, double mu, double* UW);
int launch_rod_unpack(sc_ctx* ctx, const double4* u4, double* UW);
int launch_count_active(sc_ctx* ctx, const double* gam, int32_t* out);
int launch_loop_continue(sc_ctx* ctx, cudaGraphConditionalHandle cond);  // device loop condition = !done
int launch_minmap(sc_ctx* ctx, const double* gam, const double* g, int64_t nc, double* out);
int launch_q(sc_ctx* ctx, double dt, const double* dtu, double* q);
struct WallRates {
  double r[SC_MAX_WALLS];  // n_k . V_k of each wall (moving boundaries; 0: static)
};

// ---- persistent small-problem BBPGD loop (persist.cu) ------------------------
bool persist_eligible(const sc_ctx* ctx);
int bbpgd_persistent(sc_ctx* ctx, double mu);

// ---- APGD comparison solver (apgd.cu) --------------------------------------
int apgd_launch_step(sc_ctx* ctx, const double* y, const double* g, const double* gam, double t, double* gam_new);
int apgd_launch_momentum(sc_ctx* ctx, const double* gam_new, const double* gam, double beta, double* y);
int launch_sum_chunks(sc_ctx* ctx, double* out4);

}  // namespace sc
