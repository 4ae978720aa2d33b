// api.cu -- the C ABI (include/stokescol.h): context, staging, NCCL, and the
// BBPGD control loop (Alg. 1) around the device kernels.
//
// The loop runs on the device: one CUDA graph whose conditional WHILE node repeats the
// two-iteration kernel sequence until K-FINALIZE sets the device flag `done` (convergence, j_max
// or a non-finite value); every kernel of an iteration starts by reading `done` and returns at
// once if it is set.  The host reads the solver scalars (one pinned copy) after the loop.
// (Multi-GPU and timed runs: iterations enqueued from the host in batches, scalars read between.)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "sc_internal.h"

namespace sc {

int fail(sc_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}
int cuda_fail(sc_ctx* c, cudaError_t e, const char* what) {
  return fail(c, SC_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

static cudaEvent_t pool_get(sc_ctx* ctx) {
  auto& p = ctx->timer.pool;
  if (!p.empty()) {
    cudaEvent_t e = p.back();
    p.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void timer_begin(sc_ctx* ctx, int family) {
  if (!ctx->timer.enabled) return;
  cudaEvent_t e = pool_get(ctx);
  cudaEventRecord(e, ctx->stream);
  ctx->timer.ev[family].push_back(e);
}
void timer_end(sc_ctx* ctx, int family) {
  if (!ctx->timer.enabled) return;
  cudaEvent_t e = pool_get(ctx);
  cudaEventRecord(e, ctx->stream);
  ctx->timer.ev[family].push_back(e);
}

int check_launch(sc_ctx* ctx, const char* what) {
  ctx->launch_count += 1;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, what);
  return 0;
}

static void timer_collect(sc_ctx* ctx) {
  cudaStreamSynchronize(ctx->stream);
  for (int f = 0; f < SC_K_COUNT; ++f) {
    auto& v = ctx->timer.ev[f];
    for (size_t k = 0; k + 1 < v.size(); k += 2) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, v[k], v[k + 1]) == cudaSuccess) ctx->timer.total_ms[f] += ms;
      ctx->timer.launches[f] += 1;
    }
    for (auto e : v) ctx->timer.pool.push_back(e);
    v.clear();
  }
}

// ------------------------------------------------------------ staging
static bool is_device_ptr(const void* p) {
  if (p == nullptr) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

struct Stager {
  sc_ctx* ctx;
  std::vector<size_t> slots;  // pool buffers this call holds
  struct Pending {
    void* host;
    const void* dev;
    size_t bytes;
  };
  std::vector<Pending> outs;
  bool staged_in = false;  // a host input was copied: finish() waits for it (the caller may reuse it)
  explicit Stager(sc_ctx* c) : ctx(c) {}
  ~Stager() {
    for (size_t k : slots) ctx->stage_busy[k] = false;
  }
  // a free pool buffer of at least `bytes` (grown in place if needed; never freed per call)
  int acquire(size_t bytes, char** p) {
    size_t k = 0;
    while (k < ctx->stage_pool.size() && ctx->stage_busy[k]) ++k;
    if (k == ctx->stage_pool.size()) {
      ctx->stage_pool.emplace_back();
      ctx->stage_busy.push_back(false);
    }
    if (int rc = ensure(ctx, ctx->stage_pool[k], bytes)) return rc;
    ctx->stage_busy[k] = true;
    slots.push_back(k);
    *p = ctx->stage_pool[k].p;
    return 0;
  }
  // device view of an input (copied if host)
  template <typename T>
  int in(const T* p, size_t count, const T** out) {
    if (p == nullptr || count == 0 || is_device_ptr(p)) {
      *out = p;
      return 0;
    }
    char* b = nullptr;
    if (int rc = acquire(count * sizeof(T), &b)) return rc;
    cudaError_t e = cudaMemcpyAsync(b, p, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "stage in");
    staged_in = true;
    *out = reinterpret_cast<const T*>(b);
    return 0;
  }
  template <typename T>
  int out(T* p, size_t count, T** o) {
    if (p == nullptr || count == 0 || is_device_ptr(p)) {
      *o = p;
      return 0;
    }
    char* b = nullptr;
    if (int rc = acquire(count * sizeof(T), &b)) return rc;
    *o = reinterpret_cast<T*>(b);
    outs.push_back({p, b, count * sizeof(T)});
    return 0;
  }
  // in + out (read-modify-write)
  template <typename T>
  int inout(T* p, size_t count, T** o) {
    if (int rc = out(p, count, o)) return rc;
    if (*o != p) {
      cudaError_t e = cudaMemcpyAsync(*o, p, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "stage inout");
      staged_in = true;
    }
    return 0;
  }
  int finish() {
    for (auto& o : outs) {
      cudaError_t e = cudaMemcpyAsync(o.host, o.dev, o.bytes, cudaMemcpyDeviceToHost, ctx->stream);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "stage out");
    }
    if (!outs.empty() || staged_in) {  // host staging is synchronous (include/stokescol.h)
      cudaError_t e = cudaStreamSynchronize(ctx->stream);
      if (e != cudaSuccess) return cuda_fail(ctx, e, "stage sync");
    }
    outs.clear();
    staged_in = false;
    return 0;
  }
};

// ------------------------------------------------------------ partition
struct Part {
  int64_t rpr = 0;             // rows per rank (multiple of 256)
  int64_t row_lo = 0, row_hi = 0;  // own rows, clipped to npad
  int64_t c0 = 0, c1 = 0;      // own chunks
  int64_t l0 = 0, l1 = 0;      // own constraints
  std::vector<int64_t> loff, lcnt;  // constraint slices of every rank
};

static void plan_rows(int64_t npad, int world, int rank, int64_t* rpr, int64_t* lo, int64_t* hi) {
  const int64_t B = npad / kRpyRows;
  const int64_t bpr = (B + world - 1) / world;
  *rpr = bpr * kRpyRows;
  *lo = std::min(npad, rank * *rpr);
  *hi = std::min(npad, (rank + 1) * *rpr);
}

static Part partition(const sc_ctx* ctx, int world, int rank) {
  Part p;
  const int64_t n = ctx->n;
  auto fp = [&](int64_t b) -> int64_t { return ctx->h_first_ptr[std::min(b, n)]; };
  plan_rows(ctx->npad, world, rank, &p.rpr, &p.row_lo, &p.row_hi);
  p.c0 = p.row_lo / kChunkBodies;
  p.c1 = p.row_hi / kChunkBodies;
  p.l0 = fp(p.row_lo);
  p.l1 = fp(p.row_hi);
  for (int r = 0; r < world; ++r) {
    int64_t rpr, lo, hi;
    plan_rows(ctx->npad, world, r, &rpr, &lo, &hi);
    p.loff.push_back(fp(lo));
    p.lcnt.push_back(fp(hi) - fp(lo));
  }
  return p;
}

#define NCCL_CHECK(call)                                                                        \
  do {                                                                                          \
    ncclResult_t r_ = (call);                                                                   \
    if (r_ != ncclSuccess) return fail(ctx, SC_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

// The multi-GPU decomposition.  With world > 1 (NCCL) this
// process runs its own rank's share and the collectives move data between GPUs.  With an
// emulated world (sc_set_emulated_world, one GPU) this process runs every rank's share in
// turn on shared buffers; the collectives become what they amount to on shared memory:
// broadcast/all-gather are no-ops (every slice is already in place) and the all-reduce of
// the zero-padded chunk partials is a copy.  No kernel ever waits on another.
struct Dist {
  sc_ctx* ctx = nullptr;
  bool on = false, emul = false;
  int W = 1;
  std::vector<Part> parts;
  std::vector<int> mine;  // ranks computed by this process

  explicit Dist(sc_ctx* c) : ctx(c) {
    const int ew = c->emul_world;
    emul = c->world == 1 && ew > 1 && c->comm == nullptr;
    W = emul ? ew : c->world;
    // a context with a communicator runs the NCCL path even with one rank (sc_create_dist, world 1)
    on = (W > 1 || (c->comm != nullptr && !emul)) && c->kind == kSpheres;
    if (!on) W = 1;
    for (int r = 0; r < W; ++r) parts.push_back(partition(c, W, r));
    if (emul || !on)
      for (int r = 0; r < W; ++r) mine.push_back(r);
    else
      mine.push_back(c->rank);
  }
  const Part& own() const { return parts[emul || !on ? 0 : ctx->rank]; }
  int proj_own(int pp) {
    for (int r : mine)
      if (int rc = launch_proj_own(ctx, pp, parts[r].l0, parts[r].l1)) return rc;
    return 0;
  }
  // every rank's constraint slice of the packed state st -> full vector on every rank
  int bcast(double2* st) {
    if (!on || emul) return 0;
    const Part& p = own();
    double* v = reinterpret_cast<double*>(st);
    NCCL_CHECK(ncclGroupStart());
    for (int r = 0; r < W; ++r) {
      if (p.lcnt[r] == 0) continue;
      NCCL_CHECK(ncclBroadcast(v + 2 * p.loff[r], v + 2 * p.loff[r], 2 * p.lcnt[r], ncclDouble, r, ctx->comm,
                               ctx->stream));
    }
    NCCL_CHECK(ncclGroupEnd());
    return 0;
  }
  // u4 = RPY(f4).  Symmetric kernel: every rank evaluates its super-block pairs into fixed-point
  // row accumulators, the int64 limbs are all-reduced (exact), and every rank combines all rows.
  // Target-row kernel: own rows, then all-gather of the rows.
  int rpy(double mu, const int32_t* done) {
    if (ctx->mobility_model == 2) {  // NEXT row f4(i): the fast summation (one GPU)
      if (on && !emul && W > 1) return fail(ctx, SC_EINVAL, "the fast RPY summation runs on a 1-GPU context");
      return fmm_apply(ctx, ctx->f4.p, mu, ctx->u4.p, done);
    }
    if (rpy_use_sym(ctx)) {
      if (!on) return rpy_apply_sym(ctx, ctx->f4.p, mu, ctx->u4.p, done, 1, mine, 0, nullptr);
      if (emul) return rpy_apply_sym(ctx, ctx->f4.p, mu, ctx->u4.p, done, W, mine, 1, nullptr);
      // exact int64 sum of every rank's fixed-point limbs (9 per row): U is bitwise the 1-GPU U
      auto reduce = [&]() -> int {
        NCCL_CHECK(ncclAllReduce(ctx->sym_acc.p, ctx->sym_acc.p, ctx->npad * 9, ncclInt64, ncclSum, ctx->comm,
                                 ctx->stream));
        return 0;
      };
      return rpy_apply_sym(ctx, ctx->f4.p, mu, ctx->u4.p, done, W, mine, 2, reduce);
    }
    if (!on) return rpy_apply_rows(ctx, ctx->f4.p, 0, ctx->npad, mu, ctx->u4.p, done);
    for (int r : mine) {
      const Part& p = parts[r];
      if (int rc = rpy_apply_rows(ctx, ctx->f4.p, p.row_lo, p.row_hi - p.row_lo, mu, ctx->u4.p, done)) return rc;
    }
    if (emul) return 0;
    double* base = reinterpret_cast<double*>(ctx->u4.p);
    const int64_t cnt = own().rpr * 4;
    NCCL_CHECK(ncclAllGather(base + ctx->rank * cnt, base, cnt, ncclDouble, ctx->comm, ctx->stream));
    return 0;
  }
  // D^T over this process's chunks.  One GPU: fused with K-FINALIZE (returns fused = true).
  int dt(int mode, int pp, bool* fused) {
    *fused = !on;
    if (!on) return launch_dt(ctx, mode, pp, nullptr, nullptr, 0, ctx->nchunks, true);
    for (int r : mine)
      if (int rc = launch_dt(ctx, mode, pp, nullptr, nullptr, parts[r].c0, parts[r].c1, false)) return rc;
    return 0;
  }
  // chunk partials -> reduced vector; returns the buffer K-FINALIZE reads
  const double* reduce_chunks() {
    if (!on) return ctx->chunk_part.p;
    return ctx->chunk_red.p;
  }
  int allreduce() {
    if (!on) return 0;
    const size_t cnt = static_cast<size_t>(ctx->nchunks) * kPartials;
    if (emul) {
      SC_CUDA(cudaMemcpyAsync(ctx->chunk_red.p, ctx->chunk_part.p, cnt * sizeof(double), cudaMemcpyDeviceToDevice,
                              ctx->stream));
      return 0;
    }
    NCCL_CHECK(ncclAllReduce(ctx->chunk_part.p, ctx->chunk_red.p, cnt, ncclDouble, ncclSum, ctx->comm, ctx->stream));
    return 0;
  }
};

// ------------------------------------------------------------ bodies
__global__ void set_spheres_kernel(const double* __restrict__ pos, const double* __restrict__ radius, int64_t n,
                                   int64_t npad, double a_const, double4* __restrict__ pos4,
                                   int32_t* __restrict__ bad) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= npad) return;
  if (b < n) {
    const double a = radius ? radius[b] : a_const;
    if (!(a > 0.0) || !isfinite(a)) atomicOr(bad, 1);
    const double x = pos[3 * b], y = pos[3 * b + 1], z = pos[3 * b + 2];
    if (!(isfinite(x) && isfinite(y) && isfinite(z))) atomicOr(bad, 2);  // NaN/Inf centre
    pos4[b] = make_double4(x, y, z, 0.5 * a);
  } else {
    // padded rows: far away, distinct, zero force (never coincide with anything)
    pos4[b] = make_double4(1e30 + static_cast<double>(b - n) * 1e20, 1e30, 1e30, 0.5 * a_const);
  }
}

__global__ void radius_minmax_kernel(const double* __restrict__ radius, int64_t n, int32_t* __restrict__ poly) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= n) return;
  if (radius[b] != radius[0]) atomicOr(poly, 4);  // bit 2: polydisperse (bits 0, 1: input errors)
}

__global__ void set_rods_kernel(const double* __restrict__ c, const double* __restrict__ d,
                                const double* __restrict__ L, int64_t n, int64_t npad, double b,
                                double4* __restrict__ pos4, double4* __restrict__ dir4, int32_t* __restrict__ bad) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= npad) return;
  if (k < n) {
    const double l = L[k];
    if (!(l > 2.0 * b) || !isfinite(l)) atomicOr(bad, 1);  // drag needs ln(L/2b) > 0
    const double x = c[3 * k], y = c[3 * k + 1], z = c[3 * k + 2];
    const double tx = d[3 * k], ty = d[3 * k + 1], tz = d[3 * k + 2];
    if (!(isfinite(x) && isfinite(y) && isfinite(z) && isfinite(tx) && isfinite(ty) && isfinite(tz)))
      atomicOr(bad, 2);
    else if (!(fabs(tx * tx + ty * ty + tz * tz - 1.0) <= 1e-8))
      atomicOr(bad, 1);  // axes must be unit vectors
    pos4[k] = make_double4(x, y, z, l);
    dir4[k] = make_double4(tx, ty, tz, 0.0);
  } else {
    pos4[k] = make_double4(1e30 + static_cast<double>(k - n) * 1e20, 1e30, 1e30, 1.0);
    dir4[k] = make_double4(1, 0, 0, 0);
  }
}

// zeta_perp = 2 zeta_par = 4 pi mu L / ln(L/(2b)), zeta_rot = pi mu L^3 / (3 ln(L/(2b)))  (configs[3])
__global__ void rod_mob_kernel(const double4* __restrict__ pos4, int64_t n, double b, double mu,
                               double4* __restrict__ mob4) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double L = pos4[k].w;
  const double lg = log(L / (2.0 * b));
  const double pi = 3.14159265358979323846;
  const double zperp = 4.0 * pi * mu * L / lg;
  const double zpar = 0.5 * zperp;
  const double zrot = pi * mu * L * L * L / (3.0 * lg);
  mob4[k] = make_double4(1.0 / zpar, 1.0 / zperp, 1.0 / zrot, mu);
}

static int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

static int prepare_bodies(sc_ctx* ctx, int kind, int64_t n) {
  ctx->fmm_ready = false;  // (the fast summation's tree follows the bodies)
  ctx->kind = kind;
  ctx->n = n;
  ctx->npad = round_up(std::max<int64_t>(n, 1), kNpadQuantum);
  ctx->nsplit = choose_nsplit(ctx->npad, ctx->world);
  ctx->nc = 0;
  ctx->assembled = false;
  ctx->have_q = false;
  ctx->rod_mu = -1.0;
  int64_t rpr, lo, hi;
  plan_rows(ctx->npad, ctx->world, ctx->rank, &rpr, &lo, &hi);
  const int64_t urows = std::max(ctx->npad, rpr * ctx->world);
  if (int rc = ensure(ctx, ctx->pos4, ctx->npad)) return rc;
  if (int rc = ensure(ctx, ctx->f4, ctx->npad)) return rc;
  if (int rc = ensure(ctx, ctx->t4, ctx->npad)) return rc;
  if (int rc = ensure(ctx, ctx->u4, kind == kRods ? 2 * ctx->npad : urows)) return rc;
  if (kind == kRods) {
    if (int rc = ensure(ctx, ctx->dir4, ctx->npad)) return rc;
    if (int rc = ensure(ctx, ctx->rodmob4, ctx->npad)) return rc;
  }
  return 0;
}

// Body-input flags of set_spheres/set_rods: bit 1 -> non-finite coordinates (SC_ENONFINITE),
// bit 0 -> invalid radius / length / axis (SC_EINVAL, msg).
static int check_body_flags(sc_ctx* ctx, const char* msg) {
  SC_CUDA(cudaMemcpyAsync(ctx->herr, ctx->derr, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  SC_CUDA(cudaStreamSynchronize(ctx->stream));
  const int32_t f = *ctx->herr;
  if (f) {
    SC_CUDA(cudaMemsetAsync(ctx->derr, 0, sizeof(int32_t), ctx->stream));
    *ctx->herr = 0;
    if (f & 2) return fail(ctx, SC_ENONFINITE, "non-finite body coordinates or axes");
    return fail(ctx, SC_EINVAL, msg);
  }
  return 0;
}

static int check_flag(sc_ctx* ctx, int code, const char* msg) {
  SC_CUDA(cudaMemcpyAsync(ctx->herr, ctx->derr, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  SC_CUDA(cudaStreamSynchronize(ctx->stream));
  if (*ctx->herr) {
    SC_CUDA(cudaMemsetAsync(ctx->derr, 0, sizeof(int32_t), ctx->stream));
    *ctx->herr = 0;
    return fail(ctx, code, msg);
  }
  return 0;
}

static int ensure_rod_mob(sc_ctx* ctx, double mu) {
  if (ctx->kind != kRods || ctx->rod_mu == mu) return 0;
  if (ctx->n > 0) {
    timer_begin(ctx, SC_K_MISC);
    rod_mob_kernel<<<static_cast<unsigned>((ctx->n + 255) / 256), 256, 0, ctx->stream>>>(
        ctx->pos4.p, ctx->n, ctx->rod_b, mu, ctx->rodmob4.p);
    timer_end(ctx, SC_K_MISC);
    if (int rc = check_launch(ctx, "rod_mob")) return rc;
  }
  ctx->rod_mu = mu;
  return 0;
}

// ---------------------------------------------------------- warm start across solves
__global__ static void pair_keys_kernel(const int32_t* __restrict__ ci, const int32_t* __restrict__ cj, int64_t nc,
                                        int64_t n, const double* __restrict__ gam, int64_t* __restrict__ key,
                                        double* __restrict__ gcopy) {
  const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l >= nc) return;
  // ascending: constraints are sorted by (i, j); j < n + SC_MAX_WALLS (walls are n + k)
  key[l] = static_cast<int64_t>(ci[l]) * (n + SC_MAX_WALLS) + cj[l];
  gcopy[l] = gam[l];
}

__global__ static void warm_match_kernel(const int32_t* __restrict__ ci, const int32_t* __restrict__ cj,
                                         int64_t nc, int64_t n, const int64_t* __restrict__ pkey,
                                         const double* __restrict__ pgam, int64_t pnc, double* __restrict__ gam0) {
  const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l >= nc) return;
  const int64_t k = static_cast<int64_t>(ci[l]) * (n + SC_MAX_WALLS) + cj[l];
  int64_t lo = 0, hi = pnc;  // binary search in the previous (sorted) key list
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (pkey[mid] < k) lo = mid + 1; else hi = mid;
  }
  gam0[l] = (lo < pnc && pkey[lo] == k) ? pgam[lo] : 0.0;
}

int save_for_warm_start(sc_ctx* ctx, const double* gam) {
  const int64_t nc = ctx->nc;
  if (int rc = ensure(ctx, ctx->prev_key, std::max<int64_t>(nc, 1))) return rc;
  if (int rc = ensure(ctx, ctx->prev_gam, std::max<int64_t>(nc, 1))) return rc;
  if (nc > 0) {
    timer_begin(ctx, SC_K_MISC);
    pair_keys_kernel<<<static_cast<unsigned>((nc + 255) / 256), 256, 0, ctx->stream>>>(
        ctx->ci.p, ctx->cj.p, nc, ctx->n, gam, ctx->prev_key.p, ctx->prev_gam.p);
    timer_end(ctx, SC_K_MISC);
    if (int rc = check_launch(ctx, "pair_keys")) return rc;
  }
  ctx->prev_nc = nc;
  ctx->prev_n = ctx->n;
  return 0;
}

int launch_warm_match(sc_ctx* ctx, double* gam0) {
  timer_begin(ctx, SC_K_MISC);
  warm_match_kernel<<<static_cast<unsigned>((ctx->nc + 255) / 256), 256, 0, ctx->stream>>>(
      ctx->ci.p, ctx->cj.p, ctx->nc, ctx->n, ctx->prev_key.p, ctx->prev_gam.p, ctx->prev_nc, gam0);
  timer_end(ctx, SC_K_MISC);
  return check_launch(ctx, "warm_match");
}

}  // namespace sc

using namespace sc;

// ============================================================== C ABI
extern "C" {

int sc_version(void) { return 10000; }
int sc_build_flags(void) { return SC_CHECKS ? 1 : 0; }

static int create_common(sc_ctx** out, int device, void* stream) {
  if (out == nullptr) return SC_EINVAL;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return SC_ECUDA;
  }
  if (device < 0 || device >= ndev) return SC_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return SC_ECUDA;
  sc_ctx* ctx = new sc_ctx();
  ctx->device = device;
  if (stream != nullptr) {
    ctx->stream = static_cast<cudaStream_t>(stream);
  } else {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
      delete ctx;
      return SC_ECUDA;
    }
    ctx->own_stream = true;
  }
  if (cudaMalloc(&ctx->dsc, sizeof(DevScalars)) != cudaSuccess ||
      cudaMallocHost(&ctx->hsc, sizeof(DevScalars)) != cudaSuccess ||
      cudaMalloc(&ctx->derr, sizeof(int32_t)) != cudaSuccess ||
      cudaMalloc(&ctx->dcount, sizeof(unsigned int)) != cudaSuccess ||
      cudaMallocHost(&ctx->herr, sizeof(int32_t)) != cudaSuccess) {
    sc_destroy(ctx);
    return SC_ENOMEM;
  }
  cudaMemset(ctx->derr, 0, sizeof(int32_t));
  cudaMemset(ctx->dcount, 0, sizeof(unsigned int));
  cudaMemset(ctx->dsc, 0, sizeof(DevScalars));
  // per-device setup (kernel attributes are per device: set them on this context's device)
  size_t free_b = 0;
  if (cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess ||
      cudaMemGetInfo(&free_b, &ctx->total_mem) != cudaSuccess || rpy_init_device(ctx) != 0 ||
      persist_init_device(ctx) != 0 || fmm_init_device(ctx) != 0) {
    sc_destroy(ctx);
    return SC_ECUDA;
  }
  if (const char* v = std::getenv("SC_SYM_VARIANT")) ctx->sym_variant = std::atoi(v);
  if (const char* v = std::getenv("SC_SYM_HS")) ctx->sym_hs = std::atoi(v);
  if (const char* v = std::getenv("SC_BATCH")) ctx->batch_override = std::atoi(v);
  if (const char* v = std::getenv("SC_NO_GRAPHS")) ctx->use_graphs = std::atoi(v) == 0;
  if (const char* v = std::getenv("SC_NO_PERSIST")) ctx->use_persist = std::atoi(v) == 0;
  if (const char* v = std::getenv("SC_PERSIST_GRID")) ctx->persist_grid_cap = std::atoi(v);
  *ctx->herr = 0;
  *out = ctx;
  return SC_OK;
}

int sc_create(sc_ctx** out, int device, void* stream) { return create_common(out, device, stream); }

int sc_nccl_unique_id(void* out128) {
  if (out128 == nullptr) return SC_EINVAL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return SC_ENCCL;
  std::memcpy(out128, &id, sizeof(id));
  return SC_OK;
}

int sc_create_dist(sc_ctx** out, int device, void* stream, const void* nccl_id, int rank, int world) {
  if (nccl_id == nullptr || world < 1 || rank < 0 || rank >= world) return SC_EINVAL;
  int rc = create_common(out, device, stream);
  if (rc != SC_OK) return rc;
  sc_ctx* ctx = *out;
  ctx->rank = rank;
  ctx->world = world;
  {  // (world 1 too: a one-rank communicator runs the same NCCL code path as world > 1)
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&ctx->comm, world, id, rank);
    if (r != ncclSuccess) {
      sc_destroy(ctx);
      *out = nullptr;
      return SC_ENCCL;
    }
  }
  return SC_OK;
}

void sc_destroy(sc_ctx* ctx) {
  if (ctx == nullptr) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  release(ctx->pos4); release(ctx->dir4); release(ctx->rodmob4);
  release(ctx->ci); release(ctx->cj); release(ctx->nrm4); release(ctx->lev4); release(ctx->rxn4);
  release(ctx->rpy6_part); release(ctx->ft_tmp); release(ctx->row_ptr); release(ctx->inc); release(ctx->icol4); release(ctx->einc); release(ctx->hinc); release(ctx->first_ptr); release(ctx->near_ptr); release(ctx->near_idx);
  release(ctx->q); release(ctx->gam[0]); release(ctx->gam[1]); release(ctx->g[0]); release(ctx->g[1]);
  release(ctx->w); release(ctx->gam_user); release(ctx->uc); release(ctx->prev_key); release(ctx->prev_gam); release(ctx->chunk_part); release(ctx->chunk_red);
  release(ctx->fmm_key); release(ctx->fmm_idx0); release(ctx->fmm_sidx); release(ctx->fmm_cnt); release(ctx->fmm_lstart); release(ctx->fmm_cubtmp); release(ctx->fmm_spos4); release(ctx->fmm_sf4); release(ctx->fmm_M); release(ctx->fmm_L); release(ctx->fmm_lev_off_dev);
  release(ctx->fmm_svd_U); release(ctx->fmm_svd_C); release(ctx->fmm_Mc); release(ctx->fmm_Lc); release(ctx->fmm_svd_work);
  release(ctx->fmm_svd_li); release(ctx->fmm_svd_ptrs); release(ctx->fmm_acc); release(ctx->fmm_fx);
  fmm_destroy_handles(ctx);
  release(ctx->sym_pairs); release(ctx->sym_acc); release(ctx->fx_scale); release(ctx->trace); release(ctx->f4); release(ctx->t4); release(ctx->u4); release(ctx->rpy_part);
  release(ctx->bbox_part); release(ctx->cell_of); release(ctx->cell_cnt); release(ctx->cell_start);
  release(ctx->sorted_idx); release(ctx->pair_cnt); release(ctx->pair_off); release(ctx->scan_tmp);
  release(ctx->sorted4); release(ctx->sorted_dir4); release(ctx->stage);
  for (auto& b : ctx->stage_pool) release(b);
  if (ctx->dsc) cudaFree(ctx->dsc);
  if (ctx->hsc) cudaFreeHost(ctx->hsc);
  if (ctx->derr) cudaFree(ctx->derr);
  if (ctx->dcount) cudaFree(ctx->dcount);
  if (ctx->herr) cudaFreeHost(ctx->herr);
  for (int f = 0; f < SC_K_COUNT; ++f)
    for (auto e : ctx->timer.ev[f]) cudaEventDestroy(e);
  for (auto e : ctx->timer.pool) cudaEventDestroy(e);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* sc_last_error(const sc_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }
void* sc_stream(const sc_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int sc_plan_partition(int64_t n, int world, int rank, int64_t* out7) {
  if (n < 0 || world < 1 || rank < 0 || rank >= world || out7 == nullptr) return SC_EINVAL;
  const int64_t npad = round_up(std::max<int64_t>(n, 1), kNpadQuantum);
  int64_t rpr, lo, hi;
  plan_rows(npad, world, rank, &rpr, &lo, &hi);
  out7[0] = npad;
  out7[1] = rpr;
  out7[2] = lo;
  out7[3] = hi;
  out7[4] = lo / kChunkBodies;
  out7[5] = hi / kChunkBodies;
  out7[6] = choose_nsplit(npad, world);
  return SC_OK;
}

// ------------------------------------------------------------ residual
int sc_minmap_residual(sc_ctx* ctx, int64_t n_c, const double* gamma, const double* g, double* phi) {
  if (ctx == nullptr) return SC_EINVAL;
  if (n_c < 0 || phi == nullptr || (n_c > 0 && (gamma == nullptr || g == nullptr)))
    return fail(ctx, SC_EINVAL, "minmap_residual: bad arguments");
  cudaSetDevice(ctx->device);
  if (n_c == 0) {
    *phi = 0.0;
    return SC_OK;
  }
  Stager st(ctx);
  const double *dg = nullptr, *dgr = nullptr;
  if (int rc = st.in(gamma, n_c, &dg)) return rc;
  if (int rc = st.in(g, n_c, &dgr)) return rc;
  double* dphi = nullptr;
  if (int rc = st.out(phi, 1, &dphi)) return rc;
  if (int rc = launch_minmap(ctx, dg, dgr, n_c, dphi)) return rc;
  if (int rc = st.finish()) return rc;
  SC_CUDA(cudaStreamSynchronize(ctx->stream));
  if (dphi != phi && !std::isfinite(*phi)) return fail(ctx, SC_ENONFINITE, "non-finite residual");  // (host phi)
  return SC_OK;
}

// ------------------------------------------------------------ NEXT row f4(ii)
int sc_set_mobility_model(sc_ctx* ctx, int model) {
  if (ctx == nullptr) return SC_EINVAL;
  if (model < 0 || model > 2)
    return fail(ctx, SC_EINVAL, "set_mobility_model: 0 (RPY), 1 (full 6N RPY) or 2 (RPY by the fast summation)");
  ctx->mobility_model = model;
  return SC_OK;
}

int sc_set_fmm_params(sc_ctx* ctx, int order, int leaf_level) {
  if (ctx == nullptr) return SC_EINVAL;
  if ((order != 4 && order != 6 && order != 8) || leaf_level < 0 || leaf_level > 8)
    return fail(ctx, SC_EINVAL, "set_fmm_params: order 4, 6 or 8; leaf_level 0 (auto) .. 8");
  ctx->fmm_order = order;
  ctx->fmm_leaf_level = leaf_level;
  ctx->fmm_ready = false;
  return SC_OK;
}

int sc_set_fmm_tolerance(sc_ctx* ctx, double rel_err, int* order_out) {
  if (ctx == nullptr) return SC_EINVAL;
  // the stated relative L2 bars of the apply per order (tests/test_gpu_fmm.py)
  int order = 0;
  if (rel_err >= 2e-3) order = 4;
  else if (rel_err >= 6e-5) order = 6;
  else if (rel_err >= 3e-6) order = 8;
  if (order == 0 || !std::isfinite(rel_err))
    return fail(ctx, SC_EINVAL, "set_fmm_tolerance: below the order-8 bar (3e-6): use the direct RPY kernel");
  if (int rc = sc_set_fmm_params(ctx, order, 0)) return rc;
  if (order_out) *order_out = order;
  return SC_OK;
}

int sc_set_fmm_compression(sc_ctx* ctx, int mode) {
  if (ctx == nullptr) return SC_EINVAL;
  if (mode < 0 || mode > 2) return fail(ctx, SC_EINVAL, "set_fmm_compression: 0 (off), 1 (on) or 2 (auto)");
  ctx->fmm_compress = mode;
  ctx->fmm_ready = false;  // (the root side follows the mode)
  return SC_OK;
}

int sc_get_fmm_compression_info(const sc_ctx* ctx, int32_t* out4) {
  if (ctx == nullptr || out4 == nullptr) return SC_EINVAL;
  out4[0] = ctx->fmm_compress;
  out4[1] = fmm_uses_library_calls(ctx) ? 1 : 0;
  const bool built = ctx->fmm_svd_key[4] != 0.0 && !ctx->fmm_svd_k.empty();
  out4[2] = built ? ctx->fmm_svd_k.back() : 0;                     // rank at the leaf level
  out4[3] = built ? static_cast<int32_t>(ctx->fmm_svd_k.size()) - 1 : 0;  // leaf level of the bases
  return SC_OK;
}

int sc_get_fmm_info(const sc_ctx* ctx, int32_t* out3) {
  if (ctx == nullptr || out3 == nullptr) return SC_EINVAL;
  out3[0] = ctx->fmm_order;
  out3[1] = ctx->fmm_ready ? ctx->fmm_L_used : 0;
  out3[2] = ctx->fmm_ready ? 1 : 0;
  return SC_OK;
}

// ------------------------------------------------------------ NEXT row f2: walls
int sc_set_walls(sc_ctx* ctx, int n_walls, const double* walls) {
  if (ctx == nullptr) return SC_EINVAL;
  if (n_walls < 0 || n_walls > SC_MAX_WALLS || (n_walls > 0 && walls == nullptr))
    return fail(ctx, SC_EINVAL, "set_walls: 0 <= n_walls <= SC_MAX_WALLS and walls != NULL");
  for (int k = 0; k < n_walls; ++k) {
    const double* w = walls + 4 * k;
    const double nn = w[0] * w[0] + w[1] * w[1] + w[2] * w[2];
    if (!(std::isfinite(w[3]) && std::fabs(nn - 1.0) <= 1e-12))
      return fail(ctx, SC_EINVAL, "set_walls: normals must be unit vectors and offsets finite");
  }
  ctx->nwalls = n_walls;
  for (int k = 0; k < SC_MAX_WALLS; ++k) {
    ctx->walls[k] = k < n_walls ? make_double4(walls[4 * k], walls[4 * k + 1], walls[4 * k + 2], walls[4 * k + 3])
                                : make_double4(0, 0, 0, 0);
    ctx->wall_vel[k][0] = ctx->wall_vel[k][1] = ctx->wall_vel[k][2] = 0.0;  // static until set
  }
  ctx->prev_nc = 0;  // the constraint numbering changes: no warm start across this call
  return SC_OK;
}

int sc_set_wall_velocities(sc_ctx* ctx, int n_walls, const double* vel) {
  if (ctx == nullptr) return SC_EINVAL;
  if (n_walls != ctx->nwalls || (n_walls > 0 && vel == nullptr))
    return fail(ctx, SC_EINVAL, "set_wall_velocities: one velocity per wall of sc_set_walls");
  for (int k = 0; k < n_walls * 3; ++k)
    if (!std::isfinite(vel[k])) return fail(ctx, SC_EINVAL, "set_wall_velocities: non-finite velocity");
  for (int k = 0; k < n_walls; ++k)
    for (int c = 0; c < 3; ++c) ctx->wall_vel[k][c] = vel[3 * k + c];
  return SC_OK;
}

int sc_get_walls(const sc_ctx* ctx, double* walls) {
  if (ctx == nullptr || (ctx->nwalls > 0 && walls == nullptr)) return SC_EINVAL;
  for (int k = 0; k < ctx->nwalls; ++k) {
    walls[4 * k] = ctx->walls[k].x;
    walls[4 * k + 1] = ctx->walls[k].y;
    walls[4 * k + 2] = ctx->walls[k].z;
    walls[4 * k + 3] = ctx->walls[k].w;
  }
  return SC_OK;
}

// ------------------------------------------------------------ (a1)
int sc_build_contacts_spheres(sc_ctx* ctx, int64_t n, const double* pos, const double* radius, double gap_abs,
                              double gap_rel, int64_t* n_c) {
  if (ctx == nullptr) return SC_EINVAL;
  if (n < 0 || (n > 0 && pos == nullptr) || !(gap_rel >= 0.0) || !std::isfinite(gap_abs))
    return fail(ctx, SC_EINVAL, "build_contacts_spheres: bad arguments");
  if (n >= (int64_t(1) << 30)) return fail(ctx, SC_EINVAL, "too many bodies");
  cudaSetDevice(ctx->device);
  if (int rc = prepare_bodies(ctx, kSpheres, n)) return rc;
  Stager st(ctx);
  const double *dpos = nullptr, *drad = nullptr;
  if (int rc = st.in(pos, 3 * n, &dpos)) return rc;
  if (int rc = st.in(radius, n, &drad)) return rc;
  SC_CUDA(cudaMemsetAsync(ctx->derr, 0, sizeof(int32_t), ctx->stream));
  timer_begin(ctx, SC_K_MISC);
  set_spheres_kernel<<<static_cast<unsigned>((ctx->npad + 255) / 256), 256, 0, ctx->stream>>>(
      dpos, drad, n, ctx->npad, 1.0, ctx->pos4.p, ctx->derr);
  timer_end(ctx, SC_K_MISC);
  if (int rc = check_launch(ctx, "set_spheres")) return rc;
  // monodisperse fast path when all radii are equal (checked with the input flags: one host read)
  ctx->poly = 0;
  ctx->a_const = 1.0;
  double a0 = 1.0;
  if (radius != nullptr && n > 0) {
    timer_begin(ctx, SC_K_MISC);
    radius_minmax_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(drad, n, ctx->derr);
    timer_end(ctx, SC_K_MISC);
    if (int rc = check_launch(ctx, "radius_minmax")) return rc;
    SC_CUDA(cudaMemcpyAsync(&a0, drad, sizeof(double), cudaMemcpyDefault, ctx->stream));
  }
  SC_CUDA(cudaMemcpyAsync(ctx->herr, ctx->derr, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  SC_CUDA(cudaStreamSynchronize(ctx->stream));
  const int32_t flags = *ctx->herr;
  *ctx->herr = 0;
  if (flags) SC_CUDA(cudaMemsetAsync(ctx->derr, 0, sizeof(int32_t), ctx->stream));
  if (flags & 2) return fail(ctx, SC_ENONFINITE, "non-finite body coordinates or axes");
  if (flags & 1) return fail(ctx, SC_EINVAL, "radii must be positive and finite");
  if (radius != nullptr && n > 0) {
    ctx->poly = (flags & 4) ? 1 : 0;
    ctx->a_const = a0;
  }
  if (ctx->npad > n) {  // padded rows carry the constant radius
    // (their w only enters the far formula for zero-force sources)
  }
  if (int rc = build_contacts_spheres(ctx, gap_abs, gap_rel)) return rc;
  if (n_c) *n_c = ctx->nc;
  return SC_OK;
}

int sc_build_contacts_rods(sc_ctx* ctx, int64_t n, const double* center, const double* dir, const double* length,
                           double b, double gap_thresh, int64_t* n_c) {
  if (ctx == nullptr) return SC_EINVAL;
  if (n < 0 || (n > 0 && (center == nullptr || dir == nullptr || length == nullptr)) || !(b > 0.0) ||
      !std::isfinite(gap_thresh))
    return fail(ctx, SC_EINVAL, "build_contacts_rods: bad arguments");
  if (n >= (int64_t(1) << 30)) return fail(ctx, SC_EINVAL, "too many bodies");
  cudaSetDevice(ctx->device);
  if (int rc = prepare_bodies(ctx, kRods, n)) return rc;
  ctx->rod_b = b;
  ctx->poly = 0;
  Stager st(ctx);
  const double *dc = nullptr, *dd = nullptr, *dl = nullptr;
  if (int rc = st.in(center, 3 * n, &dc)) return rc;
  if (int rc = st.in(dir, 3 * n, &dd)) return rc;
  if (int rc = st.in(length, n, &dl)) return rc;
  SC_CUDA(cudaMemsetAsync(ctx->derr, 0, sizeof(int32_t), ctx->stream));
  timer_begin(ctx, SC_K_MISC);
  set_rods_kernel<<<static_cast<unsigned>((ctx->npad + 255) / 256), 256, 0, ctx->stream>>>(
      dc, dd, dl, n, ctx->npad, b, ctx->pos4.p, ctx->dir4.p, ctx->derr);
  timer_end(ctx, SC_K_MISC);
  if (int rc = check_launch(ctx, "set_rods")) return rc;
  if (int rc = check_body_flags(ctx, "rod lengths must exceed 2b (ln(L/2b) > 0) and axes be unit vectors")) return rc;
  if (int rc = build_contacts_rods(ctx, gap_thresh)) return rc;
  if (n_c) *n_c = ctx->nc;
  return SC_OK;
}

__global__ static void unpack_contacts_kernel(const double4* __restrict__ nrm4, const double4* __restrict__ lev4,
                                              int64_t nc, double* __restrict__ gap, double* __restrict__ normal,
                                              double* __restrict__ lever) {
  const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (l >= nc) return;
  const double4 v = nrm4[l];
  if (gap) gap[l] = v.w;
  if (normal) {
    normal[3 * l] = v.x;
    normal[3 * l + 1] = v.y;
    normal[3 * l + 2] = v.z;
  }
  if (lever) {
    const double4 a = lev4[2 * l], b = lev4[2 * l + 1];
    double* o = lever + 6 * l;
    o[0] = a.x; o[1] = a.y; o[2] = a.z; o[3] = b.x; o[4] = b.y; o[5] = b.z;
  }
}

int sc_get_contacts(sc_ctx* ctx, int32_t* ci, int32_t* cj, double* gap, double* normal, double* lever) {
  if (ctx == nullptr) return SC_EINVAL;
  if (ctx->kind == kNone) return fail(ctx, SC_EINVAL, "get_contacts before build_contacts");
  if (lever != nullptr && ctx->kind != kRods) return fail(ctx, SC_EINVAL, "lever arms exist for rods only");
  cudaSetDevice(ctx->device);
  const int64_t nc = ctx->nc;
  if (nc == 0) return SC_OK;
  Stager st(ctx);
  int32_t *oi = nullptr, *oj = nullptr;
  double *og = nullptr, *on = nullptr, *ol = nullptr;
  if (int rc = st.out(ci, nc, &oi)) return rc;
  if (int rc = st.out(cj, nc, &oj)) return rc;
  if (int rc = st.out(gap, nc, &og)) return rc;
  if (int rc = st.out(normal, 3 * nc, &on)) return rc;
  if (int rc = st.out(lever, 6 * nc, &ol)) return rc;
  if (oi) SC_CUDA(cudaMemcpyAsync(oi, ctx->ci.p, nc * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
  if (oj) SC_CUDA(cudaMemcpyAsync(oj, ctx->cj.p, nc * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
  if (og || on || ol) {
    timer_begin(ctx, SC_K_MISC);
    unpack_contacts_kernel<<<static_cast<unsigned>((nc + 255) / 256), 256, 0, ctx->stream>>>(
        ctx->nrm4.p, ctx->lev4.p, nc, og, on, ol);
    timer_end(ctx, SC_K_MISC);
    if (int rc = check_launch(ctx, "unpack_contacts")) return rc;
  }
  if (int rc = st.finish()) return rc;
  SC_CUDA(cudaStreamSynchronize(ctx->stream));
  return SC_OK;
}

// ------------------------------------------------------------ (a2)
int sc_assemble_D(sc_ctx* ctx) {
  if (ctx == nullptr) return SC_EINVAL;
  if (ctx->kind == kNone) return fail(ctx, SC_EINVAL, "assemble_D before build_contacts");
  cudaSetDevice(ctx->device);
  if (int rc = assemble(ctx)) return rc;
  const int64_t nc = ctx->nc;
  for (int k = 0; k < 2; ++k) {
    if (int rc = ensure(ctx, ctx->gam[k], nc)) return rc;
    if (int rc = ensure(ctx, ctx->g[k], nc)) return rc;
    if (int rc = ensure(ctx, ctx->st[k], nc)) return rc;
  }
  if (int rc = ensure(ctx, ctx->q, nc)) return rc;
  if (int rc = ensure(ctx, ctx->chunk_part, ctx->nchunks * kPartials)) return rc;
  if (int rc = ensure(ctx, ctx->chunk_red, ctx->nchunks * kPartials)) return rc;
  SC_CUDA(cudaMemsetAsync(ctx->chunk_part.p, 0, sizeof(double) * ctx->nchunks * kPartials, ctx->stream));
  SC_CUDA(cudaStreamSynchronize(ctx->stream));
  return SC_OK;
}

int sc_apply_D(sc_ctx* ctx, const double* gamma, double* FT) {
  if (ctx == nullptr) return SC_EINVAL;
  if (!ctx->assembled) return fail(ctx, SC_EINVAL, "apply_D before assemble_D");
  if (FT == nullptr || (ctx->nc > 0 && gamma == nullptr)) return fail(ctx, SC_EINVAL, "apply_D: NULL buffer");
  cudaSetDevice(ctx->device);
  Stager st(ctx);
  const double* dg = nullptr;
  double* dF = nullptr;
  if (int rc = st.in(gamma, ctx->nc, &dg)) return rc;
  if (int rc = st.out(FT, 6 * ctx->n, &dF)) return rc;
  if (ctx->n > 0) {
    if (int rc = launch_gather_raw(ctx, dg, 1, 1.0, dF)) return rc;
  }
  if (int rc = st.finish()) return rc;
  return SC_OK;
}

int sc_apply_DT(sc_ctx* ctx, const double* UW, double* out) {
  if (ctx == nullptr) return SC_EINVAL;
  if (!ctx->assembled) return fail(ctx, SC_EINVAL, "apply_DT before assemble_D");
  if (ctx->nc > 0 && (UW == nullptr || out == nullptr)) return fail(ctx, SC_EINVAL, "apply_DT: NULL buffer");
  cudaSetDevice(ctx->device);
  Stager st(ctx);
  const double* du = nullptr;
  double* dout = nullptr;
  if (int rc = st.in(UW, 6 * ctx->n, &du)) return rc;
  if (int rc = st.out(out, ctx->nc, &dout)) return rc;
  if (int rc = launch_dt_user(ctx, du, dout, nullptr, 0.0)) return rc;
  if (int rc = st.finish()) return rc;
  return SC_OK;
}

// ------------------------------------------------------------ (a4)
int sc_mobility_apply(sc_ctx* ctx, double mu, const double* FT, double* UW) {
  if (ctx == nullptr) return SC_EINVAL;
  if (ctx->kind == kNone) return fail(ctx, SC_EINVAL, "mobility_apply before build_contacts");
  if (!(mu > 0.0) || (ctx->n > 0 && (FT == nullptr || UW == nullptr)))
    return fail(ctx, SC_EINVAL, "mobility_apply: bad arguments");
  if (ctx->n == 0) return SC_OK;
  cudaSetDevice(ctx->device);
  Stager st(ctx);
  const double* dF = nullptr;
  double* dU = nullptr;
  if (int rc = st.in(FT, 6 * ctx->n, &dF)) return rc;
  if (int rc = st.out(UW, 6 * ctx->n, &dU)) return rc;
  if (ctx->kind == kSpheres && ctx->mobility_model == 1) {  // full grand mobility (every rank: all rows)
    if (int rc = launch_pack_ft(ctx, dF, ctx->f4.p, ctx->t4.p)) return rc;
    if (int rc = rpy6_apply(ctx, ctx->f4.p, ctx->t4.p, mu, dU)) return rc;
    if (int rc = check_flag(ctx, SC_EDEGENERATE, "coincident centres in the RPY sum")) return rc;
  } else if (ctx->kind == kSpheres) {
    if (int rc = launch_pack_ft(ctx, dF, ctx->f4.p, ctx->t4.p)) return rc;
    Dist D(ctx);
    if (int rc = D.rpy(mu, nullptr)) return rc;
    if (int rc = launch_unpack_uw_spheres(ctx, ctx->u4.p, ctx->t4.p, mu, dU)) return rc;
    if (int rc = check_flag(ctx, SC_EDEGENERATE, "coincident centres in the RPY sum")) return rc;
  } else {
    if (int rc = ensure_rod_mob(ctx, mu)) return rc;
    if (int rc = launch_rod_drag_user(ctx, dF, mu, dU)) return rc;
  }
  if (int rc = st.finish()) return rc;
  return SC_OK;
}

// ------------------------------------------------------------ q
int sc_lcp_q(sc_ctx* ctx, double dt, const double* U_nc, double* q_out) {
  if (ctx == nullptr) return SC_EINVAL;
  if (!ctx->assembled) return fail(ctx, SC_EINVAL, "lcp_q before assemble_D");
  if (!(dt > 0.0) || (ctx->n > 0 && U_nc == nullptr)) return fail(ctx, SC_EINVAL, "lcp_q: bad arguments");
  cudaSetDevice(ctx->device);
  Stager st(ctx);
  const double* du = nullptr;
  if (int rc = st.in(U_nc, 6 * ctx->n, &du)) return rc;
  if (int rc = launch_dt_user(ctx, du, ctx->q.p, ctx->q.p, 1.0 / dt)) return rc;
  if (q_out != nullptr && ctx->nc > 0) {
    double* dq = nullptr;
    if (int rc = st.out(q_out, ctx->nc, &dq)) return rc;
    SC_CUDA(cudaMemcpyAsync(dq, ctx->q.p, ctx->nc * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  }
  if (int rc = st.finish()) return rc;
  ctx->have_q = true;
  return SC_OK;
}

// ------------------------------------------------------------ (a6) BBPGD
static int read_scalars(sc_ctx* ctx) {
  SC_CUDA(cudaMemcpyAsync(ctx->hsc, ctx->dsc, sizeof(DevScalars), cudaMemcpyDeviceToHost, ctx->stream));
  SC_CUDA(cudaStreamSynchronize(ctx->stream));
  return 0;
}

int sc_bbpgd_solve(sc_ctx* ctx, const sc_bbpgd_opts* opts, double* gamma, double* g_out, double* Fc_out,
                   double* Uc_out, sc_bbpgd_stats* stats) {
  if (ctx == nullptr) return SC_EINVAL;
  if (opts == nullptr || !(opts->mu > 0.0) || !(opts->tol >= 0.0) || opts->max_iter < 0 || opts->bb_mode < 0 ||
      opts->bb_mode > 2)
    return fail(ctx, SC_EINVAL, "bbpgd_solve: bad options");
  if (!ctx->assembled || !ctx->have_q) return fail(ctx, SC_EINVAL, "bbpgd_solve needs assemble_D and lcp_q first");
  const int64_t nc = ctx->nc, n = ctx->n;
  if (nc > 0 && gamma == nullptr) return fail(ctx, SC_EINVAL, "bbpgd_solve: gamma is NULL");
  cudaSetDevice(ctx->device);
  sc_bbpgd_stats stt;
  std::memset(&stt, 0, sizeof(stt));
  const double mu = opts->mu;
  if (int rc = ensure_rod_mob(ctx, mu)) return rc;
  Stager st(ctx);
  double *dgam = nullptr, *dg = nullptr, *dF = nullptr, *dU = nullptr;
  if (opts->warm_start == 1) {
    if (int rc = st.inout(gamma, nc, &dgam)) return rc;
  } else {
    if (int rc = st.out(gamma, nc, &dgam)) return rc;
  }
  if (int rc = st.out(g_out, nc, &dg)) return rc;
  if (int rc = st.out(Fc_out, 6 * n, &dF)) return rc;
  if (int rc = st.out(Uc_out, 6 * n, &dU)) return rc;

  ctx->trace_count = 0;
  // warm start (opts->warm_start == 2) from the previous solve of this context: decided here;
  // the previous gamma is then invalidated until this solve completes (an error or an empty
  // solve below must not leave an older gamma to warm-start a later solve)
  const bool from_prev = opts->warm_start == 2 && ctx->prev_nc > 0 && ctx->prev_n == n && nc > 0;
  if (from_prev) {
    if (int rc = launch_warm_match(ctx, ctx->gam[0].p)) return rc;
  }
  ctx->prev_nc = 0;
  if (nc == 0) {  // nothing to resolve: gamma is empty, F_c = 0, U_c = 0
    if (dF) SC_CUDA(cudaMemsetAsync(dF, 0, sizeof(double) * 6 * n, ctx->stream));
    if (dU) SC_CUDA(cudaMemsetAsync(dU, 0, sizeof(double) * 6 * n, ctx->stream));
    if (int rc = st.finish()) return rc;
    stt.converged = 1;
    stt.mvops = 0;
    if (stats) *stats = stt;
    return SC_OK;
  }
  Dist D(ctx);
  const bool dist = D.on;
  const bool spheres = ctx->kind == kSpheres;
  const int32_t* done = &ctx->dsc->done;
  if (spheres && ctx->mobility_model == 2 && !ctx->fmm_ready) {  // (the tree, before any graph capture)
    if (int rc = fmm_setup(ctx)) return rc;
  }

  DevScalars h;
  std::memset(&h, 0, sizeof(h));
  h.tol = opts->tol;
  h.max_iter = opts->max_iter;
  h.bb_mode = opts->bb_mode;
  h.fixed = opts->fixed_iters ? 1 : 0;
  h.trace = ctx->trace_cap > 0 ? ctx->trace.p : nullptr;
  h.trace_cap = ctx->trace_cap;
  SC_CUDA(cudaMemcpyAsync(ctx->dsc, &h, sizeof(h), cudaMemcpyHostToDevice, ctx->stream));
  SC_CUDA(cudaMemsetAsync(ctx->derr, 0, sizeof(int32_t), ctx->stream));
  SC_CUDA(cudaMemsetAsync(ctx->chunk_part.p, 0, sizeof(double) * ctx->nchunks * kPartials, ctx->stream));

  // mvop(v): u4 = Mobility(D v)  (spheres: f4 then RPY; rods: fused gather + drag)
  auto mvop_raw = [&](const double* v, int vstride) -> int {
    if (int rc = launch_gather_raw(ctx, v, vstride, mu, nullptr)) return rc;
    if (spheres) return D.rpy(mu, done);
    return 0;
  };
  // the components of the packed state st[k] = (gamma, g) as strided vectors
  auto st_gamma = [&](int k) { return reinterpret_cast<const double*>(ctx->st[k].p); };
  auto st_g = [&](int k) { return reinterpret_cast<const double*>(ctx->st[k].p) + 1; };
  bool fused = false;  // set by D.dt: the D^T kernel already ran K-FINALIZE
  auto reduce = [&](int mode) -> int {
    if (fused) return 0;
    if (int rc = D.allreduce()) return rc;
    return launch_finalize(ctx, mode, D.reduce_chunks());
  };

  // Steps 1-5: gamma_0, g_0 = M gamma_0 + q, phi_0
  double* gam0 = ctx->gam[0].p;
  if (opts->warm_start == 1 || from_prev) {
    if (from_prev) {  // gamma_0 of each (i, j) = the previous solve's gamma of the same pair, else 0
      // (matched above, before the previous solve's list was invalidated)
    } else {
      SC_CUDA(cudaMemcpyAsync(gam0, dgam, nc * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    }
    // projection onto gamma >= 0 (Step 1), into the packed state
    if (int rc = launch_pack_gamma0(ctx, gam0)) return rc;
    if (int rc = mvop_raw(st_gamma(0), 2)) return rc;
    if (int rc = D.dt(2, 0, &fused)) return rc;
  } else {
    SC_CUDA(cudaMemsetAsync(ctx->st[0].p, 0, nc * sizeof(double2), ctx->stream));
    SC_CUDA(cudaMemsetAsync(ctx->u4.p, 0, sizeof(double4) * ctx->u4.n, ctx->stream));
    if (int rc = D.dt(5, 0, &fused)) return rc;
  }
  if (int rc = reduce(2)) return rc;
  stt.mvops = 1;
  if (int rc = read_scalars(ctx)) return rc;
  ctx->trace_count = std::min(ctx->trace_cap, 1);
  int rc_final = SC_OK;
  int parity = 0;
  if (ctx->hsc->nonfinite) return fail(ctx, SC_ENONFINITE, "non-finite initial gradient");
  if (!ctx->hsc->done) {
    // Step 6: alpha_0 = g0.g0 / g0.M g0 (second MVOP, on the full g_0)
    if (int rc = D.bcast(ctx->st[0].p)) return rc;
    if (int rc = mvop_raw(st_g(0), 2)) return rc;
    if (int rc = D.dt(1, 0, &fused)) return rc;
    if (int rc = reduce(1)) return rc;
    stt.mvops = 2;
    // Steps 7-16
    // iterations enqueued between two host reads of the scalars: enough to cover ~1 ms of
    // device work (extra iterations after convergence are no-op launches)
    const double t_iter = spheres ? 1.3e-12 * static_cast<double>(ctx->npad) * ctx->npad + 4e-5
                                  : 2e-5 + 1.2e-10 * static_cast<double>(nc + n);
    // (multi-GPU: the done flag is identical on every rank -- K-FINALIZE runs on every rank on the
    // all-reduced partials -- so every rank enqueues the same batches and the collectives match)
    int batch = std::max(1, std::min(32, static_cast<int>(1e-3 / t_iter)));
    // (the compressed fast summation's cuBLAS calls do not read the done flag: one iteration per
    // host read, so nothing runs after convergence)
    if (spheres && ctx->mobility_model == 2 && fmm_uses_library_calls(ctx)) batch = 1;
    if (ctx->batch_override > 0) batch = ctx->batch_override;  // tuning (env SC_BATCH)
    auto enqueue_iter = [&](int pp) -> int {
      if (dist) {  // Steps 8-9 on own constraints, then every rank needs the full gamma_j
        if (int rc = D.proj_own(pp)) return rc;
        if (int rc = D.bcast(ctx->st[pp ^ 1].p)) return rc;
        if (int rc = mvop_raw(st_gamma(pp ^ 1), 2)) return rc;
      } else {  // Steps 8-9 fused into the D-gather
        if (int rc = launch_gather_proj(ctx, pp, mu)) return rc;
        if (spheres) {
          if (int rc = D.rpy(mu, done)) return rc;
        }
      }
      if (int rc = D.dt(0, pp, &fused)) return rc;  // Steps 10-15
      return reduce(0);
    };
    // One GPU, no per-launch timing: the loop runs on the device.  The two-iteration kernel
    // sequence (even + odd buffer parity) is captured once as the body of a CUDA-graph
    // conditional WHILE node; a last one-thread kernel sets the loop condition to !done (the
    // flag K-FINALIZE sets on convergence, j_max or a non-finite value), so the whole Steps 7-16
    // loop is one graph launch: no host round trip per batch of iterations and at most one
    // no-op iteration after the last.  Multi-GPU (NCCL) or timed runs: iterations enqueued from
    // the host in batches, the host reading the scalars between batches.
    cudaGraphExec_t gexec = nullptr;
    const bool persist = !dist && persist_eligible(ctx) && opts->max_iter > 0;
    if (persist) {  // small problem: the whole loop in one cooperative launch (persist.cu)
      if (int rc = bbpgd_persistent(ctx, mu)) return rc;
      if (int rc = read_scalars(ctx)) return rc;
    }
    // (the compressed fast summation calls cuBLAS: host-enqueued iterations, no graph capture)
    const bool lib_calls = spheres && ctx->mobility_model == 2 && fmm_uses_library_calls(ctx);
    if (!persist && !dist && !ctx->timer.enabled && ctx->use_graphs && opts->max_iter > 0 && !lib_calls) {
      cudaGraph_t graph = nullptr;
      SC_CUDA(cudaGraphCreate(&graph, 0));
      cudaGraphConditionalHandle cond;
      cudaError_t ce = cudaGraphConditionalHandleCreate(&cond, graph, 1, cudaGraphCondAssignDefault);
      cudaGraphNodeParams np = {};
      np.type = cudaGraphNodeTypeConditional;
      np.conditional.handle = cond;
      np.conditional.type = cudaGraphCondTypeWhile;
      np.conditional.size = 1;
      cudaGraphNode_t node;
      if (ce == cudaSuccess) ce = cudaGraphAddNode(&node, graph, nullptr, 0, &np);
      if (ce != cudaSuccess) {
        cudaGraphDestroy(graph);
        return cuda_fail(ctx, ce, "conditional graph node");
      }
      cudaGraph_t body = np.conditional.phGraph_out[0];
      const int64_t l0 = ctx->launch_count;
      ce = cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
      int rc0 = ce == cudaSuccess ? 0 : cuda_fail(ctx, ce, "cudaStreamBeginCaptureToGraph");
      if (rc0 == 0) rc0 = enqueue_iter(0);
      if (rc0 == 0) rc0 = enqueue_iter(1);
      if (rc0 == 0) rc0 = launch_loop_continue(ctx, cond);
      if (ce == cudaSuccess) {
        cudaGraph_t captured = nullptr;
        cudaError_t ce2 = cudaStreamEndCapture(ctx->stream, &captured);
        if (rc0 == 0 && ce2 != cudaSuccess) rc0 = cuda_fail(ctx, ce2, "cudaStreamEndCapture");
      }
      if (rc0 == 0) {
        ce = cudaGraphInstantiate(&gexec, graph, 0);
        if (ce != cudaSuccess) rc0 = cuda_fail(ctx, ce, "cudaGraphInstantiate(conditional loop)");
      }
      cudaGraphDestroy(graph);
      const int64_t body_kernels = ctx->launch_count - l0;
      ctx->launch_count = l0;
      if (rc0 != 0) return rc0;
      ce = cudaGraphLaunch(gexec, ctx->stream);
      if (ce != cudaSuccess) {
        cudaGraphExecDestroy(gexec);
        return cuda_fail(ctx, ce, "cudaGraphLaunch(conditional loop)");
      }
      if (int rc = read_scalars(ctx)) {
        cudaGraphExecDestroy(gexec);
        return rc;
      }
      ctx->launch_count += body_kernels * std::max(1, (ctx->hsc->iter + 1) / 2);  // bodies run
    }
    int enq = (persist || gexec) ? opts->max_iter : 0;
    while (enq < opts->max_iter) {
      const int nb = std::min(batch, opts->max_iter - enq);
      for (int k = 0; k < nb; ++k)
        if (int rc = enqueue_iter((enq + k) & 1)) return rc;
      enq += nb;
      if (int rc = read_scalars(ctx)) return rc;
      if (ctx->hsc->done) break;
    }
    if (gexec) cudaGraphExecDestroy(gexec);
    parity = ctx->hsc->iter & 1;
    stt.iters = ctx->hsc->iter;
    ctx->trace_count = std::min(ctx->trace_cap, ctx->hsc->iter + 1);
    stt.mvops = 2 + ctx->hsc->iter;
  }
  const DevScalars& s = *ctx->hsc;
  if (s.nonfinite) return fail(ctx, SC_ENONFINITE, "non-finite value in the BBPGD iteration");
  stt.converged = s.conv;
  stt.residual = s.phi;
  stt.alpha = s.alpha;
  stt.bb_breakdowns = s.breakdowns;
  if (!s.conv && !opts->fixed_iters) rc_final = SC_NOT_CONVERGED;
  double* gfin = ctx->gam[parity].p;
  double* gradfin = ctx->g[parity].p;
  if (int rc = D.bcast(ctx->st[parity].p)) return rc;  // (every rank's g slice)
  if (int rc = launch_unpack_state(ctx, parity, gfin, gradfin)) return rc;
  if (int rc = check_flag(ctx, SC_EDEGENERATE, "coincident centres in the RPY sum")) return rc;
  // outputs
  SC_CUDA(cudaMemcpyAsync(dgam, gfin, nc * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  if (dg) SC_CUDA(cudaMemcpyAsync(dg, gradfin, nc * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  if (dF) {
    if (int rc = launch_gather_raw(ctx, gfin, 1, mu, dF)) return rc;
  }
  if (dU) {
    // j_max = 0: u4 holds the alpha_0 product; rods: the projected gathers of the loop write only
    // the half rates -- recompute U = M D gamma from the final gamma
    if (!spheres) {
      if (int rc = launch_gather_raw(ctx, gfin, 1, mu, nullptr, false)) return rc;
    } else if (stt.iters == 0 && stt.mvops >= 2) {
      if (int rc = mvop_raw(gfin, 1)) return rc;
    }
    if (spheres && ctx->mobility_model == 1) {  // U_c = M D gamma with the coupling blocks (Omega_c)
      if (int rc = ensure(ctx, ctx->ft_tmp, 6 * n)) return rc;
      if (int rc = launch_gather_raw(ctx, gfin, 1, mu, ctx->ft_tmp.p)) return rc;
      if (int rc = launch_pack_ft(ctx, ctx->ft_tmp.p, ctx->f4.p, ctx->t4.p)) return rc;
      if (int rc = rpy6_apply(ctx, ctx->f4.p, ctx->t4.p, mu, dU)) return rc;
    } else if (spheres) {
      if (int rc = launch_unpack_uw_spheres(ctx, ctx->u4.p, nullptr, mu, dU)) return rc;
    } else {
      if (int rc = launch_rod_unpack(ctx, ctx->u4.p, dU)) return rc;
    }
  }
  if (int rc = save_for_warm_start(ctx, gfin)) return rc;
  int32_t* dact = ctx->derr;  // reuse the flag word as a counter
  SC_CUDA(cudaMemsetAsync(dact, 0, sizeof(int32_t), ctx->stream));
  if (int rc = launch_count_active(ctx, gfin, dact)) return rc;
  SC_CUDA(cudaMemcpyAsync(ctx->herr, dact, sizeof(int32_t), cudaMemcpyDeviceToHost, ctx->stream));
  SC_CUDA(cudaMemsetAsync(dact, 0, sizeof(int32_t), ctx->stream));
  if (int rc = st.finish()) return rc;
  SC_CUDA(cudaStreamSynchronize(ctx->stream));
  stt.active = *ctx->herr;
  *ctx->herr = 0;
  if (stats) *stats = stt;
  return rc_final;
}

int sc_collision_step(sc_ctx* ctx, const sc_problem* prob, const sc_bbpgd_opts* opts, double* Fc_out,
                      double* Uc_out, int64_t* n_c, sc_bbpgd_stats* stats) {
  if (ctx == nullptr) return SC_EINVAL;
  if (prob == nullptr || opts == nullptr || !(prob->dt > 0.0) || !(prob->mu > 0.0))
    return fail(ctx, SC_EINVAL, "collision_step: bad arguments");
  int rc;
  int64_t nc = 0;
  if (prob->kind == 0)
    rc = sc_build_contacts_spheres(ctx, prob->n, prob->pos, prob->radius, prob->gap_abs, prob->gap_rel, &nc);
  else
    rc = sc_build_contacts_rods(ctx, prob->n, prob->pos, prob->dir, prob->length, prob->b, prob->gap_abs, &nc);
  if (rc != SC_OK) return rc;
  if ((rc = sc_assemble_D(ctx)) != SC_OK) return rc;
  const int64_t n = prob->n;
  if ((rc = ensure(ctx, ctx->w, 6 * std::max<int64_t>(n, 1)))) return rc;
  rc = sc_mobility_apply(ctx, prob->mu, prob->F_ext, ctx->w.p);  // U_ext = M F_ext (Step 1)
  if (rc == SC_OK) rc = sc_lcp_q(ctx, prob->dt, ctx->w.p, nullptr);
  if (rc != SC_OK) return rc;
  if ((rc = ensure(ctx, ctx->gam_user, std::max<int64_t>(nc, 1)))) return rc;
  sc_bbpgd_opts o = *opts;
  o.mu = prob->mu;
  if (o.warm_start != 2) o.warm_start = 0;  // (1 would need a caller gamma; 2 = previous solve)
  rc = sc_bbpgd_solve(ctx, &o, ctx->gam_user.p, nullptr, Fc_out, Uc_out, stats);
  if (n_c) *n_c = nc;
  return rc;
}

// ------------------------------------------------------------ NEXT row f3: APGD
// Accelerated projected gradient descent (Mazhar et al. 2015, cited at P:L546-L558), the
// comparison solver of the paper's Fig. pairshearBBPGD; readings in DESIGN.md
// (A24): gamma_0 = 0, L_0 = g0.M g0 / g0.g0 (the Cauchy-step Lipschitz estimate, one MVOP like
// BBPGD's Step 6), back-tracking L <- 2L until f(gamma') <= f(y) + g.(gamma'-y) + L/2|gamma'-y|^2,
// Nesterov theta/beta, gradient restart when g.(gamma' - gamma) > 0, L <- 0.9 L after a step,
// stop on the same residual phi = ||min(gamma, g)|| < tol.  One GPU.
int sc_apgd_solve(sc_ctx* ctx, const sc_bbpgd_opts* opts, double* gamma, double* g_out, sc_bbpgd_stats* stats) {
  if (ctx == nullptr) return SC_EINVAL;
  if (opts == nullptr || !(opts->mu > 0.0) || !(opts->tol >= 0.0) || opts->max_iter < 0)
    return fail(ctx, SC_EINVAL, "apgd_solve: bad options");
  if (!ctx->assembled || !ctx->have_q) return fail(ctx, SC_EINVAL, "apgd_solve needs assemble_D and lcp_q first");
  if (ctx->world > 1 || ctx->emul_world > 1) return fail(ctx, SC_EINVAL, "apgd_solve is a 1-GPU comparison solver");
  const int64_t nc = ctx->nc;
  if (nc > 0 && gamma == nullptr) return fail(ctx, SC_EINVAL, "apgd_solve: gamma is NULL");
  cudaSetDevice(ctx->device);
  sc_bbpgd_stats stt;
  std::memset(&stt, 0, sizeof(stt));
  const double mu = opts->mu;
  if (int rc = ensure_rod_mob(ctx, mu)) return rc;
  Stager st(ctx);
  double *dgam = nullptr, *dg = nullptr;
  if (int rc = st.out(gamma, nc, &dgam)) return rc;
  if (int rc = st.out(g_out, nc, &dg)) return rc;
  if (nc == 0) {
    stt.converged = 1;
    if (stats) *stats = stt;
    return st.finish();
  }
  if (int rc = ensure(ctx, ctx->apgd_y, nc)) return rc;
  if (int rc = ensure(ctx, ctx->apgd_sums, 4)) return rc;
  double* x = ctx->gam[0].p;   // gamma_k
  double* xn = ctx->gam[1].p;  // gamma_{k+1}
  double* y = ctx->apgd_y.p;   // extrapolated point
  double* gy = ctx->g[0].p;    // g at y
  double* gn = ctx->g[1].p;    // g at gamma_{k+1}
  const bool spheres = ctx->kind == kSpheres;
  Dist D(ctx);
  double hs[4];
  auto sums = [&](double* out) -> int {
    if (int rc = launch_sum_chunks(ctx, ctx->apgd_sums.p)) return rc;
    SC_CUDA(cudaMemcpyAsync(out, ctx->apgd_sums.p, 4 * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    SC_CUDA(cudaStreamSynchronize(ctx->stream));
    return 0;
  };
  // gout = M v + q; returns (v.Mv, q.v, phi(v)^2)
  auto mvop_grad = [&](const double* v, double* gout, double* out) -> int {
    if (int rc = launch_gather_raw(ctx, v, 1, mu, nullptr)) return rc;
    if (spheres) {
      if (int rc = D.rpy(mu, nullptr)) return rc;
    }
    if (int rc = launch_dt(ctx, 4, 0, v, gout, 0, ctx->nchunks, false)) return rc;
    return sums(out);
  };
  SC_CUDA(cudaMemsetAsync(ctx->dsc, 0, sizeof(DevScalars), ctx->stream));  // done = 0 for the kernels
  // gamma_0 = 0: g_0 = q (the zero-vector MVOP, counted as in BBPGD), phi_0
  SC_CUDA(cudaMemsetAsync(x, 0, nc * sizeof(double), ctx->stream));
  SC_CUDA(cudaMemsetAsync(y, 0, nc * sizeof(double), ctx->stream));
  if (int rc = launch_dt(ctx, 3, 0, x, gy, 0, ctx->nchunks, false)) return rc;
  if (int rc = sums(hs)) return rc;
  stt.mvops = 1;
  double phi = std::sqrt(hs[3]);
  int rc_final = SC_OK;
  if (!(phi < opts->tol)) {
    // L_0 = g0.M g0 / g0.g0: kDtGrad on v = g0 = q gives v.Mv and q.v = |q|^2
    if (int rc = mvop_grad(gy, gn, hs)) return rc;
    stt.mvops = 2;
    double L = hs[0] / hs[1];
    if (!(std::isfinite(L) && L > 0.0)) return fail(ctx, SC_ENONFINITE, "apgd: bad Lipschitz estimate");
    double t = 1.0 / L, theta = 1.0, fy = 0.0;  // f(y_0) = f(0) = 0
    int restarts = 0;
    bool conv = false;
    for (int k = 1; k <= opts->max_iter; ++k) {
      double s[4], fxn = 0.0;
      for (int bt = 0;; ++bt) {  // back-tracking on the local Lipschitz estimate
        if (int rc = apgd_launch_step(ctx, y, gy, x, t, xn)) return rc;
        if (int rc = sums(s)) return rc;
        if (int rc = mvop_grad(xn, gn, hs)) return rc;
        stt.mvops += 1;
        fxn = 0.5 * hs[0] + hs[1];
        const double rhs = fy + s[0] + 0.5 * L * s[1];
        if (fxn <= rhs + 1e-12 * (std::fabs(fxn) + std::fabs(rhs)) || bt >= 60) break;
        L *= 2.0;
        t = 1.0 / L;
      }
      stt.iters = k;
      phi = std::sqrt(hs[2]);
      if (!std::isfinite(phi)) return fail(ctx, SC_ENONFINITE, "apgd: non-finite residual");
      std::swap(x, xn);  // gamma_{k+1} accepted (xn now holds gamma_k)
      std::swap(gy, gn);  // gy <- g(gamma_{k+1}) (kept if the next y is gamma_{k+1})
      if (phi < opts->tol) {
        conv = true;
        break;
      }
      const double theta_n = 0.5 * (-theta * theta + theta * std::sqrt(theta * theta + 4.0));
      const double beta = theta * (1.0 - theta) / (theta * theta + theta_n);
      if (s[2] > 0.0) {  // gradient restart: y = gamma_{k+1}, theta = 1 (g at y already known)
        ++restarts;
        SC_CUDA(cudaMemcpyAsync(y, x, nc * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        fy = fxn;
        theta = 1.0;
      } else {
        if (int rc = apgd_launch_momentum(ctx, x, xn, beta, y)) return rc;
        if (int rc = mvop_grad(y, gy, hs)) return rc;
        stt.mvops += 1;
        fy = 0.5 * hs[0] + hs[1];
        theta = theta_n;
      }
      L *= 0.9;
      t = 1.0 / L;
    }
    stt.bb_breakdowns = restarts;
    stt.alpha = t;
    if (!conv) rc_final = SC_NOT_CONVERGED;
    stt.converged = conv ? 1 : 0;
    // the accepted iterate is x; its gradient: gy if the loop ended on convergence or restart
    // bookkeeping differs -- recompute once for the output (not counted as an MVOP of the method)
    if (int rc = mvop_grad(x, gn, hs)) return rc;
    phi = std::sqrt(hs[2]);
    if (dg) SC_CUDA(cudaMemcpyAsync(dg, gn, nc * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  } else {
    stt.converged = 1;
    if (dg) SC_CUDA(cudaMemcpyAsync(dg, gy, nc * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  }
  stt.residual = phi;
  SC_CUDA(cudaMemcpyAsync(dgam, x, nc * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  if (int rc = st.finish()) return rc;
  SC_CUDA(cudaStreamSynchronize(ctx->stream));
  if (int rc = check_flag(ctx, SC_EDEGENERATE, "coincident centres in the RPY sum")) return rc;
  if (stats) *stats = stt;
  return rc_final;
}

// Step 4: C^{k+1} = C^k + G U dt, quaternion kinematics theta' = Psi Omega
// with renormalisation; rod axes t' = normalize(t + dt Omega x t).
// Same association as the plain definition (explicit round-to-nearest).
__global__ static void euler_update_kernel(const double4* __restrict__ pos4, const double4* __restrict__ dir4,
                                          const double* __restrict__ Unc, const double* __restrict__ Uc,
                                          int64_t n, double dt, double* __restrict__ pos_out,
                                          double* __restrict__ dir_out, double* __restrict__ quat,
                                          double* __restrict__ U_out) {
  const int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= n) return;
  double U[6];
  for (int k = 0; k < 6; ++k) U[k] = __dadd_rn(Unc[6 * b + k], Uc[6 * b + k]);
  if (U_out)
    for (int k = 0; k < 6; ++k) U_out[6 * b + k] = U[k];
  const double4 c = pos4[b];
  pos_out[3 * b + 0] = __dadd_rn(c.x, __dmul_rn(dt, U[0]));
  pos_out[3 * b + 1] = __dadd_rn(c.y, __dmul_rn(dt, U[1]));
  pos_out[3 * b + 2] = __dadd_rn(c.z, __dmul_rn(dt, U[2]));
  const double* W = U + 3;
  if (quat) {
    double* th = quat + 4 * b;
    double s = th[0], px = th[1], py = th[2], pz = th[3];
    // Psi(theta) Omega = 1/2 [ -p.Omega ; s Omega - p x Omega ]
    const double ds = -0.5 * (px * W[0] + py * W[1] + pz * W[2]);
    const double cx = py * W[2] - pz * W[1], cy = pz * W[0] - px * W[2], cz = px * W[1] - py * W[0];
    const double dx = 0.5 * (s * W[0] - cx), dy = 0.5 * (s * W[1] - cy), dz = 0.5 * (s * W[2] - cz);
    s += dt * ds;
    px += dt * dx;
    py += dt * dy;
    pz += dt * dz;
    const double nn = sqrt(s * s + px * px + py * py + pz * pz);
    th[0] = s / nn;
    th[1] = px / nn;
    th[2] = py / nn;
    th[3] = pz / nn;
  }
  if (dir_out) {
    const double4 t = dir4[b];
    const double wx = W[1] * t.z - W[2] * t.y, wy = W[2] * t.x - W[0] * t.z, wz = W[0] * t.y - W[1] * t.x;
    const double ax = t.x + dt * wx, ay = t.y + dt * wy, az = t.z + dt * wz;
    const double nn = sqrt(ax * ax + ay * ay + az * az);
    dir_out[3 * b + 0] = ax / nn;
    dir_out[3 * b + 1] = ay / nn;
    dir_out[3 * b + 2] = az / nn;
  }
}

int sc_time_step(sc_ctx* ctx, const sc_problem* prob, const sc_bbpgd_opts* opts, double* pos_out, double* dir_out,
                 double* quat, double* U_out, int64_t* n_c, sc_bbpgd_stats* stats) {
  if (ctx == nullptr) return SC_EINVAL;
  if (prob == nullptr || (prob->n > 0 && pos_out == nullptr) || (prob->kind == 1 && prob->n > 0 && !dir_out))
    return fail(ctx, SC_EINVAL, "time_step: bad arguments");
  const int64_t n = prob->n;
  if (int rc = ensure(ctx, ctx->uc, 6 * std::max<int64_t>(n, 1))) return rc;
  int rc = sc_collision_step(ctx, prob, opts, nullptr, ctx->uc.p, n_c, stats);  // steps 1-3
  if (rc < 0) return rc;
  if (n == 0) return rc;
  cudaSetDevice(ctx->device);
  Stager st(ctx);
  double *dpos = nullptr, *ddir = nullptr, *dq = nullptr, *dU = nullptr;
  if (int e = st.out(pos_out, 3 * n, &dpos)) return e;
  if (prob->kind == 1) {
    if (int e = st.out(dir_out, 3 * n, &ddir)) return e;
  }
  if (int e = st.inout(quat, 4 * n, &dq)) return e;
  if (int e = st.out(U_out, 6 * n, &dU)) return e;
  timer_begin(ctx, SC_K_MISC);
  euler_update_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(
      ctx->pos4.p, ctx->dir4.p, ctx->w.p, ctx->uc.p, n, prob->dt, dpos, ddir, dq, dU);
  timer_end(ctx, SC_K_MISC);
  if (int e = check_launch(ctx, "euler_update")) return e;
  if (int e = st.finish()) return e;
  SC_CUDA(cudaStreamSynchronize(ctx->stream));
  // moving boundaries advance with their prescribed velocity: h_k' = h_k + dt n_k . V_k
  for (int k = 0; k < ctx->nwalls; ++k) {
    const double4 w = ctx->walls[k];
    const double* v = ctx->wall_vel[k];
    ctx->walls[k].w = w.w + prob->dt * ((w.x * v[0] + w.y * v[1]) + w.z * v[2]);
  }
  return rc;
}

// ------------------------------------------------------------ measurement
int sc_set_timing(sc_ctx* ctx, int enable) {
  if (ctx == nullptr) return SC_EINVAL;
  ctx->timer.enabled = enable != 0;
  return SC_OK;
}
int sc_get_timing(sc_ctx* ctx, int family, double* total_ms, int64_t* launches) {
  if (ctx == nullptr || family < 0 || family >= SC_K_COUNT) return SC_EINVAL;
  cudaSetDevice(ctx->device);
  timer_collect(ctx);
  if (total_ms) *total_ms = ctx->timer.total_ms[family];
  if (launches) *launches = ctx->timer.launches[family];
  return SC_OK;
}
int sc_reset_timing(sc_ctx* ctx) {
  if (ctx == nullptr) return SC_EINVAL;
  timer_collect(ctx);
  for (int f = 0; f < SC_K_COUNT; ++f) {
    ctx->timer.total_ms[f] = 0.0;
    ctx->timer.launches[f] = 0;
  }
  return SC_OK;
}
int64_t sc_launch_count(const sc_ctx* ctx) { return ctx ? ctx->launch_count : -1; }

int sc_set_residual_trace(sc_ctx* ctx, int32_t capacity) {
  if (ctx == nullptr) return SC_EINVAL;
  if (capacity < 0) return fail(ctx, SC_EINVAL, "set_residual_trace: capacity < 0");
  cudaSetDevice(ctx->device);
  if (capacity > 0) {
    if (int rc = ensure(ctx, ctx->trace, static_cast<size_t>(capacity))) return rc;
  }
  ctx->trace_cap = capacity;
  ctx->trace_count = 0;
  return SC_OK;
}

int sc_get_residual_trace(sc_ctx* ctx, double* out, int32_t capacity, int32_t* count) {
  if (ctx == nullptr) return SC_EINVAL;
  if (count == nullptr || capacity < 0 || (capacity > 0 && out == nullptr))
    return fail(ctx, SC_EINVAL, "get_residual_trace: bad arguments");
  cudaSetDevice(ctx->device);
  const int32_t m = std::min(capacity, ctx->trace_count);
  *count = ctx->trace_count;
  if (m == 0) return SC_OK;
  Stager st(ctx);
  double* d = nullptr;
  if (int rc = st.out(out, m, &d)) return rc;
  SC_CUDA(cudaMemcpyAsync(d, ctx->trace.p, m * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  if (int rc = st.finish()) return rc;
  SC_CUDA(cudaStreamSynchronize(ctx->stream));
  return SC_OK;
}

int sc_comm_info(const sc_ctx* ctx, int32_t* out4) {
  if (ctx == nullptr || out4 == nullptr) return SC_EINVAL;
  int nranks = 1, rank = 0, dev = ctx->device, ver = 0;
  if (ctx->comm != nullptr) {
    if (ncclCommCount(ctx->comm, &nranks) != ncclSuccess || ncclCommUserRank(ctx->comm, &rank) != ncclSuccess ||
        ncclCommCuDevice(ctx->comm, &dev) != ncclSuccess)
      return SC_ENCCL;
  }
  ncclGetVersion(&ver);
  out4[0] = nranks;
  out4[1] = rank;
  out4[2] = dev;
  out4[3] = ver;
  return SC_OK;
}

int sc_set_rpy_kernel(sc_ctx* ctx, int mode) {
  if (ctx == nullptr) return SC_EINVAL;
  if (mode < 0 || mode > 2) return fail(ctx, SC_EINVAL, "rpy kernel mode must be 0, 1 or 2");
  ctx->rpy_mode = mode;
  return SC_OK;
}

int sc_set_emulated_world(sc_ctx* ctx, int world) {
  if (ctx == nullptr) return SC_EINVAL;
  if (world < 1 || ctx->world > 1 || ctx->comm != nullptr)
    return fail(ctx, SC_EINVAL, "emulated world needs a 1-GPU context without a communicator and world >= 1");
  ctx->emul_world = world;
  return SC_OK;
}

}  // extern "C"
