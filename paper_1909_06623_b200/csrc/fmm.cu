// fmm.cu -- NEXT row f4(i): a fast O(N) summation of the RPY mobility apply (spheres, FP64).
//
// The paper evaluates its all-to-all operators in O(N) with the kernel-independent FMM (KIFMM,
// P:L888-L896); its accuracy is set by the equivalent-point density (m = 8).  Here the
// BASELINE RPY sum U_i = F_i/(6 pi mu a) + sum_{j != i} T(r_ij) F_j (configs[0]) is evaluated with
// a black-box (Chebyshev-interpolation) FMM on a uniform octree -- the configs are uniform
// suspensions -- in the same spirit: the far field of every well-separated box pair is the RPY far
// branch T(r) = (1/(8 pi mu)) [(1/r + 2a^2/(3r^3)) I + (1/r^3)(1 - 2a^2/r^2) r r^T] evaluated
// between the pseudo-particles at the boxes' Chebyshev nodes, and the near field (the 27 leaves
// around a body, incl. every overlapping pair, r < 2a) is the exact pair sum.  The interpolation
// order n (nodes per dimension) sets the accuracy (measured errors).
//
//   P2M   leaf node strengths  M_B(m) = sum_{j in B} S(m, u_j) F_j            (anterpolation)
//   M2M   parent from children M_P(m') = sum_c sum_m S_P(m', xi_c(m)) M_c(m)   (levels L-1 .. 2)
//   M2L   L_T(m) = sum_{S in IL(T)} sum_n T(x_T(m) - y_S(n)) M_S(n)           (levels 2 .. L)
//   L2L   L_C(m) += sum_m' S_P(m', xi_C(m)) L_P(m')                          (levels 3 .. L)
//   L2P+P2P  U_i = sum_m S(m, u_i) L_B(m) + sum_{j in the 27 leaves around B} T_ij F_j
// S(m, u) = prod_d (1/n + (2/n) sum_{q=1}^{n-1} T_q(xbar_{m_d}) T_q(u_d)) with the Chebyshev nodes
// xbar_k = cos((2k+1) pi / (2n)); IL(T) = the children of the parent's neighbours that are not
// adjacent to T (at most 189).  Every sum is in a fixed order (deterministic).  Polydisperse radii:
// the far branch is split into radius-free kernels (m2l_poly_kernel), 9 node components instead of 3.
// Compressed M2L (default where faster, sc_set_fmm_compression): per level one orthonormal basis U
// of the 316 offset operators K_o (eigenvectors of sum_o K_o K_o^T, cuSOLVER, once per geometry),
// C_o = U^T K_o U, and M2L as class-batched GEMMs L = U sum_o C_o U^T M (cuBLAS: plain GEMMs).
#include <cublas_v2.h>
#include <cub/device/device_radix_sort.cuh>
#include <cusolverDn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "fixed_point.cuh"
#include "rpy_common.cuh"
#include "sc_internal.h"

namespace sc {
namespace {

// Interpolation tables of the three orders, written once per device at context creation (they
// depend on the order only, so every context writes the same bytes): for order n at offset
// tab_off(n): the Chebyshev nodes xbar[n], T_q(xbar_k) at [k * n + q], and the child-parent
// transfer matrices P[sigma][m'][m] = S(xbar_m', (xbar_m + s)/2), s = -1 (sigma 0), +1 (sigma 1).
constexpr int tab_size(int n) { return n + 3 * n * n; }
constexpr int tab_off(int n) { return n == 4 ? 0 : (n == 6 ? tab_size(4) : tab_size(4) + tab_size(6)); }
__constant__ double c_tab[tab_size(4) + tab_size(6) + tab_size(8)];
#define c_xbar (c_tab + tab_off(NN))
#define c_T (c_tab + tab_off(NN) + NN)
#define c_P (c_tab + tab_off(NN) + NN + NN * NN)

#ifndef SC_FMM_P2P_SYM
#define SC_FMM_P2P_SYM 1  // near field by p2p_sym_kernel (each unordered leaf pair once; 0: per target)
#endif

struct Geom {
  double ox, oy, oz;  // root cube corner
  double H;           // root cube side
  double a;           // sphere radius (monodisperse kernels; the polydisperse ones read w = a_i/2)
  int L;              // leaf level
};

__host__ __device__ inline int64_t nbox(int l) { return int64_t(1) << (3 * l); }

// compressed M2L for this context: mode 1 (on), or mode 2 (auto, the default) where it measured
// faster (profiles/r02/fmm_compressed_vs_direct*.jsonl): monodisperse order 8 from N = 2^15, order 6
// from 2^18, order 4 from 2^21; polydisperse order 8 from 2^17, order 6 from 2^20
inline bool fmm_use_svd(const sc_ctx* ctx) {
  if (ctx->fmm_compress == 0) return false;
  if (ctx->fmm_compress == 1) return true;
  if (ctx->poly)  // (polydisperse: 4 compressed products per offset; measured faster from these N)
    return (ctx->fmm_order == 8 && ctx->n >= (int64_t(1) << 17)) || (ctx->fmm_order == 6 && ctx->n >= (int64_t(1) << 20));
  return (ctx->fmm_order == 8 && ctx->n >= (int64_t(1) << 15)) || (ctx->fmm_order == 6 && ctx->n >= (int64_t(1) << 18)) ||
         (ctx->fmm_order == 4 && ctx->n >= (int64_t(1) << 21));
}

// 1-D interpolation weights w[k] = S_n(xbar_k, u), u in [-1, 1]
template <int NN>
__device__ __forceinline__ void cheb_w(double u, double w[NN]) {
  double T[NN];
  T[0] = 1.0;
  if (NN > 1) T[1] = u;
#pragma unroll
  for (int q = 2; q < NN; ++q) T[q] = 2.0 * u * T[q - 1] - T[q - 2];
#pragma unroll
  for (int k = 0; k < NN; ++k) {
    double s = 0.0;
#pragma unroll
    for (int q = 1; q < NN; ++q) s = fma(c_T[k * NN + q], T[q], s);
    w[k] = (1.0 + 2.0 * s) / NN;
  }
}

// RPY far branch (scaled by 8 pi mu): acc += c1 f + c2 (d.f) d, d = y - x
__device__ __forceinline__ void far_pair(double dx, double dy, double dz, double fx, double fy, double fz,
                                         double a2, double& ax, double& ay, double& az) {
  const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
  const double y = rsqrt_dp(r2);
  const double h = y * y, e = y * h;
  const double c1 = fma(2.0 / 3.0 * a2, e, y);
  const double c2 = e * fma(-2.0 * a2, h, 1.0) * fma(dz, fz, fma(dy, fy, dx * fx));
  ax = fma(c2, dx, fma(c1, fx, ax));
  ay = fma(c2, dy, fma(c1, fy, ay));
  az = fma(c2, dz, fma(c1, fz, az));
}

__device__ __forceinline__ void box_center(const Geom& g, int l, int64_t bi, double& cx, double& cy, double& cz,
                                           double& w) {
  const int D = 1 << l;
  const int ix = static_cast<int>(bi % D), iy = static_cast<int>((bi / D) % D), iz = static_cast<int>(bi / D / D);
  const double h = g.H / D;
  w = 0.5 * h;
  cx = g.ox + h * (ix + 0.5);
  cy = g.oy + h * (iy + 0.5);
  cz = g.oz + h * (iz + 0.5);
}

__global__ void leaf_of_kernel(const double4* __restrict__ pos4, int64_t n, Geom g, uint32_t* __restrict__ key,
                               int32_t* __restrict__ idx, int32_t* __restrict__ cnt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int D = 1 << g.L;
  const double h = g.H / D;
  const double4 p = pos4[i];
  int ix = static_cast<int>(floor((p.x - g.ox) / h)), iy = static_cast<int>(floor((p.y - g.oy) / h)),
      iz = static_cast<int>(floor((p.z - g.oz) / h));
  ix = min(max(ix, 0), D - 1);
  iy = min(max(iy, 0), D - 1);
  iz = min(max(iz, 0), D - 1);
  const uint32_t b = static_cast<uint32_t>((iz * D + iy) * D + ix);
  key[i] = b;
  idx[i] = static_cast<int32_t>(i);
  atomicAdd(&cnt[b], 1);
}

__global__ void gather_sorted_kernel(const int32_t* __restrict__ sidx, int64_t n, const double4* __restrict__ src,
                                     double4* __restrict__ dst) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  dst[k] = src[sidx[k]];
}

// P2M: one CTA per leaf, thread m = node (blockDim >= n^3).  C = 3 (monodisperse: the node
// strengths of F) or 9 (polydisperse: of the three source densities F, w F, w^2 F, w = a/2; see
// m2l_poly_kernel).
template <int NN, int C>
__global__ void p2m_kernel(const double4* __restrict__ spos, const double4* __restrict__ sf,
                           const int32_t* __restrict__ lstart, Geom g, double* __restrict__ M,
                           const int32_t* __restrict__ done) {
  if (done != nullptr && *done) return;
  constexpr int NB = NN * NN * NN;
  constexpr int CH = 64;
  __shared__ double sw[CH][3][NN];
  __shared__ double sfrc[CH][C];
  const int64_t b = blockIdx.x;
  double cx, cy, cz, w;
  box_center(g, g.L, b, cx, cy, cz, w);
  const int32_t j0 = lstart[b], j1 = lstart[b + 1];
  const int m = threadIdx.x;
  const int mx = m % NN, my = (m / NN) % NN, mz = m / (NN * NN);
  double acc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c] = 0.0;
  for (int32_t c0 = j0; c0 < j1; c0 += CH) {
    const int cn = min(CH, j1 - c0);
    __syncthreads();
    for (int t = threadIdx.x; t < 3 * cn; t += blockDim.x) {
      const int jj = t / 3, d = t % 3;
      const double4 p = spos[c0 + jj];
      const double x = d == 0 ? p.x - cx : (d == 1 ? p.y - cy : p.z - cz);
      double u = x / w;
      u = fmin(1.0, fmax(-1.0, u));
      double ww[NN];
      cheb_w<NN>(u, ww);
#pragma unroll
      for (int k = 0; k < NN; ++k) sw[jj][d][k] = ww[k];
      if (d == 0) {
        const double4 f = sf[c0 + jj];
        sfrc[jj][0] = f.x;
        sfrc[jj][1] = f.y;
        sfrc[jj][2] = f.z;
        if constexpr (C == 9) {
          const double hw = p.w, hw2 = p.w * p.w;
          sfrc[jj][3] = hw * f.x;
          sfrc[jj][4] = hw * f.y;
          sfrc[jj][5] = hw * f.z;
          sfrc[jj][6] = hw2 * f.x;
          sfrc[jj][7] = hw2 * f.y;
          sfrc[jj][8] = hw2 * f.z;
        }
      }
    }
    __syncthreads();
    if (m < NB) {
      for (int jj = 0; jj < cn; ++jj) {
        const double s = sw[jj][0][mx] * sw[jj][1][my] * sw[jj][2][mz];
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c] = fma(s, sfrc[jj][c], acc[c]);
      }
    }
  }
  if (m < NB) {
    double* o = M + (b * NB + m) * C;
#pragma unroll
    for (int c = 0; c < C; ++c) o[c] = acc[c];
  }
}

// M2M (child level l+1 -> parent level l) and L2L (parent l -> children l+1): the 1-D transfer
// matrices c_P of the child's position sigma in its parent; C components per node.
template <int NN, bool UP, int C>
__global__ void transfer_kernel(int l, double* __restrict__ Xp, double* __restrict__ Xc,
                                const int32_t* __restrict__ done) {
  if (done != nullptr && *done) return;
  constexpr int NB = NN * NN * NN;
  __shared__ double s[NB * C];
  const int m = threadIdx.x;
  const int mx = m % NN, my = (m / NN) % NN, mz = m / (NN * NN);
  double acc[C];
#pragma unroll
  for (int c = 0; c < C; ++c) acc[c] = 0.0;
  if (UP) {  // parent box blockIdx.x at level l: sum over its 8 children
    const int D = 1 << l;
    const int64_t p = blockIdx.x;
    const int px = static_cast<int>(p % D), py = static_cast<int>((p / D) % D), pz = static_cast<int>(p / D / D);
    for (int c = 0; c < 8; ++c) {
      const int sx = c & 1, sy = (c >> 1) & 1, sz = c >> 2;
      const int64_t ci = ((2 * pz + sz) * (2 * D) + (2 * py + sy)) * (2 * D) + (2 * px + sx);
      __syncthreads();
      for (int t = threadIdx.x; t < C * NB; t += blockDim.x) s[t] = Xc[ci * NB * C + t];
      __syncthreads();
      if (m < NB) {
        const double* Px = c_P + sx * NN * NN + mx * NN;
        const double* Py = c_P + sy * NN * NN + my * NN;
        const double* Pz = c_P + sz * NN * NN + mz * NN;
        for (int kz = 0; kz < NN; ++kz)
          for (int ky = 0; ky < NN; ++ky) {
            const double pyz = Py[ky] * Pz[kz];
#pragma unroll
            for (int kx = 0; kx < NN; ++kx) {
              const double wgt = Px[kx] * pyz;
              const double* v = s + ((kz * NN + ky) * NN + kx) * C;
#pragma unroll
              for (int q = 0; q < C; ++q) acc[q] = fma(wgt, v[q], acc[q]);
            }
          }
      }
    }
    if (m < NB) {
      double* o = Xp + (p * NB + m) * C;
#pragma unroll
      for (int q = 0; q < C; ++q) o[q] = acc[q];
    }
  } else {  // child box blockIdx.x at level l+1: add its parent's local expansion at its nodes
    const int D = 2 << l;
    const int64_t c = blockIdx.x;
    const int cx = static_cast<int>(c % D), cy = static_cast<int>((c / D) % D), cz = static_cast<int>(c / D / D);
    const int64_t pi = ((cz / 2) * (D / 2) + cy / 2) * (D / 2) + cx / 2;
    for (int t = threadIdx.x; t < C * NB; t += blockDim.x) s[t] = Xp[pi * NB * C + t];
    __syncthreads();
    if (m < NB) {
      const int sx = cx & 1, sy = cy & 1, sz = cz & 1;
      for (int kz = 0; kz < NN; ++kz)
        for (int ky = 0; ky < NN; ++ky) {
          const double pyz = c_P[sy * NN * NN + ky * NN + my] * c_P[sz * NN * NN + kz * NN + mz];
#pragma unroll
          for (int kx = 0; kx < NN; ++kx) {
            const double wgt = c_P[sx * NN * NN + kx * NN + mx] * pyz;
            const double* v = s + ((kz * NN + ky) * NN + kx) * C;
#pragma unroll
            for (int q = 0; q < C; ++q) acc[q] = fma(wgt, v[q], acc[q]);
          }
        }
      double* o = Xc + (c * NB + m) * C;
#pragma unroll
      for (int q = 0; q < C; ++q) o[q] += acc[q];
    }
  }
}

// M2L: one CTA per target box (all levels 2..L: blockIdx.x over the concatenated levels),
// thread m = target node; the source boxes of the interaction list in a fixed order.
template <int NN>
__global__ void m2l_kernel(Geom g, const int64_t* __restrict__ lev_off /* box offset of level l */,
                           const double* __restrict__ M, double* __restrict__ Lc, const int32_t* __restrict__ done) {
  if (done != nullptr && *done) return;
  constexpr int NB = NN * NN * NN;
  __shared__ double4 sy[NB];  // source node positions
  __shared__ double4 sm[NB];  // source node strengths
  int64_t gb = blockIdx.x;
  int l = 2;
  while (l < g.L && gb >= lev_off[l + 1] - lev_off[2]) ++l;
  const int64_t t = gb - (lev_off[l] - lev_off[2]);
  const int D = 1 << l;
  const int tx = static_cast<int>(t % D), ty = static_cast<int>((t / D) % D), tz = static_cast<int>(t / D / D);
  double cx, cy, cz, w;
  box_center(g, l, t, cx, cy, cz, w);
  const int m = threadIdx.x;
  const int mx = m % NN, my = (m / NN) % NN, mz = m / (NN * NN);
  const double x = cx + w * c_xbar[mx], y = cy + w * c_xbar[my], z = cz + w * c_xbar[mz];
  const double a2 = g.a * g.a;
  double ax = 0, ay = 0, az = 0;
  const int px = tx >> 1, py = ty >> 1, pz = tz >> 1, Dp = D >> 1;
  for (int oz = -1; oz <= 1; ++oz)
    for (int oy = -1; oy <= 1; ++oy)
      for (int ox = -1; ox <= 1; ++ox) {
        const int qx = px + ox, qy = py + oy, qz = pz + oz;
        if (qx < 0 || qy < 0 || qz < 0 || qx >= Dp || qy >= Dp || qz >= Dp) continue;
        for (int c = 0; c < 8; ++c) {
          const int sx = 2 * qx + (c & 1), sy_ = 2 * qy + ((c >> 1) & 1), sz = 2 * qz + (c >> 2);
          if (abs(sx - tx) <= 1 && abs(sy_ - ty) <= 1 && abs(sz - tz) <= 1) continue;  // adjacent: near
          const int64_t s = (static_cast<int64_t>(sz) * D + sy_) * D + sx;
          double scx, scy, scz, sw;
          box_center(g, l, s, scx, scy, scz, sw);
          __syncthreads();
          for (int q = threadIdx.x; q < NB; q += blockDim.x) {
            const int qx_ = q % NN, qy_ = (q / NN) % NN, qz_ = q / (NN * NN);
            sy[q] = make_double4(scx + sw * c_xbar[qx_], scy + sw * c_xbar[qy_], scz + sw * c_xbar[qz_], 0.0);
            const double* v = M + ((lev_off[l] + s) * NB + q) * 3;
            sm[q] = make_double4(v[0], v[1], v[2], 0.0);
          }
          __syncthreads();
          if (m < NB) {
#pragma unroll 4
            for (int q = 0; q < NB; ++q) {
              const double4 p = sy[q], f = sm[q];
              far_pair(p.x - x, p.y - y, p.z - z, f.x, f.y, f.z, a2, ax, ay, az);
            }
          }
        }
      }
  if (m < NB) {
    double* o = Lc + ((lev_off[l] + t) * NB + m) * 3;
    o[0] = ax;
    o[1] = ay;
    o[2] = az;
  }
}

// Polydisperse M2L.  The far branch with the pair radius abar = w_i + w_j (w = a/2) splits as
//   T(r; abar) = O(r) + abar^2 D(r),  O = (1/r) I + (1/r^3) d d^T,  D = (2/3)(1/r^3) I - 2 (1/r^5) d d^T
// (8 pi mu hoisted), and abar^2 = w_i^2 + 2 w_i w_j + w_j^2, so with the source densities
// s0 = F, s1 = w F, s2 = w^2 F (the 9 node components of p2m_kernel<NN, 9>) every target field is
//   U_i = L_A + 2 w_i L_B + w_i^2 L_C,  L_A = sum O s0 + D s2,  L_B = sum D s1,  L_C = sum D s0,
// three fields of smooth kernels that the interpolation carries like the monodisperse one
// (l2p_p2p_kernel<NN, true> forms U_i).  Source node positions from the nested loop (no table).
template <int NN>
__global__ void m2l_poly_kernel(Geom g, const int64_t* __restrict__ lev_off, const double* __restrict__ M,
                                double* __restrict__ Lc, const int32_t* __restrict__ done) {
  if (done != nullptr && *done) return;
  constexpr int NB = NN * NN * NN;
  __shared__ double sm[NB * 9];
  int64_t gb = blockIdx.x;
  int l = 2;
  while (l < g.L && gb >= lev_off[l + 1] - lev_off[2]) ++l;
  const int64_t t = gb - (lev_off[l] - lev_off[2]);
  const int D = 1 << l;
  const int tx = static_cast<int>(t % D), ty = static_cast<int>((t / D) % D), tz = static_cast<int>(t / D / D);
  double cx, cy, cz, w;
  box_center(g, l, t, cx, cy, cz, w);
  const int m = threadIdx.x;
  const int mx = m % NN, my = (m / NN) % NN, mz = m / (NN * NN);
  const double x = cx + w * c_xbar[mx], y = cy + w * c_xbar[my], z = cz + w * c_xbar[mz];
  double A[3] = {0, 0, 0}, B[3] = {0, 0, 0}, Cc[3] = {0, 0, 0};
  const int px = tx >> 1, py = ty >> 1, pz = tz >> 1, Dp = D >> 1;
  for (int oz = -1; oz <= 1; ++oz)
    for (int oy = -1; oy <= 1; ++oy)
      for (int ox = -1; ox <= 1; ++ox) {
        const int qx = px + ox, qy = py + oy, qz = pz + oz;
        if (qx < 0 || qy < 0 || qz < 0 || qx >= Dp || qy >= Dp || qz >= Dp) continue;
        for (int c = 0; c < 8; ++c) {
          const int sx = 2 * qx + (c & 1), sy_ = 2 * qy + ((c >> 1) & 1), sz = 2 * qz + (c >> 2);
          if (abs(sx - tx) <= 1 && abs(sy_ - ty) <= 1 && abs(sz - tz) <= 1) continue;  // adjacent: near
          const int64_t s = (static_cast<int64_t>(sz) * D + sy_) * D + sx;
          double scx, scy, scz, sw;
          box_center(g, l, s, scx, scy, scz, sw);
          __syncthreads();
          const double* src = M + (lev_off[l] + s) * NB * 9;
          for (int q = threadIdx.x; q < NB * 9; q += blockDim.x) sm[q] = src[q];
          __syncthreads();
          if (m < NB) {
            const double* v = sm;
            for (int qz_ = 0; qz_ < NN; ++qz_) {
              const double dz = (scz + sw * c_xbar[qz_]) - z;
              for (int qy_ = 0; qy_ < NN; ++qy_) {
                const double dy = (scy + sw * c_xbar[qy_]) - y;
#pragma unroll 2
                for (int qx_ = 0; qx_ < NN; ++qx_, v += 9) {
                  const double dx = (scx + sw * c_xbar[qx_]) - x;
                  const double r2 = fma(dz, dz, fma(dy, dy, dx * dx));
                  const double yr = rsqrt_dp(r2);
                  const double h = yr * yr, e = yr * h;
                  const double d1 = (2.0 / 3.0) * e, d2 = -2.0 * e * h;  // D: c1, c2
                  const double p0 = fma(dz, v[2], fma(dy, v[1], dx * v[0]));
                  const double p1 = fma(dz, v[5], fma(dy, v[4], dx * v[3]));
                  const double p2 = fma(dz, v[8], fma(dy, v[7], dx * v[6]));
                  const double ta = fma(e, p0, d2 * p2), tb = d2 * p1, tc = d2 * p0;
                  A[0] = fma(ta, dx, fma(yr, v[0], fma(d1, v[6], A[0])));
                  A[1] = fma(ta, dy, fma(yr, v[1], fma(d1, v[7], A[1])));
                  A[2] = fma(ta, dz, fma(yr, v[2], fma(d1, v[8], A[2])));
                  B[0] = fma(tb, dx, fma(d1, v[3], B[0]));
                  B[1] = fma(tb, dy, fma(d1, v[4], B[1]));
                  B[2] = fma(tb, dz, fma(d1, v[5], B[2]));
                  Cc[0] = fma(tc, dx, fma(d1, v[0], Cc[0]));
                  Cc[1] = fma(tc, dy, fma(d1, v[1], Cc[1]));
                  Cc[2] = fma(tc, dz, fma(d1, v[2], Cc[2]));
                }
              }
            }
          }
        }
      }
  if (m < NB) {
    double* o = Lc + ((lev_off[l] + t) * NB + m) * 9;
    for (int k = 0; k < 3; ++k) {
      o[k] = A[k];
      o[3 + k] = B[k];
      o[6 + k] = Cc[k];
    }
  }
}

// ---- compressed M2L (sc_set_fmm_compression; monodisperse) ---------------------------------
// Offsets o of a source box relative to its target box at one level: o in [-3, 3]^3 with
// max |o_d| >= 2 (316 of the 7^3 grid; index oi = ((oz+3) 7 + oy+3) 7 + ox+3).  K_o is the
// 3n^3 x 3n^3 matrix of the RPY far branch (8 pi mu hoisted) between the target nodes w xi_m and
// the source nodes 2 w o + w xi_n, row (m, alpha) = 3m + alpha, column (n, beta) = 3n + beta --
// the layout of one box's node strengths / local expansion in M and L.
constexpr int kOffGrid = 343, kOffCount = 316;

// K for q offsets (oi list), column-major with leading dimension R = 3 n^3:
// K[(c R + col) R + row], c = 0..q-1.
// kind 0: the monodisperse far branch T (radius^2 a2); 1: its Oseen part O = (1/r) I + (1/r^3) d d^T;
// 2: its radius part D = (2/3)(1/r^3) I - 2 (1/r^5) d d^T (polydisperse: T = O + abar^2 D)
template <int NN>
__global__ void svd_build_k_kernel(double* __restrict__ K, const int32_t* __restrict__ ois, int q, double w,
                                   double a2, int kind) {
  constexpr int NB = NN * NN * NN, R = 3 * NB;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<int64_t>(R) * R * q) return;
  const int row = static_cast<int>(t % R);
  const int64_t cc = t / R;  // c R + col
  const int col = static_cast<int>(cc % R), c = static_cast<int>(cc / R);
  const int oi = ois[c];
  const int ox = oi % 7 - 3, oy = (oi / 7) % 7 - 3, oz = oi / 49 - 3;
  const int m = row / 3, al = row % 3, nn = col / 3, be = col % 3;
  const int mx = m % NN, my = (m / NN) % NN, mz = m / (NN * NN);
  const int nx = nn % NN, ny = (nn / NN) % NN, nz = nn / (NN * NN);
  const double d[3] = {w * (2.0 * ox + c_xbar[nx] - c_xbar[mx]), w * (2.0 * oy + c_xbar[ny] - c_xbar[my]),
                       w * (2.0 * oz + c_xbar[nz] - c_xbar[mz])};
  const double r2 = fma(d[2], d[2], fma(d[1], d[1], d[0] * d[0]));
  const double y = 1.0 / sqrt(r2), h = y * y, e = y * h;
  double c1, c2;
  if (kind == 0) {
    c1 = fma(2.0 / 3.0 * a2, e, y);
    c2 = e * fma(-2.0 * a2, h, 1.0);
  } else if (kind == 1) {
    c1 = y;
    c2 = e;
  } else {
    c1 = (2.0 / 3.0) * e;
    c2 = -2.0 * e * h;
  }
  K[t] = (al == be ? c1 : 0.0) + c2 * d[al] * d[be];
}

// L^c_T = sum_{o in IL(T)} C_o M^c_{T+o} at one level as one GEMM per parity class.  Boxes
// T = 2P + p of class p (parent P in [0, Dp)^3) see the offsets o_d in [-2 - p_d, 3 - p_d], not
// all |o_d| <= 1; the source S = T + o has class p' = (p + o) mod 2 and parent P + delta,
// delta = floor((p + o) / 2) in {-1, 0, 1}^3.  With every class's M^c stored over its parents
// padded by one zero parent on each side ((Dp+2)^3 columns of k values: McP), the sources of all
// targets of a class for one o are the target columns shifted by the constant delta_lin -- so the
// class's L^c is a plain GEMM [k x k] x [k x columns] accumulated over its 189 offsets (K dimension
// 189 k), computed here by a register-tiled FP64 kernel (64 x 64 tile, 4 x 4 per thread, K steps
// of 16 through shared memory).  Columns = the span of interior parents in the padded numbering;
// halo columns are computed and dropped.  Fixed order over o and k -> deterministic.
constexpr int kGbm = 64, kGbn = 64, kGbk = 16;
__global__ void __launch_bounds__(256) m2l_svd_gemm_kernel(int Dp, int k, const double* __restrict__ Cops,
                                                           const int32_t* __restrict__ li_of_oi,
                                                           const double* __restrict__ McP,
                                                           double* __restrict__ LcP, const int32_t* __restrict__ done) {
  if (done != nullptr && *done) return;
  __shared__ double sA[kGbk][kGbm];
  __shared__ double sB[kGbk][kGbn];
  const int pc = static_cast<int>(blockIdx.z);
  const int pxb = pc & 1, pyb = (pc >> 1) & 1, pzb = pc >> 2;
  const int Dq = Dp + 2;
  const int64_t npad = static_cast<int64_t>(Dq) * Dq * Dq;
  const int64_t cbeg = (static_cast<int64_t>(1) * Dq + 1) * Dq + 1;  // parent (1,1,1)
  const int64_t cend = (static_cast<int64_t>(Dp) * Dq + Dp) * Dq + Dp + 1;
  const int64_t col0 = cbeg + static_cast<int64_t>(blockIdx.x) * kGbn;
  const int row0 = static_cast<int>(blockIdx.y) * kGbm;
  const int tid = threadIdx.x, tr = tid >> 4, tc = tid & 15;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int oz = -2 - pzb; oz <= 3 - pzb; ++oz)
    for (int oy = -2 - pyb; oy <= 3 - pyb; ++oy)
      for (int ox = -2 - pxb; ox <= 3 - pxb; ++ox) {
        if (abs(ox) <= 1 && abs(oy) <= 1 && abs(oz) <= 1) continue;
        const int li = li_of_oi[((oz + 3) * 7 + oy + 3) * 7 + ox + 3];
        const int qx = pxb + ox, qy = pyb + oy, qz = pzb + oz;  // in [-2, 3]
        const int spc = (qx & 1) | ((qy & 1) << 1) | ((qz & 1) << 2);
        const int dx = (qx - (qx & 1)) / 2, dy = (qy - (qy & 1)) / 2, dz = (qz - (qz & 1)) / 2;
        const int64_t dl = (static_cast<int64_t>(dz) * Dq + dy) * Dq + dx;
        const double* A = Cops + static_cast<int64_t>(li) * k * k;
        const double* B = McP + static_cast<int64_t>(spc) * npad * k;
        for (int j0 = 0; j0 < k; j0 += kGbk) {
          __syncthreads();
#pragma unroll
          for (int t = 0; t < 4; ++t) {  // A tile: (row, j) = C[j k + row], row fastest
            const int e = tid + t * 256;
            const int r = e % kGbm, jj = e / kGbm;
            const int gr = row0 + r, gj = j0 + jj;
            sA[jj][r] = (gr < k && gj < k) ? __ldg(A + static_cast<int64_t>(gj) * k + gr) : 0.0;
          }
#pragma unroll
          for (int t = 0; t < 4; ++t) {  // B tile: (j, col) = McP[(col + dl) k + j], j fastest
            const int e = tid + t * 256;
            const int jj = e % kGbk, c = e / kGbk;
            const int gj = j0 + jj;
            const int64_t gc = col0 + c;
            sB[jj][c] = (gj < k && gc < cend) ? __ldg(B + (gc + dl) * k + gj) : 0.0;
          }
          __syncthreads();
#pragma unroll
          for (int jj = 0; jj < kGbk; ++jj) {
            double a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              a[u] = sA[jj][tr * 4 + u];
              b[u] = sB[jj][tc * 4 + u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
          }
        }
      }
  // interior columns only
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    const int64_t gc = col0 + tc * 4 + v;
    if (gc >= cend) continue;
    const int px = static_cast<int>(gc % Dq), py = static_cast<int>((gc / Dq) % Dq), pz = static_cast<int>(gc / Dq / Dq);
    if (px < 1 || py < 1 || pz < 1 || px > Dp || py > Dp || pz > Dp) continue;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int r = row0 + tr * 4 + u;
      if (r < k) LcP[(static_cast<int64_t>(pc) * npad + gc) * k + r] = acc[u][v];
    }
  }
}

// polydisperse node strengths [box][node][9] = (s0, s1, s2) <-> three channels [c][box][node][3]
__global__ void svd_poly_split_kernel(int64_t nvals /* nbox NB */, const double* __restrict__ M9,
                                      double* __restrict__ S) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nvals * 9) return;
  const int64_t node = t / 9;
  const int c = static_cast<int>(t % 9) / 3, a = static_cast<int>(t % 3);
  S[(c * nvals + node) * 3 + a] = M9[t];
}
__global__ void svd_poly_merge_kernel(int64_t nvals, const double* __restrict__ S, double* __restrict__ L9) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nvals * 9) return;
  const int64_t node = t / 9;
  const int c = static_cast<int>(t % 9) / 3, a = static_cast<int>(t % 3);
  L9[t] = S[(c * nvals + node) * 3 + a];
}

// natural box order (k x nbox, box T = (z D + y) D + x) <-> class-padded order (McP layout)
__global__ void svd_to_classes_kernel(int D, int k, const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nb = static_cast<int64_t>(D) * D * D;
  if (t >= nb * k) return;
  const int j = static_cast<int>(t % k);
  const int64_t T = t / k;
  const int x = static_cast<int>(T % D), y = static_cast<int>((T / D) % D), z = static_cast<int>(T / D / D);
  const int Dp = D / 2, Dq = Dp + 2;
  const int pc = (x & 1) | ((y & 1) << 1) | ((z & 1) << 2);
  const int64_t col = ((static_cast<int64_t>(z / 2 + 1)) * Dq + (y / 2 + 1)) * Dq + (x / 2 + 1);
  dst[(static_cast<int64_t>(pc) * Dq * Dq * Dq + col) * k + j] = src[T * k + j];
}
__global__ void svd_from_classes_kernel(int D, int k, const double* __restrict__ src, double* __restrict__ dst) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nb = static_cast<int64_t>(D) * D * D;
  if (t >= nb * k) return;
  const int j = static_cast<int>(t % k);
  const int64_t T = t / k;
  const int x = static_cast<int>(T % D), y = static_cast<int>((T / D) % D), z = static_cast<int>(T / D / D);
  const int Dp = D / 2, Dq = Dp + 2;
  const int pc = (x & 1) | ((y & 1) << 1) | ((z & 1) << 2);
  const int64_t col = ((static_cast<int64_t>(z / 2 + 1)) * Dq + (y / 2 + 1)) * Dq + (x / 2 + 1);
  dst[T * k + j] = src[(static_cast<int64_t>(pc) * Dq * Dq * Dq + col) * k + j];
}

// L2P + P2P: one CTA per leaf; thread = target body (chunks of blockDim); sources of the 27
// neighbouring leaves through shared memory (exact RPY incl. the overlap branch and the self term).
// POLY: the leaf's 9-component local expansion (m2l_poly_kernel) and the pair radius w_i + w_j.
// ---- symmetric near field (default): each unordered leaf pair once --------------------------
// The exact pair sum over the 27 leaves around a body is symmetric (T_ij = T_ji), so the pairs
// between leaf b and the 13 neighbours q in the "forward" half-space (plus b itself) are
// evaluated once and feed both bodies: U_i += T F_j (forward, in registers) and U_j += T F_i
// (reverse, the warp-rotation of rpy.cu's symmetric kernel: lane l meets source (l + s) mod 32 at
// step s and carries that source's accumulator, passed on by one shuffle per step).  Every
// partial sum is added as 128-bit fixed point (fixed_point.cuh) -- exact, order-independent --
// and the L2P kernel adds the limbs.  CTA: (leaf b, neighbour index f in 0..13, chunk of 128
// targets of b); 4 warps x 32 targets; sources of q in chunks of 128 through shared memory.
// f = 0 (b itself): every ordered pair, forward only.
__global__ void fmm_fx_prep_kernel(const double4* __restrict__ spos, const double4* __restrict__ sf, int64_t n,
                                   FxScale* __restrict__ fs, const int32_t* __restrict__ done) {
  if (done != nullptr && *done) return;
  double mf = 0.0, mi = 0.0;
  for (int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b < n;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double4 f = sf[b];
    mf = fmax(mf, fmax(fabs(f.x), fmax(fabs(f.y), fabs(f.z))));
    mi = fmax(mi, 0.5 / spos[b].w);  // w = a/2 (abar >= a_min)
  }
  if (!(mf <= 1.7e308)) mf = 1.7e308;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    mf = fmax(mf, __shfl_xor_sync(0xffffffffu, mf, o));
    mi = fmax(mi, __shfl_xor_sync(0xffffffffu, mi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&fs->maxf_bits, static_cast<unsigned long long>(__double_as_longlong(mf)));
    atomicMax(&fs->maxinva_bits, static_cast<unsigned long long>(__double_as_longlong(mi)));
  }
}

// The far-branch coefficients at the high-word-clamped r^2 (rpy_common.cuh) -- branch-free: a pair
// in the overlap branch (r < 2 abar) gets a bounded far value here, which the L2P kernel swaps for
// the overlap branch from the contacts' near list (the same arithmetic as rpy_far_clamped_contrib).
template <bool POLY>
__device__ __forceinline__ void clamped_far_coefs(const double4& pi, const double4& pj, double a2, int tau_hi,
                                                  double& dx, double& dy, double& dz, double& c1, double& c2) {
  const double r2 = rpy_r2(pi, pj, dx, dy, dz);
  double ab2 = a2;
  int th = tau_hi;
  if (POLY) {
    const double ab = pi.w + pj.w;
    ab2 = ab * ab;
    th = rpy_tau_hi(ab2);
  }
  const double r2c = rpy_clamp_r2(r2, th);
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2c));
  double h = r2c * y;
  double e = fma(-h, y, 1.0);
  h = fma(0.375, e, 0.5);
  e = y * e;
  y = fma(e, h, y);
  h = y * y;
  e = y * h;
  const double sc = ab2 * h;
  c1 = y * fma(sc, 2.0 / 3.0, 1.0);
  c2 = e * fma(sc, -2.0, 1.0);
}

// TPT targets per lane (each source load and shuffle serves TPT pairs): 2 for leaves of >= 192
// bodies on average, 1 for smaller leaves (fewer idle lanes) -- fmm_launch picks it.
template <bool POLY, int TPT>
__global__ void __launch_bounds__(128) p2p_sym_kernel(const double4* __restrict__ spos, const double4* __restrict__ sf,
                                                      const int32_t* __restrict__ lstart, Geom g,
                                                      long long* __restrict__ acc, FxScale* __restrict__ fs,
                                                      int64_t fx_count, int32_t* __restrict__ err,
                                                      const int32_t* __restrict__ done) {
  if (done != nullptr && *done) return;
  constexpr int TS = 128, TT = TS * TPT;  // sources per chunk, targets per CTA
  __shared__ double4 sp[TS], sfs[TS];
  __shared__ double rev[4][TS][3];
  const int64_t b = blockIdx.x;
  const int f = static_cast<int>(blockIdx.y);
  const int D = 1 << g.L;
  const int bx = static_cast<int>(b % D), by = static_cast<int>((b / D) % D), bz = static_cast<int>(b / D / D);
  // forward neighbour f: 0 = b; 1..13 = the half-space (oz > 0) | (oz = 0, oy > 0) | (0, 0, ox > 0)
  int ox = 0, oy = 0, oz = 0;
  if (f > 0) {
    int c = 0;
    for (int z = 0; z <= 1 && c < f; ++z)
      for (int y = -1; y <= 1 && c < f; ++y)
        for (int x = -1; x <= 1 && c < f; ++x) {
          const bool fwd = z > 0 || (y > 0) || (y == 0 && x > 0);
          if (!fwd) continue;
          if (++c == f) {
            ox = x;
            oy = y;
            oz = z;
          }
        }
  }
  const int qx = bx + ox, qy = by + oy, qz = bz + oz;
  if (qx < 0 || qy < 0 || qz < 0 || qx >= D || qy >= D || qz >= D) return;  // (uniform in the CTA)
  const int64_t q = (static_cast<int64_t>(qz) * D + qy) * D + qx;
  const int32_t i0 = lstart[b] + static_cast<int32_t>(blockIdx.z) * TT, i1 = min(lstart[b + 1], i0 + TT);
  if (i0 >= i1) return;
  const int32_t j0 = lstart[q], j1 = lstart[q + 1];
  if (j0 >= j1) return;
  const double a2 = g.a * g.a;
  const int tau_hi = rpy_tau_hi(a2);  // (monodisperse)
  const double scale = pow2(fx_shift(fs, fx_count));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // targets of this lane: i0 + w 32 TPT + m 32 + lane, m < TPT
  int32_t ti[TPT];
  bool tval[TPT];
  double4 pi[TPT], fi[TPT];
  double u[TPT][3];
#pragma unroll
  for (int m = 0; m < TPT; ++m) {
    ti[m] = i0 + w * 32 * TPT + m * 32 + lane;
    tval[m] = ti[m] < i1;
    pi[m] = tval[m] ? spos[ti[m]] : make_double4(1e300, 1e300, 1e300, 1.0);
    fi[m] = tval[m] ? sf[ti[m]] : make_double4(0, 0, 0, 0);
    u[m][0] = u[m][1] = u[m][2] = 0.0;
  }
  bool bad = false;
  for (int32_t c0 = j0; c0 < j1; c0 += TS) {
    const int cn = min(TS, j1 - c0);
    __syncthreads();
    if (threadIdx.x < cn) {
      sp[threadIdx.x] = spos[c0 + threadIdx.x];
      sfs[threadIdx.x] = sf[c0 + threadIdx.x];
    }
    __syncthreads();
    if (f == 0) {  // b itself: every ordered pair (i, j != i), forward only
      for (int jj = 0; jj < cn; ++jj) {
        const double4 pj = sp[jj], fj = sfs[jj];
#pragma unroll
        for (int m = 0; m < TPT; ++m) {
          if (!tval[m] || c0 + jj == ti[m]) continue;
          double dx, dy, dz, c1, c2;
          clamped_far_coefs<POLY>(pi[m], pj, a2, tau_hi, dx, dy, dz, c1, c2);
          const double t = c2 * fma(dz, fj.z, fma(dy, fj.y, dx * fj.x));
          u[m][0] = fma(t, dx, fma(c1, fj.x, u[m][0]));
          u[m][1] = fma(t, dy, fma(c1, fj.y, u[m][1]));
          u[m][2] = fma(t, dz, fma(c1, fj.z, u[m][2]));
        }
      }
      continue;
    }
    // q != b: 32-source rotation blocks; each warp's 32 TPT targets against the chunk's sources
    for (int sb = 0; sb * 32 < cn; ++sb) {
      double rx = 0.0, ry = 0.0, rz = 0.0;
#pragma unroll 1
      for (int st = 0; st < 32; ++st) {
        const int jj = sb * 32 + ((lane + st) & 31);
        if (jj < cn) {
          const double4 pj = sp[jj], fj = sfs[jj];
#pragma unroll
          for (int m = 0; m < TPT; ++m) {
            if (!tval[m]) continue;
            double dx, dy, dz, c1, c2;
            clamped_far_coefs<POLY>(pi[m], pj, a2, tau_hi, dx, dy, dz, c1, c2);
            const double t = c2 * fma(dz, fj.z, fma(dy, fj.y, dx * fj.x));
            u[m][0] = fma(t, dx, fma(c1, fj.x, u[m][0]));
            u[m][1] = fma(t, dy, fma(c1, fj.y, u[m][1]));
            u[m][2] = fma(t, dz, fma(c1, fj.z, u[m][2]));
            const double tr = c2 * fma(dz, fi[m].z, fma(dy, fi[m].y, dx * fi[m].x));  // T even in d
            rx = fma(tr, dx, fma(c1, fi[m].x, rx));
            ry = fma(tr, dy, fma(c1, fi[m].y, ry));
            rz = fma(tr, dz, fma(c1, fi[m].z, rz));
          }
        }
        const int src = (lane + 1) & 31;  // next step this lane meets the source lane+1 met now
        rx = __shfl_sync(0xffffffffu, rx, src);
        ry = __shfl_sync(0xffffffffu, ry, src);
        rz = __shfl_sync(0xffffffffu, rz, src);
      }
      // lane l now holds source sb*32 + l's reverse sum over this warp's targets
      rev[w][sb * 32 + lane][0] = rx;
      rev[w][sb * 32 + lane][1] = ry;
      rev[w][sb * 32 + lane][2] = rz;
    }
    __syncthreads();
    if (threadIdx.x < cn) {  // the 4 warps' reverse sums in warp order -> one fixed-point add
      double v[3];
#pragma unroll
      for (int c = 0; c < 3; ++c) v[c] = ((rev[0][threadIdx.x][c] + rev[1][threadIdx.x][c]) + rev[2][threadIdx.x][c]) +
                                         rev[3][threadIdx.x][c];
      fx_red3(acc + static_cast<int64_t>(c0 + threadIdx.x) * 9, v[0], v[1], v[2], scale, bad);
    }
  }
#pragma unroll
  for (int m = 0; m < TPT; ++m)
    if (tval[m]) fx_red3(acc + static_cast<int64_t>(ti[m]) * 9, u[m][0], u[m][1], u[m][2], scale, bad);
  (void)err;  // (coincident centres: flagged by the L2P kernel's near-list pass)
  if (bad) fs->bad = 1;
}

// NEAR_FX: the near field was summed by p2p_sym_kernel into fixed-point limbs (acc, scale fs); this
// kernel then adds them (and zeroes them for the next apply) instead of running the 27-leaf loop.
template <int NN, bool POLY, bool NEAR_FX>
__global__ void __launch_bounds__(128) l2p_p2p_kernel(const double4* __restrict__ spos,
                                                      const double4* __restrict__ sf,
                                                      const int32_t* __restrict__ sidx,
                                                      const int32_t* __restrict__ lstart, Geom g,
                                                      const double* __restrict__ Lc, int64_t loff_L, double scale,
                                                      double4* __restrict__ u4, int32_t* __restrict__ err,
                                                      const int32_t* __restrict__ done, long long* __restrict__ acc,
                                                      FxScale* __restrict__ fs, int64_t fx_count,
                                                      const double4* __restrict__ pos4o,
                                                      const double4* __restrict__ f4o,
                                                      const int32_t* __restrict__ near_ptr,
                                                      const int32_t* __restrict__ near_idx) {
  if (done != nullptr && *done) return;
  constexpr int NB = NN * NN * NN;
  constexpr int TS = 128;
  constexpr int C = POLY ? 9 : 3;
  __shared__ double sl[NB * C];
  __shared__ double4 sp[TS], sfs[TS];
  const int64_t b = blockIdx.x;
  // grid.y: chunk of TS targets of the leaf (the leaf's targets in parallel CTAs)
  const int32_t i0 = lstart[b] + static_cast<int32_t>(blockIdx.y) * TS, i1 = min(lstart[b + 1], i0 + TS);
  if (i0 >= i1) return;
  const int D = 1 << g.L;
  const int bx = static_cast<int>(b % D), by = static_cast<int>((b / D) % D), bz = static_cast<int>(b / D / D);
  double cx, cy, cz, w;
  box_center(g, g.L, b, cx, cy, cz, w);
  for (int t = threadIdx.x; t < C * NB; t += blockDim.x) sl[t] = Lc[(loff_L + b) * NB * C + t];
  const double a = g.a, a2 = a * a, ia = 1.0 / a;
  const long long near_bits = __double_as_longlong(4.0 * a2);
  for (int32_t k0 = i0; k0 < i1; k0 += TS) {
    const int32_t k = k0 + threadIdx.x;
    const bool act = k < i1;
    double4 pi = make_double4(0, 0, 0, 0), fi = pi;
    if (act) {
      pi = spos[k];
      fi = sf[k];
    }
    double ux = 0, uy = 0, uz = 0;
    __syncthreads();  // (sl ready; sp / sfs free)
    if (act) {  // far field: interpolate the leaf's local expansion
      double wx[NN], wy[NN], wz[NN];
      double ex[6] = {0, 0, 0, 0, 0, 0};  // POLY: L_B, L_C at u_i
      cheb_w<NN>(fmin(1.0, fmax(-1.0, (pi.x - cx) / w)), wx);
      cheb_w<NN>(fmin(1.0, fmax(-1.0, (pi.y - cy) / w)), wy);
      cheb_w<NN>(fmin(1.0, fmax(-1.0, (pi.z - cz) / w)), wz);
#pragma unroll
      for (int mz = 0; mz < NN; ++mz)
#pragma unroll
        for (int my = 0; my < NN; ++my) {
          const double wyz = wy[my] * wz[mz];
#pragma unroll
          for (int mx = 0; mx < NN; ++mx) {
            const double s = wx[mx] * wyz;
            const double* v = sl + ((mz * NN + my) * NN + mx) * C;
            ux = fma(s, v[0], ux);
            uy = fma(s, v[1], uy);
            uz = fma(s, v[2], uz);
#pragma unroll
            for (int q = 0; q < C - 3; ++q) ex[q] = fma(s, v[3 + q], ex[q]);
          }
        }
      if (POLY) {  // U = L_A + 2 w_i L_B + w_i^2 L_C
        const double tw = 2.0 * pi.w, w2 = pi.w * pi.w;
        ux = fma(w2, ex[3], fma(tw, ex[0], ux));
        uy = fma(w2, ex[4], fma(tw, ex[1], uy));
        uz = fma(w2, ex[5], fma(tw, ex[2], uz));
      }
    }
    // near field: the 27 leaves around b (incl. b), fixed order
    if (!NEAR_FX)
    for (int oz = -1; oz <= 1; ++oz)
      for (int oy = -1; oy <= 1; ++oy)
        for (int ox = -1; ox <= 1; ++ox) {
          const int qx = bx + ox, qy = by + oy, qz = bz + oz;
          if (qx < 0 || qy < 0 || qz < 0 || qx >= D || qy >= D || qz >= D) continue;
          const int64_t q = (static_cast<int64_t>(qz) * D + qy) * D + qx;
          const int32_t j0 = lstart[q], j1 = lstart[q + 1];
          SC_DCHECK(j0 >= 0 && j0 <= j1 && j1 <= lstart[int64_t(1) << (3 * g.L)]);
          for (int32_t c0 = j0; c0 < j1; c0 += TS) {
            const int cn = min(TS, j1 - c0);
            __syncthreads();
            if (threadIdx.x < cn) {
              sp[threadIdx.x] = spos[c0 + threadIdx.x];
              sfs[threadIdx.x] = sf[c0 + threadIdx.x];
            }
            __syncthreads();
            if (act) {
              for (int jj = 0; jj < cn; ++jj) {
                if (c0 + jj == k) continue;  // self: below
                const double4 pj = sp[jj], fj = sfs[jj];
                double dx, dy, dz;
                const double r2 = rpy_r2(pi, pj, dx, dy, dz);
                const double ab = POLY ? pi.w + pj.w : a;  // pair radius abar = (a_i + a_j)/2
                if (!rpy_is_near(r2, ab, POLY, near_bits)) {
                  far_pair(dx, dy, dz, fj.x, fj.y, fj.z, POLY ? ab * ab : a2, ux, uy, uz);
                } else {  // overlap branch: (4/(3a))(1 - 9r/(32a)) I + (1/(8a^2 r)) d d^T, a = abar
                  double rs = 0.0, rr = 0.0;
                  if (r2 > 0.0) {
                    rs = rsqrt_dp(r2);
                    rr = r2 * rs;
                  } else {
                    atomicExch(err, 1);  // coincident centres (reading A12)
                  }
                  const double iab = POLY ? 1.0 / ab : ia;
                  const double c1 = (4.0 / 3.0) * iab * fma(-9.0 / 32.0 * iab, rr, 1.0);
                  const double c2 = 0.125 * iab * iab * rs * fma(dz, fj.z, fma(dy, fj.y, dx * fj.x));
                  ux = fma(c2, dx, fma(c1, fj.x, ux));
                  uy = fma(c2, dy, fma(c1, fj.y, uy));
                  uz = fma(c2, dz, fma(c1, fj.z, uz));
                }
              }
            }
          }
        }
    if (act) {
      const double cs = POLY ? (2.0 / 3.0) / pi.w : (4.0 / 3.0) * ia;  // self: F/(6 pi mu a) = (1/(8 pi mu)) (4/(3a)) F
      ux = fma(cs, fi.x, ux);
      uy = fma(cs, fi.y, uy);
      uz = fma(cs, fi.z, uz);
      if (NEAR_FX) {  // + the exact near-field sums (one rounding each), then reset the limbs
        if (fs->bad) {
          ux = uy = uz = __longlong_as_double(0x7ff8000000000000LL);  // -> SC_ENONFINITE
        } else {
          const double inv = pow2(-fx_shift(fs, fx_count));
          long long* l = acc + static_cast<int64_t>(k) * 9;
          ux += fx_value(l + 0, inv);
          uy += fx_value(l + 3, inv);
          uz += fx_value(l + 6, inv);
        }
#pragma unroll
        for (int q = 0; q < 9; ++q) acc[static_cast<int64_t>(k) * 9 + q] = 0;
        // overlapping pairs (the contacts' near list, original order): the clamped far value the
        // symmetric near field used -> the overlap branch (r < 2 abar)
        const int32_t o = sidx[k];
        const double4 po = pos4o[o];
        for (int32_t e = near_ptr[o]; e < near_ptr[o + 1]; ++e) {
          const int32_t j = near_idx[e];
          const double4 pj = pos4o[j];
          const double4 fj = f4o[j];
          double dx, dy, dz;
          const double r2 = rpy_r2(po, pj, dx, dy, dz);
          const double ab = POLY ? po.w + pj.w : a;
          double rs = 0.0, rr = 0.0;
          if (r2 > 0.0) {
            rs = rsqrt_dp(r2);
            rr = r2 * rs;
          } else {
            atomicExch(err, 1);  // coincident centres (reading A12)
          }
          const double iab = 1.0 / ab;
          const double c1 = (4.0 / 3.0) * iab * fma(-9.0 / 32.0 * iab, rr, 1.0);
          const double c2 = 0.125 * iab * iab * rs * fma(dz, fj.z, fma(dy, fj.y, dx * fj.x));
          double fx_, fy_, fz_;
          rpy_far_clamped_contrib(dx, dy, dz, r2, ab, fj, fx_, fy_, fz_);
          ux += fma(c2, dx, c1 * fj.x) - fx_;
          uy += fma(c2, dy, c1 * fj.y) - fy_;
          uz += fma(c2, dz, c1 * fj.z) - fz_;
        }
      }
      SC_DCHECK(sidx[k] >= 0 && sidx[k] < lstart[int64_t(1) << (3 * g.L)]);
      u4[sidx[k]] = make_double4(scale * ux, scale * uy, scale * uz, 0.0);
    }
  }
}

#define SC_CUBLAS(call)                                                                  \
  do {                                                                                   \
    cublasStatus_t s_ = (call);                                                          \
    if (s_ != CUBLAS_STATUS_SUCCESS) return fail(ctx, SC_ECUDA, std::string(#call) + " failed"); \
  } while (0)
#define SC_CUSOLVER(call)                                                                \
  do {                                                                                   \
    cusolverStatus_t s_ = (call);                                                        \
    if (s_ != CUSOLVER_STATUS_SUCCESS) return fail(ctx, SC_ECUDA, std::string(#call) + " failed"); \
  } while (0)

int svd_handles(sc_ctx* ctx) {
  if (ctx->cublas == nullptr) {
    cublasHandle_t h = nullptr;
    SC_CUBLAS(cublasCreate(&h));
    ctx->cublas = h;
  }
  if (ctx->cusolver == nullptr) {
    cusolverDnHandle_t h = nullptr;
    SC_CUSOLVER(cusolverDnCreate(&h));
    ctx->cusolver = h;
  }
  SC_CUBLAS(cublasSetStream(static_cast<cublasHandle_t>(ctx->cublas), ctx->stream));
  SC_CUSOLVER(cusolverDnSetStream(static_cast<cusolverDnHandle_t>(ctx->cusolver), ctx->stream));
  return 0;
}

// Bases and compressed operators of every level for the current tree (cached by geometry key).
// Monodisperse: one basis for the operators K_o of the far branch.  Polydisperse: one basis for
// both radius-free parts O_o and D_o (dominant eigenvectors of their trace-normalised Gram
// matrices' sum) and two operator sets C^O_o, C^D_o.
template <int NN, bool POLY>
int fmm_svd_prepare(sc_ctx* ctx, const Geom& g) {
  double escale = 1.0;
  if (const char* v = std::getenv("SC_FMM_SVD_EPS_SCALE")) escale = std::atof(v);
  const double key[5] = {g.H, static_cast<double>(g.L), static_cast<double>(NN), POLY ? -1.0 : g.a, escale};
  bool same = true;
  for (int i = 0; i < 5; ++i) same = same && ctx->fmm_svd_key[i] == key[i];
  if (same) return 0;
  if (int rc = svd_handles(ctx)) return rc;
  cublasHandle_t cb = static_cast<cublasHandle_t>(ctx->cublas);
  cusolverDnHandle_t cs = static_cast<cusolverDnHandle_t>(ctx->cusolver);
  constexpr int NB = NN * NN * NN, R = 3 * NB;
  constexpr int NK = POLY ? 2 : 1;  // operator families
  // kept singular directions: sigma >= eps sigma_max, eps = 3% of the order's stated error bar
  const double eps = (NN == 4 ? 6e-5 : (NN == 6 ? 1.8e-6 : 9e-8)) * escale;
  const int L = g.L;
  std::vector<int32_t> tab(kOffGrid + kOffCount, -1);  // [li_of_oi (343) | oi of li (316)]
  int nl = 0;
  for (int oi = 0; oi < kOffGrid; ++oi) {
    const int ox = oi % 7 - 3, oy = (oi / 7) % 7 - 3, oz = oi / 49 - 3;
    if (std::abs(ox) <= 1 && std::abs(oy) <= 1 && std::abs(oz) <= 1) continue;
    tab[oi] = nl;
    tab[kOffGrid + nl] = oi;
    ++nl;
  }
  if (nl != kOffCount) return fail(ctx, SC_EINVAL, "fmm compression: offset table");
  ctx->fmm_svd_lih.assign(tab.begin(), tab.begin() + kOffGrid);
  if (int rc = ensure(ctx, ctx->fmm_svd_li, tab.size())) return rc;
  SC_CUDA(cudaMemcpyAsync(ctx->fmm_svd_li.p, tab.data(), sizeof(int32_t) * tab.size(), cudaMemcpyHostToDevice,
                          ctx->stream));
  const int32_t* ois = ctx->fmm_svd_li.p + kOffGrid;
  const int Q = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kOffCount, (int64_t(256) << 20) /
                                                                                        (int64_t(R) * R * 8))));
  int lwork = 0;
  SC_CUSOLVER(cusolverDnDsyevd_bufferSize(cs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, R, nullptr, R,
                                          nullptr, &lwork));
  // work: K chunk (Q R R) | G (R R) | G2 (R R) | eigenvalues (R) | syevd work | info | eigvecs per level
  const size_t nK = size_t(Q) * R * R, nG = size_t(R) * R;
  const size_t nwork = nK + 2 * nG + R + size_t(lwork) + 2 + size_t(L + 1) * R * R;
  if (int rc = ensure(ctx, ctx->fmm_svd_work, nwork)) return rc;
  double* K = ctx->fmm_svd_work.p;
  double* G = K + nK;
  double* G2 = G + nG;
  double* W = G2 + nG;
  double* wk = W + R;
  int* info = reinterpret_cast<int*>(wk + lwork);
  double* Uall = wk + lwork + 2;  // level l: R x R eigenvectors at Uall + l R R
  const double one = 1.0, zero = 0.0;
  const unsigned kb = 256;
  const double a2 = g.a * g.a;
  auto build = [&](double w, int c0, int q, int kind) -> int {
    const int64_t tot = int64_t(R) * R * q;
    svd_build_k_kernel<NN><<<static_cast<unsigned>((tot + kb - 1) / kb), kb, 0, ctx->stream>>>(K, ois + c0, q, w, a2,
                                                                                             kind);
    return check_launch(ctx, "fmm_svd_build_k");
  };
  auto gram = [&](double w, int kind, double* Gx) -> int {  // Gx = sum_o K_o K_o^T (lower)
    SC_CUDA(cudaMemsetAsync(Gx, 0, sizeof(double) * nG, ctx->stream));
    for (int c0 = 0; c0 < kOffCount; c0 += Q) {
      const int q = std::min(Q, kOffCount - c0);
      if (int rc = build(w, c0, q, kind)) return rc;
      SC_CUBLAS(cublasDsyrk(cb, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, R, R * q, &one, K, R, &one, Gx, R));
    }
    return 0;
  };
  ctx->fmm_svd_k.assign(L + 1, 0);
  std::vector<double> hW(R);
  for (int l = 2; l <= L; ++l) {
    const double w = g.H / static_cast<double>(int64_t(1) << (l + 1));
    if (!POLY) {
      if (int rc = gram(w, 0, G)) return rc;
    } else {  // G = G_O / tr(G_O) + G_D / tr(G_D): both families equally represented
      if (int rc = gram(w, 1, G)) return rc;
      if (int rc = gram(w, 2, G2)) return rc;
      double trO = 0.0, trD = 0.0;
      SC_CUBLAS(cublasDasum(cb, R, G, R + 1, &trO));  // (diagonal of a Gram matrix: >= 0)
      SC_CUBLAS(cublasDasum(cb, R, G2, R + 1, &trD));
      if (!(trO > 0.0) || !(trD > 0.0)) return fail(ctx, SC_ECUDA, "fmm compression: degenerate operators");
      const double sO = 1.0 / trO, sD = 1.0 / trD;
      SC_CUBLAS(cublasDgeam(cb, CUBLAS_OP_N, CUBLAS_OP_N, R, R, &sO, G, R, &sD, G2, R, G, R));
    }
    SC_CUSOLVER(cusolverDnDsyevd(cs, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, R, G, R, W, wk, lwork, info));
    SC_CUDA(cudaMemcpyAsync(hW.data(), W, sizeof(double) * R, cudaMemcpyDeviceToHost, ctx->stream));
    int hinfo = 0;
    SC_CUDA(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    SC_CUDA(cudaStreamSynchronize(ctx->stream));
    if (hinfo != 0) return fail(ctx, SC_ECUDA, "fmm compression: eigensolver did not converge");
    const double lmax = hW[R - 1];  // ascending; G = sum K K^T: lambda = sigma^2
    int k = 0;
    for (int i = R - 1; i >= 0 && hW[i] >= eps * eps * lmax; --i) ++k;
    k = std::max(1, k);
    ctx->fmm_svd_k[l] = k;
    SC_CUDA(cudaMemcpyAsync(Uall + size_t(l) * R * R, G + size_t(R - k) * R, sizeof(double) * R * k,
                            cudaMemcpyDeviceToDevice, ctx->stream));
  }
  // U_l and C_l ([family][316] k_l x k_l, column-major, operator index li) into their buffers
  ctx->fmm_svd_uoff.assign(L + 2, 0);
  ctx->fmm_svd_coff.assign(L + 2, 0);
  int64_t nu = 0, ncop = 0, kmax = 1;
  for (int l = 2; l <= L; ++l) {
    ctx->fmm_svd_uoff[l] = nu;
    ctx->fmm_svd_coff[l] = ncop;
    nu += int64_t(R) * ctx->fmm_svd_k[l];
    ncop += int64_t(NK) * kOffCount * ctx->fmm_svd_k[l] * ctx->fmm_svd_k[l];
    kmax = std::max<int64_t>(kmax, ctx->fmm_svd_k[l]);
  }
  if (int rc = ensure(ctx, ctx->fmm_svd_U, nu)) return rc;
  if (int rc = ensure(ctx, ctx->fmm_svd_C, ncop)) return rc;
  // T1 = K_o U in G's space
  const int Q2 = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(Q, int64_t(nG) / (int64_t(R) * kmax))));
  for (int l = 2; l <= L; ++l) {
    const int k = ctx->fmm_svd_k[l];
    const double w = g.H / static_cast<double>(int64_t(1) << (l + 1));
    double* U = ctx->fmm_svd_U.p + ctx->fmm_svd_uoff[l];
    SC_CUDA(cudaMemcpyAsync(U, Uall + size_t(l) * R * R, sizeof(double) * R * k, cudaMemcpyDeviceToDevice,
                            ctx->stream));
    for (int f = 0; f < NK; ++f) {
      double* Cl = ctx->fmm_svd_C.p + ctx->fmm_svd_coff[l] + int64_t(f) * kOffCount * k * k;
      for (int c0 = 0; c0 < kOffCount; c0 += Q2) {
        const int q = std::min(Q2, kOffCount - c0);
        if (int rc = build(w, c0, q, POLY ? 1 + f : 0)) return rc;
        SC_CUBLAS(cublasDgemmStridedBatched(cb, CUBLAS_OP_N, CUBLAS_OP_N, R, k, R, &one, K, R, int64_t(R) * R, U, R,
                                            0, &zero, G, R, int64_t(R) * k, q));
        SC_CUBLAS(cublasDgemmStridedBatched(cb, CUBLAS_OP_T, CUBLAS_OP_N, k, k, R, &one, U, R, 0, G, R,
                                            int64_t(R) * k, &zero, Cl + int64_t(c0) * k * k, k, int64_t(k) * k, q));
      }
    }
  }
  SC_CUDA(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < 5; ++i) ctx->fmm_svd_key[i] = key[i];
  if (std::getenv("SC_FMM_DEBUG"))
    for (int l = 2; l <= L; ++l)
      std::fprintf(stderr, "fmm svd: order %d %s level %d rank %d of %d\n", NN, POLY ? "poly" : "mono", l,
                   ctx->fmm_svd_k[l], R);
  return 0;
}

// The compressed M2L of every level (writes L):
//   mono  M^c = U^T M,  L^c = sum_o C_o M^c,  L = U L^c
//   poly  P_c = U^T s_c (c = 0, 1, 2);  A = sum_o C^O_o P_0 + C^D_o P_2,  B = sum_o C^D_o P_1,
//         C = sum_o C^D_o P_0;  (L_A, L_B, L_C) = U (A, B, C)
// Each level: 189 batched GEMM calls (one per offset of every parity class, distinct outputs per
// call) plus, polydisperse, 189 more for the D s2 term of A; accumulated in call order.
template <int NN, bool POLY>
int fmm_m2l_compressed(sc_ctx* ctx, const Geom& g, const double* M, double* Lx, const int32_t* done) {
  (void)done;
  constexpr int NB = NN * NN * NN, R = 3 * NB;
  constexpr int NCH = POLY ? 3 : 1;  // channels in and out
  cublasHandle_t cb = static_cast<cublasHandle_t>(ctx->cublas);
  SC_CUBLAS(cublasSetStream(cb, ctx->stream));
  const std::vector<int64_t>& lo = ctx->fmm_lev_off;
  int64_t need = 1;
  for (int l = 2; l <= g.L; ++l) {
    const int64_t Dq = (int64_t(1) << (l - 1)) + 2;
    need = std::max<int64_t>(need, int64_t(NCH) * 8 * Dq * Dq * Dq * ctx->fmm_svd_k[l]);
  }
  const int kmax = *std::max_element(ctx->fmm_svd_k.begin(), ctx->fmm_svd_k.end());
  const int64_t nat = int64_t(NCH) * nbox(g.L) * kmax;    // natural order, NCH channels
  const int64_t split = POLY ? int64_t(NCH) * nbox(g.L) * R : 0;  // poly: split / merged R-vectors
  if (int rc = ensure(ctx, ctx->fmm_Mc, nat + need + split)) return rc;
  if (int rc = ensure(ctx, ctx->fmm_Lc, nat + need)) return rc;
  constexpr int NE = POLY ? 32 : 8;  // batch entries per offset (poly: 24 + 8)
  if (int rc = ensure(ctx, ctx->fmm_svd_ptrs, 3 * 189 * NE)) return rc;
  const double one = 1.0, zero = 0.0;
  for (int l = 2; l <= g.L; ++l) {
    const int k = ctx->fmm_svd_k[l];
    const int64_t nb = nbox(l);
    const int D = 1 << l, Dp = D / 2, Dq = Dp + 2;
    const int64_t npad = int64_t(Dq) * Dq * Dq;
    const double* U = ctx->fmm_svd_U.p + ctx->fmm_svd_uoff[l];
    double* mcn = ctx->fmm_Mc.p;                 // [ch][box][k]
    double* mcp = ctx->fmm_Mc.p + nat;           // [ch][class][padded][k]
    double* sbuf = ctx->fmm_Mc.p + nat + need;   // poly: [ch][box][node][3]
    double* lcn = ctx->fmm_Lc.p;
    double* lcp = ctx->fmm_Lc.p + nat;
    const double* Ml = M + lo[l] * NB * (POLY ? 9 : 3);
    double* Ll = Lx + lo[l] * NB * (POLY ? 9 : 3);
    const int64_t nvals = nb * NB;
    if (POLY) {
      svd_poly_split_kernel<<<static_cast<unsigned>((nvals * 9 + 255) / 256), 256, 0, ctx->stream>>>(nvals, Ml, sbuf);
      SC_CUBLAS(cublasDgemm(cb, CUBLAS_OP_T, CUBLAS_OP_N, k, static_cast<int>(NCH * nb), R, &one, U, R, sbuf, R, &zero,
                            mcn, k));
    } else {
      SC_CUBLAS(cublasDgemm(cb, CUBLAS_OP_T, CUBLAS_OP_N, k, static_cast<int>(nb), R, &one, U, R, Ml, R, &zero, mcn,
                            k));
    }
    SC_CUDA(cudaMemsetAsync(mcp, 0, sizeof(double) * NCH * 8 * npad * k, ctx->stream));  // zero halo
    const int64_t tot = nb * k;
    for (int ch = 0; ch < NCH; ++ch)
      svd_to_classes_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, ctx->stream>>>(
          D, k, mcn + ch * nb * k, mcp + ch * 8 * npad * k);
    const int64_t cbeg = (int64_t(1) * Dq + 1) * Dq + 1, cend = (int64_t(Dp) * Dq + Dp) * Dq + Dp + 1;
    const int ncol = static_cast<int>(cend - cbeg);
    const double* C0 = ctx->fmm_svd_C.p + ctx->fmm_svd_coff[l];  // mono: C; poly: C^O
    const double* C1 = C0 + int64_t(kOffCount) * k * k;           // poly: C^D
    auto chan_in = [&](int ch, int spc, int64_t dl) { return mcp + ((int64_t(ch) * 8 + spc) * npad + cbeg + dl) * k; };
    auto chan_out = [&](int ch, int pc) { return lcp + ((int64_t(ch) * 8 + pc) * npad + cbeg) * k; };
    std::vector<const double*> hA(189 * NE), hB(189 * NE);
    std::vector<double*> hC(189 * NE);
    for (int pc = 0; pc < 8; ++pc) {
      const int pxb = pc & 1, pyb = (pc >> 1) & 1, pzb = pc >> 2;
      int i = 0;
      for (int oz = -2 - pzb; oz <= 3 - pzb; ++oz)
        for (int oy = -2 - pyb; oy <= 3 - pyb; ++oy)
          for (int ox = -2 - pxb; ox <= 3 - pxb; ++ox) {
            if (std::abs(ox) <= 1 && std::abs(oy) <= 1 && std::abs(oz) <= 1) continue;
            const int oi = ((oz + 3) * 7 + oy + 3) * 7 + ox + 3;
            const int qx = pxb + ox, qy = pyb + oy, qz = pzb + oz;
            const int spc = (qx & 1) | ((qy & 1) << 1) | ((qz & 1) << 2);
            const int64_t dl = ((int64_t((qz - (qz & 1)) / 2)) * Dq + (qy - (qy & 1)) / 2) * Dq + (qx - (qx & 1)) / 2;
            const int64_t li = ctx->fmm_svd_lih[oi];
            const double* cO = C0 + li * k * k;
            const double* cD = C1 + li * k * k;
            double** Cp = hC.data() + i * NE;
            const double** Ap = hA.data() + i * NE;
            const double** Bp = hB.data() + i * NE;
            if (!POLY) {
              Ap[pc] = cO;
              Bp[pc] = chan_in(0, spc, dl);
              Cp[pc] = chan_out(0, pc);
            } else {  // [A = C^O P0 | B = C^D P1 | C = C^D P0] (24), then [A += C^D P2] (8)
              Ap[pc] = cO;
              Bp[pc] = chan_in(0, spc, dl);
              Cp[pc] = chan_out(0, pc);
              Ap[8 + pc] = cD;
              Bp[8 + pc] = chan_in(1, spc, dl);
              Cp[8 + pc] = chan_out(1, pc);
              Ap[16 + pc] = cD;
              Bp[16 + pc] = chan_in(0, spc, dl);
              Cp[16 + pc] = chan_out(2, pc);
              Ap[24 + pc] = cD;
              Bp[24 + pc] = chan_in(2, spc, dl);
              Cp[24 + pc] = chan_out(0, pc);
            }
            ++i;
          }
    }
    const double** dA = reinterpret_cast<const double**>(ctx->fmm_svd_ptrs.p);
    const double** dB = dA + 189 * NE;
    double** dC = reinterpret_cast<double**>(ctx->fmm_svd_ptrs.p + 2 * 189 * NE);
    // (pageable host -> device: the copies return once the tables are staged; stream-ordered after
    // the previous level's GEMMs that read the same device tables)
    SC_CUDA(cudaMemcpyAsync(dA, hA.data(), sizeof(void*) * 189 * NE, cudaMemcpyHostToDevice, ctx->stream));
    SC_CUDA(cudaMemcpyAsync(dB, hB.data(), sizeof(void*) * 189 * NE, cudaMemcpyHostToDevice, ctx->stream));
    SC_CUDA(cudaMemcpyAsync(dC, hC.data(), sizeof(void*) * 189 * NE, cudaMemcpyHostToDevice, ctx->stream));
    const int first = POLY ? 24 : 8;
    for (int i = 0; i < 189; ++i) {
      SC_CUBLAS(cublasDgemmBatched(cb, CUBLAS_OP_N, CUBLAS_OP_N, k, ncol, k, &one, dA + i * NE, k, dB + i * NE, k,
                                   i == 0 ? &zero : &one, dC + i * NE, k, first));
      if (POLY)
        SC_CUBLAS(cublasDgemmBatched(cb, CUBLAS_OP_N, CUBLAS_OP_N, k, ncol, k, &one, dA + i * NE + 24, k,
                                     dB + i * NE + 24, k, &one, dC + i * NE + 24, k, 8));
    }
    for (int ch = 0; ch < NCH; ++ch)
      svd_from_classes_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, ctx->stream>>>(
          D, k, lcp + ch * 8 * npad * k, lcn + ch * nb * k);
    if (POLY) {
      SC_CUBLAS(cublasDgemm(cb, CUBLAS_OP_N, CUBLAS_OP_N, R, static_cast<int>(NCH * nb), k, &one, U, R, lcn, k, &zero,
                            sbuf, R));
      svd_poly_merge_kernel<<<static_cast<unsigned>((nvals * 9 + 255) / 256), 256, 0, ctx->stream>>>(nvals, sbuf, Ll);
    } else {
      SC_CUBLAS(cublasDgemm(cb, CUBLAS_OP_N, CUBLAS_OP_N, R, static_cast<int>(nb), k, &one, U, R, lcn, k, &zero, Ll, R));
    }
  }
  ctx->launch_count += (POLY ? 9 : 5) * (g.L - 1);
  return 0;
}

template <int NN, bool POLY>
int fmm_launch(sc_ctx* ctx, const Geom& g, const double4* f4, double mu, double4* u4, const int32_t* done) {
  constexpr int NB = NN * NN * NN;
  constexpr int C = POLY ? 9 : 3;
  const int nb = (NB + 31) / 32 * 32;
  const int L = g.L;
  const int64_t n = ctx->n;
  const int64_t* loff = ctx->fmm_lev_off_dev.p;
  const std::vector<int64_t>& lo = ctx->fmm_lev_off;
  double* M = ctx->fmm_M.p;
  double* Lc = ctx->fmm_L.p;
  timer_begin(ctx, SC_K_RPY);
  gather_sorted_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(ctx->fmm_sidx.p, n, f4,
                                                                                       ctx->fmm_sf4.p);
  p2m_kernel<NN, C><<<static_cast<unsigned>(nbox(L)), nb, 0, ctx->stream>>>(
      ctx->fmm_spos4.p, ctx->fmm_sf4.p, ctx->fmm_lstart.p, g, M + lo[L] * NB * C, done);
  for (int l = L - 1; l >= 2; --l)
    transfer_kernel<NN, true, C><<<static_cast<unsigned>(nbox(l)), nb, 0, ctx->stream>>>(
        l, M + lo[l] * NB * C, M + lo[l + 1] * NB * C, done);
  if (fmm_use_svd(ctx)) {
    if (int rc = fmm_m2l_compressed<NN, POLY>(ctx, g, M, Lc, done)) return rc;
  } else if (POLY)
    m2l_poly_kernel<NN><<<static_cast<unsigned>(lo[L + 1] - lo[2]), nb, 0, ctx->stream>>>(g, loff, M, Lc, done);
  else
    m2l_kernel<NN><<<static_cast<unsigned>(lo[L + 1] - lo[2]), nb, 0, ctx->stream>>>(g, loff, M, Lc, done);
  for (int l = 2; l < L; ++l)
    transfer_kernel<NN, false, C><<<static_cast<unsigned>(nbox(l + 1)), nb, 0, ctx->stream>>>(
        l, Lc + lo[l] * NB * C, Lc + lo[l + 1] * NB * C, done);
  const double scale = 1.0 / (8.0 * 3.14159265358979323846 * mu);
  const unsigned nchunk = static_cast<unsigned>(std::max<int64_t>(1, (ctx->fmm_maxleaf + 127) / 128));
  const dim3 gp(static_cast<unsigned>(nbox(L)), nchunk);
  if (SC_FMM_P2P_SYM) {
    const int64_t fx_count = 27 * std::max<int64_t>(1, ctx->fmm_maxleaf);  // sources per row, at most
    FxScale* fs = reinterpret_cast<FxScale*>(ctx->fmm_fx.p);
    SC_CUDA(cudaMemsetAsync(fs, 0, sizeof(FxScale), ctx->stream));
    fmm_fx_prep_kernel<<<static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 4 * 148)), 256, 0, ctx->stream>>>(
        ctx->fmm_spos4.p, ctx->fmm_sf4.p, n, fs, done);
    const int tpt = n >= 192 * nbox(L) ? 2 : 1;  // (measured: profiles/r02/fmm_p2p_sym_ab.txt)
    const unsigned nchunk_s =
        static_cast<unsigned>(std::max<int64_t>(1, (ctx->fmm_maxleaf + 128 * tpt - 1) / (128 * tpt)));
    const dim3 gs(static_cast<unsigned>(nbox(L)), 14, nchunk_s);
    if (tpt == 2)
      p2p_sym_kernel<POLY, 2><<<gs, 128, 0, ctx->stream>>>(ctx->fmm_spos4.p, ctx->fmm_sf4.p, ctx->fmm_lstart.p, g,
                                                            ctx->fmm_acc.p, fs, fx_count, ctx->derr, done);
    else
      p2p_sym_kernel<POLY, 1><<<gs, 128, 0, ctx->stream>>>(ctx->fmm_spos4.p, ctx->fmm_sf4.p, ctx->fmm_lstart.p, g,
                                                            ctx->fmm_acc.p, fs, fx_count, ctx->derr, done);
    l2p_p2p_kernel<NN, POLY, true><<<gp, 128, 0, ctx->stream>>>(
        ctx->fmm_spos4.p, ctx->fmm_sf4.p, ctx->fmm_sidx.p, ctx->fmm_lstart.p, g, Lc, lo[L], scale, u4, ctx->derr,
        done, ctx->fmm_acc.p, fs, fx_count, ctx->pos4.p, f4, ctx->near_ptr.p, ctx->near_idx.p);
    ctx->launch_count += 2;
  } else {
    l2p_p2p_kernel<NN, POLY, false><<<gp, 128, 0, ctx->stream>>>(
        ctx->fmm_spos4.p, ctx->fmm_sf4.p, ctx->fmm_sidx.p, ctx->fmm_lstart.p, g, Lc, lo[L], scale, u4, ctx->derr,
        done, nullptr, nullptr, 0, nullptr, nullptr, nullptr, nullptr);
  }
  timer_end(ctx, SC_K_RPY);
  ctx->launch_count += 4 + 2 * (L - 2);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_fail(ctx, e, "fmm");
  if (ctx->npad > n)
    SC_CUDA(cudaMemsetAsync(u4 + n, 0, sizeof(double4) * (ctx->npad - n), ctx->stream));
  return 0;
}

__global__ void bbox_kernel(const double4* __restrict__ pos4, int64_t n, double* __restrict__ out /* 8 */) {
  double lo[4] = {1e300, 1e300, 1e300, 1e300}, hi[4] = {-1e300, -1e300, -1e300, -1e300};
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double4 p = pos4[i];
    lo[0] = fmin(lo[0], p.x); lo[1] = fmin(lo[1], p.y); lo[2] = fmin(lo[2], p.z);
    hi[0] = fmax(hi[0], p.x); hi[1] = fmax(hi[1], p.y); hi[2] = fmax(hi[2], p.z);
    lo[3] = fmin(lo[3], p.w); hi[3] = fmax(hi[3], p.w);  // half radii
  }
  __shared__ double s[8][256];
  for (int d = 0; d < 4; ++d) {
    s[d][threadIdx.x] = lo[d];
    s[4 + d][threadIdx.x] = hi[d];
  }
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w)
      for (int d = 0; d < 4; ++d) {
        s[d][threadIdx.x] = fmin(s[d][threadIdx.x], s[d][threadIdx.x + w]);
        s[4 + d][threadIdx.x] = fmax(s[4 + d][threadIdx.x], s[4 + d][threadIdx.x + w]);
      }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int d = 0; d < 8; ++d) out[blockIdx.x * 8 + d] = s[d][0];
}

double cheb_S(int n, double xk, double u) {  // host: S_n(xbar_k, u)
  double s = 0.0, t0 = 1.0, t1 = u, tk0 = 1.0, tk1 = xk;
  for (int q = 1; q < n; ++q) {
    s += tk1 * t1;
    const double t2 = 2.0 * u * t1 - t0, tk2 = 2.0 * xk * tk1 - tk0;
    t0 = t1; t1 = t2; tk0 = tk1; tk1 = tk2;
  }
  return (1.0 + 2.0 * s) / n;
}

}  // namespace

// The interpolation tables of orders 4, 6, 8 into this device's constant memory (sc_create).
int fmm_init_device(sc_ctx* ctx) {
  double tab[tab_size(4) + tab_size(6) + tab_size(8)];
  const double pi = 3.14159265358979323846;
  for (int nn : {4, 6, 8}) {
    double* xb = tab + tab_off(nn);
    double* T = xb + nn;
    double* P = T + nn * nn;
    for (int k = 0; k < nn; ++k) xb[k] = std::cos((2 * k + 1) * pi / (2 * nn));
    for (int k = 0; k < nn; ++k) {
      double t0 = 1.0, t1 = xb[k];
      T[k * nn] = 1.0;
      if (nn > 1) T[k * nn + 1] = xb[k];
      for (int q = 2; q < nn; ++q) {
        const double t2 = 2.0 * xb[k] * t1 - t0;
        T[k * nn + q] = t2;
        t0 = t1;
        t1 = t2;
      }
    }
    for (int sg = 0; sg < 2; ++sg)
      for (int mp = 0; mp < nn; ++mp)
        for (int m = 0; m < nn; ++m) P[sg * nn * nn + mp * nn + m] = cheb_S(nn, xb[mp], 0.5 * (xb[m] + (sg ? 1.0 : -1.0)));
  }
  cudaError_t e = cudaMemcpyToSymbol(c_tab, tab, sizeof(tab));
  if (e != cudaSuccess) return cuda_fail(ctx, e, "fmm tables");
  return 0;
}

// Tree of the current bodies (after build_contacts): root cube, leaf level, bodies sorted by leaf.
int fmm_setup(sc_ctx* ctx) {
  const int nn = ctx->fmm_order;
  if (nn != 4 && nn != 6 && nn != 8) return fail(ctx, SC_EINVAL, "fmm order must be 4, 6 or 8");
  if (ctx->kind != kSpheres) return fail(ctx, SC_EINVAL, "the fast RPY summation is for spheres");
  const int64_t n = ctx->n;
  // bounding cube
  const int nbb = 64;
  if (int rc = ensure(ctx, ctx->bbox_part, 8 * nbb)) return rc;
  bbox_kernel<<<nbb, 256, 0, ctx->stream>>>(ctx->pos4.p, n, ctx->bbox_part.p);
  if (int rc = check_launch(ctx, "fmm_bbox")) return rc;
  std::vector<double> hb(8 * nbb);
  SC_CUDA(cudaMemcpyAsync(hb.data(), ctx->bbox_part.p, sizeof(double) * 8 * nbb, cudaMemcpyDeviceToHost, ctx->stream));
  SC_CUDA(cudaStreamSynchronize(ctx->stream));
  double lo[4] = {1e300, 1e300, 1e300, 1e300}, hi[4] = {-1e300, -1e300, -1e300, -1e300};
  for (int b = 0; b < nbb; ++b)
    for (int d = 0; d < 4; ++d) {
      lo[d] = std::min(lo[d], hb[b * 8 + d]);
      hi[d] = std::max(hi[d], hb[b * 8 + 4 + d]);
    }
  double ext = std::max(hi[0] - lo[0], std::max(hi[1] - lo[1], hi[2] - lo[2]));
  // the largest pair radius: every overlapping pair (r < 2 abar <= 2 a_max) must lie in
  // neighbouring leaves, and well-separated boxes are >= one leaf side >= 2 a_max apart
  const double a = ctx->poly ? 2.0 * hi[3] : ctx->a_const;
  ext = std::max(ext, 8.0 * a) * (1.0 + 1e-9) + 1e-9;  // (>= 4 leaves of side >= 2a per dimension)
  if (fmm_use_svd(ctx)) {  // root side on a ladder 8a 2^(i/8): the cached M2L bases survive small
                           // changes of the bounding box (time stepping)
    const double i = std::ceil(8.0 * std::log2(ext / (8.0 * a)) - 1e-9);
    ext = 8.0 * a * std::exp2(std::max(0.0, i) / 8.0);
  }
  // leaf level: largest useful L with leaf side >= 2a (far branch between well-separated boxes,
  // every overlapping pair in neighbouring leaves), chosen to balance the P2P and M2L work
  int L = ctx->fmm_leaf_level;
  const int Lmax = std::max(2, static_cast<int>(std::floor(std::log2(ext / (2.0 * a)))));
  if (L <= 0) {  // cost model: pair evaluations of P2P (27 leaves) and M2L (<= 189 boxes, n^6 node
                 // pairs, ~0.8 of a P2P pair's cost); at least 2 CTAs per SM of leaves when N allows
    double best = 1e300;
    const double nb3 = static_cast<double>(nn) * nn * nn;
    for (int l = 2; l <= std::min(Lmax, 7); ++l) {
      const double leaves = static_cast<double>(nbox(l));
      const double p2p = static_cast<double>(n) * 27.0 * (static_cast<double>(n) / leaves);
      double m2l = (ctx->poly ? 1.8 : 1.0) * 0.8 * 1.15 * leaves * 150.0 * nb3 * nb3;  // (poly: 3 fields)
      if (fmm_use_svd(ctx)) {  // compressed: 189 k^2 FMA per box on the GEMM path, ~7.8 FMA per P2P pair
        const double kest = nn == 4 ? 132.0 : (nn == 6 ? 286.0 : 454.0);
        m2l = (ctx->poly ? 4.4 : 1.0) * leaves * 189.0 * kest * kest / 7.8;  // (poly: 4 products, larger k)
      }
      const double fill = std::min(1.0, leaves * std::max(1.0, static_cast<double>(n) / leaves / 128.0) /
                                            (2.0 * std::max(ctx->num_sms, 1)));
      const double cost = (p2p + m2l) / fill;
      if (cost < best) {
        best = cost;
        L = l;
      }
    }
  }
  L = std::max(2, std::min(L, Lmax));
  ctx->fmm_L_used = L;
  ctx->fmm_poly = ctx->poly;
  ctx->fmm_geom[0] = 0.5 * (lo[0] + hi[0]) - 0.5 * ext;
  ctx->fmm_geom[1] = 0.5 * (lo[1] + hi[1]) - 0.5 * ext;
  ctx->fmm_geom[2] = 0.5 * (lo[2] + hi[2]) - 0.5 * ext;
  ctx->fmm_geom[3] = ext;
  Geom g{ctx->fmm_geom[0], ctx->fmm_geom[1], ctx->fmm_geom[2], ext, a, L};
  // bodies sorted by leaf (stable radix sort: within a leaf by body index -> deterministic sums)
  const int64_t nleaf = nbox(L);
  if (int rc = ensure(ctx, ctx->fmm_key, 2 * std::max<int64_t>(n, 1))) return rc;
  if (int rc = ensure(ctx, ctx->fmm_idx0, std::max<int64_t>(n, 1))) return rc;
  if (int rc = ensure(ctx, ctx->fmm_sidx, std::max<int64_t>(n, 1))) return rc;
  if (int rc = ensure(ctx, ctx->fmm_cnt, nleaf + 1)) return rc;
  if (int rc = ensure(ctx, ctx->fmm_lstart, nleaf + 1)) return rc;
  if (int rc = ensure(ctx, ctx->scan_tmp, scan_tmp_size(nleaf + 1) + 1)) return rc;
  SC_CUDA(cudaMemsetAsync(ctx->fmm_cnt.p, 0, sizeof(int32_t) * (nleaf + 1), ctx->stream));
  uint32_t* key_in = reinterpret_cast<uint32_t*>(ctx->fmm_key.p);
  uint32_t* key_out = key_in + std::max<int64_t>(n, 1);
  leaf_of_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(ctx->pos4.p, n, g, key_in,
                                                                                  ctx->fmm_idx0.p, ctx->fmm_cnt.p);
  if (int rc = check_launch(ctx, "fmm_leaf_of")) return rc;
  if (int rc = exclusive_scan_i32(ctx, ctx->fmm_cnt.p, ctx->fmm_lstart.p, nleaf, ctx->scan_tmp.p)) return rc;
  {  // the fullest leaf (the P2P grid's chunks per leaf)
    std::vector<int32_t> hc(nleaf);
    SC_CUDA(cudaMemcpyAsync(hc.data(), ctx->fmm_cnt.p, sizeof(int32_t) * nleaf, cudaMemcpyDeviceToHost, ctx->stream));
    SC_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->fmm_maxleaf = *std::max_element(hc.begin(), hc.end());
  }
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key_in, key_out, ctx->fmm_idx0.p, ctx->fmm_sidx.p,
                                  static_cast<int>(n), 0, 3 * L, ctx->stream);
  if (int rc = ensure(ctx, ctx->fmm_cubtmp, tmp_bytes + 16)) return rc;
  SC_CUDA(cub::DeviceRadixSort::SortPairs(ctx->fmm_cubtmp.p, tmp_bytes, key_in, key_out, ctx->fmm_idx0.p,
                                          ctx->fmm_sidx.p, static_cast<int>(n), 0, 3 * L, ctx->stream));
  if (int rc = ensure(ctx, ctx->fmm_spos4, std::max<int64_t>(n, 1))) return rc;
  if (ctx->fmm_acc.n < static_cast<size_t>(9 * std::max<int64_t>(n, 1)) || ctx->fmm_acc.p == nullptr) {
    if (int rc = ensure(ctx, ctx->fmm_acc, 9 * std::max<int64_t>(n, 1))) return rc;
    SC_CUDA(cudaMemsetAsync(ctx->fmm_acc.p, 0, sizeof(long long) * 9 * std::max<int64_t>(n, 1), ctx->stream));
  }
  if (int rc = ensure(ctx, ctx->fmm_fx, 4)) return rc;
  if (int rc = ensure(ctx, ctx->fmm_sf4, std::max<int64_t>(n, 1))) return rc;
  gather_sorted_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, ctx->stream>>>(ctx->fmm_sidx.p, n,
                                                                                       ctx->pos4.p, ctx->fmm_spos4.p);
  if (int rc = check_launch(ctx, "fmm_sort")) return rc;
  // expansions of levels 2..L (box offsets per level)
  ctx->fmm_lev_off.assign(L + 2, 0);
  int64_t off = 0;
  for (int l = 0; l <= L + 1; ++l) {
    ctx->fmm_lev_off[l] = off;
    if (l >= 2 && l <= L) off += nbox(l);
  }
  // (offsets relative to level 2: lev_off[l] = boxes of levels 2..l-1)
  const int64_t nb3 = static_cast<int64_t>(nn) * nn * nn;
  const int ncomp = ctx->poly ? 9 : 3;  // node components (fmm_launch's C)
  if (int rc = ensure(ctx, ctx->fmm_M, static_cast<size_t>(off) * nb3 * ncomp)) return rc;
  if (int rc = ensure(ctx, ctx->fmm_L, static_cast<size_t>(off) * nb3 * ncomp)) return rc;
  if (int rc = ensure(ctx, ctx->fmm_lev_off_dev, L + 2)) return rc;
  SC_CUDA(cudaMemcpyAsync(ctx->fmm_lev_off_dev.p, ctx->fmm_lev_off.data(), sizeof(int64_t) * (L + 2),
                          cudaMemcpyHostToDevice, ctx->stream));
  SC_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->fmm_ready = true;
  return 0;
}

bool fmm_uses_library_calls(const sc_ctx* ctx) { return fmm_use_svd(ctx); }

void fmm_destroy_handles(sc_ctx* ctx) {
  if (ctx->cublas) cublasDestroy(static_cast<cublasHandle_t>(ctx->cublas));
  if (ctx->cusolver) cusolverDnDestroy(static_cast<cusolverDnHandle_t>(ctx->cusolver));
  ctx->cublas = nullptr;
  ctx->cusolver = nullptr;
}

int fmm_apply(sc_ctx* ctx, const double4* f4, double mu, double4* u4, const int32_t* done) {
  if (!ctx->fmm_ready) {
    if (int rc = fmm_setup(ctx)) return rc;
  }
  Geom g{ctx->fmm_geom[0], ctx->fmm_geom[1], ctx->fmm_geom[2], ctx->fmm_geom[3], ctx->a_const, ctx->fmm_L_used};
  if (fmm_use_svd(ctx)) {
    int rc = 0;
    const bool pl = ctx->fmm_poly != 0;
    switch (ctx->fmm_order) {
      case 4: rc = pl ? fmm_svd_prepare<4, true>(ctx, g) : fmm_svd_prepare<4, false>(ctx, g); break;
      case 6: rc = pl ? fmm_svd_prepare<6, true>(ctx, g) : fmm_svd_prepare<6, false>(ctx, g); break;
      default: rc = pl ? fmm_svd_prepare<8, true>(ctx, g) : fmm_svd_prepare<8, false>(ctx, g); break;
    }
    if (rc) return rc;
  }
  if (ctx->fmm_poly) switch (ctx->fmm_order) {
      case 4: return fmm_launch<4, true>(ctx, g, f4, mu, u4, done);
      case 6: return fmm_launch<6, true>(ctx, g, f4, mu, u4, done);
      default: return fmm_launch<8, true>(ctx, g, f4, mu, u4, done);
    }
  switch (ctx->fmm_order) {
    case 4: return fmm_launch<4, false>(ctx, g, f4, mu, u4, done);
    case 6: return fmm_launch<6, false>(ctx, g, f4, mu, u4, done);
    default: return fmm_launch<8, false>(ctx, g, f4, mu, u4, done);
  }
}

}  // namespace sc
