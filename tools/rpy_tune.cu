// rpy_tune.cu -- standalone tuning harness for the FP64 RPY pair loop (not product code).
// Times kernel variants (targets/thread, threads/CTA, sources interleaved per step) on a
// C5-shaped problem (N = 262144 spheres, volume fraction 0.3) and checks they agree.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rpy_tune rpy_tune.cu && ./rpy_tune
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int TILE = 128;

__device__ __forceinline__ double rsq_approx(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

struct K {
  double k23a2, m2a2;
  long long near_bits;
};

// Stage-wise evaluation of TPT targets x SU sources: every stage is written for all
// KK = TPT*SU independent chains before the next stage, so the instruction stream interleaves them.
template <int TPT, int NT, int SU>
__global__ void __launch_bounds__(NT) rpy_var(const double4* __restrict__ pos4, const double4* __restrict__ f4,
                                              int64_t npad, int64_t per, K k, double* __restrict__ part,
                                              int64_t nrows) {
  __shared__ double4 sp[TILE], sf[TILE];
  const int tid = threadIdx.x;
  const int split = blockIdx.y;
  const int64_t rbase = static_cast<int64_t>(blockIdx.x) * NT * TPT;
  double4 p[TPT];
  double ax[TPT], ay[TPT], az[TPT], hx[TPT], hy[TPT], hz[TPT], lx[TPT], ly[TPT], lz[TPT];
#pragma unroll
  for (int t = 0; t < TPT; ++t) {
    p[t] = pos4[rbase + tid + t * NT];
    hx[t] = hy[t] = hz[t] = lx[t] = ly[t] = lz[t] = 0.0;
  }
  const int64_t s0 = split * per;
  const int64_t s1 = min(npad, s0 + per);
  for (int64_t sb = s0; sb < s1; sb += TILE) {
    __syncthreads();
    for (int q = tid; q < TILE; q += NT) {
      sp[q] = pos4[sb + q];
      sf[q] = f4[sb + q];
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < TPT; ++t) ax[t] = ay[t] = az[t] = 0.0;
    bool nearflag = false;
#pragma unroll 1
    for (int q = 0; q < TILE; q += SU) {
      constexpr int KK = TPT * SU;
      double4 pj[SU], fj[SU];
#pragma unroll
      for (int u = 0; u < SU; ++u) { pj[u] = sp[q + u]; fj[u] = sf[q + u]; }
      double dx[KK], dy[KK], dz[KK], r2[KK], y[KK], h[KK], e[KK];
#pragma unroll
      for (int c = 0; c < KK; ++c) {
        const int t = c % TPT, u = c / TPT;
        dx[c] = pj[u].x - p[t].x; dy[c] = pj[u].y - p[t].y; dz[c] = pj[u].z - p[t].z;
      }
#pragma unroll
      for (int c = 0; c < KK; ++c) r2[c] = fma(dz[c], dz[c], fma(dy[c], dy[c], dx[c] * dx[c]));
#pragma unroll
      for (int c = 0; c < KK; ++c) y[c] = rsq_approx(r2[c]);
#pragma unroll
      for (int c = 0; c < KK; ++c) h[c] = r2[c] * y[c];
#pragma unroll
      for (int c = 0; c < KK; ++c) e[c] = fma(-h[c], y[c], 1.0);
#pragma unroll
      for (int c = 0; c < KK; ++c) { h[c] = fma(0.375, e[c], 0.5); e[c] = y[c] * e[c]; }
#pragma unroll
      for (int c = 0; c < KK; ++c) y[c] = fma(e[c], h[c], y[c]);           // rinv
#pragma unroll
      for (int c = 0; c < KK; ++c) h[c] = y[c] * y[c];                    // rinv2
#pragma unroll
      for (int c = 0; c < KK; ++c) e[c] = y[c] * h[c];                    // rinv3
      double c1[KK], c2[KK];
#pragma unroll
      for (int c = 0; c < KK; ++c) {
        c1[c] = fma(k.k23a2, e[c], y[c]);
        c2[c] = e[c] * fma(k.m2a2, h[c], 1.0);
        const bool nr = __double_as_longlong(r2[c]) < k.near_bits;
        nearflag |= nr;
        c1[c] = nr ? 0.0 : c1[c];
        c2[c] = nr ? 0.0 : c2[c];
      }
#pragma unroll
      for (int c = 0; c < KK; ++c) {
        const int u = c / TPT;
        h[c] = fma(dz[c], fj[u].z, fma(dy[c], fj[u].y, dx[c] * fj[u].x));
      }
#pragma unroll
      for (int c = 0; c < KK; ++c) c2[c] *= h[c];
#pragma unroll
      for (int c = 0; c < KK; ++c) {
        const int t = c % TPT, u = c / TPT;
        ax[t] = fma(c2[c], dx[c], fma(c1[c], fj[u].x, ax[t]));
        ay[t] = fma(c2[c], dy[c], fma(c1[c], fj[u].y, ay[t]));
        az[t] = fma(c2[c], dz[c], fma(c1[c], fj[u].z, az[t]));
      }
    }
    (void)nearflag;
#pragma unroll
    for (int t = 0; t < TPT; ++t) {
      double s = hx[t] + ax[t], bp = s - hx[t]; lx[t] += (hx[t] - (s - bp)) + (ax[t] - bp); hx[t] = s;
      s = hy[t] + ay[t]; bp = s - hy[t]; ly[t] += (hy[t] - (s - bp)) + (ay[t] - bp); hy[t] = s;
      s = hz[t] + az[t]; bp = s - hz[t]; lz[t] += (hz[t] - (s - bp)) + (az[t] - bp); hz[t] = s;
    }
  }
#pragma unroll
  for (int t = 0; t < TPT; ++t) {
    double* o = part + (split * nrows + rbase + tid + t * NT) * 3;
    o[0] = hx[t] + lx[t]; o[1] = hy[t] + ly[t]; o[2] = hz[t] + lz[t];
  }
}

template <int TPT, int NT, int SU>
double run(const double4* pos, const double4* f, int64_t n, int nsplit, K k, double* part, int reps,
           std::vector<double>& out) {
  int64_t per = ((n + nsplit - 1) / nsplit + TILE - 1) / TILE * TILE;
  dim3 grid(n / (NT * TPT), nsplit);
  rpy_var<TPT, NT, SU><<<grid, NT>>>(pos, f, n, per, k, part, n);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) rpy_var<TPT, NT, SU><<<grid, NT>>>(pos, f, n, per, k, part, n);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaFuncAttributes at; cudaFuncGetAttributes(&at, rpy_var<TPT, NT, SU>);
  out.assign(3 * n, 0.0);
  std::vector<double> h(static_cast<size_t>(nsplit) * n * 3);
  CK(cudaMemcpy(h.data(), part, h.size() * 8, cudaMemcpyDeviceToHost));
  for (int s = 0; s < nsplit; ++s)
    for (int64_t i = 0; i < 3 * n; ++i) out[i] += h[s * 3 * n + i];
  double t = ms / reps;
  double pairs = double(n) * (n - 1);
  printf("TPT=%d NT=%3d SU=%d nsplit=%2d regs=%3d : %8.3f ms  %.3e pairs/s  %.1f%% of 37.2 TF (37 flop/pair)\n", TPT, NT,
         SU, nsplit, at.numRegs, t, pairs / (t / 1e3), 100.0 * 37 * pairs / (t / 1e3) / 37.22e12);
  return t;
}

int main(int argc, char** argv) {
  const int64_t n = 262144;
  const double L = pow(n * 4.0 / 3.0 * M_PI / 0.3, 1.0 / 3.0);
  std::vector<double4> hp(n), hf(n);
  srand(5);
  auto U = [] { return rand() / (RAND_MAX + 1.0); };
  for (int64_t i = 0; i < n; ++i) {
    hp[i] = make_double4(U() * L, U() * L, U() * L, 0.5);
    hf[i] = make_double4(U() - 0.5, U() - 0.5, U() - 0.5, 0.0);
  }
  double4 *pos, *f; double* part;
  CK(cudaMalloc(&pos, n * 32)); CK(cudaMalloc(&f, n * 32));
  CK(cudaMalloc(&part, 64ull * n * 3 * 8));
  CK(cudaMemcpy(pos, hp.data(), n * 32, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(f, hf.data(), n * 32, cudaMemcpyHostToDevice));
  K k; k.k23a2 = 2.0 / 3.0; k.m2a2 = -2.0; double n2 = 4.0; k.near_bits = *reinterpret_cast<long long*>(&n2);
  int reps = argc > 1 ? atoi(argv[1]) : 2;
  std::vector<double> ref, o;
  auto cmp = [&](const char* tag) {
    double num = 0, den = 0;
    for (size_t i = 0; i < ref.size(); ++i) { num += (o[i] - ref[i]) * (o[i] - ref[i]); den += ref[i] * ref[i]; }
    printf("   %s rel diff vs first: %.2e\n", tag, sqrt(num / den));
  };
  run<2, 128, 1>(pos, f, n, 32, k, part, reps, ref);
  run<2, 128, 2>(pos, f, n, 32, k, part, reps, o); cmp("");
  run<1, 256, 2>(pos, f, n, 32, k, part, reps, o); cmp("");
  run<1, 256, 4>(pos, f, n, 32, k, part, reps, o); cmp("");
  run<1, 128, 4>(pos, f, n, 32, k, part, reps, o); cmp("");
  run<2, 64, 2>(pos, f, n, 32, k, part, reps, o); cmp("");
  run<2, 128, 4>(pos, f, n, 32, k, part, reps, o); cmp("");
  run<4, 64, 1>(pos, f, n, 32, k, part, reps, o); cmp("");
  run<4, 64, 2>(pos, f, n, 32, k, part, reps, o); cmp("");
  run<1, 512, 2>(pos, f, n, 32, k, part, reps, o); cmp("");
  return 0;
}
