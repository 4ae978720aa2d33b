// FP64 pipe probe for B200 (sm_100a): (1) DFMA-chain throughput on all SMs,
// (2) accuracy of rsqrt.approx.f64 (MUFU.RSQ64H) and of an FP32-seeded rsqrt.
// Standalone tool; not part of the product path.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__global__ void dfma_chain(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ double rsq_approx(double x) {
  double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y;
}
__global__ void rsq_err(const double* x, double* e_approx, double* e_f32, double* e_cubic, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x; if (i >= n) return;
  double v = x[i];
  double exact = 1.0 / sqrt(v);
  double y = rsq_approx(v);
  e_approx[i] = fabs(y - exact) / exact;
  double yf = (double)rsqrtf((float)v);
  e_f32[i] = fabs(yf - exact) / exact;
  // cubic correction from the MUFU seed: e = 1 - v y^2; y' = y + y e (1/2 + 3/8 e)
  double h = v * y; double ee = fma(-h, y, 1.0); double p = fma(0.375, ee, 0.5); double t = y * ee;
  double yc = fma(t, p, y);
  e_cubic[i] = fabs(yc - exact) / exact;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("device %s SMs %d clock(kHz) %d\n", p.name, p.multiProcessorCount, p.clockRate);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 20000;
  double* out; CK(cudaMalloc(&out, sizeof(double) * blocks * threads));
  dfma_chain<<<blocks, threads>>>(out, 100, 0.999999, 1e-7);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    dfma_chain<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    double fl = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("rep %d: %.3f ms  DFMA %.2f TFLOP/s (%.3f Tinst/s)\n", rep, ms, fl / ms / 1e9, fl / 2 / ms / 1e9);
  }
  int n = 1 << 20;
  double *x, *e1, *e2, *e3; CK(cudaMallocManaged(&x, n * 8)); cudaMallocManaged(&e1, n * 8);
  cudaMallocManaged(&e2, n * 8); cudaMallocManaged(&e3, n * 8);
  for (int i = 0; i < n; ++i) x[i] = pow(10.0, -6.0 + 14.0 * (double)i / n) * (1.0 + 0.37 * (((long long)i * 7919) % 1000) / 1000.0);
  rsq_err<<<(n + 255) / 256, 256>>>(x, e1, e2, e3, n); CK(cudaDeviceSynchronize());
  double m1 = 0, m2 = 0, m3 = 0;
  for (int i = 0; i < n; ++i) { m1 = fmax(m1, e1[i]); m2 = fmax(m2, e2[i]); m3 = fmax(m3, e3[i]); }
  printf("rsqrt.approx.f64 max rel err %.3e (2^%.1f)\n", m1, log2(m1));
  printf("rsqrtf seed      max rel err %.3e (2^%.1f)\n", m2, log2(m2));
  printf("approx+cubic     max rel err %.3e (2^%.1f)\n", m3, log2(m3));
  return 0;
}
