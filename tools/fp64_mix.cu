// fp64_mix.cu -- FP64 pipe ceiling vs operand pattern (tuning probe, not product code).
// A: DFMA with one vector operand (x = x*a + b, a,b uniform)   B: DFMA with 3 vector operands
// C: DMUL/DADD with 2 vector operands                            D: the RPY-like mix (15 DFMA, 8 DMUL, 3 DADD)
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, int iters, double a, double b) {
  double x[8], y[8], z[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    x[c] = threadIdx.x * 1e-3 + c;
    y[c] = 1.0 + 1e-9 * c;
    z[c] = 1e-7 * (c + 1);
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (MODE == 0) x[c] = fma(x[c], a, b);
        if (MODE == 1) x[c] = fma(x[c], y[c], z[c]);
        if (MODE == 2) { x[c] = x[c] * y[c]; x[c] = x[c] + z[c]; }
        if (MODE == 3) {  // 1 MUFU.RSQ64H per 16 DFMA
          double r;
          asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(y[c]));
          y[c] = fma(r, 1e-30, y[c]);
#pragma unroll
          for (int q = 0; q < 15; ++q) x[c] = fma(x[c], y[c], z[c]);
        }
        if (MODE == 4) {  // FP32 seed via integer bit tricks + MUFU.RSQ (fp32), 16 DFMA
          long long bits = __double_as_longlong(y[c]);
          int fb = (int)((bits >> 29) & 0x7FFFFFFF) - ((1023 - 127) << 23);
          float rf = rsqrtf(__int_as_float(fb));
          long long db = ((long long)(__float_as_int(rf) + ((1023 - 127) << 23))) << 29;
          double r = __longlong_as_double(db);
          y[c] = fma(r, 1e-30, y[c]);
#pragma unroll
          for (int q = 0; q < 15; ++q) x[c] = fma(x[c], y[c], z[c]);
        }
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, double* out, int ops_per_chain_iter) {
  int blocks = 148 * 8, threads = 256, iters = 4000;
  k<MODE><<<blocks, threads>>>(out, 10, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double inst = double(iters) * 8 * 8 * ops_per_chain_iter * blocks * threads;
  printf("%-40s %8.3f ms  %.3f T DP-inst/s  (%.1f%% of 18.62)\n", name, ms, inst / ms / 1e9, 100 * inst / ms / 1e9 / 18.62);
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 256 * 8);
  run<0>("A: DFMA, 1 vector operand", out, 1);
  run<1>("B: DFMA, 3 vector operands", out, 1);
  run<2>("C: DMUL+DADD, 2 vector operands", out, 2);
  run<3>("D: 1 MUFU.RSQ64H + 16 DFMA", out, 16);
  run<4>("E: int-trick + MUFU.RSQ fp32 + 16 DFMA", out, 16);
  return 0;
}
