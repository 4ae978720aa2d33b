// scan.cu -- exclusive prefix sum of int32 arrays (cell counts, pair counts,
// incidence degrees).  Three-phase block scan, recursive over block totals.
#include "sc_internal.h"

namespace sc {
namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 2 * kScanThreads;  // elements per block

__device__ __forceinline__ int32_t warp_incl(int32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int32_t u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// out[k] = sum_{m<k} in[m] within the block; block total -> sums[blockIdx.x]
__global__ void scan_block(const int32_t* __restrict__ in, int32_t* __restrict__ out, int64_t n,
                           int32_t* __restrict__ sums) {
  __shared__ int32_t wsum[kScanThreads / 32];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanItems;
  const int t = threadIdx.x;
  const int64_t k0 = base + 2 * t, k1 = k0 + 1;
  const int32_t a = k0 < n ? in[k0] : 0;
  const int32_t b = k1 < n ? in[k1] : 0;
  int32_t v = a + b;
  int32_t inc = warp_incl(v);
  const int warp = t >> 5, lane = t & 31;
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int32_t w = wsum[lane];
    w = warp_incl(w);
    wsum[lane] = w;
  }
  __syncthreads();
  const int32_t before = (warp > 0 ? wsum[warp - 1] : 0) + inc - v;
  if (k0 < n) out[k0] = before;
  if (k1 < n) out[k1] = before + a;
  if (t == kScanThreads - 1) sums[blockIdx.x] = before + v;
}

__global__ void scan_add(int32_t* __restrict__ out, int64_t n, const int32_t* __restrict__ offs) {
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanItems;
  const int32_t o = offs[blockIdx.x];
  for (int k = threadIdx.x; k < kScanItems; k += blockDim.x) {
    const int64_t idx = base + k;
    if (idx < n) out[idx] += o;
  }
}

__global__ void scan_total(const int32_t* __restrict__ in, int32_t* __restrict__ out, int64_t n) {
  // out[n] = out[n-1] + in[n-1]
  out[n] = n > 0 ? out[n - 1] + in[n - 1] : 0;
}

int scan_rec(sc_ctx* ctx, const int32_t* in, int32_t* out, int64_t n, int32_t* tmp) {
  const int64_t nb = (n + kScanItems - 1) / kScanItems;
  if (nb == 0) return 0;
  int32_t* sums = tmp;
  int32_t* sums_scan = tmp + nb + 1;
  timer_begin(ctx, SC_K_MISC);
  scan_block<<<static_cast<unsigned>(nb), kScanThreads, 0, ctx->stream>>>(in, out, n, sums);
  timer_end(ctx, SC_K_MISC);
  if (int rc = check_launch(ctx, "scan_block")) return rc;
  if (nb > 1) {
    if (int rc = scan_rec(ctx, sums, sums_scan, nb, sums_scan + nb + 1)) return rc;
    timer_begin(ctx, SC_K_MISC);
    scan_add<<<static_cast<unsigned>(nb), 256, 0, ctx->stream>>>(out, n, sums_scan);
    timer_end(ctx, SC_K_MISC);
    if (int rc = check_launch(ctx, "scan_add")) return rc;
  }
  return 0;
}

}  // namespace

size_t scan_tmp_size(int64_t n) {
  size_t total = 0;
  int64_t m = n;
  while (true) {
    const int64_t nb = (m + kScanItems - 1) / kScanItems;
    total += 2 * (nb + 1);
    if (nb <= 1) break;
    m = nb;
  }
  return total + 16;
}

int exclusive_scan_i32(sc_ctx* ctx, const int32_t* in, int32_t* out, int64_t n, int32_t* tmp) {
  if (n > 0) {
    if (int rc = scan_rec(ctx, in, out, n, tmp)) return rc;
  }
  timer_begin(ctx, SC_K_MISC);
  scan_total<<<1, 1, 0, ctx->stream>>>(in, out, n);
  timer_end(ctx, SC_K_MISC);
  return check_launch(ctx, "scan_total");
}

}  // namespace sc
