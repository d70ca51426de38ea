// Probe (design input): how few CTAs saturate one PCIe link with SM zero-copy (H2D / D2H)?
#include <cuda_runtime.h>
#include <cstdio>
#include <algorithm>
#include <cstring>
template<int U> __global__ void copy16(const uint4* __restrict__ s, uint4* __restrict__ d, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x, i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) v[u] = __ldcg(s + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; u++) d[i + u * stride] = v[u];
  }
  for (; i < n; i += stride) d[i] = s[i];
}
static float timeit(auto fn) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); fn(); cudaDeviceSynchronize();
  float best = 1e9; for (int r = 0; r < 4; r++) { cudaEventRecord(a); fn(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms); }
  return best;
}
int main() {
  size_t B = 1ull << 30; char *h, *d; cudaHostAlloc(&h, B, cudaHostAllocMapped); cudaMalloc(&d, B); memset(h, 1, B);
  auto gb = [&](float ms) { return B / ms / 1e6; };
  for (int grid : {2, 4, 8, 16, 24, 32, 48, 64, 148, 592})
    for (int U : {4, 8}) {
      float a, b;
      if (U == 4) { a = timeit([&] { copy16<4><<<grid, 512>>>((const uint4*)h, (uint4*)d, B / 16); }); b = timeit([&] { copy16<4><<<grid, 512>>>((const uint4*)d, (uint4*)h, B / 16); }); }
      else { a = timeit([&] { copy16<8><<<grid, 512>>>((const uint4*)h, (uint4*)d, B / 16); }); b = timeit([&] { copy16<8><<<grid, 512>>>((const uint4*)d, (uint4*)h, B / 16); }); }
      printf("grid %4d unroll %d: h2d %.2f d2h %.2f\n", grid, U, gb(a), gb(b));
    }
}
