// Probe (design input): 32-byte vector loads/stores (ld/st.global.v8.b32, sm_100) for the
// zero-copy path, H2D and D2H, vs 16-byte vectors.
#include <cuda_runtime.h>
#include <cstdio>
#include <algorithm>
#include <cstring>
struct alignas(32) u8x32 { unsigned x[8]; };
__device__ __forceinline__ u8x32 ld32(const u8x32* p) {
  u8x32 v;
  asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.x[0]), "=r"(v.x[1]), "=r"(v.x[2]), "=r"(v.x[3]), "=r"(v.x[4]), "=r"(v.x[5]), "=r"(v.x[6]), "=r"(v.x[7]) : "l"(p));
  return v;
}
__device__ __forceinline__ void st32(u8x32* p, const u8x32& v) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               :: "l"(p), "r"(v.x[0]), "r"(v.x[1]), "r"(v.x[2]), "r"(v.x[3]), "r"(v.x[4]), "r"(v.x[5]), "r"(v.x[6]), "r"(v.x[7]) : "memory");
}
template<int U> __global__ void copy32(const u8x32* __restrict__ s, u8x32* __restrict__ d, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x, i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    u8x32 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) v[u] = ld32(s + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; u++) st32(d + i + u * stride, v[u]);
  }
  for (; i < n; i += stride) st32(d + i, ld32(s + i));
}
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
  float best = 1e9; for (int r = 0; r < 5; r++) { cudaEventRecord(a); fn(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms); }
  return best;
}
int main() {
  size_t B = 1ull << 30; char *h, *d; cudaHostAlloc(&h, B, cudaHostAllocMapped); cudaMalloc(&d, B); memset(h, 1, B);
  auto gb = [&](float ms) { return B / ms / 1e6; };
  for (int grid : {296, 592}) {
    printf("grid %d  16B: h2d %.2f d2h %.2f | 32B: h2d %.2f d2h %.2f\n", grid,
      gb(timeit([&] { copy16<4><<<grid, 512>>>((const uint4*)h, (uint4*)d, B / 16); })),
      gb(timeit([&] { copy16<4><<<grid, 512>>>((const uint4*)d, (uint4*)h, B / 16); })),
      gb(timeit([&] { copy32<4><<<grid, 512>>>((const u8x32*)h, (u8x32*)d, B / 32); })),
      gb(timeit([&] { copy32<4><<<grid, 512>>>((const u8x32*)d, (u8x32*)h, B / 32); })));
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
