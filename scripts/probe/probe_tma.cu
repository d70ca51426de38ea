// Probe (design input): can TMA bulk copies or L2 prefetch-size hints make SM zero-copy
// reach copy-engine PCIe efficiency on B200? H2D host->HBM and D2H HBM->host, 1 GiB.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <algorithm>
#include <cstring>
#define CK(x) do{cudaError_t e=(x); if(e){printf("ERR %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); exit(1);}}while(0)

__device__ __forceinline__ uint32_t smem_u32(const void* p){ return (uint32_t)__cvta_generic_to_shared(p); }

template<int NS>
__global__ void tma_copy(const char* __restrict__ src, char* __restrict__ dst, size_t ntiles, uint32_t TILE)
{
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar[NS];
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; s++) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t phase = 0;  // bit s
  const size_t stride = gridDim.x;
  size_t t = blockIdx.x;
  int issued = 0;
  auto load = [&](int s, size_t tile) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[s])), "r"(TILE) : "memory");
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      :: "r"(smem_u32(smem + (size_t)s*TILE)), "l"(src + tile*TILE), "r"(TILE), "r"(smem_u32(&bar[s])) : "memory");
  };
  for (int s = 0; s < NS; s++) { size_t tt = t + s*stride; if (tt < ntiles) load(s, tt); }
  for (size_t i = 0; t < ntiles; t += stride, i++) {
    int s = i % NS;
    uint32_t ph = (phase >> s) & 1;
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" :: "r"(smem_u32(&bar[s])), "r"(ph) : "memory");
    phase ^= (1u << s);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(dst + t*TILE), "r"(smem_u32(smem + (size_t)s*TILE)), "r"(TILE) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    size_t tn = t + NS*stride;
    if (tn < ntiles) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      load(s, tn);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template<int U, int HINT>
__global__ void ld_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U-1)*stride < n16; i += U*stride) {
    uint4 v[U];
#pragma unroll
    for (int u=0;u<U;u++) {
      const uint4* p = src + i + u*stride;
      if (HINT == 256) asm volatile("ld.global.cg.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x),"=r"(v[u].y),"=r"(v[u].z),"=r"(v[u].w) : "l"(p));
      else if (HINT == 128) asm volatile("ld.global.cg.L2::128B.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v[u].x),"=r"(v[u].y),"=r"(v[u].z),"=r"(v[u].w) : "l"(p));
      else v[u] = __ldcg(p);
    }
#pragma unroll
    for (int u=0;u<U;u++) dst[i + u*stride] = v[u];
  }
  for (; i < n16; i += stride) dst[i] = src[i];
}

// warp-contiguous: each warp owns a 2 KiB..8 KiB contiguous span (32 lanes x 16 B x U)
template<int U>
__global__ void warp_span_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  const size_t warps = (size_t)gridDim.x * blockDim.x / 32;
  const size_t w = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  const size_t span = 32 * U;
  for (size_t base = w * span; base < n16; base += warps * span) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) v[u] = __ldcg(src + base + u*32 + lane);
#pragma unroll
    for (int u = 0; u < U; u++) dst[base + u*32 + lane] = v[u];
  }
}

static float timeit(int reps, auto fn) {
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  fn(); CK(cudaDeviceSynchronize());
  float best=1e30f;
  for (int r=0;r<reps;r++){ cudaEventRecord(a); fn(); cudaEventRecord(b); CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms,a,b); best=std::min(best,ms);}
  return best;
}

int main() {
  size_t B = 1ull<<30;
  char *h, *d;
  CK(cudaHostAlloc(&h, B, cudaHostAllocMapped));
  CK(cudaMalloc(&d, B));
  memset(h, 3, B); CK(cudaMemset(d, 5, B));
  auto gb = [&](float ms){ return B/ms/1e6; };
  printf("CE h2d %.2f d2h %.2f\n", gb(timeit(5,[&]{cudaMemcpyAsync(d,h,B,cudaMemcpyHostToDevice);})), gb(timeit(5,[&]{cudaMemcpyAsync(h,d,B,cudaMemcpyDeviceToHost);})));
  for (int hint : {0, 128, 256}) {
    float m1, m2;
    if (hint==0) { m1 = timeit(5,[&]{ld_copy<4,0><<<592,512>>>((const uint4*)h,(uint4*)d,B/16);}); m2 = timeit(5,[&]{ld_copy<4,0><<<592,512>>>((const uint4*)d,(uint4*)h,B/16);}); }
    else if (hint==128) { m1 = timeit(5,[&]{ld_copy<4,128><<<592,512>>>((const uint4*)h,(uint4*)d,B/16);}); m2 = timeit(5,[&]{ld_copy<4,128><<<592,512>>>((const uint4*)d,(uint4*)h,B/16);}); }
    else { m1 = timeit(5,[&]{ld_copy<4,256><<<592,512>>>((const uint4*)h,(uint4*)d,B/16);}); m2 = timeit(5,[&]{ld_copy<4,256><<<592,512>>>((const uint4*)d,(uint4*)h,B/16);}); }
    printf("ld hint L2::%d: h2d %.2f d2h %.2f\n", hint, gb(m1), gb(m2));
  }
  for (int grid : {296, 592, 1184}) {
    float m1 = timeit(5,[&]{warp_span_copy<8><<<grid,512>>>((const uint4*)h,(uint4*)d,B/16);});
    float m2 = timeit(5,[&]{warp_span_copy<8><<<grid,512>>>((const uint4*)d,(uint4*)h,B/16);});
    printf("warp-span 4KiB grid %d: h2d %.2f d2h %.2f\n", grid, gb(m1), gb(m2));
  }
  for (uint32_t tile : {4096u, 8192u, 16384u, 32768u}) {
    for (int cps : {1, 2, 4}) {
      const int NS = 4;
      size_t smem = (size_t)NS * tile;
      if (smem > 200*1024) continue;
      CK(cudaFuncSetAttribute(tma_copy<NS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int grid = 148 * cps;
      size_t nt = B / tile;
      float m1 = timeit(5,[&]{tma_copy<NS><<<grid,32,smem>>>(h,d,nt,tile);});
      cudaError_t e = cudaGetLastError(); if (e) { printf("tma err %s\n", cudaGetErrorString(e)); return 1; }
      float m2 = timeit(5,[&]{tma_copy<NS><<<grid,32,smem>>>(d,h,nt,tile);});
      printf("TMA bulk tile %u NS %d grid %d: h2d %.2f d2h %.2f\n", tile, NS, grid, gb(m1), gb(m2));
    }
  }
  // correctness spot check of TMA path
  memset(h, 0, B); for (size_t i=0;i<B;i+=4096) h[i]=(char)(i>>12);
  tma_copy<4><<<148,32,4*16384>>>(h,d,B/16384,16384); CK(cudaDeviceSynchronize());
  char* chk = (char*)malloc(B); CK(cudaMemcpy(chk, d, B, cudaMemcpyDeviceToHost));
  printf("tma check %s\n", memcmp(chk, h, B)==0 ? "OK" : "MISMATCH");
  return 0;
}
