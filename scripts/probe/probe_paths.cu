// Path probe for a single B200 (design input, not product code): CE vs SM zero-copy
// vs concurrent CE+ZC over one PCIe link, scattered 32 KiB segments, stream memops.
#include <cuda_runtime.h>
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cstring>
#define CK(x) do{cudaError_t e=(x); if(e){printf("ERR %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); exit(1);}}while(0)

template<int U>
__global__ void zc_copy(const uint4* __restrict__ src, uint4* __restrict__ dst, size_t n16) {
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = tid;
  for (; i + (U-1)*stride < n16; i += U*stride) {
    uint4 v[U];
#pragma unroll
    for (int u=0;u<U;u++) v[u] = src[i + u*stride];
#pragma unroll
    for (int u=0;u<U;u++) dst[i + u*stride] = v[u];
  }
  for (; i < n16; i += stride) dst[i] = src[i];
}
// one warp-group per segment chunk: segments of seg bytes, src/dst offsets from tables
__global__ void zc_gather(const char* __restrict__ hbase, char* __restrict__ dbase, const long long* __restrict__ soff,
                          const long long* __restrict__ doff, int nseg, int seg) {
  int warps = blockDim.x/32, w = threadIdx.x/32, lane = threadIdx.x%32;
  for (long long s = blockIdx.x*(long long)warps + w; s < nseg; s += (long long)gridDim.x*warps) {
    const uint4* sp = (const uint4*)(hbase + soff[s]); uint4* dp = (uint4*)(dbase + doff[s]);
    int n16 = seg/16;
    for (int i = lane; i < n16; i += 32*8) {
      uint4 v[8];
#pragma unroll
      for (int u=0;u<8;u++) if (i+u*32<n16) v[u]=sp[i+u*32];
#pragma unroll
      for (int u=0;u<8;u++) if (i+u*32<n16) dp[i+u*32]=v[u];
    }
  }
}

static float timeit(cudaStream_t s, int reps, auto fn) {
  cudaEvent_t a,b; cudaEventCreate(&a); cudaEventCreate(&b);
  fn(); CK(cudaStreamSynchronize(s)); CK(cudaDeviceSynchronize());
  float best=1e30f;
  for (int r=0;r<reps;r++){ cudaEventRecord(a,s); fn(); cudaEventRecord(b,s); CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms,a,b); best=std::min(best,ms);}
  return best;
}

int main() {
  size_t B = 1ull<<30;
  char *h, *hd; char* d; char* d2;
  CK(cudaHostAlloc(&h, B, cudaHostAllocMapped|cudaHostAllocPortable));
  CK(cudaHostAlloc(&hd, B, cudaHostAllocMapped|cudaHostAllocPortable));
  memset(h, 1, B); memset(hd, 2, B);
  CK(cudaMalloc(&d, B)); CK(cudaMalloc(&d2, B));
  char* hdev; CK(cudaHostGetDevicePointer((void**)&hdev, h, 0));
  char* hddev; CK(cudaHostGetDevicePointer((void**)&hddev, hd, 0));
  printf("hostptr==devptr %d\n", (int)(hdev==h));
  int v; cudaDeviceGetAttribute(&v, cudaDevAttrAsyncEngineCount, 0); printf("asyncEngineCount %d\n", v);
  cudaDeviceGetAttribute(&v, cudaDevAttrCanUseHostPointerForRegisteredMem, 0); printf("canUseHostPtrForRegistered %d\n", v);
  cudaDeviceGetAttribute(&v, cudaDevAttrPageableMemoryAccess, 0); printf("pageableMemoryAccess %d\n", v);
  CUdevice cd; cuInit(0); cuDeviceGet(&cd, 0);
  cuDeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, cd); printf("memops64 %d\n", v);
  cuDeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_WAIT_VALUE_NOR, cd); printf("waitNOR %d\n", v);
  cudaStream_t s[4]; for (int i=0;i<4;i++) CK(cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking));
  auto gbps=[&](size_t bytes,float ms){return bytes/ms/1e6;};
  float ms;
  ms = timeit(s[0], 8, [&]{ cudaMemcpyAsync(d, h, B, cudaMemcpyHostToDevice, s[0]);}); printf("CE h2d 1GiB: %.2f GB/s\n", gbps(B,ms));
  ms = timeit(s[0], 8, [&]{ cudaMemcpyAsync(hd, d, B, cudaMemcpyDeviceToHost, s[0]);}); printf("CE d2h 1GiB: %.2f GB/s\n", gbps(B,ms));
  // simultaneous H2D + D2H (duplex)
  { cudaEvent_t e0, e1, j; cudaEventCreate(&e0); cudaEventCreate(&e1); cudaEventCreate(&j);
    ms = timeit(s[0], 5, [&]{ cudaEventRecord(e0, s[0]); cudaStreamWaitEvent(s[1], e0); cudaMemcpyAsync(d, h, B, cudaMemcpyHostToDevice, s[0]); cudaMemcpyAsync(hd, d2, B, cudaMemcpyDeviceToHost, s[1]); cudaEventRecord(j, s[1]); cudaStreamWaitEvent(s[0], j);});
    printf("CE duplex h2d+d2h: %.2f GB/s total\n", gbps(2*B,ms)); }
  // multi-stream CE H2D
  for (int ns : {2,4}) {
    cudaEvent_t f, j[4]; cudaEventCreate(&f); for(int i=0;i<4;i++) cudaEventCreate(&j[i]);
    ms = timeit(s[0], 5, [&]{ cudaEventRecord(f, s[0]); size_t part=B/ns; for (int i=0;i<ns;i++){ if(i) cudaStreamWaitEvent(s[i], f); cudaMemcpyAsync(d+i*part, h+i*part, part, cudaMemcpyHostToDevice, s[i]); if(i){cudaEventRecord(j[i], s[i]); cudaStreamWaitEvent(s[0], j[i]);} }});
    printf("CE h2d %d streams: %.2f GB/s\n", ns, gbps(B,ms));
  }
  size_t n16 = B/16;
  for (int grid : {148, 296, 592, 1184}) for (int thr : {256, 512, 1024}) {
    ms = timeit(s[0], 5, [&]{ zc_copy<4><<<grid, thr, 0, s[0]>>>((const uint4*)hdev, (uint4*)d, n16); });
    float ms2 = timeit(s[0], 5, [&]{ zc_copy<4><<<grid, thr, 0, s[0]>>>((const uint4*)d2, (uint4*)hddev, n16); });
    printf("ZC grid %d thr %d: h2d %.2f GB/s  d2h %.2f GB/s\n", grid, thr, gbps(B,ms), gbps(B,ms2));
  }
  ms = timeit(s[0], 5, [&]{ zc_copy<8><<<296, 512, 0, s[0]>>>((const uint4*)hdev, (uint4*)d, n16); }); printf("ZC U8 h2d %.2f\n", gbps(B,ms));
  ms = timeit(s[0], 5, [&]{ zc_copy<4><<<1184, 512, 0, s[0]>>>((const uint4*)d2, (uint4*)d, n16); }); printf("dev copy kernel %.2f GB/s (rd+wr %.2f)\n", gbps(B,ms), gbps(2*B,ms));
  // CE + ZC concurrent, split fraction f to ZC
  for (int pct : {5, 10, 20, 30, 50}) {
    size_t zb = (B * pct / 100) & ~size_t(4095);
    cudaEvent_t f, j; cudaEventCreate(&f); cudaEventCreate(&j);
    ms = timeit(s[0], 5, [&]{ cudaEventRecord(f, s[0]); cudaStreamWaitEvent(s[1], f);
      cudaMemcpyAsync(d, h, B-zb, cudaMemcpyHostToDevice, s[0]);
      zc_copy<4><<<148, 512, 0, s[1]>>>((const uint4*)(hdev+(B-zb)), (uint4*)(d+(B-zb)), zb/16);
      cudaEventRecord(j, s[1]); cudaStreamWaitEvent(s[0], j); });
    float ms2 = timeit(s[0], 5, [&]{ cudaEventRecord(f, s[0]); cudaStreamWaitEvent(s[1], f);
      cudaMemcpyAsync(hd, d, B-zb, cudaMemcpyDeviceToHost, s[0]);
      zc_copy<4><<<148, 512, 0, s[1]>>>((const uint4*)(d+(B-zb)), (uint4*)(hddev+(B-zb)), zb/16);
      cudaEventRecord(j, s[1]); cudaStreamWaitEvent(s[0], j); });
    printf("CE+ZC split %d%% to ZC: h2d %.2f GB/s  d2h %.2f GB/s\n", pct, gbps(B,ms), gbps(B,ms2));
  }
  // scattered 32 KiB segments: 32768 segs (1 GiB) in a 2 GiB-equivalent permuted pool (here: permuted inside B)
  int seg = 32768; int nseg = B/seg; std::vector<long long> so(nseg), dofs(nseg);
  for (int i=0;i<nseg;i++){ so[i]=(long long)i*seg; dofs[i]=(long long)i*seg; }
  srand(7); for (int i=nseg-1;i>0;i--){ int k=rand()%(i+1); std::swap(so[i],so[k]); }
  for (int i=nseg-1;i>0;i--){ int k=rand()%(i+1); std::swap(dofs[i],dofs[k]); }
  ms = timeit(s[0], 3, [&]{ for (int i=0;i<nseg;i++) cudaMemcpyAsync(d+dofs[i], h+so[i], seg, cudaMemcpyHostToDevice, s[0]); });
  printf("per-seg cudaMemcpyAsync 32KiB x %d: %.2f GB/s\n", nseg, gbps(B,ms));
  long long *dso, *ddo; CK(cudaMalloc(&dso, nseg*8)); CK(cudaMalloc(&ddo, nseg*8));
  cudaMemcpy(dso, so.data(), nseg*8, cudaMemcpyHostToDevice); cudaMemcpy(ddo, dofs.data(), nseg*8, cudaMemcpyHostToDevice);
  for (int grid : {148, 296, 592}) { ms = timeit(s[0], 5, [&]{ zc_gather<<<grid, 512, 0, s[0]>>>(hdev, d, dso, ddo, nseg, seg); });
    printf("ZC gather grid %d: %.2f GB/s\n", grid, gbps(B,ms)); }
  // stream memop latency: write/wait chain
  { auto wr = (CUresult(*)(CUstream,CUdeviceptr,cuuint64_t,unsigned))nullptr; cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPointByVersion("cuStreamWriteValue64", (void**)&wr, 12000, cudaEnableDefault, &q)); printf("entry writeValue64 %p q=%d\n", (void*)wr, (int)q);
    unsigned long long* flag; CK(cudaMalloc(&flag, 64)); cudaMemset(flag, 0, 64);
    ms = timeit(s[0], 3, [&]{ for (int i=0;i<1000;i++) wr(s[0], (CUdeviceptr)flag, i, 0); });
    printf("1000 writeValue64: %.3f ms\n", ms); }
  // API issue cost of cudaMemcpyAsync (host side)
  printf("done\n");
}
