// Probe (design input): per-chunk cost of copy-engine DMAs and stream memory operations.
// 1 GiB H2D as n chunks of C bytes: (a) one stream, DMAs only; (b) two streams alternating;
// (c) one stream with a write memop after every DMA; (d) two streams, wait + DMA + write per
// chunk with the waits already satisfied; (e) four streams, DMAs only.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <algorithm>
#include <cstring>
#define CK(x) do{cudaError_t e=(x); if(e){printf("ERR %s @%d: %s\n",#x,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)
typedef CUresult (*memop_t)(CUstream, CUdeviceptr, cuuint64_t, unsigned);
typedef CUresult (*batch_t)(CUstream, unsigned, CUstreamBatchMemOpParams*, unsigned);

int main() {
  setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 1);
  const size_t B = 1ull << 30;
  char *h, *d; CK(cudaHostAlloc(&h, B, cudaHostAllocMapped)); CK(cudaMalloc(&d, B));
  unsigned long long* flags; CK(cudaMalloc(&flags, 4096)); CK(cudaMemset(flags, 0, 4096));
  memop_t w64 = nullptr, wt64 = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuStreamWriteValue64", (void**)&w64, 12000, cudaEnableDefault, &q);
  cudaGetDriverEntryPointByVersion("cuStreamWaitValue64", (void**)&wt64, 12000, cudaEnableDefault, &q);
  batch_t bmo = nullptr; cudaGetDriverEntryPointByVersion("cuStreamBatchMemOp", (void**)&bmo, 12000, cudaEnableDefault, &q);
  cudaStream_t st[4]; for (int i = 0; i < 4; i++) CK(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
  cudaEvent_t a, b, f, j[4]; cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreateWithFlags(&f, cudaEventDisableTiming);
  for (int i = 0; i < 4; i++) cudaEventCreateWithFlags(&j[i], cudaEventDisableTiming);
  for (size_t C : {256ull << 10, 1ull << 20, 4ull << 20, 16ull << 20}) {
    const size_t n = B / C;
    for (int variant = 0; variant < 6; variant++) {
      int ns = (variant == 0 || variant == 2) ? 1 : (variant == 4 ? 4 : 2);
      float best = 1e9;
      for (int rep = 0; rep < 4; rep++) {
        cudaEventRecord(a, st[0]); cudaEventRecord(f, st[0]);
        for (int i = 1; i < ns; i++) cudaStreamWaitEvent(st[i], f, 0);
        for (size_t c = 0; c < n; c++) {
          cudaStream_t s = st[c % ns];
          if (variant == 3) wt64((CUstream)s, (CUdeviceptr)&flags[c % 2], 0, CU_STREAM_WAIT_VALUE_GEQ);
          if (variant == 5) {
            CUstreamBatchMemOpParams pr[2]; memset(pr, 0, sizeof pr); unsigned k = 0;
            if (c >= 2) { pr[k].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64; pr[k].writeValue.address = (CUdeviceptr)&flags[8 + c % 2]; pr[k].writeValue.value64 = c - 1; k++; }
            pr[k].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_64; pr[k].waitValue.address = (CUdeviceptr)&flags[c % 2]; pr[k].waitValue.value64 = 0; pr[k].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ; k++;
            bmo((CUstream)s, k, pr, 0);
          }
          cudaMemcpyAsync(d + c * C, h + c * C, C, cudaMemcpyHostToDevice, s);
          if (variant == 2 || variant == 3) w64((CUstream)s, (CUdeviceptr)&flags[8 + c % 2], c + 1, 0);
        }
        for (int i = 1; i < ns; i++) { cudaEventRecord(j[i], st[i]); cudaStreamWaitEvent(st[0], j[i], 0); }
        cudaEventRecord(b, st[0]); CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b); if (rep) best = std::min(best, ms);
      }
      const char* name[] = {"1 stream DMA", "2 streams DMA", "1 stream DMA+write", "2 streams wait+DMA+write", "4 streams DMA", "2 streams batch(write,wait)+DMA"};
      printf("C=%5zu KiB  %-26s %6.2f GB/s  %6.2f us/chunk\n", C >> 10, name[variant], B / best / 1e6, best * 1e3 / n);
    }
  }
  return 0;
}
