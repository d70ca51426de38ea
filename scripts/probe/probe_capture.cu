// Probe (design input): which calls a library may make while the caller's stream is being
// captured (global capture mode, as torch.cuda.graph uses by default).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
__global__ void k(int* p) { p[threadIdx.x] += 1; }
int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  cudaStream_t s, t; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking);
  int* d; cudaMalloc(&d, 4096); cudaMemset(d, 0, 4096); cudaDeviceSynchronize();
  char* h0; cudaHostAlloc(&h0, 1 << 20, cudaHostAllocPortable | cudaHostAllocMapped);
  cudaEvent_t fork, join; cudaEventCreateWithFlags(&fork, cudaEventDisableTiming); cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
  cudaGraph_t g;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  if (getenv("PROBE_ALLOC")) {
    void* hp = nullptr; cudaError_t e1 = cudaHostAlloc(&hp, 1 << 20, cudaHostAllocPortable | cudaHostAllocMapped);
    printf("cudaHostAlloc during capture: %s\n", cudaGetErrorString(e1)); cudaGetLastError();
    void* dm = nullptr; cudaError_t e2 = cudaMalloc(&dm, 1 << 20);
    printf("cudaMalloc during capture: %s\n", cudaGetErrorString(e2)); cudaGetLastError();
  }
  void* da = nullptr; cudaError_t e3 = cudaMallocAsync(&da, 1 << 20, s);
  printf("cudaMallocAsync on the capturing stream: %s\n", cudaGetErrorString(e3)); cudaGetLastError();
  cudaError_t e4 = da ? cudaMemcpyAsync(da, h0, 1 << 20, cudaMemcpyHostToDevice, s) : cudaErrorInvalidValue;
  printf("memcpy pinned->graph-alloc on the capturing stream: %s\n", cudaGetErrorString(e4)); cudaGetLastError();
  cudaEventRecord(fork, s); cudaError_t e5 = cudaStreamWaitEvent(t, fork, 0);
  printf("fork to a side stream: %s\n", cudaGetErrorString(e5));
  k<<<1, 32, 0, t>>>(d); cudaError_t e6 = cudaGetLastError();
  printf("kernel on the side stream: %s\n", cudaGetErrorString(e6));
  cudaEventRecord(join, t); cudaStreamWaitEvent(s, join, 0);
  cudaError_t e7 = da ? cudaFreeAsync(da, s) : cudaSuccess;
  printf("cudaFreeAsync on the capturing stream: %s\n", cudaGetErrorString(e7)); cudaGetLastError();
  cudaStreamCaptureStatus st; unsigned long long id; cudaGraph_t cg = nullptr;
  cudaError_t e8 = cudaStreamGetCaptureInfo(s, &st, &id, &cg, nullptr, nullptr);
  printf("capture info: %s status=%d graph=%p\n", cudaGetErrorString(e8), (int)st, (void*)cg);
  cudaError_t e9 = cudaStreamEndCapture(s, &g);
  printf("end capture: %s\n", cudaGetErrorString(e9));
  if (e9 != cudaSuccess) return 1;
  cudaGraphExec_t x; cudaError_t e10 = cudaGraphInstantiate(&x, g, 0);
  printf("instantiate: %s\n", cudaGetErrorString(e10));
  for (int i = 0; i < 3; i++) cudaGraphLaunch(x, s);
  cudaError_t e11 = cudaStreamSynchronize(s);
  int v = 0; cudaMemcpy(&v, d, 4, cudaMemcpyDeviceToHost);
  printf("3 replays: %s, counter %d\n", cudaGetErrorString(e11), v);
  return 0;
}
