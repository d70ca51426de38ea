// Probe: which host-side queries invalidate a global-mode capture (design input for the
// capture path's call classification).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
static const char* st(cudaStream_t s) { cudaStreamCaptureStatus c; cudaStreamIsCapturing(s, &c); return c == 0 ? "none" : c == 1 ? "active" : "INVALIDATED"; }
int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  char* d; cudaMalloc(&d, 1 << 20); char* h; cudaHostAlloc(&h, 1 << 20, 0);
  const char* names[] = {"cudaPointerGetAttributes(device)", "cudaPointerGetAttributes(pinned host)", "cudaStreamGetDevice",
                         "cudaGetDevice+cudaSetDevice", "cudaGetLastError", "cudaEventCreate", "cudaDeviceGetAttribute",
                         "cudaPointerGetAttributes(pageable)"};
  for (int relaxed = 0; relaxed < 2; relaxed++)
    for (int t = 0; t < 8; t++) {
      cudaStreamBeginCapture(s, relaxed ? cudaStreamCaptureModeRelaxed : cudaStreamCaptureModeGlobal);
      cudaPointerAttributes a; int dev; cudaEvent_t ev; static char pg[64];
      cudaError_t e = cudaSuccess;
      switch (t) {
        case 0: e = cudaPointerGetAttributes(&a, d); break;
        case 1: e = cudaPointerGetAttributes(&a, h); break;
        case 2: e = cudaStreamGetDevice(s, &dev); break;
        case 3: cudaGetDevice(&dev); e = cudaSetDevice(dev); break;
        case 4: e = cudaGetLastError(); break;
        case 5: e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming); break;
        case 6: e = cudaDeviceGetAttribute(&dev, cudaDevAttrMultiProcessorCount, 0); break;
        case 7: e = cudaPointerGetAttributes(&a, pg); break;
      }
      printf("%-8s %-40s rc=%-30s capture=%s\n", relaxed ? "relaxed" : "global", names[t], cudaGetErrorName(e), st(s));
      cudaGraph_t g; cudaStreamEndCapture(s, &g); cudaGetLastError();
    }
  return 0;
}
