// Probe (design input): DEVICE rate of a scattered 131072 x 32 KiB copy issued as
// cudaMemcpyBatchAsync split over k streams (host issue hidden behind a gate kernel), both
// directions; plus the same with the device side packed (contiguous) so only the host side
// is scattered.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>
__global__ void gate(long long ns) { long long t0 = clock64(); while (clock64() - t0 < ns) {} }
int main() {
  const size_t seg = 32768, n = 131072, B = seg * n;
  char *h, *d; cudaHostAlloc(&h, 2 * B, cudaHostAllocMapped); cudaMalloc(&d, 2 * B);
  std::vector<size_t> perm(2 * n); for (size_t i = 0; i < 2 * n; i++) perm[i] = i;
  std::shuffle(perm.begin(), perm.end(), std::mt19937(7));
  std::vector<size_t> dsamp(perm.begin(), perm.begin() + n);   // device blocks: a sorted sample
  std::shuffle(perm.begin(), perm.end(), std::mt19937(8));
  std::sort(dsamp.begin(), dsamp.end());
  cudaStream_t st[8]; for (int i = 0; i < 8; i++) cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
  cudaStream_t g; cudaStreamCreateWithFlags(&g, cudaStreamNonBlocking);
  cudaEvent_t go, end[8]; cudaEventCreate(&go); for (auto& e : end) cudaEventCreate(&e);
  cudaMemcpyAttributes at = {}; at.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
  for (int packed = 0; packed < 2; packed++)
    for (int dir = 0; dir < 2; dir++)
      for (int k : {1, 2, 3, 4, 8}) {
        std::vector<void*> dsts(n), srcs(n); std::vector<size_t> sz(n, seg);
        for (size_t i = 0; i < n; i++) {
          char* hp = h + perm[i] * seg;
          char* dp = d + (packed ? i : dsamp[i]) * seg;
          if (dir == 0) { dsts[i] = dp; srcs[i] = hp; } else { dsts[i] = hp; srcs[i] = dp; }
        }
        float best = 1e9;
        for (int rep = 0; rep < 3; rep++) {
          cudaDeviceSynchronize();
          gate<<<1, 1, 0, g>>>(400ll * 1000 * 1000 * 2);   // ~400 ms at ~2 GHz
          cudaEventRecord(go, g);
          for (int t = 0; t < k; t++) {
            cudaStreamWaitEvent(st[t], go, 0);
            size_t lo = n * t / k, hi = n * (t + 1) / k, idx = 0, fail = 0;
            cudaMemcpyBatchAsync(dsts.data() + lo, srcs.data() + lo, sz.data() + lo, hi - lo, &at, &idx, 1, &fail, st[t]);
            cudaEventRecord(end[t], st[t]);
          }
          cudaDeviceSynchronize();
          float ms = 0;
          for (int t = 0; t < k; t++) { float m; cudaEventElapsedTime(&m, go, end[t]); ms = std::max(ms, m); }
          best = std::min(best, ms);
        }
        printf("%s %s streams %d: %.2f GB/s (%.1f ms) %s\n", dir ? "d2h" : "h2d", packed ? "dev-packed" : "dev-scattered",
               k, B / best / 1e6, best, cudaGetErrorString(cudaGetLastError()));
      }
  // contiguous reference
  for (int dir = 0; dir < 2; dir++) {
    float best = 1e9;
    for (int rep = 0; rep < 3; rep++) {
      cudaEventRecord(go, st[0]);
      if (dir == 0) cudaMemcpyAsync(d, h, B, cudaMemcpyHostToDevice, st[0]); else cudaMemcpyAsync(h, d, B, cudaMemcpyDeviceToHost, st[0]);
      cudaEventRecord(end[0], st[0]); cudaEventSynchronize(end[0]);
      float m; cudaEventElapsedTime(&m, go, end[0]); best = std::min(best, m);
    }
    printf("%s contiguous 4 GiB: %.2f GB/s\n", dir ? "d2h" : "h2d", B / best / 1e6);
  }
}
