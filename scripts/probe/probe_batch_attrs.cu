// Probe (design input): host issue time of one cudaMemcpyBatchAsync of 131,072 scattered
// 32 KiB copies (the config-3 KV fetch shape) vs its attributes: source access order and
// location hints. Device time measured after the issue (events), issue time by the host clock.
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <vector>
#include <algorithm>
int main() {
  setvbuf(stdout, NULL, _IONBF, 0);
  const size_t n = 131072, sb = 32768, pool = 2 * n * sb;
  char *h, *d; cudaHostAlloc(&h, pool, cudaHostAllocPortable | cudaHostAllocMapped); cudaMalloc(&d, n * sb);
  memset(h, 1, pool);
  std::vector<size_t> slot(2 * n); for (size_t i = 0; i < 2 * n; i++) slot[i] = i;
  unsigned long long x = 0x4D4D41;
  for (size_t i = 2 * n - 1; i > 0; i--) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; std::swap(slot[i], slot[x % (i + 1)]); }
  std::vector<void*> dst(n), src(n); std::vector<size_t> len(n, sb);
  for (size_t i = 0; i < n; i++) { src[i] = h + slot[i] * sb; dst[i] = d + i * sb; }
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  struct V { const char* name; int order; int hints; unsigned flags; } vs[] = {
    {"order=stream, no hints", cudaMemcpySrcAccessOrderStream, 0, 0},
    {"order=stream, hints host->dev", cudaMemcpySrcAccessOrderStream, 1, 0},
    {"order=any, no hints", cudaMemcpySrcAccessOrderAny, 0, 0},
    {"order=any, hints", cudaMemcpySrcAccessOrderAny, 1, 0},
    {"order=stream, hints, prefer-overlap", cudaMemcpySrcAccessOrderStream, 1, cudaMemcpyFlagPreferOverlapWithCompute},
  };
  for (auto& v : vs) {
    cudaMemcpyAttributes at; memset(&at, 0, sizeof at);
    at.srcAccessOrder = (cudaMemcpySrcAccessOrder)v.order; at.flags = v.flags;
    if (v.hints) { at.srcLocHint.type = cudaMemLocationTypeHost; at.dstLocHint.type = cudaMemLocationTypeDevice; at.dstLocHint.id = 0; }
    double best_issue = 1e9; float best_dev = 1e9;
    for (int rep = 0; rep < 4; rep++) {
      size_t idx = 0, fail = 0;
      cudaStreamSynchronize(s);
      cudaEventRecord(a, s);
      auto t0 = std::chrono::steady_clock::now();
      cudaError_t e = cudaMemcpyBatchAsync(dst.data(), src.data(), len.data(), n, &at, &idx, 1, &fail, s);
      double issue = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      cudaEventRecord(b, s); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (e != cudaSuccess) { printf("%s: %s\n", v.name, cudaGetErrorString(e)); cudaGetLastError(); break; }
      if (rep) { best_issue = std::min(best_issue, issue); best_dev = std::min(best_dev, ms); }
    }
    printf("%-40s issue %7.2f ms  call->done %7.2f ms  %6.2f GB/s\n", v.name, best_issue, best_dev, n * sb / (best_dev * 1e-3) / 1e9);
  }
  return 0;
}
