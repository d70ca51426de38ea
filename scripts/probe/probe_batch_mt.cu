// Probe (design input): does issuing cudaMemcpyBatchAsync from several host threads (one
// stream each) cut the host issue time of a 131072 x 32 KiB scattered H2D?
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>
#include <random>
#include <algorithm>
int main() {
  const size_t seg = 32768, n = 131072, B = seg * n;
  char *h, *d; cudaHostAlloc(&h, 2 * B, cudaHostAllocMapped); cudaMalloc(&d, B);
  std::vector<size_t> perm(2 * n); for (size_t i = 0; i < 2 * n; i++) perm[i] = i;
  std::shuffle(perm.begin(), perm.end(), std::mt19937(7));
  std::vector<void*> dsts(n), srcs(n); std::vector<size_t> sz(n, seg);
  for (size_t i = 0; i < n; i++) { dsts[i] = d + i * seg; srcs[i] = h + perm[i] * seg; }
  cudaStream_t st[8]; for (int i = 0; i < 8; i++) cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
  cudaMemcpyAttributes at = {}; at.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
  for (int T : {1, 2, 4, 8}) {
    for (int rep = 0; rep < 3; rep++) {
      cudaDeviceSynchronize();
      auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> th; std::vector<double> issue(T);
      for (int t = 0; t < T; t++) th.emplace_back([&, t] {
        auto a = std::chrono::steady_clock::now();
        size_t lo = n * t / T, hi = n * (t + 1) / T, idx = 0, fail = 0;
        cudaMemcpyBatchAsync(dsts.data() + lo, srcs.data() + lo, sz.data() + lo, hi - lo, &at, &idx, 1, &fail, st[t]);
        issue[t] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
      });
      for (auto& x : th) x.join();
      auto t1 = std::chrono::steady_clock::now();
      cudaDeviceSynchronize();
      auto t2 = std::chrono::steady_clock::now();
      double im = std::chrono::duration<double, std::milli>(t1 - t0).count();
      double wm = std::chrono::duration<double, std::milli>(t2 - t0).count();
      if (rep) printf("threads %d: issue %.1f ms (per-thread max %.1f), wall %.1f ms -> %.2f GB/s\n", T, im,
                      *std::max_element(issue.begin(), issue.end()), wm, B / wm / 1e6);
    }
  }
}
