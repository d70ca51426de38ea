// Probe (design input, DESIGN §5 item 12): does a kernel whose CTAs wait on a flag slow the
// copy engine down? One 1 GiB pinned H2D / D2H cudaMemcpyAsync on one stream while a "waiter"
// kernel on another stream holds N CTAs of 512 threads; thread 0 of each CTA waits for a host
// release in one of several ways, the other threads sit at __syncthreads (the relay kernels'
// shape). Reported: DMA GB/s per (wait body, N).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o scripts/probe/probe_spin_ce \
//        scripts/probe/probe_spin_ce.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint64_t gtimer()
{
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// mode 0: nanosleep only (bounded by a timer), 1: ld.relaxed.sys of a device flag + sleep,
// 2: ld.acquire.sys of a device flag + sleep, 3: volatile read of a mapped host flag + sleep,
// 4 (two or more GPUs): ld.relaxed.sys of a flag in GPU 1's memory over NVLink + sleep -- the
// H2D pull kernel's seq polls in the peer form (to be measured on a multi-GPU box)
__global__ void __launch_bounds__(512) waiter(int mode, const uint64_t* dflag, const volatile int* hflag, uint64_t ns_budget)
{
    if (threadIdx.x == 0) {
        const uint64_t t0 = gtimer();
        for (;;) {
            uint64_t v = 0;
            if (mode == 1) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(dflag) : "memory");
            else if (mode == 2) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(dflag) : "memory");
            else if (mode == 3) v = *hflag;
            else if (mode == 4) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(dflag) : "memory");
            if (v) break;
            if (gtimer() - t0 > ns_budget) break;
            __nanosleep(500);
        }
    }
    __syncthreads();
}

int main()
{
    const size_t B = 1ull << 30;
    char *h, *d;
    CK(cudaHostAlloc(&h, B, cudaHostAllocDefault));
    CK(cudaMalloc(&d, B));
    uint64_t* dflag;
    CK(cudaMalloc(&dflag, 64));
    CK(cudaMemset(dflag, 0, 64));
    int* hflag;
    CK(cudaHostAlloc(&hflag, 64, cudaHostAllocMapped));
    *hflag = 0;
    cudaStream_t sc, sk;
    CK(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const char* names[] = {"nanosleep only", "ld.relaxed.sys dev flag", "ld.acquire.sys dev flag", "volatile host flag",
                           "ld.relaxed.sys peer flag"};
    int ngpu = 0;
    CK(cudaGetDeviceCount(&ngpu));
    uint64_t* pflag = nullptr;                      // a flag in GPU 1's memory (peer form)
    if (ngpu > 1) {
        int ok = 0;
        CK(cudaDeviceCanAccessPeer(&ok, 0, 1));
        if (ok) {
            CK(cudaDeviceEnablePeerAccess(1, 0));
            CK(cudaSetDevice(1));
            CK(cudaMalloc(&pflag, 64));
            CK(cudaMemset(pflag, 0, 64));
            CK(cudaDeviceSynchronize());
            CK(cudaSetDevice(0));
        }
    }
    for (int dir = 0; dir < 2; dir++) {
        for (int mode = 0; mode < (pflag ? 5 : 4); mode++) {
            for (int n : {0, 16, 56, 112, 148}) {
                if (n == 0 && mode > 0) continue;
                float best = 1e9;
                for (int rep = 0; rep < 3; rep++) {
                    if (n) waiter<<<n, 512, 0, sk>>>(mode, mode == 4 ? pflag : dflag, hflag, 400000000ull);   // <= 0.4 s
                    CK(cudaEventRecord(a, sc));
                    CK(cudaMemcpyAsync(dir ? h : d, dir ? d : h, B, dir ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice, sc));
                    CK(cudaEventRecord(b, sc));
                    CK(cudaEventSynchronize(b));
                    float ms;
                    CK(cudaEventElapsedTime(&ms, a, b));
                    if (ms < best) best = ms;
                    CK(cudaStreamSynchronize(sk));
                }
                printf("%s waiter=%-26s ctas=%4d  DMA %.2f GB/s\n", dir ? "d2h" : "h2d", names[mode], n, B / best / 1e6);
                fflush(stdout);
            }
        }
    }
    return 0;
}
