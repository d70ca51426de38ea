// zerocopy.cu — C2/C3: SM zero-copy movement over one path (north_star (d), SURVEY §8(a)
// rows a7 and a10).
//
// The kernel runs on the path's GPU and moves the chunks that path carries directly
// between mapped pinned host memory and device memory with 16-byte coalesced loads and
// stores; nothing is staged. Launched on
//   - the target GPU d: the direct path (H2D host->d HBM, D2H d HBM->host);
//   - a relay GPU r: a one-hop relay (H2D: loads of host memory cross r's PCIe link,
//     stores to d's HBM cross NVLink; D2H the reverse), which needs no ring and no flags.
// For scattered segments (paged KV blocks) it gathers host blocks and scatters them to
// device blocks in one launch, where the copy engine needs one DMA per block.
#include <cuda_runtime.h>

#include "copy.cuh"

namespace mma {

__global__ void __launch_bounds__(kThreads) zc_copy_kernel(const __grid_constant__ ZcLaunchArg A)
{
    const uint64_t U = A.unit_bytes, C = A.v.C, B = A.v.B;
    const uint64_t upc = (C + U - 1) / U;
    const uint64_t nunits = A.chunks.count * upc;
    for (uint64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
        const uint64_t j = u / upc, k = u % upc;
        const uint64_t i = chunk_index(A.chunks, j);
        const uint64_t off = i * C;
        const uint64_t len = (B - off < C) ? B - off : C;
        const uint64_t lo = k * U;
        if (lo >= len) continue;
        const uint64_t hi = (lo + U < len) ? lo + U : len;
        v_copy<V_DIRECT>(A.v, off + lo, off + hi, nullptr);
        if (!A.log) continue;
        if (!A.piece_chunk) {
            if (k == 0 && threadIdx.x == 0) A.log[i] = (uint8_t)A.path;
        } else if (A.v.nseg == 1) {
            if (threadIdx.x == 0) A.log[A.piece_chunk[0]] = (uint8_t)A.path;
        } else {   // every piece this unit touched: its chunk was carried by this path
            for (uint64_t q = v_find(A.v, off + lo) + threadIdx.x; q < A.v.nseg && A.v.start[q] < off + hi; q += blockDim.x)
                A.log[A.piece_chunk[q]] = (uint8_t)A.path;
        }
    }
}

// Dynamic pull: a CTA claims the next chunk with a system-scope atomic on the target's
// cursor (a peer atomic over NVLink for relays), moves it, and claims again. The claim for
// the next chunk is issued before the current chunk is copied, so the ~2 us NVLink
// round trip of the atomic overlaps the copy.
//
// Contention with background traffic (§3.4.2, background_policy = 1): "if
// prioritizing background traffic is desired, the outstanding queue can wait for a period
// after being blocked before fetching micro-tasks". A unit that took longer than yield_pct %
// of what the path's rate predicts means the link is blocked; the CTA then pushes the whole
// path's pause time to now + that unit's duration, and every CTA of the path waits for it
// before its next claim -- the path's link carries less of the transfer (the other links'
// CTAs keep claiming), and the background flow gets the link meanwhile.
__global__ void __launch_bounds__(kThreads) zc_dyn_kernel(const __grid_constant__ DynLaunchArg A)
{
    __shared__ unsigned long long s_next;
    const uint64_t C = A.v.C, B = A.v.B;
    if (threadIdx.x == 0) s_next = atomicAdd_system(A.cursor, 1ull);
    __syncthreads();
    uint64_t i = s_next;
    unsigned long long taken = 0, waits = 0;
    while (i < A.nchunks) {
        __syncthreads();                                   // everyone has read s_next
        uint64_t t0 = 0;
        if (threadIdx.x == 0) {
            s_next = atomicAdd_system(A.cursor, 1ull);
            if (A.yield_pct) t0 = globaltimer_ns();
        }
        const uint64_t off = i * C;
        const uint64_t len = (B - off < C) ? B - off : C;
        v_copy<V_DIRECT>(A.v, off, off + len, nullptr);
        if (threadIdx.x == 0 && A.log) A.log[i] = (uint8_t)A.path;
        taken++;
        __syncthreads();
        if (threadIdx.x == 0 && A.yield_pct) {
            const uint64_t now = globaltimer_ns(), dt = now - t0;
            if (dt * 100 > A.expect_ns * (uint64_t)A.yield_pct)   // blocked: pause the path
                atomicMax_system(A.pause, now + (dt < 1000000 ? dt : 1000000));
            const uint64_t until = *(volatile unsigned long long*)A.pause;
            if (globaltimer_ns() < until) {
                waits++;
                while (globaltimer_ns() < until) __nanosleep(1000);
            }
        }
        __syncthreads();
        i = s_next;
    }
    if (threadIdx.x == 0 && taken) atomicAdd_system(&A.counts[A.path], taken);
    if (threadIdx.x == 0 && waits && A.backoffs) atomicAdd_system(A.backoffs, waits);
}

cudaError_t launch_zc_dyn(const DynLaunchArg& a, unsigned grid, cudaStream_t s)
{
    if (grid == 0) return cudaSuccess;
    zc_dyn_kernel<<<grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_zc(const ZcLaunchArg& a, unsigned grid, cudaStream_t s)
{
    if (grid == 0) return cudaSuccess;
    zc_copy_kernel<<<grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace mma
