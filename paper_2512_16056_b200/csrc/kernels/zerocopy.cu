// zerocopy.cu — C2/C3: SM zero-copy movement over one path (north_star (d), SURVEY §8(a)
// rows a7 and a10).
//
// The kernel runs on the path's GPU and moves the chunks that path carries directly
// between mapped pinned host memory and device memory -- zc_bulk_kernel (direct paths, the
// default) through shared-memory tiles with cp.async.bulk, zc_copy_kernel with 16-byte
// coalesced register loads and stores; no staging buffer in HBM. Launched on
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

// ---- the bulk-copy (TMA) form of the zero-copy kernel (direct paths; MMA_ZC_BULK=0: off): one warp per CTA,
// lane 0 streams the CTA's units through kZcStages shared-memory tiles with cp.async.bulk
// (global -> shared completing on an mbarrier, shared -> global in bulk groups), so a CTA
// keeps up to kZcStages x 32 KiB of host reads (H2D) in flight with one issuing thread and a
// few registers, where the vector kernel holds one 64 KiB round in the registers of an
// SM's whole register file. Tiles that are not 16-byte aligned at both ends or not a multiple
// of 16 bytes long keep their 16-byte-aligned middle on the bulk engine when source and
// destination agree mod 16 (the warp copies the < 16-byte head and tail), else the warp copies
// them. Every lane runs the same tile generator over the same table (broadcast loads), so
// control flow is warp-uniform.
constexpr uint32_t kZcTile = 32u << 10;
#ifndef MMA_ZC_STAGES
#define MMA_ZC_STAGES 4
#endif
constexpr int kZcStages = MMA_ZC_STAGES;   // shared memory per CTA = kZcStages x kZcTile (4: 128 KiB; 3 loses 4% duplex, 6 gains nothing)
constexpr int kZcBulkThreads = 32;

struct ZcTileGen {
    const ZcLaunchArg& A;
    uint64_t upc, nunits, u, x, b, k;
    bool in_unit = false;
    __device__ ZcTileGen(const ZcLaunchArg& a) : A(a)
    {
        upc = (A.v.C + A.unit_bytes - 1) / A.unit_bytes;
        nunits = A.chunks.count * upc;
        u = blockIdx.x;
    }
    // the next unit's v range [x, b); logs the unit's chunk / pieces (lane 0 / the warp)
    __device__ bool enter_unit()
    {
        const uint64_t U = A.unit_bytes, C = A.v.C, B = A.v.B;
        for (; u < nunits; u += gridDim.x) {
            const uint64_t j = u / upc, kk = u % upc;
            const uint64_t i = chunk_index(A.chunks, j);
            const uint64_t off = i * C;
            const uint64_t len = (B - off < C) ? B - off : C;
            const uint64_t lo = kk * U;
            if (lo >= len) continue;
            const uint64_t hi = (lo + U < len) ? lo + U : len;
            x = off + lo;
            b = off + hi;
            k = A.v.nseg == 1 ? 0 : v_find(A.v, x);
            if (A.log) {
                if (!A.piece_chunk) {
                    if (kk == 0 && threadIdx.x == 0) A.log[i] = (uint8_t)A.path;
                } else if (A.v.nseg == 1) {
                    if (threadIdx.x == 0) A.log[A.piece_chunk[0]] = (uint8_t)A.path;
                } else {
                    for (uint64_t q = k + threadIdx.x; q < A.v.nseg && A.v.start[q] < b; q += blockDim.x)
                        A.log[A.piece_chunk[q]] = (uint8_t)A.path;
                }
            }
            u += gridDim.x;
            return true;
        }
        return false;
    }
    // next tile: src, dst, length (<= kZcTile); false when the CTA's units are done
    __device__ bool next(const char** src, char** dst, uint32_t* n)
    {
        for (;;) {
            if (!in_unit) {
                if (!enter_unit()) return false;
                in_unit = true;
            }
            if (x >= b) {
                in_unit = false;
                continue;
            }
            uint64_t vk = 0, end = b;
            const char* s0;
            char* d0;
            if (A.v.nseg == 1) {
                s0 = reinterpret_cast<const char*>(A.v.src0);
                d0 = reinterpret_cast<char*>(A.v.dst0);
            } else {
                while (A.v.start[k + 1] <= x) k++;       // skip empty / finished pieces
                vk = A.v.start[k];
                if (A.v.start[k + 1] < end) end = A.v.start[k + 1];
                s0 = reinterpret_cast<const char*>(A.v.src[k]);
                d0 = reinterpret_cast<char*>(A.v.dst[k]);
            }
            const uint64_t m = (end - x < kZcTile) ? end - x : kZcTile;
            *src = s0 + (x - vk);
            *dst = d0 + (x - vk);
            *n = (uint32_t)m;
            x += m;
            return true;
        }
    }
};

__global__ void __launch_bounds__(kZcBulkThreads) zc_bulk_kernel(const __grid_constant__ ZcLaunchArg A)
{
    extern __shared__ __align__(128) char s_tile[];
    __shared__ __align__(8) uint64_t s_bar[kZcStages];
    const bool lead = threadIdx.x == 0;
    if (lead) {
        for (int q = 0; q < kZcStages; q++)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[q])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    ZcTileGen gen(A);
    char* dst_of[kZcStages];          // lane 0: the destination and length of each stage's tile
    uint32_t n_of[kZcStages];
    uint32_t phase = 0;
    uint64_t loaded = 0, stored = 0;   // bulk tiles whose load / store was issued
    bool more = true;
    // a tile for the next free stage: bulk tiles load into it, the others are copied now
    auto fill = [&]() {
        while (more) {
            const char* s;
            char* d;
            uint32_t n;
            if (!(more = gen.next(&s, &d, &n))) return;
            const uintptr_t sa = reinterpret_cast<uintptr_t>(s), da = reinterpret_cast<uintptr_t>(d);
            if (((sa ^ da) & 15) == 0) {
                // same alignment mod 16: head and tail bytes (< 16 each) by the warp, the
                // 16-byte-aligned middle by the bulk engine
                const uint32_t head = min(n, (uint32_t)((16 - (sa & 15)) & 15));
                const uint32_t mid = (n - head) & ~15u;
                const uint32_t tail = n - head - mid;
                if (threadIdx.x < head) d[threadIdx.x] = s[threadIdx.x];
                if (threadIdx.x < tail) d[head + mid + threadIdx.x] = s[head + mid + threadIdx.x];
                if (!mid) continue;
                if (lead) {
                    const int q = (int)(loaded % kZcStages);
                    dst_of[q] = d + head;
                    n_of[q] = mid;
                    bulk_load(s_tile + (uint64_t)q * kZcTile, s + head, mid, &s_bar[q]);
                }
                loaded++;
                return;
            }
            // source and destination aligned differently mod 16: the warp copies the tile, with
            // 4-byte words when they agree mod 4, kUnroll loads per lane in flight
            if (((sa ^ da) & 3) == 0) {
                const uint32_t head = min(n, (uint32_t)((4 - (sa & 3)) & 3));
                if (threadIdx.x < head) d[threadIdx.x] = s[threadIdx.x];
                const uint32_t nw = (n - head) >> 2;
                const uint32_t* sw = reinterpret_cast<const uint32_t*>(s + head);
                uint32_t* dw = reinterpret_cast<uint32_t*>(d + head);
                for (uint32_t base = 0; base < nw; base += kZcBulkThreads * kUnroll) {
                    uint32_t r[kUnroll];
#pragma unroll
                    for (int j = 0; j < kUnroll; j++) {
                        const uint32_t i = base + j * kZcBulkThreads + threadIdx.x;
                        if (i < nw) r[j] = __ldcg(sw + i);
                    }
#pragma unroll
                    for (int j = 0; j < kUnroll; j++) {
                        const uint32_t i = base + j * kZcBulkThreads + threadIdx.x;
                        if (i < nw) __stcg(dw + i, r[j]);
                    }
                }
                const uint32_t done = head + (nw << 2);
                if (threadIdx.x < n - done) d[done + threadIdx.x] = s[done + threadIdx.x];
            } else {
                for (uint32_t base = 0; base < n; base += kZcBulkThreads * kUnroll) {
                    char r[kUnroll];
#pragma unroll
                    for (int j = 0; j < kUnroll; j++) {
                        const uint32_t i = base + j * kZcBulkThreads + threadIdx.x;
                        if (i < n) r[j] = s[i];
                    }
#pragma unroll
                    for (int j = 0; j < kUnroll; j++) {
                        const uint32_t i = base + j * kZcBulkThreads + threadIdx.x;
                        if (i < n) d[i] = r[j];
                    }
                }
            }
        }
    };
    for (int q = 0; q < kZcStages; q++) fill();
    while (stored < loaded) {
        if (lead) {
            const int q = (int)(stored % kZcStages);
            bulk_wait(&s_bar[q], (phase >> q) & 1);
            phase ^= 1u << q;
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_of[q]),
                         "r"(smem_u32(s_tile + (uint64_t)q * kZcTile)), "r"(n_of[q])
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        stored++;
        // the previous tile's stage is free once its store has read it: refill it (after the
        // first store no stage is free yet: the other K - 1 hold loads, this one the store)
        if (more && stored >= 2) {
            if (lead) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            fill();
        }
    }
    if (lead) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

cudaError_t launch_zc(const ZcLaunchArg& a, unsigned grid, cudaStream_t s, bool bulk)
{
    if (grid == 0) return cudaSuccess;
    if (bulk) {
        constexpr int smem = kZcStages * kZcTile;
        if (!allow_dyn_smem<zc_bulk_kernel>(smem)) return cudaErrorInvalidValue;
        zc_bulk_kernel<<<grid, kZcBulkThreads, smem, s>>>(a);
        return cudaGetLastError();
    }
    zc_copy_kernel<<<grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace mma
