// copy.cuh — CTA-cooperative byte movement over the virtual stream v, for sm_100a.
//
// HBM/PCIe/NVLink-bound byte copies: no tensor-core work exists on this path (SURVEY
// §8(a): "integer / bitwise semantics"). What matters is coalescing (a warp moves 512
// contiguous bytes per 16-byte-vector instruction), enough bytes in flight per SM to cover
// NVLink (~2 us) and PCIe latency (all loads of an unrolled group issue before any store),
// and L1 bypass (.cg) for data another agent rewrites during the kernel (staging slots).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../kargs.h"

namespace mma {

constexpr int kThreads = 512;
#ifndef MMA_UNROLL
#define MMA_UNROLL 8      // 64 KiB in flight per CTA per round (+8-10% per CTA over 4, probe_relay)
#endif
constexpr int kUnroll = MMA_UNROLL;

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p)
{
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// a relaxed system-scope poll: no L1 invalidation per read (an acquire load is a load plus
// CCTL.IVALL in SASS); a poll that succeeds is confirmed by one ld_acquire_sys
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p)
{
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v)
{
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer_ns()
{
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// the dynamic shared memory a bulk kernel needs, allowed once per device (the attribute is set
// per function on the current device: a kernel first launched on GPU 0 is not yet allowed it
// on GPU 1); one instantiation (and flag set) per kernel
template <auto* FN>
inline bool allow_dyn_smem(int bytes)
{
    static bool done[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return false;
    if (!done[dev]) done[dev] = cudaFuncSetAttribute(FN, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess;
    return done[dev];
}

// cp.async.bulk (TMA) helpers: a shared-memory tile filled from global memory (completing on
// an mbarrier with the tile's byte count) and its wait
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bulk_load(char* sbuf, const char* src, uint32_t n, uint64_t* bar)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sbuf)),
                 "l"(src), "r"(n), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void bulk_wait(uint64_t* bar, uint32_t parity)
{
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(smem_u32(bar)),
                 "r"(parity)
                 : "memory");
}

// Cooperative copy of len bytes by the whole CTA. 16-byte vectors when src and dst share
// their alignment modulo 16 (always true for the engine's 4 KiB-aligned chunks and
// staging slots when user pointers are 16-byte aligned); otherwise 4-byte or byte moves.
__device__ __forceinline__ void cta_copy(char* __restrict__ dst, const char* __restrict__ src,
                                         uint64_t len)
{
    const int tid = threadIdx.x;
    const uintptr_t d = reinterpret_cast<uintptr_t>(dst);
    const uintptr_t s = reinterpret_cast<uintptr_t>(src);
    if (((d ^ s) & 15) == 0) {
        uint64_t head = (16 - (d & 15)) & 15;
        if (head > len) head = len;
        if (tid < head) dst[tid] = src[tid];
        const uint64_t nvec = (len - head) >> 4;
        uint4* __restrict__ d4 = reinterpret_cast<uint4*>(dst + head);
        const uint4* __restrict__ s4 = reinterpret_cast<const uint4*>(src + head);
        // rounds of kThreads x kUnroll vectors; a partial last round is predicated rather than
        // run one vector at a time, so a 32 KiB paged-KV segment (2048 vectors) is ONE round of
        // loads in flight, not four dependent ones (probe_relay "seg" rows)
        constexpr uint64_t step = (uint64_t)kThreads * kUnroll;
        for (uint64_t base = 0; base < nvec; base += step) {
            const uint64_t i = base + tid;
            uint4 r[kUnroll];
            if (base + step <= nvec) {
#pragma unroll
                for (int u = 0; u < kUnroll; u++) r[u] = __ldcg(s4 + i + u * kThreads);
#pragma unroll
                for (int u = 0; u < kUnroll; u++) __stcg(d4 + i + u * kThreads, r[u]);
            } else {
#pragma unroll
                for (int u = 0; u < kUnroll; u++)
                    if (i + u * kThreads < nvec) r[u] = __ldcg(s4 + i + u * kThreads);
#pragma unroll
                for (int u = 0; u < kUnroll; u++)
                    if (i + u * kThreads < nvec) __stcg(d4 + i + u * kThreads, r[u]);
            }
        }
        const uint64_t done = head + (nvec << 4);
        const uint64_t tail = len - done;
        if (tid < tail) dst[done + tid] = src[done + tid];
    } else if (((d ^ s) & 3) == 0) {
        uint64_t head = (4 - (d & 3)) & 3;
        if (head > len) head = len;
        if (tid < head) dst[tid] = src[tid];
        const uint64_t nw = (len - head) >> 2;
        uint32_t* dw = reinterpret_cast<uint32_t*>(dst + head);
        const uint32_t* sw = reinterpret_cast<const uint32_t*>(src + head);
        for (uint64_t i = tid; i < nw; i += kThreads) __stcg(dw + i, __ldcg(sw + i));
        const uint64_t done = head + (nw << 2);
        if (tid < len - done) dst[done + tid] = src[done + tid];
    } else {
        for (uint64_t i = tid; i < len; i += kThreads) dst[i] = src[i];
    }
}

// first segment k with start[k+1] > x
__device__ __forceinline__ uint64_t v_find(const VStreamArg& v, uint64_t x)
{
    uint64_t lo = 0, hi = v.nseg;
    while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if (v.start[mid + 1] > x) hi = mid; else lo = mid + 1;
    }
    return lo;
}

enum VMode { V_DIRECT = 0, V_PACK = 1, V_UNPACK = 2 };

// Move v[a, b): V_DIRECT src pieces -> dst pieces; V_PACK src pieces -> buf (packed, buf[0]
// = v[a]); V_UNPACK buf -> dst pieces. Byte x of segment k: src_k + (x - v_k) -> dst_k +
// (x - v_k) (north_star (e); oracle/mma_oracle.c vs_copy states the same rule).
template <int MODE>
__device__ __forceinline__ void v_copy(const VStreamArg& v, uint64_t a, uint64_t b, char* buf)
{
    if (a >= b) return;
    if (v.nseg == 1) {
        const char* s = reinterpret_cast<const char*>(v.src0) + a;
        char* d = reinterpret_cast<char*>(v.dst0) + a;
        if (MODE == V_DIRECT) cta_copy(d, s, b - a);
        else if (MODE == V_PACK) cta_copy(buf, s, b - a);
        else cta_copy(d, buf, b - a);
        return;
    }
    // piece k of v clipped to [a, b): its source, destination and length for this MODE
    auto piece = [&](uint64_t k, const char** s, char** d) -> uint64_t {
        const uint64_t vk = v.start[k], vk1 = v.start[k + 1];
        const uint64_t lo = vk > a ? vk : a;
        const uint64_t hi = vk1 < b ? vk1 : b;
        *s = nullptr;
        *d = nullptr;
        if (lo >= hi) return 0;                      // an empty segment
        *s = MODE == V_UNPACK ? buf + (lo - a) : reinterpret_cast<const char*>(v.src[k]) + (lo - vk);
        *d = MODE == V_PACK ? buf + (lo - a) : reinterpret_cast<char*>(v.dst[k]) + (lo - vk);
        return hi - lo;
    };
#ifdef MMA_NO_GROUP
    constexpr bool kGroupPieces = false;   // probe builds: one piece per round (scripts/probe_duplex_grid.py)
#else
    constexpr bool kGroupPieces = true;
#endif
    constexpr uint64_t kRound = (uint64_t)kThreads * kUnroll * 16;   // bytes one round keeps in flight
    uint64_t k = v_find(v, a);
    while (k < v.nseg && v.start[k] < b) {
        // Small pieces (a 32 KiB paged-KV segment fills half a round) are grouped: the group's
        // loads all issue before any store, so a CTA keeps a full round in flight across piece
        // boundaries instead of one piece (under full-duplex load a host read's round trip
        // grows, and bytes in flight per SM bound the rate: scripts/probe_duplex_grid.py).
        // A group is consecutive pieces, each 16-byte aligned at both ends with a length
        // that is a multiple of 16, kMaxGroup at most, a round of bytes at most. Only the
        // zero-copy kernels group (V_DIRECT: their loads cross PCIe); in the relay kernels the
        // group's walk state spills at their 128-register bound, and their loads stay on-GPU.
        constexpr uint64_t kMaxGroup = 16;
        uint64_t k2 = k, tot = 0;
        for (; MODE == V_DIRECT && kGroupPieces && k2 < v.nseg && k2 - k < kMaxGroup && v.start[k2] < b; k2++) {
            const char* s;
            char* d;
            const uint64_t n = piece(k2, &s, &d);
            if (tot + n > kRound || ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d) | n) & 15)) break;
            tot += n;
        }
        if (k2 - k >= 2) {
            const uint64_t nv = tot >> 4;
            uint4 r[kUnroll];
            // each phase walks the group's pieces once (i grows with u); the store phase walks
            // again rather than keeping kUnroll destination pointers live across the loads
            for (int phase = 0; phase < 2; phase++) {
                uint64_t p = k, pbase = 0;      // piece p holds group vectors [pbase, pbase + pn)
                const char* ps;
                char* pd;
                uint64_t pn = piece(p, &ps, &pd) >> 4;
#pragma unroll
                for (int u = 0; u < kUnroll; u++) {
                    const uint64_t i = (uint64_t)u * kThreads + threadIdx.x;
                    if (i < nv) {
                        while (i >= pbase + pn) {
                            pbase += pn;
                            pn = piece(++p, &ps, &pd) >> 4;
                        }
                        if (phase == 0) r[u] = __ldcg(reinterpret_cast<const uint4*>(ps) + (i - pbase));
                        else __stcg(reinterpret_cast<uint4*>(pd) + (i - pbase), r[u]);
                    }
                }
            }
            k = k2;
            continue;
        }
        const char* s;
        char* d;
        const uint64_t n = piece(k, &s, &d);
        if (n) cta_copy(d, s, n);
        k++;
    }
}

__device__ __forceinline__ uint64_t chunk_index(const ChunkListArg& c, uint64_t j)
{
    return c.table ? (uint64_t)c.table[j] : c.first + j;
}

}  // namespace mma
