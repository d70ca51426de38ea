// copy.cuh — CTA-cooperative byte movement over the virtual stream v, for sm_100a.
//
// HBM/PCIe/NVLink-bound byte copies: no tensor-core work exists on this path (SURVEY
// §8(a): "integer / bitwise semantics"). What matters is coalescing (a warp moves 512
// contiguous bytes per 16-byte-vector instruction), enough bytes in flight per SM to cover
// NVLink (~2 us) and PCIe latency (all loads of an unrolled group issue before any store),
// and L1 bypass (.cg) for data another agent rewrites during the kernel (staging slots).
#pragma once
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
    for (uint64_t k = v_find(v, a); k < v.nseg; k++) {
        const uint64_t vk = v.start[k], vk1 = v.start[k + 1];
        if (vk >= b) break;
        const uint64_t lo = vk > a ? vk : a;
        const uint64_t hi = vk1 < b ? vk1 : b;
        if (lo >= hi) continue;
        const char* s = reinterpret_cast<const char*>(v.src[k]) + (lo - vk);
        char* d = reinterpret_cast<char*>(v.dst[k]) + (lo - vk);
        if (MODE == V_DIRECT) cta_copy(d, s, hi - lo);
        else if (MODE == V_PACK) cta_copy(buf + (lo - a), s, hi - lo);
        else cta_copy(d, buf + (lo - a), hi - lo);
    }
}

__device__ __forceinline__ uint64_t chunk_index(const ChunkListArg& c, uint64_t j)
{
    return c.table ? (uint64_t)c.table[j] : c.first + j;
}

}  // namespace mma
