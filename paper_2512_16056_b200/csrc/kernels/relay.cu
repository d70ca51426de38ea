// relay.cu — C1/C3: the relay kernels of MMA's dual-pipeline relay, generalised to an
// S-slot staging ring per (relay, target, direction) (§3.4.3, Fig 6; SURVEY
// §8(a) rows a6, a9, a10).
//
// H2D, on the TARGET GPU d (relay_pull_kernel): for each chunk g of ring r, in order,
//   poll seq_r[s] (relay-local, ld.acquire.sys over NVLink) until it equals g + 1, then
//   pull the slot stage_r[s] (peer HBM) with 16-byte coalesced loads and store it to the
//   destination pieces of v, then publishes credit_r[s] = g + 1 (system fence + atomicMax).
// D2H, on the RELAY GPU r (relay_pack_kernel): for each chunk g, wait credit_r[s] >=
//   g - S + 1 (the relay's copy engine drained the slot), pull the chunk's source pieces
//   from d's HBM over NVLink into stage_r[s], then publishes seq_r[s] = g + 1.
//
// "a dependency established between these operations to guarantee the correctness and
// ordering of data transfer" is the seq flag; the credit flag is the buffer
// ownership of "each relay stream has a dedicated relay buffer".
//
// Work is claimed in ring order through a monotone per-ring cursor: a chunk is split into
// units of unit_bytes; any CTA serving the ring claims the next unit. No chunk is owned
// statically by a CTA, so progress needs only one resident CTA per ring (SURVEY §7 hard
// part 4). The last CTA to finish a chunk's units releases the flag. Every spin is bounded
// by a globaltimer timeout: on expiry the kernel records a sticky error in mapped host
// memory and releases every slot so the copy-engine side of the ring cannot hang.
#include <cuda_runtime.h>

#include "copy.cuh"

namespace mma {

constexpr uint64_t kReleaseAll = 1ull << 62;

// Flags the kernel publishes only ever grow (atomicMax after a system fence = a release
// that cannot move a flag backwards), so once a ring is aborted every copy-engine wait on
// it passes even if a CTA still finishing a chunk publishes afterwards.
#ifndef MMA_PUBLISH_SC
#define MMA_PUBLISH_SC 0
#endif
__device__ __forceinline__ void publish(uint64_t* flag, uint64_t v)
{
    // a release at system scope (the flag's readers include the copy engines' stream memory
    // operations and other GPUs): fence.acq_rel.sys + the relaxed atomic is the PTX release
    // pattern; MMA_PUBLISH_SC=1 builds the stronger fence.sc.sys (__threadfence_system)
#if MMA_PUBLISH_SC
    __threadfence_system();
#else
    asm volatile("fence.acq_rel.sys;" ::: "memory");
#endif
    atomicMax_system(reinterpret_cast<unsigned long long*>(flag), (unsigned long long)v);
}

__device__ __forceinline__ void ring_abort(const RelayLaunchArg& A, const RingArg& R)
{
    if (A.err) atomicExch_system(A.err, 1);
    for (uint32_t s = 0; s < R.S; s++) {
        publish(&R.credit[s], kReleaseAll);
        publish(&R.seq[s], kReleaseAll);
        if (R.ready) publish(&R.ready[s], kReleaseAll);   // releases the chunk's followers
    }
}

// Spin (thread 0 only) until pred(*flag) holds; false on timeout or a peer's abort. *seen =
// the last value read (the one that satisfied pred on success). Polls are relaxed loads of
// the (device-memory) flag with an exponential backoff (kSpinMinNs .. kSpinMaxNs); one
// acquire load is taken on success. The abort word lives in mapped HOST memory, and
// reading host memory from waiting CTAs throttles the copy engines of the same GPU: 16 CTAs
// reading a host word every ~0.5 us cut a concurrent 1 GiB H2D DMA from 55.6 to 30 GB/s, 56
// CTAs to 8.9 (D2H: 13 and 2.8), while device-memory polls of any kind cost nothing
// (scripts/probe/probe_spin_ce.cu, profiles/r02_probe_spin_ce.txt). Relay kernels wait
// next to their own rings' DMAs, so the abort word is read only every kErrCheckNs (10 ms):
// a peer's abort still ends the wait within 10 ms.
#ifndef MMA_SPIN_MIN_NS
#define MMA_SPIN_MIN_NS 32
#endif
#ifndef MMA_SPIN_MAX_NS
#define MMA_SPIN_MAX_NS 512
#endif
#ifndef MMA_ERR_CHECK_NS
#define MMA_ERR_CHECK_NS 10000000
#endif
constexpr unsigned kSpinMinNs = MMA_SPIN_MIN_NS, kSpinMaxNs = MMA_SPIN_MAX_NS;
constexpr uint64_t kErrCheckNs = MMA_ERR_CHECK_NS;

template <typename Pred>
__device__ __forceinline__ bool spin_until(const RelayLaunchArg& A, const uint64_t* flag, Pred pred, uint64_t* seen)
{
    const uint64_t t0 = globaltimer_ns();
    uint64_t next_err = t0 + kErrCheckNs;
    unsigned ns = kSpinMinNs;
    for (;;) {
#ifdef MMA_SPIN_ACQUIRE
        const uint64_t v = ld_acquire_sys(flag);
#else
        const uint64_t v = ld_relaxed_sys(flag);
#endif
        *seen = v;
#ifdef MMA_SPIN_ACQUIRE
        if (pred(v)) return true;
#else
        // the flag satisfied the wait: one acquire load of it (flags never move past a value
        // a waiter still needs, so it satisfies pred again) orders the slot reads after it --
        // cheaper than a fence.acq_rel.sys (a MEMBAR.SYS) and the same acquire
        if (pred(v) && pred(*seen = ld_acquire_sys(flag))) return true;
#endif
        if (v >= kReleaseAll) return false;              // ring aborted elsewhere
        const uint64_t t = globaltimer_ns();
        if (t - t0 > A.timeout_ns) return false;
        if (t >= next_err) {
            if (A.err && *(volatile int*)A.err) return false;
            next_err = t + kErrCheckNs;
        }
        __nanosleep(ns);
        if (ns < kSpinMaxNs) ns <<= 1;
    }
}

// ---- the bulk-copy (TMA) form of a unit's copy: one thread streams the unit through
// shared memory with cp.async.bulk -- global -> shared completing on an mbarrier, then
// shared -> global in a bulk group -- kBulkStages tiles of kBulkTile in flight. The vector
// form keeps 64 KiB per CTA in flight in registers; this one 128 KiB in shared memory with a
// single issuing thread ("or stage through shared memory / cp.async.bulk").
// Used for contiguous transfers whose unit is 16-byte aligned (MMA_RELAY_BULK=1).
constexpr uint32_t kBulkTile = 32u << 10;
constexpr int kBulkStages = 4;

// thread 0 only: dst[0, len) = src[0, len); len % 16 == 0, both 16-byte aligned. *phase holds
// one parity bit per stage (the barriers live as long as the CTA).
__device__ __forceinline__ void bulk_copy(char* dst, const char* src, uint64_t len, char* smem, uint64_t* bar,
                                          uint32_t* phase)
{
    const uint64_t ntiles = (len + kBulkTile - 1) / kBulkTile;
    auto tile_bytes = [&](uint64_t t) { return (uint32_t)((len - t * kBulkTile) < kBulkTile ? len - t * kBulkTile : kBulkTile); };
    asm volatile("fence.proxy.async;" ::: "memory");   // the flag's acquire before the async-proxy reads
    for (uint64_t t = 0; t < ntiles && t < (uint64_t)kBulkStages; t++)
        bulk_load(smem + t * kBulkTile, src + t * kBulkTile, tile_bytes(t), &bar[t]);
    for (uint64_t t = 0; t < ntiles; t++) {
        const int s = (int)(t % kBulkStages);
        bulk_wait(&bar[s], (*phase >> s) & 1);
        *phase ^= 1u << s;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + t * kBulkTile),
                     "r"(smem_u32(smem + s * kBulkTile)), "r"(tile_bytes(t))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        // the previous tile's stage is free once its store has read it: refill it
        if (t >= 1 && t - 1 + kBulkStages < ntiles) {
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            const int sp = (int)((t - 1) % kBulkStages);
            bulk_load(smem + sp * kBulkTile, src + (t - 1 + kBulkStages) * kBulkTile, tile_bytes(t - 1 + kBulkStages), &bar[sp]);
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // every store performed
    asm volatile("fence.proxy.async;" ::: "memory");             // ... before the generic-proxy release
}

template <bool PULL, bool BULK>
__device__ __forceinline__ void relay_body(const RelayLaunchArg& A)
{
    uint32_t r = 0;
    while (r < A.nrings && blockIdx.x >= A.ring[r].cta_end) r++;
    if (r >= A.nrings || blockIdx.x < A.ring[r].cta_begin) return;
    const RingArg& R = A.ring[r];
    const uint64_t U = A.unit_bytes, C = A.v.C, B = A.v.B;
    const uint64_t upc = (C + U - 1) / U;
    const uint64_t nunits = R.chunks.count * upc;
    __shared__ unsigned long long s_u;
    __shared__ int s_ok;
    extern __shared__ __align__(128) char s_bulk[];   // BULK: kBulkStages x kBulkTile
    __shared__ __align__(8) uint64_t s_bar[kBulkStages];
    uint32_t bulk_phase = 0;
    if (BULK) {
        if (threadIdx.x == 0) {
            for (int k = 0; k < kBulkStages; k++)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&s_bar[k])));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    // thread 0: the last chunk whose flag this CTA saw satisfied. Its flag cannot move on
    // while this CTA still holds one of its units (the slot is released only when every unit
    // of the chunk is done), so a later unit of the same chunk skips the poll.
    uint64_t seen = ~0ull;
    for (;;) {
        if (threadIdx.x == 0) s_u = atomicAdd(R.cursor, 1ull) - R.unit0;
        __syncthreads();
        const uint64_t u = s_u;
        __syncthreads();
        if (u >= nunits) break;
        const uint64_t j = u / upc, k = u % upc;
        const uint64_t i = chunk_index(R.chunks, j);
        const uint64_t off = i * C;
        const uint64_t len = (B - off < C) ? B - off : C;
        const uint64_t lo = k * U;
        if (lo >= len) continue;                           // empty unit of a short chunk
        const uint64_t hi = (lo + U < len) ? lo + U : len;
        const uint64_t g = R.g0 + j;
        const uint32_t s = (uint32_t)(g % R.S);
        char* slot = R.stage + (uint64_t)s * R.slot_bytes;
        if (threadIdx.x == 0) {
            bool ok;
            uint64_t flag = 0;
            // the chunk's leader (the CTA holding its first unit) polls the ring flag, which may
            // live in a peer's memory, and passes the value it saw to the local ready word; the
            // chunk's other CTAs wait on that word. Both waits have acquire semantics, and the
            // leader's fence + atomicMax is a release at GPU scope, so a follower's slot reads
            // are ordered after the staging write the leader observed. ready[s] is monotone
            // like the flags: it can pass this chunk's value only after every unit of the chunk
            // is done (the slot must drain before chunk g + S is staged).
            const bool leader = (k == 0) || !R.ready;
            const uint64_t* wflag = leader ? (PULL ? &R.seq[s] : &R.credit[s]) : R.ready + s;
            if (g == seen) ok = true;
            else if (PULL) ok = spin_until(A, wflag, [g](uint64_t v) { return v == g + 1; }, &flag);
            else ok = (g < R.S) || spin_until(A, wflag, [g, &R](uint64_t v) { return v >= g - R.S + 1; }, &flag);
            if (ok && g != seen && leader && R.ready && (PULL || g >= R.S)) {
                __threadfence();
                atomicMax(reinterpret_cast<unsigned long long*>(R.ready + s), (unsigned long long)flag);
            }
            if (g != seen && A.fwd) {   // the observation the forward (pack) of chunk i rests on
                A.fwd[2 * i] = flag;
                A.fwd[2 * i + 1] = g + 1;
            }
            if (!ok) ring_abort(A, R);
            else seen = g;
            s_ok = ok;
        }
        __syncthreads();
        if (!s_ok) return;
        // the bulk form for a contiguous, 16-byte-aligned unit; the vector form otherwise
        const char* bsrc = PULL ? slot + lo : reinterpret_cast<const char*>(A.v.src0) + off + lo;
        char* bdst = PULL ? reinterpret_cast<char*>(A.v.dst0) + off + lo : slot + lo;
        if (BULK && A.v.nseg == 1 && !(((uintptr_t)bsrc | (uintptr_t)bdst | (hi - lo)) & 15)) {
            if (threadIdx.x == 0) bulk_copy(bdst, bsrc, hi - lo, s_bulk, s_bar, &bulk_phase);
        } else if (PULL) {
            v_copy<V_UNPACK>(A.v, off + lo, off + hi, slot + lo);
        } else {
            v_copy<V_PACK>(A.v, off + lo, off + hi, slot + lo);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const unsigned units_j = (unsigned)((len + U - 1) / U);
            const unsigned old = atomicAdd(&R.cnt[s], 1u);
            if (old == units_j - 1) {                      // last unit of chunk g
                atomicExch(&R.cnt[s], 0u);
                if (A.log) A.log[i] = (uint8_t)R.path;
                if (PULL) publish(&R.credit[s], g + 1);   // slot free for g + S
                else publish(&R.seq[s], g + 1);           // chunk g staged
            }
        }
    }
}

__global__ void __launch_bounds__(kThreads) relay_pull_kernel(const __grid_constant__ RelayLaunchArg A)
{
    relay_body<true, false>(A);
}

__global__ void __launch_bounds__(kThreads) relay_pack_kernel(const __grid_constant__ RelayLaunchArg A)
{
    relay_body<false, false>(A);
}

__global__ void __launch_bounds__(kThreads) relay_pull_bulk_kernel(const __grid_constant__ RelayLaunchArg A)
{
    relay_body<true, true>(A);
}

__global__ void __launch_bounds__(kThreads) relay_pack_bulk_kernel(const __grid_constant__ RelayLaunchArg A)
{
    relay_body<false, true>(A);
}

cudaError_t launch_relay(const RelayLaunchArg& a, bool pull, unsigned grid, cudaStream_t s, bool bulk)
{
    if (grid == 0) return cudaSuccess;
    if (bulk) {
        constexpr int smem = kBulkStages * kBulkTile;
        if (!(pull ? allow_dyn_smem<relay_pull_bulk_kernel>(smem) : allow_dyn_smem<relay_pack_bulk_kernel>(smem)))
            return cudaErrorInvalidValue;
        if (pull) relay_pull_bulk_kernel<<<grid, kThreads, smem, s>>>(a);
        else relay_pack_bulk_kernel<<<grid, kThreads, smem, s>>>(a);
        return cudaGetLastError();
    }
    if (pull) relay_pull_kernel<<<grid, kThreads, 0, s>>>(a);
    else relay_pack_kernel<<<grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace mma
