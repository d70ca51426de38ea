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
__device__ __forceinline__ void publish(uint64_t* flag, uint64_t v)
{
    __threadfence_system();
    atomicMax_system(reinterpret_cast<unsigned long long*>(flag), (unsigned long long)v);
}

__device__ __forceinline__ void ring_abort(const RelayLaunchArg& A, const RingArg& R)
{
    if (A.err) atomicExch_system(A.err, 1);
    for (uint32_t s = 0; s < R.S; s++) {
        publish(&R.credit[s], kReleaseAll);
        publish(&R.seq[s], kReleaseAll);
    }
}

// Spin (thread 0 only) until pred(*flag) holds; false on timeout or a peer's abort. *seen =
// the last value read (the one that satisfied pred on success).
template <typename Pred>
__device__ __forceinline__ bool spin_until(const RelayLaunchArg& A, const uint64_t* flag, Pred pred, uint64_t* seen)
{
    uint64_t t0 = 0;
    for (uint32_t it = 0;; it++) {
        const uint64_t v = ld_acquire_sys(flag);
        *seen = v;
        if (pred(v)) return true;
        if (v >= kReleaseAll) return false;              // ring aborted elsewhere
        if ((it & 255) == 0) {
            const uint64_t t = globaltimer_ns();
            if (it == 0) t0 = t;
            else if (t - t0 > A.timeout_ns) return false;
            if (A.err && *(volatile int*)A.err) return false;
        }
        __nanosleep(64);
    }
}

template <bool PULL>
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
            if (g == seen) ok = true;
            else if (PULL) ok = spin_until(A, &R.seq[s], [g](uint64_t v) { return v == g + 1; }, &flag);
            else ok = (g < R.S) || spin_until(A, &R.credit[s], [g, &R](uint64_t v) { return v >= g - R.S + 1; }, &flag);
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
        if (PULL) v_copy<V_UNPACK>(A.v, off + lo, off + hi, slot + lo);
        else v_copy<V_PACK>(A.v, off + lo, off + hi, slot + lo);
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
    relay_body<true>(A);
}

__global__ void __launch_bounds__(kThreads) relay_pack_kernel(const __grid_constant__ RelayLaunchArg A)
{
    relay_body<false>(A);
}

cudaError_t launch_relay(const RelayLaunchArg& a, bool pull, unsigned grid, cudaStream_t s)
{
    if (grid == 0) return cudaSuccess;
    if (pull) relay_pull_kernel<<<grid, kThreads, 0, s>>>(a);
    else relay_pack_kernel<<<grid, kThreads, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace mma
