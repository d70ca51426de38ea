// kargs.h — plain-old-data kernel arguments shared by the engine (host C++) and the
// sm_100a kernels. No CUDA types, no method logic.
#pragma once
#include <stdint.h>

#define MMA_KMAX_RINGS 16

namespace mma {

// The transfer as a "virtual stream" v of B bytes (north_star (e)): the concatenation of
// nseg segments. Byte x of segment k lives at src[k] + (x - start[k]) and goes to
// dst[k] + (x - start[k]). A contiguous copy is nseg = 1 with src0/dst0 inline.
struct VStreamArg {
    uint64_t nseg;
    uint64_t B;
    uint64_t C;              // chunk size: chunk i = [i*C, min(B, (i+1)*C))
    uint64_t src0, dst0;     // nseg == 1
    const uint64_t* start;   // nseg > 1: [nseg + 1] offsets in v
    const uint64_t* src;     // nseg > 1: [nseg] addresses
    const uint64_t* dst;     // nseg > 1: [nseg] addresses
};

// The chunks one path carries in one call, in ascending chunk order.
struct ChunkListArg {
    uint64_t count;
    uint64_t first;          // contiguous plan: chunk index of the j-th = first + j
    const uint32_t* table;   // interleaved plan: chunk index of the j-th = table[j]
};

// One relay ring: S staging slots of slot_bytes on the relay GPU,
// seq[S] / credit[S] flags (relay-local), and the consumer-side claim state.
struct RingArg {
    char* stage;
    uint64_t slot_bytes;
    uint64_t* seq;
    uint64_t* credit;
    unsigned* cnt;               // [S] units finished of the slot's current chunk
    unsigned long long* cursor;  // monotone unit-claim cursor
    // [S] on the kernel's GPU: the flag value the leader of the slot's current chunk (the CTA
    // holding its first unit) saw satisfied; the other CTAs of the chunk wait on this LOCAL
    // word instead of polling the flag, which may live in a peer's memory across NVLink
    uint64_t* ready;
    uint64_t g0;                 // global ring index of this call's first chunk
    unsigned long long unit0;    // cursor value when this call's kernel starts
    ChunkListArg chunks;
    uint32_t S;
    uint32_t path;               // path index (delivery log)
    uint32_t cta_begin, cta_end; // CTAs [cta_begin, cta_end) of the grid serve this ring
};

struct RelayLaunchArg {
    VStreamArg v;
    RingArg ring[MMA_KMAX_RINGS];
    uint32_t nrings;
    uint32_t unit_bytes;         // bytes of one claimable unit (a chunk has ceil(C/U))
    uint8_t* log;                // delivery log [n] (device) or nullptr
    // forward log (debug; SURVEY §8(c) "C1 logs the seq value it observed at forward start"):
    // for chunk i of v, [2i] = the flag value this kernel saw satisfied before moving the chunk
    // (pull: seq, must equal g + 1 -- the staging write completed; pack: credit, must be >=
    // g - S + 1 -- the slot drained; 0 when no wait was needed), [2i + 1] = g + 1. nullptr = off.
    uint64_t* fwd;
    int* err;                    // sticky error word (mapped host memory)
    uint64_t timeout_ns;         // bound on every spin
};

// GPU-driven dynamic pull (the paper's pull scheduler, §3.4.2,
// moved onto the GPU): every path's kernel claims whole chunks from one cursor in the
// target's memory until the chunks run out, so faster or less loaded links take more.
struct DynLaunchArg {
    VStreamArg v;
    uint64_t nchunks;
    unsigned long long* cursor;   // per-call claim cursor (target GPU memory, zeroed per call)
    unsigned long long* counts;   // [MMA_KMAX_RINGS] chunks taken per path (same slot)
    uint32_t path;
    uint8_t* log;
    // contention with background traffic: yield_pct > 0 -> a CTA whose unit took more
    // than yield_pct % of expect_ns waits that long again before its next claim
    uint64_t expect_ns;
    uint32_t yield_pct;
    unsigned long long* backoffs;   // waits taken (same claim slot)
    unsigned long long* pause;      // this path's "no claims before" time (%globaltimer ns)
};

struct ZcLaunchArg {
    VStreamArg v;
    ChunkListArg chunks;
    uint32_t unit_bytes;
    uint32_t path;
    uint8_t* log;
    // a private (host-ordered) stream: piece k belongs to chunk piece_chunk[k] of the call's
    // virtual stream; the kernel logs that chunk for every piece it moves. nullptr: v is the
    // call's own stream and chunk i is logged directly.
    const uint32_t* piece_chunk;
};

}  // namespace mma
