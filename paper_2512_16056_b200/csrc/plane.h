// plane.h — internal state and interfaces of the data plane (engine) shared by
// plane.cpp (configuration, devices, rings, ledger, enqueue), api.cpp (the C ABI) and
// tune.cpp (per-path measurement). Not part of the public ABI (include/mma.h is).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/mma.h"
#include "engine.h"
#include "kargs.h"
#include "planner.h"

namespace mma {

#define CK(x)                                   \
    do {                                        \
        int e_ = (int)(x);                      \
        if (e_ != 0) return e_;                 \
    } while (0)


using PFN_memop64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
using PFN_batch_memop = CUresult (*)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int);

// 8 MiB: a copy-engine DMA costs ~4 us of setup on B200, so 1 MiB chunks reach 46 GB/s,
// 4 MiB 52.6, 16 MiB 54.8 of the link's 55.6 (scripts/probe/probe_chunks.cu)
constexpr uint64_t kDefaultChunk = 8ull << 20;
constexpr uint64_t kRingBytes = 32ull << 20;   // staging per ring when cfg.ring_slots = 0
constexpr uint32_t kDefaultMbps = 50000;
// Claim unit of the relay and zero-copy kernels: a CTA claims, checks the flag, copies and
// releases per unit, so small units pay that bookkeeping often. Relay kernel alone, 8 CTAs,
// local HBM: 23 GB/s per CTA at 128 KiB, 38 at 512 KiB, 41 at 1 MiB
// (profiles/r01_probe_relay_unroll.txt)
constexpr uint32_t kDefaultUnit = 512u << 10;
constexpr int kDefaultRelayCtas = 8;
constexpr uint64_t kDefaultGroupBytes = 8ull << 20;   // MMA_GROUP_BYTES (profiles/r02_sweep_group_lanes.jsonl)
constexpr int kDefaultZcCtas = 16;     // zero-copy kernel grid (mma_config_t::zc_ctas): the link saturates from 4-8
constexpr unsigned kDynSlots = 64;        // per-call claim slots, rotating
constexpr unsigned kDynSlotWords = 64;    // cursor, counts[MMA_KMAX_RINGS], backoffs, pause[MMA_KMAX_RINGS]
constexpr unsigned kDynBackoffWord = 1 + MMA_KMAX_RINGS;
constexpr unsigned kDynPauseWord = 2 + MMA_KMAX_RINGS;

// The CUDA device behind engine GPU index g: the identity, except under the MMA_VGPUS=k test
// hook, where indices >= the physical device count are virtual GPUs g % count (plane.cpp).
int phys_dev(int g);

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d)
    {
        cudaGetDevice(&prev);
        const int p = phys_dev(d);
        if (p != prev) cudaSetDevice(p);
    }
    ~DeviceGuard()
    {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// One set of engine streams per direction, so an H2D call and a D2H call (PCIe is full
// duplex) never queue behind each other on a shared stream.
struct Lanes {
    cudaStream_t direct = nullptr;   // direct-path DMA
    cudaStream_t zc = nullptr;       // zero-copy kernels (direct or one-hop relay)
    cudaStream_t hop[2] = {};        // relay hop DMAs: dual pipeline, slot parity
    cudaStream_t kern = nullptr;     // relay kernels (pull on a target, pack on a relay)
};

struct DevRes {
    bool made = false;
    Lanes lane[2];                   // [MMA_H2D], [MMA_D2H]
    // streams of captured calls only: a call on a capturing stream pulls every engine stream
    // it uses into that capture until the user ends it, so captured calls never touch the
    // live lanes (a live call on another stream may run in that window), and a second
    // capture while these are still capturing is recorded as the native copy (api.cpp)
    Lanes cap_lane[2];
    cudaEvent_t cap_fork = nullptr;  // fork event of captured calls (live calls take one from fork_pool)
    std::vector<cudaEvent_t> fork_pool;   // fork events of live calls (one per call in flight of enqueue)
    // [dir][0 direct lane, 1 zero-copy lane]: recorded behind this GPU's own direct work when
    // a relay through this GPU must wait for it (direct path first, plane.cpp Call::gate)
    cudaEvent_t gate_ev[2][2] = {};
    cudaStream_t setup = nullptr;    // ring initialisation (never waits on user work)
    cudaEvent_t cap_ev = nullptr;    // captured calls: orders the table frees after the join
    int sms = 148;
};

struct Ring {
    bool made = false;
    int relay = -1, kdev = -1;       // GPU holding stage and flags; GPU running the kernel
    uint32_t S = 0;
    uint64_t slot_bytes = 0;
    char* stage = nullptr;
    uint64_t* seq = nullptr;         // relay-local
    uint64_t* credit = nullptr;      // relay-local
    unsigned* cnt = nullptr;         // on kdev
    unsigned long long* cursor = nullptr;   // on kdev
    uint64_t* ready = nullptr;              // on kdev: [64] leader-observed flag per slot
    uint64_t g_next = 0;             // chunks carried so far (reading R18)
    unsigned long long unit_next = 0;
    // a call failed part-way through this ring's enqueue: its flags and counters may be out
    // of step with g_next / unit_next. get_ring drains both devices (every wait already
    // enqueued is satisfiable, DESIGN §5 item 8) and makes the ring afresh.
    bool broken = false;
};

struct PathState {
    int gpu;
    int kind;       // MMA_PATH_DIRECT / MMA_PATH_RELAY
    uint32_t mbps;
    int mode;       // mma_hop_t
    uint32_t seg_mbps = 0;   // measured for scattered transfers (mma_tune_segments); 0 = unset
    int seg_mode = -1;       // idem; -1 = unset
    // calibration evidence (mma_get_calibration): [0] contiguous, [1] scattered
    uint32_t solo_mbps[2] = {0, 0};   // solo rate of the chosen mode
    uint32_t conc_mbps[2] = {0, 0};   // rate with every path of the set active (0 = not measured)
    int node = -1;                    // NUMA node of the path's GPU (R23; -1 = unknown)
};

struct Scratch {    // per-call table uploads, double-buffered by call parity
    void* host = nullptr;
    size_t host_cap = 0;
    void* dev[MMA_MAX_GPUS] = {};
    size_t dev_cap[MMA_MAX_GPUS] = {};
    cudaEvent_t done = nullptr;       // recorded on the user stream at the call's join
    int done_dev = -1;
    bool pending = false;
};

struct Target {
    bool paths_made = false;
    std::vector<PathState> paths[2];
    Ring rings[2][MMA_MAX_PATHS];
    mma_stats_t stats{};
    uint8_t* log = nullptr;
    size_t log_cap = 0, log_n = 0;
    uint64_t* fwd = nullptr;         // forward log (debug_log): 2 words per chunk (kargs.h)
    size_t fwd_cap = 0, fwd_n = 0;
    // debug_log: the table order of the last scattered call's virtual stream (R23 regrouping;
    // identity when not regrouped): last_order[k] = table index of v's k-th segment
    std::vector<uint32_t> last_order;
    Scratch scratch[4];   // table buffers of the last 4 calls (a ring)
    unsigned parity = 0;
    unsigned long long* dyn = nullptr;        // dynamic-pull slots: cursor + per-path counts
    unsigned dyn_next = 0;
    unsigned long long* last_dyn = nullptr;
    int last_dyn_paths = 0;
};

struct Engine {
    std::mutex mu;                   // one multipath enqueue at a time
    std::atomic<bool> inited{false};   // read without the mutex by ensure_init's fast path
    mma_config_t cfg{};
    int ndev = 0;
    // MMA_VGPUS=k (test hook, read at init): the engine sees k GPUs although the box has fewer;
    // GPU index g >= the physical count is a virtual GPU on CUDA device phys[g] = g % count,
    // with its own streams, rings, flags, ledger entries and path index. Relays through a
    // virtual GPU therefore run every code path of a peer relay (relay index != target: the
    // pack kernel on the relay, cross-index fork/join, gates, peer rings) except the NVLink
    // transport itself, which a one-GPU box cannot provide.
    int phys[MMA_MAX_GPUS];
    bool virt = false;
    Engine()
    {
        for (int g = 0; g < MMA_MAX_GPUS; g++) phys[g] = g;
    }
    bool p2p[MMA_MAX_GPUS][MMA_MAX_GPUS] = {};
    bool p2p_atomic[MMA_MAX_GPUS][MMA_MAX_GPUS] = {};   // [a][b]: a kernel on a may atomically update b's memory
    DevRes dev[MMA_MAX_GPUS];
    Target tgt[MMA_MAX_GPUS];
    std::map<cudaStream_t, cudaEvent_t> join_ev;   // join event per engine stream
    // backlog ledger (NEXT-1): bytes in flight per (direction, link GPU), and of those the
    // link's own target's direct bytes; each call's share is retired when its done event
    // (recorded on the user stream at the join) has completed
    struct InFlight {
        cudaEvent_t done;
        int dev, dir;
        uint64_t bytes[MMA_MAX_GPUS];
        uint64_t own[MMA_MAX_GPUS];
        uint64_t shared;             // attach generation of the cross-process ledger it entered (0 = none)
    };
    std::vector<InFlight> inflight;
    std::vector<std::pair<int, cudaEvent_t>> free_events;
    uint64_t ledger[2][MMA_MAX_GPUS] = {};
    uint64_t ledger_own[2][MMA_MAX_GPUS] = {};
    int* err = nullptr;              // mapped pinned host word (sticky async error)
    // tables of captured calls (graph replays read them): an append-only pinned arena made at
    // init, since nothing may be allocated while a stream is captured
    char* arena = nullptr;
    size_t arena_cap = 0, arena_used = 0;
    PFN_memop64 wait64 = nullptr, write64 = nullptr;
    PFN_batch_memop batch_memop = nullptr;   // several flag waits / writes in one stream operation
    uint64_t timeout_ns = 20ull * 1000 * 1000 * 1000;
    uint32_t unit_bytes = kDefaultUnit;
    uint64_t group_bytes = kDefaultGroupBytes;   // ring hop groups (plane.cpp group_chunks)
    int hop_lanes = 2;                           // relay hop streams per direction used (1 or 2)
    bool relay_bulk = false;                     // MMA_RELAY_BULK=1: the cp.async.bulk relay kernels
    bool zc_bulk = true;                         // MMA_ZC_BULK=0: direct zero-copy paths use the vector kernel
    int zc_ctas_dir[2] = {0, 0};                 // MMA_ZC_CTAS_{H2D,D2H}: per-direction zero-copy grid (0 = cfg.zc_ctas)
    bool upload_by_kernel = true;    // MMA_UPLOAD=ce: table uploads by the copy engine
    // fault injection (tests only, MMA_FAULT_DROP_PUBLISH=g): the hop-1 publish of global
    // ring chunk g is never issued, so the relay kernel must time out, record the sticky
    // error and release the ring instead of hanging (SURVEY §5 failure detection)
    long long fault_drop_publish = -1;
    // fault injection (tests only, MMA_FAULT_FAIL_RINGS=1): the ring stage of every call fails
    // after the direct path was enqueued, to check that a failed call still joins its streams
    bool fault_fail_rings = false;
    // fault injection (tests only, MMA_FAULT_FAIL_HOP=k): the k-th copy-engine ring hop the
    // engine enqueues (counted from init, 0-based) fails once, in the middle of a call whose
    // rings have already advanced, to check ring poisoning and the join of a failed call
    long long fault_fail_hop = -1;
    // fault injection (tests only, MMA_FAULT_MISROUTE=1): after planning, path 0's last chunk
    // is moved to path 1's work list, so the engine carries a plan other than the one it
    // reports; the delivery log (written by the hop that moves each chunk) must show it
    bool fault_misroute = false;
    long long hops_issued = 0;
};

Engine& E();

size_t env_size(const char* name, size_t dflt);

int env_int(const char* name, int dflt);


// ------------------------------------------------------------------ transfer job ---

struct Piece {
    uint64_t v;       // offset in v
    uint64_t len;
    const char* src;
    char* dst;
};

// Measurement runs (concurrent calibration): per path, timing events
// bracketing the work each engine stream does for that path, recorded on that stream. A
// path's time is the longest of its spans; every span starts when its stream passes the
// call's fork, so the spans of one call share an origin.
struct PathTiming {
    struct Span {
        int dev;
        cudaStream_t s;
        cudaEvent_t a, b;
    };
    std::vector<std::vector<Span>> path;
    std::vector<uint64_t> bytes;      // bytes the plan gave each path
    explicit PathTiming(int P) : path(P), bytes(P, 0) {}
    ~PathTiming();
    void start(int p, int dev, cudaStream_t s);   // once per (path, stream)
    void end(int p);                              // closes every open span of p
    int collect(std::vector<float>& ms);          // synchronises; 0 ms = no span
};

struct Job {
    int dir = 0;
    int d = 0;                       // target GPU
    cudaStream_t user = nullptr;
    int user_dev = 0;
    uint64_t B = 0;
    uint64_t C = 0;
    bool contiguous = true;
    const char* src0 = nullptr;
    char* dst0 = nullptr;
    const mma_segment_t* segs = nullptr;
    uint64_t nseg = 0;
    std::vector<uint64_t> vstart;    // segmented: prefix offsets [nseg + 1]
    bool mapped = false;             // every host address is usable by GPU SMs
    bool pageable = false;           // segmented: some host segment is pageable (native copy)
    double validate_us = 0;          // segmented: host time classifying the table
    uint64_t ptr_queries = 0;
    const uint32_t* bw_override = nullptr;   // measurement runs: per-path bandwidth
    const int* mode_override = nullptr;      // measurement runs: per-path mode
    const std::vector<uint8_t>* plan_override = nullptr;   // joint plans: path of each chunk
    bool interleaved_plan = false;           // the given plan is not contiguous per path
    bool no_log = false;                     // joint plans: another transfer to this GPU keeps the log
    bool no_small_fallback = false;          // measurement runs: ignore the threshold
    PathTiming* timing = nullptr;            // measurement runs: per-path events (planned plans only)
    bool capturing = false;                  // the user stream is being captured into a graph

    // pieces of v[a, b) (the per-segment parts; one piece when contiguous)
    template <typename F>
    void pieces(uint64_t a, uint64_t b, F f) const
    {
        if (a >= b) return;
        if (contiguous) { f(Piece{a, b - a, src0 + a, dst0 + a}); return; }
        uint64_t k = std::upper_bound(vstart.begin(), vstart.end(), a) - vstart.begin() - 1;
        for (; k < nseg && vstart[k] < b; k++) {
            uint64_t lo = std::max(vstart[k], a), hi = std::min(vstart[k + 1], b);
            if (lo >= hi) continue;
            f(Piece{lo, hi - lo, (const char*)segs[k].src + (lo - vstart[k]),
                    (char*)segs[k].dst + (lo - vstart[k])});
        }
    }
    void extent(uint64_t i, uint64_t* off, uint64_t* len) const
    {
        *off = i * C;
        *len = std::min(C, B - *off);
    }
};

void order_by_key(const uint64_t* key, size_t n, std::vector<uint32_t>& perm);

// Pieces copied by the copy engine: one cudaMemcpyAsync per merged run of pieces. Scattered
// transfers with many pieces go to the zero-copy kernels instead (MMA_HOP_AUTO), since each
// DMA costs host issue time.
struct DmaBatch {
    std::vector<void*> dst, src;
    std::vector<size_t> len;
    void add(void* d, const void* s, size_t n)
    {
        if (!n) return;
        if (!dst.empty() && (char*)dst.back() + len.back() == (char*)d && (const char*)src.back() + len.back() == (const char*)s) {
            len.back() += n;    // merge adjacent pieces
            return;
        }
        dst.push_back(d);
        src.push_back(const_cast<void*>(s));
        len.push_back(n);
    }
    // issue order = ascending host address (the copies are independent; config host_order)
    void sort_by_host(cudaMemcpyKind kind)
    {
        if (dst.size() < 2) return;
        const std::vector<void*>& h = kind == cudaMemcpyDeviceToHost ? dst : src;
        std::vector<uint64_t> key(h.size());
        for (size_t i = 0; i < h.size(); i++) key[i] = (uint64_t)h[i];
        std::vector<uint32_t> perm;
        order_by_key(key.data(), key.size(), perm);
        std::vector<void*> d2(dst.size()), s2(src.size());
        std::vector<size_t> l2(len.size());
        for (size_t i = 0; i < perm.size(); i++) {
            d2[i] = dst[perm[i]];
            s2[i] = src[perm[i]];
            l2[i] = len[perm[i]];
        }
        dst.swap(d2);
        src.swap(s2);
        len.swap(l2);
    }
    int issue(cudaMemcpyKind kind, cudaStream_t s)
    {
        for (size_t i = 0; i < dst.size(); i++) CK(cudaMemcpyAsync(dst[i], src[i], len[i], kind, s));
        return cudaSuccess;
    }
};

// ---- plane.cpp
void apply_env(mma_config_t* c);
void defaults(mma_config_t* c);
int validate_cfg(const mma_config_t& c);
int make_device(int d);
// grid of a zero-copy path kernel on device d moving direction dir (cfg.zc_ctas, or the
// engine's per-direction grid; capped at 4 CTAs per SM)
uint64_t zc_grid(int d, int dir);
uint32_t ring_slots_for(uint64_t C);   // the ring depth for chunks of C bytes
int do_init(const mma_config_t* cfg);
int ensure_init();
void make_paths(int d);
void free_ring(Ring& r);
int get_ring(int d, int dir, int p, uint64_t C, uint32_t S, bool push, Ring** out);
int ring_kdev(int d, int dir, int relay, int mode);   // the GPU running a kernel ring's relay kernel
inline bool kernel_ring(int mode) { return mode == MMA_HOP_CE || mode == MMA_HOP_PUSH; }
// gate (optional): GPUs whose own direct work is in flight in this process; a relay through
// one of them is planned behind that backlog and waits for it (direct path first)
void ledger_inputs(int d, int dir, const std::vector<PathState>& ps, std::vector<PlanPath>& pp,
                   std::vector<int>* gate = nullptr);
// record gate_ev of GPU g for direction dir behind its direct and zero-copy lanes
int record_gates(int g, int dir);
void ledger_retire();
// ---- ledger_shm.cpp: the cross-process ledger (mma_ledger_attach)
bool shm_ledger_on();
uint64_t shm_ledger_gen();   // attach generation; 0 when detached
// adds to this process's entry, if `gen` is still the current attach (else the bytes left
// the ledger with the old attach)
void shm_ledger_add(int dir, int dev, int64_t bytes, int64_t own, uint64_t gen);
void shm_ledger_get(int dir, int dev, uint64_t* bytes, uint64_t* own);
int shm_ledger_slot(int dev);   // -1 when detached; resolves the bus id (a CUDA call)
void shm_ledger_add_slot(int dir, int slot, int64_t bytes, int64_t own, uint64_t gen);   // no CUDA calls
int run_job(Job& j);
int run_multi(std::vector<Job>& jobs);   // a joint plan of concurrent transfers (NEXT-1)
void mp_finalize();                      // mp.cpp: free the copy-engine share rings
int reserve_tables(const Job& j);
int sticky();
extern bool g_ktime;
extern thread_local bool tl_capturing;   // no timing / trace events inside a capture
struct KRec {
    int dev;
    int kind;   // 0 zero-copy, 1 relay pull (H2D), 2 relay pack (D2H), 3 dynamic | dir << 4 | path << 8 | dev << 16
    cudaEvent_t a, b;
};
extern std::vector<KRec> g_kpending;
extern std::mutex g_kmu;
// CUDA events around one kernel launch on its stream while kernel timing is on
struct KTimer {
    bool on = false;
    KRec r{};
    cudaStream_t s = nullptr;
    KTimer(int dev, cudaStream_t st, int kind)
    {
        if (!g_ktime || tl_capturing) return;
        DeviceGuard g(dev);
        if (cudaEventCreate(&r.a) != cudaSuccess || cudaEventCreate(&r.b) != cudaSuccess) return;
        r.dev = dev;
        r.kind = kind | (dev << 16);
        s = st;
        on = cudaEventRecord(r.a, s) == cudaSuccess;
    }
    ~KTimer()
    {
        if (!on) return;
        DeviceGuard g(r.dev);
        cudaEventRecord(r.b, s);
        std::lock_guard<std::mutex> lk(g_kmu);
        g_kpending.push_back(r);
    }
};

// ---- trace.cpp: a span of stream work bracketed by CUDA events while a trace is active
struct TSpan {
    long long idx_ = -1;
    TSpan(int dev, cudaStream_t s, const char* name, int path, long long chunk, uint64_t bytes);
    ~TSpan();
};
bool trace_on();
// ---- api.cpp
int load_calibration_locked(const char* path, int* applied);
int prepare_segments(int dir, const mma_segment_t* segs, size_t nsegs, int device, cudaStream_t stream, Job& j);

}  // namespace mma
