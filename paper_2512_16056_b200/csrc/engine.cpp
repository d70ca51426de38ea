// engine.cpp — the multipath data plane (C6) and its C ABI (C7).
//
// One user copy of B bytes between pinned host memory and GPU d becomes n chunks; each
// chunk travels over exactly one path:
//   direct   d's own PCIe link: copy-engine DMA ("a single H2D transfer operation")
//            or SM zero-copy (north_star (d));
//   relay r  r's PCIe link into r's HBM staging ring, then NVLink r -> d pulled by the
//            relay kernel on d ("an H2D operation and a P2P operation ... with a
//            dependency"; dual pipeline generalised to S slots); D2H mirrors it. In
//            zero-copy mode a relay is one hop: a kernel on r reads host memory over r's
//            PCIe and stores into d's HBM over NVLink.
// The paper's Dummy Task + callback + spin kernel (§3.3, §4) is
// replaced by GPU-ordered fork/join: an event recorded on the user stream gates every path
// stream and every path stream's completion event gates the user stream, so the copy is
// ordered exactly like cudaMemcpyAsync with no CPU thread in the per-chunk loop (the
// paper's 2 threads per GPU, cost 822% CPU at 8 GPUs). Per relay chunk
// the host enqueues: wait(credit) -> DMA -> write(seq) on the relay's stream (cuda.h stream
// memory operations); the relay kernel polls seq and releases credit on the GPU.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
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

namespace {

using PFN_memop64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);

constexpr uint64_t kDefaultChunk = 4ull << 20;
constexpr unsigned kDefaultSlots = 4;
constexpr uint32_t kDefaultMbps = 50000;
constexpr uint32_t kDefaultUnit = 128u << 10;
constexpr int kDefaultRelayCtas = 8;
constexpr unsigned kDynSlots = 64;        // per-call claim slots, rotating
constexpr unsigned kDynSlotWords = 32;    // cursor + counts[MMA_KMAX_RINGS] (+ padding)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int d)
    {
        cudaGetDevice(&prev);
        if (d != prev) cudaSetDevice(d);
    }
    ~DeviceGuard()
    {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

struct DevRes {
    bool made = false;
    cudaStream_t direct = nullptr;   // direct-path DMA
    cudaStream_t zc = nullptr;       // zero-copy kernels (direct or one-hop relay)
    cudaStream_t hop[2] = {};        // relay hop DMAs: dual pipeline, slot parity
    cudaStream_t kern = nullptr;     // relay kernels (pull on a target, pack on a relay)
    cudaEvent_t fork = nullptr;      // recorded on a user stream of this device
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
    uint64_t g_next = 0;             // chunks carried so far (reading R18)
    unsigned long long unit_next = 0;
};

struct PathState {
    int gpu;
    int kind;       // MMA_PATH_DIRECT / MMA_PATH_RELAY
    uint32_t mbps;
    int mode;       // mma_hop_t
    uint32_t seg_mbps = 0;   // measured for scattered transfers (mma_tune_segments); 0 = unset
    int seg_mode = -1;       // idem; -1 = unset
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
    Scratch scratch[4];   // table buffers of the last 4 calls (a ring)
    unsigned parity = 0;
    unsigned long long* dyn = nullptr;        // dynamic-pull slots: cursor + per-path counts
    unsigned dyn_next = 0;
    unsigned long long* last_dyn = nullptr;
    int last_dyn_paths = 0;
};

struct Engine {
    std::mutex mu;                   // one multipath enqueue at a time
    bool inited = false;
    mma_config_t cfg{};
    int ndev = 0;
    bool p2p[MMA_MAX_GPUS][MMA_MAX_GPUS] = {};
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
    };
    std::vector<InFlight> inflight;
    std::vector<std::pair<int, cudaEvent_t>> free_events;
    uint64_t ledger[2][MMA_MAX_GPUS] = {};
    uint64_t ledger_own[2][MMA_MAX_GPUS] = {};
    int* err = nullptr;              // mapped pinned host word (sticky async error)
    PFN_memop64 wait64 = nullptr, write64 = nullptr;
    uint64_t timeout_ns = 20ull * 1000 * 1000 * 1000;
    uint32_t unit_bytes = kDefaultUnit;
    // fault injection (tests only, MMA_FAULT_DROP_PUBLISH=g): the hop-1 publish of global
    // ring chunk g is never issued, so the relay kernel must time out, record the sticky
    // error and release the ring instead of hanging (SURVEY §5 failure detection)
    long long fault_drop_publish = -1;
};

Engine& E()
{
    static Engine* e = new Engine();   // never destroyed: safe at process exit
    return *e;
}

size_t env_size(const char* name, size_t dflt)
{
    const char* s = getenv(name);
    if (!s || !*s) return dflt;
    char* end = nullptr;
    double v = strtod(s, &end);
    std::string suf = end ? end : "";
    if (suf == "K" || suf == "k" || suf == "KiB") v *= 1024;
    else if (suf == "M" || suf == "m" || suf == "MiB") v *= 1024 * 1024;
    else if (suf == "G" || suf == "g" || suf == "GiB") v *= 1024.0 * 1024 * 1024;
    return (size_t)v;
}

int env_int(const char* name, int dflt)
{
    const char* s = getenv(name);
    return (s && *s) ? atoi(s) : dflt;
}

}  // namespace

// ------------------------------------------------------------------- configuration ---

static void apply_env(mma_config_t* c)
{
    c->chunk_bytes[0] = env_size("MMA_CHUNK_BYTES_H2D", env_size("MMA_CHUNK_BYTES", c->chunk_bytes[0]));
    c->chunk_bytes[1] = env_size("MMA_CHUNK_BYTES_D2H", env_size("MMA_CHUNK_BYTES", c->chunk_bytes[1]));
    c->ring_slots = (unsigned)env_int("MMA_RING_SLOTS", (int)c->ring_slots);
    c->fallback_bytes[0] = env_size("MMA_FALLBACK_BYTES_H2D", env_size("MMA_FALLBACK_BYTES", c->fallback_bytes[0]));
    c->fallback_bytes[1] = env_size("MMA_FALLBACK_BYTES_D2H", env_size("MMA_FALLBACK_BYTES", c->fallback_bytes[1]));
    c->loopback_relays = env_int("MMA_LOOPBACK", c->loopback_relays);
    c->plan_mode = env_int("MMA_PLAN_MODE", c->plan_mode);
    c->hop_mode[0] = env_int("MMA_HOP_H2D", env_int("MMA_HOP", c->hop_mode[0]));
    c->hop_mode[1] = env_int("MMA_HOP_D2H", env_int("MMA_HOP", c->hop_mode[1]));
    c->relay_ctas = env_int("MMA_RELAY_CTAS", c->relay_ctas);
    c->numa_mode = env_int("MMA_NUMA", c->numa_mode);
    c->debug_log = env_int("MMA_DEBUG_LOG", c->debug_log);
    c->ledger = env_int("MMA_LEDGER", c->ledger);
    if (const char* s = getenv("MMA_PATHS")) {   // comma-separated relay GPU ids
        c->npaths = 0;
        for (const char* p = s; *p && c->npaths < MMA_MAX_PATHS;) {
            char* end;
            long v = strtol(p, &end, 10);
            if (end == p) break;
            c->path_gpus[c->npaths++] = (int)v;
            p = (*end == ',') ? end + 1 : end;
        }
    }
}

static void defaults(mma_config_t* c)
{
    memset(c, 0, sizeof(*c));
    c->chunk_bytes[0] = c->chunk_bytes[1] = kDefaultChunk;
    c->ring_slots = kDefaultSlots;
    // Fallback threshold: "between two and five chunks" (§5.1.3); 2 chunks until the
    // B200 break-even sweep replaces it.
    c->fallback_bytes[0] = c->fallback_bytes[1] = 2 * kDefaultChunk;
    c->plan_mode = PLAN_CONTIGUOUS;
    c->hop_mode[0] = c->hop_mode[1] = MMA_HOP_AUTO;
    c->relay_ctas = kDefaultRelayCtas;
    c->ledger = 1;
}

static int validate_cfg(const mma_config_t& c)
{
    for (int d = 0; d < 2; d++)
        if (c.chunk_bytes[d] == 0 || c.chunk_bytes[d] % 4096) return cudaErrorInvalidValue;
    if (c.ring_slots < 1 || c.ring_slots > 64) return cudaErrorInvalidValue;
    if (c.npaths < 0 || c.npaths > MMA_MAX_PATHS) return cudaErrorInvalidValue;
    if (c.loopback_relays < 0 || c.loopback_relays > 8) return cudaErrorInvalidValue;
    if (c.plan_mode < PLAN_CONTIGUOUS || c.plan_mode > PLAN_DYNAMIC) return cudaErrorInvalidValue;
    for (int d = 0; d < 2; d++)
        if (c.hop_mode[d] < MMA_HOP_AUTO || c.hop_mode[d] > MMA_HOP_ZC) return cudaErrorInvalidValue;
    if (c.relay_ctas < 1 || c.relay_ctas > 64) return cudaErrorInvalidValue;
    return cudaSuccess;
}

// Streams, peer access and flags for device d (lazily, once).
static int make_device(int d)
{
    Engine& e = E();
    DevRes& r = e.dev[d];
    if (r.made) return cudaSuccess;
    DeviceGuard g(d);
    int lo, hi;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    // Five streams created back to back so they land on distinct hardware queues: a
    // spinning relay kernel must never sit in front of the DMAs it waits for.
    CK(cudaStreamCreateWithPriority(&r.kern, cudaStreamNonBlocking, hi));
    CK(cudaStreamCreateWithPriority(&r.hop[0], cudaStreamNonBlocking, hi));
    CK(cudaStreamCreateWithPriority(&r.hop[1], cudaStreamNonBlocking, hi));
    CK(cudaStreamCreateWithPriority(&r.direct, cudaStreamNonBlocking, hi));
    CK(cudaStreamCreateWithPriority(&r.zc, cudaStreamNonBlocking, hi));
    CK(cudaEventCreateWithFlags(&r.fork, cudaEventDisableTiming));
    CK(cudaDeviceGetAttribute(&r.sms, cudaDevAttrMultiProcessorCount, d));
    for (int p = 0; p < e.ndev; p++) {
        if (p == d || !e.p2p[d][p]) continue;
        cudaError_t pe = cudaDeviceEnablePeerAccess(p, 0);
        if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else if (pe != cudaSuccess) { cudaGetLastError(); e.p2p[d][p] = false; }
    }
    r.made = true;
    return cudaSuccess;
}

static int do_init(const mma_config_t* cfg)
{
    Engine& e = E();
    mma_config_t c;
    if (cfg) c = *cfg;
    else { defaults(&c); apply_env(&c); }
    CK((cudaError_t)validate_cfg(c));
    if (!e.inited) {
        CK(cudaGetDeviceCount(&e.ndev));
        if (e.ndev > MMA_MAX_GPUS) e.ndev = MMA_MAX_GPUS;
        for (int a = 0; a < e.ndev; a++)
            for (int b = 0; b < e.ndev; b++) {
                int ok = 0;
                if (a != b) cudaDeviceCanAccessPeer(&ok, a, b);
                e.p2p[a][b] = ok != 0;
            }
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue64", &fn, 12000, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            e.wait64 = (PFN_memop64)fn;
        fn = nullptr;
        if (cudaGetDriverEntryPointByVersion("cuStreamWriteValue64", &fn, 12000, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            e.write64 = (PFN_memop64)fn;
        CK(cudaHostAlloc((void**)&e.err, sizeof(int) * 16, cudaHostAllocPortable | cudaHostAllocMapped));
        memset(e.err, 0, sizeof(int) * 16);
        e.timeout_ns = (uint64_t)env_size("MMA_SPIN_TIMEOUT_MS", 20000) * 1000000ull;
        e.unit_bytes = (uint32_t)env_size("MMA_UNIT_BYTES", kDefaultUnit);
        const char* f = getenv("MMA_FAULT_DROP_PUBLISH");
        e.fault_drop_publish = f ? atoll(f) : -1;
        if (e.unit_bytes < 4096) e.unit_bytes = 4096;
    }
    e.cfg = c;
    for (int d = 0; d < e.ndev; d++) e.tgt[d].paths_made = false;   // re-derive path sets
    e.inited = true;
    return cudaSuccess;
}

static int ensure_init()
{
    Engine& e = E();
    if (e.inited) return cudaSuccess;
    std::lock_guard<std::mutex> g(e.mu);
    if (e.inited) return cudaSuccess;
    return do_init(nullptr);
}

// Path set of target d: path 0 = d's own link, then relay GPUs in calibration order, then
// loopback relays (reading R11).
static void make_paths(int d)
{
    Engine& e = E();
    Target& t = e.tgt[d];
    if (t.paths_made) return;
    for (int dir = 0; dir < 2; dir++) {
        std::vector<PathState> ps;
        ps.push_back({d, MMA_PATH_DIRECT, kDefaultMbps, e.cfg.hop_mode[dir]});
        std::vector<int> cand;
        if (e.cfg.npaths > 0) cand.assign(e.cfg.path_gpus, e.cfg.path_gpus + e.cfg.npaths);
        else for (int g = 0; g < e.ndev; g++) cand.push_back(g);
        for (int g : cand) {
            if (g < 0 || g >= e.ndev || g == d || !e.p2p[d][g] || !e.p2p[g][d]) continue;
            bool dup = false;
            for (auto& p : ps) dup |= (p.gpu == g);
            if (!dup && ps.size() < MMA_MAX_PATHS) ps.push_back({g, MMA_PATH_RELAY, kDefaultMbps, e.cfg.hop_mode[dir]});
        }
        for (int k = 0; k < e.cfg.loopback_relays && ps.size() < MMA_MAX_PATHS; k++)
            ps.push_back({d, MMA_PATH_RELAY, kDefaultMbps, e.cfg.hop_mode[dir]});
        // keep a previously pinned vector when the set is unchanged
        if (t.paths[dir].size() == ps.size()) {
            bool same = true;
            for (size_t i = 0; i < ps.size(); i++) same &= ps[i].gpu == t.paths[dir][i].gpu && ps[i].kind == t.paths[dir][i].kind;
            if (same)
                for (size_t i = 0; i < ps.size(); i++) {   // measured / pinned values survive
                    ps[i].mbps = t.paths[dir][i].mbps;
                    ps[i].seg_mbps = t.paths[dir][i].seg_mbps;
                    ps[i].seg_mode = t.paths[dir][i].seg_mode;
                }
        }
        t.paths[dir] = ps;
    }
    t.paths_made = true;
}

// --------------------------------------------------------------------- the rings ---

static void free_ring(Ring& r)
{
    if (!r.made) return;
    { DeviceGuard g(r.relay); cudaFree(r.stage); cudaFree(r.seq); }
    { DeviceGuard g(r.kdev); cudaFree(r.cnt); }
    r = Ring();
}

// Ring of path p of target d in direction dir: S slots of C bytes on the relay.
static int get_ring(int d, int dir, int p, uint64_t C, uint32_t S, Ring** out)
{
    Engine& e = E();
    Ring& r = e.tgt[d].rings[dir][p];
    const int relay = e.tgt[d].paths[dir][p].gpu;
    const int kdev = (dir == MMA_H2D) ? d : relay;
    if (r.made && (r.slot_bytes < C || r.S != S || r.relay != relay)) {
        // tunables changed: drain everything that may still use the old ring
        { DeviceGuard g(r.relay); cudaDeviceSynchronize(); }
        { DeviceGuard g(r.kdev); cudaDeviceSynchronize(); }
        free_ring(r);
    }
    if (!r.made) {
        r.relay = relay;
        r.kdev = kdev;
        r.S = S;
        r.slot_bytes = C;
        {
            DeviceGuard g(relay);
            CK(cudaMalloc(&r.stage, (size_t)S * C));
            CK(cudaMalloc(&r.seq, 2 * 64 * sizeof(uint64_t)));
            CK(cudaMemset(r.seq, 0, 2 * 64 * sizeof(uint64_t)));
            r.credit = r.seq + 64;
        }
        {
            DeviceGuard g(kdev);
            CK(cudaMalloc(&r.cnt, 64 * sizeof(unsigned) + 64));
            CK(cudaMemset(r.cnt, 0, 64 * sizeof(unsigned) + 64));
            r.cursor = (unsigned long long*)((char*)r.cnt + 64 * sizeof(unsigned));
        }
        CK(cudaDeviceSynchronize());
        r.g_next = 0;
        r.unit_next = 0;
        r.made = true;
    }
    *out = &r;
    return cudaSuccess;
}

// ------------------------------------------------------------------ transfer job ---

struct Piece {
    uint64_t v;       // offset in v
    uint64_t len;
    const char* src;
    char* dst;
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
    const uint32_t* bw_override = nullptr;   // measurement runs: per-path bandwidth
    const int* mode_override = nullptr;      // measurement runs: per-path mode
    bool no_small_fallback = false;          // measurement runs: ignore the threshold

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

// Pieces copied by one DMA call: cudaMemcpyAsync for one, cudaMemcpyBatchAsync for many.
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
    int issue(cudaMemcpyKind kind, cudaStream_t s)
    {
        if (dst.empty()) return cudaSuccess;
        if (dst.size() == 1) return (int)cudaMemcpyAsync(dst[0], src[0], len[0], kind, s);
        if (s == nullptr || s == cudaStreamLegacy) {   // the batch API rejects the legacy stream
            for (size_t i = 0; i < dst.size(); i++) CK(cudaMemcpyAsync(dst[i], src[i], len[i], kind, s));
            return cudaSuccess;
        }
        cudaMemcpyAttributes at;
        memset(&at, 0, sizeof(at));
        at.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
        size_t idx = 0, fail = 0;
        cudaError_t e = cudaMemcpyBatchAsync(dst.data(), src.data(), len.data(), dst.size(), &at, &idx, 1, &fail, s);
        if (e == cudaSuccess) return cudaSuccess;
        cudaGetLastError();
        for (size_t i = 0; i < dst.size(); i++) CK(cudaMemcpyAsync(dst[i], src[i], len[i], kind, s));
        return cudaSuccess;
    }
};

static cudaEvent_t join_event(cudaStream_t s, int dev)
{
    Engine& e = E();
    auto it = e.join_ev.find(s);
    if (it != e.join_ev.end()) return it->second;
    DeviceGuard g(dev);
    cudaEvent_t ev = nullptr;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    e.join_ev[s] = ev;
    return ev;
}

// Grow-only device scratch on device `dev` for this call's tables.
static int scratch_dev(Scratch& sc, int dev, size_t bytes, void** out)
{
    if (sc.dev_cap[dev] < bytes) {
        DeviceGuard g(dev);
        if (sc.dev[dev]) cudaFree(sc.dev[dev]);
        sc.dev[dev] = nullptr;
        size_t cap = std::max(bytes, (size_t)1 << 20);
        CK(cudaMalloc(&sc.dev[dev], cap));
        sc.dev_cap[dev] = cap;
    }
    *out = sc.dev[dev];
    return cudaSuccess;
}

static int scratch_host(Scratch& sc, size_t bytes, void** out)
{
    if (sc.host_cap < bytes) {
        if (sc.host) cudaFreeHost(sc.host);
        sc.host = nullptr;
        size_t cap = std::max(bytes, (size_t)1 << 20);
        CK(cudaHostAlloc(&sc.host, cap, cudaHostAllocPortable));
        sc.host_cap = cap;
    }
    *out = sc.host;
    return cudaSuccess;
}

// Optional per-launch CUDA-event timing of the engine's kernels, recorded on the stream
// the kernel is launched on (mma_set_kernel_timing / mma_kernel_times).
struct KRec {
    int dev;
    int kind;   // 0 zero-copy, 1 relay pull (H2D), 2 relay pack (D2H) | dir << 4 | path << 8 | dev << 16
    cudaEvent_t a, b;
};
static std::vector<KRec> g_kpending;
static bool g_ktime = false;

struct KTimer {
    bool on = false;
    KRec r{};
    cudaStream_t s = nullptr;
    KTimer(int dev, cudaStream_t st, int kind)
    {
        if (!g_ktime) return;
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
        g_kpending.push_back(r);
    }
};

static int resolve_mode(const Job& j, int mode)
{
    if (mode == MMA_HOP_AUTO) mode = j.contiguous ? MMA_HOP_CE : MMA_HOP_ZC;
    if (mode == MMA_HOP_ZC && !j.mapped) mode = MMA_HOP_CE;
    return mode;
}

// ---- backlog ledger (NEXT-1) ---------------------------------------------------------
static void ledger_retire()
{
    Engine& e = E();
    for (size_t i = 0; i < e.inflight.size();) {
        auto& f = e.inflight[i];
        if (cudaEventQuery(f.done) == cudaErrorNotReady) { i++; continue; }
        cudaGetLastError();
        for (int g = 0; g < MMA_MAX_GPUS; g++) {
            e.ledger[f.dir][g] -= f.bytes[g];
            e.ledger_own[f.dir][g] -= f.own[g];
        }
        e.free_events.push_back({f.dev, f.done});
        e.inflight[i] = e.inflight.back();
        e.inflight.pop_back();
    }
}

static int ledger_add(int dir, int user_dev, cudaStream_t user, const uint64_t* bytes, const uint64_t* own)
{
    Engine& e = E();
    Engine::InFlight f{};
    f.dir = dir;
    f.dev = user_dev;
    for (size_t i = 0; i < e.free_events.size(); i++)
        if (e.free_events[i].first == user_dev) {
            f.done = e.free_events[i].second;
            e.free_events.erase(e.free_events.begin() + i);
            break;
        }
    DeviceGuard g(user_dev);
    if (!f.done) CK(cudaEventCreateWithFlags(&f.done, cudaEventDisableTiming));
    CK(cudaEventRecord(f.done, user));
    for (int k = 0; k < MMA_MAX_GPUS; k++) {
        f.bytes[k] = bytes[k];
        f.own[k] = own[k];
        e.ledger[dir][k] += bytes[k];
        e.ledger_own[dir][k] += own[k];
    }
    e.inflight.push_back(f);
    return cudaSuccess;
}

// Planner inputs of target d's paths: bandwidth (0 = not usable for this call) and
// backlog from the ledger.
static void ledger_inputs(int d, int dir, const std::vector<PathState>& ps, std::vector<PlanPath>& pp)
{
    Engine& e = E();
    if (!e.cfg.ledger) return;
    ledger_retire();
    for (size_t p = 0; p < ps.size(); p++) {
        const int g = ps[p].gpu;
        pp[p].backlog = e.ledger[dir][g];
        // direct path first: a GPU whose link still carries its own target's bytes takes
        // no relay work for another target
        if (ps[p].kind == MMA_PATH_RELAY && g != d && e.ledger_own[dir][g] > 0) pp[p].mbps = 0;
    }
}

// MMA_TRACE=1: per-call host-time breakdown of the enqueue on stderr.
struct Trace {
    bool on;
    std::chrono::steady_clock::time_point last;
    std::string s;
    Trace() : on(getenv("MMA_TRACE") != nullptr), last(std::chrono::steady_clock::now()) {}
    void mark(const char* what)
    {
        if (!on) return;
        auto now = std::chrono::steady_clock::now();
        char buf[64];
        snprintf(buf, sizeof buf, " %s=%.0fus", what, std::chrono::duration<double, std::micro>(now - last).count());
        s += buf;
        last = now;
    }
    ~Trace()
    {
        if (on && !s.empty()) fprintf(stderr, "[mma]%s\n", s.c_str());
    }
};

// Enqueue one multipath copy (engine mutex held).
static int run_job(Job& j)
{
    Engine& e = E();
    Target& t = e.tgt[j.d];
    Trace tr;
    const auto t0 = std::chrono::steady_clock::now();
    const cudaMemcpyKind kind = (j.dir == MMA_H2D) ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
    make_paths(j.d);
    std::vector<PathState>& ps = t.paths[j.dir];
    const int P = (int)ps.size();

    // ---- plan (a2)
    std::vector<PlanPath> pp(P);
    std::vector<int> pmode(P);
    for (int p = 0; p < P; p++) {
        uint32_t bw = (!j.contiguous && ps[p].seg_mbps) ? ps[p].seg_mbps : ps[p].mbps;
        if (j.bw_override) bw = j.bw_override[p];
        pp[p] = PlanPath{ps[p].kind == MMA_PATH_DIRECT, bw, 0};
        pmode[p] = (!j.contiguous && ps[p].seg_mode >= 0) ? ps[p].seg_mode : ps[p].mode;
        if (j.mode_override) pmode[p] = j.mode_override[p];
    }
    const uint64_t thr = j.no_small_fallback ? 0 : e.cfg.fallback_bytes[j.dir];
    if (!j.bw_override) ledger_inputs(j.d, j.dir, ps, pp);
    Plan plan;
    const int pmode_plan = e.cfg.plan_mode == PLAN_DYNAMIC ? PLAN_CONTIGUOUS : e.cfg.plan_mode;
    if (make_plan(pp.data(), P, j.B, j.C, thr, pmode_plan, plan) != 0)
        return cudaErrorInvalidValue;
    t.stats.calls++;
    t.stats.bytes += j.B;
    tr.mark("plan");

    // ---- fallback (a1): the native copy on the user stream (§3.2)
    if (plan.fallback) {
        t.stats.fallbacks++;
        const int mode0 = resolve_mode(j, pmode[0]);
        const bool small = j.B < thr;
        if (small || mode0 == MMA_HOP_CE) {
            DmaBatch b;
            j.pieces(0, j.B, [&](const Piece& x) { b.add(x.dst, x.src, x.len); });
            CK((cudaError_t)b.issue(kind, j.user));
            t.stats.path_bytes[j.dir][0] += j.B;
            t.stats.path_chunks[j.dir][0] += 1;
            t.log_n = 0;
            if (e.cfg.ledger) {
                uint64_t lb[MMA_MAX_GPUS] = {}, lo[MMA_MAX_GPUS] = {};
                lb[j.d] = lo[j.d] = j.B;
                CK(ledger_add(j.dir, j.user_dev, j.user, lb, lo));
            }
            t.stats.issue_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
            return cudaSuccess;
        }
        // single direct path moved by SM zero-copy: fall through with a one-path plan
        plan.fallback = false;
        plan.n = (j.B - 1) / j.C + 1;
        plan.path.assign(plan.n, 0);
        plan.count.assign(P, 0);
        plan.count[0] = plan.n;
    }

    const uint64_t n = plan.n;
    Scratch& sc = t.scratch[t.parity & 3];
    t.parity++;
    if (sc.pending) {   // the call four back used these tables: it must be finished
        const auto w0 = std::chrono::steady_clock::now();
        CK(cudaEventSynchronize(sc.done));
        sc.pending = false;
        t.stats.wait_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - w0).count();
    }
    // every GPU of the path set gets its streams and peer access before any enqueue
    for (int p = 0; p < P; p++) CK(make_device(ps[p].gpu));
    tr.mark("scratch");

    // ---- per-path chunk lists, ascending
    std::vector<std::vector<uint32_t>> lists(P);
    for (uint64_t i = 0; i < n; i++) lists[plan.path[i]].push_back((uint32_t)i);
    std::vector<int> mode(P);
    for (int p = 0; p < P; p++) mode[p] = resolve_mode(j, pmode[p]);
    // GPU-driven dynamic pull when every usable path moves bytes with SMs:
    // the assignment is then observed (delivery log, per-path counts), not planned
    bool dynamic = e.cfg.plan_mode == PLAN_DYNAMIC && !plan.fallback;
    std::vector<char> active(P, 0);
    for (int p = 0; p < P; p++) {
        active[p] = !lists[p].empty();
        if (dynamic && pp[p].mbps && mode[p] != MMA_HOP_ZC) dynamic = false;
    }
    if (dynamic)
        for (int p = 0; p < P; p++) active[p] = pp[p].mbps > 0;

    // ---- host tables: chunk lists (interleaved plans) and the segment table
    const bool need_ctab = e.cfg.plan_mode == PLAN_INTERLEAVED && !dynamic;
    const uint64_t seg_words = j.contiguous ? 0 : (j.nseg + 1) + 2 * j.nseg;
    const size_t tab_bytes = (need_ctab ? n * 4 : 0) + ((need_ctab && (n & 1)) ? 4 : 0) + seg_words * 8;
    std::vector<size_t> ctab_off(P, 0);
    void* htab = nullptr;
    if (tab_bytes) {
        CK((cudaError_t)scratch_host(sc, tab_bytes, &htab));
        char* h = (char*)htab;
        size_t o = 0;
        if (!j.contiguous) {
            uint64_t* w = (uint64_t*)h;
            memcpy(w, j.vstart.data(), (j.nseg + 1) * 8);
            for (uint64_t k = 0; k < j.nseg; k++) {
                w[j.nseg + 1 + k] = (uint64_t)j.segs[k].src;
                w[2 * j.nseg + 1 + k] = (uint64_t)j.segs[k].dst;
            }
            o = seg_words * 8;
        }
        if (need_ctab)
            for (int p = 0; p < P; p++) {
                ctab_off[p] = o;
                memcpy(h + o, lists[p].data(), lists[p].size() * 4);
                o += lists[p].size() * 4;
            }
    }
    tr.mark("tables");
    // devices whose kernels read the tables
    bool needs_tab[MMA_MAX_GPUS] = {};
    for (int p = 0; p < P; p++) {
        if (!active[p]) continue;
        const bool relay = ps[p].kind == MMA_PATH_RELAY;
        if (mode[p] == MMA_HOP_ZC) needs_tab[ps[p].gpu] = true;
        else if (relay) needs_tab[j.dir == MMA_H2D ? j.d : ps[p].gpu] = true;
    }

    // ---- fork (a3)
    {
        DeviceGuard g(j.user_dev);
        CK(make_device(j.user_dev));
        CK(cudaEventRecord(e.dev[j.user_dev].fork, j.user));
    }
    const cudaEvent_t fork = e.dev[j.user_dev].fork;
    std::vector<std::pair<cudaStream_t, int>> used;
    auto use = [&](cudaStream_t s, int dev) -> int {
        for (auto& u : used) if (u.first == s) return cudaSuccess;
        used.push_back({s, dev});
        DeviceGuard g(dev);
        return (int)cudaStreamWaitEvent(s, fork, 0);
    };

    // table uploads, one per device that runs a kernel (before its kernels, same streams)
    void* dtab[MMA_MAX_GPUS] = {};
    for (int g = 0; g < e.ndev; g++) {
        if (!needs_tab[g] || !tab_bytes) continue;
        CK(make_device(g));
        CK((cudaError_t)scratch_dev(sc, g, tab_bytes, &dtab[g]));
        DeviceGuard dg(g);
        // upload on the kernel stream and the direct stream's order: kern first, then
        // the direct stream waits for it through an event-free trick: upload on both
        // streams' common predecessor = kern; the direct stream waits on kern below.
        CK((cudaError_t)use(e.dev[g].kern, g));
        CK(cudaMemcpyAsync(dtab[g], htab, tab_bytes, cudaMemcpyHostToDevice, e.dev[g].kern));
    }
    tr.mark("upload");
    // streams that launch table-reading kernels other than kern wait for the upload
    auto after_upload = [&](cudaStream_t s, int g) -> int {
        if (!dtab[g] || s == e.dev[g].kern) return cudaSuccess;
        cudaEvent_t ev = join_event(e.dev[g].kern, g);
        DeviceGuard dg(g);
        CK(cudaEventRecord(ev, e.dev[g].kern));
        return (int)cudaStreamWaitEvent(s, ev, 0);
    };

    auto vstream_on = [&](int g) {
        VStreamArg v{};
        v.B = j.B;
        v.C = j.C;
        if (j.contiguous) {
            v.nseg = 1;
            v.src0 = (uint64_t)j.src0;
            v.dst0 = (uint64_t)j.dst0;
        } else {
            v.nseg = j.nseg;
            const uint64_t* w = (const uint64_t*)dtab[g];
            v.start = w;
            v.src = w + j.nseg + 1;
            v.dst = w + 2 * j.nseg + 1;
        }
        return v;
    };
    auto chunks_on = [&](int p, int g) {
        ChunkListArg c{};
        c.count = lists[p].size();
        if (c.count == 0) return c;
        if (need_ctab) c.table = (const uint32_t*)((const char*)dtab[g] + ctab_off[p]);
        else c.first = lists[p][0];
        return c;
    };

    // delivery log (debug)
    uint8_t* log = nullptr;
    if (e.cfg.debug_log) {
        if (t.log_cap < n) {
            DeviceGuard g(j.d);
            if (t.log) cudaFree(t.log);
            CK(cudaMalloc(&t.log, n));
            t.log_cap = n;
        }
        log = t.log;
        t.log_n = n;
        DeviceGuard g(j.d);
        CK((cudaError_t)use(e.dev[j.d].direct, j.d));
        CK(cudaMemsetAsync(log, 0xff, n, e.dev[j.d].direct));
    } else {
        t.log_n = 0;
    }

    // ---- dynamic pull: one claim cursor per call in d's memory, one kernel per path GPU
    if (dynamic) {
        if (!t.dyn) {
            DeviceGuard g(j.d);
            CK(cudaMalloc(&t.dyn, kDynSlots * kDynSlotWords * sizeof(unsigned long long)));
        }
        unsigned long long* slot = t.dyn + (t.dyn_next++ % kDynSlots) * kDynSlotWords;
        cudaStream_t zs = e.dev[j.d].zc;
        CK((cudaError_t)use(zs, j.d));
        cudaEvent_t zeroed = join_event(zs, j.d);
        {
            DeviceGuard g(j.d);
            CK(cudaMemsetAsync(slot, 0, kDynSlotWords * sizeof(unsigned long long), zs));
            CK(cudaEventRecord(zeroed, zs));
        }
        t.last_dyn = slot;
        t.last_dyn_paths = P;
        t.stats.dynamic_calls++;
        for (int p = 0; p < P; p++) {
            if (!active[p]) continue;
            const int g = ps[p].gpu;
            cudaStream_t s = e.dev[g].zc;
            CK((cudaError_t)use(s, g));
            CK((cudaError_t)after_upload(s, g));
            DeviceGuard dg(g);
            if (s != zs) CK(cudaStreamWaitEvent(s, zeroed, 0));
            DynLaunchArg a{};
            a.v = vstream_on(g);
            a.nchunks = n;
            a.cursor = slot;
            a.counts = slot + 1;
            a.path = (uint32_t)p;
            a.log = log;
            const unsigned grid = (unsigned)std::min<uint64_t>(n, (uint64_t)e.dev[g].sms * 4);
            KTimer kt(g, s, 3 | (j.dir << 4) | (p << 8));
            CK(launch_zc_dyn(a, grid, s));
            t.stats.kernels++;
        }
    }

    // ---- direct path and zero-copy paths (a4, a7)
    for (int p = 0; p < P && !dynamic; p++) {
        if (lists[p].empty()) continue;
        const int g = ps[p].gpu;
        CK(make_device(g));
        const bool relay = ps[p].kind == MMA_PATH_RELAY;
        uint64_t bytes_p = 0;
        for (uint32_t i : lists[p]) { uint64_t o, l; j.extent(i, &o, &l); bytes_p += l; }
        t.stats.path_bytes[j.dir][p] += bytes_p;
        t.stats.path_chunks[j.dir][p] += lists[p].size();
        if (relay) t.stats.relay_bytes += bytes_p;
        if (mode[p] == MMA_HOP_ZC) {
            // one kernel per path: on d for the direct path, on r for a one-hop relay
            cudaStream_t s = e.dev[g].zc;
            CK((cudaError_t)use(s, g));
            CK((cudaError_t)after_upload(s, g));
            ZcLaunchArg a{};
            a.v = vstream_on(g);
            a.chunks = chunks_on(p, g);
            a.unit_bytes = e.unit_bytes;
            a.path = (uint32_t)p;
            a.log = log;
            const uint64_t upc = (j.C + e.unit_bytes - 1) / e.unit_bytes;
            const uint64_t units = a.chunks.count * upc;
            const unsigned grid = (unsigned)std::min<uint64_t>(units, (uint64_t)e.dev[g].sms * 4);
            DeviceGuard dg(g);
            KTimer kt(g, s, 0 | (j.dir << 4) | (p << 8));
            CK(launch_zc(a, grid, s));
            t.stats.kernels++;
            continue;
        }
        if (relay) continue;                         // CE relays below
        // direct CE: one DMA (or batch) per run of consecutive chunks
        cudaStream_t s = e.dev[g].direct;
        CK((cudaError_t)use(s, g));
        DeviceGuard dg(g);
        size_t a = 0;
        while (a < lists[p].size()) {
            size_t b = a + 1;
            while (b < lists[p].size() && lists[p][b] == lists[p][b - 1] + 1) b++;
            uint64_t o0, l0, o1, l1;
            j.extent(lists[p][a], &o0, &l0);
            j.extent(lists[p][b - 1], &o1, &l1);
            DmaBatch batch;
            j.pieces(o0, o1 + l1, [&](const Piece& x) { batch.add(x.dst, x.src, x.len); });
            CK((cudaError_t)batch.issue(kind, s));
            if (log) CK(cudaMemsetAsync(log + lists[p][a], p, b - a, s));
            a = b;
        }
    }

    tr.mark("direct+zc");
    // ---- CE relay rings (a5, a6 for H2D; a9 for D2H)
    std::vector<int> rp;   // relay paths using rings
    for (int p = 0; p < P; p++)
        if (!lists[p].empty() && ps[p].kind == MMA_PATH_RELAY && mode[p] == MMA_HOP_CE) rp.push_back(p);
    if (!rp.empty() && !dynamic) {
        if (!e.wait64 || !e.write64) return MMA_ERR_NO_MEMOPS;
        const uint32_t S = e.cfg.ring_slots;
        const uint64_t upc = (j.C + e.unit_bytes - 1) / e.unit_bytes;
        std::vector<Ring*> rings(P, nullptr);
        std::vector<uint64_t> g0(P, 0);
        for (int p : rp) {
            CK((cudaError_t)get_ring(j.d, j.dir, p, j.C, S, &rings[p]));
            g0[p] = rings[p]->g_next;
        }
        // relay kernels: one launch per kernel GPU covering all of its rings
        std::map<int, RelayLaunchArg> launches;
        std::map<int, unsigned> grids;
        for (int p : rp) {
            Ring* r = rings[p];
            const int kd = r->kdev;
            auto& A = launches[kd];
            if (grids.find(kd) == grids.end()) {
                memset(&A, 0, sizeof(A));
                A.v = vstream_on(kd);
                A.unit_bytes = e.unit_bytes;
                A.log = log;
                A.err = e.err;
                A.timeout_ns = e.timeout_ns;
                grids[kd] = 0;
            }
            if (A.nrings >= MMA_KMAX_RINGS) return cudaErrorInvalidValue;
            RingArg& R = A.ring[A.nrings++];
            R.stage = r->stage;
            R.slot_bytes = r->slot_bytes;
            R.seq = r->seq;
            R.credit = r->credit;
            R.cnt = r->cnt;
            R.cursor = r->cursor;
            R.g0 = g0[p];
            R.unit0 = r->unit_next;
            R.chunks = chunks_on(p, kd);
            R.S = S;
            R.path = (uint32_t)p;
            R.cta_begin = grids[kd];
            grids[kd] += (unsigned)e.cfg.relay_ctas;
            R.cta_end = grids[kd];
            r->g_next += lists[p].size();
            // every CTA of the ring claims until it draws one unit past the end, so the
            // cursor advances by the units plus one claim per CTA
            r->unit_next += (unsigned long long)lists[p].size() * upc + (unsigned)e.cfg.relay_ctas;
        }
        for (auto& kv : launches) {
            const int kd = kv.first;
            cudaStream_t s = e.dev[kd].kern;
            CK(make_device(kd));
            CK((cudaError_t)use(s, kd));
            DeviceGuard dg(kd);
            KTimer kt(kd, s, (j.dir == MMA_H2D ? 1 : 2) | (j.dir << 4) | (0xff << 8));
            CK(launch_relay(kv.second, j.dir == MMA_H2D, grids[kd], s));
            t.stats.kernels++;
        }
        // host issue of the copy-engine hops, round-robin across rings chunk by chunk
        size_t maxc = 0;
        for (int p : rp) maxc = std::max(maxc, lists[p].size());
        for (size_t c = 0; c < maxc; c++) {
            for (int p : rp) {
                if (c >= lists[p].size()) continue;
                Ring* r = rings[p];
                const uint64_t g = g0[p] + c;
                const uint32_t s = (uint32_t)(g % S);
                cudaStream_t hs = e.dev[r->relay].hop[s & 1];
                CK((cudaError_t)use(hs, r->relay));
                DeviceGuard dg(r->relay);
                char* slot = r->stage + (uint64_t)s * r->slot_bytes;
                uint64_t off, len;
                j.extent(lists[p][c], &off, &len);
                DmaBatch batch;
                if (j.dir == MMA_H2D) {
                    if (g >= S && e.wait64((CUstream)hs, (CUdeviceptr)&r->credit[s], g - S + 1, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
                        return cudaErrorUnknown;
                    j.pieces(off, off + len, [&](const Piece& x) { batch.add(slot + (x.v - off), x.src, x.len); });
                    CK((cudaError_t)batch.issue(kind, hs));
                    if ((long long)g != e.fault_drop_publish &&
                        e.write64((CUstream)hs, (CUdeviceptr)&r->seq[s], g + 1, 0) != CUDA_SUCCESS)
                        return cudaErrorUnknown;
                } else {
                    if (e.wait64((CUstream)hs, (CUdeviceptr)&r->seq[s], g + 1, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
                        return cudaErrorUnknown;
                    j.pieces(off, off + len, [&](const Piece& x) { batch.add(x.dst, slot + (x.v - off), x.len); });
                    CK((cudaError_t)batch.issue(kind, hs));
                    if (e.write64((CUstream)hs, (CUdeviceptr)&r->credit[s], g + 1, 0) != CUDA_SUCCESS) return cudaErrorUnknown;
                }
            }
        }
    }

    tr.mark("rings");
    // ---- join (a8)
    for (auto& u : used) {
        cudaEvent_t ev = join_event(u.first, u.second);
        {
            DeviceGuard g(u.second);
            CK(cudaEventRecord(ev, u.first));
        }
        DeviceGuard g(j.user_dev);
        CK(cudaStreamWaitEvent(j.user, ev, 0));
    }
    if (tab_bytes) {
        DeviceGuard g(j.user_dev);
        if (!sc.done || sc.done_dev != j.user_dev) {
            if (sc.done) cudaEventDestroy(sc.done);
            CK(cudaEventCreateWithFlags(&sc.done, cudaEventDisableTiming));
            sc.done_dev = j.user_dev;
        }
        CK(cudaEventRecord(sc.done, j.user));
        sc.pending = true;
    }
    if (e.cfg.ledger && !dynamic) {
        uint64_t lb[MMA_MAX_GPUS] = {}, lo[MMA_MAX_GPUS] = {};
        for (int p = 0; p < P; p++) {
            uint64_t bytes_p = 0;
            for (uint32_t i : lists[p]) { uint64_t o, l; j.extent(i, &o, &l); bytes_p += l; }
            lb[ps[p].gpu] += bytes_p;
            if (ps[p].kind == MMA_PATH_DIRECT) lo[ps[p].gpu] += bytes_p;
        }
        CK(ledger_add(j.dir, j.user_dev, j.user, lb, lo));
    }
    tr.mark("join");
    t.stats.issue_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    return cudaSuccess;
}

// ------------------------------------------------------------- classification ---

static int sticky()
{
    Engine& e = E();
    if (e.err && *(volatile int*)e.err) return MMA_ERR_RELAY_TIMEOUT;
    return cudaSuccess;
}

static int stream_device(cudaStream_t s, int* dev)
{
    cudaError_t e = cudaStreamGetDevice(s, dev);
    if (e != cudaSuccess) { cudaGetLastError(); return cudaGetDevice(dev); }
    return cudaSuccess;
}

// type of pointer: 0 host pinned (mapped if *mapped), 1 device (dev), 2 pageable/unknown
static int classify(const void* p, int* dev, bool* mapped)
{
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) { cudaGetLastError(); return 2; }
    if (a.type == cudaMemoryTypeDevice) { *dev = a.device; return 1; }
    if (a.type == cudaMemoryTypeHost) { *mapped = a.devicePointer != nullptr; return 0; }
    return 2;
}

static int copy_contiguous(int dir, void* dst, const void* src, size_t bytes, cudaStream_t stream)
{
    CK((cudaError_t)ensure_init());
    if (int se = sticky()) return se;
    if (bytes == 0) return cudaSuccess;
    if (!dst || !src) return cudaErrorInvalidValue;
    Engine& e = E();
    const void* dptr = (dir == MMA_H2D) ? dst : src;
    const void* hptr = (dir == MMA_H2D) ? src : dst;
    int d = -1, hd = -1;
    bool mapped = false, dummy = false;
    if (classify(dptr, &d, &dummy) != 1) return cudaErrorInvalidValue;
    const int hk = classify(hptr, &hd, &mapped);
    if (hk == 1) return cudaErrorInvalidValue;   // device -> device is not this API
    const cudaMemcpyKind kind = (dir == MMA_H2D) ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(stream, &cap);
    if (hk == 2 || cap != cudaStreamCaptureStatusNone || d >= e.ndev)
        return (int)cudaMemcpyAsync(dst, src, bytes, kind, stream);   // native (R7)
    Job j;
    j.dir = dir;
    j.d = d;
    j.user = stream;
    CK((cudaError_t)stream_device(stream, &j.user_dev));
    j.B = bytes;
    j.C = e.cfg.chunk_bytes[dir];
    j.contiguous = true;
    j.src0 = (const char*)src;
    j.dst0 = (char*)dst;
    j.mapped = mapped;
    std::lock_guard<std::mutex> g(e.mu);
    CK((cudaError_t)make_device(d));
    return run_job(j);
}

// Validate a segment table and fill the job (no engine lock held).
static int prepare_segments(int dir, const mma_segment_t* segs, size_t nsegs, int device,
                            cudaStream_t stream, Job& j)
{
    Engine& e = E();
    j.dir = dir;
    j.d = device;
    j.user = stream;
    CK((cudaError_t)stream_device(stream, &j.user_dev));
    j.C = e.cfg.chunk_bytes[dir];
    j.contiguous = false;
    j.segs = segs;
    j.nseg = nsegs;
    j.vstart.resize(nsegs + 1);
    j.vstart[0] = 0;
    // destinations must be pairwise disjoint: O(n) when they are in ascending order,
    // else a sort -- skipped when the table is byte-identical to the last one validated
    bool sorted = true;
    uintptr_t prev_end = 0;
    for (size_t k = 0; k < nsegs; k++) {
        if (!segs[k].bytes) { j.vstart[k + 1] = j.vstart[k]; continue; }
        if (!segs[k].src || !segs[k].dst) return cudaErrorInvalidValue;
        j.vstart[k + 1] = j.vstart[k] + segs[k].bytes;
        if ((uintptr_t)segs[k].dst < prev_end) sorted = false;
        prev_end = (uintptr_t)segs[k].dst + segs[k].bytes;
    }
    j.B = j.vstart[nsegs];
    if (j.B == 0) return cudaSuccess;
    if (!sorted) {
        static std::mutex mu;
        static std::vector<mma_segment_t> last_ok[2];
        std::lock_guard<std::mutex> g(mu);
        std::vector<mma_segment_t>& ok = last_ok[dir];
        if (!(ok.size() == nsegs && memcmp(ok.data(), segs, nsegs * sizeof(mma_segment_t)) == 0)) {
            std::vector<std::pair<uintptr_t, size_t>> v;
            v.reserve(nsegs);
            for (size_t k = 0; k < nsegs; k++)
                if (segs[k].bytes) v.push_back({(uintptr_t)segs[k].dst, segs[k].bytes});
            std::sort(v.begin(), v.end());
            for (size_t k = 1; k < v.size(); k++)
                if (v[k - 1].first + v[k - 1].second > v[k].first) return cudaErrorInvalidValue;
            ok.assign(segs, segs + nsegs);
        }
    }
    // classify a bounded sample of the table (first, last, evenly spaced): a pointer query
    // costs ~0.1 ms, so the sample stays small; the caller guarantees the memory kinds
    j.mapped = true;
    const size_t nsample = std::min<size_t>(nsegs, 5);
    for (size_t q = 0; q < nsample; q++) {
        size_t k = (nsample == 1) ? 0 : q * (nsegs - 1) / (nsample - 1);
        if (!segs[k].bytes) continue;
        const void* dp = (dir == MMA_H2D) ? segs[k].dst : segs[k].src;
        const void* hp = (dir == MMA_H2D) ? segs[k].src : segs[k].dst;
        int d = -1, hd = -1;
        bool m = false, dummy = false;
        if (classify(dp, &d, &dummy) != 1 || d != device) return cudaErrorInvalidValue;
        int hk = classify(hp, &hd, &m);
        if (hk == 1) return cudaErrorInvalidValue;
        if (hk == 2) j.mapped = false;   // pageable: CE only
        j.mapped = j.mapped && m;
    }
    if (nsegs == 1) {   // one segment is a contiguous copy (the kernels' nseg == 1 form)
        j.contiguous = true;
        j.src0 = (const char*)segs[0].src;
        j.dst0 = (char*)segs[0].dst;
    }
    return cudaSuccess;
}

static int copy_segments(int dir, const mma_segment_t* segs, size_t nsegs, int device, cudaStream_t stream)
{
    CK((cudaError_t)ensure_init());
    if (int se = sticky()) return se;
    Engine& e = E();
    if (nsegs == 0) return cudaSuccess;
    if (!segs) return cudaErrorInvalidValue;
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    Job j;
    CK(prepare_segments(dir, segs, nsegs, device, stream, j));
    if (j.B == 0) return cudaSuccess;
    std::lock_guard<std::mutex> g(e.mu);
    CK((cudaError_t)make_device(device));
    return run_job(j);
}

}  // namespace mma

// ====================================================================== C ABI (C7) ===

using namespace mma;

extern "C" {

int mma_default_config(mma_config_t* cfg)
{
    if (!cfg) return cudaErrorInvalidValue;
    defaults(cfg);
    apply_env(cfg);
    return cudaSuccess;
}

int mma_init(const mma_config_t* cfg)
{
    std::lock_guard<std::mutex> g(E().mu);
    return do_init(cfg);
}

int mma_finalize(void)
{
    Engine& e = E();
    std::lock_guard<std::mutex> g(e.mu);
    if (!e.inited) return cudaSuccess;
    for (int d = 0; d < e.ndev; d++) {
        if (!e.dev[d].made) continue;
        DeviceGuard dg(d);
        cudaDeviceSynchronize();
    }
    for (int d = 0; d < e.ndev; d++) {
        Target& t = e.tgt[d];
        for (int dir = 0; dir < 2; dir++)
            for (int p = 0; p < MMA_MAX_PATHS; p++) free_ring(t.rings[dir][p]);
        if (t.log) { DeviceGuard dg(d); cudaFree(t.log); }
        if (t.dyn) { DeviceGuard dg(d); cudaFree(t.dyn); }
        for (auto& sc : t.scratch) {
            for (int g2 = 0; g2 < MMA_MAX_GPUS; g2++)
                if (sc.dev[g2]) { DeviceGuard dg(g2); cudaFree(sc.dev[g2]); }
            if (sc.host) cudaFreeHost(sc.host);
            if (sc.done) cudaEventDestroy(sc.done);
        }
        t = Target();
    }
    for (auto& kv : e.join_ev) cudaEventDestroy(kv.second);
    e.join_ev.clear();
    for (auto& f : e.inflight) cudaEventDestroy(f.done);
    for (auto& f : e.free_events) cudaEventDestroy(f.second);
    e.inflight.clear();
    e.free_events.clear();
    memset(e.ledger, 0, sizeof e.ledger);
    memset(e.ledger_own, 0, sizeof e.ledger_own);
    for (int d = 0; d < e.ndev; d++) {
        DevRes& r = e.dev[d];
        if (!r.made) continue;
        DeviceGuard dg(d);
        cudaStreamDestroy(r.kern);
        cudaStreamDestroy(r.hop[0]);
        cudaStreamDestroy(r.hop[1]);
        cudaStreamDestroy(r.direct);
        cudaStreamDestroy(r.zc);
        cudaEventDestroy(r.fork);
        r = DevRes();
    }
    if (e.err) { cudaFreeHost(e.err); e.err = nullptr; }
    e.inited = false;
    return cudaSuccess;
}

int mma_memcpy_h2d(void* dst, const void* src, size_t bytes, mma_stream_t stream)
{
    return copy_contiguous(MMA_H2D, dst, src, bytes, (cudaStream_t)stream);
}

int mma_memcpy_d2h(void* dst, const void* src, size_t bytes, mma_stream_t stream)
{
    return copy_contiguous(MMA_D2H, dst, src, bytes, (cudaStream_t)stream);
}

int mma_memcpy_h2d_segments(const mma_segment_t* segs, size_t nsegs, int dst_device, mma_stream_t stream)
{
    return copy_segments(MMA_H2D, segs, nsegs, dst_device, (cudaStream_t)stream);
}

int mma_memcpy_d2h_segments(const mma_segment_t* segs, size_t nsegs, int src_device, mma_stream_t stream)
{
    return copy_segments(MMA_D2H, segs, nsegs, src_device, (cudaStream_t)stream);
}

int mma_get_paths(int device, mma_dir_t dir, int* gpus, int* kinds, uint32_t* mbps, int* modes,
                  int cap, int* npaths)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    if ((dir != MMA_H2D && dir != MMA_D2H) || !npaths) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> g(e.mu);
    make_paths(device);
    auto& ps = e.tgt[device].paths[dir];
    *npaths = (int)ps.size();
    for (int i = 0; i < (int)ps.size() && i < cap; i++) {
        if (gpus) gpus[i] = ps[i].gpu;
        if (kinds) kinds[i] = ps[i].kind;
        if (mbps) mbps[i] = ps[i].mbps;
        if (modes) modes[i] = ps[i].mode;
    }
    return cudaSuccess;
}

int mma_set_plan_mode(int mode)
{
    CK((cudaError_t)ensure_init());
    if (mode < PLAN_CONTIGUOUS || mode > PLAN_DYNAMIC) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> g(E().mu);
    E().cfg.plan_mode = mode;
    return cudaSuccess;
}

int mma_get_segment_tuning(int device, mma_dir_t dir, uint32_t* mbps, int* modes, int cap, int* npaths)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    if ((dir != MMA_H2D && dir != MMA_D2H) || !npaths) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> g(e.mu);
    make_paths(device);
    auto& ps = e.tgt[device].paths[dir];
    *npaths = (int)ps.size();
    for (int i = 0; i < (int)ps.size() && i < cap; i++) {
        if (mbps) mbps[i] = ps[i].seg_mbps;
        if (modes) modes[i] = ps[i].seg_mode;
    }
    return cudaSuccess;
}

int mma_set_bandwidth(int device, mma_dir_t dir, const uint32_t* mbps, int npaths)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    if ((dir != MMA_H2D && dir != MMA_D2H) || !mbps) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> g(e.mu);
    make_paths(device);
    auto& ps = e.tgt[device].paths[dir];
    if (npaths != (int)ps.size()) return cudaErrorInvalidValue;
    bool any = false;
    for (int i = 0; i < npaths; i++) any |= mbps[i] > 0;
    if (!any) return cudaErrorInvalidValue;
    for (int i = 0; i < npaths; i++) { ps[i].mbps = mbps[i]; ps[i].seg_mbps = 0; }
    return cudaSuccess;
}

int mma_set_path_modes(int device, mma_dir_t dir, const int* modes, int npaths)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    if ((dir != MMA_H2D && dir != MMA_D2H) || !modes) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> g(e.mu);
    make_paths(device);
    auto& ps = e.tgt[device].paths[dir];
    if (npaths != (int)ps.size()) return cudaErrorInvalidValue;
    for (int i = 0; i < npaths; i++)
        if (modes[i] < MMA_HOP_AUTO || modes[i] > MMA_HOP_ZC) return cudaErrorInvalidValue;
    for (int i = 0; i < npaths; i++) { ps[i].mode = modes[i]; ps[i].seg_mode = -1; }
    return cudaSuccess;
}

int mma_get_plan(int device, mma_dir_t dir, size_t bytes, uint8_t* path_of_chunk, size_t cap,
                 size_t* nchunks, int* fallback)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    if ((dir != MMA_H2D && dir != MMA_D2H) || !nchunks) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> g(e.mu);
    make_paths(device);
    auto& ps = e.tgt[device].paths[dir];
    std::vector<PlanPath> pp;
    for (auto& p : ps) pp.push_back(PlanPath{p.kind == MMA_PATH_DIRECT, p.mbps, 0});
    ledger_inputs(device, dir, ps, pp);
    Plan plan;
    if (make_plan(pp.data(), (int)pp.size(), bytes, e.cfg.chunk_bytes[dir], e.cfg.fallback_bytes[dir],
                  e.cfg.plan_mode == PLAN_DYNAMIC ? PLAN_CONTIGUOUS : e.cfg.plan_mode, plan))
        return cudaErrorInvalidValue;
    *nchunks = plan.n;
    if (fallback) *fallback = plan.fallback;
    if (path_of_chunk) {
        if (cap < plan.n) return cudaErrorInvalidValue;
        memcpy(path_of_chunk, plan.path.data(), plan.n);
    }
    return cudaSuccess;
}

int mma_plan_chunks(const uint32_t* mbps, const int* kinds, const uint64_t* backlog, int npaths,
                    uint64_t bytes, uint64_t chunk_bytes, uint64_t thr, int mode,
                    uint8_t* path_of_chunk, size_t cap, size_t* nchunks, int* fallback)
{
    if (!mbps || !kinds || !nchunks || npaths < 1 || npaths > 255) return cudaErrorInvalidValue;
    std::vector<PlanPath> pp(npaths);
    for (int p = 0; p < npaths; p++) {
        if (kinds[p] != MMA_PATH_DIRECT && kinds[p] != MMA_PATH_RELAY) return cudaErrorInvalidValue;
        pp[p] = PlanPath{kinds[p] == MMA_PATH_DIRECT, mbps[p], backlog ? backlog[p] : 0};
    }
    Plan plan;
    if (make_plan(pp.data(), npaths, bytes, chunk_bytes, thr, mode, plan)) return cudaErrorInvalidValue;
    *nchunks = plan.n;
    if (fallback) *fallback = plan.fallback;
    if (path_of_chunk) {
        if (cap < plan.n) return cudaErrorInvalidValue;
        memcpy(path_of_chunk, plan.path.data(), plan.n);
    }
    return cudaSuccess;
}

// Measure every path alone in each hop mode on the transfer `proto` describes and keep,
// per path, the faster mode and its rate (integer MB/s, reading R17: llround). Runs the
// copy (1 + reps) times per (path, mode); the best of `reps` timed runs counts. The host
// thread that enqueues a call is one resource shared by all P paths of a multipath call,
// so a mode's rate is min(device rate, host-issue rate / P): a copy-engine path that needs
// one descriptor per 32 KiB segment (~0.6 us each) cannot feed 8 links from one thread
// (DESIGN.md §5.3).
static int tune_paths(Job proto, int reps, std::vector<uint32_t>& mbps, std::vector<int>& modes)
{
    Engine& e = E();
    auto& ps = e.tgt[proto.d].paths[proto.dir];
    const int P = (int)ps.size();
    mbps.assign(P, 0);
    modes.assign(P, MMA_HOP_CE);
    std::vector<uint32_t> bw(P);
    std::vector<int> md(P, MMA_HOP_CE);
    cudaEvent_t a = nullptr, b = nullptr;
    {
        DeviceGuard g(proto.user_dev);
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
    }
    int rc = cudaSuccess;
    for (int p = 0; p < P && rc == cudaSuccess; p++) {
        float best_rate = 0.f;
        for (int m : {MMA_HOP_CE, MMA_HOP_ZC}) {
            if (m == MMA_HOP_ZC && !proto.mapped) continue;
            for (int q = 0; q < P; q++) bw[q] = (q == p) ? 1 : 0;
            md[p] = m;
            float best = 1e30f, best_issue = 1e30f;
            for (int rep = 0; rep <= reps && rc == cudaSuccess; rep++) {
                Job j = proto;
                j.bw_override = bw.data();
                j.mode_override = md.data();
                j.no_small_fallback = true;
                DeviceGuard g(j.user_dev);
                cudaEventRecord(a, j.user);
                const auto h0 = std::chrono::steady_clock::now();
                rc = run_job(j);
                const float issue_ms = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - h0).count();
                cudaEventRecord(b, j.user);
                if (cudaEventSynchronize(b) != cudaSuccess) rc = cudaErrorUnknown;
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                if (rep > 0 && ms > 0) {                             // rep 0 warms up
                    best = std::min(best, ms);
                    best_issue = std::min(best_issue, issue_ms);
                }
            }
            const float eff_ms = std::max(best, best_issue * (float)P);
            const float rate = best < 1e29f ? (float)((double)proto.B / (eff_ms * 1e-3) / 1e6) : 0.f;
            if (rate > best_rate) {
                best_rate = rate;
                modes[p] = m;
                mbps[p] = (uint32_t)llround(rate);
            }
        }
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (rc == cudaSuccess && sticky()) rc = sticky();
    return rc;
}

int mma_calibrate(int device, mma_dir_t dir, size_t bytes)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    if ((dir != MMA_H2D && dir != MMA_D2H) || bytes == 0) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> g(e.mu);
    CK(make_device(device));
    make_paths(device);
    DeviceGuard dg(device);
    char* hbuf = nullptr;
    char* dbuf = nullptr;
    cudaStream_t s = nullptr;
    CK(cudaHostAlloc((void**)&hbuf, bytes, cudaHostAllocPortable | cudaHostAllocMapped));
    CK(cudaMalloc((void**)&dbuf, bytes));
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    Job j;
    j.dir = dir;
    j.d = device;
    j.user = s;
    j.user_dev = device;
    j.B = bytes;
    j.C = e.cfg.chunk_bytes[dir];
    j.src0 = dir == MMA_H2D ? hbuf : dbuf;
    j.dst0 = dir == MMA_H2D ? dbuf : hbuf;
    j.mapped = true;
    std::vector<uint32_t> mbps;
    std::vector<int> modes;
    int rc = tune_paths(j, 3, mbps, modes);
    if (rc == cudaSuccess) {
        auto& ps = e.tgt[device].paths[dir];
        for (size_t p = 0; p < ps.size(); p++)
            if (mbps[p]) { ps[p].mbps = mbps[p]; ps[p].mode = modes[p]; }
    }
    cudaStreamDestroy(s);
    cudaFree(dbuf);
    cudaFreeHost(hbuf);
    return rc;
}

int mma_tune_segments(const mma_segment_t* segs, size_t nsegs, int device, mma_dir_t dir,
                      mma_stream_t stream, int reps)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    if ((dir != MMA_H2D && dir != MMA_D2H) || !segs || nsegs == 0 || reps < 1) return cudaErrorInvalidValue;
    Job j;
    CK(prepare_segments(dir, segs, nsegs, device, (cudaStream_t)stream, j));
    if (j.B == 0) return cudaSuccess;
    std::lock_guard<std::mutex> g(e.mu);
    CK(make_device(device));
    make_paths(device);
    std::vector<uint32_t> mbps;
    std::vector<int> modes;
    int rc = tune_paths(j, reps, mbps, modes);
    if (rc == cudaSuccess) {
        auto& ps = e.tgt[device].paths[dir];
        for (size_t p = 0; p < ps.size(); p++)
            if (mbps[p]) { ps[p].seg_mbps = mbps[p]; ps[p].seg_mode = modes[p]; }
    }
    return rc;
}

int mma_get_delivery_log(int device, uint8_t* path_of_chunk, size_t cap, size_t* nchunks)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    if (!nchunks) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> g(e.mu);
    Target& t = e.tgt[device];
    *nchunks = t.log_n;
    if (!t.log_n || !path_of_chunk) return cudaSuccess;
    if (cap < t.log_n) return cudaErrorInvalidValue;
    DeviceGuard dg(device);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(path_of_chunk, t.log, t.log_n, cudaMemcpyDeviceToHost));
    return cudaSuccess;
}

int mma_host_alloc(void** ptr, size_t bytes, unsigned flags)
{
    CK((cudaError_t)ensure_init());
    (void)flags;
    return host_alloc(ptr, bytes, E().cfg.numa_mode, 0);
}

int mma_host_free(void* ptr) { return host_free(ptr); }

int mma_get_stats(int device, mma_stats_t* out)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    if (!out) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> g(e.mu);
    *out = e.tgt[device].stats;
    return cudaSuccess;
}

int mma_reset_stats(int device)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> g(e.mu);
    e.tgt[device].stats = mma_stats_t{};
    return cudaSuccess;
}

int mma_set_kernel_timing(int on)
{
    std::lock_guard<std::mutex> g(E().mu);
    g_ktime = on != 0;
    return cudaSuccess;
}

int mma_kernel_times(float* ms, int* kinds, size_t cap, size_t* n)
{
    if (!n) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> g(E().mu);
    size_t k = 0;
    int rc = cudaSuccess;
    for (auto& r : g_kpending) {
        DeviceGuard dg(r.dev);
        float t = 0.f;
        if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&t, r.a, r.b) != cudaSuccess)
            rc = cudaErrorUnknown;
        if (k < cap) {
            if (ms) ms[k] = t;
            if (kinds) kinds[k] = r.kind;
        }
        k++;
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    g_kpending.clear();
    *n = k;
    return rc;
}

int mma_get_dynamic_counts(int device, uint64_t* chunks, int cap, int* npaths)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    if (!npaths) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> g(e.mu);
    Target& t = e.tgt[device];
    *npaths = t.last_dyn ? t.last_dyn_paths : 0;
    if (!t.last_dyn || !chunks) return cudaSuccess;
    unsigned long long c[MMA_KMAX_RINGS] = {};
    DeviceGuard dg(device);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(c, t.last_dyn + 1, sizeof c, cudaMemcpyDeviceToHost));
    for (int p = 0; p < t.last_dyn_paths && p < cap; p++) chunks[p] = c[p];
    return cudaSuccess;
}

int mma_get_last_error(void)
{
    if (!E().inited) return cudaSuccess;
    return sticky();
}

const char* mma_error_string(int err)
{
    if (err == MMA_ERR_RELAY_TIMEOUT) return "mma: relay kernel spin timed out (sticky; mma_finalize to reset)";
    if (err == MMA_ERR_NO_MEMOPS) return "mma: CUDA stream memory operations unavailable";
    return cudaGetErrorString((cudaError_t)err);
}

int mma_fill_pattern(void* ptr, size_t bytes, uint64_t seed, uint64_t offset, mma_stream_t s)
{
    if (bytes && !ptr) return cudaErrorInvalidValue;
    return (int)launch_fill(ptr, bytes, seed, offset, (cudaStream_t)s);
}

int mma_verify_pattern(const void* ptr, size_t bytes, uint64_t seed, uint64_t offset,
                       uint64_t* mismatches, mma_stream_t s)
{
    if ((bytes && !ptr) || !mismatches) return cudaErrorInvalidValue;
    return (int)launch_verify(ptr, bytes, seed, offset, mismatches, (cudaStream_t)s);
}

int mma_verify_segments(void* const* dst, const uint64_t* offset, const uint64_t* bytes,
                        size_t nsegs, uint64_t seed, uint64_t* mismatches, mma_stream_t s)
{
    if (!mismatches || (nsegs && (!dst || !offset || !bytes))) return cudaErrorInvalidValue;
    if (!nsegs) return cudaSuccess;
    uint64_t* tab = nullptr;
    CK(cudaMallocAsync((void**)&tab, 3 * nsegs * 8, (cudaStream_t)s));
    CK(cudaMemcpyAsync(tab, dst, nsegs * 8, cudaMemcpyHostToDevice, (cudaStream_t)s));
    CK(cudaMemcpyAsync(tab + nsegs, offset, nsegs * 8, cudaMemcpyHostToDevice, (cudaStream_t)s));
    CK(cudaMemcpyAsync(tab + 2 * nsegs, bytes, nsegs * 8, cudaMemcpyHostToDevice, (cudaStream_t)s));
    CK(launch_verify_segments(tab, tab + nsegs, tab + 2 * nsegs, nsegs, seed, mismatches, (cudaStream_t)s));
    CK(cudaFreeAsync(tab, (cudaStream_t)s));
    return cudaSuccess;
}

// Raise the hardware queue count before the first CUDA context exists, so the engine's
// streams do not alias one queue (SURVEY §7 hard part 4).
__attribute__((constructor)) static void mma_preinit(void)
{
    setenv("CUDA_DEVICE_MAX_CONNECTIONS", "32", 0);
}

}  // extern "C"
