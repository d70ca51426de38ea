// plane.cpp — the multipath data plane (C6): configuration, devices, rings, ledger, enqueue.
//
// One user copy of B bytes between pinned host memory and GPU d becomes n chunks; each
// chunk travels over exactly one path:
//   direct   d's own PCIe link: copy-engine DMA ("a single H2D transfer operation")
//            or SM zero-copy (north_star (d));
//   relay r  r's PCIe link into r's HBM staging ring, then NVLink r -> d, pulled by the
//            relay kernel on d or pushed by a peer DMA on r's own stream (MMA_HOP_CE_P2P)
//            ("an H2D operation and a P2P operation ... with a dependency"; dual
//            pipeline generalised to S slots); D2H mirrors it. In zero-copy mode a relay is
//            one hop: a kernel on r reads host memory over r's PCIe and stores into d's HBM
//            over NVLink.
// A call on a stream being captured is recorded as a replayable graph (class Call, capture
// mode); scattered tables may be regrouped by host NUMA node (R23) and moved in host-address
// order inside a path (R22).
// The paper's Dummy Task + callback + spin kernel (§3.3, §4) is
// replaced by GPU-ordered fork/join: an event recorded on the user stream gates every path
// stream and every path stream's completion event gates the user stream, so the copy is
// ordered exactly like cudaMemcpyAsync with no CPU thread in the per-chunk loop (the
// paper's 2 threads per GPU, cost 822% CPU at 8 GPUs). Per relay chunk
// the host enqueues: wait(credit) -> DMA -> write(seq) on the relay's stream (cuda.h stream
// memory operations); the relay kernel polls seq and releases credit on the GPU.
#include <nvtx3/nvToolsExt.h>   // header-only: ranges are free unless a tool (nsys) attaches

#include <memory>

#include "plane.h"

namespace mma {

Engine& E()
{
    static Engine* e = new Engine();   // never destroyed: safe at process exit
    return *e;
}

int phys_dev(int g)
{
    return (g >= 0 && g < MMA_MAX_GPUS) ? E().phys[g] : g;
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

// ------------------------------------------------------------------- configuration ---

void apply_env(mma_config_t* c)
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
    c->claim_bytes = env_size("MMA_CLAIM_BYTES", c->claim_bytes);
    c->zc_ctas = env_int("MMA_ZC_CTAS", c->zc_ctas);
    c->calib_rounds = env_int("MMA_CALIB_ROUNDS", c->calib_rounds);
    c->host_order = env_int("MMA_HOST_ORDER", c->host_order);
    c->numa_plan = env_int("MMA_NUMA_PLAN", c->numa_plan);
    c->background_policy = env_int("MMA_BACKGROUND", c->background_policy);
    c->yield_pct = (unsigned)env_int("MMA_YIELD_PCT", (int)c->yield_pct);
    c->relay_prefer = env_int("MMA_RELAY_PREFER", c->relay_prefer);
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

void defaults(mma_config_t* c)
{
    memset(c, 0, sizeof(*c));
    c->chunk_bytes[0] = c->chunk_bytes[1] = kDefaultChunk;
    c->ring_slots = 0;   // auto: ring_slots_for(C)
    // Fallback threshold: "between two and five chunks" (§5.1.3); 2 chunks until the
    // B200 break-even sweep replaces it.
    c->fallback_bytes[0] = c->fallback_bytes[1] = 2 * kDefaultChunk;
    c->plan_mode = PLAN_CONTIGUOUS;
    c->hop_mode[0] = c->hop_mode[1] = MMA_HOP_AUTO;
    c->relay_ctas = kDefaultRelayCtas;
    c->ledger = 1;
    c->claim_bytes = 256u << 10;
    c->zc_ctas = kDefaultZcCtas;
    c->calib_rounds = 2;
    c->host_order = 1;
    c->numa_plan = 1;
    c->background_policy = 0;
    c->yield_pct = 150;
}

int validate_cfg(const mma_config_t& c)
{
    for (int d = 0; d < 2; d++)
        if (c.chunk_bytes[d] == 0 || c.chunk_bytes[d] % 4096) return cudaErrorInvalidValue;
    if (c.ring_slots > 64) return cudaErrorInvalidValue;
    if (c.npaths < 0 || c.npaths > MMA_MAX_PATHS) return cudaErrorInvalidValue;
    if (c.loopback_relays < 0 || c.loopback_relays > 8) return cudaErrorInvalidValue;
    if (c.plan_mode < PLAN_CONTIGUOUS || c.plan_mode > PLAN_DYNAMIC) return cudaErrorInvalidValue;
    for (int d = 0; d < 2; d++)
        if (c.hop_mode[d] < MMA_HOP_AUTO || c.hop_mode[d] > MMA_HOP_PUSH) return cudaErrorInvalidValue;
    if (c.relay_ctas < 1 || c.relay_ctas > 64) return cudaErrorInvalidValue;
    if (c.claim_bytes % 16) return cudaErrorInvalidValue;
    if (c.zc_ctas < 0 || c.zc_ctas > 4096) return cudaErrorInvalidValue;
    if (c.calib_rounds < 0 || c.calib_rounds > 16) return cudaErrorInvalidValue;
    if (c.host_order < 0 || c.host_order > 2) return cudaErrorInvalidValue;
    if (c.numa_plan < 0 || c.numa_plan > 1) return cudaErrorInvalidValue;
    if (c.background_policy < 0 || c.background_policy > 1 || c.yield_pct > 100000) return cudaErrorInvalidValue;
    if (c.relay_prefer < 0 || c.relay_prefer > MMA_MAX_GPUS) return cudaErrorInvalidValue;
    return cudaSuccess;
}

// Permutation that orders n keys ascending (stable): LSD radix sort on (key - min) >> 12
// (4 KiB pages) in 11-bit digits, std::sort below 4096 keys. O(n) per digit; the digit count
// follows the key range (a few passes for one host pool).
void order_by_key(const uint64_t* key, size_t n, std::vector<uint32_t>& perm)
{
    perm.resize(n);
    for (size_t i = 0; i < n; i++) perm[i] = (uint32_t)i;
    if (n < 2) return;
    if (n < 4096) {
        std::stable_sort(perm.begin(), perm.end(), [&](uint32_t a, uint32_t b) { return key[a] < key[b]; });
        return;
    }
    uint64_t lo = key[0], hi = key[0];
    for (size_t i = 1; i < n; i++) {
        lo = std::min(lo, key[i]);
        hi = std::max(hi, key[i]);
    }
    const uint64_t range = (hi - lo) >> 12;
    std::vector<uint32_t> tmp(n);
    std::vector<size_t> cnt(1u << 11);
    for (int shift = 0; shift < 64 && (range >> shift); shift += 11) {
        std::fill(cnt.begin(), cnt.end(), 0);
        for (size_t i = 0; i < n; i++) cnt[(((key[perm[i]] - lo) >> 12) >> shift) & 2047]++;
        size_t sum = 0;
        for (auto& c : cnt) { const size_t t = c; c = sum; sum += t; }
        for (size_t i = 0; i < n; i++) tmp[cnt[(((key[perm[i]] - lo) >> 12) >> shift) & 2047]++] = perm[i];
        perm.swap(tmp);
    }
    // within one 4 KiB page keep ascending addresses too (pieces of a page are few)
    for (size_t a = 0; a < n;) {
        size_t b = a + 1;
        while (b < n && ((key[perm[b]] - lo) >> 12) == ((key[perm[a]] - lo) >> 12)) b++;
        if (b - a > 1)
            std::stable_sort(perm.begin() + a, perm.begin() + b, [&](uint32_t x, uint32_t y) { return key[x] < key[y]; });
        a = b;
    }
}

// Ring depth S: cfg.ring_slots, or (0, the default) a constant 32 MiB of staging per ring,
// 4..32 slots. A ring pays per-wave and per-group costs (a kernel launch per wave of S chunks,
// a DMA and a batched flag operation per group), so small chunks want deep rings: one loopback
// kernel ring carries 0.79 / 0.85 / 0.89 of the native copy at C = 1 MiB and S = 8 / 16 / 32,
// and 0.93 at 8 MiB with S = 4 (profiles/r02_sweep_ring_depth.jsonl).
uint32_t ring_slots_for(uint64_t C)
{
    const Engine& e = E();
    if (e.cfg.ring_slots) return e.cfg.ring_slots;
    const uint64_t s = kRingBytes / std::max<uint64_t>(C, 1);
    return (uint32_t)std::min<uint64_t>(32, std::max<uint64_t>(4, s));
}

uint64_t zc_grid(int d, int dir)
{
    const Engine& e = E();
    const uint64_t cap = (uint64_t)e.dev[d].sms * 4;
    const int per_dir = (dir == MMA_H2D || dir == MMA_D2H) ? e.zc_ctas_dir[dir] : 0;
    const uint64_t want = per_dir > 0 ? (uint64_t)per_dir
                        : e.cfg.zc_ctas > 0 ? (uint64_t)e.cfg.zc_ctas : (uint64_t)kDefaultZcCtas;
    return std::min(want, cap);
}

static cudaEvent_t join_event(cudaStream_t s, int dev);

// test hook (MMA_DENY_PEER="a,b;c,d"): cudaDeviceEnablePeerAccess is taken to fail for these
// ordered pairs, so the refused-peer branch below runs on a box where every pair works
static bool peer_denied(int a, int b)
{
    const char* s = getenv("MMA_DENY_PEER");
    if (!s) return false;
    for (const char* q = s; *q;) {
        char* end;
        const long x = strtol(q, &end, 10);
        if (end == q || *end != ',') break;
        const long y = strtol(end + 1, &end, 10);
        if (x == a && y == b) return true;
        while (*end && *end != ';') end++;
        q = *end ? end + 1 : end;
    }
    return false;
}

// Streams, peer access and flags for device d (lazily, once).
int make_device(int d)
{
    Engine& e = E();
    DevRes& r = e.dev[d];
    if (r.made) return cudaSuccess;
    DeviceGuard g(d);
    int lo, hi;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    // Ten streams (five per direction) created back to back so they land on distinct
    // hardware queues: a spinning relay kernel must never sit in front of the DMAs it waits for.
    for (Lanes& l : r.lane) {
        CK(cudaStreamCreateWithPriority(&l.kern, cudaStreamNonBlocking, hi));
        CK(cudaStreamCreateWithPriority(&l.hop[0], cudaStreamNonBlocking, hi));
        CK(cudaStreamCreateWithPriority(&l.hop[1], cudaStreamNonBlocking, hi));
        CK(cudaStreamCreateWithPriority(&l.direct, cudaStreamNonBlocking, hi));
        CK(cudaStreamCreateWithPriority(&l.zc, cudaStreamNonBlocking, hi));
    }
    for (Lanes& l : r.cap_lane) {
        CK(cudaStreamCreateWithPriority(&l.kern, cudaStreamNonBlocking, hi));
        CK(cudaStreamCreateWithPriority(&l.hop[0], cudaStreamNonBlocking, hi));
        CK(cudaStreamCreateWithPriority(&l.hop[1], cudaStreamNonBlocking, hi));
        CK(cudaStreamCreateWithPriority(&l.direct, cudaStreamNonBlocking, hi));
        CK(cudaStreamCreateWithPriority(&l.zc, cudaStreamNonBlocking, hi));
    }
    CK(cudaEventCreateWithFlags(&r.cap_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&r.cap_ev, cudaEventDisableTiming));
    for (auto& gd : r.gate_ev)
        for (cudaEvent_t& ev : gd) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CK(cudaStreamCreateWithFlags(&r.setup, cudaStreamNonBlocking));
    // join events exist before any call: a captured call may not create one
    for (Lanes* ls : {r.lane, r.cap_lane})
        for (int k = 0; k < 2; k++)
            for (cudaStream_t s : {ls[k].kern, ls[k].hop[0], ls[k].hop[1], ls[k].direct, ls[k].zc})
                if (!join_event(s, d)) return cudaErrorMemoryAllocation;
    CK(cudaDeviceGetAttribute(&r.sms, cudaDevAttrMultiProcessorCount, phys_dev(d)));
    for (int p = 0; p < e.ndev; p++) {
        if (p == d || !e.p2p[d][p]) continue;
        cudaError_t pe = peer_denied(d, p)                  ? cudaErrorPeerAccessUnsupported
                         : phys_dev(p) == phys_dev(d) ? cudaSuccess   // virtual GPUs of one device
                                                      : cudaDeviceEnablePeerAccess(phys_dev(p), 0);
        if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else if (pe != cudaSuccess) { cudaGetLastError(); e.p2p[d][p] = false; }   // never a path
    }
    r.made = true;
    return cudaSuccess;
}

int do_init(const mma_config_t* cfg)
{
    Engine& e = E();
    mma_config_t c;
    if (cfg) c = *cfg;
    else { defaults(&c); apply_env(&c); }
    CK((cudaError_t)validate_cfg(c));
    if (!e.inited) {
        CK(cudaGetDeviceCount(&e.ndev));
        if (e.ndev > MMA_MAX_GPUS) e.ndev = MMA_MAX_GPUS;
        const int nphys = e.ndev;
        const int nv = env_int("MMA_VGPUS", 0);
        e.virt = nphys > 0 && nv > nphys;
        if (e.virt) e.ndev = std::min(nv, MMA_MAX_GPUS);
        for (int g = 0; g < MMA_MAX_GPUS; g++) e.phys[g] = (e.virt && g >= nphys) ? g % nphys : g;
        for (int a = 0; a < e.ndev; a++)
            for (int b = 0; b < e.ndev; b++) {
                int ok = 0, at = 0;
                const int pa = e.phys[a], pb = e.phys[b];
                if (a != b && pa == pb) ok = at = 1;   // two indices of one device (MMA_VGPUS)
                else if (a != b) {
                    cudaDeviceCanAccessPeer(&ok, pa, pb);
                    if (cudaDeviceGetP2PAttribute(&at, cudaDevP2PAttrNativeAtomicSupported, pa, pb) != cudaSuccess) {
                        cudaGetLastError();
                        at = 0;
                    }
                }
                e.p2p[a][b] = ok != 0;
                // a kernel on a that updates flags / cursors in b's memory needs native atomics
                // over the link (system-scope atomics to a peer); MMA_NO_P2P_ATOMICS: test hook
                e.p2p_atomic[a][b] = a == b || (at != 0 && !getenv("MMA_NO_P2P_ATOMICS"));
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
        fn = nullptr;
        if (cudaGetDriverEntryPointByVersion("cuStreamBatchMemOp", &fn, 12000, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess && !getenv("MMA_NO_BATCH_MEMOP"))
            e.batch_memop = (PFN_batch_memop)fn;
        CK(cudaHostAlloc((void**)&e.err, sizeof(int) * 16, cudaHostAllocPortable | cudaHostAllocMapped));
        memset(e.err, 0, sizeof(int) * 16);
        e.arena_cap = env_size("MMA_GRAPH_ARENA", 16u << 20);
        e.arena_used = 0;
        if (e.arena_cap) CK(cudaHostAlloc((void**)&e.arena, e.arena_cap, cudaHostAllocPortable));
        e.timeout_ns = (uint64_t)env_size("MMA_SPIN_TIMEOUT_MS", 20000) * 1000000ull;
        e.unit_bytes = (uint32_t)env_size("MMA_UNIT_BYTES", kDefaultUnit);
        e.group_bytes = env_size("MMA_GROUP_BYTES", kDefaultGroupBytes);
        e.hop_lanes = env_int("MMA_HOP_LANES", 2) == 1 ? 1 : 2;
        e.relay_bulk = env_int("MMA_RELAY_BULK", 0) != 0;
        e.zc_bulk = env_int("MMA_ZC_BULK", 1) != 0;
        e.zc_ctas_dir[MMA_H2D] = std::max(0, env_int("MMA_ZC_CTAS_H2D", 0));
        e.zc_ctas_dir[MMA_D2H] = std::max(0, env_int("MMA_ZC_CTAS_D2H", 0));
        if (const char* u = getenv("MMA_UPLOAD")) e.upload_by_kernel = strcmp(u, "ce") != 0;
        const char* f = getenv("MMA_FAULT_DROP_PUBLISH");
        e.fault_drop_publish = f ? atoll(f) : -1;
        e.fault_fail_rings = getenv("MMA_FAULT_FAIL_RINGS") != nullptr;
        const char* fh = getenv("MMA_FAULT_FAIL_HOP");
        e.fault_fail_hop = fh ? atoll(fh) : -1;
        e.hops_issued = 0;
        e.fault_misroute = getenv("MMA_FAULT_MISROUTE") != nullptr;
        if (e.unit_bytes < 4096) e.unit_bytes = 4096;
    }
    e.cfg = c;
    for (int d = 0; d < e.ndev; d++) e.tgt[d].paths_made = false;   // re-derive path sets
    e.inited = true;
    if (const char* cal = getenv("MMA_CALIB")) load_calibration_locked(cal, nullptr);
    if (const char* led = getenv("MMA_LEDGER_SHM")) mma_ledger_attach(led);
    return cudaSuccess;
}

int ensure_init()
{
    Engine& e = E();
    if (e.inited) return cudaSuccess;
    std::lock_guard<std::mutex> g(e.mu);
    if (e.inited) return cudaSuccess;
    return do_init(nullptr);
}

// Path set of target d: path 0 = d's own link, then relay GPUs in calibration order, then
// loopback relays (reading R11).
void make_paths(int d)
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
        // peer access is enabled (make_device) before a relay is admitted: a pair whose
        // cudaDeviceEnablePeerAccess failed is marked non-P2P there and never becomes a path
        const bool dev_ok = make_device(d) == cudaSuccess;
        for (int g : cand) {
            if (g < 0 || g >= e.ndev || g == d || !dev_ok || !e.p2p[d][g] || !e.p2p[g][d]) continue;
            if (make_device(g) != cudaSuccess || !e.p2p[d][g] || !e.p2p[g][d]) continue;
            bool dup = false;
            for (auto& p : ps) dup |= (p.gpu == g);
            if (!dup && ps.size() < MMA_MAX_PATHS) ps.push_back({g, MMA_PATH_RELAY, kDefaultMbps, e.cfg.hop_mode[dir]});
        }
        for (int k = 0; k < e.cfg.loopback_relays && ps.size() < MMA_MAX_PATHS; k++)
            ps.push_back({d, MMA_PATH_RELAY, kDefaultMbps, e.cfg.hop_mode[dir]});
        // NUMA (reading R23): each path's GPU node; relays on the target's node first (stable),
        // so the first group of a node-grouped table meets the target's own link
        for (auto& p : ps) p.node = gpu_numa_node(p.gpu);
        if (e.cfg.numa_plan) {
            const int nd = ps[0].node;
            std::stable_sort(ps.begin() + 1, ps.end(), [nd](const PathState& a, const PathState& b) {
                return (a.node != nd) < (b.node != nd);
            });
        }
        if (const char* fk = getenv("MMA_FAKE_PATH_NODES")) {   // test hook: node per path index
            size_t i = 0;
            for (const char* q = fk; *q && i < ps.size(); i++) {
                char* end;
                const long x = strtol(q, &end, 10);
                if (end == q) break;
                ps[i].node = (int)x;
                q = (*end == ',') ? end + 1 : end;
            }
        }
        // MMA_BW="mbps0,mbps1,...": a pinned vector for parity runs (SURVEY §7 hard part 7),
        // applied when it names exactly this set's paths
        if (const char* bwenv = getenv("MMA_BW")) {
            std::vector<uint32_t> v;
            for (const char* q = bwenv; *q;) {
                char* end;
                const unsigned long x = strtoul(q, &end, 10);
                if (end == q) break;
                v.push_back((uint32_t)x);
                q = (*end == ',') ? end + 1 : end;
            }
            if (v.size() == ps.size())
                for (size_t i = 0; i < ps.size(); i++) ps[i].mbps = v[i];
        }
        // keep a previously pinned vector when the set is unchanged
        if (t.paths[dir].size() == ps.size()) {
            bool same = true;
            for (size_t i = 0; i < ps.size(); i++) same &= ps[i].gpu == t.paths[dir][i].gpu && ps[i].kind == t.paths[dir][i].kind;
            if (same)
                for (size_t i = 0; i < ps.size(); i++) {   // measured / pinned values survive
                    ps[i].mbps = t.paths[dir][i].mbps;
                    ps[i].seg_mbps = t.paths[dir][i].seg_mbps;
                    ps[i].seg_mode = t.paths[dir][i].seg_mode;
                    for (int k = 0; k < 2; k++) {
                        ps[i].solo_mbps[k] = t.paths[dir][i].solo_mbps[k];
                        ps[i].conc_mbps[k] = t.paths[dir][i].conc_mbps[k];
                    }
                }
        }
        t.paths[dir] = ps;
    }
    t.paths_made = true;
}

// --------------------------------------------------------------------- the rings ---

void free_ring(Ring& r)
{
    if (!r.made) return;
    { DeviceGuard g(r.relay); cudaFree(r.stage); cudaFree(r.seq); }
    { DeviceGuard g(r.kdev); cudaFree(r.cnt); }
    r = Ring();
}

// The GPU that runs a kernel ring's relay kernel: the pull form on the side that receives
// over NVLink (H2D: the target; D2H: the relay), the push form (MMA_HOP_PUSH) on the side
// that sends (H2D: the relay; D2H: the target).
int ring_kdev(int d, int dir, int relay, int mode)
{
    const bool push = mode == MMA_HOP_PUSH;
    return (dir == MMA_H2D) != push ? d : relay;
}

// Ring of path p of target d in direction dir: S slots of C bytes on the relay.
int get_ring(int d, int dir, int p, uint64_t C, uint32_t S, bool push, Ring** out)
{
    Engine& e = E();
    Ring& r = e.tgt[d].rings[dir][p];
    const int relay = e.tgt[d].paths[dir][p].gpu;
    const int kdev = ring_kdev(d, dir, relay, push ? MMA_HOP_PUSH : MMA_HOP_CE);
    if (r.made && (r.broken || r.slot_bytes < C || r.S != S || r.relay != relay || r.kdev != kdev)) {
        // tunables changed, or a failed call left the ring out of step: drain everything
        // that may still use the old ring
        { DeviceGuard g(r.relay); cudaDeviceSynchronize(); }
        { DeviceGuard g(r.kdev); cudaDeviceSynchronize(); }
        free_ring(r);
    }
    if (!r.made) {
        CK(make_device(relay));
        CK(make_device(kdev));
        r.relay = relay;
        r.kdev = kdev;
        r.S = S;
        r.slot_bytes = C;
        // flags are zeroed on each device's setup stream and waited for there alone: a new
        // ring never waits on (possibly long) user work already queued on the device
        {
            DeviceGuard g(relay);
            CK(cudaMalloc(&r.stage, (size_t)S * C));
            CK(cudaMalloc(&r.seq, 2 * 64 * sizeof(uint64_t)));
            CK(cudaMemsetAsync(r.seq, 0, 2 * 64 * sizeof(uint64_t), e.dev[relay].setup));
            r.credit = r.seq + 64;
        }
        {
            DeviceGuard g(kdev);
            // unit counters [64], the claim cursor, the leaders' observed flags [64]
            const size_t bytes = 64 * sizeof(unsigned) + 64 + 64 * sizeof(uint64_t);
            CK(cudaMalloc(&r.cnt, bytes));
            CK(cudaMemsetAsync(r.cnt, 0, bytes, e.dev[kdev].setup));
            r.cursor = (unsigned long long*)((char*)r.cnt + 64 * sizeof(unsigned));
            r.ready = (uint64_t*)((char*)r.cnt + 64 * sizeof(unsigned) + 64);
        }
        CK(cudaStreamSynchronize(e.dev[relay].setup));
        CK(cudaStreamSynchronize(e.dev[kdev].setup));
        r.g_next = 0;
        r.unit_next = 0;
        r.made = true;
    }
    *out = &r;
    return cudaSuccess;
}

// ------------------------------------------------------------------ transfer job ---


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

// Table buffers start at 4 MiB (a 131,072-segment table is 3 MiB) and grow by 1.5x: an
// allocation of pinned or device memory while copies are in flight can stall the enqueueing
// thread for tens of ms (scripts/probe_e2e.py with MMA_TRACE=1), so it should happen rarely.
constexpr size_t kScratchMin = 4u << 20;

// Grow-only device scratch on device `dev` for this call's tables.
static int scratch_dev(Scratch& sc, int dev, size_t bytes, void** out)
{
    if (sc.dev_cap[dev] < bytes) {
        DeviceGuard g(dev);
        if (sc.dev[dev]) cudaFree(sc.dev[dev]);
        sc.dev[dev] = nullptr;
        size_t cap = std::max(bytes + bytes / 2, kScratchMin);
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
        size_t cap = std::max(bytes + bytes / 2, kScratchMin);
        CK(cudaHostAlloc(&sc.host, cap, cudaHostAllocPortable | cudaHostAllocMapped));   // kernels read it
        sc.host_cap = cap;
    }
    *out = sc.host;
    return cudaSuccess;
}

// Measurement runs: grow every rotating table buffer of target d (host and each path GPU)
// to what a call of j's shape can need, so no timed call pays a first-use allocation.
int reserve_tables(const Job& j)
{
    Engine& e = E();
    Target& t = e.tgt[j.d];
    make_paths(j.d);
    const uint64_t n = j.B ? (j.B - 1) / j.C + 1 : 0;
    const uint64_t seg_words = j.contiguous ? 0 : (j.nseg + 1) + 2 * j.nseg;
    const size_t bytes = n * 4 + 4 + seg_words * 8;
    for (Scratch& sc : t.scratch) {
        if (sc.pending) {
            CK(cudaEventSynchronize(sc.done));
            sc.pending = false;
        }
        void* p = nullptr;
        CK((cudaError_t)scratch_host(sc, bytes, &p));
        for (const PathState& ps : t.paths[j.dir]) {
            CK(make_device(ps.gpu));
            CK((cudaError_t)scratch_dev(sc, ps.gpu, bytes, &p));
        }
        CK((cudaError_t)scratch_dev(sc, j.d, bytes, &p));
    }
    return cudaSuccess;
}

// Optional per-launch CUDA-event timing of the engine's kernels, recorded on the stream
// the kernel is launched on (mma_set_kernel_timing / mma_kernel_times).
std::vector<KRec> g_kpending;
bool g_ktime = false;
thread_local bool tl_capturing = false;
std::mutex g_kmu;

static int resolve_mode(const Job& j, int mode)
{
    if (mode == MMA_HOP_AUTO) mode = j.contiguous ? MMA_HOP_CE : MMA_HOP_ZC;
    if (mode == MMA_HOP_ZC && !j.mapped) mode = MMA_HOP_CE;
    return mode;
}

// ---- backlog ledger (NEXT-1) ---------------------------------------------------------
void ledger_retire()
{
    Engine& e = E();
    for (size_t i = 0; i < e.inflight.size();) {
        auto& f = e.inflight[i];
        if (cudaEventQuery(f.done) == cudaErrorNotReady) { i++; continue; }
        cudaGetLastError();
        for (int g = 0; g < MMA_MAX_GPUS; g++) {
            e.ledger[f.dir][g] -= f.bytes[g];
            e.ledger_own[f.dir][g] -= f.own[g];
            if (f.shared && (f.bytes[g] || f.own[g]))
                shm_ledger_add(f.dir, g, -(int64_t)f.bytes[g], -(int64_t)f.own[g], f.shared);
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
    // with a cross-process ledger attached, every process plans against every process's bytes
    f.shared = shm_ledger_gen();
    if (f.shared)
        for (int k = 0; k < MMA_MAX_GPUS; k++)
            if (bytes[k] || own[k]) shm_ledger_add(dir, k, (int64_t)bytes[k], (int64_t)own[k], f.shared);
    e.inflight.push_back(f);
    return cudaSuccess;
}

// Planner inputs of target d's paths: backlog from the ledger (bytes in flight on each
// link, the link's own target's direct bytes included), so a relay's chunks are planned
// behind whatever its link still carries. "Direct path first" (§3.4.2): a relay
// GPU whose own direct work is in flight in this process is returned in `gate`, and the
// call's relay work on it waits for that work (Call::gate); own direct work of ANOTHER process
// (cross-process ledger) cannot be waited for, so such a relay is not used (bandwidth 0).
void ledger_inputs(int d, int dir, const std::vector<PathState>& ps, std::vector<PlanPath>& pp,
                   std::vector<int>* gate)
{
    Engine& e = E();
    if (!e.cfg.ledger) return;
    ledger_retire();
    const bool shared = shm_ledger_on();
    for (size_t p = 0; p < ps.size(); p++) {
        const int g = ps[p].gpu;
        const uint64_t local_own = e.ledger_own[dir][g];
        uint64_t bytes = e.ledger[dir][g], own = local_own;
        if (shared) shm_ledger_get(dir, g, &bytes, &own);   // includes this process's bytes
        pp[p].backlog = bytes;
        if (ps[p].kind != MMA_PATH_RELAY || g == d) continue;
        if (own > local_own) pp[p].mbps = 0;
        else if (local_own > 0 && gate && std::find(gate->begin(), gate->end(), g) == gate->end())
            gate->push_back(g);
    }
}

int record_gates(int g, int dir)
{
    Engine& e = E();
    DevRes& r = e.dev[g];
    if (!r.made) return cudaSuccess;
    DeviceGuard dg(g);
    CK(cudaEventRecord(r.gate_ev[dir][0], r.lane[dir].direct));
    CK(cudaEventRecord(r.gate_ev[dir][1], r.lane[dir].zc));
    return cudaSuccess;
}

// MMA_TRACE=1: per-call host-time breakdown of the enqueue on stderr.
struct Trace {
    bool on;
    std::chrono::steady_clock::time_point last;
    std::string s;
    bool cap_debug = getenv("MMA_CAPTURE_DEBUG") != nullptr;
    cudaStream_t cap_stream = nullptr;
    Trace() : on(getenv("MMA_TRACE") != nullptr), last(std::chrono::steady_clock::now()) {}
    void mark(const char* what)
    {
        if (cap_debug) {   // MMA_CAPTURE_DEBUG: the capture status of the user stream per stage
            cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
            cudaStreamIsCapturing(cap_stream, &st);
            fprintf(stderr, "[mma capture] after %s: status %d\n", what, (int)st);
        }
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

// One multipath call being enqueued (engine mutex held). The stages run in this order:
// plan (a2) -> native fallback (a1) -> chunk lists and modes -> host tables -> fork (a3) ->
// table uploads -> delivery log -> measurement spans -> dynamic pull | direct and zero-copy
// paths (a4, a7) -> copy-engine relay rings (a5, a6, a9) -> join (a8).
class Call {
public:
    explicit Call(Job& j)
        : j_(j), eng_(E()), t_(eng_.tgt[j.d]),
          kind_(j.dir == MMA_H2D ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost)
    {
    }

    int run()
    {
        struct CaptureFlag {   // no timing / trace events inside a capture
            explicit CaptureFlag(bool on) { tl_capturing = on; }
            ~CaptureFlag() { tl_capturing = false; }
        } cflag(j_.capturing);
        int rc = begin();
        if (rc != cudaSuccess) return forked_ ? end(rc) : rc;   // a failure after the fork still joins
        if (done_) return rc;
        rc = enqueue_side(false);
        if (rc == cudaSuccess) rc = enqueue_side(true);
        return end(rc);
    }

    // ---- the phases run() strings together; run_multi interleaves them across the calls of
    // one joint plan (every call's direct side, then every call's relay side, gated)

    // plan .. fork .. uploads: everything before a byte moves. done() after it: the call was
    // completed by a native copy. An error after the fork must still go through end().
    int begin()
    {
        t0_ = std::chrono::steady_clock::now();
        char m[96];
        snprintf(m, sizeof m, "mma %s %s %.1f MiB -> gpu %d%s", j_.dir == MMA_H2D ? "h2d" : "d2h",
                 j_.contiguous ? "contig" : "segments", (double)j_.B / (1 << 20), j_.d,
                 j_.capturing ? " (captured)" : "");
        nvtxRangePushA(m);   // one NVTX range per call (SURVEY §5 tracing) around the enqueue
        nvtx_open_ = true;
        tr_.cap_stream = j_.user;
        tr_.mark("start");
        make_paths(j_.d);
        ps_ = &t_.paths[j_.dir];
        P_ = (int)ps_->size();
        host_order_ = !j_.contiguous && (eng_.cfg.host_order == 2 || (eng_.cfg.host_order == 1 && j_.dir == MMA_D2H));
        CK(plan());
        if (plan_.fallback) {
            bool done = false;
            CK(native_fallback(&done));
            if (done) { done_ = true; return finish(); }
        }
        CK(prepare());
        const int tb = build_tables();
        if (tb == kArenaFull) {   // a captured call whose tables do not fit: the native copy
            bool done = false;
            thr_ = ~0ull;
            CK(native_fallback(&done));
            done_ = true;
            return finish();
        }
        CK(tb);
        CK(fork());
        forked_ = true;
        // after the fork, a failing stage still joins every stream it enqueued on, so the
        // user stream never runs ahead of partial engine work; the error is returned
        int rc = upload_tables();
        if (rc == cudaSuccess) rc = delivery_log();
        if (rc == cudaSuccess) rc = open_timing();
        return rc;
    }

    bool done() const { return done_; }
    bool forked() const { return forked_; }

    // the direct side (relay = false: the target's own link, or a dynamic pull launch) or the
    // relay side (zero-copy relays and relay rings) of the call
    int enqueue_side(bool relay)
    {
        if (dynamic_) return relay ? cudaSuccess : enqueue_dynamic();
        CK(enqueue_paths(relay));
        return relay ? enqueue_rings() : cudaSuccess;
    }

    // relay work that crosses GPU g's PCIe link first waits for `ev` (recorded behind g's own
    // direct work): "the outstanding queue prioritizes completing direct tasks before
    // processing micro-tasks from other queues" (§3.4.2)
    void gate(int g, cudaEvent_t ev)
    {
        if (g >= 0 && g < MMA_MAX_GPUS && g != j_.d) gates_[g].push_back(ev);
    }

    int end(int rc)
    {
        if (rc != cudaSuccess) {
            if (forked_) {
                join_streams();
                if (!j_.capturing) mark_tables_busy();   // partial work may still read the tables
            }
            close_range();
            return rc;
        }
        rc = join();
        close_range();
        if (rc != cudaSuccess) return rc;
        return finish();
    }

    ~Call()
    {
        close_range();
        // every stream wait on the fork event is enqueued by now: the event can be reused
        if (pooled_fork_) eng_.dev[j_.user_dev].fork_pool.push_back(fork_);
    }

private:
    bool done_ = false, forked_ = false, nvtx_open_ = false, pooled_fork_ = false;
    std::vector<cudaEvent_t> gates_[MMA_MAX_GPUS];
    std::vector<cudaStream_t> gated_;   // streams already made to wait on their GPU's gates

    void close_range()
    {
        if (nvtx_open_) nvtxRangePop();
        nvtx_open_ = false;
    }

    // a relay stream on GPU g waits for g's gates once per call
    int apply_gates(cudaStream_t s, int g)
    {
        if (g < 0 || g >= MMA_MAX_GPUS || gates_[g].empty()) return cudaSuccess;
        if (std::find(gated_.begin(), gated_.end(), s) != gated_.end()) return cudaSuccess;
        gated_.push_back(s);
        DeviceGuard dg(g);
        for (cudaEvent_t ev : gates_[g]) CK(cudaStreamWaitEvent(s, ev, 0));
        return cudaSuccess;
    }

    Job& j_;
    Engine& eng_;
    Target& t_;
    const cudaMemcpyKind kind_;
    Trace tr_;
    std::chrono::steady_clock::time_point t0_;
    std::vector<PathState>* ps_ = nullptr;
    int P_ = 0;
    std::vector<PlanPath> pp_;
    std::vector<int> pmode_, mode_;
    uint64_t thr_ = 0;
    Plan plan_;
    uint64_t n_ = 0, n_log_ = 0, claimC_ = 0;
    Scratch* sc_ = nullptr;
    std::vector<std::vector<uint32_t>> lists_;
    std::vector<char> active_;
    bool dynamic_ = false;
    bool needs_tab_[MMA_MAX_GPUS] = {};
    bool need_ctab_ = false;
    size_t tab_bytes_ = 0;
    std::vector<size_t> ctab_off_;
    void* htab_ = nullptr;
    void* dtab_[MMA_MAX_GPUS] = {};
    cudaEvent_t fork_ = nullptr;
    std::vector<std::pair<cudaStream_t, int>> used_;   // engine streams this call enqueued on
    uint8_t* log_ = nullptr;
    uint64_t* fwd_ = nullptr;   // forward log (debug_log), on the target
    // host-address order (config host_order): a zero-copy path of a scattered transfer gets a
    // private table of its own pieces sorted by host address, copy-engine batches are sorted
    bool host_order_ = false;
    struct Priv {
        bool on = false;
        size_t off = 0;          // byte offset of its table in the upload
        uint64_t npieces = 0, B = 0;
        uint64_t src0 = 0, dst0 = 0;   // the first piece (the stream's one-piece form)
    };
    std::vector<Priv> priv_;
    struct HostSorted {   // the table's segments in host-address order (host_order_perm)
        std::vector<uint64_t> src, dst, vs, ve;   // addresses and [start, end) in v
    };
    std::shared_ptr<const HostSorted> sorted_;
    std::vector<uint8_t> owner_;   // path carrying each chunk (from the work lists)
    static constexpr int kArenaFull = -1000;
    struct CapturedAlloc {
        int dev;
        cudaStream_t s;
        void* p;
    };
    std::vector<CapturedAlloc> captured_;   // captured relay staging, freed behind the join
    // NUMA (R23): the host node of every segment (when the path set spans two or more nodes)
    // and, with numa_plan, the table regrouped by node in path order
    std::vector<int> seg_node_;
    std::vector<mma_segment_t> reseg_;

    PathState& path(int p) { return (*ps_)[p]; }
    Lanes& lanes(int g) { return j_.capturing ? eng_.dev[g].cap_lane[j_.dir] : eng_.dev[g].lane[j_.dir]; }

    int finish()
    {
        t_.stats.issue_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0_).count();
        return cudaSuccess;
    }

    uint64_t path_bytes(int p) const
    {
        uint64_t b = 0;
        for (uint32_t i : lists_[p]) {
            uint64_t o, l;
            j_.extent(i, &o, &l);
            b += l;
        }
        return b;
    }

    // ---- plan (a2): bandwidth and mode per path (scattered tuning, measurement overrides),
    // backlog from the ledger, then the integer earliest-finish plan
    int plan()
    {
        pp_.resize(P_);
        pmode_.resize(P_);
        for (int p = 0; p < P_; p++) {
            const PathState& q = path(p);
            uint32_t bw = (!j_.contiguous && q.seg_mbps) ? q.seg_mbps : q.mbps;
            if (j_.bw_override) bw = j_.bw_override[p];
            pp_[p] = PlanPath{q.kind == MMA_PATH_DIRECT, bw, 0};
            pmode_[p] = (!j_.contiguous && q.seg_mode >= 0) ? q.seg_mode : q.mode;
            if (j_.mode_override) pmode_[p] = j_.mode_override[p];
        }
        thr_ = j_.no_small_fallback ? 0 : eng_.cfg.fallback_bytes[j_.dir];
        if (j_.capturing) {
            // a graph replays this call any number of times: kernel rings (whose sequence
            // numbers advance per call) and the ledger (which retires calls by events) stay
            // out; zero-copy paths, the direct copy engine and all-copy-engine relays (on
            // staging of their own, enqueue_captured_p2p) replay as they are
            for (int p = 0; p < P_; p++)
                if (path(p).kind == MMA_PATH_RELAY && kernel_ring(resolve_mode(j_, pmode_[p]))) pp_[p].mbps = 0;
        } else if (!j_.bw_override && !j_.plan_override) {
            std::vector<int> gate;
            ledger_inputs(j_.d, j_.dir, *ps_, pp_, &gate);
            for (int g : gate) {   // relays behind their own links' direct work
                CK(record_gates(g, j_.dir));
                for (cudaEvent_t ev : eng_.dev[g].gate_ev[j_.dir]) this->gate(g, ev);
            }
        }
        const int pm = eng_.cfg.plan_mode == PLAN_DYNAMIC ? PLAN_CONTIGUOUS : eng_.cfg.plan_mode;
        if (j_.plan_override) {   // a joint plan (run_multi): the chunk -> path map is given
            plan_ = Plan();
            plan_.n = j_.plan_override->size();
            plan_.path = *j_.plan_override;
            plan_.count.assign(P_, 0);
            for (uint8_t p : plan_.path) {
                if (p >= P_) return cudaErrorInvalidValue;
                plan_.count[p]++;
            }
            if (plan_.n != (j_.B ? (j_.B - 1) / j_.C + 1 : 0)) return cudaErrorInvalidValue;
        } else if (make_plan(pp_.data(), P_, j_.B, j_.C, thr_, pm, plan_) != 0) {
            return cudaErrorInvalidValue;
        }
        t_.stats.calls++;
        t_.stats.bytes += j_.B;
        t_.stats.validate_us += j_.validate_us;
        t_.last_order.clear();
        t_.stats.ptr_queries += j_.ptr_queries;
        tr_.mark("plan");
        return cudaSuccess;
    }

    // ---- fallback (a1): the native copy on the user stream (§3.2). A single direct
    // path in zero-copy mode is not native: it continues as a one-path plan.
    int native_fallback(bool* done)
    {
        const bool small = j_.B < thr_;
        if (small || resolve_mode(j_, pmode_[0]) != MMA_HOP_ZC) {
            t_.stats.fallbacks++;
            DmaBatch b;
            j_.pieces(0, j_.B, [&](const Piece& x) { b.add(x.dst, x.src, x.len); });
            if (!small && host_order_) b.sort_by_host(kind_);   // a one-path plan, not a small copy
            TSpan ts(j_.user_dev, j_.user, "DMA native (fallback)", 0, -1, j_.B);
            CK((cudaError_t)b.issue(kind_, j_.user));
            t_.stats.path_bytes[j_.dir][0] += j_.B;
            t_.stats.path_chunks[j_.dir][0] += 1;
            t_.log_n = 0;
            t_.fwd_n = 0;
            if (eng_.cfg.ledger && !j_.capturing) {
                uint64_t lb[MMA_MAX_GPUS] = {}, lo[MMA_MAX_GPUS] = {};
                lb[j_.d] = lo[j_.d] = j_.B;
                CK(ledger_add(j_.dir, j_.user_dev, j_.user, lb, lo));
            }
            *done = true;
            return cudaSuccess;
        }
        t_.stats.single_path_calls++;
        plan_.fallback = false;
        plan_.n = (j_.B - 1) / j_.C + 1;
        plan_.path.assign(plan_.n, 0);
        plan_.count.assign(P_, 0);
        plan_.count[0] = plan_.n;
        return cudaSuccess;
    }

    // ---- NUMA-affine regrouping (reading R23): segments stably grouped by the NUMA node of
    // their host memory, groups in the order of the usable paths' nodes (the target's first),
    // then other nodes, unknown last. The virtual stream is the regrouped table, so the
    // contiguous plan gives each path the bytes of its own node except at group boundaries.
    int numa_regroup()
    {
        if (j_.contiguous || j_.nseg < 2) return cudaSuccess;
        if (eng_.cfg.debug_log) {   // identity unless regrouped below
            t_.last_order.resize(j_.nseg);
            for (uint64_t k = 0; k < j_.nseg; k++) t_.last_order[k] = (uint32_t)k;
        }
        std::vector<int> order;   // distinct known nodes of the paths that may carry bytes
        for (int p = 0; p < P_; p++) {
            const int nd = path(p).node;
            if (pp_[p].mbps == 0 || nd < 0) continue;
            if (std::find(order.begin(), order.end(), nd) == order.end()) order.push_back(nd);
        }
        if (order.size() < 2) return cudaSuccess;
        const uint64_t n = j_.nseg;
        std::vector<const void*> hp(n);
        for (uint64_t k = 0; k < n; k++) hp[k] = j_.dir == MMA_H2D ? j_.segs[k].src : j_.segs[k].dst;
        seg_node_.resize(n);
        host_nodes(hp.data(), n, seg_node_.data());
        if (!eng_.cfg.numa_plan) return cudaSuccess;   // nodes kept for the statistics only
        // group rank of each segment: the paths' nodes in path order, other known nodes by id,
        // unknown last; a stable counting sort over the ranks (O(n), the table is large)
        int maxnode = -1;
        for (uint64_t k = 0; k < n; k++) maxnode = std::max(maxnode, seg_node_[k]);
        const int R = (int)order.size() + std::max(0, maxnode + 1) + 1;   // last rank: unknown
        std::vector<int> rank_of(std::max(0, maxnode + 1), -1);
        for (size_t r = 0; r < order.size(); r++)
            if (order[r] <= maxnode) rank_of[order[r]] = (int)r;
        auto rank = [&](int nd) -> int {
            if (nd < 0) return R - 1;
            return rank_of[nd] >= 0 ? rank_of[nd] : (int)order.size() + nd;
        };
        std::vector<uint32_t> start(R + 1, 0);
        for (uint64_t k = 0; k < n; k++) start[rank(seg_node_[k]) + 1]++;
        for (int r = 0; r < R; r++) start[r + 1] += start[r];
        std::vector<uint32_t> idx(n);
        for (uint64_t k = 0; k < n; k++) idx[start[rank(seg_node_[k])]++] = (uint32_t)k;
        if (eng_.cfg.debug_log) t_.last_order = idx;
        reseg_.resize(n);
        std::vector<int> nodes(n);
        for (uint64_t k = 0; k < n; k++) {
            reseg_[k] = j_.segs[idx[k]];
            nodes[k] = seg_node_[idx[k]];
        }
        seg_node_.swap(nodes);
        j_.segs = reseg_.data();
        for (uint64_t k = 0; k < n; k++) j_.vstart[k + 1] = j_.vstart[k] + j_.segs[k].bytes;
        return cudaSuccess;
    }

    // bytes whose host node is known, and of those the bytes carried by a path on that node
    void numa_stats()
    {
        if (seg_node_.empty() || dynamic_) return;
        uint64_t known = 0, local = 0;
        for (uint64_t i = 0; i < n_; i++) {
            const int pn = path(plan_.path[i]).node;
            uint64_t a, len;
            j_.extent(i, &a, &len);
            const uint64_t b = a + len;
            uint64_t k = std::upper_bound(j_.vstart.begin(), j_.vstart.end(), a) - j_.vstart.begin() - 1;
            for (; k < j_.nseg && j_.vstart[k] < b; k++) {
                const uint64_t lo = std::max(j_.vstart[k], a), hi = std::min(j_.vstart[k + 1], b);
                if (lo >= hi || seg_node_[k] < 0) continue;
                known += hi - lo;
                if (seg_node_[k] == pn) local += hi - lo;
            }
        }
        t_.stats.numa_known_bytes[j_.dir] += known;
        t_.stats.numa_local_bytes[j_.dir] += local;
    }

    // ---- table buffers, devices, per-path chunk lists and modes
    int prepare()
    {
        CK(numa_regroup());
        n_ = plan_.n;
        sc_ = &t_.scratch[t_.parity & 3];
        if (!j_.capturing) t_.parity++;
        if (!j_.capturing && sc_->pending) {   // the call four back used these tables: it must be finished
            const auto w0 = std::chrono::steady_clock::now();
            CK(cudaEventSynchronize(sc_->done));
            sc_->pending = false;
            t_.stats.wait_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - w0).count();
        }
        // every GPU of the path set gets its streams and peer access before any enqueue
        for (int p = 0; p < P_; p++) CK(make_device(path(p).gpu));
        tr_.mark("scratch");
        lists_.assign(P_, {});
        for (uint64_t i = 0; i < n_; i++) lists_[plan_.path[i]].push_back((uint32_t)i);
        if (eng_.fault_misroute && P_ >= 2 && !lists_[0].empty() && !lists_[1].empty()) {   // test hook
            const uint32_t c = lists_[0].back();
            lists_[0].pop_back();
            lists_[1].insert(std::lower_bound(lists_[1].begin(), lists_[1].end(), c), c);
        }
        mode_.resize(P_);
        for (int p = 0; p < P_; p++) {
            mode_[p] = resolve_mode(j_, pmode_[p]);
            if ((mode_[p] == MMA_HOP_CE_P2P || mode_[p] == MMA_HOP_PUSH) && path(p).kind == MMA_PATH_DIRECT)
                mode_[p] = MMA_HOP_CE;
            // a kernel ring whose relay kernel updates the ring's flags across the link needs
            // native peer atomics (H2D pull: flags on the relay, kernel on the target; D2H
            // push: the same); without them the ring's copy-engine form carries the chunks
            if (kernel_ring(mode_[p]) && path(p).kind == MMA_PATH_RELAY) {
                const int kd = ring_kdev(j_.d, j_.dir, path(p).gpu, mode_[p]);
                if (!eng_.p2p_atomic[kd][path(p).gpu]) mode_[p] = MMA_HOP_CE_P2P;
            }
        }
        // GPU-driven dynamic pull when every usable path moves bytes with SMs:
        // the assignment is then observed (delivery log, per-path counts), not planned
        dynamic_ = eng_.cfg.plan_mode == PLAN_DYNAMIC && !j_.timing && !j_.capturing;
        active_.assign(P_, 0);
        for (int p = 0; p < P_; p++) {
            active_[p] = !lists_[p].empty();
            if (dynamic_ && pp_[p].mbps && mode_[p] != MMA_HOP_ZC) dynamic_ = false;
            // every path's kernel claims from a cursor in the target's memory
            if (dynamic_ && pp_[p].mbps && !eng_.p2p_atomic[path(p).gpu][j_.d]) dynamic_ = false;
        }
        if (dynamic_)
            for (int p = 0; p < P_; p++) active_[p] = pp_[p].mbps > 0;
        claimC_ = eng_.cfg.claim_bytes ? eng_.cfg.claim_bytes : (256u << 10);
        n_log_ = dynamic_ ? (j_.B - 1) / claimC_ + 1 : n_;
        numa_stats();
        return cudaSuccess;
    }

    // ---- host tables: the shared segment table and (interleaved plans) the chunk lists,
    // built only when some kernel reads them (copy-engine-only calls build none), then the
    // private host-ordered tables of zero-copy paths
    int build_tables()
    {
        bool shared = false, any_priv = false;
        priv_.assign(P_, Priv());
        for (int p = 0; p < P_; p++) {
            if (!active_[p]) continue;
            if (mode_[p] == MMA_HOP_ZC) {
                needs_tab_[path(p).gpu] = true;
                if (host_order_ && !dynamic_) priv_[p].on = any_priv = true;
                else shared = true;
            } else if (path(p).kind == MMA_PATH_RELAY && kernel_ring(mode_[p])) {   // the relay kernel
                needs_tab_[ring_kdev(j_.d, j_.dir, path(p).gpu, mode_[p])] = shared = true;
            }
        }
        if (any_priv) count_privates();
        if (any_priv) tr_.mark("count");
        need_ctab_ = shared && e_plan_interleaved() && !dynamic_;
        const uint64_t seg_words = (shared && !j_.contiguous) ? (j_.nseg + 1) + 2 * j_.nseg : 0;
        size_t bytes = seg_words * 8 + (need_ctab_ ? n_ * 4 + (n_ & 1) * 4 : 0);
        for (auto& q : priv_)
            if (q.on) {
                q.off = bytes;
                bytes += (3 * q.npieces + 1) * 8 + ((q.npieces * 4 + 7) & ~(uint64_t)7);
            }
        tab_bytes_ = bytes;
        ctab_off_.assign(P_, 0);
        if (tab_bytes_ && j_.capturing) {   // replays read the tables: they live in the arena
            const size_t need = (tab_bytes_ + 255) & ~(size_t)255;
            if (!eng_.arena || eng_.arena_used + need > eng_.arena_cap) return kArenaFull;
            htab_ = eng_.arena + eng_.arena_used;
            eng_.arena_used += need;
        } else if (tab_bytes_) {
            CK((cudaError_t)scratch_host(*sc_, tab_bytes_, &htab_));
        }
        if (tab_bytes_) {
            char* h = (char*)htab_;
            size_t o = 0;
            if (seg_words) {
                uint64_t* w = (uint64_t*)h;
                memcpy(w, j_.vstart.data(), (j_.nseg + 1) * 8);
                for (uint64_t k = 0; k < j_.nseg; k++) {
                    w[j_.nseg + 1 + k] = (uint64_t)j_.segs[k].src;
                    w[2 * j_.nseg + 1 + k] = (uint64_t)j_.segs[k].dst;
                }
                o = seg_words * 8;
            }
            if (need_ctab_)
                for (int p = 0; p < P_; p++) {
                    ctab_off_[p] = o;
                    memcpy(h + o, lists_[p].data(), lists_[p].size() * 4);
                    o += lists_[p].size() * 4;
                }
            tr_.mark("shared");
            if (any_priv) fill_privates(h);
        }
        tr_.mark("tables");
        return cudaSuccess;
    }

    bool e_plan_interleaved() const { return eng_.cfg.plan_mode == PLAN_INTERLEAVED || j_.interleaved_plan; }

    // the private streams of the zero-copy paths that get one (priv_[p].on): each path's
    // pieces -- the parts of the chunks it carries -- in host-address order, a virtual stream
    // of B_p bytes that the path's zero-copy kernel moves alone. One pass over the segments in
    // host order (a single sort, cached for a table identical to the previous one) assigns
    // every piece to the path carrying its chunk (the work lists, i.e. what is executed); each
    // piece keeps the chunk's index, which the kernel logs. count_privates sizes the tables,
    // fill_privates writes them straight into the pinned table buffer:
    //   [npieces + 1] start offsets | [npieces] src | [npieces] dst | [npieces] u32 chunk
    template <typename F>
    void each_private_piece(F&& f)
    {
        const uint64_t C = j_.C;
        const HostSorted& hs = *sorted_;
        for (size_t x = 0; x < hs.vs.size(); x++) {   // segments in host order, read in sequence
            const uint64_t vk = hs.vs[x], vk1 = hs.ve[x];
            for (uint64_t c = vk / C; c * C < vk1; c++) {
                const int p = owner_[c];
                if (!priv_[p].on) continue;
                const uint64_t lo = std::max(vk, c * C), hi = std::min(vk1, (c + 1) * C);
                f(p, x, c, lo - vk, hi - lo);
            }
        }
    }

    void count_privates()
    {
        host_order_perm();
        tr_.mark("host-order");
        owner_.resize(n_);
        for (int p = 0; p < P_; p++)
            for (uint32_t i : lists_[p]) owner_[i] = (uint8_t)p;
        for (auto& q : priv_) q.npieces = q.B = 0;
        each_private_piece([&](int p, size_t, uint64_t, uint64_t, uint64_t len) {
            priv_[p].npieces++;
            priv_[p].B += len;
        });
    }

    void fill_privates(char* h)
    {
        std::vector<uint64_t> at(P_, 0);
        for (auto& q : priv_)
            if (q.on) ((uint64_t*)(h + q.off))[0] = 0;
        const HostSorted& hs = *sorted_;
        each_private_piece([&](int p, size_t k, uint64_t c, uint64_t off, uint64_t len) {
            Priv& q = priv_[p];
            uint64_t* w = (uint64_t*)(h + q.off);
            const uint64_t x = at[p]++, n = q.npieces;
            w[x + 1] = w[x] + len;
            w[n + 1 + x] = hs.src[k] + off;
            w[2 * n + 1 + x] = hs.dst[k] + off;
            ((uint32_t*)(w + 3 * n + 1))[x] = (uint32_t)c;
            if (x == 0) {   // the one-piece form of the stream (private_stream_on)
                q.src0 = w[n + 1];
                q.dst0 = w[2 * n + 1];
            }
        });
    }

    // the segments in ascending host address (H2D: sources, D2H: destinations), as arrays
    // read in sequence by the table passes; kept for the next call if its table is the same
    // (a repeated offload of one block table pays one memcmp instead of a sort and a gather)
    void host_order_perm()
    {
        static std::mutex mu;
        static int dir = -1;
        static std::vector<mma_segment_t> last;
        static auto cached = std::make_shared<HostSorted>();
        std::lock_guard<std::mutex> g(mu);   // (the engine mutex is held too)
        const uint64_t n = j_.nseg;
        if (dir == j_.dir && last.size() == n && !memcmp(last.data(), j_.segs, n * sizeof(mma_segment_t))) {
            sorted_ = cached;
            return;
        }
        std::vector<uint64_t> key(n);
        for (uint64_t k = 0; k < n; k++)
            key[k] = (uint64_t)(j_.dir == MMA_D2H ? (const void*)j_.segs[k].dst : j_.segs[k].src);
        std::vector<uint32_t> perm;
        order_by_key(key.data(), n, perm);
        auto hs = std::make_shared<HostSorted>();
        hs->src.resize(n);
        hs->dst.resize(n);
        hs->vs.resize(n);
        hs->ve.resize(n);
        for (uint64_t x = 0; x < n; x++) {
            const uint32_t k = perm[x];
            hs->src[x] = (uint64_t)j_.segs[k].src;
            hs->dst[x] = (uint64_t)j_.segs[k].dst;
            hs->vs[x] = j_.vstart[k];
            hs->ve[x] = j_.vstart[k + 1];
        }
        dir = j_.dir;
        last.assign(j_.segs, j_.segs + n);
        cached = hs;
        sorted_ = hs;
    }

    // ---- fork (a3): an event on the user stream gates every engine stream the call uses
    int fork()
    {
        DeviceGuard g(j_.user_dev);
        CK(make_device(j_.user_dev));
        if (j_.capturing) {
            fork_ = eng_.dev[j_.user_dev].cap_fork;
        } else {   // an event of its own: calls of one joint plan fork before any of them forks a stream
            auto& pool = eng_.dev[j_.user_dev].fork_pool;
            if (pool.empty()) {
                cudaEvent_t ev = nullptr;
                CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                pool.push_back(ev);
            }
            fork_ = pool.back();
            pool.pop_back();
            pooled_fork_ = true;
        }
        CK(cudaEventRecord(fork_, j_.user));
        return cudaSuccess;
    }

    int use(cudaStream_t s, int dev)
    {
        for (auto& u : used_)
            if (u.first == s) return cudaSuccess;
        used_.push_back({s, dev});
        DeviceGuard g(dev);
        return (int)cudaStreamWaitEvent(s, fork_, 0);
    }

    // table uploads, one per device that runs a kernel, on that device's kernel stream
    int upload_tables()
    {
        for (int g = 0; g < eng_.ndev; g++) {
            if (!needs_tab_[g] || !tab_bytes_) continue;
            CK(make_device(g));
            DeviceGuard dg(g);
            CK((cudaError_t)use(lanes(g).kern, g));
            if (j_.capturing) CK(cudaMallocAsync(&dtab_[g], tab_bytes_, lanes(g).kern));   // a graph allocation
            else CK((cudaError_t)scratch_dev(*sc_, g, tab_bytes_, &dtab_[g]));
            if (!j_.capturing && tab_bytes_ >= (64u << 10) && eng_.upload_by_kernel) {
                // a large table is fetched by the zero-copy kernel from the mapped staging
                // buffer: a copy-engine upload would queue behind whatever DMAs the copy
                // engines hold (131,072 per-segment DMAs of another call), and its enqueue
                // blocks the host once the engine's queue is full
                ZcLaunchArg a{};
                a.v.nseg = 1;
                a.v.B = a.v.C = tab_bytes_;
                a.v.src0 = (uint64_t)htab_;
                a.v.dst0 = (uint64_t)dtab_[g];
                a.chunks.count = 1;
                a.unit_bytes = eng_.unit_bytes;
                const unsigned grid = (unsigned)std::min<uint64_t>((tab_bytes_ + eng_.unit_bytes - 1) / eng_.unit_bytes, 8);
                CK(launch_zc(a, grid, lanes(g).kern));
                t_.stats.kernels++;
            } else {
                CK(cudaMemcpyAsync(dtab_[g], htab_, tab_bytes_, cudaMemcpyHostToDevice, lanes(g).kern));
            }
        }
        tr_.mark("upload");
        return cudaSuccess;
    }

    // streams other than kern that launch table-reading kernels wait for the upload
    int after_upload(cudaStream_t s, int g)
    {
        if (!dtab_[g] || s == lanes(g).kern) return cudaSuccess;
        cudaEvent_t ev = join_event(lanes(g).kern, g);
        DeviceGuard dg(g);
        CK(cudaEventRecord(ev, lanes(g).kern));
        return (int)cudaStreamWaitEvent(s, ev, 0);
    }

    VStreamArg vstream_on(int g) const
    {
        VStreamArg v{};
        v.B = j_.B;
        v.C = j_.C;
        if (j_.contiguous) {
            v.nseg = 1;
            v.src0 = (uint64_t)j_.src0;
            v.dst0 = (uint64_t)j_.dst0;
        } else {
            v.nseg = j_.nseg;
            const uint64_t* w = (const uint64_t*)dtab_[g];
            v.start = w;
            v.src = w + j_.nseg + 1;
            v.dst = w + 2 * j_.nseg + 1;
        }
        return v;
    }

    // the private stream of zero-copy path p (build_private) on device g, and its chunks
    const uint32_t* private_chunks_on(int p, int g) const
    {
        const Priv& q = priv_[p];
        return (const uint32_t*)((const char*)dtab_[g] + q.off + (3 * q.npieces + 1) * 8);
    }

    VStreamArg private_stream_on(int p, int g) const
    {
        const Priv& q = priv_[p];
        VStreamArg v{};
        v.B = q.B;
        v.C = j_.C;
        if (q.npieces == 1) {
            v.nseg = 1;
            v.src0 = q.src0;
            v.dst0 = q.dst0;
        } else {
            const uint64_t* w = (const uint64_t*)((const char*)dtab_[g] + q.off);
            v.nseg = q.npieces;
            v.start = w;
            v.src = w + q.npieces + 1;
            v.dst = w + 2 * q.npieces + 1;
        }
        return v;
    }

    ChunkListArg chunks_on(int p, int g) const
    {
        ChunkListArg c{};
        c.count = lists_[p].size();
        if (c.count == 0) return c;
        if (need_ctab_) c.table = (const uint32_t*)((const char*)dtab_[g] + ctab_off_[p]);
        else c.first = lists_[p][0];
        return c;
    }

    // delivery log (debug): one byte per chunk (per claim in dynamic pull), 0xff = unwritten
    int delivery_log()
    {
        if (j_.no_log) return cudaSuccess;   // log_ stays null; the target's log is another call's
        if (!eng_.cfg.debug_log || j_.capturing) {
            t_.log_n = 0;
            t_.fwd_n = 0;
            return cudaSuccess;
        }
        DeviceGuard g(j_.d);
        if (t_.log_cap < n_log_) {
            if (t_.log) cudaFree(t_.log);
            CK(cudaMalloc(&t_.log, n_log_));
            t_.log_cap = n_log_;
        }
        log_ = t_.log;
        t_.log_n = n_log_;
        CK((cudaError_t)use(lanes(j_.d).direct, j_.d));
        CK(cudaMemsetAsync(log_, 0xff, n_log_, lanes(j_.d).direct));
        if (dynamic_) {
            t_.fwd_n = 0;
            return cudaSuccess;
        }
        if (t_.fwd_cap < n_) {   // forward log: 0 = no relay kernel observed this chunk
            if (t_.fwd) cudaFree(t_.fwd);
            CK(cudaMalloc(&t_.fwd, n_ * 16));
            t_.fwd_cap = n_;
        }
        fwd_ = t_.fwd;
        t_.fwd_n = n_;
        return (int)cudaMemsetAsync(fwd_, 0, n_ * 16, lanes(j_.d).direct);
    }

    // ---- measurement runs: every path's spans open at the fork, before any path's work is
    // enqueued, so a path's time counts from the start of the call even where paths share a
    // stream (loopback relays share their GPU's streams)
    int open_timing()
    {
        if (!j_.timing) return cudaSuccess;
        for (int p = 0; p < P_; p++) {
            if (lists_[p].empty()) continue;
            const int g = path(p).gpu;
            CK(make_device(g));
            Lanes& L = lanes(g);
            if (mode_[p] == MMA_HOP_ZC || path(p).kind == MMA_PATH_DIRECT) {
                cudaStream_t s = mode_[p] == MMA_HOP_ZC ? L.zc : L.direct;
                CK((cudaError_t)use(s, g));
                j_.timing->start(p, g, s);
                continue;
            }
            if (!eng_.wait64 || !eng_.write64) return MMA_ERR_NO_MEMOPS;
            Ring* r = nullptr;   // enqueue_rings gets the same ring and base
            CK((cudaError_t)get_ring(j_.d, j_.dir, p, j_.C, ring_slots_for(j_.C), mode_[p] == MMA_HOP_PUSH, &r));
            for (size_t c = 0; c < lists_[p].size() && c < 2 * (size_t)r->S; c++) {
                cudaStream_t hs = L.hop[((r->g_next + c) % r->S) & 1];
                CK((cudaError_t)use(hs, g));
                j_.timing->start(p, g, hs);
            }
        }
        return cudaSuccess;
    }

    // ---- dynamic pull: one claim cursor per call in d's memory, one kernel per path GPU
    int enqueue_dynamic()
    {
        if (!t_.dyn) {
            DeviceGuard g(j_.d);
            CK(cudaMalloc(&t_.dyn, kDynSlots * kDynSlotWords * sizeof(unsigned long long)));
        }
        unsigned long long* slot = t_.dyn + (t_.dyn_next++ % kDynSlots) * kDynSlotWords;
        cudaStream_t zs = lanes(j_.d).zc;
        CK((cudaError_t)use(zs, j_.d));
        cudaEvent_t zeroed = join_event(zs, j_.d);
        {
            DeviceGuard g(j_.d);
            CK(cudaMemsetAsync(slot, 0, kDynSlotWords * sizeof(unsigned long long), zs));
            CK(cudaEventRecord(zeroed, zs));
        }
        t_.last_dyn = slot;
        t_.last_dyn_paths = P_;
        t_.stats.dynamic_calls++;
        for (int p = 0; p < P_; p++) {
            if (!active_[p]) continue;
            const int g = path(p).gpu;
            cudaStream_t s = lanes(g).zc;
            CK((cudaError_t)use(s, g));
            CK((cudaError_t)after_upload(s, g));
            DeviceGuard dg(g);
            if (s != zs) CK(cudaStreamWaitEvent(s, zeroed, 0));
            DynLaunchArg a{};
            a.v = vstream_on(g);
            a.v.C = claimC_;   // the claim unit plays the chunk's role
            a.nchunks = n_log_;
            a.cursor = slot;
            a.counts = slot + 1;
            a.backoffs = slot + kDynBackoffWord;
            a.pause = slot + kDynPauseWord + p;
            if (eng_.cfg.background_policy == 1 && pp_[p].mbps) {   // yield to background traffic
                a.yield_pct = eng_.cfg.yield_pct ? eng_.cfg.yield_pct : 150;
                const uint64_t ctas = std::min<uint64_t>(n_log_, zc_grid(g, j_.dir));
                // ns one claim unit takes when the path's measured rate is split over its CTAs
                a.expect_ns = claimC_ * ctas * 1000ull / pp_[p].mbps;
            }
            a.path = (uint32_t)p;
            a.log = log_;
            const unsigned grid = (unsigned)std::min<uint64_t>(n_log_, zc_grid(g, j_.dir));
            KTimer kt(g, s, 3 | (j_.dir << 4) | (p << 8));
            TSpan ts(g, s, "zero-copy dynamic pull", p, -1, 0);
            CK(launch_zc_dyn(a, grid, s));
            t_.stats.kernels++;
        }
        return cudaSuccess;
    }

    // ---- direct path (a4, a7) when relay = false; zero-copy relays (a7) when relay = true;
    // copy-engine relays are enqueue_rings'
    int enqueue_paths(bool relay_side)
    {
        for (int p = 0; p < P_; p++) {
            if (lists_[p].empty()) continue;
            const bool relay = path(p).kind == MMA_PATH_RELAY;
            if (relay != relay_side) continue;
            const int g = path(p).gpu;
            CK(make_device(g));
            const uint64_t bytes_p = path_bytes(p);
            t_.stats.path_bytes[j_.dir][p] += bytes_p;
            t_.stats.path_chunks[j_.dir][p] += lists_[p].size();
            if (relay) t_.stats.relay_bytes += bytes_p;
            if (j_.timing) j_.timing->bytes[p] = bytes_p;
            if (mode_[p] == MMA_HOP_ZC) CK(enqueue_zero_copy(p, g, relay, bytes_p));
            else if (!relay) CK(enqueue_direct_ce(p, g));
            // (copy-engine relays: their bytes are counted here, moved by enqueue_rings)
        }
        tr_.mark(relay_side ? "zc relays" : "direct");
        return cudaSuccess;
    }

    // one kernel per path: on d for the direct path, on r for a one-hop relay
    int enqueue_zero_copy(int p, int g, bool relay, uint64_t bytes_p)
    {
        cudaStream_t s = lanes(g).zc;
        CK((cudaError_t)use(s, g));
        if (relay) CK(apply_gates(s, g));
        CK((cudaError_t)after_upload(s, g));
        ZcLaunchArg a{};
        const bool own = priv_[p].on;
        if (own) {   // its own host-ordered stream: chunks 0..ceil(B_p/C)-1 of it
            a.v = private_stream_on(p, g);
            a.chunks.count = (priv_[p].B + j_.C - 1) / j_.C;
            a.chunks.first = 0;
        } else {
            a.v = vstream_on(g);
            a.chunks = chunks_on(p, g);
        }
        a.unit_bytes = eng_.unit_bytes;
        a.path = (uint32_t)p;
        a.log = log_;
        if (own) a.piece_chunk = private_chunks_on(p, g);   // the kernel logs each piece's chunk
        const uint64_t upc = (j_.C + eng_.unit_bytes - 1) / eng_.unit_bytes;
        const unsigned grid = (unsigned)std::min<uint64_t>(a.chunks.count * upc, zc_grid(g, j_.dir));
        DeviceGuard dg(g);
        {
            const bool bulk = eng_.zc_bulk && !relay;   // the bulk kernel: direct paths (no peer addresses)
            KTimer kt(g, s, (bulk ? 4 : 0) | (j_.dir << 4) | (p << 8));
            TSpan ts(g, s, relay ? "zero-copy one-hop relay kernel" : "zero-copy direct kernel", p, -1, bytes_p);
            CK(launch_zc(a, grid, s, bulk));
        }
        t_.stats.kernels++;
        if (j_.timing) j_.timing->end(p);
        return cudaSuccess;
    }

    // direct copy engine: one DMA (or batch) per run of consecutive chunks
    int enqueue_direct_ce(int p, int g)
    {
        cudaStream_t s = lanes(g).direct;
        CK((cudaError_t)use(s, g));
        DeviceGuard dg(g);
        const auto& L = lists_[p];
        for (size_t a = 0; a < L.size();) {
            size_t b = a + 1;
            while (b < L.size() && L[b] == L[b - 1] + 1) b++;
            uint64_t o0, l0, o1, l1;
            j_.extent(L[a], &o0, &l0);
            j_.extent(L[b - 1], &o1, &l1);
            DmaBatch batch;
            j_.pieces(o0, o1 + l1, [&](const Piece& x) { batch.add(x.dst, x.src, x.len); });
            if (host_order_) batch.sort_by_host(kind_);
            {
                TSpan ts(g, s, "DMA direct", p, L[a], o1 + l1 - o0);
                CK((cudaError_t)batch.issue(kind_, s));
            }
            if (log_) CK(cudaMemsetAsync(log_ + L[a], p, b - a, s));
            a = b;
        }
        if (j_.timing) j_.timing->end(p);
        return cudaSuccess;
    }

    // ---- copy-engine relay rings (a5, a6 for H2D; a9 for D2H), enqueued in WAVES of at most
    // S chunks per ring, so that every wait the call enqueues depends only on work enqueued
    // before it:
    //   H2D wave w: the hops of w first (hop 1 of chunk c waits for the credit of chunk c - S,
    //     which the pull kernel of an earlier wave releases), then the pull kernel of w;
    //   D2H wave w: the pack kernel of w first (its credit waits name chunks of earlier waves,
    //     whose hops are already enqueued), then the hops of w (they wait for its seq flags).
    // The copy therefore completes when launches are serialised (CUDA_LAUNCH_BLOCKING, a
    // profiler that runs each kernel alone), and a call that fails part-way leaves nothing
    // waiting on work that was never issued. A wave holds at most S chunks of a ring because
    // chunk c's slot last held chunk c - S, which must belong to an earlier wave.
    int enqueue_rings()
    {
        std::vector<int> rp;   // relay paths using rings
        for (int p = 0; p < P_; p++)
            if (!lists_[p].empty() && path(p).kind == MMA_PATH_RELAY &&
                (kernel_ring(mode_[p]) || mode_[p] == MMA_HOP_CE_P2P))
                rp.push_back(p);
        if (rp.empty()) return cudaSuccess;
        if (eng_.fault_fail_rings) return cudaErrorUnknown;   // test hook (plane.h)
        if (j_.capturing) {
            for (int p : rp) CK(enqueue_captured_p2p(p));   // plan() left only CE_P2P relays
            tr_.mark("rings");
            return cudaSuccess;
        }
        if (!eng_.wait64 || !eng_.write64) return MMA_ERR_NO_MEMOPS;
        const uint32_t S = ring_slots_for(j_.C);
        std::vector<Ring*> rings(P_, nullptr);
        std::vector<uint64_t> g0(P_, 0);
        for (int p : rp) {
            CK((cudaError_t)get_ring(j_.d, j_.dir, p, j_.C, S, mode_[p] == MMA_HOP_PUSH, &rings[p]));
            g0[p] = rings[p]->g_next;
        }
        size_t maxc = 0;
        for (int p : rp) maxc = std::max(maxc, lists_[p].size());
        int rc = cudaSuccess;
        for (size_t w0 = 0; w0 < maxc && rc == cudaSuccess; w0 += S) {
            const size_t w1 = std::min<size_t>(maxc, w0 + S);
            if (j_.dir == MMA_H2D) {
                rc = wave_hops(rp, rings, g0, S, w0, w1);
                if (rc == cudaSuccess) rc = wave_kernels(rp, rings, g0, S, w0, w1);
            } else {
                rc = wave_kernels(rp, rings, g0, S, w0, w1);
                if (rc == cudaSuccess) rc = wave_hops(rp, rings, g0, S, w0, w1);
            }
        }
        if (rc != cudaSuccess) {   // flags and counters may now be out of step with g_next
            for (int p : rp) rings[p]->broken = true;
            return rc;
        }
        for (int p : rp) rings[p]->g_next = g0[p] + lists_[p].size();
        tr_.mark("rings");
        return cudaSuccess;
    }

    // chunks per hop group: small chunks are grouped up to eng_.group_bytes (at most S/2, so a
    // wave still holds two groups, one per hop stream: the dual pipeline); a chunk
    // of group_bytes or more goes alone. A group's chunks are published together when its DMA
    // ends, so large groups delay the relay's pull and the slots' reuse (measured: grouping
    // 8 MiB chunks in pairs cut a loopback kernel ring from 0.93 to 0.90 of native).
    size_t group_chunks(uint32_t S) const
    {
        const uint64_t k = eng_.group_bytes / std::max<uint64_t>(1, j_.C);
        return (size_t)std::max<uint64_t>(1, std::min<uint64_t>(k, S / 2));
    }

    // the copy-engine side of ring chunks [w0, w1) of every ring. A ring's chunks go in groups
    // (group_chunks) of consecutive chunks on consecutive slots: one DMA (or batch) and one
    // batched flag operation per group instead of per chunk -- a stream memory operation and
    // a DMA each cost microseconds of setup, which 1 MiB chunks feel. Groups are
    // issued round-robin across rings.
    int wave_hops(const std::vector<int>& rp, std::vector<Ring*>& rings, const std::vector<uint64_t>& g0,
                  uint32_t S, size_t w0, size_t w1)
    {
        const size_t k = group_chunks(S);
        std::vector<size_t> next(P_, w0);
        for (bool any = true; any;) {
            any = false;
            for (int p : rp) {
                const size_t end = std::min(lists_[p].size(), w1);
                const size_t c0 = next[p];
                if (c0 >= end) continue;
                const uint32_t s0 = (uint32_t)((g0[p] + c0) % S);
                const size_t c1 = c0 + std::min<size_t>({k, S - s0, end - c0});
                CK(ring_hops(p, rings[p], g0[p], c0, c1, S, eng_.hop_lanes > 1 ? (int)((s0 / k) & 1) : 0,
                             mode_[p] == MMA_HOP_CE_P2P));
                next[p] = c1;
                // the path's last hop-1 (H2D) / last hop-2 (D2H) DMA closes its spans; the
                // H2D forward of that chunk (one chunk over NVLink) is not attributed
                if (j_.timing && c1 == lists_[p].size()) j_.timing->end(p);
                any = true;
            }
        }
        return cudaSuccess;
    }

    // one relay kernel launch per kernel GPU for ring chunks [w0, w1) of its kernel rings
    int wave_kernels(const std::vector<int>& rp, std::vector<Ring*>& rings, const std::vector<uint64_t>& g0,
                     uint32_t S, size_t w0, size_t w1)
    {
        const uint64_t upc = (j_.C + eng_.unit_bytes - 1) / eng_.unit_bytes;
        std::map<int, RelayLaunchArg> launches;
        std::map<int, unsigned> grids;
        for (int p : rp) {
            if (mode_[p] == MMA_HOP_CE_P2P || lists_[p].size() <= w0) continue;   // no kernel
            Ring* r = rings[p];
            const size_t c1 = std::min(lists_[p].size(), w1);
            const int kd = r->kdev;
            auto& A = launches[kd];
            if (grids.find(kd) == grids.end()) {
                memset(&A, 0, sizeof(A));
                A.v = vstream_on(kd);
                A.unit_bytes = eng_.unit_bytes;
                A.log = log_;
                A.fwd = fwd_;
                A.err = eng_.err;
                A.timeout_ns = eng_.timeout_ns;
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
            R.ready = r->ready;
            R.g0 = g0[p] + w0;
            R.unit0 = r->unit_next;
            R.chunks = chunks_on(p, kd);
            R.chunks.count = c1 - w0;
            if (R.chunks.table) R.chunks.table += w0;
            else R.chunks.first += w0;
            R.S = S;
            R.path = (uint32_t)p;
            R.cta_begin = grids[kd];
            const unsigned ctas = (unsigned)std::min<uint64_t>((uint64_t)eng_.cfg.relay_ctas, R.chunks.count * upc);
            grids[kd] += ctas;
            R.cta_end = grids[kd];
            // every CTA of the ring claims until it draws one unit past the end, so the
            // cursor advances by the units plus one claim per CTA
            r->unit_next += (unsigned long long)R.chunks.count * upc + ctas;
        }
        for (auto& kv : launches) {
            const int kd = kv.first;
            cudaStream_t s = lanes(kd).kern;
            CK(make_device(kd));
            CK((cudaError_t)use(s, kd));
            DeviceGuard dg(kd);
            KTimer kt(kd, s, (j_.dir == MMA_H2D ? 1 : 2) | (j_.dir << 4) | (0xff << 8));
            TSpan ts(kd, s, j_.dir == MMA_H2D ? "relay pull kernel" : "relay pack kernel", -1, (long long)w0, 0);
            CK(launch_relay(kv.second, j_.dir == MMA_H2D, grids[kd], s, eng_.relay_bulk));
            t_.stats.kernels++;
        }
        return cudaSuccess;
    }

    // captured all-copy-engine relay: two staging slots of its own (graph allocations on the
    // relay, freed at the end of each replay), chunk c on hop stream c & 1 with slot c & 1, so
    // stream order alone keeps a slot's two uses apart -- no flags, nothing shared with live
    // rings, and every replay moves the same chunks again
    int enqueue_captured_p2p(int p)
    {
        const int r = path(p).gpu;
        Lanes& L = lanes(r);
        const uint64_t C = j_.C;
        char* slots[2] = {nullptr, nullptr};
        DeviceGuard dg(r);
        for (int k = 0; k < 2 && k < (int)lists_[p].size(); k++) {
            CK((cudaError_t)use(L.hop[k], r));
            CK(cudaMallocAsync((void**)&slots[k], C, L.hop[k]));
            captured_.push_back({r, L.hop[k], slots[k]});
        }
        for (size_t c = 0; c < lists_[p].size(); c++) {
            const int k = (int)(c & 1);
            cudaStream_t hs = L.hop[k];
            char* slot = slots[k];
            uint64_t off, len;
            j_.extent(lists_[p][c], &off, &len);
            DmaBatch in, out;
            if (j_.dir == MMA_H2D) {
                j_.pieces(off, off + len, [&](const Piece& x) { in.add(slot + (x.v - off), x.src, x.len); });
                j_.pieces(off, off + len, [&](const Piece& x) { out.add(x.dst, slot + (x.v - off), x.len); });
                if (host_order_) in.sort_by_host(cudaMemcpyHostToDevice);
                CK((cudaError_t)in.issue(cudaMemcpyHostToDevice, hs));
                CK((cudaError_t)out.issue(cudaMemcpyDeviceToDevice, hs));
            } else {
                j_.pieces(off, off + len, [&](const Piece& x) { in.add(slot + (x.v - off), x.src, x.len); });
                j_.pieces(off, off + len, [&](const Piece& x) { out.add(x.dst, slot + (x.v - off), x.len); });
                if (host_order_) out.sort_by_host(cudaMemcpyDeviceToHost);
                CK((cudaError_t)in.issue(cudaMemcpyDeviceToDevice, hs));
                CK((cudaError_t)out.issue(cudaMemcpyDeviceToHost, hs));
            }
        }
        return cudaSuccess;
    }

    // the copy-engine side of ring chunks c0..c1-1 of path p (ring index g = gbase + c, slot
    // g mod S, consecutive slots) on the relay's hop stream `lane`.
    // H2D: wait credit[s] >= g-S+1 (slot drained) -> DMA host -> slots -> publish seq[s] = g+1.
    // D2H: wait seq[s] >= g+1 (slot packed by the relay kernel) -> DMA slots -> host ->
    // release credit[s] = g+1.
    // p2p (MMA_HOP_CE_P2P): the same stream also does the other hop with a peer DMA, so the
    // slot protocol (seq / credit per slot) is the kernel ring's and the two kinds of ring may
    // follow each other on one ring. H2D: ... publish seq -> DMA slots -> target pieces ->
    // release credit. D2H: wait credit -> DMA source pieces -> slots -> publish seq -> DMA
    // slots -> host -> release credit. The delivery log is written behind the final DMA.
    int ring_hops(int p, Ring* r, uint64_t gbase, size_t c0, size_t c1, uint32_t S, int lane, bool p2p)
    {
        if (eng_.fault_fail_hop >= 0 && eng_.hops_issued++ == eng_.fault_fail_hop) return cudaErrorUnknown;   // test hook
        cudaStream_t hs = lanes(r->relay).hop[lane];
        CK((cudaError_t)use(hs, r->relay));
        CK(apply_gates(hs, r->relay));
        DeviceGuard dg(r->relay);
        auto slot_of = [&](size_t c) { return (uint32_t)((gbase + c) % S); };
        // one batched stream memory operation: wait (GEQ) or write each listed flag
        auto flags = [&](bool wait, uint64_t* base, uint64_t delta, bool credit_wait) -> int {
            CUstreamBatchMemOpParams op[64];
            unsigned n = 0;
            for (size_t c = c0; c < c1; c++) {
                const uint64_t g = gbase + c;
                if (credit_wait && g < S) continue;                        // slot never used yet
                if (!wait && base == r->seq && (long long)g == eng_.fault_drop_publish) continue;   // test hook
                const uint64_t v = credit_wait ? g - S + 1 : g + delta;
                uint64_t* addr = base + slot_of(c);
                if (!eng_.batch_memop) {
                    const CUresult e = wait ? eng_.wait64((CUstream)hs, (CUdeviceptr)addr, v, CU_STREAM_WAIT_VALUE_GEQ)
                                            : eng_.write64((CUstream)hs, (CUdeviceptr)addr, v, 0);
                    if (e != CUDA_SUCCESS) return cudaErrorUnknown;
                    continue;
                }
                memset(&op[n], 0, sizeof(op[n]));
                if (wait) {
                    op[n].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_64;
                    op[n].waitValue.address = (CUdeviceptr)addr;
                    op[n].waitValue.value64 = v;
                    op[n].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
                } else {
                    op[n].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
                    op[n].writeValue.address = (CUdeviceptr)addr;
                    op[n].writeValue.value64 = v;
                }
                n++;
            }
            if (n && eng_.batch_memop((CUstream)hs, n, op, 0) != CUDA_SUCCESS) return cudaErrorUnknown;
            return cudaSuccess;
        };
        auto dma = [&](bool to_slot, cudaMemcpyKind kind, bool host_side, const char* name) -> int {
            DmaBatch batch;
            uint64_t bytes = 0;
            for (size_t c = c0; c < c1; c++) {
                uint64_t off, len;
                j_.extent(lists_[p][c], &off, &len);
                char* slot = r->stage + (uint64_t)slot_of(c) * r->slot_bytes;
                bytes += len;
                if (to_slot) j_.pieces(off, off + len, [&](const Piece& x) { batch.add(slot + (x.v - off), x.src, x.len); });
                else j_.pieces(off, off + len, [&](const Piece& x) { batch.add(x.dst, slot + (x.v - off), x.len); });
            }
            if (host_side && host_order_) batch.sort_by_host(kind);
            TSpan ts(r->relay, hs, name, p, (long long)lists_[p][c0], bytes);
            return batch.issue(kind, hs);
        };
        if (j_.dir == MMA_H2D) {
            CK(flags(true, r->credit, 0, true));
            CK(dma(true, cudaMemcpyHostToDevice, true, "DMA hop 1: host -> relay ring"));
            CK(flags(false, r->seq, 1, false));
            if (p2p) {
                CK(dma(false, cudaMemcpyDeviceToDevice, false, "DMA hop 2: relay ring -> target (peer)"));
                CK(flags(false, r->credit, 1, false));
            }
        } else {
            if (p2p) {
                CK(flags(true, r->credit, 0, true));
                CK(dma(true, cudaMemcpyDeviceToDevice, false, "DMA hop 1: source (peer) -> relay ring"));
                CK(flags(false, r->seq, 1, false));
            } else {
                CK(flags(true, r->seq, 1, false));
            }
            CK(dma(false, cudaMemcpyDeviceToHost, true, "DMA hop 2: relay ring -> host"));
            CK(flags(false, r->credit, 1, false));
        }
        if (p2p && log_)
            for (size_t c = c0; c < c1; c++) CK(cudaMemsetAsync(log_ + lists_[p][c], p, 1, hs));
        return cudaSuccess;
    }

    // ---- join (a8): the user stream waits on every engine stream used; table buffers and
    // ledger entries are released by events on the user stream
    int join_streams()
    {
        for (auto& u : used_) {
            cudaEvent_t ev = join_event(u.first, u.second);
            {
                DeviceGuard g(u.second);
                CK(cudaEventRecord(ev, u.first));
            }
            DeviceGuard g(j_.user_dev);
            CK(cudaStreamWaitEvent(j_.user, ev, 0));
        }
        return cudaSuccess;
    }

    // this call's table buffers stay in use until the user stream passes the join
    int mark_tables_busy()
    {
        if (!tab_bytes_ || !sc_) return cudaSuccess;
        DeviceGuard g(j_.user_dev);
        if (!sc_->done || sc_->done_dev != j_.user_dev) {
            if (sc_->done) cudaEventDestroy(sc_->done);
            CK(cudaEventCreateWithFlags(&sc_->done, cudaEventDisableTiming));
            sc_->done_dev = j_.user_dev;
        }
        CK(cudaEventRecord(sc_->done, j_.user));
        sc_->pending = true;
        return cudaSuccess;
    }

    int join()
    {
        CK(join_streams());
        if (j_.capturing) {
            CK(free_captured_tables());
            tr_.mark("join");
            return cudaSuccess;
        }
        CK(mark_tables_busy());
        if (eng_.cfg.ledger && !dynamic_) {
            uint64_t lb[MMA_MAX_GPUS] = {}, lo[MMA_MAX_GPUS] = {};
            for (int p = 0; p < P_; p++) {
                const uint64_t bytes_p = path_bytes(p);
                lb[path(p).gpu] += bytes_p;
                if (path(p).kind == MMA_PATH_DIRECT) lo[path(p).gpu] += bytes_p;
            }
            CK(ledger_add(j_.dir, j_.user_dev, j_.user, lb, lo));
        }
        tr_.mark("join");
        return cudaSuccess;
    }

    // captured call: each device's graph-allocated tables are freed on its kernel stream once
    // the user stream has joined every path (fork -> free -> join, all inside the capture)
    int free_captured_tables()
    {
        cudaEvent_t done = eng_.dev[j_.user_dev].cap_ev;
        {
            DeviceGuard g(j_.user_dev);
            CK(cudaEventRecord(done, j_.user));
        }
        for (const CapturedAlloc& c : captured_) {   // staging slots, on the stream that made them
            DeviceGuard dg(c.dev);
            CK(cudaStreamWaitEvent(c.s, done, 0));
            CK(cudaFreeAsync(c.p, c.s));
            cudaEvent_t ev = join_event(c.s, c.dev);
            CK(cudaEventRecord(ev, c.s));
            DeviceGuard ug(j_.user_dev);
            CK(cudaStreamWaitEvent(j_.user, ev, 0));
        }
        for (int g = 0; g < eng_.ndev; g++) {
            if (!dtab_[g]) continue;
            cudaStream_t k = lanes(g).kern;
            DeviceGuard dg(g);
            CK(cudaStreamWaitEvent(k, done, 0));
            CK(cudaFreeAsync(dtab_[g], k));
            cudaEvent_t ev = join_event(k, g);
            CK(cudaEventRecord(ev, k));
            DeviceGuard ug(j_.user_dev);
            CK(cudaStreamWaitEvent(j_.user, ev, 0));
        }
        return cudaSuccess;
    }
};

// Enqueue one multipath copy (engine mutex held).
int run_job(Job& j)
{
    Call c(j);
    return c.run();
}

// Link id of path p of target d in a joint plan: the path GPU's own link, or for a loopback
// relay (relay GPU == target, one-GPU test mode) a virtual link MMA_MAX_GPUS + its ordinal.
static int link_of_path(const std::vector<PathState>& ps, int d, size_t p)
{
    if (ps[p].kind == MMA_PATH_DIRECT || ps[p].gpu != d) return ps[p].gpu;
    int k = 0;
    for (size_t q = 1; q < p; q++) k += ps[q].kind == MMA_PATH_RELAY && ps[q].gpu == d;
    return MMA_MAX_GPUS + k;
}

// Enqueue concurrent transfers under one joint plan (engine mutex held): per
// direction, make_plan_multi over the links of every transfer's path set (a link's rate is
// its own GPU's direct-path rate; a loopback relay's is its path's), then every call's direct
// side, then -- behind gates recorded on the direct lanes of every target GPU of the batch --
// every call's relay side, so a link finishes its own target's work before it relays
// ("direct path first", §3.4.2), as the joint plan assumed.
int run_multi(std::vector<Job>& jobs)
{
    Engine& e = E();
    const int L = MMA_MAX_GPUS + 8;
    std::vector<std::vector<uint8_t>> plans(jobs.size());
    for (int dir = 0; dir < 2; dir++) {
        std::vector<MultiLink> links(L, MultiLink{0});
        std::vector<std::vector<uint8_t>> carry(L, std::vector<uint8_t>(L, 0));
        std::vector<int> target;
        std::vector<uint64_t> nchunks;
        std::vector<size_t> idx;
        for (size_t t = 0; t < jobs.size(); t++) {
            if (jobs[t].dir != dir) continue;
            const int d = jobs[t].d;
            make_paths(d);
            const auto& ps = e.tgt[d].paths[dir];
            for (size_t p = 0; p < ps.size(); p++) {
                const int l = link_of_path(ps, d, p);
                if (l >= L || !ps[p].mbps) continue;
                if (l < MMA_MAX_GPUS) {
                    make_paths(l);
                    links[l].mbps = e.tgt[l].paths[dir][0].mbps;
                } else if (!links[l].mbps) {
                    links[l].mbps = ps[p].mbps;
                }
                carry[d][l] = 1;
            }
            target.push_back(d);
            nchunks.push_back(jobs[t].B ? (jobs[t].B - 1) / jobs[t].C + 1 : 0);
            idx.push_back(t);
        }
        if (idx.empty()) continue;
        const int mode = e.cfg.plan_mode == PLAN_INTERLEAVED ? PLAN_INTERLEAVED : PLAN_CONTIGUOUS;
        std::vector<std::vector<int>> lk;
        const int prefer = e.cfg.relay_prefer > 0 ? e.cfg.relay_prefer - 1 : -1;
        if (make_plan_multi(links, carry, target, nchunks, jobs[idx[0]].C, mode, lk, prefer)) return cudaErrorInvalidValue;
        for (size_t k = 0; k < idx.size(); k++) {
            Job& j = jobs[idx[k]];
            const auto& ps = e.tgt[j.d].paths[dir];
            auto& pl = plans[idx[k]];
            pl.resize(lk[k].size());
            for (size_t c = 0; c < lk[k].size(); c++) {
                size_t p = 0;
                while (p < ps.size() && link_of_path(ps, j.d, p) != lk[k][c]) p++;
                if (p == ps.size()) return cudaErrorInvalidValue;
                pl[c] = (uint8_t)p;
            }
            j.plan_override = &pl;
            j.interleaved_plan = mode == PLAN_INTERLEAVED;
        }
    }
    for (size_t t = 0; t < jobs.size(); t++)   // one delivery log per GPU: the last transfer's
        for (size_t u = t + 1; u < jobs.size(); u++) jobs[t].no_log |= jobs[u].d == jobs[t].d;
    std::vector<std::unique_ptr<Call>> calls;
    for (Job& j : jobs) calls.emplace_back(new Call(j));
    std::vector<int> rc(jobs.size(), cudaSuccess);
    for (size_t t = 0; t < calls.size(); t++) {
        rc[t] = calls[t]->begin();
        if (rc[t] == cudaSuccess && !calls[t]->done()) rc[t] = calls[t]->enqueue_side(false);
    }
    for (size_t t = 0; t < jobs.size(); t++)   // every target's own work, per direction
        if (rc[t] == cudaSuccess && !calls[t]->done()) {
            const int r = record_gates(jobs[t].d, jobs[t].dir);
            if (r != cudaSuccess) rc[t] = r;
        }
    for (size_t t = 0; t < calls.size(); t++) {
        if (calls[t]->done()) continue;
        if (rc[t] == cudaSuccess) {
            for (size_t u = 0; u < jobs.size(); u++)
                if (jobs[u].dir == jobs[t].dir)
                    for (cudaEvent_t ev : e.dev[jobs[u].d].gate_ev[jobs[u].dir]) calls[t]->gate(jobs[u].d, ev);
            rc[t] = calls[t]->enqueue_side(true);
        }
        if (rc[t] != cudaSuccess && !calls[t]->forked()) continue;
        rc[t] = calls[t]->end(rc[t]);
    }
    for (int r : rc)
        if (r != cudaSuccess) return r;
    return cudaSuccess;
}

int sticky()
{
    Engine& e = E();
    if (e.err && *(volatile int*)e.err) return MMA_ERR_RELAY_TIMEOUT;
    return cudaSuccess;
}

}  // namespace mma
