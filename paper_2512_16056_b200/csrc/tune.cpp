// tune.cpp — "chosen per path by measurement" (north_star (d)): time
// every path alone in each hop mode and keep the faster mode; then measure every path's rate
// with all paths of the set active (a0) and keep that rate for the planner.
#include "plane.h"

namespace mma {

// ---- per-path timing spans (Job::timing) ---------------------------------------------

PathTiming::~PathTiming()
{
    for (auto& v : path)
        for (auto& sp : v) {
            DeviceGuard g(sp.dev);
            if (sp.a) cudaEventDestroy(sp.a);
            if (sp.b) cudaEventDestroy(sp.b);
        }
}

void PathTiming::start(int p, int dev, cudaStream_t s)
{
    for (auto& sp : path[p])
        if (sp.s == s) return;
    Span sp{dev, s, nullptr, nullptr};
    DeviceGuard g(dev);
    if (cudaEventCreate(&sp.a) != cudaSuccess) { cudaGetLastError(); return; }
    cudaEventRecord(sp.a, s);
    path[p].push_back(sp);
}

void PathTiming::end(int p)
{
    for (auto& sp : path[p]) {
        if (sp.b) continue;
        DeviceGuard g(sp.dev);
        if (cudaEventCreate(&sp.b) != cudaSuccess) { cudaGetLastError(); continue; }
        cudaEventRecord(sp.b, sp.s);
    }
}

int PathTiming::collect(std::vector<float>& ms)
{
    ms.assign(path.size(), 0.f);
    for (size_t p = 0; p < path.size(); p++)
        for (auto& sp : path[p]) {
            if (!sp.a || !sp.b) continue;
            DeviceGuard g(sp.dev);
            CK(cudaEventSynchronize(sp.b));
            float t = 0.f;
            CK(cudaEventElapsedTime(&t, sp.a, sp.b));
            ms[p] = std::max(ms[p], t);
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
    CK(reserve_tables(proto));
    cudaEvent_t a = nullptr, b = nullptr;
    {
        DeviceGuard g(proto.user_dev);
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
    }
    int rc = cudaSuccess;
    for (int p = 0; p < P && rc == cudaSuccess; p++) {
        // candidates in order of SM use: a relay's all-copy-engine ring uses none, the kernel
        // ring the relay kernel, zero-copy its own grid; a later candidate must win by 2%
        const bool relay = ps[p].kind == MMA_PATH_RELAY;
        std::vector<int> cands;
        if (relay) cands.push_back(MMA_HOP_CE_P2P);
        cands.push_back(MMA_HOP_CE);
        if (relay) cands.push_back(MMA_HOP_PUSH);
        if (proto.mapped) cands.push_back(MMA_HOP_ZC);
        // zero-copy is measured first: a copy-engine candidate whose warm-up run's host issue
        // alone (x P, see above) bounds it below 0.8 of the zero-copy rate cannot be chosen,
        // so its timed runs are skipped -- a scattered table costs the copy engine one DMA per
        // piece (~5 us each since the batched API closed, DESIGN §5 item 11), i.e. seconds per
        // candidate run at config-3 size. The choice itself is made below in SM-use order.
        std::vector<float> rate_of(cands.size(), 0.f);
        std::vector<size_t> order;
        for (size_t c = 0; c < cands.size(); c++)
            if (cands[c] == MMA_HOP_ZC) order.push_back(c);
        for (size_t c = 0; c < cands.size(); c++)
            if (cands[c] != MMA_HOP_ZC) order.push_back(c);
        float zc_rate = 0.f;
        for (size_t c : order) {
            const int m = cands[c];
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
                // (only a long issue counts: a first use may spend a few ms creating the ring)
                if (rep == 0 && m != MMA_HOP_ZC && zc_rate > 0.f && issue_ms >= 50.f) {
                    const double bound = (double)proto.B / ((double)issue_ms * P * 1e-3) / 1e6;
                    if (bound < 0.8 * zc_rate) break;                // cannot win: skip the timed runs
                }
            }
            const float eff_ms = std::max(best, best_issue * (float)P);
            rate_of[c] = best < 1e29f ? (float)((double)proto.B / (eff_ms * 1e-3) / 1e6) : 0.f;
            if (m == MMA_HOP_ZC) zc_rate = rate_of[c];
        }
        float best_rate = 0.f;
        for (size_t c = 0; c < cands.size(); c++) {
            // a candidate that uses more SMs must win by 2%: on a near-tie the path keeps its SMs
            // free (§3.4.3) and the run-to-run noise of one timed call cannot flip it
            if (rate_of[c] > best_rate * (best_rate > 0.f ? 1.02f : 1.0f)) {
                best_rate = rate_of[c];
                modes[p] = cands[c];
                mbps[p] = (uint32_t)llround(rate_of[c]);
            }
        }
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (rc == cudaSuccess && sticky()) rc = sticky();
    return rc;
}

// Concurrent refinement (bw[p] "measured with all paths of the set
// active"). Starting from the solo vector, run the transfer `rounds` times with every path
// active, planned from the current vector (same modes); a path's new rate is the bytes the
// plan gave it over the longest of its own stream spans (best of `reps`). Paths that get no
// chunk keep their rate (conc = 0 in the evidence). A link that shares DRAM, a switch uplink
// or a socket link with others thus enters the planner at the rate it actually gets. The
// iteration moves toward equal finish times, where every path is busy for the whole call
// and the measured rates are the concurrent ones.
static int refine_concurrent(Job proto, int rounds, int reps, std::vector<uint32_t>& mbps,
                             const std::vector<int>& modes, std::vector<uint32_t>& conc)
{
    const int P = (int)mbps.size();
    conc.assign(P, 0);
    int active = 0;
    for (int p = 0; p < P; p++) active += mbps[p] > 0;
    if (active < 2 || rounds <= 0) return cudaSuccess;
    int rc = cudaSuccess;
    for (int r = 0; r < rounds && rc == cudaSuccess; r++) {
        std::vector<float> best(P, 0.f);
        std::vector<uint64_t> bytes(P, 0);
        for (int rep = 0; rep <= reps && rc == cudaSuccess; rep++) {
            Job j = proto;
            j.bw_override = mbps.data();
            j.mode_override = modes.data();
            j.no_small_fallback = true;
            PathTiming pt(P);
            j.timing = &pt;
            {
                DeviceGuard g(j.user_dev);
                rc = run_job(j);
            }
            if (rc != cudaSuccess) break;
            std::vector<float> ms;
            rc = pt.collect(ms);
            if (rc != cudaSuccess || rep == 0) continue;   // rep 0 warms up
            for (int p = 0; p < P; p++)
                if (ms[p] > 0.f && (best[p] == 0.f || ms[p] < best[p])) best[p] = ms[p];
            bytes = pt.bytes;
        }
        if (rc != cudaSuccess) break;
        for (int p = 0; p < P; p++) {
            if (!bytes[p] || best[p] <= 0.f) { conc[p] = 0; continue; }
            const long long v = llround((double)bytes[p] / ((double)best[p] * 1e-3) / 1e6);
            conc[p] = (uint32_t)std::max(1ll, v);
            mbps[p] = conc[p];
        }
    }
    {
        DeviceGuard g(proto.user_dev);
        if (rc == cudaSuccess && cudaStreamSynchronize(proto.user) != cudaSuccess) rc = cudaErrorUnknown;
    }
    if (rc == cudaSuccess && sticky()) rc = sticky();
    return rc;
}

// Solo mode choice, then the concurrent refinement; results stored for contiguous (k = 0)
// or scattered (k = 1) transfers.
static int calibrate_job(Job& j, int reps, int k)
{
    Engine& e = E();
    std::vector<uint32_t> mbps, conc;
    std::vector<int> modes;
    CK(tune_paths(j, reps, mbps, modes));
    std::vector<uint32_t> solo = mbps;
    CK(refine_concurrent(j, e.cfg.calib_rounds, reps, mbps, modes, conc));
    auto& ps = e.tgt[j.d].paths[j.dir];
    for (size_t p = 0; p < ps.size(); p++) {
        if (!mbps[p]) continue;
        if (k == 0) { ps[p].mbps = mbps[p]; ps[p].mode = modes[p]; }
        else { ps[p].seg_mbps = mbps[p]; ps[p].seg_mode = modes[p]; }
        ps[p].solo_mbps[k] = solo[p];
        ps[p].conc_mbps[k] = conc[p];
    }
    return cudaSuccess;
}

// Library-owned buffers for a contiguous measurement transfer of `bytes` to/from `device`:
// pinned mapped host memory, device memory and a private stream; freed on scope exit.
struct CalBuffers {
    int dev;
    char* h = nullptr;
    char* d = nullptr;
    cudaStream_t s = nullptr;
    int rc = cudaSuccess;
    CalBuffers(int device, size_t bytes) : dev(device)
    {
        DeviceGuard g(dev);
        if ((rc = cudaHostAlloc((void**)&h, bytes, cudaHostAllocPortable | cudaHostAllocMapped))) return;
        if ((rc = cudaMalloc((void**)&d, bytes))) return;
        rc = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    }
    ~CalBuffers()
    {
        DeviceGuard g(dev);
        if (s) cudaStreamDestroy(s);
        if (d) cudaFree(d);
        if (h) cudaFreeHost(h);
    }
    Job job(int dir, size_t bytes) const
    {
        Job j;
        j.dir = dir;
        j.d = dev;
        j.user = s;
        j.user_dev = dev;
        j.B = bytes;
        j.C = E().cfg.chunk_bytes[dir];
        j.src0 = dir == MMA_H2D ? h : d;
        j.dst0 = dir == MMA_H2D ? d : h;
        j.mapped = true;
        return j;
    }
};

}  // namespace mma

using namespace mma;

extern "C" {

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
    CalBuffers cb(device, bytes);
    CK(cb.rc);
    Job j = cb.job(dir, bytes);
    return calibrate_job(j, 3, 0);
}

// Chunk size by measurement (§3.4.1: the Task Manager "dynamically adjusts" the chunk
// size; P:902 tuned optima 2.81 / 5.37 MB on H20; reading R3). Each candidate C in
// {1, 2, 4, 8, 16, 32} MiB not above bytes / 2 is timed on a contiguous copy of `bytes` with
// the current vector and modes (best of 3 after a warm-up); the fastest is kept, a smaller
// chunk only when it is >= 1% faster (fewer DMAs, memops and flags per byte otherwise).
int mma_tune_chunk(int device, mma_dir_t dir, size_t bytes, size_t* chunk_out)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    if ((dir != MMA_H2D && dir != MMA_D2H) || bytes < (2u << 20)) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> g(e.mu);
    CK(make_device(device));
    make_paths(device);
    DeviceGuard dg(device);
    CalBuffers cb(device, bytes);
    CK(cb.rc);
    cudaEvent_t a = nullptr, b = nullptr;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const size_t keep = e.cfg.chunk_bytes[dir];
    size_t best_c = keep;
    float best_ms = 1e30f;
    int rc = cudaSuccess;
    for (size_t C = 32u << 20; C >= (1u << 20) && rc == cudaSuccess; C >>= 1) {   // large first
        if (C > bytes / 2) continue;
        e.cfg.chunk_bytes[dir] = C;
        Job proto = cb.job(dir, bytes);
        if ((rc = reserve_tables(proto)) != cudaSuccess) break;
        float best = 1e30f;
        for (int rep = 0; rep <= 3 && rc == cudaSuccess; rep++) {
            Job j = cb.job(dir, bytes);
            j.no_small_fallback = true;
            cudaEventRecord(a, cb.s);
            rc = run_job(j);
            cudaEventRecord(b, cb.s);
            if (rc == cudaSuccess && cudaEventSynchronize(b) != cudaSuccess) rc = cudaErrorUnknown;
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            if (rep > 0 && ms > 0) best = std::min(best, ms);
        }
        if (best < best_ms * 0.99f) {
            best_ms = best;
            best_c = C;
        }
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (rc == cudaSuccess && sticky()) rc = sticky();
    e.cfg.chunk_bytes[dir] = rc == cudaSuccess ? best_c : keep;
    if (chunk_out) *chunk_out = e.cfg.chunk_bytes[dir];
    return rc;
}

// Break-even ("thr defaults to the measured B200 break-even"; the paper's
// 11.3 MB H2D / 13 MB D2H on H20, §5.1.3). Sizes C, 2C, 4C, ... up to max_bytes: each
// is timed as the native copy on one stream and as the multipath copy with the current
// vector and modes (best of 5 after a warm-up, CUDA events). The threshold becomes the
// smallest swept size from which every larger swept size is at least 3% faster by
// multipath. When even the largest is not, no break-even exists up to max_bytes and the
// threshold is left as it was (*found = 0): the path set, not the size, is the problem then,
// and a direct path in zero-copy mode must still serve large scattered copies.
int mma_tune_threshold(int device, mma_dir_t dir, size_t max_bytes, size_t* thr_out, int* found)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    if ((dir != MMA_H2D && dir != MMA_D2H) || max_bytes == 0) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> g(e.mu);
    CK(make_device(device));
    make_paths(device);
    DeviceGuard dg(device);
    const uint64_t C = e.cfg.chunk_bytes[dir];
    if (max_bytes < C) max_bytes = C;
    {   // a set whose only usable path is the direct one has nothing to gain: no break-even
        const auto& ps = e.tgt[device].paths[dir];
        int usable = 0;
        for (const PathState& q : ps) usable += q.mbps > 0;
        if (usable < 2) {
            if (thr_out) *thr_out = e.cfg.fallback_bytes[dir];
            if (found) *found = 0;
            return cudaSuccess;
        }
    }
    CalBuffers cb(device, max_bytes);
    CK(cb.rc);
    CK(reserve_tables(cb.job(dir, max_bytes)));
    cudaEvent_t a = nullptr, b = nullptr;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const cudaMemcpyKind kind = dir == MMA_H2D ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
    std::vector<uint64_t> sizes;
    std::vector<char> faster;
    int rc = cudaSuccess;
    for (uint64_t B = C; B <= max_bytes && rc == cudaSuccess; B *= 2) {
        float best[2] = {1e30f, 1e30f};
        for (int how = 0; how < 2 && rc == cudaSuccess; how++)
            for (int rep = 0; rep <= 5 && rc == cudaSuccess; rep++) {
                cudaEventRecord(a, cb.s);
                if (how == 0) {
                    rc = cudaMemcpyAsync(dir == MMA_H2D ? cb.d : cb.h, dir == MMA_H2D ? cb.h : cb.d, B, kind, cb.s);
                } else {
                    Job j = cb.job(dir, B);
                    j.no_small_fallback = true;
                    rc = run_job(j);
                }
                cudaEventRecord(b, cb.s);
                if (rc == cudaSuccess && cudaEventSynchronize(b) != cudaSuccess) rc = cudaErrorUnknown;
                float ms = 0;
                cudaEventElapsedTime(&ms, a, b);
                if (rep > 0 && ms > 0) best[how] = std::min(best[how], ms);
            }
        sizes.push_back(B);
        faster.push_back(best[1] < 0.97f * best[0]);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (rc == cudaSuccess && sticky()) rc = sticky();
    if (rc != cudaSuccess) return rc;
    // the smallest size from which every larger swept size wins; at least two winning sizes
    // (one timed point alone cannot tell a break-even from noise)
    size_t thr = 0;
    int wins = 0;
    for (size_t k = sizes.size(); k-- > 0;) {
        if (!faster[k]) break;
        thr = sizes[k];
        wins++;
    }
    const bool any = wins >= 2 || (wins == 1 && sizes.size() == 1);
    if (any) e.cfg.fallback_bytes[dir] = thr;
    if (thr_out) *thr_out = e.cfg.fallback_bytes[dir];
    if (found) *found = any ? 1 : 0;
    return cudaSuccess;
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
    if (j.pageable) return cudaErrorInvalidValue;   // tuning measures pinned transfers only
    std::lock_guard<std::mutex> g(e.mu);
    CK(make_device(device));
    make_paths(device);
    return calibrate_job(j, reps, 1);
}

int mma_get_calibration(int device, mma_dir_t dir, int scattered, uint32_t* solo_mbps,
                        uint32_t* conc_mbps, int cap, int* npaths)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    if ((dir != MMA_H2D && dir != MMA_D2H) || !npaths || cap < 0) return cudaErrorInvalidValue;
    const int k = scattered ? 1 : 0;
    std::lock_guard<std::mutex> g(e.mu);
    make_paths(device);
    auto& ps = e.tgt[device].paths[dir];
    *npaths = (int)ps.size();
    for (int i = 0; i < (int)ps.size() && i < cap; i++) {
        if (solo_mbps) solo_mbps[i] = ps[i].solo_mbps[k];
        if (conc_mbps) conc_mbps[i] = ps[i].conc_mbps[k];
    }
    return cudaSuccess;
}

}  // extern "C"
