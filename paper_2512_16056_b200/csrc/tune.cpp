// tune.cpp — "chosen per path by measurement" (north_star (d)): time
// every path alone in each hop mode and keep the faster mode and its rate for the planner.
#include "plane.h"

namespace mma {

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

}  // extern "C"
