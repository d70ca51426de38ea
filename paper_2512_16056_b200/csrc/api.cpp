// api.cpp — C7: the C ABI of include/mma.h (validation, fallback decisions, pointer
// classification) over the data plane in plane.cpp. Every function returns a cudaError_t
// value as int; validation happens before anything is enqueued.
#include <unistd.h>

#include <cctype>
#include <string>

#include "plane.h"
#include "ranges.h"

namespace mma {

// ------------------------------------------------------------- classification ---


static int stream_device(cudaStream_t s, int* dev)
{
    // cudaStreamGetDevice invalidates a capture in progress on s (either capture mode,
    // profiles/r01_probe_capture_calls.txt): a capturing stream is taken to be on the
    // current device, where torch.cuda.graph and cudaStreamBeginCapture users create it
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone) return cudaGetDevice(dev);
    cudaGetLastError();
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

// Memory-kind query behind the per-call range cache (ranges.h): cudaPointerGetAttributes for
// the kind, the driver's RANGE_START_ADDR / RANGE_SIZE for the allocation's bounds.
using PFN_ptrattrs = CUresult (*)(unsigned, CUpointer_attribute*, void**, CUdeviceptr);

static PFN_ptrattrs ptr_attrs()
{
    static PFN_ptrattrs fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuPointerGetAttributes", &f, 12000, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            f = nullptr;
        }
        return (PFN_ptrattrs)f;
    }();
    return fn;
}

static MemRange query_range(uintptr_t p, uintptr_t end, void*)
{
    MemRange r{p, end, MK_PAGEABLE, -1, false};
    r.kind = classify((const void*)p, &r.dev, &r.mapped);
    CUdeviceptr start = 0;
    size_t size = 0;
    CUpointer_attribute at[2] = {CU_POINTER_ATTRIBUTE_RANGE_START_ADDR, CU_POINTER_ATTRIBUTE_RANGE_SIZE};
    void* data[2] = {&start, &size};
    if (PFN_ptrattrs f = ptr_attrs(); f && r.kind != MK_PAGEABLE)
        if (f(2, at, data, (CUdeviceptr)p) == CUDA_SUCCESS && size && start <= p && p < start + size) {
            r.lo = (uintptr_t)start;
            r.hi = (uintptr_t)start + size;
            return r;
        }
    if (end - p > 1) {   // no bounds (pageable, or none reported): both ends of the piece must agree
        int dev2 = -1;
        bool m2 = false;
        const int k2 = classify((const void*)(end - 1), &dev2, &m2);
        if (k2 != r.kind || dev2 != r.dev) r.kind = MK_MIXED;
        r.mapped = r.mapped && m2;
    }
    return r;
}

// Capture status of the user stream. A captured call may not initialise anything (the
// engine, a device's streams, the graph arena): those are made by an uncaptured call first,
// else the copy is the native one. Returns 1 = capture the multipath copy, 0 = not
// capturing, -1 = capturing but not ready (native copy).
static int capture_state(cudaStream_t stream, int d)
{
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    unsigned long long id = 0;
    if (cudaStreamGetCaptureInfo(stream, &cap, &id) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    if (cap == cudaStreamCaptureStatusNone) return 0;
    if (cap != cudaStreamCaptureStatusActive) return -1;
    Engine& e = E();
    if (!e.inited || !e.arena || d < 0 || d >= e.ndev || !e.tgt[d].paths_made) return -1;
    make_paths(d);
    for (int dir = 0; dir < 2; dir++)
        for (const PathState& p : e.tgt[d].paths[dir]) {
            const DevRes& r = e.dev[p.gpu];
            if (!r.made) return -1;
            // another capture still holds the capture lanes (its user has not ended it yet):
            // joining them would tie the two graphs together. Lanes already in THIS capture
            // (an earlier call of the same graph) are fine.
            for (const Lanes& l : r.cap_lane)
                for (cudaStream_t s : {l.kern, l.hop[0], l.hop[1], l.direct, l.zc}) {
                    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
                    unsigned long long lid = 0;
                    if (cudaStreamGetCaptureInfo(s, &st, &lid) != cudaSuccess) {
                        cudaGetLastError();
                        return -1;
                    }
                    if (st != cudaStreamCaptureStatusNone && lid != id) return -1;
                }
        }
    return 1;
}

static int copy_contiguous(int dir, void* dst, const void* src, size_t bytes, cudaStream_t stream)
{
    {   // the first call of a process must not initialise inside a capture
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        if (!E().inited && cudaStreamIsCapturing(stream, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone)
            return (int)cudaMemcpyAsync(dst, src, bytes, dir == MMA_H2D ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
                                        stream);
        cudaGetLastError();
    }
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
    if (hk == 2 || d >= e.ndev) return (int)cudaMemcpyAsync(dst, src, bytes, kind, stream);   // native (R7)
    std::lock_guard<std::mutex> g(e.mu);
    const int cs = capture_state(stream, d);
    if (cs < 0) return (int)cudaMemcpyAsync(dst, src, bytes, kind, stream);   // native (R7)
    Job j;
    j.capturing = cs == 1;
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
    if (!j.capturing) CK((cudaError_t)make_device(d));
    return run_job(j);
}

// Validate a segment table and fill the job (no engine lock held).
int prepare_segments(int dir, const mma_segment_t* segs, size_t nsegs, int device,
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
    // every segment's memory kind, through a per-call cache of the allocations seen so far
    // (a few driver queries per call; one per segment only for memory CUDA does not know)
    const auto v0 = std::chrono::steady_clock::now();
    RangeCache hc(query_range, nullptr), dc(query_range, nullptr);
    j.mapped = true;
    j.pageable = false;
    for (size_t k = 0; k < nsegs; k++) {
        if (!segs[k].bytes) continue;
        const void* dp = (dir == MMA_H2D) ? segs[k].dst : segs[k].src;
        const void* hp = (dir == MMA_H2D) ? segs[k].src : segs[k].dst;
        int d = -1;
        bool m = false;
        if (dc.kind((uintptr_t)dp, segs[k].bytes, &d, &m) != MK_DEVICE || d != phys_dev(device)) return cudaErrorInvalidValue;
        const int hk = hc.kind((uintptr_t)hp, segs[k].bytes, &d, &m);
        if (hk == MK_DEVICE || hk == MK_MIXED) return cudaErrorInvalidValue;
        if (hk == MK_PAGEABLE) {   // pageable or unregistered: the whole table goes native (R7)
            j.pageable = true;
            break;
        }
        j.mapped = j.mapped && m;
    }
    j.validate_us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - v0).count();
    j.ptr_queries = hc.queries() + dc.queries();
    if (nsegs == 1) {   // one segment is a contiguous copy (the kernels' nseg == 1 form)
        j.contiguous = true;
        j.src0 = (const char*)segs[0].src;
        j.dst0 = (char*)segs[0].dst;
    }
    return cudaSuccess;
}

// the native form of a segment table: one cudaMemcpyAsync per segment (capturable)
static int native_segments(int dir, const mma_segment_t* segs, size_t nsegs, cudaStream_t stream)
{
    const cudaMemcpyKind kind = dir == MMA_H2D ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost;
    for (size_t k = 0; k < nsegs; k++)
        if (segs[k].bytes) CK(cudaMemcpyAsync(segs[k].dst, segs[k].src, segs[k].bytes, kind, stream));
    return cudaSuccess;
}

static int copy_segments(int dir, const mma_segment_t* segs, size_t nsegs, int device, cudaStream_t stream)
{
    {   // the first call of a process must not initialise inside a capture
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        if (!E().inited && cudaStreamIsCapturing(stream, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone)
            return (nsegs && !segs) ? cudaErrorInvalidValue : native_segments(dir, segs, nsegs, stream);
        cudaGetLastError();
    }
    CK((cudaError_t)ensure_init());
    if (int se = sticky()) return se;
    Engine& e = E();
    if (nsegs == 0) return cudaSuccess;
    if (!segs) return cudaErrorInvalidValue;
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    Job j;
    CK(prepare_segments(dir, segs, nsegs, device, stream, j));
    if (j.B == 0) return cudaSuccess;
    if (j.pageable) {   // some host segment is not page-locked: the native copy (R7)
        std::lock_guard<std::mutex> g(e.mu);
        e.tgt[device].stats.fallbacks++;
        e.tgt[device].stats.calls++;
        e.tgt[device].stats.bytes += j.B;
        e.tgt[device].stats.validate_us += j.validate_us;
        e.tgt[device].stats.ptr_queries += j.ptr_queries;
        return native_segments(dir, segs, nsegs, stream);
    }
    std::lock_guard<std::mutex> g(e.mu);
    const int cs = capture_state(stream, device);
    if (cs < 0) return native_segments(dir, segs, nsegs, stream);
    j.capturing = cs == 1;
    if (!j.capturing) CK((cudaError_t)make_device(device));
    return run_job(j);
}

// (engine mutex held)
int load_calibration_locked(const char* path, int* applied)
{
    if (!path) return cudaErrorInvalidValue;
    Engine& e = E();
    FILE* f = fopen(path, "r");
    if (!f) return cudaErrorInvalidValue;
    char line[256];
    int n = 0;
    while (fgets(line, sizeof line, f)) {
        if (line[0] == '#') continue;
        int d, dir, gpu, kind, mode, seg_mode;
        size_t p;
        unsigned mbps, seg_mbps;
        if (sscanf(line, "%d %d %zu %d %d %u %d %u %d", &d, &dir, &p, &gpu, &kind, &mbps, &mode, &seg_mbps, &seg_mode) != 9)
            continue;
        if (d < 0 || d >= e.ndev || dir < 0 || dir > 1 || mode < MMA_HOP_AUTO || mode > MMA_HOP_PUSH ||
            seg_mode < -1 || seg_mode > MMA_HOP_PUSH)
            continue;
        make_paths(d);
        auto& ps = e.tgt[d].paths[dir];
        if (p >= ps.size() || ps[p].gpu != gpu || ps[p].kind != kind) continue;
        ps[p].mbps = mbps ? mbps : ps[p].mbps;
        ps[p].mode = mode;
        ps[p].seg_mbps = seg_mbps;
        ps[p].seg_mode = seg_mode;
        n++;
    }
    fclose(f);
    if (applied) *applied = n;
    return cudaSuccess;
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
    mp_finalize();
    for (int d = 0; d < e.ndev; d++) {
        Target& t = e.tgt[d];
        for (int dir = 0; dir < 2; dir++)
            for (int p = 0; p < MMA_MAX_PATHS; p++) free_ring(t.rings[dir][p]);
        if (t.log) { DeviceGuard dg(d); cudaFree(t.log); }
        if (t.dyn) { DeviceGuard dg(d); cudaFree(t.dyn); }
        if (t.fwd) { DeviceGuard dg(d); cudaFree(t.fwd); }
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
    ledger_retire();   // every call has completed: their bytes leave the (shared) ledger
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
        for (Lanes* ls : {r.lane, r.cap_lane})
            for (int k = 0; k < 2; k++) {
                cudaStreamDestroy(ls[k].kern);
                cudaStreamDestroy(ls[k].hop[0]);
                cudaStreamDestroy(ls[k].hop[1]);
                cudaStreamDestroy(ls[k].direct);
                cudaStreamDestroy(ls[k].zc);
            }
        cudaEventDestroy(r.cap_fork);
        for (cudaEvent_t ev : r.fork_pool) cudaEventDestroy(ev);
        for (auto& gd : r.gate_ev)
            for (cudaEvent_t ev : gd) cudaEventDestroy(ev);
        cudaEventDestroy(r.cap_ev);
        cudaStreamDestroy(r.setup);
        r = DevRes();
    }
    if (e.err) { cudaFreeHost(e.err); e.err = nullptr; }
    if (e.arena) { cudaFreeHost(e.arena); e.arena = nullptr; }   // graphs with captured copies die with it
    e.arena_used = e.arena_cap = 0;
    e.inited = false;
    return cudaSuccess;
}

int mma_order_by_address(const uint64_t* addr, size_t n, uint32_t* perm)
{
    if ((n && (!addr || !perm)) || n > 0xffffffffull) return cudaErrorInvalidValue;
    std::vector<uint32_t> p;
    order_by_key(addr, n, p);
    if (n) memcpy(perm, p.data(), n * sizeof(uint32_t));
    return cudaSuccess;
}

int mma_get_topology(mma_topology_t* out)
{
    if (!out) return cudaErrorInvalidValue;
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    memset(out, 0, sizeof(*out));
    out->ngpu = e.ndev;
    for (int a = 0; a < e.ndev; a++) {
        for (int b = 0; b < e.ndev; b++) out->p2p[a][b] = e.p2p[a][b] ? 1 : 0;
        const int pa = phys_dev(a);   // a virtual GPU (MMA_VGPUS) reports its device's values
        CK(cudaDeviceGetAttribute(&out->copy_engines[a], cudaDevAttrAsyncEngineCount, pa));
        CK(cudaDeviceGetAttribute(&out->sms[a], cudaDevAttrMultiProcessorCount, pa));
        CK(cudaDeviceGetPCIBusId(out->bus_id[a], sizeof out->bus_id[a], pa));
        out->numa_node[a] = gpu_numa_node(a);
    }
    for (int i = 0; i < 256; i++) {
        char p[96];
        snprintf(p, sizeof p, "/sys/devices/system/node/node%d", i);
        if (access(p, F_OK) == 0) out->host_numa_nodes = i + 1;
    }
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

int mma_memcpy_multi(const mma_transfer_t* xf, size_t n)
{
    CK((cudaError_t)ensure_init());
    if (int se = sticky()) return se;
    if (n == 0) return cudaSuccess;
    if (!xf) return cudaErrorInvalidValue;
    Engine& e = E();
    std::vector<Job> jobs;
    jobs.reserve(n);
    std::vector<size_t> single;   // copied on their own: native (pageable, small) or capturing
    for (size_t k = 0; k < n; k++) {   // validate everything before anything is enqueued
        const mma_transfer_t& x = xf[k];
        if (x.dir != MMA_H2D && x.dir != MMA_D2H) return cudaErrorInvalidValue;
        if (x.device < 0 || x.device >= e.ndev) return cudaErrorInvalidDevice;
        if (x.nsegs && !x.segs) return cudaErrorInvalidValue;
        if (!x.nsegs) continue;
        cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing((cudaStream_t)x.stream, &cap) != cudaSuccess) cudaGetLastError();
        Job j;
        CK(prepare_segments(x.dir, x.segs, x.nsegs, x.device, (cudaStream_t)x.stream, j));
        if (j.B == 0) continue;
        if (cap != cudaStreamCaptureStatusNone || j.pageable || j.B < e.cfg.fallback_bytes[x.dir]) {
            single.push_back(k);
            continue;
        }
        jobs.push_back(std::move(j));
    }
    for (size_t k : single) {   // the ordinary single-transfer path (it takes the engine lock)
        const mma_transfer_t& x = xf[k];
        CK(copy_segments(x.dir, x.segs, x.nsegs, x.device, (cudaStream_t)x.stream));
    }
    if (jobs.empty()) return cudaSuccess;
    std::lock_guard<std::mutex> g(e.mu);
    for (Job& j : jobs) CK((cudaError_t)make_device(j.d));
    return run_multi(jobs);
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

// Calibration file (SURVEY §5 "checkpoint / resume": only the calibration persists): one
// line per (device, direction, path): device dir path gpu kind mbps mode seg_mbps seg_mode.
// Loading applies a line only where the current path set has the same (gpu, kind) at that
// index, so a file from another topology is ignored path by path, never misapplied.
int mma_save_calibration(const char* path)
{
    CK((cudaError_t)ensure_init());
    if (!path) return cudaErrorInvalidValue;
    Engine& e = E();
    std::lock_guard<std::mutex> g(e.mu);
    FILE* f = fopen(path, "w");
    if (!f) return cudaErrorInvalidValue;
    fprintf(f, "# mma calibration v1: device dir path gpu kind mbps mode seg_mbps seg_mode\n");
    for (int d = 0; d < e.ndev; d++) {
        make_paths(d);
        for (int dir = 0; dir < 2; dir++) {
            const auto& ps = e.tgt[d].paths[dir];
            for (size_t p = 0; p < ps.size(); p++)
                fprintf(f, "%d %d %zu %d %d %u %d %u %d\n", d, dir, p, ps[p].gpu, ps[p].kind, ps[p].mbps,
                        ps[p].mode, ps[p].seg_mbps, ps[p].seg_mode);
        }
    }
    fclose(f);
    return cudaSuccess;
}

int mma_load_calibration(const char* path, int* applied)
{
    CK((cudaError_t)ensure_init());
    std::lock_guard<std::mutex> g(E().mu);
    return load_calibration_locked(path, applied);
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
        if (modes[i] < MMA_HOP_AUTO || modes[i] > MMA_HOP_PUSH) return cudaErrorInvalidValue;
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

int mma_plan_multi(int nlinks, const uint32_t* link_mbps, const uint8_t* carry, int ntransfers,
                   const int* target, const uint64_t* nchunks, uint64_t chunk_bytes, int mode,
                   int prefer, int32_t* link_of_chunk)
{
    if (nlinks < 1 || nlinks > 128 || ntransfers < 0 || !link_mbps || !carry ||
        (ntransfers && (!target || !nchunks || !link_of_chunk)))
        return cudaErrorInvalidValue;
    std::vector<MultiLink> links(nlinks);
    std::vector<std::vector<uint8_t>> ok(nlinks, std::vector<uint8_t>(nlinks));
    for (int l = 0; l < nlinks; l++) links[l].mbps = link_mbps[l];
    for (int d = 0; d < nlinks; d++)
        for (int l = 0; l < nlinks; l++) ok[d][l] = carry[(size_t)d * nlinks + l];
    std::vector<int> tg(target, target + ntransfers);
    std::vector<uint64_t> nc(nchunks, nchunks + ntransfers);
    std::vector<std::vector<int>> out;
    if (make_plan_multi(links, ok, tg, nc, chunk_bytes, mode, out, prefer)) return cudaErrorInvalidValue;
    size_t i = 0;
    for (const auto& v : out)
        for (int l : v) link_of_chunk[i++] = l;
    return cudaSuccess;
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

int mma_get_forward_log(int device, uint64_t* observed, uint64_t* expected, size_t cap, size_t* nchunks)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    if (!nchunks) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> g(e.mu);
    Target& t = e.tgt[device];
    *nchunks = t.fwd_n;
    if (!t.fwd_n || (!observed && !expected)) return cudaSuccess;
    if (cap < t.fwd_n) return cudaErrorInvalidValue;
    DeviceGuard dg(device);
    CK(cudaDeviceSynchronize());
    std::vector<uint64_t> w(2 * t.fwd_n);
    CK(cudaMemcpy(w.data(), t.fwd, w.size() * 8, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < t.fwd_n; i++) {
        if (observed) observed[i] = w[2 * i];
        if (expected) expected[i] = w[2 * i + 1];
    }
    return cudaSuccess;
}

int mma_get_segment_order(int device, uint32_t* order, size_t cap, size_t* nsegs)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    if (!nsegs) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> g(e.mu);
    const auto& o = e.tgt[device].last_order;
    *nsegs = o.size();
    if (!order || o.empty()) return cudaSuccess;
    if (cap < o.size()) return cudaErrorInvalidValue;
    memcpy(order, o.data(), o.size() * sizeof(uint32_t));
    return cudaSuccess;
}

int mma_host_alloc(void** ptr, size_t bytes, unsigned flags)
{
    CK((cudaError_t)ensure_init());
    (void)flags;
    return host_alloc(ptr, bytes, E().cfg.numa_mode, 0);
}

int mma_host_free(void* ptr) { return host_free(ptr); }

int mma_host_alloc_size(const void* ptr, size_t* bytes) { return host_alloc_size(ptr, bytes); }

int mma_host_alloc_for(void** ptr, size_t bytes, int device, mma_dir_t dir)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    if (!ptr || (dir != MMA_H2D && dir != MMA_D2H)) return cudaErrorInvalidValue;
    std::vector<uint64_t> ends;
    std::vector<int> nodes;
    {
        std::lock_guard<std::mutex> g(e.mu);
        make_paths(device);
        const auto& ps = e.tgt[device].paths[dir];
        std::vector<PlanPath> pp;
        for (auto& p : ps) pp.push_back(PlanPath{p.kind == MMA_PATH_DIRECT, p.mbps, 0});
        Plan plan;
        const uint64_t C = e.cfg.chunk_bytes[dir];
        if (make_plan(pp.data(), (int)pp.size(), bytes, C, 0, PLAN_CONTIGUOUS, plan)) return cudaErrorInvalidValue;
        uint64_t end = 0;
        for (size_t p = 0; p < ps.size(); p++) {   // contiguous plan: path p's range, in path order
            end = std::min<uint64_t>(bytes, end + plan.count[p] * C);
            ends.push_back(end);
            nodes.push_back(gpu_numa_node(ps[p].gpu));
        }
    }
    return host_alloc_ranges(ptr, bytes, ends.data(), nodes.data(), (int)ends.size());
}

int mma_host_page_node(const void* ptr) { return host_page_node(ptr); }

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
    std::lock_guard<std::mutex> gk(g_kmu);
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

int mma_get_dynamic_backoffs(int device, uint64_t* waits)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    if (!waits) return cudaErrorInvalidValue;
    std::lock_guard<std::mutex> g(e.mu);
    Target& t = e.tgt[device];
    *waits = 0;
    if (!t.last_dyn) return cudaSuccess;
    DeviceGuard dg(device);
    CK(cudaDeviceSynchronize());
    unsigned long long w = 0;
    CK(cudaMemcpy(&w, t.last_dyn + kDynBackoffWord, sizeof w, cudaMemcpyDeviceToHost));
    *waits = w;
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

