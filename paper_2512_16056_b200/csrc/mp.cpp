// mp.cpp — multi-process mode: one process per GPU, as in vLLM tensor
// parallel serving. The target's process exports its destination memory (CUDA IPC) and the
// host buffer lives in shared memory registered by every process; each process then moves
// its own share of the transfer on its own GPU with the zero-copy kernel -- the chunks the
// common plan gives its path (planned mode), or the chunks it claims from a cursor in the
// target's memory (the dynamic pull of plane.cpp, across processes). No process creates a
// context on another process's GPU, and nothing on the data path is a collective.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <sys/statvfs.h>
#include <unistd.h>

#include "plane.h"

namespace mma {

namespace {

struct SharedMap {
    size_t len;
    int fd;
};
std::mutex g_mp_mu;
std::map<void*, SharedMap> g_shared;      // mapping -> length, fd
std::map<void*, void*> g_ipc_base;        // user pointer -> IPC base to close

using PFN_range = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

// A directory for the shared buffer: /dev/shm when it has room (tmpfs), else MMA_SHM_DIR or
// /tmp (a file-backed shared mapping; its pages are locked by cudaHostRegister).
std::string shared_path(const char* name, size_t bytes)
{
    std::string dir = "/dev/shm";
    struct statvfs v;
    if (statvfs(dir.c_str(), &v) != 0 || (uint64_t)v.f_bavail * v.f_frsize < bytes + (64u << 20)) {
        const char* d = getenv("MMA_SHM_DIR");
        dir = d ? d : "/tmp";
    }
    return dir + "/mma_" + name;
}

// Segment table (and chunk list) on the device for one launch: allocated and freed in
// stream order.
int upload(const void* host, size_t bytes, cudaStream_t s, void** dev)
{
    *dev = nullptr;
    if (!bytes) return cudaSuccess;
    CK(cudaMallocAsync(dev, bytes, s));
    return (int)cudaMemcpyAsync(*dev, host, bytes, cudaMemcpyHostToDevice, s);
}

int vstream_from(const mma_segment_t* segs, size_t nsegs, uint64_t C, cudaStream_t s,
                 VStreamArg& v, void** dtab)
{
    v = VStreamArg{};
    v.C = C;
    *dtab = nullptr;
    if (nsegs == 1) {
        v.nseg = 1;
        v.B = segs[0].bytes;
        v.src0 = (uint64_t)segs[0].src;
        v.dst0 = (uint64_t)segs[0].dst;
        return cudaSuccess;
    }
    std::vector<uint64_t> w(3 * nsegs + 1);
    w[0] = 0;
    for (size_t k = 0; k < nsegs; k++) {
        if (segs[k].bytes && (!segs[k].src || !segs[k].dst)) return cudaErrorInvalidValue;
        w[k + 1] = w[k] + segs[k].bytes;
        w[nsegs + 1 + k] = (uint64_t)segs[k].src;
        w[2 * nsegs + 1 + k] = (uint64_t)segs[k].dst;
    }
    v.nseg = nsegs;
    v.B = w[nsegs];
    CK(upload(w.data(), w.size() * 8, s, dtab));
    const uint64_t* d = (const uint64_t*)*dtab;
    v.start = d;
    v.src = d + nsegs + 1;
    v.dst = d + 2 * nsegs + 1;
    return cudaSuccess;
}

// Multi-process shares enter the cross-process ledger (mma_ledger_attach) while queued: the
// bytes are added at enqueue and removed by a host function on the stream once the kernel
// has run (the function makes no CUDA call: the ledger slot is resolved here).
struct LedgerRelease {
    int dir, slot;
    int64_t bytes, own;
    uint64_t gen;   // the attach it entered (a re-attach drops it)
};

void CUDART_CB release_share(void* p)
{
    LedgerRelease* r = (LedgerRelease*)p;
    shm_ledger_add_slot(r->dir, r->slot, -r->bytes, -r->own, r->gen);
    delete r;
}

// direction of a segment table from the memory kinds: a device source is an offload (D2H)
static int seg_dir(const mma_segment_t* segs)
{
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, segs[0].src) == cudaSuccess && a.type == cudaMemoryTypeDevice) return MMA_D2H;
    return MMA_H2D;
}

int ledger_share(const mma_segment_t* segs, int device, uint64_t bytes, bool own, cudaStream_t s)
{
    const int slot = shm_ledger_slot(device);
    if (slot < 0 || !bytes) return cudaSuccess;
    const int dir = seg_dir(segs);
    cudaGetLastError();
    LedgerRelease* r = new LedgerRelease{dir, slot, (int64_t)bytes, own ? (int64_t)bytes : 0, shm_ledger_gen()};
    shm_ledger_add_slot(dir, slot, r->bytes, r->own, r->gen);
    const cudaError_t e = cudaLaunchHostFunc(s, release_share, r);
    if (e != cudaSuccess) release_share(r);
    return (int)e;
}

// The copy-engine relay ring of this process for one (device, direction) (NEXT-4): S slots
// of C bytes in this GPU's HBM and the dual relay pipeline's two streams. Slot s
// is always used on stream s & 1, so stream order alone keeps a slot's next hop-1 DMA behind
// its previous hop-2 DMA: the ring needs no flags, and a share of another process's transfer
// moves through it with this process's copy engines only.
struct ShareRing {
    char* stage = nullptr;
    uint64_t C = 0;
    uint32_t S = 0;
    cudaStream_t hop[2] = {};
    cudaEvent_t fork = nullptr, done[2] = {};
    uint64_t next = 0;   // chunks carried so far: the slot of the next one
};
ShareRing g_share_ring[MMA_MAX_GPUS][2];

int share_ring(int device, int dir, uint64_t C, uint32_t S, ShareRing** out)
{
    ShareRing& r = g_share_ring[device][dir];
    DeviceGuard g(device);
    if (r.stage && (r.C < C || r.S != S)) {   // re-sized: drain, then make it afresh
        for (cudaStream_t h : r.hop) CK(cudaStreamSynchronize(h));
        CK(cudaFree(r.stage));
        r.stage = nullptr;
    }
    if (!r.hop[0]) {
        for (int k = 0; k < 2; k++) {
            CK(cudaStreamCreateWithFlags(&r.hop[k], cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&r.done[k], cudaEventDisableTiming));
        }
        CK(cudaEventCreateWithFlags(&r.fork, cudaEventDisableTiming));
    }
    if (!r.stage) {
        CK(cudaMalloc(&r.stage, (size_t)S * C));
        r.C = C;
        r.S = S;
        r.next = 0;
    }
    *out = &r;
    return cudaSuccess;
}

}  // namespace

// mma_finalize: the share rings die with the engine (every device was synchronised)
void mp_finalize()
{
    std::lock_guard<std::mutex> lk(g_mp_mu);
    for (int d = 0; d < MMA_MAX_GPUS; d++)
        for (ShareRing& r : g_share_ring[d]) {
            if (!r.hop[0] && !r.stage) continue;
            DeviceGuard g(d);
            if (r.stage) cudaFree(r.stage);
            for (int k = 0; k < 2; k++) {
                if (r.hop[k]) cudaStreamDestroy(r.hop[k]);
                if (r.done[k]) cudaEventDestroy(r.done[k]);
            }
            if (r.fork) cudaEventDestroy(r.fork);
            r = ShareRing();
        }
}

}  // namespace mma

using namespace mma;

extern "C" {

int mma_shared_host_alloc(const char* name, size_t bytes, int create, void** ptr)
{
    if (!name || !*name || !ptr || bytes == 0) return cudaErrorInvalidValue;
    CK((cudaError_t)ensure_init());
    *ptr = nullptr;
    const std::string path = shared_path(name, bytes);
    int fd = open(path.c_str(), create ? (O_RDWR | O_CREAT | O_TRUNC) : O_RDWR, 0600);
    if (fd < 0) return cudaErrorInvalidValue;
    if (create && ftruncate(fd, (off_t)bytes) != 0) { close(fd); return cudaErrorMemoryAllocation; }
    struct stat st;
    if (fstat(fd, &st) != 0 || (size_t)st.st_size < bytes) { close(fd); return cudaErrorInvalidValue; }
    void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    if (p == MAP_FAILED) { close(fd); return cudaErrorMemoryAllocation; }
    if (create) memset(p, 0, bytes);           // allocate every page before pinning
    cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped);
    if (e != cudaSuccess) { munmap(p, bytes); close(fd); return e; }
    std::lock_guard<std::mutex> g(g_mp_mu);
    g_shared[p] = SharedMap{bytes, fd};
    *ptr = p;
    return cudaSuccess;
}

int mma_shared_host_free(void* ptr, const char* unlink_name)
{
    SharedMap m;
    {
        std::lock_guard<std::mutex> g(g_mp_mu);
        auto it = g_shared.find(ptr);
        if (it == g_shared.end()) return cudaErrorInvalidValue;
        m = it->second;
        g_shared.erase(it);
    }
    cudaError_t e = cudaHostUnregister(ptr);
    munmap(ptr, m.len);
    close(m.fd);
    if (unlink_name && *unlink_name) unlink(shared_path(unlink_name, 0).c_str());
    return e;
}

int mma_ipc_export(const void* dev_ptr, void* handle, uint64_t* offset)
{
    if (!dev_ptr || !handle || !offset) return cudaErrorInvalidValue;
    CK((cudaError_t)ensure_init());
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &fn, 12000, cudaEnableDefault, &q) != cudaSuccess || !fn)
        return cudaErrorNotSupported;
    CUdeviceptr base = 0;
    size_t size = 0;
    if (((PFN_range)fn)(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS) return cudaErrorInvalidValue;
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, (void*)base));
    memcpy(handle, &h, sizeof h);
    *offset = (uint64_t)dev_ptr - (uint64_t)base;
    return cudaSuccess;
}

int mma_ipc_open(const void* handle, uint64_t offset, int device, void** dev_ptr)
{
    if (!handle || !dev_ptr) return cudaErrorInvalidValue;
    CK((cudaError_t)ensure_init());
    DeviceGuard g(device);
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    void* base = nullptr;
    CK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *dev_ptr = (char*)base + offset;
    std::lock_guard<std::mutex> lk(g_mp_mu);
    g_ipc_base[*dev_ptr] = base;
    return cudaSuccess;
}

int mma_ipc_close(void* dev_ptr)
{
    void* base;
    {
        std::lock_guard<std::mutex> lk(g_mp_mu);
        auto it = g_ipc_base.find(dev_ptr);
        if (it == g_ipc_base.end()) return cudaErrorInvalidValue;
        base = it->second;
        g_ipc_base.erase(it);
    }
    return (int)cudaIpcCloseMemHandle(base);
}

int mma_copy_share_segments(const mma_segment_t* segs, size_t nsegs, size_t chunk_bytes,
                            const uint8_t* path_of_chunk, size_t nchunks, int path, int device,
                            mma_stream_t stream)
{
    CK((cudaError_t)ensure_init());
    if (int se = sticky()) return se;
    if (!nsegs) return cudaSuccess;
    if (!segs || !path_of_chunk || chunk_bytes == 0 || path < 0) return cudaErrorInvalidValue;
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    CK(make_device(device));
    DeviceGuard g(device);
    cudaStream_t s = (cudaStream_t)stream;
    VStreamArg v;
    void* dtab = nullptr;
    CK(vstream_from(segs, nsegs, chunk_bytes, s, v, &dtab));
    if ((v.B + chunk_bytes - 1) / chunk_bytes != nchunks && !(nchunks == 1 && v.B > 0)) {
        if (dtab) cudaFreeAsync(dtab, s);
        return cudaErrorInvalidValue;
    }
    if (nchunks == 1) v.C = v.B;             // a one-piece (fallback) plan
    std::vector<uint32_t> mine;
    for (size_t i = 0; i < nchunks; i++)
        if (path_of_chunk[i] == path) mine.push_back((uint32_t)i);
    int rc = cudaSuccess;
    if (!mine.empty()) {
        void* dlist = nullptr;
        rc = upload(mine.data(), mine.size() * 4, s, &dlist);
        if (rc == cudaSuccess) {
            ZcLaunchArg a{};
            a.v = v;
            a.chunks.count = mine.size();
            a.chunks.table = (const uint32_t*)dlist;
            a.unit_bytes = e.unit_bytes;
            a.path = (uint32_t)path;
            const uint64_t upc = (v.C + e.unit_bytes - 1) / e.unit_bytes;
            const unsigned grid = (unsigned)std::min<uint64_t>(mine.size() * upc, zc_grid(device, seg_dir(segs)));
            KTimer kt(device, s, 0 | (path << 8));
            rc = launch_zc(a, grid, s);   // the share's dst may be a peer's (IPC): vector form
            cudaFreeAsync(dlist, s);
        }
        if (rc == cudaSuccess) {   // this share's bytes, queued on this GPU's link
            uint64_t mine_bytes = 0;
            for (uint32_t i : mine) mine_bytes += std::min<uint64_t>(v.C, v.B - (uint64_t)i * v.C);
            rc = ledger_share(segs, device, mine_bytes, path == 0, s);
        }
    }
    if (dtab) cudaFreeAsync(dtab, s);
    return rc;
}

int mma_copy_share_segments_ring(const mma_segment_t* segs, size_t nsegs, size_t chunk_bytes,
                                 const uint8_t* path_of_chunk, size_t nchunks, int path, int device,
                                 unsigned slots, mma_stream_t stream)
{
    CK((cudaError_t)ensure_init());
    if (int se = sticky()) return se;
    if (!nsegs) return cudaSuccess;
    if (!segs || !path_of_chunk || chunk_bytes == 0 || path < 0 || slots < 1 || slots > 64) return cudaErrorInvalidValue;
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    std::vector<uint64_t> start(nsegs + 1, 0);
    for (size_t k = 0; k < nsegs; k++) {
        if (segs[k].bytes && (!segs[k].src || !segs[k].dst)) return cudaErrorInvalidValue;
        start[k + 1] = start[k] + segs[k].bytes;
    }
    const uint64_t B = start[nsegs];
    uint64_t C = chunk_bytes;
    if ((B + C - 1) / C != nchunks && !(nchunks == 1 && B > 0)) return cudaErrorInvalidValue;
    if (nchunks == 1) C = B;                   // a one-piece (fallback) plan
    const int dir = seg_dir(segs);
    cudaGetLastError();
    CK(make_device(device));
    std::lock_guard<std::mutex> lk(g_mp_mu);
    ShareRing* r = nullptr;
    CK(share_ring(device, dir, C, slots, &r));
    DeviceGuard g(device);
    cudaStream_t user = (cudaStream_t)stream;
    CK(cudaEventRecord(r->fork, user));
    bool used[2] = {false, false};
    uint64_t mine_bytes = 0;
    for (size_t i = 0; i < nchunks; i++) {
        if (path_of_chunk[i] != path) continue;
        const uint64_t off = (uint64_t)i * C, len = std::min<uint64_t>(C, B - off);
        const uint32_t slot = (uint32_t)(r->next++ % r->S);
        const int k = slot & 1;
        cudaStream_t hs = r->hop[k];
        if (!used[k]) { CK(cudaStreamWaitEvent(hs, r->fork, 0)); used[k] = true; }
        char* buf = r->stage + (uint64_t)slot * r->C;
        DmaBatch in, out;
        size_t q = std::upper_bound(start.begin(), start.end(), off) - start.begin() - 1;
        for (; q < nsegs && start[q] < off + len; q++) {   // the chunk's pieces, packed in the slot
            const uint64_t lo = std::max(start[q], off), hi = std::min(start[q + 1], off + len);
            if (lo >= hi) continue;
            const char* sp = (const char*)segs[q].src + (lo - start[q]);
            char* dp = (char*)segs[q].dst + (lo - start[q]);
            in.add(buf + (lo - off), sp, hi - lo);
            out.add(dp, buf + (lo - off), hi - lo);
        }
        // hop 1 into the slot over this GPU's link (H2D) or from the source GPU (D2H, a peer
        // copy over NVLink), hop 2 out of it: the same stream, so the slot is free again after
        CK(in.issue(dir == MMA_H2D ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, hs));
        CK(out.issue(dir == MMA_H2D ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, hs));
        mine_bytes += len;
    }
    for (int k = 0; k < 2; k++)   // join: the user stream waits for both relay streams
        if (used[k]) {
            CK(cudaEventRecord(r->done[k], r->hop[k]));
            CK(cudaStreamWaitEvent(user, r->done[k], 0));
        }
    return ledger_share(segs, device, mine_bytes, path == 0, user);
}

int mma_copy_claim_segments(const mma_segment_t* segs, size_t nsegs, size_t claim_bytes,
                            uint64_t* cursor, uint64_t* counts, int path, int device,
                            mma_stream_t stream)
{
    CK((cudaError_t)ensure_init());
    if (int se = sticky()) return se;
    if (!nsegs) return cudaSuccess;
    if (!segs || !cursor || !counts || claim_bytes == 0 || path < 0 || path >= MMA_KMAX_RINGS)
        return cudaErrorInvalidValue;
    Engine& e = E();
    if (device < 0 || device >= e.ndev) return cudaErrorInvalidDevice;
    CK(make_device(device));
    DeviceGuard g(device);
    cudaStream_t s = (cudaStream_t)stream;
    VStreamArg v;
    void* dtab = nullptr;
    CK(vstream_from(segs, nsegs, claim_bytes, s, v, &dtab));
    DynLaunchArg a{};
    a.v = v;
    a.nchunks = (v.B + claim_bytes - 1) / claim_bytes;
    a.cursor = (unsigned long long*)cursor;
    a.counts = (unsigned long long*)counts;
    a.path = (uint32_t)path;
    const unsigned grid = (unsigned)std::min<uint64_t>(a.nchunks, zc_grid(device, seg_dir(segs)));
    int rc = cudaSuccess;
    if (a.nchunks) {
        KTimer kt(device, s, 3 | (path << 8));
        rc = launch_zc_dyn(a, grid, s);
    }
    if (dtab) cudaFreeAsync(dtab, s);
    return rc;
}

}  // extern "C"
