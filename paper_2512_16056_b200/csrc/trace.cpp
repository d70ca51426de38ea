// trace.cpp — timeline tracing of the data plane (SURVEY §5 "tracing / profiling").
//
// While a trace is active, every copy-engine DMA (or batch) and every kernel the engine
// enqueues is bracketed by CUDA events on the stream it runs on. mma_trace_end writes the
// spans as a Chrome trace (chrome://tracing, Perfetto): one process row per GPU, one
// thread row per engine stream, so overlapping copy engines, relay kernels and zero-copy
// kernels are visible directly. Times are relative to a reference event recorded on every
// device when the trace began (per-device clocks; rows of different GPUs are aligned to
// within the host's launch skew).
#include "plane.h"

namespace mma {

namespace {

struct Span {
    int dev;
    cudaStream_t stream;
    std::string name;
    int path;
    long long chunk;
    uint64_t bytes;
    cudaEvent_t a, b;
};

std::mutex g_tmu;
bool g_on = false;
size_t g_cap = 0;
std::vector<Span> g_spans;
cudaEvent_t g_ref[MMA_MAX_GPUS] = {};

std::string stream_name(cudaStream_t s)
{
    Engine& e = E();
    for (int d = 0; d < e.ndev; d++) {
        const DevRes& r = e.dev[d];
        if (!r.made) continue;
        for (int k = 0; k < 4; k++) {
            const int dir = k & 1;
            const Lanes& l = k < 2 ? r.lane[dir] : r.cap_lane[dir];
            const std::string sfx = std::string(dir == MMA_H2D ? " (H2D" : " (D2H") + (k < 2 ? ")" : ", captured)");
            if (s == l.direct) return "direct DMA" + sfx;
            if (s == l.hop[0]) return "relay hop stream 0" + sfx;
            if (s == l.hop[1]) return "relay hop stream 1" + sfx;
            if (s == l.kern) return "relay kernels" + sfx;
            if (s == l.zc) return "zero-copy kernels" + sfx;
        }
    }
    return "user stream";
}

}  // namespace

bool trace_on() { return g_on; }

TSpan::TSpan(int dev, cudaStream_t s, const char* name, int path, long long chunk, uint64_t bytes)
{
    if (!g_on || tl_capturing) return;
    std::lock_guard<std::mutex> g(g_tmu);
    if (g_spans.size() >= g_cap) return;
    DeviceGuard dg(dev);
    Span sp{dev, s, name, path, chunk, bytes, nullptr, nullptr};
    if (cudaEventCreate(&sp.a) != cudaSuccess || cudaEventCreate(&sp.b) != cudaSuccess) return;
    if (cudaEventRecord(sp.a, s) != cudaSuccess) return;
    idx_ = (long long)g_spans.size();
    g_spans.push_back(sp);
}

TSpan::~TSpan()
{
    if (idx_ < 0) return;
    std::lock_guard<std::mutex> g(g_tmu);
    Span& sp = g_spans[(size_t)idx_];
    DeviceGuard dg(sp.dev);
    cudaEventRecord(sp.b, sp.stream);
}

}  // namespace mma

using namespace mma;

extern "C" {

int mma_trace_begin(size_t max_spans)
{
    CK((cudaError_t)ensure_init());
    Engine& e = E();
    std::lock_guard<std::mutex> lk(e.mu);
    std::lock_guard<std::mutex> g(g_tmu);
    if (g_on) return cudaErrorInvalidValue;
    for (int d = 0; d < e.ndev; d++) {
        DeviceGuard dg(d);
        CK(cudaDeviceSynchronize());
        if (!g_ref[d]) CK(cudaEventCreate(&g_ref[d]));
        CK(cudaEventRecord(g_ref[d], 0));
    }
    g_spans.clear();
    g_cap = max_spans ? max_spans : 100000;
    g_on = true;
    return cudaSuccess;
}

int mma_trace_end(const char* json_path, size_t* nspans)
{
    Engine& e = E();
    std::lock_guard<std::mutex> lk(e.mu);
    std::lock_guard<std::mutex> g(g_tmu);
    if (!g_on) return cudaErrorInvalidValue;
    g_on = false;
    FILE* f = json_path ? fopen(json_path, "w") : nullptr;
    if (json_path && !f) return cudaErrorInvalidValue;
    if (f) fprintf(f, "{\"traceEvents\": [\n");
    size_t k = 0;
    int rc = cudaSuccess;
    for (auto& sp : g_spans) {
        DeviceGuard dg(sp.dev);
        float t0 = 0, t1 = 0;
        if (cudaEventSynchronize(sp.b) != cudaSuccess || cudaEventElapsedTime(&t0, g_ref[sp.dev], sp.a) != cudaSuccess ||
            cudaEventElapsedTime(&t1, g_ref[sp.dev], sp.b) != cudaSuccess)
            rc = cudaErrorUnknown;
        if (f)
            fprintf(f, "%s{\"name\": \"%s\", \"ph\": \"X\", \"pid\": \"GPU %d\", \"tid\": \"%s\", \"ts\": %.3f, "
                       "\"dur\": %.3f, \"args\": {\"path\": %d, \"chunk\": %lld, \"bytes\": %llu}}",
                    k ? ",\n" : "", sp.name.c_str(), sp.dev, stream_name(sp.stream).c_str(), t0 * 1e3,
                    (t1 - t0) * 1e3, sp.path, sp.chunk, (unsigned long long)sp.bytes);
        cudaEventDestroy(sp.a);
        cudaEventDestroy(sp.b);
        k++;
    }
    if (f) {
        fprintf(f, "\n]}\n");
        fclose(f);
    }
    if (nspans) *nspans = k;
    g_spans.clear();
    return rc;
}

}  // extern "C"
