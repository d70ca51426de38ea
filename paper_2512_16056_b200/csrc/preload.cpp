// preload.cpp — C10: transparent injection (§4: "Users can load the MMA dynamic
// library via the LD_PRELOAD mechanism, achieving transparent substitution for the native
// CUDA memory API"; §3.2 Transfer Task Interceptor).
//
// libmma_preload.so exports cudaMemcpyAsync / cudaMemcpyAsync_ptsz / cudaMemcpy. A host <->
// device copy (kind H2D / D2H, or cudaMemcpyDefault classified by pointer attributes) of
// at least MMA_PRELOAD_MIN_BYTES goes to mma_memcpy_h2d / mma_memcpy_d2h (which apply the
// engine's own fallback rules); everything else, and any engine error at enqueue, goes to
// the next definition in the lookup order (the application's libcudart) via
// dlsym(RTLD_NEXT). A thread-local guard keeps the engine's own copies native. The shim
// links no CUDA runtime: every runtime function it needs is looked up with RTLD_NEXT.
//
// Pinned allocations: cudaHostAlloc / cudaMallocHost of at least
// MMA_PRELOAD_ALLOC_MIN_BYTES (default 2 MiB; 0 = off) become mma_host_alloc (C8: NUMA-placed
// per the engine's numa_mode, page-locked, mapped into every GPU), so a torch pin_memory()
// buffer is the engine's own and usable by its zero-copy kernels; cudaFreeHost of such a
// buffer is mma_host_free. Write-combined requests and every failure go to the runtime.
//
// Scattered block swaps (paged KV caches) are not interposed: an application that wants the
// multipath scattered copy calls mma_memcpy_{h2d,d2h}_segments (north_star (e)) itself.
#include <dlfcn.h>
#include <stdint.h>
#include <stdlib.h>


#include "../../include/mma.h"

namespace {

typedef int (*memcpy_async_fn)(void*, const void*, size_t, int, void*);
typedef int (*memcpy_fn)(void*, const void*, size_t, int);
typedef int (*sync_fn)(void*);
typedef int (*attr_fn)(void*, const void*);

constexpr int kH2D = 1, kD2H = 2, kDefault = 4;   // cudaMemcpyKind values
constexpr int kTypeHost = 1, kTypeDevice = 2;     // cudaMemoryType values

thread_local int g_inside = 0;

template <typename F>
F next(const char* name)
{
    return reinterpret_cast<F>(dlsym(RTLD_NEXT, name));
}

size_t min_bytes()
{
    static size_t v = [] {
        const char* s = getenv("MMA_PRELOAD_MIN_BYTES");
        return s ? (size_t)strtoull(s, nullptr, 10) : (size_t)(8u << 20);
    }();
    return v;
}

// cudaPointerAttributes layout (CUDA >= 11): int type; int device; void* devicePointer;
// void* hostPointer.
struct PtrAttr {
    int type;
    int device;
    void* devicePointer;
    void* hostPointer;
};

int classify(const void* p)
{
    static attr_fn get = next<attr_fn>("cudaPointerGetAttributes");
    static auto clear = next<int (*)()>("cudaGetLastError");
    if (!get) return 0;
    PtrAttr a{};
    if (get(&a, p) != 0) {
        if (clear) clear();
        return 0;
    }
    return a.type;
}

// Returns the effective kind (kH2D / kD2H) if the engine should take the copy, else 0.
int route(void* dst, const void* src, size_t n, int kind)
{
    if (g_inside || n < min_bytes()) return 0;
    if (kind == kDefault) {
        const int td = classify(dst), ts = classify(src);
        if (td == kTypeDevice && ts != kTypeDevice) kind = kH2D;
        else if (ts == kTypeDevice && td != kTypeDevice) kind = kD2H;
        else return 0;
    }
    return (kind == kH2D || kind == kD2H) ? kind : 0;
}

int engine(void* dst, const void* src, size_t n, int kind, void* stream)
{
    g_inside = 1;
    const int rc = (kind == kH2D) ? mma_memcpy_h2d(dst, src, n, (mma_stream_t)stream)
                                  : mma_memcpy_d2h(dst, src, n, (mma_stream_t)stream);
    g_inside = 0;
    return rc;
}

typedef int (*host_alloc_fn)(void**, size_t, unsigned);
typedef int (*malloc_host_fn)(void**, size_t);
typedef int (*free_host_fn)(void*);

constexpr unsigned kWriteCombined = 0x04;   // cudaHostAllocWriteCombined

size_t alloc_min_bytes()
{
    static size_t v = [] {
        const char* s = getenv("MMA_PRELOAD_ALLOC_MIN_BYTES");
        return s ? (size_t)strtoull(s, nullptr, 10) : (size_t)(2u << 20);
    }();
    return v;
}

// 0 if the engine allocated it (C8), else nonzero
int engine_alloc(void** p, size_t n, unsigned flags)
{
    if (g_inside || !p || alloc_min_bytes() == 0 || n < alloc_min_bytes() || (flags & kWriteCombined)) return 1;
    g_inside = 1;
    const int rc = mma_host_alloc(p, n, 0);
    g_inside = 0;
    return rc;
}

}  // namespace

extern "C" {

__attribute__((visibility("default"))) int cudaMemcpyAsync(void* dst, const void* src, size_t n, int kind, void* stream)
{
    static memcpy_async_fn real = next<memcpy_async_fn>("cudaMemcpyAsync");
    if (const int k = route(dst, src, n, kind)) {
        if (engine(dst, src, n, k, stream) == 0) return 0;
    }
    return real(dst, src, n, kind, stream);
}

__attribute__((visibility("default"))) int cudaMemcpyAsync_ptsz(void* dst, const void* src, size_t n, int kind, void* stream)
{
    static memcpy_async_fn real = next<memcpy_async_fn>("cudaMemcpyAsync_ptsz");
    if (const int k = route(dst, src, n, kind)) {
        // the per-thread default stream handle (cudaStreamPerThread = 0x2) for stream 0
        if (engine(dst, src, n, k, stream ? stream : (void*)0x2) == 0) return 0;
    }
    return real(dst, src, n, kind, stream);
}

__attribute__((visibility("default"))) int cudaHostAlloc(void** p, size_t n, unsigned flags)
{
    static host_alloc_fn real = next<host_alloc_fn>("cudaHostAlloc");
    if (engine_alloc(p, n, flags) == 0) return 0;
    return real(p, n, flags);
}

__attribute__((visibility("default"))) int cudaMallocHost(void** p, size_t n)
{
    static malloc_host_fn real = next<malloc_host_fn>("cudaMallocHost");
    if (engine_alloc(p, n, 0) == 0) return 0;
    return real(p, n);
}

__attribute__((visibility("default"))) int cudaFreeHost(void* p)
{
    static free_host_fn real = next<free_host_fn>("cudaFreeHost");
    size_t n = 0;
    if (p && mma_host_alloc_size(p, &n) == 0) return mma_host_free(p);   // the engine's (C8)
    return real(p);
}

__attribute__((visibility("default"))) int cudaMemcpy(void* dst, const void* src, size_t n, int kind)
{
    static memcpy_fn real = next<memcpy_fn>("cudaMemcpy");
    static sync_fn sync = next<sync_fn>("cudaStreamSynchronize");
    if (const int k = route(dst, src, n, kind)) {
        // synchronous semantics: enqueue on the legacy stream, then wait for it
        if (sync && engine(dst, src, n, k, nullptr) == 0) return sync(nullptr);
    }
    return real(dst, src, n, kind);
}

}  // extern "C"
