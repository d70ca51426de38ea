// hostmem.cpp — C8: NUMA-aware pinned host buffers (layer L1).
//
// A multipath copy reads host DRAM through every participating GPU's PCIe link; the paper
// attributes its 6-path plateau to the cross-NUMA link (§5.1.1). Buffers from
// mma_host_alloc are anonymous mappings whose pages are bound with mbind(2) (raw syscall:
// libnuma is absent) to the requested node(s) before first touch, then registered with
// cudaHostRegister(PORTABLE | MAPPED) so every GPU's copy engine and SMs can reach them.
// numa_mode: 0 = kernel default placement, 1 = node `node0`, 2 = interleave across nodes
// (page by page), 3 = 2 MiB blocks round-robin over the nodes (every block on one node, so a
// paged-KV block never straddles nodes and the planner's regrouping, R23, sees whole blocks).
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "engine.h"

namespace mma {

namespace {
std::mutex g_mu;
std::map<void*, size_t> g_allocs;   // base -> mapped length
std::map<void*, bool> g_interleaved;   // bases placed page by page (numa_mode 2): never cached

// host_nodes' cache: 2 MiB region -> node. Pinned pages do not move, but a freed range can be
// mapped again on another node, so host_free drops its regions.
std::mutex g_node_mu;
std::unordered_map<uintptr_t, int> g_node_cache;

constexpr int kMpolBind = 2;
constexpr int kMpolInterleave = 3;

int numa_nodes()
{
    int n = 0;
    for (int i = 0; i < 64; i++) {
        char path[96];
        snprintf(path, sizeof path, "/sys/devices/system/node/node%d", i);
        if (access(path, F_OK) == 0) n = i + 1;
    }
    return n < 1 ? 1 : n;
}
}  // namespace

int host_alloc(void** ptr, size_t bytes, int numa_mode, int node0)
{
    if (!ptr) return cudaErrorInvalidValue;
    *ptr = nullptr;
    if (bytes == 0) return cudaSuccess;
    const size_t align = 2u << 20;
    const size_t len = (bytes + align - 1) / align * align;
    void* p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) return cudaErrorMemoryAllocation;
    madvise(p, len, MADV_HUGEPAGE);
    const int nodes = numa_nodes();
    if (numa_mode == 3 && nodes > 1) {
        for (size_t off = 0; off < len; off += align) {
            unsigned long mask[4] = {0, 0, 0, 0};
            const int nd = (int)((off / align) % nodes);
            mask[nd / 64] |= 1ul << (nd % 64);
            syscall(SYS_mbind, (char*)p + off, align, kMpolBind, mask, 256ul, 0u);   // best effort
        }
    } else if (numa_mode != 0 && nodes > 1) {
        unsigned long mask[4] = {0, 0, 0, 0};
        int mode = kMpolBind;
        if (numa_mode == 2) {
            mode = kMpolInterleave;
            for (int i = 0; i < nodes && i < 256; i++) mask[i / 64] |= 1ul << (i % 64);
        } else {
            int nd = node0 < 0 ? 0 : node0 % nodes;
            mask[nd / 64] |= 1ul << (nd % 64);
        }
        syscall(SYS_mbind, p, len, mode, mask, 256ul, 0u);   // best effort
    }
    memset(p, 0, len);   // first touch places the pages
    cudaError_t e = cudaHostRegister(p, len, cudaHostRegisterPortable | cudaHostRegisterMapped);
    if (e != cudaSuccess) {
        munmap(p, len);
        return e;
    }
    std::lock_guard<std::mutex> g(g_mu);
    g_allocs[p] = len;
    if (numa_mode == 2 && nodes > 1) g_interleaved[p] = true;
    *ptr = p;
    return cudaSuccess;
}

// numa_mode 3 ("spread"): bind consecutive byte ranges to given nodes before first
// touch -- range k = [end[k-1], end[k]) on node[k] (node < 0: default placement). Used for a
// contiguous transfer whose plan gives path p one range, placed on the node of p's GPU.
int host_alloc_ranges(void** ptr, size_t bytes, const uint64_t* range_end, const int* node, int nranges)
{
    if (!ptr || (nranges && (!range_end || !node))) return cudaErrorInvalidValue;
    *ptr = nullptr;
    if (bytes == 0) return cudaSuccess;
    const size_t align = 2u << 20, page = 4096;
    const size_t len = (bytes + align - 1) / align * align;
    void* p = mmap(nullptr, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) return cudaErrorMemoryAllocation;
    const int nodes = numa_nodes();
    uint64_t a = 0;
    for (int k = 0; k < nranges && nodes > 1; k++) {
        const uint64_t b = std::min<uint64_t>(range_end[k], len);
        const uint64_t pa = a / page * page, pb = (b + page - 1) / page * page;
        if (node[k] >= 0 && node[k] < nodes && pb > pa) {
            unsigned long mask[4] = {0, 0, 0, 0};
            mask[node[k] / 64] |= 1ul << (node[k] % 64);
            syscall(SYS_mbind, (char*)p + pa, pb - pa, kMpolBind, mask, 256ul, 0u);   // best effort
        }
        a = b;
    }
    memset(p, 0, len);   // first touch places the pages
    cudaError_t e = cudaHostRegister(p, len, cudaHostRegisterPortable | cudaHostRegisterMapped);
    if (e != cudaSuccess) {
        munmap(p, len);
        return e;
    }
    std::lock_guard<std::mutex> g(g_mu);
    g_allocs[p] = len;
    *ptr = p;
    return cudaSuccess;
}

int host_alloc_size(const void* ptr, size_t* bytes)
{
    std::lock_guard<std::mutex> g(g_mu);
    auto it = g_allocs.find(const_cast<void*>(ptr));
    if (it == g_allocs.end()) return cudaErrorInvalidValue;
    if (bytes) *bytes = it->second;
    return cudaSuccess;
}

int host_free(void* ptr)
{
    if (!ptr) return cudaSuccess;
    size_t len;
    {
        std::lock_guard<std::mutex> g(g_mu);
        auto it = g_allocs.find(ptr);
        if (it == g_allocs.end()) return cudaErrorInvalidValue;
        len = it->second;
        g_allocs.erase(it);
        g_interleaved.erase(ptr);
    }
    {
        std::lock_guard<std::mutex> g(g_node_mu);
        const uintptr_t a = reinterpret_cast<uintptr_t>(ptr) >> 21, b = (reinterpret_cast<uintptr_t>(ptr) + len - 1) >> 21;
        for (uintptr_t r = a; r <= b; r++) g_node_cache.erase(r);
    }
    cudaError_t e = cudaHostUnregister(ptr);
    munmap(ptr, len);
    return e;
}

// NUMA node of page `p` (move_pages with nodes = NULL queries), or -1.
int host_page_node(const void* p)
{
    void* pages[1] = {const_cast<void*>(p)};
    int status[1] = {-1};
    if (syscall(SYS_move_pages, 0, 1ul, pages, nullptr, status, 0) != 0) return -1;
    return status[0];
}

int host_numa_count() { return numa_nodes(); }

void host_nodes(const void* const* p, size_t n, int* nodes)
{
    if (const char* fk = getenv("MMA_FAKE_HOST_NODES")) {   // test hook: 2 MiB regions round-robin
        const long k = atol(fk);
        for (size_t i = 0; i < n; i++) nodes[i] = k > 0 ? (int)((reinterpret_cast<uintptr_t>(p[i]) >> 21) % k) : -1;
        return;
    }
    if (numa_nodes() < 2) {
        for (size_t i = 0; i < n; i++) nodes[i] = 0;
        return;
    }
    // regions inside page-interleaved allocations are asked page by page, never cached
    std::vector<char> nocache(n, 0);
    {
        std::lock_guard<std::mutex> g(g_mu);
        if (!g_interleaved.empty())
            for (size_t i = 0; i < n; i++) {
                auto it = g_allocs.upper_bound(const_cast<void*>(p[i]));
                if (it == g_allocs.begin()) continue;
                --it;
                if ((const char*)p[i] < (const char*)it->first + it->second && g_interleaved.count(it->first)) nocache[i] = 1;
            }
    }
    std::unordered_map<uintptr_t, int>& cache = g_node_cache;
    std::lock_guard<std::mutex> g(g_node_mu);
    std::vector<void*> ask;
    std::vector<size_t> who;
    for (size_t i = 0; i < n; i++) {
        const uintptr_t r = reinterpret_cast<uintptr_t>(p[i]) >> 21;
        auto it = nocache[i] ? cache.end() : cache.find(r);
        if (it != cache.end()) nodes[i] = it->second;
        else { nodes[i] = -2; ask.push_back(const_cast<void*>(p[i])); who.push_back(i); }
    }
    if (!ask.empty()) {   // one move_pages query (nodes = NULL: report) for every unknown region
        std::vector<int> st(ask.size(), -1);
        if (syscall(SYS_move_pages, 0, (unsigned long)ask.size(), ask.data(), nullptr, st.data(), 0) != 0)
            std::fill(st.begin(), st.end(), -1);
        for (size_t q = 0; q < ask.size(); q++) {
            const int nd = st[q] >= 0 ? st[q] : -1;
            if (!nocache[who[q]]) cache[reinterpret_cast<uintptr_t>(ask[q]) >> 21] = nd;
            nodes[who[q]] = nd;
        }
        for (size_t i = 0; i < n; i++)   // repeats of a region asked in this call
            if (nodes[i] == -2) nodes[i] = cache[reinterpret_cast<uintptr_t>(p[i]) >> 21];
    }
}

int gpu_numa_node(int dev)
{
    char bus[32] = {0};
    if (cudaDeviceGetPCIBusId(bus, sizeof bus - 1, phys_dev(dev)) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    std::string b = bus;
    for (char& c : b) c = (char)tolower((unsigned char)c);
    int node = -1;
    if (FILE* f = fopen(("/sys/bus/pci/devices/" + b + "/numa_node").c_str(), "r")) {
        if (fscanf(f, "%d", &node) != 1) node = -1;
        fclose(f);
    }
    return node;
}

}  // namespace mma
