// ledger_shm.cpp — the backlog ledger shared between processes ("a
// shared-memory path ledger"; §5.1.2: with one process per GPU each process keeps
// its own multipath queue, so without a shared view two flows relay through each other's
// links blindly -- Fig 9b's two MMA flows).
//
// One POSIX shared-memory object per name holds, per (direction, GPU), the bytes that calls
// of every attached process still have queued on that GPU's link, and of those the bytes of
// the GPU's own (direct) transfers. GPUs are keyed by PCI bus id, so processes with different
// CUDA_VISIBLE_DEVICES agree on them. An all-zero object is a valid empty ledger, so creation
// needs no initialisation protocol. Counters are lock-free 64-bit atomics in the mapping.
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>

#include "plane.h"

namespace mma {

namespace {

struct ShmLedger {
    std::atomic<uint32_t> lock;                    // guards the slot table
    uint32_t pad;
    char bus[MMA_MAX_GPUS][32];                    // PCI bus id per slot ("" = free)
    std::atomic<uint64_t> bytes[2][MMA_MAX_GPUS];  // queued on the slot's link
    std::atomic<uint64_t> own[2][MMA_MAX_GPUS];    // of which the slot's own target's direct bytes
};
static_assert(std::atomic<uint64_t>::is_always_lock_free, "cross-process atomics must be lock-free");

std::mutex g_mu;
ShmLedger* g_shm = nullptr;
int g_slot_cache[MMA_MAX_GPUS];   // local device -> slot (-2 = not looked up); reset on attach
bool g_cache_init = false;

std::string shm_name(const char* name) { return std::string("/mma_ledger_") + name; }

// slot of a bus id (claimed on first use); -1 when the table is full
int slot_of(const char* bus)
{
    if (!g_shm || !bus || !*bus) return -1;
    while (g_shm->lock.exchange(1, std::memory_order_acquire)) {
    }
    int found = -1, free_slot = -1;
    for (int s = 0; s < MMA_MAX_GPUS; s++) {
        if (!strncmp(g_shm->bus[s], bus, sizeof g_shm->bus[s])) { found = s; break; }
        if (free_slot < 0 && !g_shm->bus[s][0]) free_slot = s;
    }
    if (found < 0 && free_slot >= 0) {
        strncpy(g_shm->bus[free_slot], bus, sizeof g_shm->bus[free_slot] - 1);
        found = free_slot;
    }
    g_shm->lock.store(0, std::memory_order_release);
    return found;
}

// slot of local device `dev` (bus id from the driver), cached per attach (g_mu held)
int slot_of_device(int dev)
{
    if (!g_cache_init) {
        for (int& c : g_slot_cache) c = -2;
        g_cache_init = true;
    }
    if (dev < 0 || dev >= MMA_MAX_GPUS) return -1;
    if (g_slot_cache[dev] == -2) {
        char bus[32] = {0};
        if (cudaDeviceGetPCIBusId(bus, sizeof bus - 1, dev) != cudaSuccess) {
            cudaGetLastError();
            return -1;
        }
        g_slot_cache[dev] = slot_of(bus);
    }
    return g_slot_cache[dev];
}
}  // namespace

bool shm_ledger_on()
{
    std::lock_guard<std::mutex> g(g_mu);
    return g_shm != nullptr;
}

void shm_ledger_add(int dir, int dev, int64_t bytes, int64_t own)
{
    std::lock_guard<std::mutex> g(g_mu);
    const int s = slot_of_device(dev);
    if (s < 0) return;
    g_shm->bytes[dir][s].fetch_add((uint64_t)bytes, std::memory_order_relaxed);
    g_shm->own[dir][s].fetch_add((uint64_t)own, std::memory_order_relaxed);
}

int shm_ledger_slot(int dev)
{
    std::lock_guard<std::mutex> g(g_mu);
    return g_shm ? slot_of_device(dev) : -1;
}

void shm_ledger_add_slot(int dir, int slot, int64_t bytes, int64_t own)
{
    std::lock_guard<std::mutex> g(g_mu);
    if (!g_shm || slot < 0 || slot >= MMA_MAX_GPUS) return;
    g_shm->bytes[dir][slot].fetch_add((uint64_t)bytes, std::memory_order_relaxed);
    g_shm->own[dir][slot].fetch_add((uint64_t)own, std::memory_order_relaxed);
}

void shm_ledger_get(int dir, int dev, uint64_t* bytes, uint64_t* own)
{
    std::lock_guard<std::mutex> g(g_mu);
    *bytes = *own = 0;
    const int s = slot_of_device(dev);
    if (s < 0) return;
    *bytes = g_shm->bytes[dir][s].load(std::memory_order_relaxed);
    *own = g_shm->own[dir][s].load(std::memory_order_relaxed);
}

}  // namespace mma

using namespace mma;

extern "C" {

int mma_ledger_attach(const char* name)
{
    std::lock_guard<std::mutex> g(g_mu);
    if (g_shm) {
        munmap(g_shm, sizeof(ShmLedger));
        g_shm = nullptr;
    }
    g_cache_init = false;
    if (!name || !*name) return cudaSuccess;
    if (strchr(name, '/') || strlen(name) > 200) return cudaErrorInvalidValue;
    const int fd = shm_open(shm_name(name).c_str(), O_CREAT | O_RDWR, 0600);
    if (fd < 0) return cudaErrorInvalidValue;
    if (ftruncate(fd, sizeof(ShmLedger)) != 0) {
        close(fd);
        return cudaErrorInvalidValue;
    }
    void* p = mmap(nullptr, sizeof(ShmLedger), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) return cudaErrorMemoryAllocation;
    g_shm = (ShmLedger*)p;
    return cudaSuccess;
}

int mma_device_bus_id(int device, char* buf, int len)
{
    if (!buf || len < 13) return cudaErrorInvalidValue;
    return (int)cudaDeviceGetPCIBusId(buf, len, device);
}

int mma_ledger_unlink(const char* name)
{
    if (!name || !*name || strchr(name, '/')) return cudaErrorInvalidValue;
    shm_unlink(shm_name(name).c_str());
    return cudaSuccess;
}

int mma_ledger_shared_add(const char* bus_id, int dir, int64_t bytes, int64_t own)
{
    std::lock_guard<std::mutex> g(g_mu);
    if (!g_shm) return cudaErrorInvalidValue;
    if (dir != MMA_H2D && dir != MMA_D2H) return cudaErrorInvalidValue;
    const int s = slot_of(bus_id);
    if (s < 0) return cudaErrorInvalidValue;
    g_shm->bytes[dir][s].fetch_add((uint64_t)bytes, std::memory_order_relaxed);
    g_shm->own[dir][s].fetch_add((uint64_t)own, std::memory_order_relaxed);
    return cudaSuccess;
}

int mma_ledger_shared_get(const char* bus_id, int dir, uint64_t* bytes, uint64_t* own)
{
    std::lock_guard<std::mutex> g(g_mu);
    if (!g_shm || !bytes || !own) return cudaErrorInvalidValue;
    if (dir != MMA_H2D && dir != MMA_D2H) return cudaErrorInvalidValue;
    const int s = slot_of(bus_id);
    if (s < 0) return cudaErrorInvalidValue;
    *bytes = g_shm->bytes[dir][s].load(std::memory_order_relaxed);
    *own = g_shm->own[dir][s].load(std::memory_order_relaxed);
    return cudaSuccess;
}

}  // extern "C"
