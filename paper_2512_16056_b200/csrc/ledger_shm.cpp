// ledger_shm.cpp — the backlog ledger shared between processes ("a
// shared-memory path ledger"; §5.1.2: with one process per GPU each process keeps
// its own multipath queue, so without a shared view two flows relay through each other's
// links blindly -- Fig 9b's two MMA flows).
//
// One POSIX shared-memory object per name holds, per attached process and per (direction,
// GPU), the bytes that the process's calls still have queued on that GPU's link, and of those
// the bytes of the GPU's own (direct) transfers; a reader sums the live processes' entries. GPUs are keyed by PCI bus id, so processes with different
// CUDA_VISIBLE_DEVICES agree on them. An all-zero object is a valid empty ledger, so creation
// needs no initialisation protocol. Counters are lock-free 64-bit atomics in the mapping.
#include <fcntl.h>
#include <signal.h>
#include <sys/mman.h>
#include <unistd.h>

#include <cerrno>

#include <atomic>

#include "plane.h"

namespace mma {

namespace {

// One entry per attached process, written only by its owner: a process that dies with
// calls in flight leaves counters that readers then ignore (its pid is gone) and the next
// attacher reclaims. Entry 0 holds bytes entered by hand (mma_ledger_shared_add).
constexpr int kEntries = 64;
struct Entry {
    std::atomic<int32_t> pid;                      // 0 = free; entry 0: always live
    uint32_t pad;
    std::atomic<uint64_t> bytes[2][MMA_MAX_GPUS];  // queued on the slot's link
    std::atomic<uint64_t> own[2][MMA_MAX_GPUS];    // of which the slot's own target's direct bytes
};
struct ShmLedger {
    std::atomic<uint32_t> lock;                    // guards the slot and entry tables
    uint32_t pad;
    char bus[MMA_MAX_GPUS][32];                    // PCI bus id per slot ("" = free)
    Entry entry[kEntries];
};
static_assert(std::atomic<uint64_t>::is_always_lock_free, "cross-process atomics must be lock-free");

std::mutex g_mu;
ShmLedger* g_shm = nullptr;
int g_entry = -1;                  // this process's entry
uint64_t g_gen = 0;                // attach generation (InFlight records it)
int g_slot_cache[MMA_MAX_GPUS];    // local device -> slot (-2 = not looked up); reset on attach
bool g_cache_init = false;

std::string shm_name(const char* name) { return std::string("/mma_ledger2_") + name; }

void lock_table()
{
    while (g_shm->lock.exchange(1, std::memory_order_acquire)) {
    }
}
void unlock_table() { g_shm->lock.store(0, std::memory_order_release); }

bool alive(int32_t pid) { return pid > 0 && (kill(pid, 0) == 0 || errno == EPERM); }

// slot of a bus id (claimed on first use); -1 when the table is full
int slot_of(const char* bus)
{
    if (!g_shm || !bus || !*bus) return -1;
    lock_table();
    int found = -1, free_slot = -1;
    for (int s = 0; s < MMA_MAX_GPUS; s++) {
        if (!strncmp(g_shm->bus[s], bus, sizeof g_shm->bus[s])) { found = s; break; }
        if (free_slot < 0 && !g_shm->bus[s][0]) free_slot = s;
    }
    if (found < 0 && free_slot >= 0) {
        strncpy(g_shm->bus[free_slot], bus, sizeof g_shm->bus[free_slot] - 1);
        found = free_slot;
    }
    unlock_table();
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
        // a virtual GPU (MMA_VGPUS) shares its device's entry
        if (cudaDeviceGetPCIBusId(bus, sizeof bus - 1, phys_dev(dev)) != cudaSuccess) {
            cudaGetLastError();
            return -1;
        }
        g_slot_cache[dev] = slot_of(bus);
    }
    return g_slot_cache[dev];
}

void clear_entry(Entry& e)
{
    for (int d = 0; d < 2; d++)
        for (int s = 0; s < MMA_MAX_GPUS; s++) {
            e.bytes[d][s].store(0, std::memory_order_relaxed);
            e.own[d][s].store(0, std::memory_order_relaxed);
        }
}

void add(Entry& e, int dir, int slot, int64_t bytes, int64_t own)
{
    e.bytes[dir][slot].fetch_add((uint64_t)bytes, std::memory_order_relaxed);
    e.own[dir][slot].fetch_add((uint64_t)own, std::memory_order_relaxed);
}

// sum over the live entries
void sum(int dir, int slot, uint64_t* bytes, uint64_t* own)
{
    *bytes = *own = 0;
    for (int k = 0; k < kEntries; k++) {
        Entry& e = g_shm->entry[k];
        if (k != 0 && !alive(e.pid.load(std::memory_order_relaxed))) continue;
        *bytes += e.bytes[dir][slot].load(std::memory_order_relaxed);
        *own += e.own[dir][slot].load(std::memory_order_relaxed);
    }
}

// give this process's entry back (its in-flight bytes leave the ledger with it)
void detach_locked()
{
    if (!g_shm) return;
    if (g_entry > 0) {
        clear_entry(g_shm->entry[g_entry]);
        g_shm->entry[g_entry].pid.store(0, std::memory_order_release);
    }
    munmap(g_shm, sizeof(ShmLedger));
    g_shm = nullptr;
    g_entry = -1;
}
}  // namespace

bool shm_ledger_on()
{
    std::lock_guard<std::mutex> g(g_mu);
    return g_shm != nullptr;
}

uint64_t shm_ledger_gen()
{
    std::lock_guard<std::mutex> g(g_mu);
    return g_shm ? g_gen : 0;
}

void shm_ledger_add(int dir, int dev, int64_t bytes, int64_t own, uint64_t gen)
{
    std::lock_guard<std::mutex> g(g_mu);
    if (!g_shm || g_entry < 0 || gen != g_gen) return;   // entered under another attach: gone with it
    const int s = slot_of_device(dev);
    if (s < 0) return;
    add(g_shm->entry[g_entry], dir, s, bytes, own);
}

int shm_ledger_slot(int dev)
{
    std::lock_guard<std::mutex> g(g_mu);
    return g_shm ? slot_of_device(dev) : -1;
}

void shm_ledger_add_slot(int dir, int slot, int64_t bytes, int64_t own, uint64_t gen)
{
    std::lock_guard<std::mutex> g(g_mu);
    if (!g_shm || g_entry < 0 || gen != g_gen || slot < 0 || slot >= MMA_MAX_GPUS) return;
    add(g_shm->entry[g_entry], dir, slot, bytes, own);
}

void shm_ledger_get(int dir, int dev, uint64_t* bytes, uint64_t* own)
{
    std::lock_guard<std::mutex> g(g_mu);
    *bytes = *own = 0;
    const int s = slot_of_device(dev);
    if (s < 0) return;
    sum(dir, s, bytes, own);
}

}  // namespace mma

using namespace mma;

extern "C" {

int mma_ledger_attach(const char* name)
{
    std::lock_guard<std::mutex> g(g_mu);
    detach_locked();
    g_cache_init = false;
    g_gen++;
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
    // claim an entry: our own (re-attach), a dead process's, or a free one
    const int32_t me = (int32_t)getpid();
    lock_table();
    int pick = -1;
    for (int k = 1; k < kEntries && pick < 0; k++)
        if (g_shm->entry[k].pid.load(std::memory_order_relaxed) == me) pick = k;
    for (int k = 1; k < kEntries && pick < 0; k++)
        if (!alive(g_shm->entry[k].pid.load(std::memory_order_relaxed))) pick = k;
    if (pick > 0) {
        clear_entry(g_shm->entry[pick]);
        g_shm->entry[pick].pid.store(me, std::memory_order_release);
    }
    unlock_table();
    if (pick < 0) {   // 63 live processes already: no room
        munmap(g_shm, sizeof(ShmLedger));
        g_shm = nullptr;
        return cudaErrorMemoryAllocation;
    }
    g_entry = pick;
    return cudaSuccess;
}

int mma_device_bus_id(int device, char* buf, int len)
{
    if (!buf || len < 13) return cudaErrorInvalidValue;
    return (int)cudaDeviceGetPCIBusId(buf, len, phys_dev(device));
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
    add(g_shm->entry[0], dir, s, bytes, own);   // the hand-entered entry (always live)
    return cudaSuccess;
}

int mma_ledger_process_add(const char* bus_id, int dir, int64_t bytes, int64_t own)
{
    std::lock_guard<std::mutex> g(g_mu);
    if (!g_shm || g_entry < 0) return cudaErrorInvalidValue;
    if (dir != MMA_H2D && dir != MMA_D2H) return cudaErrorInvalidValue;
    const int s = slot_of(bus_id);
    if (s < 0) return cudaErrorInvalidValue;
    add(g_shm->entry[g_entry], dir, s, bytes, own);   // this process's entry, as its calls do
    return cudaSuccess;
}

int mma_ledger_shared_get(const char* bus_id, int dir, uint64_t* bytes, uint64_t* own)
{
    std::lock_guard<std::mutex> g(g_mu);
    if (!g_shm || !bytes || !own) return cudaErrorInvalidValue;
    if (dir != MMA_H2D && dir != MMA_D2H) return cudaErrorInvalidValue;
    const int s = slot_of(bus_id);
    if (s < 0) return cudaErrorInvalidValue;
    sum(dir, s, bytes, own);
    return cudaSuccess;
}

}  // extern "C"
