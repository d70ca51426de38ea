// Probe (evidence for SURVEY §8(a) a6/a9): throughput of the relay kernels themselves, with
// hop 1 already complete. A ring of S = n slots holds the whole transfer, every seq flag is
// pre-published (H2D pull) or every credit is free (D2H pack: chunk g < S never waits), so the
// kernel runs at its own speed: claim, flag check, 16-byte coalesced copy slot -> dst, release.
// On one GPU the slot is local HBM (loopback); on an 8-GPU box the pull reads the slot over
// NVLink. Reported: GB/s of payload per configuration (rings x CTAs per ring), and the HBM
// traffic rate (2 bytes per payload byte: read the slot, write the destination).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
//        -I include scripts/probe/probe_relay.cu -o scripts/probe/probe_relay
//   ./scripts/probe/probe_relay [ncu]      (ncu: one launch of the 7 x 8 configuration only)
// "seg" rows (C3): the destination is a table of 32 KiB segments at a seeded
// permutation of block slots (the paged-KV layout), so the pull scatters every slot into 256
// blocks and the pack gathers them.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>
#include <algorithm>

#include "../../paper_2512_16056_b200/csrc/kernels/relay.cu"

#define CK(x) do { cudaError_t e_ = (x); if (e_) { printf("ERR %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

using namespace mma;

static bool g_bulk = false;   // the cp.async.bulk form of the relay kernels

struct RingMem {
    char* stage;
    uint64_t* flags;     // seq[64], credit[64]
    unsigned* cnt;       // cnt[64] + cursor + ready[64] (the engine's layout, plane.cpp get_ring)
};

int main(int argc, char** argv)
{
    const bool ncu = argc > 1 && !strcmp(argv[1], "ncu");

    const uint64_t C = 8ull << 20;          // engine default chunk
    const uint32_t S = 32;                  // slots = chunks per ring: 256 MiB per ring
    const uint64_t per_ring = S * C;
    const int max_rings = 7;                // a target with 7 relay GPUs
    std::vector<RingMem> rm(max_rings);
    char* dst;
    CK(cudaMalloc(&dst, per_ring * max_rings));
    for (auto& r : rm) {
        CK(cudaMalloc(&r.stage, per_ring));
        CK(cudaMemset(r.stage, 0x5A, per_ring));
        CK(cudaMalloc(&r.flags, 128 * sizeof(uint64_t)));
        CK(cudaMalloc(&r.cnt, 64 * sizeof(unsigned) + 64 + 64 * sizeof(uint64_t)));
    }
    int* err;
    CK(cudaHostAlloc(&err, 64, cudaHostAllocMapped));
    memset(err, 0, 64);
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    std::vector<uint64_t> seqs(128, 0);
    for (uint32_t s = 0; s < S; s++) seqs[s] = s + 1;   // chunk g = s staged (g0 = 0)

    // segment table of the scattered form: segment k (32 KiB) of v lives at block perm[k]
    const uint64_t SB = 32 << 10, nseg_max = per_ring * max_rings / SB;
    std::vector<uint64_t> tab(3 * nseg_max + 1);
    {
        std::vector<uint64_t> perm(nseg_max);
        for (uint64_t k = 0; k < nseg_max; k++) perm[k] = k;
        uint64_t x = 0x4D4D41;
        for (uint64_t k = nseg_max - 1; k > 0; k--) {   // seeded Fisher-Yates (splitmix64)
            x += 0x9e3779b97f4a7c15ull;
            uint64_t z = x;
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
            z ^= z >> 31;
            std::swap(perm[k], perm[z % (k + 1)]);
        }
        for (uint64_t k = 0; k <= nseg_max; k++) tab[k] = k * SB;
        for (uint64_t k = 0; k < nseg_max; k++) {
            tab[nseg_max + 1 + k] = (uint64_t)dst + perm[k] * SB;       // src (pack reads it)
            tab[2 * nseg_max + 1 + k] = (uint64_t)dst + perm[k] * SB;   // dst (pull writes it)
        }
    }
    uint64_t* dtab;
    CK(cudaMalloc(&dtab, tab.size() * 8));
    CK(cudaMemcpy(dtab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice));

    auto run = [&](int rings, int ctas, bool pull, uint32_t unit, float* ms_out, bool seg = false) -> int {
        RelayLaunchArg A;
        memset(&A, 0, sizeof(A));
        A.v.nseg = 1;
        A.v.B = per_ring * rings;
        A.v.C = C;
        if (seg) {   // v = the first B / 32 KiB segments of the table
            A.v.nseg = A.v.B / SB;
            A.v.start = dtab;
            A.v.src = dtab + nseg_max + 1;
            A.v.dst = dtab + 2 * nseg_max + 1;
        }
        A.unit_bytes = unit;
        A.err = err;
        A.timeout_ns = 5ull * 1000 * 1000 * 1000;
        // the transfer v = rings contiguous ranges; ring r carries chunks [r*S, (r+1)*S)
        // H2D pull: slot -> dst ; D2H pack: src (dst buffer reused as the source) -> slot
        A.v.src0 = (uint64_t)dst;
        A.v.dst0 = (uint64_t)dst;
        for (int r = 0; r < rings; r++) {
            RingArg& R = A.ring[r];
            R.stage = rm[r].stage;
            R.slot_bytes = C;
            R.seq = rm[r].flags;
            R.credit = rm[r].flags + 64;
            R.cnt = rm[r].cnt;
            R.cursor = (unsigned long long*)((char*)rm[r].cnt + 64 * sizeof(unsigned));
            R.ready = (uint64_t*)((char*)rm[r].cnt + 64 * sizeof(unsigned) + 64);   // leaders / followers
            R.g0 = 0;
            R.unit0 = 0;
            R.chunks.count = S;
            R.chunks.first = (uint64_t)r * S;
            R.S = S;
            R.path = r + 1;
            R.cta_begin = r * ctas;
            R.cta_end = (r + 1) * ctas;
            // reset the ring: seq pre-published (pull) / all zero (pack), counters zero
            if (cudaMemcpy(rm[r].flags, pull ? seqs.data() : std::vector<uint64_t>(128, 0).data(),
                           128 * sizeof(uint64_t), cudaMemcpyHostToDevice)) return 1;
            if (cudaMemset(rm[r].cnt, 0, 64 * sizeof(unsigned) + 64 + 64 * sizeof(uint64_t))) return 1;
        }
        A.nrings = rings;
        cudaEventRecord(a, st);
        if (launch_relay(A, pull, rings * ctas, st, g_bulk) != cudaSuccess) return 1;
        cudaEventRecord(b, st);
        if (cudaEventSynchronize(b) != cudaSuccess) return 1;
        cudaEventElapsedTime(ms_out, a, b);
        return *(volatile int*)err;
    };

    if (argc > 1 && !strcmp(argv[1], "bulk")) {   // vector vs bulk form, contiguous, 1 and 7 rings
        printf("# relay kernels alone, vector form (16-byte loads in registers) vs bulk form (cp.async.bulk\n");
        printf("# through shared memory, 4 x 32 KiB in flight per CTA), 512 KiB units; best of 5\n");
        printf("%-5s %-6s %-6s %-5s %10s %10s\n", "kern", "form", "rings", "ctas", "GB/s", "GB/s/CTA");
        for (int pull = 1; pull >= 0; pull--)
            for (int bulk = 0; bulk < 2; bulk++)
                for (int rings : {1, 7})
                    for (int ctas : {1, 2, 4, 8, 16}) {
                        g_bulk = bulk;
                        float best = 1e30f;
                        for (int rep = 0; rep < 6; rep++) {
                            float ms = 0;
                            int rc = run(rings, ctas, pull, 512u << 10, &ms);
                            if (rc) { printf("ERR run rc=%d\n", rc); return 1; }
                            if (rep) best = std::min(best, ms);
                        }
                        const double gbs = (double)per_ring * rings / (best * 1e-3) / 1e9;
                        printf("%-5s %-6s %-6d %-5d %10.1f %10.1f\n", pull ? "pull" : "pack", bulk ? "bulk" : "vector",
                               rings, ctas, gbs, gbs / (rings * ctas));
                    }
        g_bulk = false;
        return 0;
    }
    if (ncu) {     // one profiled launch per kernel: 7 rings x 8 CTAs (the engine default)
        float ms;
        CK((cudaError_t)run(7, 8, true, 128u << 10, &ms));
        CK((cudaError_t)run(7, 8, false, 128u << 10, &ms));
        CK((cudaError_t)run(7, 8, true, 512u << 10, &ms, true));
        CK((cudaError_t)run(7, 8, false, 512u << 10, &ms, true));
        printf("ncu launches done\n");
        return 0;
    }
    printf("# MMA_UNROLL = %d\n", kUnroll);
    printf("# relay kernels alone (hop 1 complete), 1 x B200 loopback: slots in local HBM\n");
    printf("# C = 8 MiB chunks, S = 32 slots per ring (256 MiB per ring), unit = claim size; best of 5\n");
    printf("%-5s %-6s %-5s %-8s %10s %10s %12s\n", "kern", "rings", "ctas", "unit", "GB/s", "GB/s/CTA", "HBM GB/s");
    for (int pull = 1; pull >= 0; pull--)
        for (int rings : {1, 7})
            for (int ctas : {1, 2, 4, 8, 16, 32})
                for (uint32_t unit : {128u << 10, 512u << 10, 1024u << 10}) {
                    if (rings * ctas > 296) continue;
                    float best = 1e30f;
                    for (int rep = 0; rep < 6; rep++) {
                        float ms = 0;
                        int rc = run(rings, ctas, pull, unit, &ms);
                        if (rc) { printf("ERR run rc=%d\n", rc); return 1; }
                        if (rep) best = std::min(best, ms);
                    }
                    const double gbs = (double)per_ring * rings / (best * 1e-3) / 1e9;
                    printf("%-5s %-6d %-5d %-8u %10.1f %10.1f %12.1f\n", pull ? "pull" : "pack", rings, ctas,
                           unit >> 10, gbs, gbs / (rings * ctas), 2 * gbs);
                }
    printf("# C3 scattered form: v = 32 KiB segments at permuted blocks (the pull scatters, the pack gathers)\n");
    for (int pull = 1; pull >= 0; pull--)
        for (int rings : {1, 7})
            for (int ctas : {8, 32}) {
                float best = 1e30f;
                for (int rep = 0; rep < 6; rep++) {
                    float ms = 0;
                    int rc = run(rings, ctas, pull, 512u << 10, &ms, true);
                    if (rc) { printf("ERR run rc=%d\n", rc); return 1; }
                    if (rep) best = std::min(best, ms);
                }
                const double gbs = (double)per_ring * rings / (best * 1e-3) / 1e9;
                printf("%-5s %-6d %-5d %-8s %10.1f %10.1f %12.1f\n", pull ? "pull" : "pack", rings, ctas, "512seg",
                       gbs, gbs / (rings * ctas), 2 * gbs);
            }
    return 0;
}
