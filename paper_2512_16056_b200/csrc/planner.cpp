// planner.cpp — C5: integer earliest-finish assignment of equal chunks to paths.
//
// The paper assigns micro-tasks online: every PCIe link's outstanding queue pulls work
// while it has room, its own target's queue first (§3.4.2). For a fixed measured
// bandwidth vector (north_star (b)) the same intent -- each chunk goes where it completes
// first, the direct path winning ties -- is the earliest-finish rule, which is optimal for
// equal chunks on uniform links (reading R1). Implemented here with a binary
// heap keyed by each path's finish time after one more chunk, compared exactly as
// rationals in 128-bit integers.
#include "planner.h"

#include <algorithm>

namespace mma {

namespace {

using u128 = unsigned __int128;

struct Key {
    u128 num;       // backlog + (k + 1) * C
    uint32_t den;   // MB/s
    int idx;
};

// strict weak order: earlier finish first, then lower path index ("direct path first")
inline bool earlier(const Key& a, const Key& b)
{
    const u128 l = a.num * b.den, r = b.num * a.den;
    if (l != r) return l < r;
    return a.idx < b.idx;
}

struct HeapCmp {   // std::push_heap builds a max-heap: invert
    bool operator()(const Key& a, const Key& b) const { return earlier(b, a); }
};

}  // namespace

int make_plan(const PlanPath* paths, int npaths, uint64_t B, uint64_t C, uint64_t thr,
              int mode, Plan& out)
{
    out = Plan();
    if (!paths || npaths < 1 || npaths > 255 || C == 0) return -22;
    if (mode != PLAN_CONTIGUOUS && mode != PLAN_INTERLEAVED) return -22;
    int live = 0;
    for (int p = 0; p < npaths; p++) {
        if (paths[p].direct && p != 0) return -22;
        live += paths[p].mbps > 0;
    }
    if (live == 0) return -22;
    out.count.assign(npaths, 0);
    if (B == 0) return 0;

    const bool only_direct = live == 1 && paths[0].direct && paths[0].mbps > 0;
    if (B < thr || only_direct) {       // native single path (§3.2; strict <)
        out.fallback = true;
        out.n = 1;
        out.path.assign(1, 0);
        out.count[0] = 1;
        return 0;
    }

    const uint64_t n = (B - 1) / C + 1;
    out.n = n;
    out.path.resize(n);
    std::vector<Key> heap;
    heap.reserve(npaths);
    for (int p = 0; p < npaths; p++)
        if (paths[p].mbps) heap.push_back(Key{(u128)paths[p].backlog + C, paths[p].mbps, p});
    std::make_heap(heap.begin(), heap.end(), HeapCmp());
    for (uint64_t i = 0; i < n; i++) {
        std::pop_heap(heap.begin(), heap.end(), HeapCmp());
        Key& k = heap.back();
        out.path[i] = (uint8_t)k.idx;
        out.count[k.idx]++;
        k.num += C;
        std::push_heap(heap.begin(), heap.end(), HeapCmp());
    }
    if (mode == PLAN_CONTIGUOUS) {      // each path takes one contiguous range, in path order
        uint64_t i = 0;
        for (int p = 0; p < npaths; p++)
            std::fill_n(out.path.begin() + i, out.count[p], (uint8_t)p), i += out.count[p];
    }
    return 0;
}

}  // namespace mma
