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

// ---- joint plan (NEXT-1). Links wait in a heap keyed by the time they become free (chunks
// pulled x C / rate, compared exactly); each endpoint's queue is a FIFO cursor over its
// transfers. Queue lengths are few (<= the link count), so the longest is found by a scan.
int make_plan_multi(const std::vector<MultiLink>& links, const std::vector<std::vector<uint8_t>>& carry,
                    const std::vector<int>& target, const std::vector<uint64_t>& nchunks, uint64_t C, int mode,
                    std::vector<std::vector<int>>& link_of_chunk, int prefer)
{
    const int L = (int)links.size(), T = (int)target.size();
    if (L < 1 || L > 128 || C == 0 || (int)nchunks.size() != T || (int)carry.size() != L) return -22;
    if (mode != PLAN_CONTIGUOUS && mode != PLAN_INTERLEAVED) return -22;
    auto may = [&](int d, int l) { return l == d || carry[d][l] != 0; };
    struct Queue {
        uint64_t left = 0;
        std::vector<int> transfers;   // to this endpoint, in call order
        size_t ti = 0;                // current transfer (index into transfers)
        uint64_t next = 0;            // next chunk of it
    };
    std::vector<Queue> q(L);
    link_of_chunk.assign(T, {});
    for (int t = 0; t < T; t++) {
        if (target[t] < 0 || target[t] >= L) return -22;
        link_of_chunk[t].assign(nchunks[t], -1);
        if (!nchunks[t]) continue;
        bool any = false;
        for (int l = 0; l < L && !any; l++) any = links[l].mbps && may(target[t], l);
        if (!any) return -22;
        q[target[t]].left += nchunks[t];
        q[target[t]].transfers.push_back(t);
    }
    std::vector<Key> heap;   // num = chunks pulled * C, den = rate, idx = link
    for (int l = 0; l < L; l++)
        if (links[l].mbps) heap.push_back(Key{0, links[l].mbps, l});
    std::make_heap(heap.begin(), heap.end(), HeapCmp());
    std::vector<std::vector<uint64_t>> cnt(T, std::vector<uint64_t>(L, 0));
    uint64_t remaining = 0;
    for (const Queue& x : q) remaining += x.left;
    while (remaining && !heap.empty()) {
        std::pop_heap(heap.begin(), heap.end(), HeapCmp());
        Key k = heap.back();
        heap.pop_back();
        const int l = k.idx;
        int d = -1;
        if (q[l].left) d = l;   // direct path first
        else if (prefer >= 0 && prefer < L && prefer != l && q[prefer].left && may(prefer, l)) d = prefer;
        else
            for (int e = 0; e < L; e++)   // longest queue it may relay for; ties: lower id
                if (e != l && q[e].left && may(e, l) && (d < 0 || q[e].left > q[d].left)) d = e;
        if (d < 0) continue;   // nothing this link may take, now or later: it leaves the heap
        Queue& Q = q[d];
        while (Q.next >= nchunks[Q.transfers[Q.ti]]) { Q.ti++; Q.next = 0; }
        const int t = Q.transfers[Q.ti];
        link_of_chunk[t][Q.next++] = l;
        cnt[t][l]++;
        Q.left--;
        remaining--;
        k.num += C;
        heap.push_back(k);
        std::push_heap(heap.begin(), heap.end(), HeapCmp());
    }
    if (remaining) return -22;
    if (mode == PLAN_CONTIGUOUS)
        for (int t = 0; t < T; t++) {
            auto& v = link_of_chunk[t];
            size_t i = 0;
            const int d = target[t];
            for (uint64_t c = 0; c < cnt[t][d]; c++) v[i++] = d;
            for (int l = 0; l < L; l++)
                if (l != d)
                    for (uint64_t c = 0; c < cnt[t][l]; c++) v[i++] = l;
        }
    return 0;
}

}  // namespace mma
