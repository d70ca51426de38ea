// ranges.h — memory-kind classification of a segment table through a per-call cache of
// allocation ranges (SURVEY §8(b) Errors). Header-only and free of CUDA
// types so that tests/test_ranges_cpu.py can compile it against a fake allocation map.
//
// A segment inside a known range takes that range's kind. Ranges come from `query` (in the
// library: cudaPointerGetAttributes for the kind, the driver's RANGE_START_ADDR / RANGE_SIZE
// for the bounds); a piece the query cannot bound (pageable memory, or no range reported) is
// classified as a whole from both of its ends. A piece that crosses the end of a range
// continues in the next one; every part must agree.
#pragma once
#include <stdint.h>

#include <algorithm>
#include <vector>

namespace mma {

enum { MK_HOST = 0, MK_DEVICE = 1, MK_PAGEABLE = 2, MK_MIXED = 3 };

struct MemRange {
    uintptr_t lo, hi;   // [lo, hi)
    int kind;           // MK_*
    int dev;            // device ordinal (MK_DEVICE)
    bool mapped;        // host memory usable by GPU SMs
};

// query(p, end, ctx): the range holding p, or {p, end, kind, ...} when no bounds are known
// (kind MK_MIXED if the two ends of [p, end) differ)
using RangeQueryFn = MemRange (*)(uintptr_t p, uintptr_t end, void* ctx);

class RangeCache {
public:
    RangeCache(RangeQueryFn q, void* ctx) : q_(q), ctx_(ctx) {}

    size_t queries() const { return queries_; }
    size_t cached() const { return v_.size(); }

    // kind of [ptr, ptr + len), len > 0: MK_HOST (*mapped), MK_DEVICE (*dev), MK_PAGEABLE,
    // or MK_MIXED
    int kind(uintptr_t p, uint64_t len, int* dev, bool* mapped)
    {
        const uintptr_t end = p + len;
        int k = -1;
        *mapped = true;
        *dev = -1;
        while (p < end) {
            MemRange r;
            const long at = find(p);
            if (at >= 0) {
                r = v_[(size_t)at];
            } else {
                queries_++;
                r = q_(p, end, ctx_);
                if (r.kind == MK_MIXED) return MK_MIXED;
                if (!(r.lo <= p && p < r.hi)) return MK_MIXED;   // a query that does not hold p
                if (r.lo != p || r.hi != end) insert(r);          // a real range: remember it
                else r.hi = end;
            }
            if (k >= 0 && (r.kind != k || (k == MK_DEVICE && r.dev != *dev))) return MK_MIXED;
            k = r.kind;
            *dev = r.dev;
            *mapped = *mapped && r.mapped;
            p = r.hi;
        }
        return k < 0 ? MK_PAGEABLE : k;
    }

private:
    RangeQueryFn q_;
    void* ctx_;
    std::vector<MemRange> v_;   // sorted by lo, disjoint
    size_t last_ = 0;
    size_t queries_ = 0;

    // index of the cached range holding p, or -1
    long find(uintptr_t p)
    {
        if (last_ < v_.size() && v_[last_].lo <= p && p < v_[last_].hi) return (long)last_;
        size_t lo = 0, hi = v_.size();   // first range with lo > p
        while (lo < hi) {
            const size_t mid = (lo + hi) / 2;
            if (v_[mid].lo > p) hi = mid;
            else lo = mid + 1;
        }
        if (lo == 0 || p >= v_[lo - 1].hi) return -1;
        last_ = lo - 1;
        return (long)last_;
    }

    void insert(const MemRange& r)
    {
        size_t lo = 0, hi = v_.size();
        while (lo < hi) {
            const size_t mid = (lo + hi) / 2;
            if (v_[mid].lo > r.lo) hi = mid;
            else lo = mid + 1;
        }
        v_.insert(v_.begin() + (long)lo, r);
        last_ = lo;
    }
};

}  // namespace mma
