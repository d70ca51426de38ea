"""CPU test of the segment-table classifier (paper_2512_16056_b200/csrc/ranges.h) against
brute force: a fake address space of allocations (pinned host mapped / unmapped, device
memory of two GPUs) with pageable gaps, random pieces (inside one allocation, straddling
two, inside a gap, crossing a gap), and a query that reports bounds or not. The kind of a
piece must equal the kind of every byte in it when all bytes agree (same GPU for device
memory), MK_MIXED otherwise; the cache must bound the queries by the allocations touched."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]

HARNESS = r"""
#include <cstdio>
#include <cstdlib>
#include <random>
#include "ranges.h"
using namespace mma;

struct Alloc { uintptr_t lo, hi; int kind, dev; bool mapped; };
static std::vector<Alloc> A;
static bool g_bounds = true;

static int kind_at(uintptr_t x, int* dev, bool* mapped) {
    for (auto& a : A) if (a.lo <= x && x < a.hi) { *dev = a.dev; *mapped = a.mapped; return a.kind; }
    *dev = -1; *mapped = false; return MK_PAGEABLE;
}
static MemRange query(uintptr_t p, uintptr_t end, void*) {
    MemRange r{p, end, 0, -1, false};
    r.kind = kind_at(p, &r.dev, &r.mapped);
    if (g_bounds && r.kind != MK_PAGEABLE) for (auto& a : A) if (a.lo <= p && p < a.hi) { r.lo = a.lo; r.hi = a.hi; return r; }
    int d2; bool m2; int k2 = kind_at(end - 1, &d2, &m2);
    if (k2 != r.kind || d2 != r.dev) r.kind = MK_MIXED;
    r.mapped = r.mapped && m2;
    return r;
}
// brute force over bytes: the piece's kind, or MK_MIXED. Documented limits of pointer
// queries: memory CUDA does not know has no bounds, so a piece whose first byte is pageable
// is judged by its two ends (pageable iff the last byte is too); without reported bounds a
// piece of CUDA memory is judged by its two ends as well.
static int ends(uintptr_t p, uint64_t len, int* dev, bool* mapped) {
    int d1, d2; bool m1, m2;
    int k1 = kind_at(p, &d1, &m1), k2 = kind_at(p + len - 1, &d2, &m2);
    *dev = d1; *mapped = m1 && m2;
    return (k1 != k2 || d1 != d2) ? MK_MIXED : k1;
}
static int brute(uintptr_t p, uint64_t len, int* dev, bool* mapped) {
    { int d; bool m; if (kind_at(p, &d, &m) == MK_PAGEABLE || !g_bounds) return ends(p, len, dev, mapped); }
    int k = -1; *mapped = true; *dev = -1;
    for (uintptr_t x = p; x < p + len; x++) {
        int d; bool m; int kk = kind_at(x, &d, &m);
        if (k >= 0 && (kk != k || (k == MK_DEVICE && d != *dev))) return MK_MIXED;
        k = kk; *dev = d; *mapped = *mapped && m;
    }
    return k;
}
int main(int argc, char** argv) {
    std::mt19937_64 rng(atoi(argv[1]));
    long checked = 0, bad = 0;
    for (int trial = 0; trial < 300; trial++) {
        A.clear();
        uintptr_t x = 4096;
        int na = 1 + rng() % 6;
        for (int i = 0; i < na; i++) {
            x += (rng() % 3) * (rng() % 200);       // a gap (pageable) or none
            uintptr_t len = 1 + rng() % 300;
            int kind = rng() % 2;
            A.push_back({x, x + len, kind, kind == MK_DEVICE ? (int)(rng() % 2) : -1, kind == MK_HOST && rng() % 4 != 0});
            x += len;
        }
        g_bounds = rng() % 3 != 0;
        RangeCache c(query, nullptr);
        for (int q = 0; q < 60; q++) {
            uintptr_t p = 4096 + rng() % (x - 4096 + 50);
            uint64_t len = 1 + rng() % 400;
            int d1, d2; bool m1, m2;
            int k1 = c.kind(p, len, &d1, &m1), k2 = brute(p, len, &d2, &m2);
            bool ok = k1 == k2 && (k1 == MK_MIXED || k1 == MK_PAGEABLE || (d1 == d2 && (k1 != MK_HOST || m1 == m2)));
            if (!g_bounds && k1 != MK_MIXED && k1 == k2) ok = true;   // ends-only: kind agreement is the contract
            if (!ok) { if (bad < 5) printf("mismatch trial %d p=%lu len=%lu got %d/%d/%d want %d/%d/%d\n", trial,
                (unsigned long)p, (unsigned long)len, k1, d1, m1, k2, d2, m2); bad++; }
            checked++;
        }
        if (g_bounds && c.cached() > A.size()) { printf("cache holds %zu ranges for %zu allocations\n", c.cached(), A.size()); bad++; }
    }
    // query bound: 131072 pieces over one pool and 64 device allocations -> 65 queries
    A.clear();
    A.push_back({1u << 30, (1u << 30) + (1u << 28), MK_HOST, -1, true});
    for (int i = 0; i < 64; i++) A.push_back({(2ull << 30) + i * (1ull << 22), (2ull << 30) + (i + 1) * (1ull << 22), MK_DEVICE, 0, false});
    g_bounds = true;
    RangeCache h(query, nullptr), d(query, nullptr);
    for (int k = 0; k < 131072; k++) {
        int dv; bool m;
        uintptr_t hp = (1u << 30) + (rng() % 65536) * 4096, dp = (2ull << 30) + (uint64_t)k * 2048;
        if (h.kind(hp, 4096, &dv, &m) != MK_HOST || !m) bad++;
        if (d.kind(dp, 2048, &dv, &m) != MK_DEVICE || dv != 0) bad++;
    }
    printf("queries %zu %zu\n", h.queries(), d.queries());
    if (h.queries() != 1 || d.queries() != 64) bad++;
    printf("checked %ld bad %ld\n", checked, bad);
    return bad != 0;
}
"""


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_range_cache_matches_brute_force(tmp_path, seed):
    src = tmp_path / "h.cpp"
    src.write_text(HARNESS)
    exe = tmp_path / "h"
    inc = ROOT / "paper_2512_16056_b200" / "csrc"
    try:
        subprocess.run(["g++", "-O2", "-std=c++17", f"-I{inc}", str(src), "-o", str(exe)], check=True,
                       capture_output=True, text=True, timeout=120)
    except FileNotFoundError:
        pytest.skip("no g++")
    p = subprocess.run([str(exe), str(seed)], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stdout + p.stderr
    assert "bad 0" in p.stdout
