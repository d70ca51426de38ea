/*
 * mma_oracle.c — CPU oracle for MMA's multipath host<->GPU copy (arXiv 2512.16056).
 * TEST INFRASTRUCTURE ONLY (see mma_oracle.h): never linked into the product path.
 *
 * Written from the paper (P: = /root/reference/PAPER.md line) and the readings listed in
 * DESIGN.md §3. Plain C11 + pthreads; no blocking, fusion or reordering beyond what the
 * cited passages state. Slow on purpose.
 */
#include "mma_oracle.h"

#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ---------------------------------------------------------------- chunking --- */

/* "divides the original transfer task into multiple micro-tasks according to a fixed chunk
 * size" (§3.4.1). The last micro-task holds the remainder, unpadded (reading R4). */
uint64_t orc_nchunks(uint64_t B, uint64_t C)
{
    if (B == 0 || C == 0) return 0;   /* C = 0 is invalid; callers reject it */
    return B / C + (B % C != 0);
}

void orc_chunk_extent(uint64_t i, uint64_t B, uint64_t C, uint64_t* off, uint64_t* len)
{
    uint64_t a = i * C;
    uint64_t b = a + C;
    if (b > B) b = B;
    *off = a;
    *len = b - a;
}

/* ------------------------------------------------------------- assignment --- */

/* Earliest finish: is path p's finish time after taking one more chunk strictly earlier
 * than path q's?  (backlog_p + (k_p+1)C)/bw_p < (backlog_q + (k_q+1)C)/bw_q, compared by
 * cross-multiplication in 128-bit integers (reading R1). */
static int ef_less(const orc_path* paths, const uint64_t* k, uint64_t C, int p, int q)
{
    u128 fp = (u128)paths[p].backlog + (u128)(k[p] + 1) * C;
    u128 fq = (u128)paths[q].backlog + (u128)(k[q] + 1) * C;
    return fp * paths[q].bw_mbps < fq * paths[p].bw_mbps;
}

/* Pull rule under constant rates: the path that becomes free first takes the next chunk
 * ("links without congestion can continuously consume micro-tasks"). Compares the
 * current free times (backlog_p + k_p C)/bw_p. Oracle-only comparison mode. */
static int pull_less(const orc_path* paths, const uint64_t* k, uint64_t C, int p, int q)
{
    u128 fp = (u128)paths[p].backlog + (u128)k[p] * C;
    u128 fq = (u128)paths[q].backlog + (u128)k[q] * C;
    return fp * paths[q].bw_mbps < fq * paths[p].bw_mbps;
}

int orc_plan(const orc_path* paths, int P, uint64_t B, uint64_t C, uint64_t thr, int mode,
             uint8_t* path_of_chunk, uint64_t cap, uint64_t* nchunks, uint64_t* counts,
             int* fallback)
{
    if (!paths || P < 1 || P > 255 || C == 0 || !nchunks || !counts || !fallback)
        return ORC_EINVAL;
    if (mode != ORC_CONTIG && mode != ORC_INTERLEAVED && mode != ORC_PULL) return ORC_EINVAL;
    int usable = 0;
    for (int p = 0; p < P; p++) {
        if (paths[p].kind != ORC_RELAY && !(p == 0 && paths[p].kind == ORC_DIRECT))
            return ORC_EINVAL;               /* a direct path may only be path 0 (R2) */
        counts[p] = 0;
        if (paths[p].bw_mbps > 0) usable++;  /* a path with bw = 0 is dropped */
    }
    if (usable == 0) return ORC_EINVAL;
    *fallback = 0;
    *nchunks = 0;
    if (B == 0) return 0;                    /* cudaMemcpyAsync semantics: no-op (R6) */

    /* Fallback: "Transfer tasks with data sizes below a specific threshold automatically
     * revert to native single-path transfer" (§3.2), strict < (R5). A set whose only
     * usable path is the direct one is the native copy as well. */
    int direct_only = (usable == 1 && paths[0].kind == ORC_DIRECT && paths[0].bw_mbps > 0);
    if (B < thr || direct_only) {
        if (cap < 1 || !path_of_chunk) return ORC_ENOSPC;
        path_of_chunk[0] = 0;
        counts[0] = 1;
        *nchunks = 1;
        *fallback = 1;
        return 0;
    }

    uint64_t n = orc_nchunks(B, C);
    if (cap < n || !path_of_chunk) return ORC_ENOSPC;
    /* Chunk i goes to the best path by the mode's rule; ties keep the lower path index,
     * which makes the direct path (index 0) win ties: "direct path first". */
    for (uint64_t i = 0; i < n; i++) {
        int best = -1;
        for (int p = 0; p < P; p++) {
            if (paths[p].bw_mbps == 0) continue;
            if (best < 0) { best = p; continue; }
            int less = (mode == ORC_PULL) ? pull_less(paths, counts, C, p, best)
                                          : ef_less(paths, counts, C, p, best);
            if (less) best = p;
        }
        counts[best] += 1;
        if (mode != ORC_CONTIG) path_of_chunk[i] = (uint8_t)best;
    }
    if (mode == ORC_CONTIG) {                /* [0]*k0 ++ [1]*k1 ++ ... (reading R1) */
        uint64_t i = 0;
        for (int p = 0; p < P; p++)
            for (uint64_t c = 0; c < counts[p]; c++) path_of_chunk[i++] = (uint8_t)p;
    }
    *nchunks = n;
    return 0;
}

/* ------------------------------------ joint plan of concurrent transfers --- */

/* May link l take chunks of endpoint GPU d? Its own GPU's queue always; others by relay_ok. */
static int may_carry(int L, const uint8_t* relay_ok, int d, int l)
{
    return l == d || relay_ok[(size_t)d * L + l];
}

int orc_plan_multi(int L, const uint32_t* link_bw, const uint8_t* relay_ok, int T,
                   const int32_t* target, const uint64_t* nchunks, uint64_t C, int mode,
                   int prefer, int32_t* link_of_chunk)
{
    if (L < 1 || L > 128 || T < 0 || !link_bw || !relay_ok || (T && (!target || !nchunks)) || C == 0)
        return ORC_EINVAL;
    if (mode != ORC_INTERLEAVED && mode != ORC_CONTIG) return ORC_EINVAL;
    uint64_t total = 0;
    for (int t = 0; t < T; t++) {
        if (target[t] < 0 || target[t] >= L) return ORC_EINVAL;
        int any = 0;
        for (int l = 0; l < L; l++) any |= link_bw[l] > 0 && may_carry(L, relay_ok, target[t], l);
        if (!any && nchunks[t]) return ORC_EINVAL;
        total += nchunks[t];
    }
    /* the queue of GPU d: transfers to d in order, each transfer's chunks in order */
    uint64_t* first = calloc((size_t)T + 1, sizeof(uint64_t));   /* transfer t's first out index */
    uint64_t* left = calloc((size_t)L, sizeof(uint64_t));        /* chunks waiting per queue */
    int* cur_t = calloc((size_t)L, sizeof(int));                 /* head: transfer, chunk */
    uint64_t* cur_c = calloc((size_t)L, sizeof(uint64_t));
    uint64_t* taken = calloc((size_t)L, sizeof(uint64_t));       /* chunks pulled per link */
    int* live = calloc((size_t)L, sizeof(int));
    uint64_t* cnt = calloc((size_t)T * L + 1, sizeof(uint64_t)); /* per transfer, per link */
    if (!first || !left || !cur_t || !cur_c || !taken || !live || !cnt) {
        free(first); free(left); free(cur_t); free(cur_c); free(taken); free(live); free(cnt);
        return ORC_EINVAL;
    }
    for (int t = 0; t < T; t++) first[t + 1] = first[t] + nchunks[t];
    for (int d = 0; d < L; d++) {
        cur_t[d] = -1;
        for (int t = 0; t < T; t++)
            if (target[t] == d) {
                left[d] += nchunks[t];
                if (cur_t[d] < 0 && nchunks[t]) cur_t[d] = t;
            }
    }
    for (int l = 0; l < L; l++) live[l] = link_bw[l] > 0;
    for (uint64_t step = 0; step < total; step++) {
        /* the live link that is free first: taken_l * C / bw_l smallest, ties -> lower id */
        int best = -1;
        for (int l = 0; l < L; l++) {
            if (!live[l]) continue;
            if (best < 0) { best = l; continue; }
            u128 a = (u128)taken[l] * C * link_bw[best], b = (u128)taken[best] * C * link_bw[l];
            if (a < b) best = l;
        }
        if (best < 0) break;
        /* what it takes: its own queue first, else the longest queue it may relay for */
        int q = -1;
        if (left[best] > 0) q = best;
        else if (prefer >= 0 && prefer < L && prefer != best && left[prefer] > 0 && may_carry(L, relay_ok, prefer, best))
            q = prefer;                                      /* the preferred GPU's queue */
        else
            for (int d = 0; d < L; d++)
                if (d != best && left[d] > 0 && may_carry(L, relay_ok, d, best) && (q < 0 || left[d] > left[q])) q = d;
        if (q < 0) { live[best] = 0; step--; continue; }   /* nothing to take, ever again */
        int t = cur_t[q];
        uint64_t c = cur_c[q];
        link_of_chunk[first[t] + c] = best;
        cnt[(size_t)t * L + best]++;
        taken[best]++;
        left[q]--;
        if (++cur_c[q] == nchunks[t]) {                      /* next transfer of this queue */
            cur_c[q] = 0;
            int nt = -1;
            for (int u = t + 1; u < T; u++)
                if (target[u] == q && nchunks[u]) { nt = u; break; }
            cur_t[q] = nt;
        }
    }
    if (mode == ORC_CONTIG)                                  /* own link first, then by id */
        for (int t = 0; t < T; t++) {
            uint64_t i = first[t];
            int d = target[t];
            for (uint64_t c = 0; c < cnt[(size_t)t * L + d]; c++) link_of_chunk[i++] = d;
            for (int l = 0; l < L; l++)
                if (l != d)
                    for (uint64_t c = 0; c < cnt[(size_t)t * L + l]; c++) link_of_chunk[i++] = l;
        }
    free(first); free(left); free(cur_t); free(cur_c); free(taken); free(live); free(cnt);
    return 0;
}

void orc_predict(const orc_path* paths, int P, uint64_t B, uint64_t C,
                 const uint8_t* path_of_chunk, uint64_t n, double* T_s, double* agg_gbps)
{
    uint64_t bytes[256] = {0};
    for (uint64_t i = 0; i < n; i++) {
        uint64_t off, len;
        if (n == 1) { off = 0; len = B; }     /* a fallback plan is one piece [0, B) */
        else orc_chunk_extent(i, B, C, &off, &len);
        bytes[path_of_chunk[i]] += len;
    }
    double T = 0.0;
    for (int p = 0; p < P; p++) {
        if (bytes[p] == 0 || paths[p].bw_mbps == 0) continue;
        double t = (double)(paths[p].backlog + bytes[p]) / ((double)paths[p].bw_mbps * 1e6);
        if (t > T) T = t;
    }
    *T_s = T;
    *agg_gbps = (T > 0.0) ? (double)B / T / 1e9 : 0.0;
}

/* ------------------------------------------------- the virtual stream v (segments) --- */

typedef struct {
    const orc_segment* segs;
    uint64_t nsegs;
    uint64_t* start;      /* start[k] = offset of segment k in v; start[nsegs] = B */
    uint32_t* wcount;     /* per-byte write counters of v, or NULL */
} vstream;

static int vs_init(vstream* vs, const orc_segment* segs, uint64_t nsegs, uint32_t* wc)
{
    vs->segs = segs;
    vs->nsegs = nsegs;
    vs->wcount = wc;
    vs->start = (uint64_t*)malloc((nsegs + 1) * sizeof(uint64_t));
    if (!vs->start) return ORC_EINVAL;
    vs->start[0] = 0;
    for (uint64_t k = 0; k < nsegs; k++) vs->start[k + 1] = vs->start[k] + segs[k].len;
    return 0;
}

/* first segment k with start[k+1] > x */
static uint64_t vs_find(const vstream* vs, uint64_t x)
{
    uint64_t lo = 0, hi = vs->nsegs;
    while (lo < hi) {
        uint64_t mid = (lo + hi) / 2;
        if (vs->start[mid + 1] > x) hi = mid; else lo = mid + 1;
    }
    return lo;
}

/* what: 0 = src -> dst (direct), 1 = src -> buf (pack, relay hop1), 2 = buf -> dst (unpack,
 * relay hop2). Copies the part of each segment that overlaps v[a, b): byte x of v lives at
 * src_k + (x - v_k) and goes to dst_k + (x - v_k) (north_star (e)). */
static void vs_copy(const vstream* vs, uint64_t a, uint64_t b, int what, unsigned char* buf)
{
    if (a >= b) return;
    for (uint64_t k = vs_find(vs, a); k < vs->nsegs && vs->start[k] < b; k++) {
        uint64_t lo = vs->start[k] > a ? vs->start[k] : a;
        uint64_t hi = vs->start[k + 1] < b ? vs->start[k + 1] : b;
        if (lo >= hi) continue;
        const unsigned char* s = (const unsigned char*)vs->segs[k].src + (lo - vs->start[k]);
        unsigned char* d = (unsigned char*)vs->segs[k].dst + (lo - vs->start[k]);
        if (what == 0) memcpy(d, s, hi - lo);
        else if (what == 1) memcpy(buf + (lo - a), s, hi - lo);
        else memcpy(d, buf + (lo - a), hi - lo);
        if (what != 1 && vs->wcount)
            for (uint64_t x = lo; x < hi; x++) vs->wcount[x] += 1;
    }
}

/* ---------------------------------------------------- NUMA-affine order (R23) --- */

/* Bucket pass, one group at a time, written for the eye rather than for speed: collect the
 * groups' nodes in the reading's order, then for each group append its segments in table
 * order; the unknown group last. */
void orc_numa_order(const int32_t* seg_node, uint64_t nsegs, const orc_path* paths,
                    const int32_t* path_node, int P, uint32_t* order)
{
    int32_t groups[256];
    int ng = 0, npath_nodes;
    for (int p = 0; p < P; p++) {                       /* path nodes, in path order */
        if (paths[p].bw_mbps == 0 || path_node[p] < 0) continue;
        int seen = 0;
        for (int g = 0; g < ng; g++) seen |= groups[g] == path_node[p];
        if (!seen && ng < 256) groups[ng++] = path_node[p];
    }
    npath_nodes = ng;
    for (uint64_t k = 0; k < nsegs; k++) order[k] = (uint32_t)k;
    if (npath_nodes < 2 || nsegs < 2) return;           /* as given */
    for (;;) {                                          /* other known nodes, ascending */
        int32_t next = -1;
        for (uint64_t k = 0; k < nsegs; k++) {
            int32_t nd = seg_node[k], listed = 0;
            if (nd < 0) continue;
            for (int g = 0; g < ng; g++) listed |= groups[g] == nd;
            if (!listed && (next < 0 || nd < next)) next = nd;
        }
        if (next < 0 || ng >= 255) break;
        groups[ng++] = next;
    }
    groups[ng++] = -1;                                  /* unknown last */
    uint64_t o = 0;
    for (int g = 0; g < ng; g++)
        for (uint64_t k = 0; k < nsegs; k++) {
            int32_t nd = seg_node[k] < 0 ? -1 : seg_node[k];
            if (nd == groups[g]) order[o++] = (uint32_t)k;
        }
}

static int cmp_dst(const void* x, const void* y)
{
    const orc_segment* a = (const orc_segment*)x;
    const orc_segment* b = (const orc_segment*)y;
    uintptr_t pa = (uintptr_t)a->dst, pb = (uintptr_t)b->dst;
    return pa < pb ? -1 : pa > pb;
}

int orc_segments_disjoint(const orc_segment* segs, uint64_t nsegs)
{
    orc_segment* s = (orc_segment*)malloc((nsegs ? nsegs : 1) * sizeof(orc_segment));
    if (!s) return 0;
    uint64_t m = 0;
    for (uint64_t k = 0; k < nsegs; k++)
        if (segs[k].len > 0) s[m++] = segs[k];   /* empty segments cover no bytes */
    qsort(s, m, sizeof(orc_segment), cmp_dst);
    int ok = 1;
    for (uint64_t k = 1; k < m; k++)
        if ((uintptr_t)s[k - 1].dst + s[k - 1].len > (uintptr_t)s[k].dst) { ok = 0; break; }
    free(s);
    return ok;
}

/* --------------------------------------------------- the relay ring --- */
/*
 * One ring per relay path: S staging slots of C bytes, seq[S] and credit[S] flags.
 * The ring's j-th chunk in this call has global index g = base + j, uses slot s = g mod S
 * and sequence value g + 1 (readings R8, R18).
 *   producer (hop1: relay's PCIe):  if g >= S wait credit[s] >= g - S + 1;
 *                                   copy chunk into slot s; release seq[s] = g + 1
 *   consumer (hop2: NVLink):        acquire-wait seq[s] == g + 1; copy slot s to dst;
 *                                   release credit[s] = g + 1
 * This is the dual-pipeline relay of P:588-594 ("two relay streams ... each relay stream
 * has a dedicated relay buffer ... limited to one data chunk") with S buffers; S = 2 is the
 * paper's configuration. "a dependency established between these operations" is
 * the seq flag.
 */
typedef struct {
    int path;
    uint64_t base;
    uint32_t S;
    uint64_t* chunks;     /* chunk indices carried by this ring, ascending */
    uint64_t nchunks;
    unsigned char* stage; /* S * C bytes */
    _Atomic uint64_t* seq;
    _Atomic uint64_t* credit;
    /* actor program counters (deterministic mode) */
    uint64_t pj, cj;
    int pstep, cstep;
} ring_t;

typedef struct {
    vstream vs;
    uint64_t B, C, n;
    uint64_t slot_bytes;  /* C, or B for a one-piece (fallback) plan */
    const uint8_t* path_of_chunk;
    uint64_t* events;
    _Atomic uint64_t clock;
    int fault;
    uint64_t* direct;     /* chunk indices on the direct path, ascending */
    uint64_t ndirect;
    ring_t* rings;
    int nrings;
} mover_t;

static uint64_t tick(mover_t* m) { return atomic_fetch_add(&m->clock, 1) + 1; }

static void stamp(mover_t* m, uint64_t chunk, int ev, uint64_t t)
{
    if (m->events) m->events[chunk * ORC_NEV + ev] = t;
}

static void extent(const mover_t* m, uint64_t i, uint64_t* a, uint64_t* b)
{
    uint64_t off, len;
    if (m->n == 1) { off = 0; len = m->B; }
    else orc_chunk_extent(i, m->B, m->C, &off, &len);
    *a = off;
    *b = off + len;
}

/* Initial flag values of a ring that has already carried `base` chunks: slot s last held
 * the largest g < base with g mod S = s, whose seq and credit both equal g + 1. */
static void ring_init_flags(ring_t* r)
{
    for (uint32_t s = 0; s < r->S; s++) {
        uint64_t v = 0;
        if (r->base > s) {
            uint64_t g = r->base - 1 - ((r->base - 1 - s) % r->S);
            v = g + 1;
        }
        atomic_store(&r->seq[s], v);
        atomic_store(&r->credit[s], v);
    }
}

/* Deterministic single-thread execution: actors take one step each in round-robin order;
 * a blocked wait skips its turn. Producer steps: 0 wait credit, 1 copy first half (stage
 * begins), 2 copy second half (stage ends), 3 publish. Consumer steps: 0 wait seq, 1 copy
 * first half (forward begins), 2 copy second half (forward ends), 3 credit. */
static int producer_step(mover_t* m, ring_t* r)
{
    if (r->pj >= r->nchunks) return 0;
    uint64_t i = r->chunks[r->pj], g = r->base + r->pj, a, b;
    uint32_t s = (uint32_t)(g % r->S);
    unsigned char* slot = r->stage + (uint64_t)s * m->slot_bytes;
    extent(m, i, &a, &b);
    uint64_t mid = a + (b - a) / 2;
    int step = r->pstep;
    if (m->fault == ORC_FAULT_PUBLISH_EARLY) {   /* seeded bug: publish before the copy */
        static const int order[4] = {0, 3, 1, 2};
        step = order[r->pstep];
    }
    switch (step) {
    case 0:
        if (m->fault != ORC_FAULT_SKIP_CREDIT && g >= r->S &&
            atomic_load_explicit(&r->credit[s], memory_order_acquire) < g - r->S + 1)
            return 0;                                 /* blocked */
        break;
    case 1:
        stamp(m, i, ORC_EV_STAGE_BEGIN, tick(m));
        vs_copy(&m->vs, a, mid, 1, slot);
        break;
    case 2:
        vs_copy(&m->vs, mid, b, 1, slot + (mid - a));
        stamp(m, i, ORC_EV_STAGE_END, tick(m));
        break;
    case 3:
        stamp(m, i, ORC_EV_PUBLISH, tick(m));
        atomic_store_explicit(&r->seq[s], g + 1, memory_order_release);
        break;
    }
    if (++r->pstep == 4) { r->pstep = 0; r->pj++; }
    return 1;
}

static int consumer_step(mover_t* m, ring_t* r)
{
    if (r->cj >= r->nchunks) return 0;
    uint64_t i = r->chunks[r->cj], g = r->base + r->cj, a, b;
    uint32_t s = (uint32_t)(g % r->S);
    unsigned char* slot = r->stage + (uint64_t)s * m->slot_bytes;
    extent(m, i, &a, &b);
    uint64_t mid = a + (b - a) / 2;
    switch (r->cstep) {
    case 0:
        if (atomic_load_explicit(&r->seq[s], memory_order_acquire) != g + 1) return 0;
        break;
    case 1:
        stamp(m, i, ORC_EV_FWD_BEGIN, tick(m));
        vs_copy(&m->vs, a, mid, 2, slot);
        break;
    case 2:
        vs_copy(&m->vs, mid, b, 2, slot + (mid - a));
        stamp(m, i, ORC_EV_FWD_END, tick(m));
        break;
    case 3:
        stamp(m, i, ORC_EV_CREDIT, tick(m));
        atomic_store_explicit(&r->credit[s], g + 1, memory_order_release);
        break;
    }
    if (++r->cstep == 4) { r->cstep = 0; r->cj++; }
    return 1;
}

static int run_deterministic(mover_t* m)
{
    uint64_t dj = 0;
    for (;;) {
        int progressed = 0, pending = 0;
        if (dj < m->ndirect) {            /* direct path: one DMA per chunk */
            uint64_t a, b;
            extent(m, m->direct[dj], &a, &b);
            vs_copy(&m->vs, a, b, 0, NULL);
            dj++;
            progressed = 1;
        }
        for (int k = 0; k < m->nrings; k++) {
            ring_t* r = &m->rings[k];
            progressed |= producer_step(m, r);
            progressed |= consumer_step(m, r);
            pending |= (r->pj < r->nchunks) || (r->cj < r->nchunks);
        }
        pending |= dj < m->ndirect;
        if (!pending) return 0;
        if (!progressed) return ORC_EDEADLK;
    }
}

/* Threaded execution: one thread for the direct path, a producer and a consumer thread per
 * relay ring, synchronised only through the acquire/release seq and credit flags. Each
 * spin is bounded so a protocol bug reports EDEADLK instead of hanging. */
typedef struct { mover_t* m; ring_t* r; int role; int rc; } thr_arg;

#define SPIN_LIMIT (1ull << 34)

static void* thread_main(void* p)
{
    thr_arg* t = (thr_arg*)p;
    mover_t* m = t->m;
    ring_t* r = t->r;
    t->rc = 0;
    if (t->role == 0) {
        for (uint64_t j = 0; j < m->ndirect; j++) {
            uint64_t a, b;
            extent(m, m->direct[j], &a, &b);
            vs_copy(&m->vs, a, b, 0, NULL);
        }
        return NULL;
    }
    for (uint64_t j = 0; j < r->nchunks; j++) {
        uint64_t i = r->chunks[j], g = r->base + j, a, b;
        uint32_t s = (uint32_t)(g % r->S);
        unsigned char* slot = r->stage + (uint64_t)s * m->slot_bytes;
        extent(m, i, &a, &b);
        if (t->role == 1) {                                   /* producer */
            if (m->fault != ORC_FAULT_SKIP_CREDIT && g >= r->S) {
                uint64_t spins = 0;
                while (atomic_load_explicit(&r->credit[s], memory_order_acquire) < g - r->S + 1)
                    if (++spins > SPIN_LIMIT) { t->rc = ORC_EDEADLK; return NULL; }
            }
            if (m->fault == ORC_FAULT_PUBLISH_EARLY) {
                stamp(m, i, ORC_EV_PUBLISH, tick(m));
                atomic_store_explicit(&r->seq[s], g + 1, memory_order_release);
            }
            stamp(m, i, ORC_EV_STAGE_BEGIN, tick(m));
            vs_copy(&m->vs, a, b, 1, slot);
            stamp(m, i, ORC_EV_STAGE_END, tick(m));
            if (m->fault != ORC_FAULT_PUBLISH_EARLY) {
                stamp(m, i, ORC_EV_PUBLISH, tick(m));
                atomic_store_explicit(&r->seq[s], g + 1, memory_order_release);
            }
        } else {                                              /* consumer */
            uint64_t spins = 0;
            while (atomic_load_explicit(&r->seq[s], memory_order_acquire) != g + 1)
                if (++spins > SPIN_LIMIT) { t->rc = ORC_EDEADLK; return NULL; }
            stamp(m, i, ORC_EV_FWD_BEGIN, tick(m));
            vs_copy(&m->vs, a, b, 2, slot);
            stamp(m, i, ORC_EV_FWD_END, tick(m));
            stamp(m, i, ORC_EV_CREDIT, tick(m));
            atomic_store_explicit(&r->credit[s], g + 1, memory_order_release);
        }
    }
    return NULL;
}

static int run_threaded(mover_t* m)
{
    int nt = 1 + 2 * m->nrings;
    pthread_t* th = (pthread_t*)calloc((size_t)nt, sizeof(pthread_t));
    thr_arg* args = (thr_arg*)calloc((size_t)nt, sizeof(thr_arg));
    if (!th || !args) { free(th); free(args); return ORC_EINVAL; }
    args[0] = (thr_arg){m, NULL, 0, 0};
    for (int k = 0; k < m->nrings; k++) {
        args[1 + 2 * k] = (thr_arg){m, &m->rings[k], 1, 0};
        args[2 + 2 * k] = (thr_arg){m, &m->rings[k], 2, 0};
    }
    for (int t = 0; t < nt; t++) pthread_create(&th[t], NULL, thread_main, &args[t]);
    int rc = 0;
    for (int t = 0; t < nt; t++) {
        pthread_join(th[t], NULL);
        if (args[t].rc) rc = args[t].rc;
    }
    free(th);
    free(args);
    return rc;
}

int orc_move(const orc_segment* segs, uint64_t nsegs, uint64_t C,
             const orc_path* paths, int P, const uint8_t* path_of_chunk, uint64_t n,
             uint32_t S, const uint64_t* base, int exec, uint64_t* events,
             uint32_t* write_count, int fault)
{
    if ((nsegs && !segs) || C == 0 || !paths || P < 1 || P > 255 || S < 1) return ORC_EINVAL;
    if (!orc_segments_disjoint(segs, nsegs)) return ORC_EINVAL;
    mover_t m;
    memset(&m, 0, sizeof(m));
    if (vs_init(&m.vs, segs, nsegs, write_count)) return ORC_EINVAL;
    m.B = m.vs.start[nsegs];
    m.C = C;
    m.n = n;
    m.path_of_chunk = path_of_chunk;
    m.events = events;
    m.fault = fault;
    atomic_store(&m.clock, 0);
    int rc = 0;
    if (n != orc_nchunks(m.B, C) && !(n == 1 && m.B > 0)) { rc = ORC_EINVAL; goto out_vs; }
    m.slot_bytes = (n == 1 && m.B > C) ? m.B : C;
    if (events) memset(events, 0, n * ORC_NEV * sizeof(uint64_t));

    /* Split the plan into per-path lists, ascending chunk order. */
    m.direct = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    m.rings = (ring_t*)calloc((size_t)P, sizeof(ring_t));
    if (!m.direct || !m.rings) { rc = ORC_EINVAL; goto out; }
    for (uint64_t i = 0; i < n; i++) {
        int p = path_of_chunk[i];
        if (p >= P) { rc = ORC_EINVAL; goto out; }
        if (paths[p].kind == ORC_DIRECT) m.direct[m.ndirect++] = i;
    }
    for (int p = 0; p < P; p++) {
        if (paths[p].kind != ORC_RELAY) continue;
        uint64_t cnt = 0;
        for (uint64_t i = 0; i < n; i++) cnt += (path_of_chunk[i] == p);
        if (cnt == 0) continue;
        ring_t* r = &m.rings[m.nrings++];
        r->path = p;
        r->base = base ? base[p] : 0;
        r->S = S;
        r->nchunks = cnt;
        r->chunks = (uint64_t*)malloc(cnt * sizeof(uint64_t));
        r->stage = (unsigned char*)malloc((size_t)S * m.slot_bytes);
        r->seq = (_Atomic uint64_t*)malloc(S * sizeof(_Atomic uint64_t));
        r->credit = (_Atomic uint64_t*)malloc(S * sizeof(_Atomic uint64_t));
        if (!r->chunks || !r->stage || !r->seq || !r->credit) { rc = ORC_EINVAL; goto out; }
        uint64_t c = 0;
        for (uint64_t i = 0; i < n; i++)
            if (path_of_chunk[i] == p) r->chunks[c++] = i;
        ring_init_flags(r);
    }
    rc = (exec == ORC_EXEC_THREADED) ? run_threaded(&m) : run_deterministic(&m);
out:
    for (int k = 0; k < m.nrings; k++) {
        free(m.rings[k].chunks);
        free(m.rings[k].stage);
        free((void*)m.rings[k].seq);
        free((void*)m.rings[k].credit);
    }
    free(m.rings);
    free(m.direct);
out_vs:
    free(m.vs.start);
    return rc;
}

/* ------------------------------------------------------------ invariant checker --- */

uint64_t orc_check_events(const uint64_t* ev, const orc_path* paths, int P,
                          const uint8_t* path_of_chunk, uint64_t n, uint32_t S,
                          const uint64_t* base)
{
    uint64_t bad = 0;
    for (int p = 0; p < P; p++) {
        if (paths[p].kind != ORC_RELAY) continue;
        uint64_t j = 0;
        uint64_t* prev = (uint64_t*)calloc(S, sizeof(uint64_t));   /* chunk+1 per slot */
        for (uint64_t i = 0; i < n; i++) {
            if (path_of_chunk[i] != p) continue;
            const uint64_t* e = ev + i * ORC_NEV;
            uint64_t g = (base ? base[p] : 0) + j;
            /* every event happened */
            for (int k = 0; k < ORC_NEV; k++) bad += (e[k] == 0);
            /* (a) forward only after the staging write completed and was published */
            bad += !(e[ORC_EV_STAGE_END] < e[ORC_EV_PUBLISH]);
            bad += !(e[ORC_EV_PUBLISH] <= e[ORC_EV_FWD_BEGIN]);
            bad += !(e[ORC_EV_FWD_BEGIN] < e[ORC_EV_FWD_END]);
            bad += !(e[ORC_EV_FWD_END] < e[ORC_EV_CREDIT]);
            /* (b) slot reuse only after the previous occupant's credit */
            uint32_t s = (uint32_t)(g % S);
            if (prev[s]) bad += !(ev[(prev[s] - 1) * ORC_NEV + ORC_EV_CREDIT] <= e[ORC_EV_STAGE_BEGIN]);
            prev[s] = i + 1;
            j++;
        }
        free(prev);
    }
    return bad;
}

/* ------------------------------------------------------ exhaustive interleavings --- */

#define XN 8
#define XS 4
typedef struct {
    int8_t pj, ps, cj, cs;          /* producer / consumer: chunk index and step */
    int8_t slot[XS][2];             /* chunk id held by each half of each slot; -2 stale */
    int8_t dst[XN][2];              /* chunk id delivered into each half of each dst chunk */
    uint64_t seq[XS], credit[XS];
} xstate;

typedef struct {
    xstate* tab;
    unsigned char* used;
    uint64_t cap, count;
} xset;

static uint64_t xhash(const xstate* s)
{
    const unsigned char* p = (const unsigned char*)s;
    uint64_t h = 1469598103934665603ull;
    for (size_t k = 0; k < sizeof(*s); k++) { h ^= p[k]; h *= 1099511628211ull; }
    return h;
}

static int xset_insert(xset* set, const xstate* s);

static void xset_grow(xset* set)
{
    xset old = *set;
    set->cap = old.cap ? old.cap * 2 : 1024;
    set->tab = (xstate*)calloc(set->cap, sizeof(xstate));
    set->used = (unsigned char*)calloc(set->cap, 1);
    set->count = 0;
    for (uint64_t k = 0; k < old.cap; k++)
        if (old.used[k]) xset_insert(set, &old.tab[k]);
    free(old.tab);
    free(old.used);
}

/* returns 1 if newly inserted */
static int xset_insert(xset* set, const xstate* s)
{
    if ((set->count + 1) * 2 > set->cap) xset_grow(set);
    uint64_t h = xhash(s) & (set->cap - 1);
    while (set->used[h]) {
        if (memcmp(&set->tab[h], s, sizeof(*s)) == 0) return 0;
        h = (h + 1) & (set->cap - 1);
    }
    set->used[h] = 1;
    set->tab[h] = *s;
    set->count++;
    return 1;
}

/* Apply one producer (who=0) or consumer (who=1) step; returns 0 if blocked/done,
 * 1 if taken; *viol set when the step reads data that is not the chunk's. */
static int xstep(const xstate* in, xstate* out, int who, int n, int S, uint64_t base,
                 int fault, int* viol)
{
    *out = *in;
    *viol = 0;
    if (who == 0) {
        if (in->pj >= n) return 0;
        uint64_t g = base + (uint64_t)in->pj;
        int s = (int)(g % (uint64_t)S);
        int step = in->ps;
        if (fault == ORC_FAULT_PUBLISH_EARLY) { static const int o[4] = {0, 3, 1, 2}; step = o[in->ps]; }
        switch (step) {
        case 0:
            if (fault != ORC_FAULT_SKIP_CREDIT && g >= (uint64_t)S &&
                in->credit[s] < g - (uint64_t)S + 1) return 0;
            break;
        case 1: out->slot[s][0] = in->pj; break;
        case 2: out->slot[s][1] = in->pj; break;
        case 3: out->seq[s] = g + 1; break;
        }
        if (++out->ps == 4) { out->ps = 0; out->pj++; }
        return 1;
    }
    if (in->cj >= n) return 0;
    uint64_t g = base + (uint64_t)in->cj;
    int s = (int)(g % (uint64_t)S);
    switch (in->cs) {
    case 0:
        if (in->seq[s] != g + 1) return 0;
        break;
    case 1:
        out->dst[in->cj][0] = in->slot[s][0];
        *viol = in->slot[s][0] != in->cj;
        break;
    case 2:
        out->dst[in->cj][1] = in->slot[s][1];
        *viol = in->slot[s][1] != in->cj;
        break;
    case 3: out->credit[s] = g + 1; break;
    }
    if (++out->cs == 4) { out->cs = 0; out->cj++; }
    return 1;
}

int orc_ring_explore(int n, int S, uint64_t base, int fault, uint64_t* states,
                     uint64_t* violations)
{
    if (n < 0 || n > XN || S < 1 || S > XS || !states || !violations) return ORC_EINVAL;
    xstate init;
    memset(&init, 0, sizeof(init));
    for (int s = 0; s < XS; s++) init.slot[s][0] = init.slot[s][1] = -2;
    for (int j = 0; j < XN; j++) init.dst[j][0] = init.dst[j][1] = -1;
    for (int s = 0; s < S; s++) {            /* flags left behind by `base` earlier chunks */
        uint64_t v = 0;
        if (base > (uint64_t)s) v = base - 1 - ((base - 1 - (uint64_t)s) % (uint64_t)S) + 1;
        init.seq[s] = init.credit[s] = v;
    }
    xset set = {0};
    xset_grow(&set);
    uint64_t stack_cap = 1024, sp = 0, bad = 0;
    xstate* stack = (xstate*)malloc(stack_cap * sizeof(xstate));
    xset_insert(&set, &init);
    stack[sp++] = init;
    while (sp) {
        xstate cur = stack[--sp];
        int moved = 0;
        for (int who = 0; who < 2; who++) {
            xstate nxt;
            int viol;
            if (!xstep(&cur, &nxt, who, n, S, base, fault, &viol)) continue;
            moved = 1;
            bad += viol;
            if (xset_insert(&set, &nxt)) {
                if (sp == stack_cap) {
                    stack_cap *= 2;
                    stack = (xstate*)realloc(stack, stack_cap * sizeof(xstate));
                }
                stack[sp++] = nxt;
            }
        }
        if (!moved) {
            int done = cur.pj >= n && cur.cj >= n;
            if (!done) { bad++; continue; }                       /* deadlock */
            for (int j = 0; j < n; j++)                           /* wrong delivery */
                bad += (cur.dst[j][0] != j) || (cur.dst[j][1] != j);
        }
    }
    *states = set.count;
    *violations = bad;
    free(stack);
    free(set.tab);
    free(set.used);
    return 0;
}


/* ---- steady-state path throughput model (performance; header comment) ------------------ */

double orc_direct_rate(double C, unsigned depth, double B, double t0)
{
    if (C <= 0 || B <= 0 || depth == 0) return 0.0;
    const double per_slot = depth * C / (t0 + C / B);   /* each slot: setup then transfer */
    return per_slot < B ? per_slot : B;                  /* the link cannot exceed B */
}

double orc_relay_rate(double C, unsigned streams, double Bp, double Bn, double t0)
{
    if (C <= 0 || Bp <= 0 || Bn <= 0 || streams == 0) return 0.0;
    const double hop1 = t0 + C / Bp, hop2 = C / Bn;
    if (streams == 1) return C / (hop1 + hop2);         /* Fig 6a: the hops serialise */
    return C / (hop1 > hop2 ? hop1 : hop2);             /* Fig 6b: hop 2 of i under hop 1 of i+1 */
}
