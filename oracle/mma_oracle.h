/*
 * mma_oracle.h — plain, slow, obviously-correct CPU oracle for MMA's multipath copy
 * (arXiv 2512.16056, "MultiPath Transfer Engine"; /root/reference/PAPER.md = "P:").
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library. The product path
 * (paper_2512_16056_b200/) never includes, links or executes anything under oracle/, and
 * this file includes no header from the product tree. The two sides share no code.
 *
 * What it computes (DESIGN.md §3 lists every reading of the paper it depends on):
 *   - chunking of one transfer into micro-tasks        (§3.4.1 "fixed chunk size")
 *   - the fallback decision                            (§3.2; reading R5)
 *   - chunk -> path assignment for a FIXED bandwidth vector: integer earliest-finish
 *     greedy, ties to the lower path index (direct path first, §3.4.2;
 *     readings R1/R2), plus the paper's pull rule under constant rates as a
 *     comparison mode
 *   - the byte movement, direct and via an S-slot relay staging ring with per-slot
 *     sequence/credit flags (§3.4.3 dual-pipeline relay, generalised to S slots;
 *     reading R8), run deterministically, with threads, or over every interleaving
 *   - the scattered-segment (paged KV) variant (north_star (e); §2.1)
 *   - the paper's invariants (north_star): every byte delivered exactly once; a chunk is
 *     forwarded only after its staging write completes; a slot is reused only after its
 *     forward completes.
 *   - a steady-state throughput model of one path (performance, not bytes): direct path
 *     with `depth` outstanding DMAs, relay with one or two pipelines (Fig 6;
 *     SPEC S:462-486), pinned by SPEC's worked numbers and a discrete-event schedule.
 * Every function is pinned by tests/test_oracle_*.py against closed forms, worked
 * examples (tests/golden/) or brute force; see DESIGN.md §3 "Pins".
 */
#ifndef MMA_ORACLE_H
#define MMA_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_DIRECT = 0, ORC_RELAY = 1 };                      /* path kinds */
enum { ORC_CONTIG = 0, ORC_INTERLEAVED = 1, ORC_PULL = 2 };  /* plan modes */
enum { ORC_EXEC_DETERMINISTIC = 0, ORC_EXEC_THREADED = 1 };  /* mover modes */
/* seeded protocol bugs: the checkers must catch each (tests/test_oracle_ring.py) */
enum { ORC_FAULT_NONE = 0, ORC_FAULT_PUBLISH_EARLY = 1, ORC_FAULT_SKIP_CREDIT = 2 };
/* per relay chunk event slots in the log, logical clock values (0 = not a relay chunk) */
enum { ORC_EV_STAGE_BEGIN = 0, ORC_EV_STAGE_END = 1, ORC_EV_PUBLISH = 2,
       ORC_EV_FWD_BEGIN = 3, ORC_EV_FWD_END = 4, ORC_EV_CREDIT = 5, ORC_NEV = 6 };

/* error codes (negative errno style) */
#define ORC_EINVAL (-22)
#define ORC_ENOSPC (-28)
#define ORC_EDEADLK (-35)

typedef struct {
    int32_t  kind;      /* ORC_DIRECT (only legal at index 0) or ORC_RELAY */
    uint32_t bw_mbps;   /* measured bandwidth, integer MB/s; 0 = path dropped */
    uint64_t backlog;   /* bytes already queued on this path (default 0) */
} orc_path;

typedef struct {        /* one scattered segment (north_star (e)) */
    const void* src;
    void*       dst;
    uint64_t    len;
} orc_segment;

/* n = 0 if B = 0, else ceil(B / C). C must be > 0. */
uint64_t orc_nchunks(uint64_t B, uint64_t C);

/* Chunk i covers [*off, *off + *len) of the transfer: [i*C, min(B, (i+1)*C)). */
void orc_chunk_extent(uint64_t i, uint64_t B, uint64_t C, uint64_t* off, uint64_t* len);

/*
 * Plan one transfer of B bytes in chunks of C over paths[0..P).
 *   thr      fallback threshold: B < thr (strict) -> native single copy (R5)
 *   mode     ORC_CONTIG | ORC_INTERLEAVED | ORC_PULL
 * Outputs: path_of_chunk[0..*nchunks), counts[0..P) (chunks per path), *fallback.
 * A fallback plan is reported as *nchunks = 1, path_of_chunk[0] = 0, *fallback = 1.
 * Returns 0, ORC_EINVAL (bad arguments / no usable path), ORC_ENOSPC (cap too small).
 */
int orc_plan(const orc_path* paths, int P, uint64_t B, uint64_t C, uint64_t thr, int mode,
             uint8_t* path_of_chunk, uint64_t cap, uint64_t* nchunks, uint64_t* counts,
             int* fallback);

/* Predicted makespan T = max_p (backlog_p + bytes_p) / bw_p in seconds (bw in 1e6 B/s),
 * bytes_p counting the real (possibly short) chunk lengths; *agg_gbps = B / T / 1e9. */
void orc_predict(const orc_path* paths, int P, uint64_t B, uint64_t C,
                 const uint8_t* path_of_chunk, uint64_t n, double* T_s, double* agg_gbps);

/*
 * Steady-state throughput model of one path (performance, not bytes; §3.4.3,
 * Fig 6; SPEC S:462-486 launch_direct / launch_relay). Rates in bytes/s, C in bytes, t0 =
 * the DMA setup time in seconds of one chunk.
 *   orc_direct_rate: `depth` outstanding DMAs on a link of rate B. A chunk occupies its
 *     slot for t0 + C/B; the link is busy whenever another slot is in setup, so
 *     rate = min(B, depth * C / (t0 + C/B)).
 *   orc_relay_rate: a relay with `streams` relay pipelines: hop 1 (t0 + C/Bp on the relay's
 *     PCIe link) then hop 2 (C/Bn over NVLink). One pipeline serialises the hops:
 *     rate = C / (t0 + C/Bp + C/Bn); two or more overlap hop 2 of chunk i with hop 1 of
 *     chunk i+1: rate = C / max(t0 + C/Bp, C/Bn).
 */
double orc_direct_rate(double C, unsigned depth, double B, double t0);
double orc_relay_rate(double C, unsigned streams, double Bp, double Bn, double t0);

/*
 * Move a transfer according to a plan. The host buffers stand in for both host memory and
 * device memory (D2H is the same program with the roles of src and dst swapped).
 *   segs/nsegs  the transfer as a list of segments; the contiguous case is one segment
 *               {src, dst, B}. B = sum(len) is the "virtual stream" v that is chunked.
 *   S           relay ring slots (>= 1); base[p] = chunks ring p carried before (R18)
 *   exec        ORC_EXEC_DETERMINISTIC (round-robin actors, logical clock) or
 *               ORC_EXEC_THREADED (1 thread for the direct path, 2 per relay ring)
 *   events      NULL or n*ORC_NEV uint64 logical timestamps per chunk (relay chunks only)
 *   write_count NULL or one uint32 counter per byte of v, incremented on every write of
 *               that byte's final destination (exactly-once check)
 *   fault       ORC_FAULT_* seeded bug (tests only)
 * Returns 0, ORC_EINVAL (bad plan / overlapping segment destinations), ORC_EDEADLK.
 */
int orc_move(const orc_segment* segs, uint64_t nsegs, uint64_t C,
             const orc_path* paths, int P, const uint8_t* path_of_chunk, uint64_t n,
             uint32_t S, const uint64_t* base, int exec, uint64_t* events,
             uint32_t* write_count, int fault);

/*
 * Joint plan of concurrent transfers: the paper's Path Selector under
 * constant link rates (§3.4.2). One micro-task queue per endpoint GPU holds the
 * chunks of every transfer to that GPU, FIFO in transfer order; every link
 * has an outstanding queue that pulls. The link that becomes free first -- free time =
 * chunks taken x C / link_bw, compared exactly; ties -> lower link id -- takes
 *   the head of its own GPU's queue when that is non-empty ("the Outstanding queue
 *   corresponding to each GPU always has priority in fetching transfer tasks from the
 *   associated Mico-task Queue"), else
 *   the head of the longest queue it may relay for ("prioritizing tasks from the longest
 *   micro-task queue"; ties -> lower GPU id) -- or, with prefer >= 0,
 *   GPU prefer's queue first when it is non-empty and the link may carry it ("tasks can be
 *   preferentially fetched from the corresponding micro-task queue"; SPEC PreferGpu),
 * and a link with nothing it may take drops out (queues only shrink).
 *   L                  links (ids 0..L-1; a GPU's own link has the GPU's id), L <= 128
 *   link_bw[l]         MB/s; 0 = absent
 *   relay_ok[d*L + l]  1 if link l may carry chunks for endpoint GPU d (d's own link always may)
 *   T, target[t], nchunks[t]   the transfers (target[t] < L)
 *   mode  ORC_INTERLEAVED: chunks numbered in FIFO order as pulled; ORC_CONTIG: per
 *         transfer, the same per-link counts laid out as contiguous ranges, the target's own
 *         link first, then the other links by id (reading R1's contiguous form)
 *   link_of_chunk      out: sum(nchunks) entries, transfer after transfer
 * Returns 0 or ORC_EINVAL (a transfer no link may carry, bad arguments).
 */
int orc_plan_multi(int L, const uint32_t* link_bw, const uint8_t* relay_ok, int T,
                   const int32_t* target, const uint64_t* nchunks, uint64_t C, int mode,
                   int prefer, int32_t* link_of_chunk);

/*
 * NUMA-affine order of a scattered transfer's segments (reading R23): the
 * paper's bandwidth saturates at six GPUs because "typically four GPUs reside within a
 * single NUMA node, while cross-NUMA H2D transfers rely on the UPI link" (§5.1.1),
 * so the virtual stream v is the segment table regrouped by the host node of each segment:
 *   groups, in this order: each distinct node of the paths that may carry bytes (bw > 0,
 *   path_node >= 0), in path order; then every other known node, ascending; then unknown
 *   nodes (-1). Inside a group, table order.
 * With fewer than two distinct path nodes (or fewer than two segments) v is the table as
 * given. order[k] = table index of the k-th segment of v. The planner then runs on v
 * unchanged (§8(c) step 6).
 */
void orc_numa_order(const int32_t* seg_node, uint64_t nsegs, const orc_path* paths,
                    const int32_t* path_node, int P, uint32_t* order);

/* 1 if the segment destinations are pairwise disjoint, else 0. */
int orc_segments_disjoint(const orc_segment* segs, uint64_t nsegs);

/*
 * Check the protocol invariants on a move's event log:
 *   (a) stage_end(j) < publish(j) <= fwd_begin(j)   forward only after staging completes
 *   (b) credit(j - S) <= stage_begin(j)             slot reused only after its forward
 * for every relay chunk. Returns the number of violations.
 */
uint64_t orc_check_events(const uint64_t* events, const orc_path* paths, int P,
                          const uint8_t* path_of_chunk, uint64_t n, uint32_t S,
                          const uint64_t* base);

/*
 * Exhaustive interleavings of ONE relay ring (producer = hop1, consumer = hop2) carrying
 * n chunks through S slots, each copy split into two half-steps so partial writes are
 * visible. Explores every reachable state. Outputs the number of distinct states and the
 * number of violating states (a forward reading a half that is not chunk j's, a wrong
 * final destination, or a deadlock). n <= 8, S <= 4.
 */
int orc_ring_explore(int n, int S, uint64_t base, int fault, uint64_t* states,
                     uint64_t* violations);

#ifdef __cplusplus
}
#endif
#endif
