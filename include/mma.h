/*
 * mma.h — C ABI of the B200-native multipath host<->GPU copy engine (MMA, arXiv 2512.16056).
 *
 * Citations: P:NNN = line of the paper's text, S:NNN = line of SPEC.md; the
 * section is named beside each. DESIGN.md §2 maps every entry point to the paper.
 *
 * Conventions for every function below
 *  - Return value: a cudaError_t value as int (0 = cudaSuccess). Validation happens
 *    before anything is enqueued: a call that fails validation enqueued nothing. A CUDA
 *    error while enqueueing (after validation) is returned after the user stream has been
 *    made to wait for whatever part of the copy was already enqueued.
 *  - Asynchronous failures (a relay kernel whose bounded spin timed out) are sticky: they
 *    are returned by the next mma_* call and by mma_get_last_error().
 *  - Thread safety: every call may be made from any thread. Multipath calls serialise at
 *    enqueue time. One engine per process (§5.1.2 "each process in MMA maintains
 *    its own multipath queue").
 *  - Ordering between calls: the engine's path streams are shared, so multipath calls run
 *    in enqueue order on them. Like any shared resource this adds one rule that plain
 *    cudaMemcpyAsync does not have: a call must not be made to wait (through stream or
 *    event dependencies) on a multipath call enqueued after it.
 *  - Pointers are plain host or device virtual addresses (UVA). The library never takes
 *    ownership of caller memory; it owns its streams, events, staging rings and flags,
 *    all released by mma_finalize().
 */
#ifndef MMA_H
#define MMA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* mma_stream_t;   /* == cudaStream_t; NULL = legacy default stream */

#define MMA_MAX_GPUS 16
#define MMA_MAX_PATHS 16

typedef enum { MMA_H2D = 0, MMA_D2H = 1 } mma_dir_t;

/* How a path moves host bytes (§3.4.3 uses copy-engine DMA only; the SM
 * zero-copy mode is north_star (d), chosen per path by measurement). */
typedef enum {
    MMA_HOP_AUTO = 0,  /* CE for contiguous copies, ZC for scattered segments */
    MMA_HOP_CE = 1,    /* copy-engine DMA; a relay stages through its HBM ring */
    MMA_HOP_ZC = 2,    /* SM loads/stores of mapped pinned host memory; a relay writes the
                          target over NVLink directly (one hop, no staging) */
    MMA_HOP_PUSH = 4,  /* relays only: the kernel ring with the relay kernel on the OTHER side of
                          NVLink -- H2D on the relay GPU (it reads its own slot and writes the
                          target over NVLink: posted writes), D2H on the target (it reads its own
                          memory and writes the relay's slot). Same slots, flags and waves as
                          MMA_HOP_CE; chosen against it by measurement (pull / push /
                          copy engine) */
    MMA_HOP_CE_P2P = 3 /* relays only: the copy engine for both hops, the paper's own design
                          ("an H2D operation and a P2P operation"): host <-> the relay's
                          ring slot, then a peer DMA slot <-> the target, on the same relay
                          stream, under the ring's seq/credit flags -- no SM work anywhere.
                          A direct path given this mode uses MMA_HOP_CE. */
} mma_hop_t;

typedef enum { MMA_PATH_DIRECT = 0, MMA_PATH_RELAY = 1 } mma_path_kind_t;

/* One scattered segment (north_star (e); paged KV blocks, §2.1). */
typedef struct {
    const void* src;
    void* dst;
    size_t bytes;
} mma_segment_t;

typedef struct {
    /* chunk size per direction in bytes (§3.4.1 "fixed chunk size"; P:902 tuned
     * optima 2.81 MB H2D / 5.37 MB D2H on H20). Default 8 MiB (B200 DMA setup cost,
     * DESIGN.md §6). Multiple of 4096. */
    size_t chunk_bytes[2];
    /* relay staging slots per ring, 1..64 (P:588-594 dual pipeline = 2). 0 = default: 32 MiB
     * of staging per ring, i.e. S = 32 MiB / chunk_bytes clamped to 4..32 (S = 4 at the 8 MiB
     * default chunk, 32 at 1 MiB chunks; reading R25). */
    unsigned ring_slots;
    /* fallback threshold per direction (§3.2, §5.1.3): a copy of B < thr
     * bytes takes the native single path. (size_t)-1 = always native; 0 = never. */
    size_t fallback_bytes[2];
    /* relay GPUs in calibration order; npaths = 0 -> every P2P-capable peer, ascending */
    int path_gpus[MMA_MAX_PATHS];
    int npaths;
    /* extra relay paths through the target GPU itself (loopback rings): a diagnostic
     * mode that exercises the full relay protocol on a single GPU. Default 0. */
    int loopback_relays;
    /* 0 = contiguous (each path carries one contiguous range), 1 = interleaved,
     * 2 = dynamic: when every usable path is in zero-copy mode, the path kernels claim
     * chunks from one cursor on the target GPU (the paper's pull scheduler, P:549-557,
     * run by the GPUs); the assignment is observed (delivery log, mma_get_dynamic_counts)
     * instead of planned; otherwise the contiguous plan is used */
    int plan_mode;
    /* hop mode per direction for every path (mma_hop_t), refined per path by
     * mma_set_path_modes() */
    int hop_mode[2];
    /* CTAs per relay ring for the relay kernels; 0 = default (8) */
    int relay_ctas;
    /* NUMA placement for mma_host_alloc: 0 = default, 1 = bind to node 0, 2 = interleave
     * across all nodes page by page, 3 = 2 MiB blocks round-robin over the nodes (a paged-KV
     * block then never straddles nodes, for the planner's regrouping, numa_plan) -- all a
     * no-op on a single-node host */
    int numa_mode;
    /* record the per-chunk delivery log (debug; off in timed runs) */
    int debug_log;
    /* backlog ledger: plan each call against the bytes other in-flight
     * calls still have queued on every link ("remaining tasks in the buffer provide an
     * effective proxy for link congestion", §2.3); a relay GPU whose own target's
     * direct bytes are still in flight takes relay work only behind them ("direct path
     * first", §3.4.2; R27). 0 = off, 1 = on (default). */
    int ledger;
    /* dynamic pull (plan_mode 2): bytes one CTA claims at a time; the delivery log has one
     * entry per claim. Small claims keep every link's share proportional to its speed
     * (the paper's outstanding-queue depth). 0 = default (256 KiB). */
    size_t claim_bytes;
    /* CTAs per zero-copy path kernel, planned or dynamic (the vector kernels: 512 threads;
     * the cp.async.bulk kernel of direct paths: one warp and 128 KiB of shared memory). A
     * PCIe link saturates with 4 vector CTAs (profiles/r01_probe_grid.txt), so a small grid
     * leaves the relay GPU's other SMs to its own work (§3.4.3: relaying must not
     * steal the peer's compute). 0 = default (16); at most 4 x the SM count. The environment
     * variables MMA_ZC_CTAS_H2D / MMA_ZC_CTAS_D2H (read at the first init) override it per
     * direction. */
    int zc_ctas;
    /* Concurrent calibration rounds (the bandwidth vector is "measured with
     * all paths of the set active"). After mma_calibrate / mma_tune_segments pick each
     * path's mode and solo rate, the transfer is run this many more times with every path
     * active, planned from the current vector; each path's rate becomes the bytes it carried
     * over the time its own streams took (events on those streams), quantised as in R17.
     * Shared host DRAM, switch uplinks or socket links then show up in the vector the
     * planner uses. 0 = solo rates only; default 2. */
    int calib_rounds;
    /* Host-address order for scattered transfers: each path moves its pieces in ascending
     * host address instead of table order (the bytes and the chunk -> path plan are
     * unchanged; only the order of work inside a path's share). Random 32 KiB host writes
     * cost the copy engine 7% on B200 and, on some hosts, the SM scatter 12%
     * (profiles/r01_probe_sort.jsonl). 0 = table order, 1 = D2H (default), 2 = both
     * directions. */
    int host_order;
    /* NUMA-affine planning of scattered transfers (north_star (b); reading R23): when the
     * path GPUs sit on more than one NUMA node, a scattered table is planned as the stable
     * regrouping of its segments by host node, groups in path order, and relays are ordered
     * with the target's node first, so the contiguous plan gives each path (mostly) the
     * bytes on its own GPU's node. Bytes are unchanged; mma_get_stats reports local bytes.
     * 0 = off, 1 = auto (default; inert on a one-node host). */
    int numa_plan;
    /* Contention with background traffic (§3.4.2), dynamic pull only: 0 = keep
     * claiming as soon as a unit is done ("maximize link utilization", default); 1 = yield to
     * background traffic: a CTA whose last unit took longer than yield_pct percent of the
     * unit time the path's bandwidth predicts ("blocked") waits that long before it claims
     * again, so a link shared with other traffic carries less of the transfer and the other
     * links more. mma_get_dynamic_backoffs counts the waits. */
    int background_policy;
    unsigned yield_pct;   /* 0 = default (150) */
    /* Relay task scheduling of joint plans (mma_memcpy_multi; §3.4.2): 0 = longest
     * micro-task queue first (default); g + 1 = GPU g's queue first ("prioritize data
     * transfer for a specific GPU"), then longest first. A link's own queue always first. */
    int relay_prefer;
} mma_config_t;

typedef struct {
    uint64_t calls, fallbacks, bytes;
    /* path_bytes / path_chunks / relay_bytes count PLANNED work at enqueue; a dynamic-pull
     * call (plan_mode 2) splits on the device, so it adds to none of them: its split is
     * mma_get_dynamic_counts after completion (its bytes stay in `bytes`) */
    uint64_t path_bytes[2][MMA_MAX_PATHS];   /* [direction][path] of this target */
    uint64_t path_chunks[2][MMA_MAX_PATHS];
    uint64_t relay_bytes;                 /* bytes that crossed NVLink (relayed) */
    uint64_t kernels;                     /* relay / zero-copy kernel launches */
    double issue_us;                      /* host time spent enqueueing (incl. wait_us) */
    double wait_us;                       /* of which blocked on table-buffer reuse */
    uint64_t dynamic_calls;               /* calls moved by GPU-driven dynamic pull */
    uint64_t numa_known_bytes[2];         /* [direction] bytes whose host NUMA node is known */
    uint64_t numa_local_bytes[2];         /* of those, carried by a path on the same node */
    /* fallbacks counts calls moved by the NATIVE copy (below the threshold, pageable, or a
     * one-path plan on the copy engine); a one-path plan that runs the engine's zero-copy
     * kernel is counted here instead */
    uint64_t single_path_calls;
    double validate_us;                   /* host time classifying segment memory kinds */
    uint64_t ptr_queries;                 /* driver pointer queries made for it */
} mma_stats_t;

/* Fill cfg with defaults (then env MMA_* overrides). */
int mma_default_config(mma_config_t* cfg);

/* Initialise the engine: enable peer access between P2P-capable GPUs, create path streams,
 * resolve the stream memory-op entry points. cfg = NULL -> defaults + env. Idempotent
 * (a second call with a different cfg re-applies the tunables). Lazy on first copy. */
int mma_init(const mma_config_t* cfg);
int mma_finalize(void);

/*
 * Multipath copies with cudaMemcpyAsync(dst, src, bytes, kind, stream) semantics
 * (§3.1 "preserving the semantics of existing transfer APIs"; P:447-448 workflow):
 * ordered after prior work on `stream`; later work on `stream` sees the bytes; returns
 * before completion. The GPU is the one owning the device pointer (not the current
 * device). H2D: dst is device memory, src host memory; D2H the reverse. bytes = 0 is a
 * no-op. Falls back to the native single-path copy (byte-identical by definition) when
 * bytes < fallback threshold, host memory is pageable, or the target has a single path
 * (§3.2).
 * Graph capture: a call on a stream being captured is recorded as a replayable multipath
 * copy -- zero-copy paths, the direct copy engine and MMA_HOP_CE_P2P relays on two staging
 * slots of their own (graph allocations); kernel-driven relay rings and the backlog ledger
 * stay out (ring sequence numbers advance per call) -- tables in a pinned arena made at init
 * (MMA_GRAPH_ARENA bytes, default 16 MiB; when full, the native copy is captured) and on the
 * device as graph allocations. The engine must have made a copy on that device before the
 * capture (nothing may be allocated while capturing); else the native copy is captured.
 * While such a capture is open, other threads must not make multipath calls (the engine's
 * streams are part of it). Graphs holding captured copies must not be replayed after
 * mma_finalize.
 * Errors: cudaErrorInvalidValue (null pointer with bytes > 0, wrong memory kinds),
 * cudaErrorInvalidDevice, or the CUDA error of an enqueue.
 */
int mma_memcpy_h2d(void* dst, const void* src, size_t bytes, mma_stream_t stream);
int mma_memcpy_d2h(void* dst, const void* src, size_t bytes, mma_stream_t stream);

/*
 * Scattered variant (north_star (e)): segs[k] copies segs[k].bytes from src to dst. The
 * segments form one virtual stream v (their concatenation in table order) that is chunked
 * and planned like a contiguous copy. H2D: every src is pinned host memory, every dst is
 * device memory of dst_device; D2H the reverse with src_device. The table is copied at
 * call time. Destinations must be pairwise disjoint (cudaErrorInvalidValue otherwise).
 * Every segment's memory is classified before anything is enqueued (a per-call cache of
 * the driver's allocation ranges, mma_stats_t.validate_us / ptr_queries): a device-side
 * piece that is not device memory of that GPU, a host-side piece that is device memory, or
 * a piece that spans two kinds of memory -> cudaErrorInvalidValue, nothing enqueued. A
 * host-side piece that is pageable (not page-locked) -> the whole table is copied by the
 * native cudaMemcpyAsync per segment on `stream` (byte-identical; its errors are that
 * call's), as for a contiguous copy (reading R7).
 */
int mma_memcpy_h2d_segments(const mma_segment_t* segs, size_t nsegs, int dst_device,
                            mma_stream_t stream);
int mma_memcpy_d2h_segments(const mma_segment_t* segs, size_t nsegs, int src_device,
                            mma_stream_t stream);

/* Concurrent transfers under ONE joint plan (config 5: every GPU reloading
 * its weights while some also fetch KV): the paper's Path Selector, §3.4.2. Per
 * direction, one micro-task queue per target GPU (its transfers' chunks, FIFO in array
 * order); the link that is free first takes its own GPU's next chunk ("direct path first"),
 * else the next chunk of the longest queue it may relay for; link rates are each GPU's
 * direct-path rate (mma_set_bandwidth on that GPU, path 0). The plan is mma_plan_multi's.
 * Each transfer is then enqueued like mma_memcpy_*_segments on its own stream with that
 * plan: first every transfer's direct part, then every relay part, the relay work on a GPU
 * waiting for that GPU's own direct work of the batch. Semantics per transfer are
 * cudaMemcpyAsync's on x.stream. A transfer that is pageable, below the direction's fallback
 * threshold, or on a capturing stream is copied on its own instead. Every transfer is
 * validated before anything is enqueued (errors as mma_memcpy_*_segments). */
typedef struct {
    int dir;                     /* MMA_H2D or MMA_D2H */
    int device;                  /* H2D: the destination GPU; D2H: the source GPU */
    const mma_segment_t* segs;   /* the transfer; one segment = a contiguous copy */
    size_t nsegs;
    mma_stream_t stream;
} mma_transfer_t;
int mma_memcpy_multi(const mma_transfer_t* xfers, size_t n);

/* Paths of a target GPU for a direction: path 0 = its own PCIe link (direct), then relays
 * in calibration order. Arrays of length cap; *npaths receives the count. */
int mma_get_paths(int device, mma_dir_t dir, int* gpus, int* kinds, uint32_t* mbps,
                  int* modes, int cap, int* npaths);

/* Pin the bandwidth vector (integer MB/s, index-aligned with mma_get_paths) used by the
 * planner; bit-exact plan parity runs pin it (SURVEY §7 hard part 7). 0 drops a path. */
int mma_set_bandwidth(int device, mma_dir_t dir, const uint32_t* mbps, int npaths);

/* Switch the plan mode (mma_config_t.plan_mode) without re-initialising. */
int mma_set_plan_mode(int mode);

/* Per-path hop mode (mma_hop_t), index-aligned with mma_get_paths. */
int mma_set_path_modes(int device, mma_dir_t dir, const int* modes, int npaths);

/* "Chosen per path by measurement" (north_star (d)): time each path of `device` alone in
 * each hop mode (copy engine, SM zero-copy) on a contiguous copy of `bytes` through
 * library-owned buffers, and keep per path the faster mode and its rate as the planner's
 * bandwidth (integer MB/s, reading R17: llround). Synchronous. */
int mma_calibrate(int device, mma_dir_t dir, size_t bytes);

/* Chunk size by measurement (§3.4.1 "dynamically adjusts"; reading R3): times
 * a contiguous copy of `bytes` (>= 2 MiB) through library-owned buffers at chunk sizes
 * 32, 16, 8, 4, 2, 1 MiB (those <= bytes / 2) with the current bandwidth vector and modes,
 * and sets cfg.chunk_bytes[dir] to the fastest (a smaller chunk must be >= 1% faster).
 * *chunk_out (may be NULL) receives it. Synchronous; rings are re-made for the new size. */
int mma_tune_chunk(int device, mma_dir_t dir, size_t bytes, size_t* chunk_out);

/* Fallback threshold by measurement (§3.2, §5.1.3: below a break-even size
 * the native single-path copy wins). Times the native copy and the multipath copy (current
 * bandwidth vector and modes) at sizes chunk, 2*chunk, 4*chunk, ... <= max_bytes through
 * library-owned buffers, and sets cfg.fallback_bytes[dir] to the smallest swept size from
 * which every larger swept size is >= 3% faster by multipath (at least two such sizes when
 * two or more are swept). If even max_bytes is not (a single-path set, or relays that share
 * the target's link), there is no break-even:
 * the threshold is left unchanged and *found = 0. *thr_out receives the threshold in effect.
 * Either pointer may be NULL. Synchronous. */
int mma_tune_threshold(int device, mma_dir_t dir, size_t max_bytes, size_t* thr_out, int* found);

/* The same measurement on the caller's scattered transfer (segment table as in
 * mma_memcpy_*_segments): the copy is executed (1 + reps) times per (path, mode) on
 * `stream`, so the destinations are written. The result applies to scattered transfers
 * only; mma_set_bandwidth / mma_set_path_modes clear it. Synchronous. */
int mma_tune_segments(const mma_segment_t* segs, size_t nsegs, int device, mma_dir_t dir,
                      mma_stream_t stream, int reps);
/* Persist / restore what calibration measured (bandwidth and mode per path, contiguous and
 * scattered), one text line per (device, direction, path). Loading applies a line only
 * where the current path set has the same GPU and kind at that index; *applied receives the
 * number of paths updated. MMA_CALIB=<file> loads it at init. */
int mma_save_calibration(const char* path);
int mma_load_calibration(const char* path, int* applied);

/* What mma_tune_segments chose, index-aligned with mma_get_paths (0 / -1 = not tuned). */
int mma_get_segment_tuning(int device, mma_dir_t dir, uint32_t* mbps, int* modes, int cap,
                           int* npaths);

/* Evidence of the last calibration of (device, dir): per path, the solo rate of the chosen
 * mode and the rate measured with all paths active (integer MB/s; 0 = not measured: the
 * path carried no bytes, or calib_rounds = 0 / a single path). scattered = 0 reads
 * mma_calibrate's result, 1 mma_tune_segments'. Arrays of length cap (either may be NULL);
 * *npaths receives the path count. */
int mma_get_calibration(int device, mma_dir_t dir, int scattered, uint32_t* solo_mbps,
                        uint32_t* conc_mbps, int cap, int* npaths);

/* The plan the engine would use for a copy of `bytes`: path index per chunk. A fallback
 * plan is reported as nchunks = 1, path_of_chunk[0] = 0, *fallback = 1. */
int mma_get_plan(int device, mma_dir_t dir, size_t bytes, uint8_t* path_of_chunk,
                 size_t cap, size_t* nchunks, int* fallback);

/* The planner alone, on the host (no GPU, no engine state): the assignment for a given
 * path vector. kinds[p] is MMA_PATH_DIRECT (index 0 only) or MMA_PATH_RELAY; backlog may
 * be NULL (all 0); mode 0 = contiguous, 1 = interleaved; thr = fallback threshold.
 * Same outputs as mma_get_plan. Returns cudaErrorInvalidValue on bad arguments. */
int mma_plan_chunks(const uint32_t* mbps, const int* kinds, const uint64_t* backlog, int npaths,
                    uint64_t bytes, uint64_t chunk_bytes, uint64_t thr, int mode,
                    uint8_t* path_of_chunk, size_t cap, size_t* nchunks, int* fallback);

/* The joint planner alone (no GPU, no engine state): the plan of concurrent transfers that
 * mma_memcpy_multi uses (the paper's Path Selector under constant link rates,
 * P:549-574 §3.4.2, reading R24 in DESIGN.md). One micro-task queue per endpoint holds the
 * chunks of every transfer to it, FIFO in array order; the link that is free first (chunks
 * pulled x chunk_bytes / link_mbps, exact; ties to the lower id) takes its own endpoint's
 * head ("direct path first"), else the head of the longest queue it may carry
 * (ties to the lower endpoint id).
 *   nlinks, link_mbps[nlinks]     link rates (0 = absent); a GPU's own link has its id
 *   carry[d * nlinks + l]         1 if link l may carry chunks for endpoint d
 *   target[t], nchunks[t]         transfers
 *   mode                          MMA plan mode: 0 contiguous (per transfer, own link's range
 *                                 first, then the other links by id), 1 interleaved (as pulled)
 *   prefer                        -1, or an endpoint whose queue links relay first (P:569:
 *                                 "tasks can be preferentially fetched from the corresponding
 *                                 micro-task queue"; the own queue still comes first)
 *   link_of_chunk                 out: sum(nchunks) link ids, transfer after transfer
 * cudaErrorInvalidValue: bad arguments, or a transfer no link may carry. */
int mma_plan_multi(int nlinks, const uint32_t* link_mbps, const uint8_t* carry, int ntransfers,
                   const int* target, const uint64_t* nchunks, uint64_t chunk_bytes, int mode,
                   int prefer, int32_t* link_of_chunk);

/* Debug: the path that delivered each chunk of the most recent multipath copy to/from
 * `device`, as written on the GPU by the final hop (needs cfg.debug_log; synchronises). */
int mma_get_delivery_log(int device, uint8_t* path_of_chunk, size_t cap, size_t* nchunks);

/* Debug (cfg.debug_log): what the relay kernels observed before moving each chunk of the
 * most recent multipath copy to/from `device` -- the GPU-side evidence of the north_star
 * invariant "a chunk is forwarded only after its staging write completes". For
 * chunk i carried by a kernel-driven ring: H2D (pull) observed[i] = the seq value the kernel
 * read before pulling the slot, expected[i] = g + 1 (they must be equal); D2H (pack)
 * observed[i] = the credit value it read before overwriting the slot, expected[i] = g + 1,
 * and observed[i] >= expected[i] - S must hold (0 when the slot had never been used).
 * Chunks no relay kernel moved: both 0. Synchronises. */
int mma_get_forward_log(int device, uint64_t* observed, uint64_t* expected, size_t cap, size_t* nchunks);

/* Debug (cfg.debug_log): the order of the segments in the virtual stream v of the last
 * scattered call to `device` -- order[k] = table index of v's k-th segment. It is the table
 * order unless the call was regrouped by host NUMA node (reading R23, §5.1.1; the
 * oracle's orc_numa_order). With mma_get_delivery_log it gives the path that carried every
 * byte. *nsegs = 0 after a contiguous or native call. cap < *nsegs -> cudaErrorInvalidValue. */
int mma_get_segment_order(int device, uint32_t* order, size_t cap, size_t* nsegs);

/* Waits taken by yielding CTAs (background_policy = 1) in the last dynamic-pull call to
 * `device` (synchronises). */
int mma_get_dynamic_backoffs(int device, uint64_t* waits);
/* Chunks each path took in the most recent dynamic-pull call to/from `device`
 * (synchronises; *npaths = 0 if none). */
int mma_get_dynamic_counts(int device, uint64_t* chunks, int cap, int* npaths);

/* Pinned, mapped, portable host memory, NUMA-placed per cfg.numa_mode (C8). */
int mma_host_alloc(void** ptr, size_t bytes, unsigned flags);
int mma_host_free(void* ptr);
/* Whether ptr is the base of a live mma_host_alloc buffer (C8): cudaSuccess and its mapped
 * length (a 2 MiB multiple) in *bytes, else cudaErrorInvalidValue. The LD_PRELOAD shim uses
 * it to route cudaFreeHost of buffers it allocated through the engine. */
int mma_host_alloc_size(const void* ptr, size_t* bytes);

/* NUMA "spread" placement (C8): a buffer for a contiguous transfer of `bytes`
 * to / from `device` whose byte range carried by each path of the current contiguous plan
 * lives on the NUMA node of that path's GPU, so every link reads node-local memory (the
 * paper's 6-path plateau came from the cross-socket link). Pinned, mapped, freed with
 * mma_host_free. mma_host_page_node returns the node holding the page at ptr (-1 if
 * unknown). */
int mma_host_alloc_for(void** ptr, size_t bytes, int device, mma_dir_t dir);
int mma_host_page_node(const void* ptr);

/* Measurement: when on, every relay / zero-copy kernel launch is bracketed by CUDA events
 * on the stream it is launched on. mma_kernel_times synchronises on the recorded launches,
 * returns their durations (ms) and tags in launch order (up to cap; *n = number recorded)
 * and clears the record. tag = kind | direction << 4 | path << 8 | device << 16, kind 0 =
 * zero-copy (vector kernel), 1 = relay pull (H2D), 2 = relay pack (D2H), 3 = dynamic-pull
 * zero-copy, 4 = zero-copy (cp.async.bulk kernel, direct paths); path 255 = all rings of the
 * launch. */
int mma_set_kernel_timing(int on);
int mma_kernel_times(float* ms, int* kinds, size_t cap, size_t* n);

/*
 * Multi-process mode (one process per GPU, as in tensor-parallel serving).
 * The target's process exports its destination memory; the host buffer is shared memory
 * registered in every process; each process moves its own share on its own GPU with the
 * zero-copy kernel. Nothing here is a collective: the processes agree on the plan by
 * computing it with mma_plan_chunks from the same inputs.
 *  - mma_shared_host_alloc: `bytes` of pinned, mapped host memory shared by name between
 *    processes (create = 1 in one process first, 0 in the others); /dev/shm when it has
 *    room, else MMA_SHM_DIR or /tmp. mma_shared_host_free unmaps (and unlinks `name` if
 *    given).
 *  - mma_ipc_export writes a 64-byte CUDA IPC handle of the allocation holding dev_ptr and
 *    dev_ptr's offset in it; mma_ipc_open maps it on `device` of another process (peer
 *    access enabled lazily) and returns the matching pointer; mma_ipc_close unmaps.
 *  - mma_copy_share_segments moves the chunks i of the table with path_of_chunk[i] == path
 *    (a plan from mma_plan_chunks for the same bytes and chunk size) with a zero-copy kernel
 *    on `device`; pointers must be valid in this process. Direction follows the pointers.
 *  - mma_copy_share_segments_ring moves the same share through this process's own
 *    copy-engine relay ring on `device` (`slots` slots of chunk_bytes in its HBM, the dual
 *    relay pipeline of P:588-590): per chunk, hop 1 into a slot -- host -> this GPU (H2D) or
 *    the source GPU -> this GPU over NVLink (D2H, source IPC-mapped) -- then hop 2 out of it
 *    to the destination (the target GPU over NVLink, or host memory), both DMAs on this
 *    process's streams; slot s always uses stream s & 1, so stream order reuses slots and no
 *    flag crosses a process. Ordered on `stream` like mma_copy_share_segments.
 *  - mma_copy_claim_segments is the dynamic-pull form: claim_bytes units are claimed from
 *    *cursor (device memory, e.g. IPC-mapped from the target, zeroed before the transfer)
 *    until none is left; counts[path] += units taken.
 */
int mma_shared_host_alloc(const char* name, size_t bytes, int create, void** ptr);
int mma_shared_host_free(void* ptr, const char* unlink_name);
int mma_ipc_export(const void* dev_ptr, void* handle, uint64_t* offset);
int mma_ipc_open(const void* handle, uint64_t offset, int device, void** dev_ptr);
int mma_ipc_close(void* dev_ptr);
int mma_copy_share_segments(const mma_segment_t* segs, size_t nsegs, size_t chunk_bytes,
                            const uint8_t* path_of_chunk, size_t nchunks, int path, int device,
                            mma_stream_t stream);
int mma_copy_share_segments_ring(const mma_segment_t* segs, size_t nsegs, size_t chunk_bytes,
                                 const uint8_t* path_of_chunk, size_t nchunks, int path, int device,
                                 unsigned slots, mma_stream_t stream);
int mma_copy_claim_segments(const mma_segment_t* segs, size_t nsegs, size_t claim_bytes,
                            uint64_t* cursor, uint64_t* counts, int path, int device,
                            mma_stream_t stream);

/*
 * Cross-process backlog ledger (SURVEY NEXT-4 "a shared-memory path ledger"; §5.1.2:
 * one multipath queue per process). mma_ledger_attach(name) maps the POSIX shared-memory
 * object /mma_ledger_<name> (created on first use, all-zero = empty); from then on every call
 * of this process adds its per-link bytes to it until the call completes, and every plan uses
 * the bytes all attached processes have queued on each link as the backlog (and skips a relay
 * whose own target's direct bytes are in flight). Attach before the first copy.
 * name = NULL or "" detaches. MMA_LEDGER_SHM=<name> attaches at init. Links are keyed by PCI
 * bus id, so processes with different CUDA_VISIBLE_DEVICES agree. A process that dies with
 * calls in flight leaves its bytes counted: mma_ledger_unlink removes the object.
 * mma_ledger_shared_add / _get read or adjust one link's counters directly (bus id as from
 * cudaDeviceGetPCIBusId), for schedulers outside the engine and for tests. Host-only.
 */
int mma_ledger_attach(const char* name);
int mma_ledger_unlink(const char* name);
int mma_ledger_shared_add(const char* bus_id, int dir, int64_t bytes, int64_t own);
/* Adds to THIS process's entry of the attached ledger, as the engine's own calls do (they
 * are removed when the call completes, or with the entry when the process detaches or dies:
 * readers skip entries whose process is gone, and the next attacher reclaims them).
 * mma_ledger_shared_add instead adds to a hand-entered entry that no process owns. */
int mma_ledger_process_add(const char* bus_id, int dir, int64_t bytes, int64_t own);
int mma_ledger_shared_get(const char* bus_id, int dir, uint64_t* bytes, uint64_t* own);
/* The order the engine issues a path's pieces in under cfg.host_order (reading R22): perm
 * receives the stable ascending order of the n addresses (radix sort on 4 KiB page numbers,
 * then by address inside a page). Host-only; exposed for tests and external schedulers. */
int mma_order_by_address(const uint64_t* addr, size_t n, uint32_t* perm);

/* PCI bus id of a device ("dddd:bb:dd.f", as cudaDeviceGetPCIBusId) for the calls above. */
int mma_device_bus_id(int device, char* buf, int len);

/* Timeline tracing: while active, every DMA and kernel the engine enqueues is bracketed by
 * CUDA events on its stream; mma_trace_end synchronises, writes the spans as a Chrome trace
 * JSON (one row per GPU and engine stream) to json_path (NULL: discard) and reports their
 * number. max_spans = 0 -> 100000. */
int mma_trace_begin(size_t max_spans);
int mma_trace_end(const char* json_path, size_t* nspans);

/* Topology probe ("P2P matrix, NUMA node per GPU, CE count"), as the
 * engine sees it: peer access is what cudaDeviceCanAccessPeer reports (and what the engine
 * enabled), the NUMA node comes from sysfs for the GPU's PCI device (-1 = unknown), copy
 * engines from cudaDevAttrAsyncEngineCount. */
typedef struct {
    int ngpu;
    int p2p[MMA_MAX_GPUS][MMA_MAX_GPUS];  /* 1 = device i can access device j's memory */
    int numa_node[MMA_MAX_GPUS];
    int copy_engines[MMA_MAX_GPUS];
    int sms[MMA_MAX_GPUS];
    char bus_id[MMA_MAX_GPUS][16];        /* "dddd:bb:dd.f" */
    int host_numa_nodes;                  /* NUMA nodes the host exposes */
} mma_topology_t;
int mma_get_topology(mma_topology_t* out);

int mma_get_stats(int device, mma_stats_t* out);
int mma_reset_stats(int device);
int mma_get_last_error(void);
const char* mma_error_string(int err);

/* Verification kernels (C4): the seeded offset-unique pattern of SURVEY §8(c) generated on
 * the device. Word w (8 bytes, little endian) of the stream = splitmix64((seed << 40) ^ w);
 * `offset` is the stream byte offset of ptr[0].
 *  - mma_fill_pattern writes bytes [offset, offset+bytes) of the stream to device ptr.
 *  - mma_verify_pattern counts mismatching bytes of device ptr against the stream and
 *    adds them to *mismatches (device memory, uint64).
 *  - mma_verify_segments does the same per segment: dst[k] (device) holds stream bytes
 *    [offset[k], offset[k] + bytes[k]); tables are host arrays. */
int mma_fill_pattern(void* ptr, size_t bytes, uint64_t seed, uint64_t offset, mma_stream_t s);
int mma_verify_pattern(const void* ptr, size_t bytes, uint64_t seed, uint64_t offset,
                       uint64_t* mismatches, mma_stream_t s);
int mma_verify_segments(void* const* dst, const uint64_t* offset, const uint64_t* bytes,
                        size_t nsegs, uint64_t seed, uint64_t* mismatches, mma_stream_t s);

#ifdef __cplusplus
}
#endif
#endif /* MMA_H */
