// planner.h — chunk -> path assignment from a measured bandwidth vector (C5, layer L2).
// Pure C++, no CUDA. Written from SURVEY §8(c) steps 1-3 and DESIGN.md readings R1-R6,
// independently of oracle/ (the two share no code; tests compare them bit for bit).
#pragma once
#include <stdint.h>

#include <vector>

namespace mma {

struct PlanPath {
    bool direct;        // the target's own link; only legal at index 0
    uint32_t mbps;      // integer MB/s; 0 drops the path
    uint64_t backlog;   // bytes already queued on the path
};

enum PlanMode { PLAN_CONTIGUOUS = 0, PLAN_INTERLEAVED = 1, PLAN_DYNAMIC = 2 /* engine only */ };

struct Plan {
    bool fallback = false;          // one piece [0, B) on path 0 (native)
    uint64_t n = 0;                 // chunks
    std::vector<uint8_t> path;      // path of each chunk
    std::vector<uint64_t> count;    // chunks per path
};

// Returns 0 or a negative errno (-22 invalid arguments / no usable path).
int make_plan(const PlanPath* paths, int npaths, uint64_t B, uint64_t C, uint64_t thr,
              int mode, Plan& out);

// Joint plan of concurrent transfers (the paper's Path Selector under constant
// link rates, §3.4.2): one micro-task queue per endpoint, FIFO over the transfers
// to it; the link free first pulls its own endpoint's queue head ("direct path first",
// P:564-565), else the head of the longest queue it may relay for (ties to the lower
// id). links: rate per link id (0 = absent); carry(d, l): may link l carry chunks of endpoint d
// (its own queue always). prefer >= 0: a link with an empty own queue takes endpoint
// prefer's head first when it may ("tasks can be preferentially fetched from the
// corresponding micro-task queue"). Output: for each transfer, the link id of each chunk; contiguous
// mode lays each transfer's per-link counts out as ranges, own link first, then by link id.
struct MultiLink {
    uint32_t mbps;
};
int make_plan_multi(const std::vector<MultiLink>& links, const std::vector<std::vector<uint8_t>>& carry,
                    const std::vector<int>& target, const std::vector<uint64_t>& nchunks, uint64_t C, int mode,
                    std::vector<std::vector<int>>& link_of_chunk, int prefer = -1);

}  // namespace mma
