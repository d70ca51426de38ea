#!/usr/bin/env python3
"""Probe (design input): when request A's KV fetch (H2D) and request B's offload (D2H) run at
once on one full-duplex link, both by the SM zero-copy kernels, does the kernels' grid bound
the pair? Under duplex load a host read's round trip grows (the upstream direction also
carries the offload's writes), so a fixed number of bytes in flight per CTA moves fewer bytes
per second (Little's law). Rows: zc grid (cfg.zc_ctas) x {fetch alone, offload alone, both};
the copy engine's contiguous duplex (1 GiB each way, native cudaMemcpyAsync) is the link's
reference. GB/s = bytes / device time (CUDA events), best of 3 after one warm-up.
argv[1]: comma-separated grids, each "n" (both directions) or "h2d:d2h" (MMA_ZC_CTAS_H2D /
MMA_ZC_CTAS_D2H, read at engine init: one subprocess per grid)."""
import json
import os
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_16056_b200 as mma  # noqa: E402
from mma_inputs import workloads as W  # noqa: E402


def timed(fn, streams, reps=4):
    best = None
    for rep in range(reps):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        a.record(streams[0])
        for s in streams[1:]:
            s.wait_event(a)
        fn()
        ends = []
        for s in streams:
            e = torch.cuda.Event(enable_timing=True)
            e.record(s)
            ends.append(e)
        torch.cuda.synchronize()
        per = [a.elapsed_time(e) for e in ends]
        if rep and (best is None or max(per) < max(best)):
            best = per
    return best   # per stream: ms from the common start to that stream's end (best rep by the max)


def main():
    if len(sys.argv) > 2 and sys.argv[2] == "--one":
        return one(sys.argv[1])
    torch.cuda.set_device(0)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    # the link's own duplex reference: contiguous native copies, 1 GiB each way
    n = 1 << 30
    hsrc = torch.empty(n, dtype=torch.uint8).pin_memory()
    hdst = torch.empty(n, dtype=torch.uint8).pin_memory()
    d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")

    def ce_h2d():
        with torch.cuda.stream(s1):
            d1.copy_(hsrc, non_blocking=True)

    def ce_d2h():
        with torch.cuda.stream(s2):
            hdst.copy_(d2, non_blocking=True)

    ms_h = max(timed(ce_h2d, [s1, s2]))
    ms_d = max(timed(ce_d2h, [s1, s2]))
    ms_b = max(timed(lambda: (ce_d2h(), ce_h2d()), [s1, s2]))
    print(json.dumps({"what": "native CE contiguous 1 GiB", "h2d_gbps": round(n / ms_h / 1e6, 2),
                      "d2h_gbps": round(n / ms_d / 1e6, 2), "duplex_gbps": round(2 * n / ms_b / 1e6, 2)}), flush=True)
    del hsrc, hdst, d1, d2
    torch.cuda.synchronize()
    for g in (sys.argv[1] if len(sys.argv) > 1 else "8,16,32,64,148").split(","):
        subprocess.run([sys.executable, __file__, g, "--one"], check=True)


def one(grid):
    torch.cuda.set_device(0)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    h, _, d = grid.partition(":")
    os.environ["MMA_ZC_CTAS_H2D"] = h
    os.environ["MMA_ZC_CTAS_D2H"] = d or h
    shape = W.KVShape()
    ho, do, sb, hpool, dbytes = W.kv_segments(shape)
    ho2, do2, _, _, _ = W.kv_segments(shape, request=1)
    hp = mma.host_alloc(hpool)
    cache = torch.empty(dbytes, dtype=torch.uint8, device="cuda")
    lens = np.full(len(ho), sb, dtype=np.int64)
    KB = int(lens.sum())
    fetch = mma.make_segments(hp + ho, cache.data_ptr() + do, lens)
    offload = mma.make_segments(cache.data_ptr() + do2, hp + ho2, lens)
    for _ in (0,):
        cfg = mma.default_config()
        cfg.npaths = 1
        cfg.path_gpus[0] = 0
        cfg.debug_log = 0
        mma.init(cfg)
        mma.set_path_modes(0, mma.H2D, [mma.HOP_ZC])
        mma.set_path_modes(0, mma.D2H, [mma.HOP_ZC])
        f = lambda: mma.memcpy_h2d_segments(*fetch, 0, stream=s1)       # noqa: E731
        o = lambda: mma.memcpy_d2h_segments(*offload, 0, stream=s2)     # noqa: E731
        ms_f = max(timed(f, [s1, s2]))
        ms_o = max(timed(o, [s1, s2]))
        t_f, t_o = timed(lambda: (o(), f()), [s1, s2])
        ms_fo = max(t_f, t_o)
        print(json.dumps({"zc_ctas_h2d": int(h), "zc_ctas_d2h": int(d or h), "fetch_gbps": round(KB / ms_f / 1e6, 2),
                          "offload_gbps": round(KB / ms_o / 1e6, 2),
                          "duplex_gbps": round(2 * KB / ms_fo / 1e6, 2),
                          "duplex_fetch_ms": round(t_f, 2), "duplex_offload_ms": round(t_o, 2)}), flush=True)
        assert mma.get_last_error() == 0
    mma.host_free(hp)


if __name__ == "__main__":
    main()
