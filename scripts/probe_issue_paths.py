#!/usr/bin/env python3
"""Host issue cost of one config-3 call (131,072 x 32 KiB segments) vs the number of paths,
every path in zero-copy mode (the mode the measured choice picks for scattered transfers on
more than one link), using loopback relays on one GPU: the enqueue time per call, split by
stage with MMA_TRACE=1 (stderr), and the device time. At N = 8 the device step shrinks ~8x
while the enqueue does not, so the enqueue bounds the end-to-end rate."""
import json, os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2512_16056_b200 as mma
from mma_inputs import workloads as W

shape = W.KVShape()
ho, do, sb, hpool, dbytes = W.kv_segments(shape, 0x4D4D44)
pool = mma.host_alloc(hpool)
cache = torch.empty(dbytes, dtype=torch.uint8, device="cuda")
lens = np.full(len(ho), sb, dtype=np.int64)
fetch = mma.make_segments(pool + ho, cache.data_ptr() + do, lens)
off = mma.make_segments(cache.data_ptr() + do, pool + ho, lens)
s = torch.cuda.Stream()
for lb in [int(x) for x in (sys.argv[1:] or ["0", "1", "3", "7"])]:
    cfg = mma.default_config()
    cfg.loopback_relays = lb
    cfg.hop_mode[0] = cfg.hop_mode[1] = mma.HOP_ZC
    cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = 0
    cfg.debug_log = 0
    cfg.npaths = 1
    cfg.path_gpus[0] = 0
    mma.init(cfg)
    for d in (mma.H2D, mma.D2H):
        mma.set_bandwidth(0, d, [1] * (1 + lb))
    for name, segs, fn in (("h2d", fetch, mma.memcpy_h2d_segments), ("d2h", off, mma.memcpy_d2h_segments)):
        fn(*segs, 0, stream=s)
        s.synchronize()
        mma.reset_stats(0)
        t = []
        for _ in range(5):
            s.synchronize()
            t0 = time.perf_counter()
            fn(*segs, 0, stream=s)
            t.append(time.perf_counter() - t0)
        s.synchronize()
        st = mma.get_stats(0)
        print(json.dumps({"paths": 1 + lb, "dir": name, "enqueue_ms": round(1e3 * sorted(t)[2], 3),
                          "issue_us_per_call": round(st["issue_us"] / st["calls"], 1),
                          "validate_us_per_call": round(st["validate_us"] / st["calls"], 1)}), flush=True)
