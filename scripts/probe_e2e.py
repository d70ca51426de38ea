#!/usr/bin/env python3
"""Where the synchronous (e2e) step time goes: host time of each API call, device time,
for the config-3 fetch + offload with each mode combination (design input)."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2512_16056_b200 as mma
from mma_inputs import workloads as W

torch.cuda.set_device(0)
s = torch.cuda.Stream()
shape = W.KVShape()
ho, do, sb, hpool, dbytes = W.kv_segments(shape)
ptr = mma.host_alloc(hpool)
cache = torch.empty(dbytes, dtype=torch.uint8, device="cuda")
lens = np.full(len(ho), sb, dtype=np.int64)
fetch = mma.make_segments(ptr + ho, cache.data_ptr() + do, lens)
off = mma.make_segments(cache.data_ptr() + do, ptr + ho, lens)
B = int(lens.sum())
for hm, dm in ((1, 2), (2, 2), (1, 1)):
    cfg = mma.default_config(); cfg.npaths = 1; cfg.path_gpus[0] = 0; cfg.debug_log = 0
    mma.init(cfg)
    mma.set_path_modes(0, mma.H2D, [hm]); mma.set_path_modes(0, mma.D2H, [dm])
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        mma.memcpy_h2d_segments(*fetch, 0, stream=s)
        t1 = time.perf_counter()
        mma.memcpy_d2h_segments(*off, 0, stream=s)
        t2 = time.perf_counter()
        s.synchronize()
        t3 = time.perf_counter()
        if rep:
            print(json.dumps(dict(h2d={1: "ce", 2: "zc"}[hm], d2h={1: "ce", 2: "zc"}[dm],
                                  h2d_call_ms=round((t1 - t0) * 1e3, 2), d2h_call_ms=round((t2 - t1) * 1e3, 2),
                                  wait_ms=round((t3 - t2) * 1e3, 2), step_ms=round((t3 - t0) * 1e3, 2),
                                  e2e_gbps=round(2 * B / (t3 - t0) / 1e9, 2))), flush=True)
