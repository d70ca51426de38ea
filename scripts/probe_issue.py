#!/usr/bin/env python3
"""Host issue cost vs device time of the config-3 KV fetch/offload per mode (design input)."""
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
pool = torch.empty(hpool, dtype=torch.uint8).pin_memory()
cache = torch.empty(dbytes, dtype=torch.uint8, device="cuda")
lens = np.full(len(ho), sb, dtype=np.int64)
fetch = mma.make_segments(pool.data_ptr() + ho, cache.data_ptr() + do, lens)
off = mma.make_segments(cache.data_ptr() + do, pool.data_ptr() + ho, lens)
B = int(lens.sum())
for mode in (1, 2):
    cfg = mma.default_config(); cfg.hop_mode[0] = cfg.hop_mode[1] = mode; cfg.npaths = 1; cfg.path_gpus[0] = 0
    mma.init(cfg)
    for name, segs, fn in (("h2d", fetch, mma.memcpy_h2d_segments), ("d2h", off, mma.memcpy_d2h_segments)):
        for rep in range(3):
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            # gate the stream so the device does not start before the whole call is issued
            a.record(s)
            t0 = time.perf_counter(); fn(*segs, 0, stream=s); t1 = time.perf_counter()
            b.record(s); b.synchronize(); t2 = time.perf_counter()
            print(json.dumps(dict(mode={1: "ce", 2: "zc"}[mode], dir=name, issue_ms=round((t1 - t0) * 1e3, 2),
                                  wall_ms=round((t2 - t0) * 1e3, 2), event_ms=round(a.elapsed_time(b), 2),
                                  wall_gbps=round(B / (t2 - t0) / 1e9, 2))), flush=True)
