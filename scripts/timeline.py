#!/usr/bin/env python3
"""A short workload for an nsys timeline (design evidence): one H2D and one D2H of 512 MiB
with the direct path in copy-engine mode plus two loopback relay rings (relay kernels
overlapping the copy engines), then a dynamic-pull KV fetch."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2512_16056_b200 as mma
from mma_inputs import workloads as W

torch.cuda.set_device(0)
s = torch.cuda.Stream()
B = 512 << 20
host = torch.empty(B, dtype=torch.uint8).pin_memory()
dev = torch.empty(B, dtype=torch.uint8, device="cuda")
cfg = mma.default_config()
cfg.chunk_bytes[0] = cfg.chunk_bytes[1] = 4 << 20
cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = 0
cfg.loopback_relays = 2
cfg.hop_mode[0] = cfg.hop_mode[1] = mma.HOP_CE
mma.init(cfg)
for d in (mma.H2D, mma.D2H):
    mma.set_bandwidth(0, d, [2, 1, 1])
for _ in range(2):
    mma.memcpy_h2d(dev, host, B, stream=s)
    mma.memcpy_d2h(host, dev, B, stream=s)
s.synchronize()
shape = W.scaled_kv(4096)
ho, do, sb, hpool, dbytes = W.kv_segments(shape)
pool = torch.empty(hpool, dtype=torch.uint8).pin_memory()
cache = torch.empty(dbytes, dtype=torch.uint8, device="cuda")
lens = np.full(len(ho), sb, dtype=np.int64)
segs = mma.make_segments(pool.data_ptr() + ho, cache.data_ptr() + do, lens)
cfg.hop_mode[0] = cfg.hop_mode[1] = mma.HOP_ZC
cfg.plan_mode = 2
mma.init(cfg)
for _ in range(2):
    mma.memcpy_h2d_segments(*segs, 0, stream=s)
s.synchronize()
print("counts", mma.get_dynamic_counts(0), "err", mma.get_last_error())
