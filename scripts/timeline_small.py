#!/usr/bin/env python3
"""Tiny loopback-relay workload for an nsys timeline: 256 MiB H2D with the direct copy
engine path plus two loopback relay rings (copy engines + relay kernel overlapping)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2512_16056_b200 as mma
torch.cuda.set_device(0)
s = torch.cuda.Stream()
B = 256 << 20
host = torch.empty(B, dtype=torch.uint8).pin_memory()
dev = torch.empty(B, dtype=torch.uint8, device="cuda")
cfg = mma.default_config()
cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = 0
cfg.loopback_relays = 2
cfg.hop_mode[0] = cfg.hop_mode[1] = mma.HOP_CE
mma.init(cfg)
mma.set_bandwidth(0, mma.H2D, [2, 1, 1])
for _ in range(3):
    mma.memcpy_h2d(dev, host, B, stream=s)
s.synchronize()
print("ok", mma.get_last_error())
