#!/usr/bin/env python3
"""Relay kernels in the engine's real protocol (for ncu; VERDICT r1 missing #7): one H2D and
one D2H copy carried entirely by copy-engine relay rings (3 loopback rings, or with --peers
every other GPU as a relay of GPU 0), 8 MiB chunks, S = 4, through mma_memcpy_h2d/d2h --
the same waves, flags and launches as a production call. ncu serialises the launches; the
waves keep every kernel's waits on work enqueued before it (plane.cpp enqueue_rings)."""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2512_16056_b200 as mma

ap = argparse.ArgumentParser()
ap.add_argument("--bytes", type=int, default=768 << 20)
ap.add_argument("--peers", action="store_true")
a = ap.parse_args()
torch.cuda.set_device(0)
cfg = mma.default_config()
cfg.chunk_bytes[0] = cfg.chunk_bytes[1] = 8 << 20
cfg.ring_slots = 4
cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = 0
cfg.hop_mode[0] = cfg.hop_mode[1] = mma.HOP_CE
if a.peers and torch.cuda.device_count() > 1:
    cfg.loopback_relays = 0
else:
    cfg.loopback_relays = 3
    cfg.npaths = 1
    cfg.path_gpus[0] = 0
mma.init(cfg)
for d in (mma.H2D, mma.D2H):
    n = len(mma.get_paths(0, d))
    mma.set_bandwidth(0, d, [0] + [1] * (n - 1))   # the relay rings carry every byte
B = a.bytes
host = torch.empty(B, dtype=torch.uint8).pin_memory()
dev = torch.empty(B, dtype=torch.uint8, device="cuda")
mma.fill_pattern(dev, B, 7, 0)
torch.cuda.synchronize()
mma.memcpy_d2h(host, dev, B)
torch.cuda.synchronize()
dev.zero_()
mma.memcpy_h2d(dev, host, B)
torch.cuda.synchronize()
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
mma.verify_pattern(dev, B, 7, 0, cnt)
torch.cuda.synchronize()
assert int(cnt.item()) == 0 and mma.get_last_error() == 0
print("ok relay protocol", B, mma.get_stats(0)["kernels"])
