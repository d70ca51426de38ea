#!/usr/bin/env python3
"""Relay-ring efficiency on one link (design input): a copy carried entirely by one
loopback copy-engine relay ring (hop 1 DMA into the staging ring + relay kernel), swept
over chunk size C and ring depth S, vs the native copy -- the per-chunk cost the paper's
chunk-size and queue-length study measures (Fig 10). Both kinds of ring: the relay
kernel pulling the slot (hop mode ce) and the relay stream's own peer DMA (ce_p2p, the
paper's design, no SM work)."""
import json, statistics, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2512_16056_b200 as mma

torch.cuda.set_device(0)
s = torch.cuda.Stream()
B = 1 << 30
host = torch.empty(B, dtype=torch.uint8).pin_memory()
dev = torch.empty(B, dtype=torch.uint8, device="cuda")

def timed(fn, reps=5):
    fn(); s.synchronize(); out = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(s); fn(); b.record(s); b.synchronize(); out.append(a.elapsed_time(b))
    return statistics.median(out)

cfg = mma.default_config(); cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = (1 << 64) - 1; mma.init(cfg)
with torch.cuda.stream(s):
    nat = {d: B / timed(f) / 1e6 for d, f in (("h2d", lambda: mma.memcpy_h2d(dev, host, B, stream=s)),
                                              ("d2h", lambda: mma.memcpy_d2h(host, dev, B, stream=s)))}
print(json.dumps({"variant": "native", **{k: round(v, 2) for k, v in nat.items()}}), flush=True)
for kind, hop in (("kernel", mma.HOP_CE), ("ce_p2p", mma.HOP_CE_P2P)):
  for C in (1 << 20, 4 << 20, 8 << 20, 16 << 20):
    for S in (1, 2, 4, 8):
        cfg = mma.default_config()
        cfg.chunk_bytes[0] = cfg.chunk_bytes[1] = C
        cfg.ring_slots = S
        cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = 0
        cfg.loopback_relays = 1
        cfg.hop_mode[0] = cfg.hop_mode[1] = hop
        cfg.debug_log = 0
        mma.init(cfg)
        for d in (mma.H2D, mma.D2H):
            mma.set_bandwidth(0, d, [0, 1])        # the relay ring carries everything
        with torch.cuda.stream(s):
            h = B / timed(lambda: mma.memcpy_h2d(dev, host, B, stream=s)) / 1e6
            d2 = B / timed(lambda: mma.memcpy_d2h(host, dev, B, stream=s)) / 1e6
        print(json.dumps({"variant": "ring", "kind": kind, "C": C, "S": S, "h2d": round(h, 2), "d2h": round(d2, 2),
                          "h2d_frac": round(h / nat["h2d"], 3), "d2h_frac": round(d2 / nat["d2h"], 3)}), flush=True)
        assert mma.get_last_error() == 0
