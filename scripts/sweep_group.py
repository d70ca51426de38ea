#!/usr/bin/env python3
"""Ring hop grouping (plane.cpp group_chunks): a copy carried entirely by one loopback relay
ring, both ring kinds, over chunk size C, ring depth S and MMA_GROUP_BYTES (0 = one chunk per
DMA and flag operation), against the native copy. Each group-bytes value runs in its own
process (the knob is read at engine init)."""
import json, os, statistics, subprocess, sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CHILD = r'''
import json, os, statistics, sys
sys.path.insert(0, %r)
import torch
import paper_2512_16056_b200 as mma
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
nat = {d: B / timed(f) / 1e6 for d, f in (("h2d", lambda: mma.memcpy_h2d(dev, host, B, stream=s)),
                                          ("d2h", lambda: mma.memcpy_d2h(host, dev, B, stream=s)))}
for kind, hop in (("kernel", mma.HOP_CE), ("ce_p2p", mma.HOP_CE_P2P)):
  for C in [int(x) for x in os.environ.get("SWEEP_C", "1048576,2097152,4194304,8388608").split(",")]:
    for S in [int(x) for x in os.environ.get("SWEEP_S", "4,8").split(",")]:
        cfg = mma.default_config()
        cfg.chunk_bytes[0] = cfg.chunk_bytes[1] = C
        cfg.ring_slots = S
        cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = 0
        cfg.loopback_relays = 1
        cfg.hop_mode[0] = cfg.hop_mode[1] = hop
        cfg.debug_log = 0
        mma.init(cfg)
        for d in (mma.H2D, mma.D2H):
            mma.set_bandwidth(0, d, [0, 1])
        h = B / timed(lambda: mma.memcpy_h2d(dev, host, B, stream=s)) / 1e6
        d2 = B / timed(lambda: mma.memcpy_d2h(host, dev, B, stream=s)) / 1e6
        print(json.dumps({"group_bytes": %d, "lanes": os.environ.get("MMA_HOP_LANES", "2"), "kind": kind, "C": C, "S": S, "h2d_frac": round(h / nat["h2d"], 3),
                          "d2h_frac": round(d2 / nat["d2h"], 3), "native": {k: round(v, 2) for k, v in nat.items()}}), flush=True)
        assert mma.get_last_error() == 0
'''
# argv: group-bytes values; MMA_HOP_LANES from the environment is passed through
for gb in [int(x) for x in (sys.argv[1:] or ["0", str(2 << 20), str(4 << 20)])]:
    env = dict(os.environ, MMA_GROUP_BYTES=str(gb))
    subprocess.run([sys.executable, "-c", CHILD % (str(ROOT), gb)], env=env, check=False)
