#!/usr/bin/env python3
"""Engine timeline (Chrome trace) of a loopback multipath copy on one GPU, plus an overlap
summary: the direct DMA stream, two relay hop streams and the relay kernel run at once.
Writes gpurun_out/trace_loopback_{h2d,d2h}.json; with `p2p` as argument the relays are
all-copy-engine rings (hop 1 and the peer hop 2 on the same relay stream, the two streams
overlapping: the paper's dual pipeline, Fig 6b) -> trace_loopback_p2p_{h2d,d2h}.json."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2512_16056_b200 as mma

def overlap(path):
    ev = json.load(open(path))["traceEvents"]
    rows = {}
    for e in ev:
        rows.setdefault(e["tid"], []).append((e["ts"], e["ts"] + e["dur"]))
    t0 = min(a for v in rows.values() for a, _ in v); t1 = max(b for v in rows.values() for _, b in v)
    # sweep: time with >= 2 rows busy
    pts = sorted({x for v in rows.values() for s in v for x in s})
    busy2 = 0.0
    for a, b in zip(pts, pts[1:]):
        m = (a + b) / 2
        if sum(any(s <= m < e for s, e in v) for v in rows.values()) >= 2:
            busy2 += b - a
    return {"span_us": round(t1 - t0, 1), "rows": {k: round(sum(e - s for s, e in v), 1) for k, v in rows.items()},
            "time_with_2plus_rows_busy_us": round(busy2, 1), "events": len(ev)}

torch.cuda.set_device(0)
s = torch.cuda.Stream()
B = 512 << 20
host = torch.empty(B, dtype=torch.uint8).pin_memory()
dev = torch.empty(B, dtype=torch.uint8, device="cuda")
cfg = mma.default_config()
cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = 0
cfg.loopback_relays = 2
cfg.hop_mode[0] = cfg.hop_mode[1] = mma.HOP_CE
p2p = len(sys.argv) > 1 and sys.argv[1] == "p2p"
mma.init(cfg)
if p2p:
    for d in (mma.H2D, mma.D2H):
        mma.set_path_modes(0, d, [mma.HOP_CE, mma.HOP_CE_P2P, mma.HOP_CE_P2P])
for d in (mma.H2D, mma.D2H):
    mma.set_bandwidth(0, d, [2, 1, 1])
mma.memcpy_h2d(dev, host, B, stream=s); mma.memcpy_d2h(host, dev, B, stream=s); s.synchronize()
out = Path("gpurun_out"); out.mkdir(exist_ok=True)
for name, fn in (("h2d", lambda: mma.memcpy_h2d(dev, host, B, stream=s)),
                 ("d2h", lambda: mma.memcpy_d2h(host, dev, B, stream=s))):
    mma.trace_begin()
    fn()
    s.synchronize()
    p = out / (f"trace_loopback_p2p_{name}.json" if p2p else f"trace_loopback_{name}.json")
    n = mma.trace_end(str(p))
    print(json.dumps({"dir": name, "spans": n, **overlap(p)}), flush=True)
assert mma.get_last_error() == 0
