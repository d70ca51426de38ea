#!/usr/bin/env python3
"""Engine timeline (Chrome trace) of a 1 GiB contiguous copy carried by K loopback kernel
rings plus the direct path, at a given relay CTA count (RINGS=7 CTAS=16 by default):
where does a wave's time go when the rings have many CTAs? Writes
gpurun_out/trace_rings_{h2d,d2h}_k{K}_c{CTAS}.json and prints per-row busy time."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2512_16056_b200 as mma  # noqa: E402

K = int(os.environ.get("RINGS", "7"))
CTAS = int(os.environ.get("CTAS", "16"))
MiB = 1 << 20
CHUNK = int(os.environ.get("CHUNK", str(8 * MiB)))
RING_ONLY = os.environ.get("RING_ONLY") == "1"          # the direct path gets no chunk
torch.cuda.set_device(0)
s = torch.cuda.Stream()
B = 1 << 30
host = torch.empty(B, dtype=torch.uint8).pin_memory()
dev = torch.empty(B, dtype=torch.uint8, device="cuda")
cfg = mma.default_config()
cfg.chunk_bytes[0] = cfg.chunk_bytes[1] = CHUNK
cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = 0
cfg.loopback_relays = K
cfg.npaths, cfg.path_gpus[0] = 1, 0
cfg.relay_ctas = CTAS
cfg.debug_log = 0
mma.init(cfg)
for d in (mma.H2D, mma.D2H):
    mma.set_path_modes(0, d, [mma.HOP_CE] * (K + 1))
    mma.set_bandwidth(0, d, [0 if RING_ONLY else 1] + [1] * K)
mma.memcpy_h2d(dev, host, B, stream=s)
mma.memcpy_d2h(host, dev, B, stream=s)
s.synchronize()
out = Path("gpurun_out")
out.mkdir(exist_ok=True)
for name, fn in (("h2d", lambda: mma.memcpy_h2d(dev, host, B, stream=s)),
                 ("d2h", lambda: mma.memcpy_d2h(host, dev, B, stream=s))):
    mma.trace_begin()
    fn()
    s.synchronize()
    p = out / f"trace_rings_{name}_k{K}_c{CTAS}_C{CHUNK >> 20}M{'_ringonly' if RING_ONLY else ''}.json"
    n = mma.trace_end(str(p))
    ev = json.load(open(p))["traceEvents"]
    t0 = min(e["ts"] for e in ev)
    t1 = max(e["ts"] + e["dur"] for e in ev)
    rows = {}
    for e in ev:
        r = rows.setdefault(f'{e["pid"]}/{e["tid"]}', [0.0, 0, []])
        r[0] += e["dur"]
        r[1] += 1
        if len(r[2]) < 6:
            r[2].append((e["name"][:28], round(e["ts"] - t0, 1), round(e["dur"], 1)))
    print(json.dumps({"dir": name, "rings": K, "ctas": CTAS, "chunk": CHUNK, "ring_only": RING_ONLY,
                      "gbps": round(B / (t1 - t0) / 1e3, 2), "span_us": round(t1 - t0, 1), "spans": n,
                      "rows": {k: {"busy_us": round(v[0], 1), "n": v[1], "first": v[2]} for k, v in rows.items()}}),
          flush=True)
assert mma.get_last_error() == 0
