#!/usr/bin/env python3
"""Contention with background traffic (§3.4.2) on one B200: a native 4 GiB H2D copy
(the background flow, its own stream) runs while the engine moves 4 GiB by dynamic pull over
the direct path and one loopback path (both zero-copy, both on the same PCIe link). With
background_policy = 0 the engine keeps claiming; with 1 its CTAs wait after a unit that took
longer than yield_pct % of the pinned per-path rate predicts. Reported: completion time of
each flow alone and together, and the waits taken."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2512_16056_b200 as mma

B = 4 << 30
hb = torch.empty(B, dtype=torch.uint8).pin_memory()
db = torch.empty(B, dtype=torch.uint8, device="cuda")
hm = torch.empty(B, dtype=torch.uint8).pin_memory()
dm = torch.empty(B, dtype=torch.uint8, device="cuda")
sb, sm = torch.cuda.Stream(), torch.cuda.Stream()


def run(policy, with_bg, with_mma, yield_pct):
    cfg = mma.default_config()
    cfg.loopback_relays = 1
    cfg.plan_mode = 2
    cfg.hop_mode[0] = cfg.hop_mode[1] = mma.HOP_ZC
    cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = 0
    cfg.debug_log = 0
    cfg.background_policy = policy
    cfg.yield_pct = yield_pct
    mma.init(cfg)
    mma.set_bandwidth(0, mma.H2D, [27000, 27000])     # each path's share of the one link
    torch.cuda.synchronize()
    ev = {k: torch.cuda.Event(enable_timing=True) for k in ("b0", "b1", "m0", "m1")}
    if with_bg:
        ev["b0"].record(sb)
        with torch.cuda.stream(sb):
            db.copy_(hb, non_blocking=True)
        ev["b1"].record(sb)
    if with_mma:
        ev["m0"].record(sm)
        mma.memcpy_h2d(dm, hm, B, stream=sm)
        ev["m1"].record(sm)
    torch.cuda.synchronize()
    out = {"policy": policy, "yield_pct": yield_pct}
    if with_bg:
        out["background_ms"] = round(ev["b0"].elapsed_time(ev["b1"]), 2)
    if with_mma:
        out["mma_ms"] = round(ev["m0"].elapsed_time(ev["m1"]), 2)
        out["waits"] = mma.get_dynamic_backoffs(0)
    return out


run(0, True, True, 150)                                  # warm-up
res = [run(0, True, False, 150), run(0, False, True, 150)]
for pol, pct in ((0, 150), (1, 250), (1, 150)):
    for _ in range(2):
        res.append(run(pol, True, True, pct))
for r in res:
    print(json.dumps(r), flush=True)
