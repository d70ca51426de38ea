#!/usr/bin/env python3
"""Probe (design input): does the ORDER of a scattered transfer's segments matter?

Config-3 KV (131,072 x 32 KiB): the host slots are a random permutation of an 8 GiB pool, so
consecutive segments of the table hit random host pages. Same segment set, three orders:
table order (layer-major, host-random), sorted by host address, sorted by device address.
Each order is timed as one copy-engine batch (native) and as one SM zero-copy kernel, H2D and
D2H (CUDA events around the call, best of reps)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_16056_b200 as mma  # noqa: E402
from mma_inputs import workloads as W  # noqa: E402


def timed(fn, stream, reps=4):
    fn()
    stream.synchronize()
    best = None
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ms = a.elapsed_time(b)
        best = ms if best is None else min(best, ms)
    return best


def main():
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    shape = W.KVShape()
    ho, do, sb, hpool, dbytes = W.kv_segments(shape)
    hp = mma.host_alloc(hpool)
    cache = torch.empty(dbytes, dtype=torch.uint8, device="cuda")
    lens = np.full(len(ho), sb, dtype=np.int64)
    KB = int(lens.sum())
    orders = {"table": np.arange(len(ho)), "host_sorted": np.argsort(ho, kind="stable"),
              "device_sorted": np.argsort(do, kind="stable")}
    for mode_name, cfg_fb, hop in (("ce_native", (1 << 64) - 1, mma.HOP_CE), ("zc_kernel", 0, mma.HOP_ZC)):
        cfg = mma.default_config()
        cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = cfg_fb
        cfg.hop_mode[0] = cfg.hop_mode[1] = hop
        cfg.npaths = 1
        cfg.path_gpus[0] = 0
        cfg.debug_log = 0
        mma.init(cfg)
        for oname, perm in orders.items():
            h, d = ho[perm], do[perm]
            fetch = mma.make_segments(hp + h, cache.data_ptr() + d, lens)
            offload = mma.make_segments(cache.data_ptr() + d, hp + h, lens)
            res = {"mode": mode_name, "order": oname}
            res["h2d_gbps"] = round(KB / timed(lambda: mma.memcpy_h2d_segments(*fetch, 0, stream=s), s) / 1e6, 2)
            res["d2h_gbps"] = round(KB / timed(lambda: mma.memcpy_d2h_segments(*offload, 0, stream=s), s) / 1e6, 2)
            assert mma.get_last_error() == 0
            print(json.dumps(res), flush=True)
    mma.host_free(hp)


if __name__ == "__main__":
    main()
