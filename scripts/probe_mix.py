#!/usr/bin/env python3
"""Probe (design input): one PCIe link carrying a scattered transfer in two modes at once.

The direct path moves its share with the copy engine (one descriptor per 32 KiB block) while
a loopback path (a zero-copy kernel on the same GPU) moves the rest, split by the planner at
the given CE fraction. Alone, CE scattered D2H is limited by per-descriptor cost (51.5 GB/s
device rate, profiles/r01_probe_batch_dev.txt) and SM zero-copy by TLP overhead (128-byte
writes, 1.19x payload on the link, profiles/r01_bench.json pcie_hw) -- different limits, so
a mix may beat both. Workload: config-3 KV (4 GiB, 131,072 x 32 KiB). Timing: CUDA events on
the user stream around the call (host issue included, as in bench.py), best of reps."""
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
    pool = torch.empty(hpool, dtype=torch.uint8).pin_memory()
    cache = torch.empty(dbytes, dtype=torch.uint8, device="cuda")
    lens = np.full(len(ho), sb, dtype=np.int64)
    fetch = mma.make_segments(pool.data_ptr() + ho, cache.data_ptr() + do, lens)
    offload = mma.make_segments(cache.data_ptr() + do, pool.data_ptr() + ho, lens)
    KB = int(lens.sum())
    cfg = mma.default_config()
    cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = 0
    cfg.loopback_relays = 1
    cfg.debug_log = 0
    mma.init(cfg)
    for ce_pct in (0, 30, 40, 50, 60, 70, 80, 90, 100):
        res = {"ce_fraction": ce_pct / 100}
        for d, name, segs in ((mma.H2D, "h2d", fetch), (mma.D2H, "d2h", offload)):
            if ce_pct == 0:
                modes, bw = [mma.HOP_ZC, mma.HOP_ZC], [1, 0]
            elif ce_pct == 100:
                modes, bw = [mma.HOP_CE, mma.HOP_ZC], [1, 0]
            else:
                modes, bw = [mma.HOP_CE, mma.HOP_ZC], [ce_pct, 100 - ce_pct]
            mma.set_path_modes(0, d, modes)
            mma.set_bandwidth(0, d, bw)
            fn = (lambda: mma.memcpy_h2d_segments(*segs, 0, stream=s)) if d == mma.H2D else \
                 (lambda: mma.memcpy_d2h_segments(*segs, 0, stream=s))
            res[name + "_gbps"] = round(KB / timed(fn, s) / 1e6, 2)
        assert mma.get_last_error() == 0
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
