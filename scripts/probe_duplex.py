#!/usr/bin/env python3
"""Probe (design input): PCIe is full duplex -- how fast do request A's KV fetch (H2D) and
request B's offload (D2H, disjoint blocks) run AT ONCE on one link, per mode pair?
Config-3 shapes (4 GiB each way, 131,072 x 32 KiB). The offload is enqueued first (its
issue is short in zero-copy mode), both on their own streams; GB/s = 8 GiB / wall time of
the pair (CUDA events), best of 3. Alone-rates for reference."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_16056_b200 as mma  # noqa: E402
from mma_inputs import workloads as W  # noqa: E402


def main():
    torch.cuda.set_device(0)
    shape = W.KVShape()
    ho, do, sb, hpool, dbytes = W.kv_segments(shape)
    ho2, do2, _, _, _ = W.kv_segments(shape, request=1)
    hp = mma.host_alloc(hpool)
    cache = torch.empty(dbytes, dtype=torch.uint8, device="cuda")
    lens = np.full(len(ho), sb, dtype=np.int64)
    KB = int(lens.sum())
    fetch = mma.make_segments(hp + ho, cache.data_ptr() + do, lens)
    offload = mma.make_segments(cache.data_ptr() + do2, hp + ho2, lens)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cfg = mma.default_config()
    cfg.npaths = 1
    cfg.path_gpus[0] = 0
    cfg.debug_log = 0
    mma.init(cfg)
    names = {mma.HOP_CE: "ce", mma.HOP_ZC: "zc"}
    for fm in (mma.HOP_CE, mma.HOP_ZC):
        for om in (mma.HOP_CE, mma.HOP_ZC):
            mma.set_path_modes(0, mma.H2D, [fm])
            mma.set_path_modes(0, mma.D2H, [om])
            best = None
            for rep in range(4):
                torch.cuda.synchronize()
                a = torch.cuda.Event(enable_timing=True)
                b1 = torch.cuda.Event(enable_timing=True)
                b2 = torch.cuda.Event(enable_timing=True)
                a.record(s1)
                s2.wait_event(a)
                mma.memcpy_d2h_segments(*offload, 0, stream=s2)
                mma.memcpy_h2d_segments(*fetch, 0, stream=s1)
                b1.record(s1)
                b2.record(s2)
                torch.cuda.synchronize()
                ms = max(a.elapsed_time(b1), a.elapsed_time(b2))
                if rep:
                    best = ms if best is None else min(best, ms)
            print(json.dumps({"fetch": names[fm], "offload": names[om],
                              "duplex_gbps": round(2 * KB / (best * 1e-3) / 1e9, 2)}), flush=True)
            assert mma.get_last_error() == 0
    mma.host_free(hp)


if __name__ == "__main__":
    main()
