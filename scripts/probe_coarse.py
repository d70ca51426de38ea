#!/usr/bin/env python3
"""Probe (design input): config 3's coarse variant ("coarse 2 MiB host blocks,
all layers per block") -- the host keeps each 16-token block's KV of all 32 layers in one
2 MiB slot (LMCache-style chunks), the device keeps the paged layer-major cache. The table
is in host order, so consecutive segments are host-adjacent inside a block. Compared on the
one link: the direct path by SM zero-copy; and one loopback relay ring carrying every byte
(its copy-engine hop merges each block's host-adjacent pieces into one 2 MiB DMA into the
slot, the relay kernel scatters the slot to the 32 KiB device blocks). One JSON line per mode."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_16056_b200 as mma  # noqa: E402
from mma_inputs import permutation  # noqa: E402
from mma_inputs import workloads as W  # noqa: E402

MiB = 1 << 20


def main():
    torch.cuda.set_device(0)
    shape = W.KVShape()
    sb = shape.seg_bytes
    per_block = shape.layers * 2                       # segments of one block, host-adjacent
    nb = shape.nblocks
    _, dev_off, _, _, dbytes = W.kv_segments(shape)
    # host: block b's 2 MiB slot at a seeded permutation of a 2x pool of block slots
    slot = permutation(7, 2 * nb)[:nb].astype(np.int64)
    k = np.arange(shape.nsegs, dtype=np.int64)
    lkv, blk = k // nb, k % nb
    host_off = slot[blk] * (per_block * sb) + lkv * sb
    order = np.lexsort((lkv, blk))                   # host order: block-major
    host_off, dev_off = host_off[order], dev_off[order]
    lens = np.full(len(host_off), sb, dtype=np.int64)
    pool = mma.host_alloc(2 * nb * per_block * sb)
    cache = torch.empty(dbytes, dtype=torch.uint8, device="cuda")
    B = int(lens.sum())
    s = torch.cuda.Stream()
    fetch = mma.make_segments(pool + host_off, cache.data_ptr() + dev_off, lens)
    offload = mma.make_segments(cache.data_ptr() + dev_off, pool + host_off, lens)

    def rate(fn, reps=3):
        fn()
        s.synchronize()
        out = []
        for _ in range(reps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            fn()
            b.record(s)
            b.synchronize()
            out.append(a.elapsed_time(b))
        return round(B / statistics.median(out) / 1e6, 2)

    for name, lb, modes, bw in (("direct zero-copy", 0, [mma.HOP_ZC], [1]),
                                ("loopback kernel ring only", 1, [mma.HOP_ZC, mma.HOP_CE], [0, 1]),
                                ("loopback copy-engine ring only", 1, [mma.HOP_ZC, mma.HOP_CE_P2P], [0, 1])):
        cfg = mma.default_config()
        cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = 0
        cfg.loopback_relays = lb
        cfg.npaths, cfg.path_gpus[0] = 1, 0
        cfg.debug_log = 0
        cfg.host_order = 0
        mma.init(cfg)
        for d in (mma.H2D, mma.D2H):
            mma.set_path_modes(0, d, modes)
            mma.set_bandwidth(0, d, bw)
        with torch.cuda.stream(s):
            h = rate(lambda: mma.memcpy_h2d_segments(*fetch, 0, stream=s))
            o = rate(lambda: mma.memcpy_d2h_segments(*offload, 0, stream=s))
        print(json.dumps({"mode": name, "h2d_gbps": h, "d2h_gbps": o, "bytes": B,
                          "host_runs_bytes": per_block * sb, "segments": len(lens)}), flush=True)
    assert mma.get_last_error() == 0


if __name__ == "__main__":
    main()
