#!/usr/bin/env python3
"""Measure how each single-GPU path mode moves the BASELINE workloads (design input for the
per-path mode choice, north_star (d) "chosen per path by measurement").

Modes on one B200 (one PCIe link): copy engine only, SM zero-copy only, and both at once
(the direct path in CE mode plus a loopback path in zero-copy mode, split by the planner at
the stated ratio). Workloads: contiguous 1 GiB (config 2 point) and a 1 GiB paged-KV
fetch/offload (config 3 shape, 8192 tokens). Prints one JSON object per line."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2512_16056_b200 as mma  # noqa: E402
from mma_inputs import workloads as W  # noqa: E402

GiB = 1 << 30


def timed(fn, stream, reps=5):
    fn()
    stream.synchronize()
    best = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        best.append(a.elapsed_time(b))
    return statistics.median(best)


def main():
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    B = GiB
    host = torch.empty(B, dtype=torch.uint8).pin_memory()
    host2 = torch.empty(B, dtype=torch.uint8).pin_memory()
    dev = torch.empty(B, dtype=torch.uint8, device="cuda")
    shape = W.scaled_kv(8192)
    ho, do, sb, hpool, dbytes = W.kv_segments(shape)
    pool = torch.empty(hpool, dtype=torch.uint8).pin_memory()
    cache = torch.empty(dbytes, dtype=torch.uint8, device="cuda")
    lens = np.full(len(ho), sb, dtype=np.int64)
    fetch = mma.make_segments(pool.data_ptr() + ho, cache.data_ptr() + do, lens)
    offload = mma.make_segments(cache.data_ptr() + do, pool.data_ptr() + ho, lens)
    KB = int(lens.sum())

    configs = [("ce", [1, 1], [1, 0]), ("zc", [2, 2], [1, 0])]
    for r in ((3, 1), (2, 1), (1, 1), (1, 2)):
        configs.append((f"ce+zc {r[0]}:{r[1]}", [1, 2], list(r)))
    for chunk in (1 << 20, 4 << 20):
        for name, modes, bw in configs:
            cfg = mma.default_config()
            cfg.chunk_bytes[0] = cfg.chunk_bytes[1] = chunk
            cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = 0
            cfg.loopback_relays = 1
            cfg.debug_log = 0
            mma.init(cfg)
            for d in (mma.H2D, mma.D2H):
                mma.set_path_modes(0, d, modes)
                mma.set_bandwidth(0, d, bw)
            res = {"chunk": chunk, "mode": name, "bw": bw}
            with torch.cuda.stream(s):
                res["contig_h2d"] = B / timed(lambda: mma.memcpy_h2d(dev, host, B, stream=s), s) / 1e6
                res["contig_d2h"] = B / timed(lambda: mma.memcpy_d2h(host2, dev, B, stream=s), s) / 1e6
                res["kv_h2d"] = KB / timed(lambda: mma.memcpy_h2d_segments(*fetch, 0, stream=s), s) / 1e6
                res["kv_d2h"] = KB / timed(lambda: mma.memcpy_d2h_segments(*offload, 0, stream=s), s) / 1e6
            assert mma.get_last_error() == 0
            print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in res.items()}), flush=True)
    # native references on the same buffers
    cfg = mma.default_config()
    cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = (1 << 64) - 1
    mma.init(cfg)
    with torch.cuda.stream(s):
        res = {"mode": "native (cudaMemcpyAsync per copy)",
               "contig_h2d": B / timed(lambda: mma.memcpy_h2d(dev, host, B, stream=s), s) / 1e6,
               "contig_d2h": B / timed(lambda: mma.memcpy_d2h(host2, dev, B, stream=s), s) / 1e6,
               "kv_h2d": KB / timed(lambda: mma.memcpy_h2d_segments(*fetch, 0, stream=s), s) / 1e6,
               "kv_d2h": KB / timed(lambda: mma.memcpy_d2h_segments(*offload, 0, stream=s), s) / 1e6}
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in res.items()}), flush=True)


if __name__ == "__main__":
    main()
