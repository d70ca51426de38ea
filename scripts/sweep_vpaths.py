#!/usr/bin/env python3
"""Path-count overhead on one link: k = 1/2/4/8 paths into GPU 0 through the engine's
virtual GPUs (MMA_VGPUS=8), every path sharing the one PCIe link. The metric's
k axis cannot be measured on a one-GPU box; what can be measured is what k paths' machinery
(per-path streams, staging rings and their flags, relay kernels, k-way fork / join) costs
when it has no extra link to win: GB/s of the k-path copy vs the native copy of the same
bytes on the same link. Relay kinds forced per row (kernel ring, all-copy-engine ring,
one-hop zero-copy) at equal bandwidths, so 1 - 1/k of the bytes take the relay machinery,
plus the engine's own per-path measurement ("calibrated"). One JSON object per row."""
import json
import os
import statistics
import sys
from pathlib import Path

os.environ.setdefault("MMA_VGPUS", "8")
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2512_16056_b200 as mma  # noqa: E402

MiB, GiB = 1 << 20, 1 << 30
CE, ZC, P2P = 1, 2, 3


def timed(fn, s, reps):
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
    return statistics.median(out)


def main():
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    sizes = [int(x) for x in os.environ.get("SWEEP_SIZES", f"{64 * MiB},{GiB}").split(",")]
    chunk = int(os.environ.get("SWEEP_CHUNK", str(8 * MiB)))
    host = torch.empty(max(sizes), dtype=torch.uint8).pin_memory()
    dev = torch.empty(max(sizes), dtype=torch.uint8, device="cuda")
    native = {}
    for k in (1, 2, 4, 8):
        for kind, mode in (("calibrated", None), ("kernel_ring", CE), ("ce_p2p_ring", P2P), ("zc_one_hop", ZC)):
            if k == 1 and mode is not None:
                continue
            cfg = mma.default_config()
            cfg.chunk_bytes[0] = cfg.chunk_bytes[1] = chunk
            cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = (1 << 64) - 1 if k == 1 else 0
            cfg.npaths = k
            for i in range(k):
                cfg.path_gpus[i] = i
            cfg.debug_log = 0
            mma.init(cfg)
            for d in (mma.H2D, mma.D2H):
                assert len(mma.get_paths(0, d)) == k
                if k == 1:
                    continue
                if mode is None:
                    mma.calibrate(0, d, GiB)
                else:
                    mma.set_path_modes(0, d, [CE] + [mode] * (k - 1))
                    mma.set_bandwidth(0, d, [1] * k)
            for B in sizes:
                reps = 10 if B <= GiB else 3
                with torch.cuda.stream(s):
                    for d, fn in ((mma.H2D, lambda: mma.memcpy_h2d(dev, host, B, stream=s)),
                                  (mma.D2H, lambda: mma.memcpy_d2h(host, dev, B, stream=s))):
                        mma.reset_stats(0)
                        ms = timed(fn, s, reps)
                        gbps = B / ms / 1e6
                        key = (B, d)
                        if k == 1:
                            native[key] = gbps
                        st = mma.get_stats(0)
                        row = {"k": k, "relay_kind": "native" if k == 1 else kind,
                               "dir": "h2d" if d == 0 else "d2h", "bytes": B, "chunk": chunk, "gbps": round(gbps, 2),
                               "of_native": round(gbps / native[key], 4),
                               "relay_fraction": round(st["relay_bytes"] / max(1, st["bytes"]), 3),
                               "modes": [p["mode"] for p in mma.get_paths(0, d)],
                               "mbps": [p["mbps"] for p in mma.get_paths(0, d)]}
                        print(json.dumps(row), flush=True)
            assert mma.get_last_error() == 0
    mma.finalize()


if __name__ == "__main__":
    main()
