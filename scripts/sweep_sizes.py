#!/usr/bin/env python3
"""BASELINE config 2 on the GPUs this box exposes: contiguous H2D and D2H size sweep
4 MiB .. 16 GiB into GPU 0 (the paper's Fig 7 shape, §5.1.1), native
cudaMemcpyAsync vs the engine with every visible GPU as a path. With one GPU the engine has
one link; the loopback rows then show what the relay machinery itself costs on that link
(staging ring + relay kernel, or one-hop zero-copy, sharing the link 1:1 with the direct
path) -- the overhead the paper's fallback threshold exists for.
One JSON object per (size, direction, variant) on stdout."""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2512_16056_b200 as mma  # noqa: E402

MiB, GiB = 1 << 20, 1 << 30


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
    return statistics.median(out), min(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max", type=int, default=16 * GiB)
    ap.add_argument("--chunk", type=int, default=4 * MiB)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    sizes = [4 * MiB << j for j in range(13) if (4 * MiB << j) <= args.max]
    top = sizes[-1]
    host = torch.empty(top, dtype=torch.uint8).pin_memory()
    dev = torch.empty(top, dtype=torch.uint8, device="cuda")
    ngpu = torch.cuda.device_count()
    variants = [("native", None), ("mma", dict(loopback=0, modes=None, bw=None))]
    if ngpu == 1:
        variants += [("loopback-ring 1:1", dict(loopback=1, modes=[1, 1], bw=[1, 1])),
                     ("loopback-ce-p2p-ring 1:1", dict(loopback=1, modes=[1, 3], bw=[1, 1])),
                     ("loopback-zc 1:1", dict(loopback=1, modes=[1, 2], bw=[1, 1]))]
    for name, v in variants:
        cfg = mma.default_config()
        cfg.chunk_bytes[0] = cfg.chunk_bytes[1] = args.chunk
        cfg.debug_log = 0
        if v is None:
            cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = (1 << 64) - 1
        else:
            cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = 0
            cfg.loopback_relays = v["loopback"]
        mma.init(cfg)
        if v is not None:
            for d in (mma.H2D, mma.D2H):
                if v["modes"]:
                    mma.set_path_modes(0, d, v["modes"])
                    mma.set_bandwidth(0, d, v["bw"])
                else:
                    mma.calibrate(0, d, GiB)
        for B in sizes:
            reps = 10 if B <= GiB else 3
            with torch.cuda.stream(s):
                for d, fn in ((mma.H2D, lambda: mma.memcpy_h2d(dev, host, B, stream=s)),
                              (mma.D2H, lambda: mma.memcpy_d2h(host, dev, B, stream=s))):
                    med, best = timed(fn, s, reps)
                    print(json.dumps({"variant": name, "dir": "h2d" if d == 0 else "d2h", "bytes": B,
                                      "paths": len(mma.get_paths(0, d)), "chunk": args.chunk,
                                      "gbps_median": round(B / med / 1e6, 2), "gbps_best": round(B / best / 1e6, 2),
                                      "reps": reps}), flush=True)
        assert mma.get_last_error() == 0


if __name__ == "__main__":
    main()
