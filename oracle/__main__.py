"""Oracle CLI (test infrastructure): plan a transfer, move a seeded one, or explore the ring.

    python -m oracle plan --bw 55000,55000 --bytes 64MiB --chunk 1MiB [--mode interleaved]
    python -m oracle move --bw 3,1 --bytes 10MiB --chunk 1MiB --slots 2 [--threaded]
    python -m oracle ring --n 6 --slots 3 [--fault publish-early|skip-credit]
"""
from __future__ import annotations

import argparse
import json
import sys

import numpy as np

import oracle


def size(s: str) -> int:
    s = s.strip()
    for suf, mul in (("GiB", 1 << 30), ("MiB", 1 << 20), ("KiB", 1 << 10), ("GB", 10**9), ("MB", 10**6), ("KB", 10**3)):
        if s.endswith(suf):
            return int(float(s[: -len(suf)]) * mul)
    return int(s)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m oracle")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("plan", "move"):
        p = sub.add_parser(name)
        p.add_argument("--bw", required=True, help="comma-separated MB/s per path, path 0 first")
        p.add_argument("--relay-only", action="store_true", help="path 0 is a relay too")
        p.add_argument("--bytes", type=size, required=True)
        p.add_argument("--chunk", type=size, required=True)
        p.add_argument("--thr", type=size, default=0)
        p.add_argument("--mode", choices=["contiguous", "interleaved", "pull"], default="contiguous")
        if name == "move":
            p.add_argument("--slots", type=int, default=2)
            p.add_argument("--threaded", action="store_true")
            p.add_argument("--seed", type=int, default=0x4D4D41)
    r = sub.add_parser("ring")
    r.add_argument("--n", type=int, default=6)
    r.add_argument("--slots", type=int, default=2)
    r.add_argument("--base", type=int, default=0)
    r.add_argument("--fault", choices=["none", "publish-early", "skip-credit"], default="none")
    a = ap.parse_args(argv)
    if a.cmd == "ring":
        fault = {"none": 0, "publish-early": 1, "skip-credit": 2}[a.fault]
        rc, states, bad = oracle.ring_explore(a.n, a.slots, a.base, fault)
        print(json.dumps({"rc": rc, "states": states, "violations": bad}))
        return 0 if rc == 0 else 1
    bw = [int(x) for x in a.bw.split(",")]
    kinds = [1] * len(bw) if a.relay_only else None
    mode = {"contiguous": 0, "interleaved": 1, "pull": 2}[a.mode]
    rc, path, counts, fb = oracle.plan(bw, a.bytes, a.chunk, a.thr, mode, kinds=kinds)
    if rc:
        print(json.dumps({"rc": rc}))
        return 1
    T, agg = oracle.predict(bw, a.bytes, a.chunk, path, kinds=kinds)
    out = {"nchunks": int(path.size), "fallback": fb, "counts": counts, "predicted_s": T,
           "predicted_gbps": agg, "path": path.tolist() if path.size <= 4096 else "(omitted)"}
    if a.cmd == "move":
        import mma_inputs
        src = mma_inputs.pattern_bytes(a.seed, a.bytes)
        dst = np.zeros_like(src)
        ev = np.zeros(max(path.size, 1) * oracle.NEV, np.uint64)
        wc = np.zeros(max(a.bytes, 1), np.uint32)
        rc = oracle.move_contiguous(dst, src, a.chunk, bw, path, S=a.slots, kinds=kinds, events=ev,
                                    write_count=wc,
                                    exec_mode=oracle.THREADED if a.threaded else oracle.DETERMINISTIC)
        out.update(rc=rc, bytes_equal=bool(np.array_equal(dst, src)),
                   exactly_once=bool((wc[:a.bytes] == 1).all()),
                   invariant_violations=oracle.check_events(ev, bw, path, a.slots, kinds=kinds))
    print(json.dumps(out))
    return 0


if __name__ == "__main__":
    sys.exit(main())
