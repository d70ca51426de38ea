"""Deployment CLI of the engine (every measurement runs in libmma.so through the C ABI):

    python -m paper_2512_16056_b200 show                       # topology, paths, current vectors
    python -m paper_2512_16056_b200 calibrate --out cal.txt    # per device x direction: modes,
                                                               # concurrent rates, break-even
    python -m paper_2512_16056_b200 plan --device 0 --bytes 1GiB [--dir d2h]

`calibrate` is the once-per-box step; a serving process then loads the file
at init with MMA_CALIB=cal.txt (mma_load_calibration). Prints one JSON object.
"""
from __future__ import annotations

import argparse
import json
import sys


def size(s: str) -> int:
    s = s.strip()
    for suf, mul in (("GiB", 1 << 30), ("MiB", 1 << 20), ("KiB", 1 << 10)):
        if s.endswith(suf):
            return int(float(s[: -len(suf)]) * mul)
    return int(s)


def _paths(mma, d):
    return {name: mma.get_paths(d, dv) for name, dv in (("h2d", mma.H2D), ("d2h", mma.D2H))}


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2512_16056_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    sub.add_parser("show")
    c = sub.add_parser("calibrate")
    c.add_argument("--out", required=True, help="calibration file (mma_save_calibration format)")
    c.add_argument("--bytes", type=size, default=256 << 20, help="contiguous calibration transfer")
    c.add_argument("--devices", default="", help="comma-separated targets (default: all)")
    c.add_argument("--no-threshold", action="store_true", help="skip the break-even sweep")
    p = sub.add_parser("plan")
    p.add_argument("--device", type=int, default=0)
    p.add_argument("--bytes", type=size, required=True)
    p.add_argument("--dir", choices=["h2d", "d2h"], default="h2d")
    a = ap.parse_args(argv)

    import paper_2512_16056_b200 as mma
    mma.init()
    topo = mma.get_topology()
    if a.cmd == "show":
        out = {"topology": topo, "paths": {str(d): _paths(mma, d) for d in range(topo["ngpu"])}}
    elif a.cmd == "calibrate":
        devs = [int(x) for x in a.devices.split(",") if x] or list(range(topo["ngpu"]))
        out = {"topology": topo, "calibration": {}, "file": a.out}
        for d in devs:
            row = {}
            for name, dv in (("h2d", mma.H2D), ("d2h", mma.D2H)):
                mma.calibrate(d, dv, a.bytes)
                r = {"paths": mma.get_paths(d, dv), "rates": mma.get_calibration(d, dv)}
                if len(r["paths"]) > 1 and a.bytes >= (2 << 20):
                    r["chunk_bytes"] = mma.tune_chunk(d, dv, a.bytes)   # set MMA_CHUNK_BYTES_H2D/_D2H
                if not a.no_threshold and len(r["paths"]) > 1:
                    thr, found = mma.tune_threshold(d, dv, a.bytes)
                    r["fallback_bytes"] = thr if found else None
                row[name] = r
            out["calibration"][str(d)] = row
        mma.save_calibration(a.out)
    else:
        dv = mma.H2D if a.dir == "h2d" else mma.D2H
        path, fb = mma.get_plan(a.device, dv, a.bytes)
        counts = {}
        for p in path:
            counts[p] = counts.get(p, 0) + 1
        out = {"device": a.device, "dir": a.dir, "bytes": a.bytes, "fallback": fb, "nchunks": len(path),
               "chunks_per_path": {str(k): v for k, v in sorted(counts.items())}, "paths": _paths(mma, a.device)[a.dir]}
    print(json.dumps(out))
    mma.finalize()
    return 0


if __name__ == "__main__":
    sys.exit(main())
