#!/usr/bin/env python3
"""Probe: k loopback relay rings on GPU 0 (relays share GPU 0's engine streams, so no stream
shares a hardware queue with another engine GPU's) by ring kind and relay CTAs, 1 GiB
contiguous, equal bandwidths. Compared with scripts/sweep_vpaths.py's virtual-GPU rows, it
separates what many kernel rings cost from what 80 streams on one device's 32 hardware
queues cost. One JSON object per row."""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2512_16056_b200 as mma  # noqa: E402
import os  # noqa: E402

if os.environ.get("MMA_LIB_VARIANT"):       # a variant build of libmma.so (scripts/build_variant.sh)
    from paper_2512_16056_b200 import mma as _binding
    _binding.LIB_PATH = Path(os.environ["MMA_LIB_VARIANT"])

MiB, GiB = 1 << 20, 1 << 30


def main():
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    B = GiB
    host = torch.empty(B, dtype=torch.uint8).pin_memory()
    dev = torch.empty(B, dtype=torch.uint8, device="cuda")

    def timed(fn, reps=8):
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
        return B / statistics.median(out) / 1e6

    import os
    rings = [int(x) for x in os.environ.get("PROBE_RINGS", "1,3,7").split(",")]
    kinds = [int(x) for x in os.environ.get("PROBE_KINDS", "1,3").split(",")]
    ctas_list = [int(x) for x in os.environ.get("PROBE_CTAS", "8,4").split(",")]
    for lb in rings:
        for mode in kinds:
            for ctas in ctas_list:
                cfg = mma.default_config()
                cfg.chunk_bytes[0] = cfg.chunk_bytes[1] = 8 * MiB
                cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = 0
                cfg.loopback_relays = lb
                cfg.npaths, cfg.path_gpus[0] = 1, 0
                cfg.debug_log = 0
                cfg.relay_ctas = ctas
                mma.init(cfg)
                r = {"loopback_rings": lb, "kind": {1: "kernel_ring", 3: "ce_p2p_ring"}[mode], "relay_ctas": ctas,
                     "unit_bytes": int(os.environ.get("MMA_UNIT_BYTES", 512 << 10))}
                for d in (0, 1):
                    mma.set_path_modes(0, d, [1] + [mode] * lb)
                    mma.set_bandwidth(0, d, [1] * (lb + 1))
                with torch.cuda.stream(s):
                    r["h2d"] = round(timed(lambda: mma.memcpy_h2d(dev, host, B, stream=s)), 2)
                    r["d2h"] = round(timed(lambda: mma.memcpy_d2h(host, dev, B, stream=s)), 2)
                print(json.dumps(r), flush=True)
    assert mma.get_last_error() == 0


if __name__ == "__main__":
    main()
