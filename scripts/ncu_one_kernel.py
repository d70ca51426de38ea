#!/usr/bin/env python3
"""One zero-copy launch of the config-3 shape (for ncu): --dir h2d|d2h, --tokens N."""
import argparse, os, sys
from pathlib import Path
os.environ.setdefault("MMA_UPLOAD", "ce")   # tables by DMA: the only zc_copy_kernel launch is the copy
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2512_16056_b200 as mma
from mma_inputs import workloads as W

ap = argparse.ArgumentParser(); ap.add_argument("--dir", default="d2h"); ap.add_argument("--tokens", type=int, default=32768)
a = ap.parse_args()
torch.cuda.set_device(0)
shape = W.KVShape() if a.tokens == 32768 else W.scaled_kv(a.tokens)
ho, do, sb, hpool, dbytes = W.kv_segments(shape)
pool = torch.zeros(hpool, dtype=torch.uint8).pin_memory()
cache = torch.zeros(dbytes, dtype=torch.uint8, device="cuda")
lens = np.full(len(ho), sb, dtype=np.int64)
cfg = mma.default_config(); cfg.hop_mode[0] = cfg.hop_mode[1] = mma.HOP_ZC; cfg.npaths = 1; cfg.path_gpus[0] = 0
mma.init(cfg)
if a.dir == "h2d":
    segs = mma.make_segments(pool.data_ptr() + ho, cache.data_ptr() + do, lens); mma.memcpy_h2d_segments(*segs, 0)
else:
    segs = mma.make_segments(cache.data_ptr() + do, pool.data_ptr() + ho, lens); mma.memcpy_d2h_segments(*segs, 0)
torch.cuda.synchronize(); assert mma.get_last_error() == 0; print("ok", a.dir, int(lens.sum()))
