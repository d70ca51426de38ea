"""Helpers shared by the GPU tests (no method arithmetic: configuration and buffers)."""
from __future__ import annotations

import numpy as np

import mma_inputs

G = 4096   # guard band bytes on each side of a destination


def configure(mma, *, loopback=1, chunk=1 << 20, slots=2, plan_mode=0, hop=(0, 0),
              thr=0, ctas=8, debug=1, paths=None, claim=None, host_order=None):
    cfg = mma.default_config()
    cfg.chunk_bytes[0] = cfg.chunk_bytes[1] = chunk
    cfg.claim_bytes = chunk if claim is None else claim   # dynamic pull claims = chunks
    cfg.ring_slots = slots
    cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = thr
    cfg.loopback_relays = loopback
    cfg.plan_mode = plan_mode
    cfg.hop_mode[0], cfg.hop_mode[1] = hop
    cfg.relay_ctas = ctas
    cfg.debug_log = debug
    if host_order is not None:
        cfg.host_order = host_order
    if paths is not None:
        cfg.npaths = len(paths)
        for i, g in enumerate(paths):
            cfg.path_gpus[i] = g
    mma.init(cfg)
    return cfg


def pinned(torch, nbytes, seed=None, offset=0):
    t = torch.empty(max(nbytes, 1), dtype=torch.uint8).pin_memory()
    if seed is not None and nbytes:
        mma_inputs.fill_pattern(t.numpy()[:nbytes], seed, offset)
    return t


def guarded_device(torch, nbytes, dev=0):
    return torch.full((nbytes + 2 * G,), 0xA5, dtype=torch.uint8, device=f"cuda:{dev}")


def guarded_host(nbytes):
    return np.full(nbytes + 2 * G, 0xA5, dtype=np.uint8)
