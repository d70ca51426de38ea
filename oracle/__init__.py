"""ctypes front-end of the CPU oracle (oracle/mma_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs. The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"

DIRECT, RELAY = 0, 1
CONTIG, INTERLEAVED, PULL = 0, 1, 2
DETERMINISTIC, THREADED = 0, 1
FAULT_NONE, FAULT_PUBLISH_EARLY, FAULT_SKIP_CREDIT = 0, 1, 2
EV_STAGE_BEGIN, EV_STAGE_END, EV_PUBLISH, EV_FWD_BEGIN, EV_FWD_END, EV_CREDIT = range(6)
NEV = 6
EINVAL, ENOSPC, EDEADLK = -22, -28, -35


class Path_(C.Structure):
    _fields_ = [("kind", C.c_int32), ("bw_mbps", C.c_uint32), ("backlog", C.c_uint64)]


class Segment(C.Structure):
    _fields_ = [("src", C.c_void_p), ("dst", C.c_void_p), ("len", C.c_uint64)]


def build(force: bool = False) -> Path:
    """Compile liboracle.so with gcc (plain C11 + pthreads)."""
    src = HERE / "mma_oracle.c"
    if force or not LIB.exists() or LIB.stat().st_mtime < max(src.stat().st_mtime, (HERE / "mma_oracle.h").stat().st_mtime):
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-Wall", "-Wextra", "-fPIC", "-shared",
                               "-pthread", "-o", str(LIB), str(src)])
    return LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(str(LIB))
        u64, p = C.c_uint64, C.POINTER
        L.orc_nchunks.restype = u64
        L.orc_nchunks.argtypes = [u64, u64]
        L.orc_chunk_extent.argtypes = [u64, u64, u64, p(u64), p(u64)]
        L.orc_plan.argtypes = [p(Path_), C.c_int, u64, u64, u64, C.c_int, C.c_void_p, u64,
                               p(u64), C.c_void_p, p(C.c_int)]
        L.orc_predict.argtypes = [p(Path_), C.c_int, u64, u64, C.c_void_p, u64,
                                  p(C.c_double), p(C.c_double)]
        L.orc_move.argtypes = [p(Segment), u64, u64, p(Path_), C.c_int, C.c_void_p, u64,
                               C.c_uint32, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
        L.orc_segments_disjoint.argtypes = [p(Segment), u64]
        L.orc_check_events.restype = u64
        L.orc_check_events.argtypes = [C.c_void_p, p(Path_), C.c_int, C.c_void_p, u64,
                                       C.c_uint32, C.c_void_p]
        L.orc_ring_explore.argtypes = [C.c_int, C.c_int, u64, C.c_int, p(u64), p(u64)]
        L.orc_plan_multi.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, u64,
                                     C.c_int, C.c_int, C.c_void_p]
        L.orc_numa_order.argtypes = [C.c_void_p, u64, p(Path_), C.c_void_p, C.c_int, C.c_void_p]
        _lib = L
    return _lib


def make_paths(bw, kinds=None, backlog=None):
    P = len(bw)
    arr = (Path_ * P)()
    for i in range(P):
        arr[i].kind = (kinds[i] if kinds is not None else (DIRECT if i == 0 else RELAY))
        arr[i].bw_mbps = int(bw[i])
        arr[i].backlog = int(backlog[i]) if backlog is not None else 0
    return arr


def plan_multi(link_bw, relay_ok, targets, nchunks, C_, mode=INTERLEAVED, prefer=-1):
    """Joint pull plan of concurrent transfers (NEXT-1). relay_ok: L x L 0/1
    (row = endpoint GPU, column = link). Returns (rc, list of per-transfer link arrays)."""
    L = len(link_bw)
    bw = np.ascontiguousarray(link_bw, dtype=np.uint32)
    ok = np.ascontiguousarray(relay_ok, dtype=np.uint8).reshape(L, L)
    tg = np.ascontiguousarray(targets, dtype=np.int32)
    nc = np.ascontiguousarray(nchunks, dtype=np.uint64)
    out = np.full(max(1, int(nc.sum())), -1, dtype=np.int32)
    rc = lib().orc_plan_multi(L, bw.ctypes.data, ok.ctypes.data, len(tg), tg.ctypes.data, nc.ctypes.data,
                              C_, mode, prefer, out.ctypes.data)
    offs = np.concatenate([[0], np.cumsum(nc)]).astype(np.int64)
    return rc, [out[offs[t]:offs[t + 1]].copy() for t in range(len(tg))]


def numa_order(seg_node, bw, path_node, kinds=None):
    """Reading R23: the table order of v's segments, regrouped by host node."""
    sn = np.ascontiguousarray(seg_node, dtype=np.int32)
    pn = np.ascontiguousarray(path_node, dtype=np.int32)
    out = np.zeros(max(1, sn.size), dtype=np.uint32)
    lib().orc_numa_order(sn.ctypes.data, sn.size, make_paths(bw, kinds), pn.ctypes.data, len(bw), out.ctypes.data)
    return out[: sn.size]


def nchunks(B: int, C_: int) -> int:
    return int(lib().orc_nchunks(B, C_))


def chunk_extent(i: int, B: int, C_: int):
    off, ln = C.c_uint64(), C.c_uint64()
    lib().orc_chunk_extent(i, B, C_, C.byref(off), C.byref(ln))
    return off.value, ln.value


def plan(bw, B: int, C_: int, thr: int = 0, mode: int = CONTIG, kinds=None, backlog=None):
    """Returns (rc, path_of_chunk uint8 array, counts list, fallback bool)."""
    paths = make_paths(bw, kinds, backlog)
    P = len(bw)
    cap = max(1, nchunks(B, C_)) if (B and C_) else 1
    out = np.zeros(cap, dtype=np.uint8)
    counts = np.zeros(P, dtype=np.uint64)
    n = C.c_uint64()
    fb = C.c_int()
    rc = lib().orc_plan(paths, P, B, C_, thr, mode, out.ctypes.data, cap, C.byref(n),
                        counts.ctypes.data, C.byref(fb))
    return rc, out[: n.value].copy(), [int(x) for x in counts], bool(fb.value)


def predict(bw, B, C_, path_of_chunk, kinds=None, backlog=None):
    paths = make_paths(bw, kinds, backlog)
    poc = np.ascontiguousarray(path_of_chunk, dtype=np.uint8)
    T, g = C.c_double(), C.c_double()
    lib().orc_predict(paths, len(bw), B, C_, poc.ctypes.data, poc.size, C.byref(T), C.byref(g))
    return T.value, g.value


def direct_rate(C_, depth, B, t0):
    """Steady-state rate (bytes/s) of a direct path with `depth` outstanding DMAs (model)."""
    f = lib().orc_direct_rate
    f.restype = C.c_double
    f.argtypes = [C.c_double, C.c_uint, C.c_double, C.c_double]
    return f(C_, depth, B, t0)


def relay_rate(C_, streams, Bp, Bn, t0):
    """Steady-state rate (bytes/s) of a relay path with `streams` relay pipelines (model)."""
    f = lib().orc_relay_rate
    f.restype = C.c_double
    f.argtypes = [C.c_double, C.c_uint, C.c_double, C.c_double, C.c_double]
    return f(C_, streams, Bp, Bn, t0)


def segments_from_arrays(src_ptrs, dst_ptrs, lens):
    n = len(lens)
    arr = (Segment * max(n, 1))()
    for k in range(n):
        arr[k].src = int(src_ptrs[k])
        arr[k].dst = int(dst_ptrs[k])
        arr[k].len = int(lens[k])
    return arr, n


def move(segs, nsegs, C_, bw, path_of_chunk, S=2, base=None, exec_mode=DETERMINISTIC,
         events=None, write_count=None, fault=FAULT_NONE, kinds=None):
    """Run the mover; segs from segments_from_arrays. Returns rc."""
    paths = make_paths(bw, kinds)
    P = len(bw)
    poc = np.ascontiguousarray(path_of_chunk, dtype=np.uint8)
    b = np.zeros(P, dtype=np.uint64) if base is None else np.ascontiguousarray(base, dtype=np.uint64)
    return lib().orc_move(segs, nsegs, C_, paths, P, poc.ctypes.data, poc.size, S,
                          b.ctypes.data, exec_mode,
                          events.ctypes.data if events is not None else None,
                          write_count.ctypes.data if write_count is not None else None, fault)


def move_contiguous(dst: np.ndarray, src: np.ndarray, C_, bw, path_of_chunk, **kw):
    segs, n = segments_from_arrays([src.ctypes.data], [dst.ctypes.data], [src.size])
    return move(segs, n if src.size else 0, C_, bw, path_of_chunk, **kw)


def check_events(events, bw, path_of_chunk, S, base=None, kinds=None):
    paths = make_paths(bw, kinds)
    P = len(bw)
    poc = np.ascontiguousarray(path_of_chunk, dtype=np.uint8)
    b = np.zeros(P, dtype=np.uint64) if base is None else np.ascontiguousarray(base, dtype=np.uint64)
    return int(lib().orc_check_events(events.ctypes.data, paths, P, poc.ctypes.data, poc.size,
                                      S, b.ctypes.data))


def ring_explore(n, S, base=0, fault=FAULT_NONE):
    st, v = C.c_uint64(), C.c_uint64()
    rc = lib().orc_ring_explore(n, S, base, fault, C.byref(st), C.byref(v))
    return rc, st.value, v.value


def segments_disjoint(segs, nsegs) -> bool:
    return bool(lib().orc_segments_disjoint(segs, nsegs))


def cpu_count_used(paths_threads: int) -> int:
    return min(paths_threads, os.cpu_count() or 1)
