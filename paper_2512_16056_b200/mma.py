"""Python binding of libmma.so (include/mma.h): argument marshalling only.

Every byte of a copy is moved by the library's CUDA path (copy engines + the sm_100a
kernels in csrc/kernels); nothing here computes. torch is used only to read tensor data
pointers and CUDA stream handles. If libmma.so is missing the import fails loudly: there
is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libmma.so"

H2D, D2H = 0, 1
HOP_AUTO, HOP_CE, HOP_ZC, HOP_CE_P2P, HOP_PUSH = 0, 1, 2, 3, 4
PATH_DIRECT, PATH_RELAY = 0, 1
MAX_PATHS = 16
MAX_GPUS = 16
ERR_RELAY_TIMEOUT = 2001

SYMBOLS = [
    "mma_default_config", "mma_init", "mma_finalize", "mma_memcpy_h2d", "mma_memcpy_d2h",
    "mma_memcpy_h2d_segments", "mma_memcpy_d2h_segments", "mma_get_paths", "mma_set_bandwidth",
    "mma_set_path_modes", "mma_calibrate", "mma_get_plan", "mma_plan_chunks",
    "mma_get_delivery_log", "mma_get_segment_order", "mma_plan_multi", "mma_memcpy_multi",
    "mma_host_alloc_size", "mma_copy_share_segments_ring", "mma_ledger_process_add",
    "mma_get_dynamic_backoffs", "mma_get_forward_log", "mma_host_alloc", "mma_host_free", "mma_get_stats",
    "mma_reset_stats", "mma_get_last_error", "mma_error_string", "mma_fill_pattern",
    "mma_verify_pattern", "mma_verify_segments", "mma_set_kernel_timing", "mma_kernel_times",
    "mma_tune_segments", "mma_get_segment_tuning", "mma_get_dynamic_counts", "mma_set_plan_mode",
    "mma_shared_host_alloc", "mma_shared_host_free", "mma_ipc_export", "mma_ipc_open", "mma_ipc_close",
    "mma_copy_share_segments", "mma_copy_claim_segments", "mma_trace_begin", "mma_trace_end",
    "mma_save_calibration", "mma_load_calibration", "mma_host_alloc_for", "mma_host_page_node",
    "mma_get_calibration", "mma_tune_threshold", "mma_ledger_attach", "mma_ledger_unlink",
    "mma_ledger_shared_add", "mma_ledger_shared_get", "mma_device_bus_id", "mma_get_topology", "mma_order_by_address", "mma_tune_chunk",
]


class Config(C.Structure):
    _fields_ = [
        ("chunk_bytes", C.c_size_t * 2),
        ("ring_slots", C.c_uint),
        ("fallback_bytes", C.c_size_t * 2),
        ("path_gpus", C.c_int * MAX_PATHS),
        ("npaths", C.c_int),
        ("loopback_relays", C.c_int),
        ("plan_mode", C.c_int),
        ("hop_mode", C.c_int * 2),
        ("relay_ctas", C.c_int),
        ("numa_mode", C.c_int),
        ("debug_log", C.c_int),
        ("ledger", C.c_int),
        ("claim_bytes", C.c_size_t),
        ("zc_ctas", C.c_int),
        ("calib_rounds", C.c_int),
        ("host_order", C.c_int),
        ("numa_plan", C.c_int),
        ("background_policy", C.c_int),
        ("yield_pct", C.c_uint),
        ("relay_prefer", C.c_int),
    ]


class Topology(C.Structure):
    _fields_ = [
        ("ngpu", C.c_int),
        ("p2p", (C.c_int * MAX_GPUS) * MAX_GPUS),
        ("numa_node", C.c_int * MAX_GPUS),
        ("copy_engines", C.c_int * MAX_GPUS),
        ("sms", C.c_int * MAX_GPUS),
        ("bus_id", (C.c_char * 16) * MAX_GPUS),
        ("host_numa_nodes", C.c_int),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("calls", C.c_uint64), ("fallbacks", C.c_uint64), ("bytes", C.c_uint64),
        ("path_bytes", (C.c_uint64 * MAX_PATHS) * 2), ("path_chunks", (C.c_uint64 * MAX_PATHS) * 2),
        ("relay_bytes", C.c_uint64), ("kernels", C.c_uint64), ("issue_us", C.c_double),
        ("wait_us", C.c_double), ("dynamic_calls", C.c_uint64),
        ("numa_known_bytes", C.c_uint64 * 2), ("numa_local_bytes", C.c_uint64 * 2),
        ("single_path_calls", C.c_uint64), ("validate_us", C.c_double), ("ptr_queries", C.c_uint64),
    ]


class Segment(C.Structure):
    _fields_ = [("src", C.c_void_p), ("dst", C.c_void_p), ("bytes", C.c_size_t)]


class Transfer(C.Structure):
    _fields_ = [("dir", C.c_int), ("device", C.c_int), ("segs", C.POINTER(Segment)), ("nsegs", C.c_size_t),
                ("stream", C.c_void_p)]


class MMAError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: {lib().mma_error_string(code).decode()} ({code})")
        self.code = code


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: build it with "
                              "`python -m paper_2512_16056_b200.build` (no CPU fallback exists)")
        L = C.CDLL(str(LIB_PATH))
        vp, sz, u64p = C.c_void_p, C.c_size_t, C.POINTER(C.c_uint64)
        L.mma_default_config.argtypes = [C.POINTER(Config)]
        L.mma_init.argtypes = [C.POINTER(Config)]
        L.mma_memcpy_h2d.argtypes = [vp, vp, sz, vp]
        L.mma_memcpy_d2h.argtypes = [vp, vp, sz, vp]
        L.mma_memcpy_h2d_segments.argtypes = [C.POINTER(Segment), sz, C.c_int, vp]
        L.mma_memcpy_d2h_segments.argtypes = [C.POINTER(Segment), sz, C.c_int, vp]
        L.mma_get_paths.argtypes = [C.c_int, C.c_int, vp, vp, vp, vp, C.c_int, C.POINTER(C.c_int)]
        L.mma_set_bandwidth.argtypes = [C.c_int, C.c_int, vp, C.c_int]
        L.mma_set_path_modes.argtypes = [C.c_int, C.c_int, vp, C.c_int]
        L.mma_calibrate.argtypes = [C.c_int, C.c_int, sz]
        L.mma_get_plan.argtypes = [C.c_int, C.c_int, sz, vp, sz, C.POINTER(sz), C.POINTER(C.c_int)]
        L.mma_plan_chunks.argtypes = [vp, vp, vp, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64,
                                      C.c_int, vp, sz, C.POINTER(sz), C.POINTER(C.c_int)]
        L.mma_get_delivery_log.argtypes = [C.c_int, vp, sz, C.POINTER(sz)]
        L.mma_get_segment_order.argtypes = [C.c_int, vp, sz, C.POINTER(sz)]
        L.mma_memcpy_multi.argtypes = [C.POINTER(Transfer), sz]
        L.mma_host_alloc_size.argtypes = [vp, C.POINTER(sz)]
        L.mma_get_dynamic_backoffs.argtypes = [C.c_int, C.POINTER(C.c_uint64)]
        L.mma_get_forward_log.argtypes = [C.c_int, vp, vp, sz, C.POINTER(sz)]
        L.mma_copy_share_segments_ring.argtypes = [C.POINTER(Segment), sz, sz, vp, sz, C.c_int, C.c_int, C.c_uint, vp]
        L.mma_plan_multi.argtypes = [C.c_int, vp, vp, C.c_int, vp, vp, C.c_uint64, C.c_int, C.c_int, vp]
        L.mma_host_alloc.argtypes = [C.POINTER(vp), sz, C.c_uint]
        L.mma_host_free.argtypes = [vp]
        L.mma_get_stats.argtypes = [C.c_int, C.POINTER(Stats)]
        L.mma_reset_stats.argtypes = [C.c_int]
        L.mma_error_string.restype = C.c_char_p
        L.mma_error_string.argtypes = [C.c_int]
        L.mma_fill_pattern.argtypes = [vp, sz, C.c_uint64, C.c_uint64, vp]
        L.mma_verify_pattern.argtypes = [vp, sz, C.c_uint64, C.c_uint64, vp, vp]
        L.mma_verify_segments.argtypes = [vp, vp, vp, sz, C.c_uint64, vp, vp]
        L.mma_set_kernel_timing.argtypes = [C.c_int]
        L.mma_tune_segments.argtypes = [C.POINTER(Segment), sz, C.c_int, C.c_int, vp, C.c_int]
        L.mma_kernel_times.argtypes = [vp, vp, sz, C.POINTER(sz)]
        L.mma_get_segment_tuning.argtypes = [C.c_int, C.c_int, vp, vp, C.c_int, C.POINTER(C.c_int)]
        L.mma_ledger_attach.argtypes = [C.c_char_p]
        L.mma_device_bus_id.argtypes = [C.c_int, C.c_char_p, C.c_int]
        L.mma_get_topology.argtypes = [C.POINTER(Topology)]
        L.mma_order_by_address.argtypes = [vp, sz, vp]
        L.mma_ledger_unlink.argtypes = [C.c_char_p]
        L.mma_ledger_shared_add.argtypes = [C.c_char_p, C.c_int, C.c_int64, C.c_int64]
        L.mma_ledger_process_add.argtypes = [C.c_char_p, C.c_int, C.c_int64, C.c_int64]
        L.mma_ledger_shared_get.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.mma_tune_chunk.argtypes = [C.c_int, C.c_int, sz, C.POINTER(sz)]
        L.mma_tune_threshold.argtypes = [C.c_int, C.c_int, sz, C.POINTER(sz), C.POINTER(C.c_int)]
        L.mma_get_calibration.argtypes = [C.c_int, C.c_int, C.c_int, vp, vp, C.c_int, C.POINTER(C.c_int)]
        L.mma_get_dynamic_counts.argtypes = [C.c_int, vp, C.c_int, C.POINTER(C.c_int)]
        L.mma_set_plan_mode.argtypes = [C.c_int]
        L.mma_trace_begin.argtypes = [sz]
        L.mma_save_calibration.argtypes = [C.c_char_p]
        L.mma_host_alloc_for.argtypes = [C.POINTER(vp), sz, C.c_int, C.c_int]
        L.mma_host_page_node.argtypes = [vp]
        L.mma_load_calibration.argtypes = [C.c_char_p, C.POINTER(C.c_int)]
        L.mma_trace_end.argtypes = [C.c_char_p, C.POINTER(sz)]
        L.mma_shared_host_alloc.argtypes = [C.c_char_p, sz, C.c_int, C.POINTER(vp)]
        L.mma_shared_host_free.argtypes = [vp, C.c_char_p]
        L.mma_ipc_export.argtypes = [vp, vp, C.POINTER(C.c_uint64)]
        L.mma_ipc_open.argtypes = [vp, C.c_uint64, C.c_int, C.POINTER(vp)]
        L.mma_ipc_close.argtypes = [vp]
        L.mma_copy_share_segments.argtypes = [C.POINTER(Segment), sz, sz, vp, sz, C.c_int, C.c_int, vp]
        L.mma_copy_claim_segments.argtypes = [C.POINTER(Segment), sz, sz, vp, vp, C.c_int, C.c_int, vp]
        _lib = L
    return _lib


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise MMAError(rc, what)


def _ptr(x) -> int:
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    if hasattr(x, "ctypes"):
        return int(x.ctypes.data)
    raise TypeError(f"cannot take a pointer of {type(x)}")


def _nbytes(x) -> int:
    if hasattr(x, "untyped_storage") and hasattr(x, "element_size"):
        return x.numel() * x.element_size()
    if hasattr(x, "nbytes"):
        return int(x.nbytes)
    raise TypeError("pass nbytes explicitly")


def _stream(stream, device=None) -> int:
    if stream is None:
        import torch
        return int(torch.cuda.current_stream(device).cuda_stream)
    if isinstance(stream, int):
        return stream
    return int(stream.cuda_stream)


def default_config() -> Config:
    c = Config()
    _check(lib().mma_default_config(C.byref(c)), "mma_default_config")
    return c


def init(cfg: Config | None = None) -> None:
    _check(lib().mma_init(C.byref(cfg) if cfg is not None else None), "mma_init")


def finalize() -> None:
    _check(lib().mma_finalize(), "mma_finalize")


def _dev_of(t):
    return t.device if hasattr(t, "device") and getattr(t.device, "type", "") == "cuda" else None


def memcpy_h2d(dst, src, nbytes: int | None = None, stream=None) -> None:
    """dst: CUDA tensor or device pointer; src: pinned CPU tensor / ndarray or pointer."""
    n = _nbytes(src) if nbytes is None else int(nbytes)
    _check(lib().mma_memcpy_h2d(_ptr(dst), _ptr(src), n, _stream(stream, _dev_of(dst))), "mma_memcpy_h2d")


def memcpy_d2h(dst, src, nbytes: int | None = None, stream=None) -> None:
    n = _nbytes(src) if nbytes is None else int(nbytes)
    _check(lib().mma_memcpy_d2h(_ptr(dst), _ptr(src), n, _stream(stream, _dev_of(src))), "mma_memcpy_d2h")


def make_segments(src_ptrs, dst_ptrs, lens):
    """Segment table from three integer sequences / numpy arrays."""
    import numpy as np
    n = len(lens)
    arr = (Segment * max(n, 1))()
    view = np.frombuffer(arr, dtype=np.uint64, count=3 * max(n, 1)).reshape(-1, 3)
    if n:
        view[:n, 0] = np.asarray(src_ptrs, dtype=np.uint64)
        view[:n, 1] = np.asarray(dst_ptrs, dtype=np.uint64)
        view[:n, 2] = np.asarray(lens, dtype=np.uint64)
    return arr, n


def memcpy_h2d_segments(segs, nsegs: int, dst_device: int, stream=None) -> None:
    _check(lib().mma_memcpy_h2d_segments(segs, nsegs, dst_device, _stream(stream, dst_device)),
           "mma_memcpy_h2d_segments")


def memcpy_d2h_segments(segs, nsegs: int, src_device: int, stream=None) -> None:
    _check(lib().mma_memcpy_d2h_segments(segs, nsegs, src_device, _stream(stream, src_device)),
           "mma_memcpy_d2h_segments")


def memcpy_multi(transfers) -> None:
    """Concurrent transfers under one joint plan (mma_memcpy_multi). `transfers`: sequence of
    (direction, device, (segs, nsegs) from make_segments, stream or None)."""
    arr = (Transfer * max(1, len(transfers)))()
    keep = []
    for i, (d, dev, (segs, n), stream) in enumerate(transfers):
        keep.append(segs)
        arr[i].dir, arr[i].device = d, dev
        arr[i].segs = C.cast(segs, C.POINTER(Segment))
        arr[i].nsegs = n
        arr[i].stream = _stream(stream, dev)
    _check(lib().mma_memcpy_multi(arr, len(transfers)), "mma_memcpy_multi")


def get_paths(device: int, direction: int):
    gpus = (C.c_int * MAX_PATHS)()
    kinds = (C.c_int * MAX_PATHS)()
    mbps = (C.c_uint32 * MAX_PATHS)()
    modes = (C.c_int * MAX_PATHS)()
    n = C.c_int()
    _check(lib().mma_get_paths(device, direction, gpus, kinds, mbps, modes, MAX_PATHS, C.byref(n)),
           "mma_get_paths")
    smbps = (C.c_uint32 * MAX_PATHS)()
    smodes = (C.c_int * MAX_PATHS)()
    _check(lib().mma_get_segment_tuning(device, direction, smbps, smodes, MAX_PATHS, C.byref(n)),
           "mma_get_segment_tuning")
    return [dict(gpu=gpus[i], kind=kinds[i], mbps=mbps[i], mode=modes[i], seg_mbps=smbps[i],
                 seg_mode=smodes[i]) for i in range(n.value)]


def set_bandwidth(device: int, direction: int, mbps) -> None:
    arr = (C.c_uint32 * len(mbps))(*[int(x) for x in mbps])
    _check(lib().mma_set_bandwidth(device, direction, arr, len(mbps)), "mma_set_bandwidth")


def set_path_modes(device: int, direction: int, modes) -> None:
    arr = (C.c_int * len(modes))(*[int(x) for x in modes])
    _check(lib().mma_set_path_modes(device, direction, arr, len(modes)), "mma_set_path_modes")


def calibrate(device: int, direction: int, nbytes: int = 256 << 20) -> None:
    _check(lib().mma_calibrate(device, direction, nbytes), "mma_calibrate")


def tune_segments(segs, nsegs: int, device: int, direction: int, stream=None, reps: int = 2) -> None:
    """Measure CE vs SM zero-copy per path on this scattered transfer (writes the dsts)."""
    _check(lib().mma_tune_segments(segs, nsegs, device, direction, _stream(stream, device), reps),
           "mma_tune_segments")


def tune_chunk(device: int, direction: int, nbytes: int = 512 << 20) -> int:
    """Pick the chunk size by measurement (returns the size now in effect)."""
    c = C.c_size_t()
    _check(lib().mma_tune_chunk(device, direction, nbytes, C.byref(c)), "mma_tune_chunk")
    return int(c.value)


def tune_threshold(device: int, direction: int, max_bytes: int = 256 << 20):
    """Measure the native/multipath break-even and set it as the fallback threshold.
    Returns (threshold in effect, found): found is False when multipath did not win even at
    max_bytes (threshold unchanged)."""
    thr = C.c_size_t()
    found = C.c_int()
    _check(lib().mma_tune_threshold(device, direction, max_bytes, C.byref(thr), C.byref(found)),
           "mma_tune_threshold")
    return int(thr.value), bool(found.value)


def ledger_attach(name: str | None) -> None:
    """Attach this process's engine to the cross-process ledger `name` (None detaches)."""
    _check(lib().mma_ledger_attach(name.encode() if name else None), "mma_ledger_attach")


def order_by_address(addr):
    """The engine's host-address issue order (R22): stable ascending permutation of addr."""
    import numpy as np
    a = np.ascontiguousarray(addr, dtype=np.uint64)
    perm = np.empty(a.size, dtype=np.uint32)
    _check(lib().mma_order_by_address(a.ctypes.data, a.size, perm.ctypes.data), "mma_order_by_address")
    return perm


def get_topology() -> dict:
    """P2P matrix, NUMA node, copy engines, SMs and PCI bus id per GPU (SURVEY a0 probe)."""
    t = Topology()
    _check(lib().mma_get_topology(C.byref(t)), "mma_get_topology")
    n = t.ngpu
    return {"ngpu": n, "p2p": [[int(t.p2p[a][b]) for b in range(n)] for a in range(n)],
            "numa_node": [int(t.numa_node[a]) for a in range(n)],
            "copy_engines": [int(t.copy_engines[a]) for a in range(n)],
            "sms": [int(t.sms[a]) for a in range(n)],
            "bus_id": [t.bus_id[a].value.decode() for a in range(n)],
            "host_numa_nodes": int(t.host_numa_nodes)}


def device_bus_id(device: int) -> str:
    buf = C.create_string_buffer(64)
    _check(lib().mma_device_bus_id(device, buf, 64), "mma_device_bus_id")
    return buf.value.decode()


def ledger_unlink(name: str) -> None:
    _check(lib().mma_ledger_unlink(name.encode()), "mma_ledger_unlink")


def ledger_shared_add(bus_id: str, direction: int, nbytes: int, own: int = 0) -> None:
    _check(lib().mma_ledger_shared_add(bus_id.encode(), direction, nbytes, own), "mma_ledger_shared_add")


def ledger_process_add(bus_id: str, direction: int, nbytes: int, own: int = 0) -> None:
    _check(lib().mma_ledger_process_add(bus_id.encode(), direction, nbytes, own), "mma_ledger_process_add")


def ledger_shared_get(bus_id: str, direction: int):
    """(bytes, own) queued on the link of the GPU with this PCI bus id, all processes."""
    b, o = C.c_uint64(), C.c_uint64()
    _check(lib().mma_ledger_shared_get(bus_id.encode(), direction, C.byref(b), C.byref(o)),
           "mma_ledger_shared_get")
    return int(b.value), int(o.value)


def get_calibration(device: int, direction: int, scattered: bool = False):
    """Per path: {"solo": MB/s alone, "conc": MB/s with every path active (0 = not measured)}."""
    solo = (C.c_uint32 * MAX_PATHS)()
    conc = (C.c_uint32 * MAX_PATHS)()
    n = C.c_int()
    _check(lib().mma_get_calibration(device, direction, int(scattered), solo, conc, MAX_PATHS, C.byref(n)),
           "mma_get_calibration")
    return [{"solo": int(solo[i]), "conc": int(conc[i])} for i in range(n.value)]


def get_plan(device: int, direction: int, nbytes: int):
    """Returns (path_of_chunk bytes, fallback bool)."""
    n = C.c_size_t()
    fb = C.c_int()
    _check(lib().mma_get_plan(device, direction, nbytes, None, 0, C.byref(n), C.byref(fb)), "mma_get_plan")
    buf = (C.c_uint8 * max(n.value, 1))()
    _check(lib().mma_get_plan(device, direction, nbytes, buf, n.value, C.byref(n), C.byref(fb)), "mma_get_plan")
    return bytes(buf[: n.value]), bool(fb.value)


def plan_chunks(mbps, kinds, nbytes: int, chunk: int, thr: int = 0, mode: int = 0, backlog=None):
    """Host-only planner (no GPU): returns (rc, path_of_chunk bytes, fallback)."""
    P = len(mbps)
    m = (C.c_uint32 * P)(*[int(x) for x in mbps])
    k = (C.c_int * P)(*[int(x) for x in kinds])
    b = (C.c_uint64 * P)(*[int(x) for x in backlog]) if backlog is not None else None
    n = C.c_size_t()
    fb = C.c_int()
    rc = lib().mma_plan_chunks(m, k, b, P, nbytes, chunk, thr, mode, None, 0, C.byref(n), C.byref(fb))
    if rc:
        return rc, b"", False
    buf = (C.c_uint8 * max(n.value, 1))()
    rc = lib().mma_plan_chunks(m, k, b, P, nbytes, chunk, thr, mode, buf, n.value, C.byref(n), C.byref(fb))
    return rc, bytes(buf[: n.value]), bool(fb.value)


def get_delivery_log(device: int):
    n = C.c_size_t()
    _check(lib().mma_get_delivery_log(device, None, 0, C.byref(n)), "mma_get_delivery_log")
    buf = (C.c_uint8 * max(n.value, 1))()
    _check(lib().mma_get_delivery_log(device, buf, n.value, C.byref(n)), "mma_get_delivery_log")
    return bytes(buf[: n.value])


def plan_multi(link_mbps, carry, targets, nchunks, chunk: int, mode: int = 0, prefer: int = -1):
    """The joint planner alone (mma_plan_multi): per transfer, the link id of each chunk."""
    import numpy as np
    L = len(link_mbps)
    bw = np.ascontiguousarray(link_mbps, dtype=np.uint32)
    ok = np.ascontiguousarray(carry, dtype=np.uint8).reshape(L, L)
    tg = np.ascontiguousarray(targets, dtype=np.int32)
    nc = np.ascontiguousarray(nchunks, dtype=np.uint64)
    out = np.full(max(1, int(nc.sum())), -1, dtype=np.int32)
    rc = lib().mma_plan_multi(L, bw.ctypes.data, ok.ctypes.data, len(tg), tg.ctypes.data, nc.ctypes.data, chunk,
                              mode, prefer, out.ctypes.data)
    offs = np.concatenate([[0], np.cumsum(nc)]).astype(np.int64)
    return rc, [out[offs[t]:offs[t + 1]].copy() for t in range(len(tg))]


def get_forward_log(device: int):
    """Debug: (observed, expected) flag values per chunk of the last call (mma_get_forward_log)."""
    import numpy as np
    n = C.c_size_t()
    _check(lib().mma_get_forward_log(device, None, None, 0, C.byref(n)), "mma_get_forward_log")
    obs = np.zeros(max(1, n.value), dtype=np.uint64)
    exp = np.zeros(max(1, n.value), dtype=np.uint64)
    _check(lib().mma_get_forward_log(device, obs.ctypes.data, exp.ctypes.data, n.value, C.byref(n)),
           "mma_get_forward_log")
    return obs[: n.value], exp[: n.value]


def get_segment_order(device: int):
    """Debug: table index of each segment of the last scattered call's virtual stream."""
    import numpy as np
    n = C.c_size_t()
    _check(lib().mma_get_segment_order(device, None, 0, C.byref(n)), "mma_get_segment_order")
    out = np.zeros(max(1, n.value), dtype=np.uint32)
    _check(lib().mma_get_segment_order(device, out.ctypes.data, n.value, C.byref(n)),
           "mma_get_segment_order")
    return out[: n.value]


def host_alloc(nbytes: int) -> int:
    p = C.c_void_p()
    _check(lib().mma_host_alloc(C.byref(p), nbytes, 0), "mma_host_alloc")
    return int(p.value or 0)


def host_free(ptr: int) -> None:
    _check(lib().mma_host_free(ptr), "mma_host_free")


def host_array(ptr: int, nbytes: int):
    """A numpy uint8 view of library-owned pinned memory (no copy)."""
    import numpy as np
    return np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(ptr))


def get_stats(device: int) -> dict:
    s = Stats()
    _check(lib().mma_get_stats(device, C.byref(s)), "mma_get_stats")
    return dict(calls=s.calls, fallbacks=s.fallbacks, bytes=s.bytes,
                path_bytes=[list(x) for x in s.path_bytes], path_chunks=[list(x) for x in s.path_chunks],
                relay_bytes=s.relay_bytes, kernels=s.kernels, issue_us=s.issue_us,
                wait_us=s.wait_us, dynamic_calls=s.dynamic_calls,
                numa_known_bytes=list(s.numa_known_bytes), numa_local_bytes=list(s.numa_local_bytes),
                single_path_calls=s.single_path_calls, validate_us=s.validate_us, ptr_queries=s.ptr_queries)


def set_plan_mode(mode: int) -> None:
    """0 contiguous, 1 interleaved, 2 GPU-driven dynamic pull."""
    _check(lib().mma_set_plan_mode(mode), "mma_set_plan_mode")


def get_dynamic_counts(device: int):
    """Chunks each path took in the last dynamic-pull call (synchronises)."""
    buf = (C.c_uint64 * MAX_PATHS)()
    n = C.c_int()
    _check(lib().mma_get_dynamic_counts(device, buf, MAX_PATHS, C.byref(n)), "mma_get_dynamic_counts")
    return [int(buf[i]) for i in range(n.value)]


def get_dynamic_backoffs(device: int) -> int:
    """Waits yielding CTAs took in the last dynamic-pull call (background_policy = 1)."""
    n = C.c_uint64()
    _check(lib().mma_get_dynamic_backoffs(device, C.byref(n)), "mma_get_dynamic_backoffs")
    return int(n.value)


def reset_stats(device: int) -> None:
    _check(lib().mma_reset_stats(device), "mma_reset_stats")


def get_last_error() -> int:
    return int(lib().mma_get_last_error())


def fill_pattern(dst, nbytes: int, seed: int, offset: int = 0, stream=None) -> None:
    _check(lib().mma_fill_pattern(_ptr(dst), nbytes, seed, offset, _stream(stream, _dev_of(dst))),
           "mma_fill_pattern")


def verify_pattern(src, nbytes: int, seed: int, offset: int, counter, stream=None) -> None:
    """Adds the number of mismatching bytes to `counter` (a CUDA uint64/int64 tensor)."""
    _check(lib().mma_verify_pattern(_ptr(src), nbytes, seed, offset, _ptr(counter),
                                    _stream(stream, _dev_of(src))), "mma_verify_pattern")


def verify_segments(dst_ptrs, offsets, lens, seed: int, counter, stream=None) -> None:
    import numpy as np
    d = np.ascontiguousarray(dst_ptrs, dtype=np.uint64)
    o = np.ascontiguousarray(offsets, dtype=np.uint64)
    n = np.ascontiguousarray(lens, dtype=np.uint64)
    _check(lib().mma_verify_segments(d.ctypes.data, o.ctypes.data, n.ctypes.data, d.size, seed,
                                     _ptr(counter), _stream(stream, _dev_of(counter))),
           "mma_verify_segments")


def set_kernel_timing(on: bool) -> None:
    _check(lib().mma_set_kernel_timing(1 if on else 0), "mma_set_kernel_timing")


def kernel_times():
    """[(ms, kind)] of the kernel launches recorded since the last call (kind 0 zero-copy,
    1 relay pull, 2 relay pack, 3 dynamic-pull zero-copy, 4 cp.async.bulk zero-copy);
    synchronises on them."""
    n = C.c_size_t()
    cap = 1 << 16
    ms = (C.c_float * cap)()
    kinds = (C.c_int * cap)()
    _check(lib().mma_kernel_times(ms, kinds, cap, C.byref(n)), "mma_kernel_times")
    out = []
    for i in range(min(n.value, cap)):
        t = kinds[i]
        out.append(dict(ms=ms[i], kind=t & 15, dir=(t >> 4) & 15, path=(t >> 8) & 255, dev=t >> 16))
    return out


# ---- multi-process mode (one process per GPU) -------------------------------

def shared_host_alloc(name: str, nbytes: int, create: bool) -> int:
    p = C.c_void_p()
    _check(lib().mma_shared_host_alloc(name.encode(), nbytes, 1 if create else 0, C.byref(p)),
           "mma_shared_host_alloc")
    return int(p.value)


def shared_host_free(ptr: int, unlink_name: str | None = None) -> None:
    _check(lib().mma_shared_host_free(ptr, unlink_name.encode() if unlink_name else None),
           "mma_shared_host_free")


def ipc_export(dev_ptr) -> tuple[bytes, int]:
    h = (C.c_uint8 * 64)()
    off = C.c_uint64()
    _check(lib().mma_ipc_export(_ptr(dev_ptr), h, C.byref(off)), "mma_ipc_export")
    return bytes(h), off.value


def ipc_open(handle: bytes, offset: int, device: int) -> int:
    h = (C.c_uint8 * 64).from_buffer_copy(handle)
    p = C.c_void_p()
    _check(lib().mma_ipc_open(h, offset, device, C.byref(p)), "mma_ipc_open")
    return int(p.value)


def ipc_close(dev_ptr: int) -> None:
    _check(lib().mma_ipc_close(dev_ptr), "mma_ipc_close")


def copy_share_segments(segs, nsegs: int, chunk_bytes: int, path_of_chunk: bytes, path: int,
                        device: int, stream=None) -> None:
    buf = (C.c_uint8 * max(len(path_of_chunk), 1)).from_buffer_copy(path_of_chunk or b"\0")
    _check(lib().mma_copy_share_segments(segs, nsegs, chunk_bytes, buf, len(path_of_chunk), path, device,
                                         _stream(stream, device)), "mma_copy_share_segments")


def copy_share_segments_ring(segs, nsegs: int, chunk_bytes: int, path_of_chunk: bytes, path: int,
                             device: int, slots: int = 4, stream=None) -> None:
    """This process's share moved through its own copy-engine relay ring (NEXT-4)."""
    buf = (C.c_uint8 * max(len(path_of_chunk), 1)).from_buffer_copy(path_of_chunk or b"\0")
    _check(lib().mma_copy_share_segments_ring(segs, nsegs, chunk_bytes, buf, len(path_of_chunk), path, device,
                                              slots, _stream(stream, device)), "mma_copy_share_segments_ring")


def copy_claim_segments(segs, nsegs: int, claim_bytes: int, cursor_ptr: int, counts_ptr: int,
                        path: int, device: int, stream=None) -> None:
    _check(lib().mma_copy_claim_segments(segs, nsegs, claim_bytes, cursor_ptr, counts_ptr, path, device,
                                         _stream(stream, device)), "mma_copy_claim_segments")


def trace_begin(max_spans: int = 0) -> None:
    _check(lib().mma_trace_begin(max_spans), "mma_trace_begin")


def trace_end(json_path: str | None) -> int:
    n = C.c_size_t()
    _check(lib().mma_trace_end(json_path.encode() if json_path else None, C.byref(n)), "mma_trace_end")
    return n.value


def save_calibration(path: str) -> None:
    _check(lib().mma_save_calibration(path.encode()), "mma_save_calibration")


def load_calibration(path: str) -> int:
    n = C.c_int()
    _check(lib().mma_load_calibration(path.encode(), C.byref(n)), "mma_load_calibration")
    return n.value


def host_alloc_for(nbytes: int, device: int, direction: int) -> int:
    """Pinned buffer whose per-path ranges live on each path GPU's NUMA node."""
    p = C.c_void_p()
    _check(lib().mma_host_alloc_for(C.byref(p), nbytes, device, direction), "mma_host_alloc_for")
    return int(p.value or 0)


def host_alloc_size(ptr: int):
    """Mapped length of an mma_host_alloc buffer based at ptr, or None if it is not one."""
    n = C.c_size_t()
    return int(n.value) if lib().mma_host_alloc_size(ptr, C.byref(n)) == 0 else None


def host_page_node(ptr: int) -> int:
    return int(lib().mma_host_page_node(ptr))
