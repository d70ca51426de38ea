"""B200-native multipath host<->GPU copy engine (MMA, arXiv 2512.16056).

The product is the C-ABI library libmma.so (include/mma.h); `mma` is its thin binding.
Importing this package loads the library first so that its constructor raises
CUDA_DEVICE_MAX_CONNECTIONS before any CUDA context exists. A missing or stale library
makes every call raise (there is no CPU fallback); importing still works so that
`python -m paper_2512_16056_b200.build` can rebuild it.
"""
from . import mma  # noqa: F401
from .mma import (  # noqa: F401
    H2D, D2H, HOP_AUTO, HOP_CE, HOP_ZC, HOP_CE_P2P, HOP_PUSH, PATH_DIRECT, PATH_RELAY, Config, MMAError,
    calibrate, default_config, finalize, get_delivery_log, get_last_error, get_paths, get_plan,
    get_stats, host_alloc, host_array, host_free, init, make_segments, memcpy_d2h,
    memcpy_d2h_segments, memcpy_h2d, memcpy_h2d_segments, plan_chunks, reset_stats,
    set_bandwidth, set_path_modes, tune_segments, get_dynamic_counts, set_plan_mode, set_kernel_timing, kernel_times, fill_pattern,
    verify_pattern, verify_segments, shared_host_alloc, shared_host_free, ipc_export, ipc_open,
    ipc_close, copy_share_segments, copy_claim_segments, trace_begin, trace_end,
    save_calibration, load_calibration, host_alloc_for, host_page_node, get_calibration, tune_threshold,
    ledger_attach, ledger_unlink, ledger_shared_add, ledger_shared_get, device_bus_id, get_topology,
    order_by_address, tune_chunk, get_segment_order, plan_multi, memcpy_multi, host_alloc_size, copy_share_segments_ring, ledger_process_add, get_dynamic_backoffs, get_forward_log,
)

try:
    mma.lib()
except (ImportError, OSError, AttributeError):
    mma._lib = None
