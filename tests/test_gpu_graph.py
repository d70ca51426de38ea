"""Graph capture: a multipath copy on a stream being captured (torch.cuda.graph) is recorded
as a replayable copy -- zero-copy paths, the direct copy engine and all-copy-engine relays
(on staging of their own), tables in the engine's pinned arena and graph allocations. Each replay must move the CURRENT bytes of the source,
bit-exact, in both directions and for scattered tables; a capture that cannot be served
(engine not yet initialised, arena full) records the native copy instead, still correct."""
import os

import numpy as np
import pytest

import mma_inputs

from gpu_util import configure, pinned

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]

MiB = 1 << 20


@pytest.fixture(scope="module")
def mma():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    os.environ.setdefault("MMA_SPIN_TIMEOUT_MS", "8000")
    import paper_2512_16056_b200 as m
    torch.cuda.init()
    yield m
    m.finalize()


def _two_paths(mma, dirn):
    """direct path by copy engine + one loopback path by SM zero-copy, split 1:1"""
    mma.set_path_modes(0, dirn, [mma.HOP_CE, mma.HOP_ZC])
    mma.set_bandwidth(0, dirn, [1, 1])


def test_captured_h2d_replays_current_bytes(mma):
    configure(mma, loopback=1, chunk=MiB, debug=0)
    _two_paths(mma, mma.H2D)
    B = 24 * MiB + 4096 + 16
    src = pinned(torch, B, seed=1)
    dst = torch.zeros(B, dtype=torch.uint8, device="cuda")
    mma.memcpy_h2d(dst, src, B)                       # uncaptured first: device state exists
    torch.cuda.synchronize()
    k0 = mma.get_stats(0)["kernels"]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        mma.memcpy_h2d(dst, src, B)
    assert mma.get_stats(0)["kernels"] == k0 + 1      # the zero-copy path was captured
    for seed in (11, 12, 13):
        mma_inputs.fill_pattern(src.numpy()[:B], seed)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(dst.cpu(), src[:B]), seed
    mma.memcpy_h2d(dst, src, B)                       # the engine keeps working uncaptured
    torch.cuda.synchronize()
    assert torch.equal(dst.cpu(), src[:B]) and mma.get_last_error() == 0


@pytest.mark.parametrize("order", [0, 1], ids=["table_order", "host_order"])
def test_captured_kv_offload_replays(mma, order):
    """scattered D2H (the KV offload shape), with and without host-ordered private tables"""
    configure(mma, loopback=1, chunk=MiB, debug=0, host_order=order)
    _two_paths(mma, mma.D2H)
    nseg, sb = 1024, 32 << 10
    rng = np.random.default_rng(3)
    slots = rng.permutation(2 * nseg)[:nseg]
    blocks = rng.permutation(nseg)
    cache = torch.empty(nseg * sb, dtype=torch.uint8, device="cuda")
    pool = torch.zeros(2 * nseg * sb, dtype=torch.uint8).pin_memory()
    segs, n = mma.make_segments([cache.data_ptr() + int(b) * sb for b in blocks],
                                [pool.data_ptr() + int(s) * sb for s in slots], [sb] * nseg)
    mma.memcpy_d2h_segments(segs, n, 0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        mma.memcpy_d2h_segments(segs, n, 0)
    for seed in (21, 22):
        mma.fill_pattern(cache, nseg * sb, seed, 0)
        torch.cuda.synchronize()
        pool.zero_()
        g.replay()
        torch.cuda.synchronize()
        got = pool.numpy().reshape(2 * nseg, sb)[slots]
        exp = cache.cpu().numpy().reshape(nseg, sb)[blocks]
        assert np.array_equal(got, exp), seed
        free = np.setdiff1d(np.arange(2 * nseg), slots)
        assert not pool.numpy().reshape(2 * nseg, sb)[free].any()
    assert mma.get_last_error() == 0


def test_capture_as_first_call_is_native(mma):
    """nothing may be initialised inside a capture: the first call of a fresh engine records
    the native copy, which replays correctly"""
    mma.finalize()
    B = 8 * MiB
    src = pinned(torch, B, seed=4)
    dst = torch.zeros(B, dtype=torch.uint8, device="cuda")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        mma.memcpy_h2d(dst, src, B)
    mma_inputs.fill_pattern(src.numpy()[:B], 5)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(dst.cpu(), src[:B])


def test_arena_full_captures_native(mma):
    mma.finalize()
    os.environ["MMA_GRAPH_ARENA"] = "4096"            # too small for the table below
    try:
        configure(mma, loopback=1, chunk=MiB, debug=0)
        _two_paths(mma, mma.H2D)
        nseg, sb = 512, 16 << 10
        pool = pinned(torch, nseg * sb, seed=6)
        cache = torch.zeros(nseg * sb, dtype=torch.uint8, device="cuda")
        perm = np.random.default_rng(9).permutation(nseg)
        segs, n = mma.make_segments([pool.data_ptr() + int(k) * sb for k in range(nseg)],
                                    [cache.data_ptr() + int(p) * sb for p in perm], [sb] * nseg)
        mma.memcpy_h2d_segments(segs, n, 0)
        torch.cuda.synchronize()
        k0 = mma.get_stats(0)["kernels"]
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            mma.memcpy_h2d_segments(segs, n, 0)
        assert mma.get_stats(0)["kernels"] == k0       # native: no kernel captured
        mma_inputs.fill_pattern(pool.numpy(), 7)
        cache.zero_()
        g.replay()
        torch.cuda.synchronize()
        got = cache.cpu().numpy().reshape(nseg, sb)[perm]
        assert np.array_equal(got, pool.numpy().reshape(nseg, sb))
    finally:
        del os.environ["MMA_GRAPH_ARENA"]
        mma.finalize()


@pytest.mark.parametrize("dirn", [0, 1], ids=["h2d", "d2h"])
@pytest.mark.parametrize("scattered", [False, True], ids=["contig", "segments"])
def test_captured_all_copy_engine_relay(mma, dirn, scattered):
    """an all-copy-engine relay (MMA_HOP_CE_P2P) is captured on staging of its own: replays
    move the current bytes through it (the relay's bytes counted at capture prove it took part)"""
    configure(mma, loopback=1, chunk=MiB, slots=4, debug=0)
    mma.set_path_modes(0, dirn, [mma.HOP_CE, mma.HOP_CE_P2P])
    mma.set_bandwidth(0, dirn, [1, 1])
    nseg, sb = 256, 48 << 10
    B = nseg * sb
    rng = np.random.default_rng(12)
    perm = rng.permutation(nseg) if scattered else np.arange(nseg)
    host = pinned(torch, B)
    dev = torch.zeros(B, dtype=torch.uint8, device="cuda")
    if dirn == 0:
        segs = ([host.data_ptr() + k * sb for k in range(nseg)], [dev.data_ptr() + int(p) * sb for p in perm])
    else:
        segs = ([dev.data_ptr() + int(p) * sb for p in perm], [host.data_ptr() + k * sb for k in range(nseg)])
    table, n = mma.make_segments(*segs, [sb] * nseg)

    def copy():
        if scattered:
            (mma.memcpy_h2d_segments if dirn == 0 else mma.memcpy_d2h_segments)(table, n, 0)
        elif dirn == 0:
            mma.memcpy_h2d(dev, host, B)
        else:
            mma.memcpy_d2h(host, dev, B)
    copy()
    torch.cuda.synchronize()
    r0 = mma.get_stats(0)["relay_bytes"]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        copy()
    assert mma.get_stats(0)["relay_bytes"] > r0
    for seed in (31, 32):
        if dirn == 0:
            mma_inputs.fill_pattern(host.numpy()[:B], seed)
        else:
            mma.fill_pattern(dev, B, seed, 0)
            torch.cuda.synchronize()
            host.numpy()[:] = 0
        g.replay()
        torch.cuda.synchronize()
        h = host.numpy()[:B].reshape(nseg, sb)
        d = dev.cpu().numpy().reshape(nseg, sb)
        assert np.array_equal(d[perm], h), seed
    assert mma.get_last_error() == 0


def test_replays_concurrent_with_live_ring_calls(mma):
    """a replayed graph (all-copy-engine relay on its own staging) and live calls through the
    kernel-driven ring of the same relay path, on two streams at once: both stay exact"""
    configure(mma, loopback=1, chunk=MiB, slots=2, debug=0)
    mma.set_path_modes(0, mma.H2D, [mma.HOP_CE, mma.HOP_CE_P2P])
    mma.set_bandwidth(0, mma.H2D, [1, 1])
    B = 16 * MiB + 4096
    gsrc = pinned(torch, B, seed=41)
    gdst = torch.zeros(B, dtype=torch.uint8, device="cuda")
    mma.memcpy_h2d(gdst, gsrc, B)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        mma.memcpy_h2d(gdst, gsrc, B)
    mma.set_path_modes(0, mma.H2D, [mma.HOP_CE, mma.HOP_CE])     # live calls: the kernel ring
    mma.set_bandwidth(0, mma.H2D, [1, 1])
    lsrc = pinned(torch, B, seed=42)
    ldst = torch.zeros(B, dtype=torch.uint8, device="cuda")
    s_graph, s_live = torch.cuda.Stream(), torch.cuda.Stream()
    for it in range(4):
        mma_inputs.fill_pattern(gsrc.numpy()[:B], 50 + it)
        mma_inputs.fill_pattern(lsrc.numpy()[:B], 60 + it)
        with torch.cuda.stream(s_graph):
            g.replay()
        mma.memcpy_h2d(ldst, lsrc, B, stream=s_live)
        torch.cuda.synchronize()
        assert torch.equal(gdst.cpu(), gsrc[:B]), it
        assert torch.equal(ldst.cpu(), lsrc[:B]), it
    assert mma.get_last_error() == 0


def test_live_call_while_a_capture_is_open(mma):
    """a captured call must not pull the streams live calls use into its capture.
    Between a captured mma call and the end of that capture, a live call on another stream
    runs at once (its bytes are there when its stream is synchronised, still inside the
    capture window), and the graph replays correctly afterwards."""
    configure(mma, loopback=1, chunk=MiB, debug=0)
    _two_paths(mma, mma.H2D)
    B = 12 * MiB + 4096
    gsrc, lsrc = pinned(torch, B, seed=71), pinned(torch, B, seed=72)
    gdst = torch.zeros(B, dtype=torch.uint8, device="cuda")
    ldst = torch.zeros(B, dtype=torch.uint8, device="cuda")
    mma.memcpy_h2d(gdst, gsrc, B)                     # uncaptured first: device state exists
    torch.cuda.synchronize()
    gdst.zero_()
    torch.cuda.synchronize()
    live = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, capture_error_mode="relaxed"):
        mma.memcpy_h2d(gdst, gsrc, B)                 # captured
        with torch.cuda.stream(live):                 # live, same paths, capture still open
            mma.memcpy_h2d(ldst, lsrc, B, stream=live)
            live_ok = torch.equal(ldst.cpu(), lsrc[:B])
    assert live_ok
    assert not gdst.any().item()                      # nothing ran at capture time
    mma_inputs.fill_pattern(gsrc.numpy()[:B], 73)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(gdst.cpu(), gsrc[:B])
    assert mma.get_last_error() == 0


def test_second_open_capture_records_native(mma):
    """two captures open at once: the second finds the capture lanes still capturing and
    records the native copy (no edge ties the two graphs); both replay correctly"""
    configure(mma, loopback=1, chunk=MiB, debug=0)
    _two_paths(mma, mma.H2D)
    B = 8 * MiB
    s1, s2 = pinned(torch, B, seed=81), pinned(torch, B, seed=82)
    d1 = torch.zeros(B, dtype=torch.uint8, device="cuda")
    d2 = torch.zeros(B, dtype=torch.uint8, device="cuda")
    mma.memcpy_h2d(d1, s1, B)
    torch.cuda.synchronize()
    st1, st2 = torch.cuda.Stream(), torch.cuda.Stream()
    g1, g2 = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    k0 = mma.get_stats(0)["kernels"]
    # raw capture API through torch streams: begin both, record one call into each, end both
    with torch.cuda.stream(st1):
        g1.capture_begin(capture_error_mode="relaxed")
        mma.memcpy_h2d(d1, s1, B, stream=st1)
    k1 = mma.get_stats(0)["kernels"]
    with torch.cuda.stream(st2):
        g2.capture_begin(capture_error_mode="relaxed")
        mma.memcpy_h2d(d2, s2, B, stream=st2)
    k2 = mma.get_stats(0)["kernels"]
    with torch.cuda.stream(st2):
        g2.capture_end()
    with torch.cuda.stream(st1):
        g1.capture_end()
    assert k1 == k0 + 1 and k2 == k1                  # the second call is the native copy
    for seed in (83, 84):
        mma_inputs.fill_pattern(s1.numpy()[:B], seed)
        mma_inputs.fill_pattern(s2.numpy()[:B], seed + 10)
        g1.replay()
        g2.replay()
        torch.cuda.synchronize()
        assert torch.equal(d1.cpu(), s1[:B]) and torch.equal(d2.cpu(), s2[:B]), seed
    assert mma.get_last_error() == 0


def test_two_calls_in_one_capture(mma):
    """two multipath calls recorded into ONE graph both stay multipath (the capture lanes are
    already in this capture after the first), and the graph replays both"""
    configure(mma, loopback=1, chunk=MiB, debug=0)
    _two_paths(mma, mma.H2D)
    B = 10 * MiB + 4096
    s1, s2 = pinned(torch, B, seed=91), pinned(torch, B, seed=92)
    d1 = torch.zeros(B, dtype=torch.uint8, device="cuda")
    d2 = torch.zeros(B, dtype=torch.uint8, device="cuda")
    mma.memcpy_h2d(d1, s1, B)
    torch.cuda.synchronize()
    k0 = mma.get_stats(0)["kernels"]
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        mma.memcpy_h2d(d1, s1, B)
        mma.memcpy_h2d(d2, s2, B)
    assert mma.get_stats(0)["kernels"] == k0 + 2        # both captured as multipath copies
    for seed in (93, 94):
        mma_inputs.fill_pattern(s1.numpy()[:B], seed)
        mma_inputs.fill_pattern(s2.numpy()[:B], seed + 7)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(d1.cpu(), s1[:B]) and torch.equal(d2.cpu(), s2[:B]), seed
    assert mma.get_last_error() == 0


@pytest.mark.parametrize("dirn", [0, 1], ids=["h2d", "d2h"])
@pytest.mark.parametrize("mode", ["zc", "ce_p2p"])
def test_captured_relay_on_another_gpu(mma, dirn, mode):
    """the relay path on engine GPU 1 (a peer on a multi-GPU box, else the engine's virtual GPU
    on the same device): the capture joins the relay GPU's capture lanes, and
    every replay moves the current bytes through it"""
    virtual = torch.cuda.device_count() < 2
    if virtual:
        mma.finalize()
        os.environ["MMA_VGPUS"] = "2"
    try:
        configure(mma, loopback=0, chunk=MiB, slots=4, debug=0, paths=[0, 1])
        assert [p["gpu"] for p in mma.get_paths(0, dirn)] == [0, 1]
        mma.set_path_modes(0, dirn, [mma.HOP_CE, mma.HOP_ZC if mode == "zc" else mma.HOP_CE_P2P])
        mma.set_bandwidth(0, dirn, [1, 1])
        B = 20 * MiB + 4096 + 48
        host = pinned(torch, B, seed=5)
        dev = torch.zeros(B, dtype=torch.uint8, device="cuda")

        def copy():
            if dirn == 0:
                mma.memcpy_h2d(dev, host, B)
            else:
                mma.memcpy_d2h(host, dev, B)
        copy()
        torch.cuda.synchronize()
        r0 = mma.get_stats(0)["relay_bytes"]
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            copy()
        assert mma.get_stats(0)["relay_bytes"] > r0            # the relay took part in the capture
        for seed in (71, 72, 73):
            if dirn == 0:
                mma_inputs.fill_pattern(host.numpy()[:B], seed)
            else:
                mma.fill_pattern(dev, B, seed, 0)
                torch.cuda.synchronize()
                host.numpy()[:] = 0
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(dev.cpu(), host[:B]), seed
        del g
        assert mma.get_last_error() == 0
    finally:
        if virtual:
            mma.finalize()
            os.environ.pop("MMA_VGPUS", None)
