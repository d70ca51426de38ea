"""Backlog ledger: a call is planned against the bytes that calls still in
flight have queued on each link. The plan with a pending call must equal the oracle's
earliest-finish plan with that backlog as input, and return to the unloaded plan once the
pending call has completed."""
import pytest

from gpu_util import configure, pinned

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]

MiB = 1 << 20


@pytest.fixture(scope="module")
def mma():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_16056_b200 as m
    yield m
    m.finalize()


def test_plan_sees_in_flight_backlog(mma, orc):
    C = MiB
    configure(mma, loopback=1, chunk=C, plan_mode=1, hop=(1, 1), debug=0)
    bw = [3, 1]
    mma.set_bandwidth(0, mma.H2D, bw)
    B = 8 * C
    rc, idle_plan, _, _ = orc.plan(bw, B, C, 0, 1)
    assert mma.get_plan(0, mma.H2D, B)[0] == idle_plan.tobytes()
    # a call held behind a sleeping kernel stays in flight
    Ba = 24 * MiB
    src = pinned(torch, Ba, seed=2)
    dst = torch.empty(Ba, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    mma.memcpy_h2d(dst, src, Ba, stream=s)        # rings and table buffers exist from here on
    s.synchronize()
    assert mma.get_plan(0, mma.H2D, B)[0] == idle_plan.tobytes()
    with torch.cuda.stream(s):
        torch.cuda._sleep(3_000_000_000)          # ~1.5 s at 1.9 GHz
        mma.memcpy_h2d(dst, src, Ba, stream=s)
    busy_path, _ = mma.get_plan(0, mma.H2D, B)
    # both paths live on GPU 0's link: each carries the pending call's Ba bytes
    rc, exp, _, _ = orc.plan(bw, B, C, 0, 1, backlog=[Ba, Ba])
    assert busy_path == exp.tobytes()
    assert busy_path != idle_plan.tobytes()
    s.synchronize()
    assert torch.equal(dst.cpu(), src[:Ba])
    assert mma.get_plan(0, mma.H2D, B)[0] == idle_plan.tobytes()


def test_ledger_off_ignores_backlog(mma, orc):
    C = MiB
    cfg = configure(mma, loopback=1, chunk=C, plan_mode=1, hop=(1, 1), debug=0)
    cfg.ledger = 0
    mma.init(cfg)
    bw = [3, 1]
    mma.set_bandwidth(0, mma.H2D, bw)
    B = 8 * C
    rc, idle_plan, _, _ = orc.plan(bw, B, C, 0, 1)
    src = pinned(torch, 24 * MiB, seed=2)
    dst = torch.empty(24 * MiB, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        torch.cuda._sleep(1_000_000_000)
        mma.memcpy_h2d(dst, src, 24 * MiB, stream=s)
    assert mma.get_plan(0, mma.H2D, B)[0] == idle_plan.tobytes()
    s.synchronize()


def test_new_ring_does_not_wait_on_user_work(mma):
    """Creating a relay ring zeroes its flags on a private setup stream: the first multipath
    call returns (is enqueued) while unrelated user work still runs on the device."""
    import time
    mma.finalize()
    configure(mma, loopback=1, chunk=MiB, plan_mode=0, hop=(1, 1), debug=0)
    mma.set_bandwidth(0, mma.H2D, [1, 1])
    B = 16 * MiB
    src = pinned(torch, B, seed=3)
    dst = torch.empty(B, dtype=torch.uint8, device="cuda")
    busy, s = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(busy):
        torch.cuda._sleep(2_000_000_000)          # ~1 s of unrelated work
    t0 = time.perf_counter()
    mma.memcpy_h2d(dst, src, B, stream=s)         # creates the ring
    enqueue_s = time.perf_counter() - t0
    s.synchronize()
    torch.cuda.synchronize()
    assert enqueue_s < 0.4, enqueue_s
    assert torch.equal(dst.cpu(), src[:B])
    assert mma.get_stats(0)["relay_bytes"] > 0


def test_shared_ledger_backlog_from_another_process(mma, orc):
    """Cross-process ledger (NEXT-4): bytes another process has queued on a link (entered
    here through mma_ledger_shared_add, as that process's engine would) become the backlog
    of this process's plan; removing them restores the idle plan."""
    import os
    name = f"gpu{os.getpid()}"
    mma.finalize()
    mma.ledger_attach(name)
    try:
        C = MiB
        configure(mma, loopback=1, chunk=C, plan_mode=1, hop=(1, 1), debug=0)
        bw = [3, 1]
        mma.set_bandwidth(0, mma.H2D, bw)
        B = 8 * C
        rc, idle_plan, _, _ = orc.plan(bw, B, C, 0, 1)
        assert mma.get_plan(0, mma.H2D, B)[0] == idle_plan.tobytes()
        bus = mma.device_bus_id(0)
        Ba = 24 * MiB
        mma.ledger_shared_add(bus, mma.H2D, Ba, 0)
        rc, exp, _, _ = orc.plan(bw, B, C, 0, 1, backlog=[Ba, Ba])    # both paths are GPU 0's link
        assert mma.get_plan(0, mma.H2D, B)[0] == exp.tobytes() != idle_plan.tobytes()
        mma.ledger_shared_add(bus, mma.H2D, -Ba, 0)
        assert mma.get_plan(0, mma.H2D, B)[0] == idle_plan.tobytes()
    finally:
        mma.finalize()
        mma.ledger_attach(None)
        mma.ledger_unlink(name)


def test_engine_calls_enter_the_shared_ledger(mma):
    """A call in flight is visible in the shared ledger with its per-link bytes (all of it on
    GPU 0's link here, the direct share as `own`) and leaves it once it has completed."""
    import os
    name = f"gpu{os.getpid()}b"
    mma.finalize()
    mma.ledger_attach(name)
    try:
        C = MiB
        configure(mma, loopback=1, chunk=C, plan_mode=1, hop=(1, 1), debug=0)
        mma.set_bandwidth(0, mma.H2D, [3, 1])
        bus = mma.device_bus_id(0)
        Ba = 24 * MiB
        src = pinned(torch, Ba, seed=5)
        dst = torch.empty(Ba, dtype=torch.uint8, device="cuda")
        s = torch.cuda.Stream()
        mma.memcpy_h2d(dst, src, Ba, stream=s)      # rings and tables exist from here on
        s.synchronize()
        mma.get_plan(0, mma.H2D, Ba)                # retires the completed call
        assert mma.ledger_shared_get(bus, mma.H2D) == (0, 0)
        with torch.cuda.stream(s):
            torch.cuda._sleep(2_000_000_000)
            mma.memcpy_h2d(dst, src, Ba, stream=s)
        got = mma.ledger_shared_get(bus, mma.H2D)
        assert got == (Ba, 18 * MiB), got          # plan 3:1 -> 18 MiB on the direct path
        s.synchronize()
        mma.get_plan(0, mma.H2D, Ba)
        assert mma.ledger_shared_get(bus, mma.H2D) == (0, 0)
        assert torch.equal(dst.cpu(), src[:Ba])
    finally:
        mma.finalize()
        mma.ledger_attach(None)
        mma.ledger_unlink(name)
