"""GPU-driven dynamic pull (the paper's pull scheduler, §3.4.2,
run by the path kernels). The assignment is observed, not planned, so parity is: the
destination bytes equal the oracle moving the same transfer with the OBSERVED assignment
(the delivery log), every chunk was taken by exactly one valid path, and the per-path
counts the GPU reports match the log."""
import numpy as np
import pytest

import mma_inputs
from mma_inputs import workloads as W

from gpu_util import G, configure, guarded_device, guarded_host, pinned

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


def _check_log(mma, n, P):
    log = np.frombuffer(mma.get_delivery_log(0), dtype=np.uint8)
    assert log.size == n and (log < P).all()          # every chunk taken by a valid path
    counts = mma.get_dynamic_counts(0)
    assert len(counts) == P and sum(counts) == n
    assert counts == [int((log == p).sum()) for p in range(P)]
    return log


@pytest.mark.parametrize("B,C,lb", [(64 * MiB, MiB, 2), (13 * MiB + 77, 256 << 10, 1), (MiB + 3, MiB, 3)])
def test_dynamic_contiguous_h2d(mma, orc, B, C, lb):
    configure(mma, loopback=lb, chunk=C, plan_mode=2, hop=(2, 2))
    src = pinned(torch, B, seed=61)
    dst = guarded_device(torch, B)
    mma.reset_stats(0)
    mma.memcpy_h2d(dst[G:G + B], src, B)
    torch.cuda.synchronize()
    assert mma.get_last_error() == 0 and mma.get_stats(0)["dynamic_calls"] == 1
    n = (B + C - 1) // C
    log = _check_log(mma, n, 1 + lb)
    exp = guarded_host(B)
    assert orc.move_contiguous(exp[G:G + B], src.numpy()[:B], C, [1] * (1 + lb), log, S=2) == 0
    assert np.array_equal(dst.cpu().numpy(), exp)


def test_dynamic_kv_fetch_and_offload(mma, orc):
    configure(mma, loopback=2, chunk=MiB, plan_mode=2, hop=(2, 2))
    shape = W.scaled_kv(512)
    ho, do, sb, hpool, dbytes = W.kv_segments(shape)
    host = torch.empty(hpool, dtype=torch.uint8).pin_memory()
    mma_inputs.fill_pattern(host.numpy(), 71)
    cache = torch.full((dbytes,), 0xA5, dtype=torch.uint8, device="cuda")
    lens = np.full(len(ho), sb, dtype=np.int64)
    segs, nseg = mma.make_segments(host.data_ptr() + ho, cache.data_ptr() + do, lens)
    mma.memcpy_h2d_segments(segs, nseg, 0)
    torch.cuda.synchronize()
    B = int(lens.sum())
    n = (B + MiB - 1) // MiB
    log = _check_log(mma, n, 3)
    exp = np.full(dbytes, 0xA5, dtype=np.uint8)
    osegs, on = orc.segments_from_arrays(host.numpy().ctypes.data + ho, exp.ctypes.data + do, lens)
    assert orc.move(osegs, on, MiB, [1, 1, 1], log, S=2) == 0
    assert np.array_equal(cache.cpu().numpy(), exp)
    # offload the cache back into a fresh pool
    back = torch.full((hpool,), 0xA5, dtype=torch.uint8).pin_memory()
    segs2, n2 = mma.make_segments(cache.data_ptr() + do, back.data_ptr() + ho, lens)
    mma.memcpy_d2h_segments(segs2, n2, 0)
    torch.cuda.synchronize()
    _check_log(mma, n, 3)
    got = back.numpy()
    hn = host.numpy()
    for k in range(0, len(ho), 13):
        assert np.array_equal(got[ho[k]:ho[k] + sb], hn[ho[k]:ho[k] + sb])


def test_dynamic_needs_all_zero_copy(mma):
    """A copy-engine path in the set keeps the planned (static) assignment."""
    configure(mma, loopback=1, chunk=MiB, plan_mode=2, hop=(1, 1))
    mma.reset_stats(0)
    src = pinned(torch, 8 * MiB, seed=5)
    dst = torch.empty(8 * MiB, dtype=torch.uint8, device="cuda")
    mma.memcpy_h2d(dst, src, 8 * MiB)
    torch.cuda.synchronize()
    assert mma.get_stats(0)["dynamic_calls"] == 0
    assert torch.equal(dst.cpu(), src[:8 * MiB])


@pytest.mark.parametrize("policy", [0, 1], ids=["maximize", "yield"])
def test_background_policy_mechanism(mma, orc, policy):
    """P:574 contention with background traffic: with background_policy = 1 a CTA whose unit
    took longer than the path's bandwidth predicts waits before claiming again. Pinning an
    absurdly high bandwidth makes every unit look "blocked": the yield policy must then wait
    (and still move every byte exactly once); the default policy never waits."""
    cfg = configure(mma, loopback=1, chunk=MiB, plan_mode=2, hop=(2, 2), claim=256 << 10)
    cfg.background_policy = policy
    mma.init(cfg)
    mma.set_bandwidth(0, mma.H2D, [10_000_000, 10_000_000])
    B = 32 * MiB + 99
    src = pinned(torch, B, seed=17)
    dst = guarded_device(torch, B)
    mma.memcpy_h2d(dst[G:G + B], src, B)
    torch.cuda.synchronize()
    log = np.frombuffer(mma.get_delivery_log(0), dtype=np.uint8)
    assert set(log.tolist()) <= {0, 1}
    exp = guarded_host(B)
    assert orc.move_contiguous(exp[G:G + B], src.numpy()[:B], 256 << 10, [1, 1], log.copy(), S=2) == 0
    assert np.array_equal(dst.cpu().numpy(), exp)
    waits = mma.get_dynamic_backoffs(0)
    assert (waits > 0) if policy else (waits == 0), waits
