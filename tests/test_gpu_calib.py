"""Concurrent calibration (the bandwidth vector is "measured with all paths
of the set active"). On one B200 the relay paths are loopback rings through the target's own
link, so all paths share one PCIe link: alone each runs near the link rate, together they
split it. The concurrent vector must show that (its sum near one link, far below the sum of
the solo rates), the planner must use it, and copies planned from it stay byte-exact and
plan-exact against the oracle."""
import numpy as np
import pytest

import mma_inputs

from gpu_util import G, configure, guarded_device, guarded_host, pinned

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

MiB = 1 << 20


@pytest.fixture(scope="module")
def mma():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import os
    os.environ.setdefault("MMA_SPIN_TIMEOUT_MS", "8000")
    import paper_2512_16056_b200 as m
    torch.cuda.init()
    yield m
    m.finalize()


@pytest.mark.parametrize("dirn", [0, 1], ids=["h2d", "d2h"])
def test_concurrent_vector_sees_the_shared_link(mma, orc, dirn):
    cfg = configure(mma, loopback=2, chunk=4 * MiB, slots=4, debug=1)
    assert cfg.calib_rounds == 2                       # the default
    mma.calibrate(0, dirn, 256 * MiB)
    cal = mma.get_calibration(0, dirn)
    paths = mma.get_paths(0, dirn)
    assert len(cal) == len(paths) == 3
    solo = [c["solo"] for c in cal]
    conc = [c["conc"] for c in cal]
    link = solo[0]                                                 # the direct path alone
    assert all(s > 0.5 * link for s in solo), (solo, link)          # each path alone ~ the link
    assert all(c > 0 for c in conc), conc                          # every path carried bytes
    assert sum(conc) < 0.6 * sum(solo), (conc, solo)               # together they share it
    assert 0.6 * link < sum(conc) < 1.5 * link, (conc, link)
    assert [p["mbps"] for p in paths] == conc                      # the planner's vector

    # a copy planned from the measured vector: plan parity and bytes vs the oracle
    B = 96 * MiB + 4321
    C = 4 * MiB
    rc, path, _, fb = orc.plan(conc, B, C, 0, orc.CONTIG)
    assert rc == 0 and not fb
    got, gfb = mma.get_plan(0, dirn, B)
    assert not gfb and got == path.tobytes()
    S = cfg.ring_slots
    if dirn == 0:
        src = pinned(torch, B, seed=0x4D4D41)
        dst = guarded_device(torch, B)
        mma.memcpy_h2d(dst[G:G + B], src, B)
        torch.cuda.synchronize()
        exp = guarded_host(B)
        assert orc.move_contiguous(exp[G:G + B], src.numpy()[:B], C, conc, path, S=S) == 0
        assert np.array_equal(dst.cpu().numpy(), exp)
    else:
        dsrc = torch.empty(B, dtype=torch.uint8, device="cuda:0")
        mma.fill_pattern(dsrc, B, 0x4D4D42, 0)
        host = pinned(torch, B + 2 * G)
        host.numpy()[:] = 0xA5
        mma.memcpy_d2h(host[G:G + B], dsrc, B)
        torch.cuda.synchronize()
        exp = guarded_host(B)
        exp[G:G + B] = mma_inputs.pattern_bytes(0x4D4D42, B, 0)
        assert np.array_equal(host.numpy(), exp)
    assert mma.get_delivery_log(0) == path.tobytes()
    assert mma.get_last_error() == 0


def test_zero_rounds_keeps_solo_rates(mma):
    cfg = configure(mma, loopback=1, chunk=4 * MiB, slots=4, debug=0)
    cfg.calib_rounds = 0
    mma.init(cfg)
    mma.calibrate(0, mma.H2D, 128 * MiB)
    cal = mma.get_calibration(0, mma.H2D)
    assert [c["conc"] for c in cal] == [0, 0]
    assert [p["mbps"] for p in mma.get_paths(0, mma.H2D)] == [c["solo"] for c in cal]


def test_single_path_is_not_refined(mma):
    cfg = configure(mma, loopback=0, chunk=4 * MiB, debug=0)
    mma.init(cfg)
    mma.calibrate(0, mma.H2D, 64 * MiB)
    cal = mma.get_calibration(0, mma.H2D)
    assert len(cal) == 1 and cal[0]["solo"] > 0 and cal[0]["conc"] == 0


def test_scattered_tuning_is_refined(mma, orc):
    """mma_tune_segments on a scattered table: modes by solo measurement, rates concurrent."""
    configure(mma, loopback=1, chunk=MiB, slots=4, debug=1)
    nseg, sb = 2048, 32 << 10
    rng = np.random.default_rng(7)
    pool = pinned(torch, 2 * nseg * sb, seed=0x4D4D43)
    slots = rng.permutation(2 * nseg)[:nseg]
    cache = torch.zeros(nseg * sb + 2 * G, dtype=torch.uint8, device="cuda:0")
    dperm = rng.permutation(nseg)
    segs, _ = mma.make_segments([pool.data_ptr() + int(s) * sb for s in slots],
                             [cache.data_ptr() + G + int(k) * sb for k in dperm], [sb] * nseg)
    mma.tune_segments(segs, nseg, 0, mma.H2D, reps=1)
    cal = mma.get_calibration(0, mma.H2D, scattered=True)
    conc = [c["conc"] for c in cal]
    assert all(c > 0 for c in conc) and sum(conc) < 0.75 * sum(c["solo"] for c in cal), cal
    # the scattered copy planned from the refined vector is byte-exact
    cache.zero_()
    mma.memcpy_h2d_segments(segs, nseg, 0)
    torch.cuda.synchronize()
    got = cache.cpu().numpy()
    blocks = got[G:G + nseg * sb].reshape(nseg, sb)
    assert np.array_equal(blocks[dperm], pool.numpy()[:2 * nseg * sb].reshape(2 * nseg, sb)[slots])
    assert not got[:G].any() and not got[G + nseg * sb:].any()
    assert mma.get_last_error() == 0


@pytest.mark.parametrize("dirn", [0, 1], ids=["h2d", "d2h"])
def test_threshold_by_measurement(mma, dirn):
    """mma_tune_threshold (SURVEY a1, P:910 break-even): on one B200 a loopback relay shares
    the target's own link, so multipath never beats the native copy at any size: no
    break-even is found and the configured threshold stays. A direct-only set gives the same
    answer (nothing to gain)."""
    cfg = configure(mma, loopback=1, chunk=4 * MiB, slots=4, debug=0, thr=12 * MiB)
    mma.set_bandwidth(0, dirn, [1, 1])
    assert mma.get_plan(0, dirn, 8 * MiB)[1] is True               # below the threshold
    assert mma.get_plan(0, dirn, 64 * MiB)[1] is False
    thr, found = mma.tune_threshold(0, dirn, 128 * MiB)
    assert (thr, found) == (12 * MiB, False)
    assert mma.get_plan(0, dirn, 64 * MiB)[1] is False
    configure(mma, loopback=0, chunk=4 * MiB, debug=0, thr=0)
    assert mma.tune_threshold(0, dirn, 32 * MiB) == (0, False)
    assert mma.get_last_error() == 0


def test_chunk_size_by_measurement(mma, orc):
    """mma_tune_chunk (P:526 'dynamically adjusts', reading R3): the chosen size is one of the
    candidates, becomes the planner's chunk, and copies stay byte- and plan-exact with it"""
    configure(mma, loopback=1, chunk=4 * MiB, slots=4, debug=1)
    mma.set_path_modes(0, mma.H2D, [mma.HOP_CE, mma.HOP_CE_P2P])
    mma.set_bandwidth(0, mma.H2D, [1, 1])
    C = mma.tune_chunk(0, mma.H2D, 256 * MiB)
    assert C in [k * MiB for k in (1, 2, 4, 8, 16, 32)], C
    B = 3 * C + 12345
    path, fb = mma.get_plan(0, mma.H2D, B)
    assert not fb and len(path) == 4
    rc, exp_path, _, _ = orc.plan([1, 1], B, C, 0, 0)
    assert path == exp_path.tobytes()
    src = pinned(torch, B, seed=8)
    dst = torch.zeros(B, dtype=torch.uint8, device="cuda")
    mma.memcpy_h2d(dst, src, B)
    torch.cuda.synchronize()
    assert torch.equal(dst.cpu(), src[:B])
    assert mma.get_delivery_log(0) == exp_path.tobytes()
    assert mma.get_last_error() == 0
