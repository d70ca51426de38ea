"""GPU parity of the scattered-segment variant (north_star (e)): a paged prefix-cache KV
fetch (config 3 shape: Llama-3-8B bf16 KV, 16-token blocks, 32 KiB segments scattered in a
pinned host pool) and its D2H offload mirror, against the oracle moving the same segment
table, byte for byte including untouched bytes of the pool and cache."""
import numpy as np
import pytest

import mma_inputs
from mma_inputs import workloads as W

from gpu_util import configure

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
    yield m
    m.finalize()


def _kv(tokens, seed=0x4D4D41 + 3):
    shape = W.scaled_kv(tokens)
    ho, do, sb, hpool, dbytes = W.kv_segments(shape, seed)
    return shape, ho, do, sb, hpool, dbytes


def _oracle_segments(orc, src_base_np, dst_np, s_off, d_off, lens, C, bw, path, S=2):
    segs, n = orc.segments_from_arrays(src_base_np.ctypes.data + s_off, dst_np.ctypes.data + d_off, lens)
    assert orc.move(segs, n, C, bw, path, S=S) == 0


CASES = [
    # tokens, chunk, loopback relays, plan mode, hop
    (256, MiB, 0, 0, 2),         # direct only, SM gather/scatter (the N=1 bench path)
    (256, MiB, 0, 0, 1),         # direct only, copy-engine batch
    (512, MiB, 1, 1, 1),         # ring: batch pack into slots + relay kernel unpack
    (512, MiB, 2, 0, 2),         # one-hop zero-copy relays
    (272, 192 << 10, 2, 1, 1),   # chunk not a multiple of the segment: pieces split
    (272, 192 << 10, 1, 1, 2),
    (2048, MiB, 1, 0, 2),        # 8192 segments: the radix path of the host-order sort
    (512, MiB, 2, 1, 3),         # all-copy-engine rings: batch into slots, peer batch out
    (272, 192 << 10, 1, 0, 3),
    (512, MiB, 2, 1, 4),         # push-form kernel rings (relay kernel on the sending side)
    (272, 192 << 10, 1, 0, 4),
]


@pytest.mark.parametrize("order", [0, 2], ids=["table_order", "host_order"])
@pytest.mark.parametrize("tokens,C,lb,mode,hop", CASES)
def test_kv_fetch_h2d(mma, orc, tokens, C, lb, mode, hop, order):
    configure(mma, loopback=lb, chunk=C, slots=2, plan_mode=mode, hop=(hop, hop), host_order=order)
    bw = [1] * (1 + lb)
    mma.set_bandwidth(0, mma.H2D, bw)
    shape, ho, do, sb, hpool, dbytes = _kv(tokens)
    host = torch.empty(hpool, dtype=torch.uint8).pin_memory()
    mma_inputs.fill_pattern(host.numpy(), 21)
    cache = torch.full((dbytes,), 0xA5, dtype=torch.uint8, device="cuda")
    lens = np.full(len(ho), sb, dtype=np.int64)
    segs, n = mma.make_segments(host.data_ptr() + ho, cache.data_ptr() + do, lens)
    B = int(lens.sum())
    rc, path, _, fb = orc.plan(bw, B, C, 0, mode)
    got_path, got_fb = mma.get_plan(0, mma.H2D, B)
    assert got_path == path.tobytes() and got_fb == fb
    mma.memcpy_h2d_segments(segs, n, 0)
    torch.cuda.synchronize()
    assert mma.get_last_error() == 0
    exp = np.full(dbytes, 0xA5, dtype=np.uint8)
    _oracle_segments(orc, host.numpy(), exp, ho, do, lens, C, bw, path)
    assert np.array_equal(cache.cpu().numpy(), exp)
    if not fb:
        assert mma.get_delivery_log(0) == path.tobytes()


@pytest.mark.parametrize("order", [0, 1], ids=["table_order", "host_order"])
@pytest.mark.parametrize("tokens,C,lb,mode,hop", CASES)
def test_kv_offload_d2h(mma, orc, tokens, C, lb, mode, hop, order):
    """host_order 1 (the default) moves each path's pieces in ascending host address: the
    plan, the bytes and the delivery log must not change."""
    configure(mma, loopback=lb, chunk=C, slots=2, plan_mode=mode, hop=(hop, hop), host_order=order)
    bw = [1] * (1 + lb)
    mma.set_bandwidth(0, mma.D2H, bw)
    shape, ho, do, sb, hpool, dbytes = _kv(tokens, seed=99)
    cache_host = mma_inputs.pattern_bytes(33, dbytes)
    cache = torch.from_numpy(cache_host).to("cuda")
    host = torch.full((hpool,), 0xA5, dtype=torch.uint8).pin_memory()
    lens = np.full(len(ho), sb, dtype=np.int64)
    segs, n = mma.make_segments(cache.data_ptr() + do, host.data_ptr() + ho, lens)
    B = int(lens.sum())
    rc, path, _, fb = orc.plan(bw, B, C, 0, mode)
    assert mma.get_plan(0, mma.D2H, B)[0] == path.tobytes()
    mma.memcpy_d2h_segments(segs, n, 0)
    torch.cuda.synchronize()
    exp = np.full(hpool, 0xA5, dtype=np.uint8)
    _oracle_segments(orc, cache_host, exp, do, ho, lens, C, bw, path)
    assert np.array_equal(host.numpy(), exp)
    if not fb:
        assert mma.get_delivery_log(0) == path.tobytes()
    assert mma.get_last_error() == 0


def test_irregular_segments(mma, orc):
    """Odd lengths, odd alignments, empty segments, destinations out of order."""
    rng = np.random.default_rng(8)
    nseg = 300
    lens = rng.integers(0, 50000, nseg)
    lens[::17] = 0
    pool = torch.empty(int(lens.sum()) * 2 + 1000, dtype=torch.uint8).pin_memory()
    mma_inputs.fill_pattern(pool.numpy(), 4)
    s_off = rng.integers(0, pool.numel() - 50000, nseg)
    order = rng.permutation(nseg)
    d_off = np.zeros(nseg, np.int64)
    pos = 3
    for k in order:
        d_off[k] = pos
        pos += int(lens[k]) + int(rng.integers(0, 40))
    for hop, lb, mode in [(1, 1, 1), (2, 2, 0), (2, 0, 1)]:
        configure(mma, loopback=lb, chunk=64 << 10, slots=2, plan_mode=mode, hop=(hop, hop))
        bw = [2] + [1] * lb
        mma.set_bandwidth(0, mma.H2D, bw)
        dev = torch.full((pos + 100,), 0xA5, dtype=torch.uint8, device="cuda")
        segs, n = mma.make_segments(pool.data_ptr() + s_off, dev.data_ptr() + d_off, lens)
        mma.memcpy_h2d_segments(segs, n, 0)
        torch.cuda.synchronize()
        B = int(lens.sum())
        rc, path, _, _ = orc.plan(bw, B, 64 << 10, 0, mode)
        exp = np.full(pos + 100, 0xA5, np.uint8)
        _oracle_segments(orc, pool.numpy(), exp, s_off, d_off, lens, 64 << 10, bw, path)
        assert np.array_equal(dev.cpu().numpy(), exp), (hop, lb, mode)


@pytest.mark.parametrize("dirn", [0, 1], ids=["h2d", "d2h"])
@pytest.mark.parametrize("C,lb,mode", [(64 << 10, 0, 0), (MiB, 2, 1), (192 << 10, 1, 2)])
def test_small_piece_groups(mma, orc, dirn, C, lb, mode):
    """The zero-copy kernels move runs of small 16-byte-friendly pieces as one round of loads
    (copy.cuh v_copy piece groups): mixed lengths (empty, 16 B, 4080 B, 32 KiB, 64 KiB + 16,
    odd), mostly 16-byte-aligned ends with some unaligned pieces breaking the groups, chunk
    and unit edges inside pieces; direct, one-hop relay and dynamic-pull zero-copy paths."""
    rng = np.random.default_rng(31 + dirn)
    nseg = 1500
    lens = rng.choice([0, 16, 32, 48, 4080, 4096, 8192, 32768, 65552, 7, 100], nseg,
                      p=[.03, .1, .1, .07, .1, .1, .1, .2, .1, .05, .05]).astype(np.int64)
    span_s = int(lens.sum()) * 2 + (1 << 20)
    s_off = (rng.integers(0, span_s - 70000, nseg) // 16) * 16
    bad = rng.random(nseg) < 0.08
    s_off[bad] += rng.integers(1, 16, int(bad.sum()))
    d_off = np.zeros(nseg, np.int64)
    pos = 0
    for k in rng.permutation(nseg):
        d_off[k] = pos + (int(rng.integers(1, 16)) if rng.random() < 0.05 else 0)
        pos = ((d_off[k] + int(lens[k]) + 15) // 16) * 16 + 16 * int(rng.integers(0, 3))
    span_d = pos + 4096
    configure(mma, loopback=lb, chunk=C, slots=2, plan_mode=mode, hop=(2, 2))
    bw = [2] + [1] * lb
    mma.set_bandwidth(0, dirn, bw)
    pat = mma_inputs.pattern_bytes(57, span_s)
    if dirn == 0:
        src = torch.from_numpy(pat.copy()).pin_memory()
        dst = torch.full((span_d,), 0xA5, dtype=torch.uint8, device="cuda")
    else:
        src = torch.from_numpy(pat.copy()).to("cuda")
        dst = torch.full((span_d,), 0xA5, dtype=torch.uint8).pin_memory()
    segs, n = mma.make_segments(src.data_ptr() + s_off, dst.data_ptr() + d_off, lens)
    (mma.memcpy_h2d_segments if dirn == 0 else mma.memcpy_d2h_segments)(segs, n, 0)
    torch.cuda.synchronize()
    assert mma.get_last_error() == 0
    B = int(lens.sum())
    rc, path, _, _ = orc.plan(bw, B, C, 0, min(mode, 1))    # bytes do not depend on the plan
    exp = np.full(span_d, 0xA5, np.uint8)
    _oracle_segments(orc, pat, exp, s_off, d_off, lens, C, bw, path)
    got = dst.cpu().numpy() if dirn == 0 else dst.numpy()
    assert np.array_equal(got, exp)


def test_overlapping_destinations_rejected(mma):
    configure(mma, loopback=0, chunk=MiB)
    host = torch.empty(MiB, dtype=torch.uint8).pin_memory()
    dev = torch.empty(MiB, dtype=torch.uint8, device="cuda")
    segs, n = mma.make_segments([host.data_ptr()] * 2, [dev.data_ptr(), dev.data_ptr() + 100],
                                [200, 200])
    with pytest.raises(mma.MMAError) as e:
        mma.memcpy_h2d_segments(segs, n, 0)
    assert e.value.code == 1


@pytest.mark.timeout(900)
def test_full_size_kv_fetch(mma, orc):
    """BASELINE config 3 at full size (131,072 x 32 KiB = 4 GiB from an 8 GiB pool) in the
    bench's launch configuration: every byte checked on the device against the seeded
    pattern, and sampled segments compared with the oracle moving those segments."""
    configure(mma, loopback=0, chunk=4 * MiB, plan_mode=0, hop=(0, 0), thr=8 * MiB, debug=0)
    shape, ho, do, sb, hpool, dbytes = _kv(32768)
    host = torch.empty(hpool, dtype=torch.uint8).pin_memory()
    seed = 0x4D4D41 + 3
    hd = torch.empty(hpool, dtype=torch.uint8, device="cuda")
    mma.fill_pattern(hd, hpool, seed, 0)
    host.copy_(hd)
    del hd
    cache = torch.full((dbytes,), 0xA5, dtype=torch.uint8, device="cuda")
    lens = np.full(len(ho), sb, dtype=np.int64)
    segs, n = mma.make_segments(host.data_ptr() + ho, cache.data_ptr() + do, lens)
    mma.memcpy_h2d_segments(segs, n, 0)
    torch.cuda.synchronize()
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    mma.verify_segments(cache.data_ptr() + do, ho, lens, seed, cnt)
    torch.cuda.synchronize()
    assert int(cnt.item()) == 0
    rng = np.random.default_rng(0)
    pick = rng.choice(len(ho), 64, replace=False)
    hnp = host.numpy()
    for k in pick:
        exp = np.zeros(sb, np.uint8)
        segs1, n1 = orc.segments_from_arrays([hnp.ctypes.data + int(ho[k])], [exp.ctypes.data], [sb])
        assert orc.move(segs1, n1, sb, [1], np.zeros(1, np.uint8)) == 0
        got = cache[int(do[k]):int(do[k]) + sb].cpu().numpy()
        assert np.array_equal(got, exp)
    # the bench's measured modes: fetch by the copy engine (batch), offload by the
    # zero-copy kernel into a fresh pool; the offloaded slots must equal the original pool
    mma.set_path_modes(0, mma.H2D, [mma.HOP_CE])
    mma.set_path_modes(0, mma.D2H, [mma.HOP_ZC])
    cache.fill_(0xA5)
    mma.memcpy_h2d_segments(segs, n, 0)
    back = torch.zeros(hpool, dtype=torch.uint8).pin_memory()
    osegs, on = mma.make_segments(cache.data_ptr() + do, back.data_ptr() + ho, lens)
    mma.memcpy_d2h_segments(osegs, on, 0)
    torch.cuda.synchronize()
    assert mma.get_last_error() == 0
    bn = back.numpy()
    for k in rng.choice(len(ho), 256, replace=False):
        assert np.array_equal(bn[ho[k]:ho[k] + sb], hnp[ho[k]:ho[k] + sb])
    untouched = np.ones(hpool // sb, bool)
    untouched[ho // sb] = False
    free_slot = int(np.flatnonzero(untouched)[0])
    assert not bn[free_slot * sb:(free_slot + 1) * sb].any()     # slots outside the table stay 0


def test_mode_choice_by_measurement(mma, orc):
    """mma_calibrate / mma_tune_segments time every path in each mode and keep the faster
    one (north_star (d)); copies afterwards stay bit-exact."""
    configure(mma, loopback=1, chunk=MiB, plan_mode=0, hop=(0, 0), debug=0)
    mma.calibrate(0, mma.H2D, 64 * MiB)
    ps = mma.get_paths(0, mma.H2D)
    # the direct path is copy engine or zero-copy; a relay may also be the all-copy-engine ring
    assert all(p["mode"] in ((1, 2) if p["kind"] == 0 else (1, 2, 3)) and p["mbps"] > 5000 for p in ps), ps
    shape, ho, do, sb, hpool, dbytes = _kv(512)
    host = torch.empty(hpool, dtype=torch.uint8).pin_memory()
    mma_inputs.fill_pattern(host.numpy(), 77)
    cache = torch.zeros(dbytes, dtype=torch.uint8, device="cuda")
    lens = np.full(len(ho), sb, dtype=np.int64)
    segs, n = mma.make_segments(host.data_ptr() + ho, cache.data_ptr() + do, lens)
    mma.tune_segments(segs, n, 0, mma.H2D, reps=1)
    ps = mma.get_paths(0, mma.H2D)
    assert all(p["seg_mode"] in ((1, 2) if p["kind"] == 0 else (1, 2, 3)) and p["seg_mbps"] > 5000 for p in ps), ps
    cache.zero_()
    mma.memcpy_h2d_segments(segs, n, 0)
    torch.cuda.synchronize()
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    got = cache.cpu().numpy()
    hn = host.numpy()
    for k in range(0, len(ho), 97):
        assert np.array_equal(got[do[k]:do[k] + sb], hn[ho[k]:ho[k] + sb])
    mma.set_bandwidth(0, mma.H2D, [1, 1])       # pinning clears the segment tuning
    assert all(p["seg_mbps"] == 0 for p in mma.get_paths(0, mma.H2D))


@pytest.mark.parametrize("zc_ctas", [1, 3, 4096])
@pytest.mark.parametrize("mode", [0, 2])
def test_zero_copy_grid_sizes(mma, orc, zc_ctas, mode):
    """mma_config_t::zc_ctas: the zero-copy kernels are grid-stride over units (planned) or
    claims (dynamic), so any grid -- one CTA, a ragged count, more CTAs than the cap --
    moves the same bytes. KV fetch and its offload mirror through two ZC paths."""
    shape, ho, do, sb, hpool, dbytes = _kv(272)
    cfg = configure(mma, loopback=1, chunk=192 << 10, plan_mode=mode, hop=(2, 2), debug=0)
    cfg.zc_ctas = zc_ctas
    mma.init(cfg)
    bw = [3, 2]
    for d in (mma.H2D, mma.D2H):
        mma.set_bandwidth(0, d, bw)
    pool = torch.empty(hpool, dtype=torch.uint8).pin_memory()
    mma_inputs.fill_pattern(pool.numpy(), 11)
    dev = torch.full((dbytes,), 0xA5, dtype=torch.uint8, device="cuda")
    lens = np.full(len(ho), sb, np.int64)
    segs, n = mma.make_segments(pool.data_ptr() + ho, dev.data_ptr() + do, lens)
    mma.memcpy_h2d_segments(segs, n, 0)
    torch.cuda.synchronize()
    rc, path, _, _ = orc.plan(bw, int(lens.sum()), 192 << 10, 0, 0)   # bytes do not depend on it
    exp = np.full(dbytes, 0xA5, np.uint8)
    _oracle_segments(orc, pool.numpy(), exp, ho, do, lens, 192 << 10, bw, path)
    assert np.array_equal(dev.cpu().numpy(), exp)
    back = torch.zeros(hpool, dtype=torch.uint8).pin_memory()
    segs, n = mma.make_segments(dev.data_ptr() + do, back.data_ptr() + ho, lens)
    mma.memcpy_d2h_segments(segs, n, 0)
    torch.cuda.synchronize()
    exp_h = np.zeros(hpool, np.uint8)
    _oracle_segments(orc, exp, exp_h, do, ho, lens, 192 << 10, bw, path)
    assert np.array_equal(back.numpy(), exp_h)
    bad = mma.default_config()
    bad.zc_ctas = -1
    with pytest.raises(mma.MMAError):
        mma.init(bad)
