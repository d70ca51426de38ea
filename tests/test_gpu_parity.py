"""GPU parity: the CUDA path (libmma.so through its C ABI) against the CPU oracle on the
same seeded inputs, element by element: destination bytes (bit-exact, guard bands
included), the chunk -> path plan, and the delivery log written on the GPU by each chunk's
final hop. A single B200 has no peers, so relay paths are LOOPBACK relays (relay GPU =
target): the staging ring, seq/credit flags, stream memory operations and the relay
kernels all run, over one PCIe link (SURVEY §4 tier T3)."""
import numpy as np
import pytest

import mma_inputs

from gpu_util import G, configure, guarded_device, guarded_host, pinned

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]

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


def _oracle_expect_contig(orc, src_np, B, C, bw, path, S):
    exp = guarded_host(B)
    dst = exp[G:G + B]
    assert orc.move_contiguous(dst, src_np[:B], C, bw, path, S=S) == 0
    return exp


def _check_plan_and_log(mma, orc, dirn, B, C, bw, thr, mode, S):
    rc, path, counts, fb = orc.plan(bw, B, C, thr, mode)
    assert rc == 0
    got_path, got_fb = mma.get_plan(0, dirn, B)
    assert got_fb == fb and got_path == path.tobytes()
    return path, fb


H2D_CASES = [
    # B, C, loopback relays, slots, plan mode
    (64 * MiB, MiB, 1, 2, 0),             # config 1: 64 MiB, 1 MiB chunks, 2 paths
    (64 * MiB, MiB, 1, 2, 1),
    (3 * MiB + 12345, MiB, 2, 1, 1),      # ragged tail, S = 1
    (10 * MiB + 7, 256 << 10, 3, 4, 1),
    (MiB - 1, MiB, 1, 2, 0),              # one short chunk
    (MiB + 1, MiB, 1, 2, 1),
    (2 * MiB + 4096, 4096, 1, 3, 1),      # 513 tiny chunks
]


@pytest.mark.parametrize("B,C,lb,S,mode", H2D_CASES)
@pytest.mark.parametrize("hop", [1, 2, 3, 4], ids=["ce", "zc", "ce_p2p", "push"])
def test_h2d_contiguous(mma, orc, B, C, lb, S, mode, hop):
    configure(mma, loopback=lb, chunk=C, slots=S, plan_mode=mode, hop=(hop, hop))
    bw = [1] * (1 + lb)
    mma.set_bandwidth(0, mma.H2D, bw)
    src = pinned(torch, B, seed=7)
    dst = guarded_device(torch, B)
    path, fb = _check_plan_and_log(mma, orc, mma.H2D, B, C, bw, 0, mode, S)
    mma.memcpy_h2d(dst[G:G + B], src, B)
    torch.cuda.synchronize()
    assert mma.get_last_error() == 0
    got = dst.cpu().numpy()
    exp = _oracle_expect_contig(orc, src.numpy(), B, C, bw, path, S)
    assert np.array_equal(got, exp)
    log = mma.get_delivery_log(0)
    assert log == path.tobytes()


@pytest.mark.parametrize("B,C,lb,S,mode", H2D_CASES)
@pytest.mark.parametrize("hop", [1, 2, 3, 4], ids=["ce", "zc", "ce_p2p", "push"])
def test_d2h_contiguous(mma, orc, B, C, lb, S, mode, hop):
    configure(mma, loopback=lb, chunk=C, slots=S, plan_mode=mode, hop=(hop, hop))
    bw = [1] * (1 + lb)
    mma.set_bandwidth(0, mma.D2H, bw)
    src_host = pinned(torch, B, seed=11)
    src = torch.empty(B, dtype=torch.uint8, device="cuda")
    src.copy_(src_host[:B])
    dst = pinned(torch, B + 2 * G)
    dst.fill_(0xA5)
    path, fb = _check_plan_and_log(mma, orc, mma.D2H, B, C, bw, 0, mode, S)
    mma.memcpy_d2h(dst[G:G + B], src, B)
    torch.cuda.synchronize()
    assert mma.get_last_error() == 0
    exp = _oracle_expect_contig(orc, src_host.numpy(), B, C, bw, path, S)
    assert np.array_equal(dst.numpy(), exp)
    assert mma.get_delivery_log(0) == path.tobytes()


def test_misaligned_pointers(mma, orc):
    """src and dst with different alignment modulo 16: byte path of the kernels."""
    B, C = 5 * MiB + 3, MiB
    for hop in (1, 2):
        configure(mma, loopback=2, chunk=C, slots=2, plan_mode=1, hop=(hop, hop))
        bw = [3, 2, 1]
        mma.set_bandwidth(0, mma.H2D, bw)
        src = pinned(torch, B + 5, seed=3)
        dst = guarded_device(torch, B + 3)
        mma.memcpy_h2d(dst[G + 3:G + 3 + B], src[5:5 + B], B)
        torch.cuda.synchronize()
        rc, path, _, _ = orc.plan(bw, B, C, 0, 1)
        exp = guarded_host(B + 3)
        orc.move_contiguous(exp[G + 3:G + 3 + B], src.numpy()[5:5 + B], C, bw, path, S=2)
        assert np.array_equal(dst.cpu().numpy(), exp)


def test_repeated_calls_ring_reuse(mma, orc):
    """Rings persist across calls with monotone sequence numbers (reading R18)."""
    B, C = 9 * MiB + 100, MiB
    configure(mma, loopback=2, chunk=C, slots=3, plan_mode=1, hop=(1, 1))
    mma.set_bandwidth(0, mma.H2D, [2, 1, 1])
    stream = torch.cuda.Stream()
    srcs = [pinned(torch, B, seed=100 + k) for k in range(5)]
    dsts = [torch.zeros(B, dtype=torch.uint8, device="cuda") for _ in range(5)]
    torch.cuda.synchronize()                  # the zero fills (default stream) precede the copies
    with torch.cuda.stream(stream):
        for k in range(5):
            mma.memcpy_h2d(dsts[k], srcs[k], B, stream=stream)
    stream.synchronize()
    for k in range(5):
        assert torch.equal(dsts[k].cpu(), srcs[k][:B])


def test_stream_ordering(mma):
    """Work before the call on the user stream completes first; work after sees the bytes
    (cudaMemcpyAsync semantics, §3.1)."""
    B, C = 32 * MiB, MiB
    configure(mma, loopback=1, chunk=C, slots=2, plan_mode=1, hop=(1, 1))
    mma.set_bandwidth(0, mma.H2D, [1, 1])
    mma.set_bandwidth(0, mma.D2H, [1, 1])
    s = torch.cuda.Stream()
    src = pinned(torch, B, seed=5)
    dev = torch.empty(B, dtype=torch.uint8, device="cuda")
    back = pinned(torch, B)
    with torch.cuda.stream(s):
        for _ in range(3):
            dev.fill_(0)                                   # before: must not clobber
            torch.cuda._sleep(2_000_000)                   # make ordering bugs visible
            mma.memcpy_h2d(dev, src, B, stream=s)
            dev2 = dev.to(torch.int16).add_(1).to(torch.uint8)   # after: must see the copy
            mma.memcpy_d2h(back, dev2, B, stream=s)
    s.synchronize()
    exp = (src.numpy()[:B].astype(np.int16) + 1).astype(np.uint8)
    assert np.array_equal(back.numpy()[:B], exp)


def test_fallback_and_errors(mma):
    configure(mma, loopback=1, chunk=MiB, thr=4 * MiB, plan_mode=1, hop=(1, 1))
    mma.set_bandwidth(0, mma.H2D, [1, 1])
    mma.reset_stats(0)
    src = pinned(torch, 3 * MiB, seed=9)
    dst = torch.zeros(3 * MiB, dtype=torch.uint8, device="cuda")
    mma.memcpy_h2d(dst, src, 3 * MiB)                      # below threshold -> native
    torch.cuda.synchronize()
    assert torch.equal(dst.cpu(), src)
    st = mma.get_stats(0)
    assert st["fallbacks"] == 1 and st["kernels"] == 0
    pageable = torch.from_numpy(mma_inputs.pattern_bytes(9, 8 * MiB))   # not pinned -> native
    dst8 = torch.zeros(8 * MiB, dtype=torch.uint8, device="cuda")
    mma.memcpy_h2d(dst8, pageable, 8 * MiB)
    torch.cuda.synchronize()
    assert torch.equal(dst8.cpu(), pageable)
    mma.memcpy_h2d(dst, src, 0)                            # zero bytes: no-op
    with pytest.raises(mma.MMAError) as e:
        mma.memcpy_h2d(0, src, 16)
    assert e.value.code == 1                               # cudaErrorInvalidValue
    with pytest.raises(mma.MMAError):
        mma.memcpy_h2d(dst, dst8, 16)                      # device -> device is not H2D
    with pytest.raises(mma.MMAError):
        mma.memcpy_d2h(src, src, 16)                       # host source for D2H
    with pytest.raises(mma.MMAError):
        mma.set_bandwidth(0, mma.H2D, [1, 1, 1])           # wrong path count


def test_stats_account_paths(mma):
    B, C = 16 * MiB, MiB
    configure(mma, loopback=1, chunk=C, plan_mode=0, hop=(1, 1))
    mma.set_bandwidth(0, mma.H2D, [3, 1])
    mma.reset_stats(0)
    src = pinned(torch, B, seed=1)
    dst = torch.empty(B, dtype=torch.uint8, device="cuda")
    mma.memcpy_h2d(dst, src, B)
    torch.cuda.synchronize()
    st = mma.get_stats(0)
    assert st["path_chunks"][0][:2] == [12, 4] and st["path_chunks"][1][:2] == [0, 0]
    assert st["path_bytes"][0][0] + st["path_bytes"][0][1] == B and st["relay_bytes"] == 4 * MiB
    assert st["kernels"] == 2                 # relay pull kernels: one per wave of S = 2 ring chunks


def test_device_generator_matches_host(mma):
    """verify.cu's splitmix64 stream == mma_inputs' (two independent implementations)."""
    for n, off in [(1, 0), (4099, 3), (1 << 20, 8), (777, 12345)]:
        d = torch.empty(n, dtype=torch.uint8, device="cuda")
        mma.fill_pattern(d, n, 0x4D4D41, off)
        torch.cuda.synchronize()
        assert np.array_equal(d.cpu().numpy(), mma_inputs.pattern_bytes(0x4D4D41, n, off))
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        mma.verify_pattern(d, n, 0x4D4D41, off, cnt)
        torch.cuda.synchronize()
        assert int(cnt.item()) == 0
        d[n // 2] ^= 1
        mma.verify_pattern(d, n, 0x4D4D41, off, cnt)
        torch.cuda.synchronize()
        assert int(cnt.item()) == 1


@pytest.mark.timeout(900)
def test_max_size_16gib(mma):
    """The sweep's largest size (16 GiB, config 2) through a copy-engine relay ring and the
    direct path, both directions; every byte checked on the device against the pattern."""
    B, C = 16 << 30, 4 * MiB
    configure(mma, loopback=1, chunk=C, slots=4, plan_mode=0, hop=(1, 2), debug=0)
    mma.set_bandwidth(0, mma.H2D, [1, 1])
    mma.set_bandwidth(0, mma.D2H, [1, 1])
    seed = 0x4D4D41 + 2
    dev = torch.empty(B, dtype=torch.uint8, device="cuda")
    mma.fill_pattern(dev, B, seed, 0)
    host = torch.empty(B, dtype=torch.uint8).pin_memory()
    mma.memcpy_d2h(host, dev, B)                       # D2H: direct ZC + loopback ZC relay
    dev2 = torch.zeros(B, dtype=torch.uint8, device="cuda")
    mma.memcpy_h2d(dev2, host, B)                      # H2D: direct CE + loopback CE ring
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    mma.verify_pattern(dev2, B, seed, 0, cnt)
    torch.cuda.synchronize()
    assert mma.get_last_error() == 0
    assert int(cnt.item()) == 0
    st = mma.get_stats(0)
    assert st["path_bytes"][0][1] > 0 and st["path_bytes"][1][1] > 0


def test_degenerate_segment_tables(mma):
    configure(mma, loopback=1, chunk=MiB, hop=(2, 2))
    host = torch.empty(MiB, dtype=torch.uint8).pin_memory()
    dev = torch.empty(MiB, dtype=torch.uint8, device="cuda")
    segs, n = mma.make_segments([], [], [])
    mma.memcpy_h2d_segments(segs, 0, 0)                                 # no segments
    segs, n = mma.make_segments([host.data_ptr()] * 3, [dev.data_ptr()] * 3, [0, 0, 0])
    mma.memcpy_h2d_segments(segs, n, 0)                                 # only empty ones
    segs, n = mma.make_segments([host.data_ptr()], [dev.data_ptr()], [1])
    mma.memcpy_h2d_segments(segs, n, 0)                                 # one byte
    torch.cuda.synchronize()
    assert dev[0].item() == host[0].item()
    with pytest.raises(mma.MMAError):
        mma.memcpy_h2d_segments(segs, n, 7, stream=torch.cuda.current_stream())  # no such device


def test_calibration_file_roundtrip(mma, tmp_path):
    """Only the calibration persists: bandwidth and mode per path survive a
    save / finalize / load cycle; lines for another path set are ignored."""
    configure(mma, loopback=2, chunk=MiB, debug=0)
    mma.set_bandwidth(0, mma.H2D, [7000, 6000, 5000])
    mma.set_path_modes(0, mma.D2H, [2, 1, 2])
    f = tmp_path / "cal.txt"
    mma.save_calibration(str(f))
    before = (mma.get_paths(0, mma.H2D), mma.get_paths(0, mma.D2H))
    mma.finalize()
    configure(mma, loopback=2, chunk=MiB, debug=0)
    assert mma.get_paths(0, mma.H2D)[0]["mbps"] != 7000
    assert mma.load_calibration(str(f)) == 6
    assert (mma.get_paths(0, mma.H2D), mma.get_paths(0, mma.D2H)) == before
    configure(mma, loopback=1, chunk=MiB, debug=0)      # a different path set
    assert mma.load_calibration(str(f)) == 4            # paths 0 and 1 still match, path 2 is gone


@pytest.mark.parametrize("dirn", [0, 1], ids=["h2d", "d2h"])
def test_ring_kinds_alternate_on_one_ring(mma, orc, dirn):
    """A relay ring driven by its kernel and the same ring driven by the copy engine alone
    (MMA_HOP_CE_P2P) share one slot protocol, so calls may alternate between them -- with an
    odd slot count, so slots change stream parity from one lap to the next."""
    C, S = 1 << 20, 3
    configure(mma, loopback=1, chunk=C, slots=S, plan_mode=1, hop=(1, 1), debug=1)
    bw = [1, 2]
    mma.set_bandwidth(0, dirn, bw)
    B = 11 * C + 777
    for k, relay_mode in enumerate([1, 3, 3, 1, 3, 1]):
        mma.set_path_modes(0, dirn, [1, relay_mode])
        mma.set_bandwidth(0, dirn, bw)
        seed = 0x4D4D41 + k
        rc, path, _, fb = orc.plan(bw, B, C, 0, 1)
        if dirn == 0:
            src = pinned(torch, B, seed=seed)
            dst = guarded_device(torch, B)
            mma.memcpy_h2d(dst[G:G + B], src, B)
            torch.cuda.synchronize()
            got = dst.cpu().numpy()
        else:
            dsrc = torch.empty(B, dtype=torch.uint8, device="cuda")
            mma.fill_pattern(dsrc, B, seed, 0)
            host = pinned(torch, B + 2 * G)
            host.numpy()[:] = 0xA5
            mma.memcpy_d2h(host[G:G + B], dsrc, B)
            torch.cuda.synchronize()
            got = host.numpy()
        exp = guarded_host(B)
        exp[G:G + B] = mma_inputs.pattern_bytes(seed, B, 0)
        assert np.array_equal(got, exp), (k, relay_mode)
        assert mma.get_delivery_log(0) == path.tobytes(), (k, relay_mode)
        assert mma.get_last_error() == 0
