"""Joint plans of concurrent transfers (mma_memcpy_multi, the paper's Path
Selector, §3.4.2) on one B200: loopback relays stand for the other links (virtual
link ids MMA_MAX_GPUS + k, as run_multi numbers them). Every transfer of a batch must be
byte-exact, each on its own stream, and the chunk -> path map of the batch must be the
oracle's orc_plan_multi over the same links (the second transfer to one GPU continues the
first's queue, FIFO). Multi-target parity across real GPUs is in test_gpu_peer.py."""
import numpy as np
import pytest

from gpu_util import G, configure, guarded_device, guarded_host, pinned

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

MiB = 1 << 20
MAX_GPUS = 16


@pytest.fixture(scope="module")
def mma():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import os
    os.environ.setdefault("MMA_SPIN_TIMEOUT_MS", "8000")
    import paper_2512_16056_b200 as m
    yield m
    m.finalize()


def _oracle_paths(orc, bw, nchunks, mode):
    """oracle joint plan of transfers to GPU 0 whose path set is [direct] + loopback relays"""
    L = MAX_GPUS + 8
    link_bw = [0] * L
    ok = np.zeros((L, L), np.uint8)
    link_bw[0] = bw[0]
    for k, b in enumerate(bw[1:]):
        link_bw[MAX_GPUS + k] = b
        ok[0, MAX_GPUS + k] = b > 0
    rc, plans = orc.plan_multi(link_bw, ok, [0] * len(nchunks), nchunks, MiB, mode)
    assert rc == 0
    to_path = {0: 0, **{MAX_GPUS + k: 1 + k for k in range(len(bw) - 1)}}
    return [np.array([to_path[int(x)] for x in p], np.uint8) for p in plans]


@pytest.mark.parametrize("mode", [0, 1], ids=["contiguous", "interleaved"])
@pytest.mark.parametrize("hop", [1, 2, 3], ids=["kernel_ring", "zc", "ce_p2p"])
def test_two_fetches_one_queue(mma, orc, mode, hop):
    configure(mma, loopback=2, chunk=MiB, slots=3, plan_mode=mode, hop=(hop, hop))
    bw = [3, 2, 1]
    mma.set_bandwidth(0, mma.H2D, bw)
    sizes = [13 * MiB + 5, 9 * MiB + 4096]
    srcs = [pinned(torch, b, seed=40 + i) for i, b in enumerate(sizes)]
    dsts = [guarded_device(torch, b) for b in sizes]
    streams = [torch.cuda.Stream() for _ in sizes]
    torch.cuda.synchronize()                      # the guard fill (default stream) is done
    xf = [(mma.H2D, 0, mma.make_segments([s.data_ptr()], [d.data_ptr() + G], [b]), st)
          for s, d, b, st in zip(srcs, dsts, sizes, streams)]
    mma.memcpy_multi(xf)
    torch.cuda.synchronize()
    assert mma.get_last_error() == 0
    nch = [(b + MiB - 1) // MiB for b in sizes]
    plans = _oracle_paths(orc, bw, nch, mode)
    for s, d, b, p in zip(srcs, dsts, sizes, plans):
        exp = guarded_host(b)
        assert orc.move_contiguous(exp[G:G + b], s.numpy()[:b], MiB, bw, p, S=3) == 0
        assert np.array_equal(d.cpu().numpy(), exp)
    assert mma.get_delivery_log(0) == plans[-1].tobytes()     # the last transfer's executed route


def test_mixed_directions_and_shapes(mma, orc):
    """an H2D contiguous fetch, an H2D scattered fetch and a D2H scattered offload in one batch
    (each direction is planned on its own), on three streams"""
    configure(mma, loopback=1, chunk=MiB, slots=2, plan_mode=0, hop=(0, 0))
    mma.set_path_modes(0, mma.H2D, [1, 2])
    mma.set_path_modes(0, mma.D2H, [2, 1])
    mma.set_bandwidth(0, mma.H2D, [1, 1])
    mma.set_bandwidth(0, mma.D2H, [1, 2])
    nseg, sb = 300, 48 << 10
    rng = np.random.default_rng(4)
    pool = pinned(torch, 2 * nseg * sb, seed=7)
    slots = rng.permutation(2 * nseg)[:nseg]
    cache = guarded_device(torch, nseg * sb)
    B = 11 * MiB + 3
    src = pinned(torch, B, seed=8)
    dst = guarded_device(torch, B)
    dev_src = torch.empty(nseg * sb, dtype=torch.uint8, device="cuda")
    mma.fill_pattern(dev_src, nseg * sb, 99, 0)
    out = pinned(torch, 2 * nseg * sb)
    out.fill_(0xA5)
    torch.cuda.synchronize()
    st = [torch.cuda.Stream() for _ in range(3)]
    fetch = mma.make_segments([pool.data_ptr() + int(s) * sb for s in slots],
                              [cache.data_ptr() + G + k * sb for k in range(nseg)], [sb] * nseg)
    off = mma.make_segments([dev_src.data_ptr() + k * sb for k in range(nseg)],
                            [out.data_ptr() + int(s) * sb for s in slots], [sb] * nseg)
    mma.memcpy_multi([(mma.H2D, 0, mma.make_segments([src.data_ptr()], [dst.data_ptr() + G], [B]), st[0]),
                      (mma.H2D, 0, fetch, st[1]), (mma.D2H, 0, off, st[2])])
    torch.cuda.synchronize()
    assert mma.get_last_error() == 0
    exp = guarded_host(B)
    exp[G:G + B] = src.numpy()[:B]
    assert np.array_equal(dst.cpu().numpy(), exp)
    c = cache.cpu().numpy()
    assert (c[:G] == 0xA5).all() and (c[G + nseg * sb:] == 0xA5).all()
    assert np.array_equal(c[G:G + nseg * sb].reshape(nseg, sb), pool.numpy().reshape(2 * nseg, sb)[slots])
    o = out.numpy().reshape(2 * nseg, sb)
    assert np.array_equal(o[slots], dev_src.cpu().numpy().reshape(nseg, sb))
    assert (o[np.setdiff1d(np.arange(2 * nseg), slots)] == 0xA5).all()


def test_each_stream_sees_its_transfer(mma):
    """work enqueued on a transfer's stream after the batch runs after that transfer"""
    configure(mma, loopback=1, chunk=MiB, slots=2, plan_mode=0, hop=(1, 1))
    mma.set_bandwidth(0, mma.H2D, [1, 1])
    B = 24 * MiB
    srcs = [torch.full((B,), 11 + i, dtype=torch.uint8).pin_memory() for i in range(3)]
    dsts = [torch.zeros(B, dtype=torch.uint8, device="cuda") for _ in range(3)]
    probes = [torch.zeros(B, dtype=torch.uint8, device="cuda") for _ in range(3)]
    st = [torch.cuda.Stream() for _ in range(3)]
    torch.cuda.synchronize()
    mma.memcpy_multi([(mma.H2D, 0, mma.make_segments([s.data_ptr()], [d.data_ptr()], [B]), t)
                      for s, d, t in zip(srcs, dsts, st)])
    for d, p, t in zip(dsts, probes, st):
        with torch.cuda.stream(t):
            p.copy_(d)
    torch.cuda.synchronize()
    for i, p in enumerate(probes):
        assert bool((p == 11 + i).all().item()), i


def test_invalid_transfer_enqueues_nothing(mma):
    configure(mma, loopback=1, chunk=MiB, slots=2, plan_mode=0, hop=(1, 1))
    mma.set_bandwidth(0, mma.H2D, [1, 1])
    B = 8 * MiB
    src = pinned(torch, B, seed=1)
    dst = torch.full((B,), 0xA5, dtype=torch.uint8, device="cuda")
    other = torch.zeros(B, dtype=torch.uint8, device="cuda")
    good = (mma.H2D, 0, mma.make_segments([src.data_ptr()], [dst.data_ptr()], [B]), None)
    bad = (mma.H2D, 0, mma.make_segments([other.data_ptr()], [dst.data_ptr()], [B]), None)   # device as host
    with pytest.raises(mma.MMAError):
        mma.memcpy_multi([good, bad])
    torch.cuda.synchronize()
    assert bool((dst == 0xA5).all().item())
    with pytest.raises(mma.MMAError):
        mma.memcpy_multi([(mma.H2D, 7, mma.make_segments([src.data_ptr()], [dst.data_ptr()], [B]), 0)])


def test_random_batches(mma, orc):
    """randomised joint batches on one GPU: 1-4 transfers (mixed directions, contiguous or
    scattered, ragged sizes), random path modes, bandwidths and plan modes; every byte
    exact, and the last transfer's delivery log equal to the oracle's joint plan"""
    import os
    rng = np.random.default_rng(int(os.environ.get("MMA_RANDOM_SEED", "77")))
    KiB = 1 << 10
    pool_h = pinned(torch, 40 * MiB, seed=5)
    pool_d = torch.empty(40 * MiB, dtype=torch.uint8, device="cuda")
    pool_d.copy_(pool_h[:40 * MiB])
    for case in range(int(os.environ.get("MMA_MULTI_CASES", "60"))):
        lb = int(rng.integers(1, 4))
        mode = int(rng.integers(0, 2))
        configure(mma, loopback=lb, chunk=MiB, slots=int(rng.integers(1, 5)), plan_mode=mode, hop=(0, 0))
        bw = [int(x) for x in rng.integers(1, 6, 1 + lb)]
        for d in (mma.H2D, mma.D2H):
            mma.set_path_modes(0, d, [int(x) for x in rng.choice([1, 2, 3], 1 + lb)])
            mma.set_bandwidth(0, d, bw)
        T = int(rng.integers(1, 5))
        xf, checks = [], []
        for t in range(T):
            dirn = int(rng.integers(0, 2))
            nseg = 1 if rng.random() < 0.5 else int(rng.integers(2, 60))
            lens = rng.integers(1, 200 * KiB, nseg) if nseg > 1 else np.array([int(rng.integers(1, 12 * MiB))])
            src_off = rng.integers(0, 20 * MiB, nseg)
            span = int(lens.sum()) + 64 * nseg
            dst_off = np.concatenate([[0], np.cumsum(lens[:-1] + 64)]).astype(np.int64)
            if dirn == 0:
                dst = torch.full((span,), 0xA5, dtype=torch.uint8, device="cuda")
                segs = mma.make_segments(pool_h.data_ptr() + src_off, dst.data_ptr() + dst_off, lens)
            else:
                dst = torch.full((span,), 0xA5, dtype=torch.uint8).pin_memory()
                segs = mma.make_segments(pool_d.data_ptr() + src_off, dst.data_ptr() + dst_off, lens)
            xf.append((dirn, 0, segs, torch.cuda.Stream()))
            checks.append((dirn, dst, src_off, dst_off, lens, span))
        torch.cuda.synchronize()
        mma.memcpy_multi(xf)
        torch.cuda.synchronize()
        assert mma.get_last_error() == 0, case
        hn = pool_h.numpy()
        for dirn, dst, src_off, dst_off, lens, span in checks:
            got = dst.cpu().numpy() if dirn == 0 else dst.numpy()
            exp = np.full(span, 0xA5, np.uint8)
            for so, do_, ln in zip(src_off, dst_off, lens):
                exp[do_:do_ + ln] = hn[so:so + ln]
            assert np.array_equal(got, exp), (case, dirn, len(lens))
        # the last transfer's executed route = its part of the oracle's joint plan
        last_dir = checks[-1][0]
        nch = [(int(c[4].sum()) + MiB - 1) // MiB for c in checks if c[0] == last_dir]
        plans = _oracle_paths(orc, bw, nch, mode)
        assert mma.get_delivery_log(0) == plans[-1].tobytes(), case
