"""Every segment of a table is classified before anything is enqueued (
SURVEY §8(b) Errors and Fallback; include/mma.h mma_memcpy_h2d_segments).

Round 1 sampled 5 segments, so a bad pointer elsewhere reached a kernel as an illegal
address. Here the offending segment sits at an index no evenly spaced sample of 5 hits:
- a device pointer where host memory is expected -> cudaErrorInvalidValue and the guarded
  destination is untouched after a synchronize (nothing was enqueued);
- a pageable host piece -> the whole table is copied natively, byte-exact (R7);
- the classification cost of a config-3-sized table (131,072 segments) stays small."""
import numpy as np
import pytest

import mma_inputs

from gpu_util import configure, pinned

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

INVALID_VALUE = 1
NSEG, SB = 2000, 8 << 10
BAD = 1237            # not first, last, nor any of the 5 evenly spaced sample points


@pytest.fixture(scope="module")
def mma():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import os
    os.environ.setdefault("MMA_SPIN_TIMEOUT_MS", "8000")
    import paper_2512_16056_b200 as m
    yield m
    m.finalize()


def _table(mma, src_ptrs, dst_ptrs):
    return mma.make_segments(src_ptrs, dst_ptrs, [SB] * len(src_ptrs))


@pytest.mark.parametrize("hop", [1, 2], ids=["ce", "zc"])
def test_device_pointer_as_host_piece_rejected(mma, hop):
    configure(mma, loopback=1, hop=(hop, hop))
    mma.set_bandwidth(0, mma.H2D, [1, 1])
    host = pinned(torch, NSEG * SB, seed=3)
    other = torch.zeros(SB, dtype=torch.uint8, device="cuda")
    dst = torch.full((NSEG * SB,), 0xA5, dtype=torch.uint8, device="cuda")
    src = [host.data_ptr() + k * SB for k in range(NSEG)]
    src[BAD] = other.data_ptr()
    segs, n = _table(mma, src, [dst.data_ptr() + k * SB for k in range(NSEG)])
    k0 = mma.get_stats(0)
    with pytest.raises(mma.MMAError) as ei:
        mma.memcpy_h2d_segments(segs, n, 0)
    assert ei.value.code == INVALID_VALUE
    torch.cuda.synchronize()
    assert bool((dst == 0xA5).all().item())             # nothing was enqueued
    assert mma.get_stats(0)["calls"] == k0["calls"]
    # the D2H mirror: a device pointer as the host destination
    dsrc = [dst.data_ptr() + k * SB for k in range(NSEG)]
    hdst = [host.data_ptr() + k * SB for k in range(NSEG)]
    hdst[BAD] = other.data_ptr()
    before = host.numpy().copy()
    segs, n = _table(mma, dsrc, hdst)
    with pytest.raises(mma.MMAError) as ei:
        mma.memcpy_d2h_segments(segs, n, 0)
    assert ei.value.code == INVALID_VALUE
    torch.cuda.synchronize()
    assert np.array_equal(host.numpy(), before)
    assert mma.get_last_error() == 0


@pytest.mark.parametrize("hop", [1, 2], ids=["ce", "zc"])
def test_pageable_piece_makes_the_table_native(mma, hop):
    configure(mma, loopback=1, hop=(hop, hop))
    mma.set_bandwidth(0, mma.H2D, [1, 1])
    mma.set_bandwidth(0, mma.D2H, [1, 1])
    host = pinned(torch, NSEG * SB, seed=4)
    pageable = np.empty(SB, dtype=np.uint8)
    mma_inputs.fill_pattern(pageable, 99)
    dst = torch.full((NSEG * SB,), 0xA5, dtype=torch.uint8, device="cuda")
    perm = np.random.default_rng(8).permutation(NSEG)
    src = [host.data_ptr() + k * SB for k in range(NSEG)]
    src[BAD] = pageable.ctypes.data
    dptr = [dst.data_ptr() + int(p) * SB for p in perm]
    segs, n = _table(mma, src, dptr)
    s0 = mma.get_stats(0)
    mma.memcpy_h2d_segments(segs, n, 0)
    torch.cuda.synchronize()
    s1 = mma.get_stats(0)
    assert s1["fallbacks"] == s0["fallbacks"] + 1 and s1["kernels"] == s0["kernels"]
    got = dst.cpu().numpy().reshape(NSEG, SB)[perm]
    exp = host.numpy()[:NSEG * SB].reshape(NSEG, SB).copy()
    exp[BAD] = pageable
    assert np.array_equal(got, exp)
    # D2H: a pageable host destination piece
    out = pinned(torch, NSEG * SB)
    out.zero_()
    page_out = np.zeros(SB, dtype=np.uint8)
    hdst = [out.data_ptr() + k * SB for k in range(NSEG)]
    hdst[BAD] = page_out.ctypes.data
    segs, n = _table(mma, dptr, hdst)
    mma.memcpy_d2h_segments(segs, n, 0)
    torch.cuda.synchronize()
    o = out.numpy()[:NSEG * SB].reshape(NSEG, SB)
    assert np.array_equal(page_out, exp[BAD])
    keep = np.arange(NSEG) != BAD
    assert np.array_equal(o[keep], exp[keep]) and not o[BAD].any()
    assert mma.get_last_error() == 0


def test_validation_cost_config3_table(mma):
    """131,072 segments (the config-3 count; 4 KiB each here to keep the buffers small),
    host slots permuted in one pinned pool, device blocks spread over 64 tensors (the
    per-layer K/V caches): the per-call classification makes a few driver queries and stays
    around a millisecond"""
    configure(mma, loopback=0, hop=(2, 2), debug=0)
    n, sb = 131072, 4096
    pool = pinned(torch, 2 * n * sb)
    caches = [torch.empty(n // 64 * sb, dtype=torch.uint8, device="cuda") for _ in range(64)]
    rng = np.random.default_rng(11)
    slots = rng.permutation(2 * n)[:n]
    src = [pool.data_ptr() + int(s) * sb for s in slots]
    dst = [caches[k // (n // 64)].data_ptr() + (k % (n // 64)) * sb for k in range(n)]
    segs, cnt = mma.make_segments(src, dst, [sb] * n)
    mma.memcpy_h2d_segments(segs, cnt, 0)       # first call: allocations warm
    torch.cuda.synchronize()
    us = []
    for _ in range(3):
        s0 = mma.get_stats(0)
        mma.memcpy_h2d_segments(segs, cnt, 0)
        s1 = mma.get_stats(0)
        us.append(s1["validate_us"] - s0["validate_us"])
        q = s1["ptr_queries"] - s0["ptr_queries"]
        assert q <= 2 * (64 + 1) + 4, q            # one query (plus range) per allocation
    torch.cuda.synchronize()
    print(f"validate_us per call: {us}")
    assert min(us) < 3000, us
    assert mma.get_last_error() == 0
