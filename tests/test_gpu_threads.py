"""Thread safety (include/mma.h conventions): several host threads enqueue multipath copies
on their own streams at the same time (ctypes releases the GIL during the C calls); every
result must equal its source."""
import threading

import numpy as np
import pytest

import mma_inputs
from mma_inputs import workloads as W

from gpu_util import configure, pinned

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

MiB = 1 << 20


@pytest.fixture(scope="module")
def mma():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_16056_b200 as m
    yield m
    m.finalize()


def test_concurrent_threads(mma):
    configure(mma, loopback=2, chunk=MiB, slots=3, plan_mode=1, hop=(1, 2), debug=0)
    mma.set_bandwidth(0, mma.H2D, [2, 1, 1])
    mma.set_bandwidth(0, mma.D2H, [1, 1, 1])
    shape = W.scaled_kv(256)
    ho, do, sb, hpool, dbytes = W.kv_segments(shape)
    errors = []

    def worker(tid):
        try:
            s = torch.cuda.Stream()
            rng = np.random.default_rng(tid)
            for it in range(6):
                B = int(rng.integers(1, 20 * MiB))
                src = pinned(torch, B, seed=1000 + 10 * tid + it)
                dev = torch.empty(B, dtype=torch.uint8, device="cuda")
                back = pinned(torch, B)
                mma.memcpy_h2d(dev, src, B, stream=s)
                mma.memcpy_d2h(back, dev, B, stream=s)
                if it % 2:
                    pool = torch.empty(hpool, dtype=torch.uint8).pin_memory()
                    mma_inputs.fill_pattern(pool.numpy(), 7 + tid)
                    cache = torch.zeros(dbytes, dtype=torch.uint8, device="cuda")
                    torch.cuda.synchronize()   # the zero fill precedes the copy on s
                    lens = np.full(len(ho), sb, dtype=np.int64)
                    segs, n = mma.make_segments(pool.data_ptr() + ho, cache.data_ptr() + do, lens)
                    mma.memcpy_h2d_segments(segs, n, 0, stream=s)
                s.synchronize()
                if not np.array_equal(back.numpy()[:B], src.numpy()[:B]):
                    errors.append((tid, it, "contig"))
                if it % 2:
                    got = cache.cpu().numpy()
                    pn = pool.numpy()
                    for k in range(0, len(ho), 29):
                        if not np.array_equal(got[do[k]:do[k] + sb], pn[ho[k]:ho[k] + sb]):
                            errors.append((tid, it, "kv", k))
                            break
        except Exception as ex:  # noqa: BLE001
            errors.append((tid, repr(ex)))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    assert mma.get_last_error() == 0
