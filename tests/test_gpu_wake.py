"""Config 4 shape (vLLM sleep-mode wake): a model's tensors reloaded one call per tensor
from one packed pinned backup buffer; small tensors take the native fallback, large ones
the multipath engine (one loopback relay on a single GPU). Bytes are compared with the
oracle moving each tensor with its own plan."""
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
    import paper_2512_16056_b200 as m
    yield m
    m.finalize()


def test_wake_and_sleep_small_qwen(mma, orc):
    tensors = W.qwen_like_tensors(layers=4, hidden=1024, inter=2816, q_heads=16, kv_heads=4,
                                  head_dim=64, vocab=8192)
    offs, sizes, total = W.packed_layout(tensors)
    thr, C = 2 * MiB, MiB
    configure(mma, loopback=1, chunk=C, thr=thr, plan_mode=1, hop=(1, 2), debug=0)
    mma.set_bandwidth(0, mma.H2D, [2, 1])
    mma.set_bandwidth(0, mma.D2H, [1, 1])
    mma.reset_stats(0)
    host = torch.empty(total, dtype=torch.uint8).pin_memory()
    mma_inputs.fill_pattern(host.numpy(), 44)
    devbuf = torch.full((total,), 0xA5, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    torch.cuda.synchronize()                  # the guard fill (default stream) precedes the copies
    hp, dp = host.data_ptr(), devbuf.data_ptr()
    for o, n in zip(offs, sizes):
        mma.memcpy_h2d(dp + o, hp + o, n, stream=s)
    s.synchronize()
    got = devbuf.cpu().numpy()
    exp = np.full(total, 0xA5, dtype=np.uint8)
    hn = host.numpy()
    for o, n in zip(offs, sizes):
        rc, path, _, fb = orc.plan([2, 1], n, C, thr, 1)
        assert rc == 0 and fb == (n < thr)
        assert orc.move_contiguous(exp[o:o + n], hn[o:o + n], C, [2, 1], path, S=4) == 0
    assert np.array_equal(got, exp)
    st = mma.get_stats(0)
    assert st["fallbacks"] == sum(n < thr for n in sizes)
    assert st["calls"] == len(sizes) and st["kernels"] > 0
    # fall asleep: D2H of every tensor into a fresh backup buffer
    back = torch.zeros(total, dtype=torch.uint8).pin_memory()
    bp = back.data_ptr()
    for o, n in zip(offs, sizes):
        mma.memcpy_d2h(bp + o, dp + o, n, stream=s)
    s.synchronize()
    assert np.array_equal(back.numpy(), got)
    assert mma.get_last_error() == 0
