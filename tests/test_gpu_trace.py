"""Timeline tracing (mma_trace_begin / mma_trace_end): a traced loopback relay copy yields a
Chrome trace whose spans cover the direct DMA, the relay hop DMAs and the relay kernel."""
import json

import pytest

from gpu_util import configure, pinned

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]

MiB = 1 << 20


def test_trace_spans(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_16056_b200 as mma
    configure(mma, loopback=1, chunk=MiB, plan_mode=0, hop=(1, 1), debug=0)
    mma.set_bandwidth(0, mma.H2D, [1, 1])
    B = 16 * MiB
    src = pinned(torch, B, seed=3)
    dst = torch.empty(B, dtype=torch.uint8, device="cuda")
    mma.trace_begin()
    mma.memcpy_h2d(dst, src, B)
    torch.cuda.synchronize()
    p = tmp_path / "t.json"
    n = mma.trace_end(str(p))
    ev = json.load(open(p))["traceEvents"]
    # one direct run, 8 relay chunks, one relay kernel per wave of S = 2 ring chunks
    assert n == len(ev) == 1 + 8 + 4
    names = {e["name"] for e in ev}
    assert {"DMA direct", "DMA hop 1: host -> relay ring", "relay pull kernel"} <= names
    assert all(e["dur"] > 0 for e in ev)
    assert sum(e["args"]["bytes"] for e in ev if e["name"].startswith("DMA")) == B
    assert torch.equal(dst.cpu(), src[:B])
    with pytest.raises(mma.MMAError):
        mma.trace_end(None)                   # no trace active
