"""Performance regression guard for DESIGN.md §5 item 12: relay kernels that wait beside the
copy engines of their own GPU must not slow them down. Seven loopback kernel rings with 16
CTAs each carry 7/8 of a 1 GiB copy on the one link; while the kernels read the engine's
host-memory error word on every few hundred polls this ran at 24 GB/s H2D / 16 GB/s D2H
(native 55 / 57), after the fix at 53 / 53 (profiles/r02_probe_lb_rings.jsonl). The bar
here is loose (0.75 of the native copy measured in the same test) so box-to-box variation
cannot fail it, while the regression would."""
import statistics

import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]

MiB, GiB = 1 << 20, 1 << 30


@pytest.fixture(scope="module")
def mma():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import os
    os.environ.setdefault("MMA_SPIN_TIMEOUT_MS", "8000")
    import paper_2512_16056_b200 as m
    yield m
    m.finalize()


def _rate(fn, s, B, reps=5):
    fn()
    s.synchronize()
    out = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        out.append(a.elapsed_time(b))
    return B / statistics.median(out) / 1e6


@pytest.mark.parametrize("dirn", [0, 1], ids=["h2d", "d2h"])
def test_waiting_relay_kernels_leave_the_copy_engines_alone(mma, dirn):
    torch.cuda.set_device(0)
    s = torch.cuda.Stream()
    B = GiB
    host = torch.empty(B, dtype=torch.uint8).pin_memory()
    dev = torch.empty(B, dtype=torch.uint8, device="cuda")
    cfg = mma.default_config()
    cfg.chunk_bytes[0] = cfg.chunk_bytes[1] = 8 * MiB
    cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = (1 << 64) - 1      # native first
    cfg.debug_log = 0
    mma.init(cfg)
    with torch.cuda.stream(s):
        copy = (lambda: mma.memcpy_h2d(dev, host, B, stream=s)) if dirn == 0 else \
               (lambda: mma.memcpy_d2h(host, dev, B, stream=s))
        native = _rate(copy, s, B)
    cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = 0
    cfg.loopback_relays = 7
    cfg.npaths, cfg.path_gpus[0] = 1, 0
    cfg.relay_ctas = 16
    mma.init(cfg)
    mma.set_path_modes(0, dirn, [mma.HOP_CE] * 8)                       # 7 kernel rings
    mma.set_bandwidth(0, dirn, [1] * 8)
    mma.reset_stats(0)
    with torch.cuda.stream(s):
        rings = _rate(copy, s, B)
    st = mma.get_stats(0)
    assert st["relay_bytes"] > 0 and st["kernels"] > 0
    assert mma.get_last_error() == 0
    assert rings > 0.75 * native, (rings, native)
