"""Randomised GPU parity sweep: seeded random transfers (size, chunk, ring slots, loopback
relay count, per-path modes, plan mode, direction, contiguous or scattered, pointer
offsets) through the C ABI, each compared byte for byte with the oracle moving the same
transfer with the same assignment (the planned one, or the observed one in dynamic mode).
Rings persist across cases, so sequence bases and slot reuse vary too. The work order inside
a path (host_order) and CUDA graph capture + replay are drawn at random as well; neither may
change a byte. In planned mode the delivery log must equal the oracle's plan and, for
scattered tables (with faked NUMA nodes a quarter of the time), the engine's virtual-stream
order must equal the oracle's orc_numa_order: together the path of every byte.

test_random_transfers_virtual_gpus draws the same cases in the engine's virtual-GPU mode
(MMA_VGPUS=4): a random target among four engine GPUs and a random set of the other three
as relays (plus loopback relays), so rings, relay kernels and gates run with relay index !=
target on a one-GPU box (on a multi-GPU box the first GPUs are real peers)."""
import numpy as np
import pytest

import mma_inputs

from gpu_util import configure

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]

KiB, MiB = 1 << 10, 1 << 20


@pytest.fixture(scope="module")
def mma():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import os
    os.environ.setdefault("MMA_SPIN_TIMEOUT_MS", "8000")
    import paper_2512_16056_b200 as m
    yield m
    m.finalize()


def test_random_transfers(mma, orc):
    import os
    rng = np.random.default_rng(int(os.environ.get("MMA_RANDOM_SEED", "20261017")))
    _sweep(mma, orc, rng, int(os.environ.get("MMA_RANDOM_CASES", "200")), ngpu=1)


def test_random_transfers_virtual_gpus(mma, orc):
    import os
    mma.finalize()
    os.environ["MMA_VGPUS"] = "4"           # read at init (plane.h): a fresh engine
    try:
        rng = np.random.default_rng(int(os.environ.get("MMA_RANDOM_SEED", "20261017")) + 1)
        _sweep(mma, orc, rng, int(os.environ.get("MMA_RANDOM_CASES_VGPU", "150")), ngpu=4)
    finally:
        mma.finalize()
        os.environ.pop("MMA_VGPUS", None)


def _sweep(mma, orc, rng, cases, ngpu):
    import os
    nphys = torch.cuda.device_count()
    pool_h = torch.empty(48 * MiB, dtype=torch.uint8).pin_memory()
    mma_inputs.fill_pattern(pool_h.numpy(), 123)
    pools_d = {}
    hn = pool_h.numpy()
    for case in range(cases):
        if ngpu > 1:       # a target and a random set of the other engine GPUs as relays
            tgt = int(rng.integers(0, ngpu))
            others = [g for g in range(ngpu) if g != tgt]
            relays = [int(x) for x in rng.permutation(others)[:int(rng.integers(0, len(others) + 1))]]
            lb = int(rng.integers(0, 2))
        else:
            tgt, relays = 0, None
            lb = int(rng.integers(0, 4))
        dev = f"cuda:{tgt % nphys}"
        if dev not in pools_d:
            pools_d[dev] = torch.empty(48 * MiB, dtype=torch.uint8, device=dev)
            pools_d[dev].copy_(pool_h)
        pool_d = pools_d[dev]
        P = 1 + lb + (len(relays) if relays else 0)
        C = int(rng.choice([4 * KiB, 64 * KiB, 256 * KiB, MiB, 3 * MiB]))
        S = int(rng.integers(1, 5))
        plan_mode = int(rng.choice([0, 1, 2]))
        modes = [int(x) for x in rng.choice([1, 2, 3, 4], P)]
        if plan_mode == 2 and rng.random() < 0.7:
            modes = [2] * P
        bw = [int(x) for x in rng.integers(1, 6, P)]
        dirn = int(rng.integers(0, 2))
        scattered = rng.random() < 0.4
        host_order = int(rng.integers(0, 3))
        capture = plan_mode != 2 and rng.random() < 0.15
        fake_numa = rng.random() < 0.25      # R23 regrouping with faked host / path nodes
        if fake_numa:
            K = int(rng.integers(2, 4))
            path_node = [int(x) for x in rng.integers(0, 3, P)]
            os.environ["MMA_FAKE_HOST_NODES"] = str(K)
            os.environ["MMA_FAKE_PATH_NODES"] = ",".join(str(x) for x in path_node)
        else:
            os.environ.pop("MMA_FAKE_HOST_NODES", None)
            os.environ.pop("MMA_FAKE_PATH_NODES", None)
        configure(mma, loopback=lb, chunk=C, slots=S, plan_mode=plan_mode, hop=(1, 1), host_order=host_order,
                  paths=None if relays is None else ([tgt] + relays))
        assert len(mma.get_paths(tgt, dirn)) == P, (case, mma.get_paths(tgt, dirn))
        mma.set_path_modes(tgt, dirn, modes)
        mma.set_bandwidth(tgt, dirn, bw)
        if scattered:
            nseg = int(rng.integers(1, 200))
            lens = rng.integers(1, 96 * KiB, nseg)
            src_off = rng.integers(0, 40 * MiB, nseg)
            order = rng.permutation(nseg)
            dst_off = np.zeros(nseg, np.int64)
            pos = int(rng.integers(0, 64))
            for k in order:
                dst_off[k] = pos
                pos += int(lens[k]) + int(rng.integers(0, 100))
            span = pos + 64
        else:
            B = int(rng.integers(1, 24 * MiB))
            lens = np.array([B])
            src_off = np.array([int(rng.integers(0, 8 * MiB))])
            dst_off = np.array([int(rng.integers(0, 64))])
            span = B + 128
        B = int(lens.sum())
        print(f"case {case}: tgt={tgt} relays={relays} lb={lb} C={C} S={S} plan={plan_mode} modes={modes} bw={bw} dir={dirn} "
              f"scattered={scattered} nseg={len(lens)} B={B} order={host_order} capture={capture} "
              f"numa={fake_numa}", flush=True)
        if dirn == 0:      # H2D: host pool -> fresh device buffer
            dst = torch.full((span,), 0xA5, dtype=torch.uint8, device=dev)
            segs, n = mma.make_segments(pool_h.data_ptr() + src_off, dst.data_ptr() + dst_off, lens)
            src_np = hn
        else:              # D2H: device pool -> fresh pinned buffer
            dst = torch.full((span,), 0xA5, dtype=torch.uint8).pin_memory()
            segs, n = mma.make_segments(pool_d.data_ptr() + src_off, dst.data_ptr() + dst_off, lens)
            src_np = hn      # pool_d holds the same bytes
        as_segments = scattered or rng.random() < 0.5 or tgt >= nphys   # a virtual target is named
        torch.cuda.synchronize()

        def copy():
            if as_segments:
                (mma.memcpy_h2d_segments if dirn == 0 else mma.memcpy_d2h_segments)(
                    segs, n, tgt, stream=torch.cuda.current_stream())
            elif dirn == 0:
                mma.memcpy_h2d(dst.data_ptr() + int(dst_off[0]), pool_h.data_ptr() + int(src_off[0]), B)
            else:
                mma.memcpy_d2h(dst.data_ptr() + int(dst_off[0]), pool_d.data_ptr() + int(src_off[0]), B)
        if capture:      # recorded into a graph (rings stay out), then replayed once
            g = torch.cuda.CUDAGraph()
            with torch.cuda.device(dev), torch.cuda.graph(g):
                copy()
            g.replay()
        else:
            with torch.cuda.device(dev):
                copy()
        torch.cuda.synchronize()
        assert mma.get_last_error() == 0, case
        dynamic = plan_mode == 2 and all(m == 2 for m in modes)
        if capture:      # the bytes are dst == src whatever the captured plan; check with the planned one
            rc, path, _, fb = orc.plan(bw, B, C, 0, plan_mode)
            assert rc == 0
        elif dynamic:
            fb = False
            path = np.frombuffer(mma.get_delivery_log(tgt), dtype=np.uint8)
            assert path.size == (B + C - 1) // C and (path < P).all(), case
        else:
            rc, path, _, fb = orc.plan(bw, B, C, 0, 0 if plan_mode == 2 else plan_mode)
            assert rc == 0
        # the virtual stream's segment order: the oracle's NUMA-affine order (R23) of the same
        # per-segment host nodes (the fake hook: 2 MiB region index mod K), else table order
        vorder = np.arange(len(lens))
        if as_segments and len(lens) >= 2 and fake_numa:
            hptr = (pool_h.data_ptr() + src_off) if dirn == 0 else (dst.data_ptr() + dst_off)
            seg_node = ((np.asarray(hptr, dtype=np.uint64) >> np.uint64(21)) % np.uint64(K)).astype(np.int32)
            vorder = orc.numa_order(seg_node, bw, path_node).astype(np.int64)
        if not capture and not dynamic and not fb:   # planned: the executed route is the oracle's, per byte
            assert mma.get_delivery_log(tgt) == path.tobytes(), case
            if as_segments and len(lens) >= 2:
                assert mma.get_segment_order(tgt).tolist() == vorder.tolist(), case
        exp = np.full(span, 0xA5, dtype=np.uint8)
        osegs, on = orc.segments_from_arrays(src_np.ctypes.data + src_off[vorder], exp.ctypes.data + dst_off[vorder],
                                             lens[vorder])
        assert orc.move(osegs, on, C, bw, path, S=S) == 0
        got = dst.cpu().numpy() if dirn == 0 else dst.numpy()
        assert np.array_equal(got, exp), (case, dict(tgt=tgt, relays=relays, lb=lb, C=C, S=S, plan=plan_mode, modes=modes, dir=dirn,
                                                     scattered=scattered, B=B, numa=fake_numa))
    os.environ.pop("MMA_FAKE_HOST_NODES", None)
    os.environ.pop("MMA_FAKE_PATH_NODES", None)
