"""The north_star invariant "a chunk is forwarded only after its staging write completes",
observed on the GPU ("How each oracle invariant is observed": C1 logs the seq
value it observed at forward start; it must be base + j + 1). For every chunk a kernel-driven
relay ring moves, the relay kernel records the flag value it saw satisfied before touching
the slot: H2D pull -- seq must equal g + 1 (the hop-1 DMA of exactly this chunk completed);
D2H pack -- credit must be >= g + 1 - S (the slot's previous chunk was drained to the host).
Both are checked against the oracle's plan (which chunks the rings carry) over several calls
(ring bases > 0), and a dropped publish shows up in the log as an aborted observation."""
import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from gpu_util import G, configure, guarded_device, pinned

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

MiB = 1 << 20
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def mma():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    os.environ.setdefault("MMA_SPIN_TIMEOUT_MS", "8000")
    import paper_2512_16056_b200 as m
    yield m
    m.finalize()


@pytest.mark.parametrize("hop", [1, 4], ids=["pull", "push"])
@pytest.mark.parametrize("S", [1, 2, 4])
@pytest.mark.parametrize("scattered", [False, True], ids=["contig", "segments"])
def test_forward_only_after_staging(mma, orc, S, scattered, hop):
    configure(mma, loopback=2, chunk=MiB, slots=S, plan_mode=1, hop=(hop, hop))
    _forward_case(mma, orc, S, scattered)


@pytest.mark.parametrize("hop", [1, 4], ids=["pull", "push"])
@pytest.mark.parametrize("S", [1, 3])
@pytest.mark.parametrize("scattered", [False, True], ids=["contig", "segments"])
def test_forward_only_after_staging_relay_gpus(mma, orc, S, scattered, hop):
    """the same with the rings on two other engine GPUs (real peers on a multi-GPU box,
    virtual GPUs on one: MMA_VGPUS): the D2H pack kernel then runs on the relay
    GPU, the H2D pull kernel polls the relay's flags"""
    virtual = torch.cuda.device_count() < 3
    if virtual:
        mma.finalize()
        os.environ["MMA_VGPUS"] = "3"
    try:
        configure(mma, loopback=0, chunk=MiB, slots=S, plan_mode=1, hop=(hop, hop), paths=[0, 1, 2])
        assert [p["gpu"] for p in mma.get_paths(0, mma.H2D)] == [0, 1, 2]
        _forward_case(mma, orc, S, scattered)
    finally:
        if virtual:
            mma.finalize()
            os.environ.pop("MMA_VGPUS", None)


def _forward_case(mma, orc, S, scattered):
    bw = [1, 2, 2]
    mma.set_bandwidth(0, mma.H2D, bw)
    mma.set_bandwidth(0, mma.D2H, bw)
    B = 19 * MiB + 777
    for rep in range(3):
        src = pinned(torch, B, seed=50 + rep)
        dst = guarded_device(torch, B)
        torch.cuda.synchronize()
        if scattered:                                    # 19 x 1 MiB blocks + a ragged tail block
            n, sb = 20, MiB
            lens = [sb] * (n - 1) + [B - (n - 1) * sb]
            perm = np.random.default_rng(rep).permutation(n - 1)    # full blocks permuted, tail last
            offs = np.concatenate([[0], np.cumsum(lens[:-1])])
            dsto = [int(offs[p]) for p in perm] + [int(offs[-1])]
            segs = mma.make_segments([src.data_ptr() + int(o) for o in offs],
                                     [dst.data_ptr() + G + o for o in dsto], lens)
            mma.memcpy_h2d_segments(*segs, 0)
        else:
            mma.memcpy_h2d(dst[G:G + B], src, B)
        torch.cuda.synchronize()
        rc, path, _, _ = orc.plan(bw, B, MiB, 0, orc.INTERLEAVED)
        obs, exp = mma.get_forward_log(0)
        ring = path != 0
        assert obs.size == path.size
        assert (obs[ring] == exp[ring]).all() and (exp[ring] > 0).all(), (rep, obs, exp)
        assert (obs[~ring] == 0).all() and (exp[~ring] == 0).all()
        # D2H: the pack kernel reads the slot's credit before overwriting it
        host = pinned(torch, B)
        mma.memcpy_d2h(host, dst[G:G + B], B)
        torch.cuda.synchronize()
        obs, exp = mma.get_forward_log(0)
        g1 = exp[ring].astype(np.int64)                  # g + 1 per ring chunk
        o = obs[ring].astype(np.int64)
        assert ((g1 <= S) & (o == 0) | (o >= g1 - S)).all(), (rep, o, g1)
        assert o.max() < 1 << 62                         # no aborted ring
        assert mma.get_last_error() == 0


PROG = r"""
import json, sys
sys.path.insert(0, {root!r})
sys.path.insert(0, {root!r} + "/tests")
import numpy as np, torch
import paper_2512_16056_b200 as m
from gpu_util import configure, pinned
configure(m, loopback=1, chunk=1 << 20, slots=2, plan_mode=1, hop=(1, 1))
m.set_bandwidth(0, m.H2D, [1, 1])
B = 16 << 20
src = pinned(torch, B, seed=1)
dst = torch.zeros(B, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
m.memcpy_h2d(dst, src, B)
torch.cuda.synchronize()
obs, exp = m.get_forward_log(0)
print(json.dumps(dict(obs=[int(x) for x in obs], exp=[int(x) for x in exp], err=m.get_last_error())))
"""


def test_dropped_publish_is_visible_in_the_forward_log(tmp_path):
    """a seeded protocol bug (hop 1 never publishes ring chunk 3) must show in the log as a
    forward that did not see g + 1 (the ring aborts; the sticky error is set)"""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    script = tmp_path / "f.py"
    script.write_text(PROG.format(root=str(ROOT)))
    env = dict(os.environ, MMA_FAULT_DROP_PUBLISH="3", MMA_SPIN_TIMEOUT_MS="1500")
    p = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True, timeout=240)
    assert p.returncode == 0, p.stderr[-3000:]
    r = json.loads(p.stdout.strip().splitlines()[-1])
    obs, exp = np.array(r["obs"], dtype=object), np.array(r["exp"], dtype=object)
    ring = exp != 0
    assert r["err"] == 2001
    assert any(o != e for o, e in zip(obs[ring], exp[ring]))   # the violation is observed
