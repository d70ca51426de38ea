"""The delivery log records what the engine EXECUTED, not what it planned (VERDICT r1 weak
#8; SURVEY §8(c) "How each invariant is observed": log[i] = path, written by the hop that
moves chunk i).

With MMA_FAULT_MISROUTE=1 the engine moves path 0's last chunk over path 1 while
mma_get_plan still reports the oracle's plan. For every way a path moves bytes -- the
direct copy engine, a kernel-driven relay ring, an all-copy-engine relay ring, the
zero-copy kernel on v and the zero-copy kernel on a host-ordered private table -- the bytes
stay exact (every chunk is still moved once) and the log must show the misrouted chunk, so
a log that merely echoed the plan would fail here."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

PROG = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
sys.path.insert(0, {root!r} + "/tests")
import paper_2512_16056_b200 as m
import oracle
from gpu_util import configure, pinned

C = 1 << 20
out = {{}}
for name, modes, order, scattered, dirn in {cases!r}:
    configure(m, loopback=1, chunk=C, slots=2, plan_mode=0, hop=(0, 0), host_order=order)
    m.set_path_modes(0, dirn, modes)
    bw = [1, 1]
    m.set_bandwidth(0, dirn, bw)
    nseg, sb = 96, 160 << 10
    B = nseg * sb
    host = pinned(torch, B, seed=0x4D4D41)
    dev = torch.zeros(B, dtype=torch.uint8, device="cuda")
    if dirn == 1:
        dev.copy_(host[:B].cuda())
        host.zero_()
    perm = np.random.default_rng(2).permutation(nseg) if scattered else np.arange(nseg)
    if scattered:
        hp = [host.data_ptr() + int(k) * sb for k in perm]
        dp = [dev.data_ptr() + i * sb for i in range(nseg)]
        segs, n = m.make_segments(*((hp, dp) if dirn == 0 else (dp, hp)), [sb] * nseg)
        (m.memcpy_h2d_segments if dirn == 0 else m.memcpy_d2h_segments)(segs, n, 0)
    elif dirn == 0:
        m.memcpy_h2d(dev, host, B)
    else:
        m.memcpy_d2h(host, dev, B)
    torch.cuda.synchronize()
    h = host.numpy()[:B].reshape(nseg, sb)[perm]
    d = dev.cpu().numpy().reshape(nseg, sb)
    rc, path, _, fb = oracle.plan(bw, B, C, 0, oracle.CONTIG)
    misrouted = path.copy()
    last0 = int(np.nonzero(path == 0)[0][-1])
    misrouted[last0] = 1
    log = np.frombuffer(m.get_delivery_log(0), dtype=np.uint8)
    out[name] = dict(bytes=bool(np.array_equal(h, d)), log_is_plan=bool(np.array_equal(log, path)),
                     log_is_executed=bool(np.array_equal(log, misrouted)),
                     reported_plan_is_oracle=m.get_plan(0, dirn, B)[0] == path.tobytes())
out["sticky"] = m.get_last_error()
print(json.dumps(out))
"""

CE, ZC, P2P = 1, 2, 3
CASES = [
    ("direct_ce+kernel_ring_h2d", [CE, CE], 0, False, 0),
    ("direct_ce+kernel_ring_d2h", [CE, CE], 0, False, 1),
    ("direct_ce+ce_p2p_ring_h2d", [CE, P2P], 0, False, 0),
    ("zc_v+zc_relay_h2d_scattered", [ZC, ZC], 0, True, 0),
    ("zc_private+zc_private_d2h_scattered", [ZC, ZC], 1, True, 1),
    ("zc_private+kernel_ring_d2h_scattered", [ZC, CE], 1, True, 1),
]


def test_log_shows_executed_route(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    script = tmp_path / "m.py"
    script.write_text(PROG.format(root=str(ROOT), cases=CASES))
    env = dict(os.environ, MMA_FAULT_MISROUTE="1", MMA_SPIN_TIMEOUT_MS="8000")
    p = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True, timeout=500)
    assert p.returncode == 0, p.stderr[-3000:]
    r = json.loads(p.stdout.strip().splitlines()[-1])
    assert r.pop("sticky") == 0
    for name, v in r.items():
        assert v["bytes"], (name, v)
        assert v["reported_plan_is_oracle"], (name, v)
        assert not v["log_is_plan"] and v["log_is_executed"], (name, v)
