"""Relay rings under serialised launches and mid-ring failures (ADVICE
r1 #1).

The engine enqueues a ring's work in waves of at most S chunks (plane.cpp enqueue_rings):
for H2D the hops of a wave precede its pull kernel, for D2H the pack kernel precedes the
hops, so every wait depends only on work enqueued before it (§3.4.3: "an H2D
operation and a P2P operation ... with a dependency established between these
operations"). With CUDA_LAUNCH_BLOCKING=1 each kernel launch returns only once the kernel
has finished -- a kernel that waited on hops enqueued after it would spin into its timeout.
Here the spin timeout is cut to 3 s, so any such wait shows as the sticky error, not as a
slow pass.

A hop that fails in the middle of a call (MMA_FAULT_FAIL_HOP) must leave the ring usable:
the failed call's rings are marked broken and remade by the next call, which must copy
byte-exactly with the oracle's plan."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

PROG = r"""
import json, sys, time
import numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2512_16056_b200 as m
import mma_inputs, oracle
sys.path.insert(0, {root!r} + "/tests")
from gpu_util import configure, pinned, guarded_device, guarded_host, G

out = {{}}
C = 1 << 20
S = {slots}
configure(m, chunk=C, slots=S, plan_mode=1, hop=(1, 1), ctas=4, **{relays})
bw = [2, 3, 3]
m.set_bandwidth(0, m.H2D, bw)
m.set_bandwidth(0, m.D2H, bw)
B = 23 * C + 12345                       # several waves per ring and a ragged tail
t0 = time.time()
for rep in range(2):                     # the second call starts mid-ring (base > 0)
    src = pinned(torch, B, seed=0x4D4D41 + rep)
    dst = guarded_device(torch, B)
    m.memcpy_h2d(dst[G:G + B], src, B)
    torch.cuda.synchronize()
    rc, path, _, fb = oracle.plan(bw, B, C, 0, oracle.INTERLEAVED)
    exp = guarded_host(B)
    assert oracle.move_contiguous(exp[G:G + B], src.numpy()[:B], C, bw, path, S=S) == 0
    out[f"h2d{{rep}}_bytes"] = bool(np.array_equal(dst.cpu().numpy(), exp))
    out[f"h2d{{rep}}_log"] = m.get_delivery_log(0) == path.tobytes()
    # D2H of a device pattern into a guarded pinned buffer
    dsrc = torch.empty(B, dtype=torch.uint8, device="cuda")
    m.fill_pattern(dsrc, B, 0x5151 + rep, 0)
    host = pinned(torch, B + 2 * G)
    host.fill_(0xA5)
    m.memcpy_d2h(host[G:G + B], dsrc, B)
    torch.cuda.synchronize()
    exp2 = guarded_host(B)
    assert oracle.move_contiguous(exp2[G:G + B], dsrc.cpu().numpy(), C, bw, path, S=S) == 0
    out[f"d2h{{rep}}_bytes"] = bool(np.array_equal(host.numpy(), exp2))
    out[f"d2h{{rep}}_log"] = m.get_delivery_log(0) == path.tobytes()
# a scattered transfer (C3) through the same rings
segs = 37
sb = 96 << 10
hsrc = pinned(torch, segs * sb, seed=0x77)
perm = np.random.default_rng(5).permutation(segs)
cache = guarded_device(torch, segs * sb)
base = cache.data_ptr() + G
table = m.make_segments([hsrc.data_ptr() + int(k) * sb for k in perm],
                        [base + i * sb for i in range(segs)], [sb] * segs)
m.memcpy_h2d_segments(*table, 0)
torch.cuda.synchronize()
got = cache.cpu().numpy()
ok = all(np.array_equal(got[G + i * sb:G + (i + 1) * sb], hsrc.numpy()[int(k) * sb:(int(k) + 1) * sb])
         for i, k in enumerate(perm))
out["seg_bytes"] = bool(ok and (got[:G] == 0xA5).all() and (got[G + segs * sb:] == 0xA5).all())
out["sticky"] = m.get_last_error()
out["secs"] = time.time() - t0
print(json.dumps(out))
"""


def _relays(kind):
    """two relay paths: loopback rings on GPU 0, or rings on engine GPUs 1 and 2 (real peers
    when the box has three GPUs, else the engine's virtual GPUs): then the
    D2H pack kernel runs on the relay GPU and the hops on the relay's own streams"""
    import torch
    if kind == "loopback":
        return "dict(loopback=2)", {}
    env = {"MMA_VGPUS": "3"} if torch.cuda.device_count() < 3 else {}
    return "dict(loopback=0, paths=[0, 1, 2])", env


@pytest.mark.parametrize("relays", ["loopback", "relay_gpus"])
@pytest.mark.parametrize("slots", [1, 2, 4])
def test_rings_complete_with_serialised_launches(tmp_path, slots, relays):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    script = tmp_path / "s.py"
    rel, renv = _relays(relays)
    script.write_text(PROG.format(root=str(ROOT), slots=slots, relays=rel))
    env = dict(os.environ, CUDA_LAUNCH_BLOCKING="1", MMA_SPIN_TIMEOUT_MS="3000", PYTHONPATH=str(ROOT), **renv)
    p = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True, timeout=500)
    assert p.returncode == 0, p.stderr[-3000:]
    r = json.loads(p.stdout.strip().splitlines()[-1])
    assert r["sticky"] == 0, r
    assert all(v for k, v in r.items() if k not in ("sticky", "secs")), r


FAULT_PROG = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import paper_2512_16056_b200 as m
import oracle
sys.path.insert(0, {root!r} + "/tests")
from gpu_util import configure, pinned, guarded_device, guarded_host, G

C = 1 << 20
S = 2
configure(m, chunk=C, slots=S, plan_mode=1, hop=({hop}, {hop}), ctas=4, **{relays})
bw = [1, 1, 1]
m.set_bandwidth(0, m.H2D, bw)
m.set_bandwidth(0, m.D2H, bw)
B = 24 * C
src = pinned(torch, B, seed=0x4D4D41)
dst = guarded_device(torch, B)
s = torch.cuda.Stream()
torch.cuda.synchronize()
out = {{}}
{direction_code}
out["sticky"] = m.get_last_error()
print(json.dumps(out))
"""

H2D_CODE = r"""
try:
    m.memcpy_h2d(dst[G:G + B], src, B, stream=s)      # the 6th hop of the engine fails
    out["failed"] = False
except m.MMAError:
    out["failed"] = True
s.synchronize()                                      # the partial call drains (no hang)
for rep in range(2):                                 # the broken rings are remade
    dst.fill_(0xA5)
    torch.cuda.synchronize()
    m.memcpy_h2d(dst[G:G + B], src, B, stream=s)
    s.synchronize()
    rc, path, _, fb = oracle.plan(bw, B, C, 0, oracle.INTERLEAVED)
    exp = guarded_host(B)
    assert oracle.move_contiguous(exp[G:G + B], src.numpy()[:B], C, bw, path, S=S) == 0
    out[f"bytes{rep}"] = bool(np.array_equal(dst.cpu().numpy(), exp))
    out[f"log{rep}"] = m.get_delivery_log(0) == path.tobytes()
"""

D2H_CODE = r"""
dsrc = dst[G:G + B]
m.fill_pattern(dsrc, B, 0x99, 0)
torch.cuda.synchronize()
host = pinned(torch, B + 2 * G)
try:
    m.memcpy_d2h(host[G:G + B], dsrc, B, stream=s)
    out["failed"] = False
except m.MMAError:
    out["failed"] = True
s.synchronize()
for rep in range(2):
    host.fill_(0xA5)
    m.memcpy_d2h(host[G:G + B], dsrc, B, stream=s)
    s.synchronize()
    rc, path, _, fb = oracle.plan(bw, B, C, 0, oracle.INTERLEAVED)
    exp = guarded_host(B)
    assert oracle.move_contiguous(exp[G:G + B], dsrc.cpu().numpy(), C, bw, path, S=S) == 0
    out[f"bytes{rep}"] = bool(np.array_equal(host.numpy(), exp))
    out[f"log{rep}"] = m.get_delivery_log(0) == path.tobytes()
"""


@pytest.mark.parametrize("relays", ["loopback", "relay_gpus"])
@pytest.mark.parametrize("direction", ["h2d", "d2h"])
@pytest.mark.parametrize("hop", [1, 3], ids=["kernel_ring", "ce_p2p_ring"])
def test_hop_failure_mid_call_poisons_and_remakes_rings(tmp_path, direction, hop, relays):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    script = tmp_path / "f.py"
    code = H2D_CODE if direction == "h2d" else D2H_CODE
    rel, renv = _relays(relays)
    script.write_text(FAULT_PROG.format(root=str(ROOT), hop=hop, direction_code=code, relays=rel))
    env = dict(os.environ, MMA_FAULT_FAIL_HOP="5", MMA_SPIN_TIMEOUT_MS="5000", PYTHONPATH=str(ROOT), **renv)
    p = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-3000:]
    r = json.loads(p.stdout.strip().splitlines()[-1])
    assert r["failed"], r
    assert r["sticky"] == 0, r
    assert r["bytes0"] and r["log0"] and r["bytes1"] and r["log1"], r
