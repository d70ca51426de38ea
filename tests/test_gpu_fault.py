"""Failure detection: a dropped hop-1 publish (fault injected with
MMA_FAULT_DROP_PUBLISH) must make the relay kernel's bounded spin expire, set the sticky
error, release the ring so the copy-engine side completes, and leave the process usable
after mma_finalize. Runs in a subprocess (the fault knob is read at engine init)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]

PROG = r"""
import json, sys, time, torch
sys.path.insert(0, {root!r})
import paper_2512_16056_b200 as m
cfg = m.default_config()
cfg.chunk_bytes[0] = cfg.chunk_bytes[1] = 1 << 20
cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = 0
cfg.loopback_relays = {loopback}
if not cfg.loopback_relays:                    # the ring on engine GPU 1 (a peer or a virtual GPU)
    cfg.npaths, cfg.path_gpus[0], cfg.path_gpus[1] = 2, 0, 1
cfg.hop_mode[0] = cfg.hop_mode[1] = m.HOP_CE
cfg.ring_slots = 2
m.init(cfg)
m.set_bandwidth(0, m.H2D, [1, 1])
n = 16 << 20
src = torch.ones(n, dtype=torch.uint8).pin_memory()
dst = torch.zeros(n, dtype=torch.uint8, device="cuda")
t0 = time.time()
m.memcpy_h2d(dst, src, n)
torch.cuda.synchronize()                       # must return: the ring is released
err = m.get_last_error()
try:
    m.memcpy_h2d(dst, src, n)
    refused = False
except m.MMAError as e:
    refused = e.code == err
m.finalize()                                   # recovery: a fresh engine works again
import os; os.environ.pop("MMA_FAULT_DROP_PUBLISH")
m.init(cfg)
m.set_bandwidth(0, m.H2D, [1, 1])
dst.zero_()
m.memcpy_h2d(dst, src, n)
torch.cuda.synchronize()
print(json.dumps(dict(err=err, refused=refused, secs=time.time() - t0, ok=bool(torch.equal(dst.cpu(), src)),
                      err2=m.get_last_error())))
"""


@pytest.mark.parametrize("relay", ["loopback", "relay_gpu"])
def test_dropped_publish_times_out_cleanly(tmp_path, relay):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    script = tmp_path / "f.py"
    script.write_text(PROG.format(root=str(ROOT), loopback=1 if relay == "loopback" else 0))
    env = dict(os.environ, MMA_FAULT_DROP_PUBLISH="3", MMA_SPIN_TIMEOUT_MS="1500")
    if relay != "loopback" and torch.cuda.device_count() < 2:
        env["MMA_VGPUS"] = "2"               # the engine's virtual GPU 1
    p = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True, timeout=240)
    assert p.returncode == 0, p.stderr[-3000:]
    r = json.loads(p.stdout.strip().splitlines()[-1])
    assert r["err"] == 2001 and r["refused"]
    assert r["ok"] and r["err2"] == 0


FAIL_PROG = r"""
import json, sys, torch
sys.path.insert(0, {root!r})
import paper_2512_16056_b200 as m
cfg = m.default_config()
cfg.chunk_bytes[0] = cfg.chunk_bytes[1] = 1 << 20
cfg.fallback_bytes[0] = cfg.fallback_bytes[1] = 0
cfg.loopback_relays = 1
cfg.hop_mode[0] = cfg.hop_mode[1] = m.HOP_CE
m.init(cfg)
m.set_bandwidth(0, m.H2D, [1, 1])          # the direct half is enqueued, then the ring stage fails
n = 512 << 20
src = torch.full((n,), 7, dtype=torch.uint8).pin_memory()
dst = torch.zeros(n, dtype=torch.uint8, device="cuda")
probe = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
try:
    m.memcpy_h2d(dst, src, n, stream=s)
    failed = False
except m.MMAError:
    failed = True
with torch.cuda.stream(s):
    probe.copy_(dst[(n // 2) - (1 << 20):n // 2])   # the tail of the direct half, right after the call
torch.cuda.synchronize()
print(json.dumps(dict(failed=failed, probe_done=bool((probe == 7).all().item()))))
"""


def test_failed_enqueue_still_orders_the_user_stream(tmp_path):
    """a CUDA error while enqueueing (injected after the direct path's DMA was enqueued) is
    returned, and work the user enqueues next on its stream still runs after that DMA"""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    script = tmp_path / "f.py"
    script.write_text(FAIL_PROG.format(root=str(ROOT)))
    env = dict(os.environ, MMA_FAULT_FAIL_RINGS="1")
    p = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True, timeout=240)
    assert p.returncode == 0, p.stderr[-3000:]
    r = json.loads(p.stdout.strip().splitlines()[-1])
    assert r["failed"] and r["probe_done"], r
