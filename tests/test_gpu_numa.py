"""NUMA-affine planning of scattered transfers (north_star (b), reading R23), on one B200 with
the test hooks MMA_FAKE_HOST_NODES (host node = 2 MiB region index mod K) and
MMA_FAKE_PATH_NODES (node per path index): the direct path on node 0, a loopback relay on
node 1. Regrouping the table by node must make (almost) every byte travel on a path of its own
node, against about half without it -- and the bytes must stay exactly the oracle's."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]

PROG = r"""
import json, sys
sys.path.insert(0, {root!r})
import numpy as np, torch
import paper_2512_16056_b200 as mma
import oracle
from gpu_util import configure
torch.cuda.init()
dirn = {dirn}
configure(mma, loopback=1, chunk=1 << 20, slots=4, plan_mode=0, hop=(1, 2), debug=1)
mma.set_bandwidth(0, dirn, [1, 1])
nseg, sb = 2048, 64 << 10                      # 128 MiB of 64 KiB blocks in a 256 MiB pool
rng = np.random.default_rng(17)
slots = rng.permutation(2 * nseg)[:nseg]
pool = torch.empty(2 * nseg * sb, dtype=torch.uint8).pin_memory()
pool.numpy()[:] = rng.integers(0, 256, pool.numel(), dtype=np.uint8)
dev = torch.empty(nseg * sb, dtype=torch.uint8, device="cuda")
if dirn == 1:
    dev.copy_(torch.from_numpy(rng.integers(0, 256, dev.numel(), dtype=np.uint8)).cuda())
    src_host = dev.cpu().numpy()
hs = [pool.data_ptr() + int(s) * sb for s in slots]
ds = [dev.data_ptr() + k * sb for k in range(nseg)]
segs, n = mma.make_segments(hs, ds, [sb] * nseg) if dirn == 0 else mma.make_segments(ds, hs, [sb] * nseg)
mma.reset_stats(0)
(mma.memcpy_h2d_segments if dirn == 0 else mma.memcpy_d2h_segments)(segs, n, 0)
torch.cuda.synchronize()
st = mma.get_stats(0)
if dirn == 0:
    ok = bool(np.array_equal(dev.cpu().numpy().reshape(nseg, sb), pool.numpy().reshape(2 * nseg, sb)[slots]))
else:
    ok = bool(np.array_equal(pool.numpy().reshape(2 * nseg, sb)[slots], src_host.reshape(nseg, sb)))
print(json.dumps(dict(ok=ok, known=st["numa_known_bytes"][dirn], local=st["numa_local_bytes"][dirn],
                      log=list(mma.get_delivery_log(0)), err=mma.get_last_error())))
"""


def _run(tmp_path, dirn, numa_plan):
    script = tmp_path / f"n{dirn}{numa_plan}.py"
    script.write_text(PROG.format(root=str(ROOT), dirn=dirn))
    env = dict(os.environ, MMA_FAKE_HOST_NODES="2", MMA_FAKE_PATH_NODES="0,1", MMA_NUMA_PLAN=str(numa_plan),
               PYTHONPATH=str(ROOT / "tests"))
    p = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True, timeout=240)
    assert p.returncode == 0, p.stderr[-3000:]
    import json
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("dirn", [0, 1], ids=["h2d", "d2h"])
def test_node_affine_plan(tmp_path, dirn):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    on, off = _run(tmp_path, dirn, 1), _run(tmp_path, dirn, 0)
    B = 2048 * (64 << 10)
    rc, path, _, _ = oracle.plan([1, 1], B, 1 << 20, 0, 0)
    for r in (on, off):
        assert r["ok"] and r["err"] == 0 and r["known"] == B
        assert bytes(r["log"]) == path.tobytes()          # the plan is the oracle's either way
    assert on["local"] / B > 0.9, on["local"] / B        # regrouped: bytes travel on their node
    assert 0.35 < off["local"] / B < 0.65, off["local"] / B   # table order: about half
