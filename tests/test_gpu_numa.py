"""NUMA-affine planning of scattered transfers (north_star (b), reading R23), on one B200 with
the test hooks MMA_FAKE_HOST_NODES (host node = 2 MiB region index mod K) and
MMA_FAKE_PATH_NODES (node per path index): the direct path on node 0, a loopback relay on
node 1. Regrouping the table by node must make (almost) every byte travel on a path of its own
node, against about half without it -- and the bytes must stay exactly the oracle's.

Parity covers WHICH path carried every byte, not only the chunk indices: the engine's
virtual-stream order (mma_get_segment_order) and delivery log give a per-byte path map,
compared with the oracle's: orc_numa_order (the regrouping step, pinned by
tests/test_oracle_numa.py) on the same per-segment nodes, then orc_plan on the regrouped
stream."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
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
                      log=list(mma.get_delivery_log(0)), err=mma.get_last_error(),
                      order=mma.get_segment_order(0).tolist(), host=[int(x) for x in hs])))
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
    # per-byte path maps: engine (its v order + its log) vs oracle (orc_numa_order + orc_plan)
    nseg, sb = 2048, 64 << 10
    seg_node = (np.array(on["host"], dtype=np.uint64) >> np.uint64(21)) % np.uint64(2)
    exp_order = oracle.numa_order(seg_node.astype(np.int32), [1, 1], [0, 1])
    assert on["order"] == exp_order.tolist()
    assert off["order"] == list(range(nseg))              # numa_plan = 0: table order
    for r, order in ((on, exp_order), (off, np.arange(nseg))):
        got = per_byte_paths(np.array(r["order"]), [sb] * nseg, bytes(r["log"]), 1 << 20)
        exp = per_byte_paths(order, [sb] * nseg, path.tobytes(), 1 << 20)
        assert np.array_equal(got, exp)
    # the oracle's map itself: regrouped, > 90% of bytes on a path of their own node
    pmap = per_byte_paths(exp_order, [sb] * nseg, path.tobytes(), 1 << 20).reshape(nseg, sb)
    local = (np.array([0, 1])[pmap] == seg_node.astype(np.int64)[:, None]).mean()
    assert local > 0.9, local


def per_byte_paths(order, lens, log, C):
    """path of every byte of the transfer, in TABLE order: v holds the table's segments in
    `order`, and byte y of v rides log[y // C]"""
    lens = np.asarray(lens, dtype=np.int64)
    vlen = lens[order]
    vstart = np.concatenate([[0], np.cumsum(vlen)])
    pbv = np.repeat(np.frombuffer(log, dtype=np.uint8), C)[: vstart[-1]]
    tstart = np.concatenate([[0], np.cumsum(lens)])
    out = np.empty(int(tstart[-1]), dtype=np.uint8)
    for k, t in enumerate(order):
        out[tstart[t]:tstart[t + 1]] = pbv[vstart[k]:vstart[k + 1]]
    return out
