"""Multi-process mode: two processes (gloo world size 2) share one GPU here;
the target process exports its destination with CUDA IPC, the host pool is shared memory,
and each process moves its share of a scattered KV fetch -- planned (mma_plan_chunks +
mma_copy_share_segments) and dynamic (mma_copy_claim_segments on an IPC-shared cursor).
The target checks every byte on the device against the seeded pattern."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]

WORKER = r"""
import json, os, sys
sys.path.insert(0, {root!r})
import numpy as np, torch, torch.distributed as dist
import paper_2512_16056_b200 as mma
import mma_inputs
from mma_inputs import workloads as W
rank = int(os.environ["RANK"]); dist.init_process_group("gloo")
torch.cuda.set_device(0)
shape = W.scaled_kv(1024); ho, do, sb, hpool, dbytes = W.kv_segments(shape)
name = "mp_test_" + os.environ["MASTER_PORT"]; seed = 91
if rank == 0:
    pool = mma.shared_host_alloc(name, hpool, True)
    mma.host_array(pool, hpool)[:] = mma_inputs.pattern_bytes(seed, hpool)
    dst = torch.zeros(dbytes, dtype=torch.uint8, device="cuda")
    ctr = torch.zeros(32, dtype=torch.int64, device="cuda")
    obj = [(mma.ipc_export(dst), mma.ipc_export(ctr))]
else:
    obj = [None]
dist.barrier()
dist.broadcast_object_list(obj, src=0)
(hd, od), (hc, oc) = obj[0]
if rank == 1:
    pool = mma.shared_host_alloc(name, hpool, False)
    dptr = mma.ipc_open(hd, od, 0); cptr = mma.ipc_open(hc, oc, 0)
else:
    dptr, cptr = dst.data_ptr(), ctr.data_ptr()
lens = np.full(len(ho), sb, dtype=np.int64)
segs, n = mma.make_segments(pool + ho, dptr + do, lens)
B = int(lens.sum()); C = 1 << 20
rc, path, fb = mma.plan_chunks([3, 1], [0, 1], B, C, 0, 1)
s = torch.cuda.Stream()
mma.copy_share_segments(segs, n, C, path, rank, 0, stream=s)
s.synchronize(); dist.barrier()
res = {{}}
if rank == 0:
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    mma.verify_segments(dst.data_ptr() + do, ho, lens, seed, cnt); torch.cuda.synchronize()
    res["planned_mismatch"] = int(cnt.item())
    dst.zero_(); ctr.zero_(); torch.cuda.synchronize()
dist.barrier()
mma.copy_claim_segments(segs, n, 256 << 10, cptr, cptr + 8, rank, 0, stream=s)
s.synchronize(); dist.barrier()
if rank == 0:
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    mma.verify_segments(dst.data_ptr() + do, ho, lens, seed, cnt); torch.cuda.synchronize()
    res["dynamic_mismatch"] = int(cnt.item())
    counts = ctr.cpu().tolist()
    res["claims"] = counts[1:3]; res["nclaims"] = (B + (256 << 10) - 1) // (256 << 10)
    res["err"] = mma.get_last_error()
dist.barrier()
# cross-process ledger: rank 1's share, held behind a sleeping kernel, is visible to rank 0
led = "mpled_" + os.environ["MASTER_PORT"]
mma.ledger_attach(led)
bus = mma.device_bus_id(0)
if rank == 1:
    with torch.cuda.stream(s):
        torch.cuda._sleep(1_500_000_000)
    mma.copy_share_segments(segs, n, C, path, 1, 0, stream=s)
dist.barrier()
if rank == 0:
    res["ledger_in_flight"] = list(mma.ledger_shared_get(bus, mma.H2D))
    res["share1_bytes"] = sum(min(C, B - i * C) for i in range(len(path)) if path[i] == 1)
dist.barrier()
s.synchronize(); dist.barrier()
if rank == 0:
    res["ledger_after"] = list(mma.ledger_shared_get(bus, mma.H2D))
    print(json.dumps(res), flush=True)
dist.barrier()
mma.ledger_attach(None)
if rank == 0:
    mma.ledger_unlink(led)
dist.barrier()
if rank == 1:
    mma.ipc_close(dptr); mma.ipc_close(cptr); mma.shared_host_free(pool)
dist.barrier()
if rank == 0:
    mma.shared_host_free(pool, name)
dist.destroy_process_group()
"""


def test_two_processes_share_a_transfer(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    script = tmp_path / "w.py"
    script.write_text(WORKER.format(root=str(ROOT)))
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK=str(r),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=280) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-3000:]
    r = json.loads(outs[0][0].strip().splitlines()[-1])
    assert r["planned_mismatch"] == 0 and r["dynamic_mismatch"] == 0 and r["err"] == 0
    assert sum(r["claims"]) == r["nclaims"]
    assert r["ledger_in_flight"] == [r["share1_bytes"], 0] and r["share1_bytes"] > 0   # a relay share: not own
    assert r["ledger_after"] == [0, 0]


RING_WORKER = r"""
import json, os, sys
sys.path.insert(0, {root!r})
import numpy as np, torch, torch.distributed as dist
import paper_2512_16056_b200 as mma
import mma_inputs
from mma_inputs import workloads as W
rank = int(os.environ["RANK"]); dist.init_process_group("gloo")
torch.cuda.set_device(0)
shape = W.scaled_kv(1024); ho, do, sb, hpool, dbytes = W.kv_segments(shape)
name = "mpring_" + os.environ["MASTER_PORT"]; seed = 93
if rank == 0:
    pool = mma.shared_host_alloc(name, hpool, True)
    mma.host_array(pool, hpool)[:] = mma_inputs.pattern_bytes(seed, hpool)
    dst = torch.zeros(dbytes, dtype=torch.uint8, device="cuda")
    obj = [mma.ipc_export(dst)]
else:
    obj = [None]
dist.barrier()
dist.broadcast_object_list(obj, src=0)
hd, od = obj[0]
if rank == 1:
    pool = mma.shared_host_alloc(name, hpool, False)
    dptr = mma.ipc_open(hd, od, 0)
else:
    dptr = dst.data_ptr()
lens = np.full(len(ho), sb, dtype=np.int64)
B = int(lens.sum()); C = 1 << 20
rc, path, fb = mma.plan_chunks([1, 2], [0, 1], B, C, 0, 1)
s = torch.cuda.Stream()
res = {{}}
# H2D: rank 0 moves path 0's chunks with its zero-copy kernel, rank 1 moves path 1's through
# ITS OWN copy-engine ring (hop 1 into its staging slots, hop 2 a DMA into rank 0's memory)
segs, n = mma.make_segments(pool + ho, dptr + do, lens)
for rep in range(2):                                          # the second pass reuses the slots
    if rank == 0:
        mma.copy_share_segments(segs, n, C, path, 0, 0, stream=s)
    else:
        mma.copy_share_segments_ring(segs, n, C, path, 1, 0, slots=3, stream=s)
    s.synchronize(); dist.barrier()
    if rank == 0:
        got = dst.cpu().numpy()
        exp = np.zeros(dbytes, np.uint8)
        import oracle
        oh = mma.host_array(pool, hpool)
        osegs, on = oracle.segments_from_arrays(oh.ctypes.data + ho, exp.ctypes.data + do, lens)
        assert oracle.move(osegs, on, C, [1, 2], np.frombuffer(path, np.uint8).copy(), S=3) == 0
        res[f"h2d_equal_{{rep}}"] = bool(np.array_equal(got, exp))
        dst.zero_(); torch.cuda.synchronize()
    dist.barrier()
# D2H: the cache (rank 0's GPU memory) back into fresh host slots, rank 1's ring doing hop 1
# as a device-to-device copy out of rank 0's memory
if rank == 0:
    mma.fill_pattern(dst, dbytes, seed + 1, 0); torch.cuda.synchronize()
    mma.host_array(pool, hpool)[:] = 0
dist.barrier()
segs2, n2 = mma.make_segments(dptr + do, pool + ho, lens)
if rank == 0:
    mma.copy_share_segments(segs2, n2, C, path, 0, 0, stream=s)
else:
    mma.copy_share_segments_ring(segs2, n2, C, path, 1, 0, slots=2, stream=s)
s.synchronize(); dist.barrier()
if rank == 0:
    h = mma.host_array(pool, hpool)
    src = dst.cpu().numpy()
    ok = all(np.array_equal(h[ho[k]:ho[k] + sb], src[do[k]:do[k] + sb]) for k in range(len(ho)))
    untouched = np.ones(hpool, bool)
    for k in range(len(ho)):
        untouched[ho[k]:ho[k] + sb] = False
    res["d2h_equal"] = bool(ok and not h[untouched].any())
    res["err"] = mma.get_last_error()
    print(json.dumps(res), flush=True)
dist.barrier()
if rank == 1:
    mma.ipc_close(dptr); mma.shared_host_free(pool)
dist.barrier()
if rank == 0:
    mma.shared_host_free(pool, name)
dist.destroy_process_group()
"""


def test_share_through_another_process_ring(tmp_path):
    """NEXT-4 (§5.1.2, one multipath queue per process): a transfer owned by process 0
    moves partly through process 1's copy-engine relay ring (its staging slots, its streams),
    H2D and D2H, byte-exact against the oracle moving the same plan"""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    script = tmp_path / "ring.py"
    script.write_text(RING_WORKER.format(root=str(ROOT)))
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", LOCAL_RANK=str(r),
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env, stdout=subprocess.PIPE,
                                      stderr=subprocess.PIPE, text=True))
    outs = [p.communicate(timeout=280) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-3000:]
    r = json.loads(outs[0][0].strip().splitlines()[-1])
    assert r["h2d_equal_0"] and r["h2d_equal_1"] and r["d2h_equal"] and r["err"] == 0, r
