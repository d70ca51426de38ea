"""bench.py modes beyond the default line, at small sizes, each must print one parseable
contract line (--engine-modes, --mp and --workload contention were
exercised only by hand). Also the N = 2 torchrun launch the driver uses for its scaling
runs, on whatever GPUs this box has (rank 0 drives every path GPU, rank 1 idles)."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(900)]


def _line(out):
    lines = [ln for ln in out.strip().splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def _bench(args, torchrun=0, timeout=700, env_extra=None):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, MMA_SPIN_TIMEOUT_MS="8000", **(env_extra or {}))
    if torchrun:
        s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={torchrun}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", "bench.py", *args]
    else:
        cmd = [sys.executable, "bench.py", *args]
    p = subprocess.run(cmd, cwd=str(ROOT), capture_output=True, text=True, timeout=timeout, env=env)
    assert p.returncode == 0, (p.stdout[-2000:], p.stderr[-3000:])
    r = _line(p.stdout)
    assert r.get("value") and r["value"] > 0 and "error" not in r, r
    return r


def test_contention_workload():
    r = _bench(["--workload", "contention", "--contention-scale", "0.02", "--steps", "2", "--warmup", "1"])
    assert r["native"]["gbps"] > 0 and r["per_call_ledger"]["gbps"] > 0


def test_engine_modes_kv():
    r = _bench(["--engine-modes", "--tokens", "2048", "--steps", "2", "--warmup", "3", "--quick"])
    assert r["verify"]["mismatched_bytes"] == 0


def test_contig_with_loopback_relay():
    r = _bench(["--workload", "contig", "--bytes", str(256 << 20), "--loopback", "1", "--hop", "1",
                "--steps", "2", "--warmup", "3", "--quick"])
    assert r["gpu_launches"] > 0 and 1 in r["kernel_kinds"]      # the relay pull kernel ran


def test_mp_two_ranks():
    r = _bench(["--mp", "--gpus", "2", "--tokens", "2048", "--steps", "2", "--warmup", "3"], torchrun=2)
    assert r["n_gpus"] == 2


def test_torchrun_two_ranks_default_line():
    r = _bench(["--gpus", "2", "--tokens", "2048", "--steps", "2", "--warmup", "3", "--quick"], torchrun=2)
    assert r["n_gpus"] == 2 and r["verify"]["mismatched_bytes"] == 0


def test_torchrun_four_ranks_virtual_gpus():
    """the driver's N = 4 scaling launch with k = 4 paths into GPU 0 -- per-path tuning, the
    concurrent calibration, the k = 1 / 2 re-runs (per_path_count), NVML counters and the
    multi-path roofline -- end to end; on a one-GPU box through the engine's virtual GPUs
    (MMA_VGPUS), where the four paths share one link"""
    import torch
    extra = {"MMA_VGPUS": "4"} if torch.cuda.is_available() and torch.cuda.device_count() < 4 else {}
    r = _bench(["--gpus", "4", "--tokens", "2048", "--steps", "2", "--warmup", "3"], torchrun=4,
               env_extra=extra)
    assert r["n_gpus"] == 4 and r["config"]["paths"] == 4 and r["verify"]["mismatched_bytes"] == 0
    assert r["config"]["multipath_error"] is None
    # a planned step counts its relay bytes at enqueue; a dynamic-pull step's split is known
    # only on the device (mma_get_dynamic_counts), so the stat stays 0 there
    assert r["engine"]["relay_bytes"] > 0 or r["plan"]["chosen"] == "dynamic"
    assert set(r["per_path_count"]) == {"1", "2", "4"}
