"""Deployment CLI (python -m paper_2512_16056_b200): show, calibrate -> file -> load at init
(MMA_CALIB), plan. Runs in subprocesses, as an operator would."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]


def _run(args, env=None):
    p = subprocess.run([sys.executable, "-m", "paper_2512_16056_b200", *args], cwd=str(ROOT), capture_output=True,
                       text=True, timeout=240, env=dict(os.environ, **(env or {})))
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


def test_cli_show_calibrate_plan(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    show = _run(["show"])
    assert show["topology"]["ngpu"] >= 1 and "0" in show["paths"]
    cal = tmp_path / "cal.txt"
    env = {"MMA_LOOPBACK": "1"}          # two paths on one GPU, so the file has relay lines
    out = _run(["calibrate", "--out", str(cal), "--devices", "0", "--bytes", str(64 << 20)], env)
    rates = out["calibration"]["0"]["h2d"]["rates"]
    assert len(rates) == 2 and all(r["solo"] > 0 for r in rates)
    assert cal.exists() and len([ln for ln in cal.read_text().splitlines() if not ln.startswith("#")]) >= 4
    # a fresh process loads the file at init: its vector is the calibrated one
    plan = _run(["plan", "--device", "0", "--bytes", str(1 << 30)], dict(env, MMA_CALIB=str(cal)))
    assert [p["mbps"] for p in plan["paths"]] == [p["mbps"] for p in out["calibration"]["0"]["h2d"]["paths"]]
    assert sum(plan["chunks_per_path"].values()) == plan["nchunks"]


def test_env_pinned_bandwidth():
    """MMA_BW pins the planner's vector from the environment (parity runs): the
    plan a fresh process reports is the oracle's plan for that vector"""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    env = {"MMA_LOOPBACK": "2", "MMA_BW": "3000,2000,1000", "MMA_PLAN_MODE": "1", "MMA_FALLBACK_BYTES": "0",
           "MMA_CHUNK_BYTES": str(1 << 20)}
    out = _run(["plan", "--device", "0", "--bytes", str(37 << 20)], env)
    assert [p["mbps"] for p in out["paths"]] == [3000, 2000, 1000]
    rc, path, counts, fb = oracle.plan([3000, 2000, 1000], 37 << 20, 1 << 20, 0, 1)
    assert out["chunks_per_path"] == {str(p): int(c) for p, c in enumerate(counts) if c}
