"""CPU checks of bench.py's host-side helpers (the round-end runs depend on them): the
clock sampler's parser, the trace summary, the oracle CPU baseline and the JSON line of the
reference arm."""
import json
import subprocess
import sys
from pathlib import Path

import bench

ROOT = Path(__file__).resolve().parents[1]


class _FakeProc:
    def __init__(self, out):
        self.out = out

    def terminate(self):
        pass

    def communicate(self, timeout=None):
        return self.out, ""


def test_clock_parser():
    c = bench.Clocks([0, 1])
    c.p = _FakeProc("0, 1965, 1965, 250.1, 0x0, Not Active, Not Active, Not Active, Not Active\n"
                    "1, 1950, 1965, 260.0, 0x4, Not Active, Not Active, Not Active, Active\n"
                    "garbage line\n")
    r = c.stop()
    assert r["sm_mhz"] == 1957.5 and r["sm_max_mhz"] == 1965.0 and r["samples"] == 2
    assert r["reasons"] == ["sw_power_cap"]
    c2 = bench.Clocks([0])
    c2.p = None
    assert c2.stop()["sm_mhz"] is None


def test_timeline_summary(tmp_path):
    ev = [{"name": "a", "ph": "X", "pid": "GPU 0", "tid": "x", "ts": 0.0, "dur": 10.0, "args": {}},
          {"name": "b", "ph": "X", "pid": "GPU 0", "tid": "y", "ts": 5.0, "dur": 10.0, "args": {}},
          {"name": "c", "ph": "X", "pid": "GPU 1", "tid": "x", "ts": 0.0, "dur": 20.0, "args": {}}]
    p = tmp_path / "t.json"
    p.write_text(json.dumps({"traceEvents": ev}))
    s = bench.timeline_summary(str(p))
    assert s["span_us"] == 20.0 and s["busy_us"] == {"GPU 0": 15.0, "GPU 1": 20.0}
    assert s["mean_gpus_busy"] == 1.75 and s["spans"] == 3
    p.write_text(json.dumps({"traceEvents": []}))
    assert bench.timeline_summary(str(p)) is None


def test_oracle_sample_bounded():
    g, threads, desc, nbytes, dt = bench.oracle_sample(2, nsegs_sample=256, reps=2)
    assert g > 0 and threads == 3 and nbytes == 2 * 256 * 32768 and dt > 0
    assert "256 of 131072" in desc


def test_cpu_baseline_legs(monkeypatch):
    """cpu_baseline: the oracle at the bench's path threads and at ~nproc threads, with the
    CPU model (SURVEY 8(d) "Oracle timing alongside")"""
    monkeypatch.setattr(bench.os, "cpu_count", lambda: 5)
    c = bench.cpu_baseline(1, nsegs_sample=128, seconds_per_leg=0.05)
    assert [leg["threads"] for leg in c["legs"]] == [1, 5]      # 1 path; (5 + 1) // 2 = 3 paths -> 5 threads
    assert c["value"] == c["legs"][0]["gbps"] and c["cores"] == 1 and c["nproc"] == 5
    assert c["kind"] == "oracle" and "cpu_model" in c


def test_reference_arm_line():
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=str(ROOT))
    assert p.returncode == 0, p.stderr[-2000:]
    j = json.loads(p.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in j, key
    assert j["impl"] == "reference" and j["metric"] == bench.METRIC


def test_widen_visible(monkeypatch):
    class D:
        world = 4
    monkeypatch.setenv("CUDA_VISIBLE_DEVICES", "4")
    note = bench.widen_visible(D(), ["4", "5", "6", "7"])
    import os
    assert os.environ["CUDA_VISIBLE_DEVICES"] == "4,5,6,7" and "widened" in note
    monkeypatch.setenv("CUDA_VISIBLE_DEVICES", "0,1,2,3")
    assert bench.widen_visible(D(), ["0,1,2,3"] * 4) is None             # already sees the job's GPUs
    monkeypatch.delenv("CUDA_VISIBLE_DEVICES")
    assert bench.widen_visible(D(), [None] * 4) is None                  # unrestricted


def test_pcie_counter_unwrap():
    """The NVML PCIe counters are 32-bit: the sampler adds deltas modulo 2^32."""
    import threading
    c = bench.PcieCounters.__new__(bench.PcieCounters)
    seq = iter([[4_000_000_000, 10], [100, 20], [4_294_967_000, 30]])
    c._read = lambda h: next(seq)
    c.h = [object()]
    c.last = [[3_000_000_000, 0]]
    c.tot = [[0, 0]]
    c.lock = threading.Lock()
    assert c.mark() == [[1_000_000_000, 10]]
    assert c.mark() == [[1_000_000_000 + 294_967_396, 20]]
    assert c.mark() == [[1_000_000_000 + 294_967_396 + 4_294_966_900, 30]]


def test_committed_bench_line_has_the_contract_keys():
    """the committed bench line (profiles/r01_bench.json) carries every key the driver's
    contract names, with the types it expects"""
    import json
    from pathlib import Path
    d = json.loads((Path(__file__).resolve().parents[1] / "profiles" / "r02_bench.json").read_text())
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["value"] > 0 and d["steps"] >= 1 and d["warmup"] >= 3 and d["higher_is_better"] is True
    assert "workload" in d["config"]
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    c = d["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in c, k
    assert c["kind"] == "oracle" and c["cores"] >= 1
    assert len(c["legs"]) >= 1 and c["nproc"] >= 1 and "cpu_model" in c     # round 2: both thread legs
    e = d["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e, k
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in d["clocks"], k


def test_engine_gpu_indices_map_to_torch_devices(monkeypatch):
    """virtual-GPU mode (MMA_VGPUS): the bench drives more engine GPUs than
    torch sees and places a virtual GPU's buffers and streams on device g mod count; with
    the variable unset (or not above the device count) every index is its own device"""
    import torch
    monkeypatch.setattr(torch.cuda, "device_count", lambda: 2)
    monkeypatch.delenv("MMA_VGPUS", raising=False)
    assert bench.engine_gpus(torch) == 2
    assert [bench.cdev(g) for g in range(2)] == [0, 1]
    monkeypatch.setenv("MMA_VGPUS", "2")
    assert bench.engine_gpus(torch) == 2
    monkeypatch.setenv("MMA_VGPUS", "8")
    assert bench.engine_gpus(torch) == 8
    assert [bench.cdev(g) for g in range(8)] == [0, 1, 0, 1, 0, 1, 0, 1]
    monkeypatch.setattr(torch.cuda, "device_count", lambda: 0)     # no GPU: nothing to map
    assert bench.engine_gpus(torch) == 0 and bench.cdev(3) == 3
