"""The oracle's steady-state path model (performance, not bytes): pinned by SPEC's worked
numbers (tests/golden/pipeline_model.json) and by a discrete-event simulation written here
that schedules chunk by chunk, independently of the closed forms."""
import json
from pathlib import Path

import pytest

GOLD = json.loads((Path(__file__).parent / "golden" / "pipeline_model.json").read_text())


@pytest.fixture(scope="module")
def orc():
    import oracle
    oracle.lib()
    return oracle


@pytest.mark.parametrize("case", GOLD["direct"], ids=lambda c: c["note"][:12])
def test_direct_rate_golden(orc, case):
    r = orc.direct_rate(case["C"], case["depth"], case["B_gbps"] * 1e9, case["t0_us"] * 1e-6) / 1e9
    assert abs(r - case["rate_gbps"]) <= case.get("tol", 1e-9) + 1e-9, r


@pytest.mark.parametrize("case", GOLD["relay"], ids=lambda c: c["note"][:12])
def test_relay_rate_golden(orc, case):
    r = orc.relay_rate(case["C"], case["streams"], case["Bp_gbps"] * 1e9, case["Bn_gbps"] * 1e9,
                       case["t0_us"] * 1e-6) / 1e9
    assert abs(r - case["rate_gbps"]) <= case.get("tol", 1e-9) + 1e-9, r


def simulate_relay(C, streams, Bp, Bn, t0, n=4000):
    """chunk-by-chunk schedule: the PCIe link serves one hop 1 at a time (setup + transfer),
    NVLink one hop 2 at a time; pipeline k (chunk i on pipeline i mod streams) holds its
    buffer from the start of hop 1 until the end of hop 2"""
    link_free = nv_free = 0.0
    buf_free = [0.0] * streams
    end = 0.0
    for i in range(n):
        k = i % streams
        h1_start = max(link_free, buf_free[k])
        h1_end = h1_start + t0 + C / Bp
        link_free = h1_end
        h2_start = max(h1_end, nv_free)
        h2_end = h2_start + C / Bn
        nv_free = h2_end
        buf_free[k] = h2_end
        end = h2_end
    return n * C / end


def simulate_direct(C, depth, B, t0, n=4000):
    """`depth` slots; a slot does setup (no link) then its transfer (link, one at a time)"""
    link_free = 0.0
    slot_free = [0.0] * depth
    end = 0.0
    for i in range(n):
        k = i % depth
        ready = slot_free[k] + t0
        start = max(ready, link_free)
        link_free = start + C / B
        slot_free[k] = link_free
        end = link_free
    return n * C / end


@pytest.mark.parametrize("streams", [1, 2, 3])
@pytest.mark.parametrize("C", [1 << 20, 5_000_000, 16 << 20])
@pytest.mark.parametrize("Bn", [40e9, 478e9, 900e9])
@pytest.mark.parametrize("t0", [0.0, 4e-6, 50e-6])
def test_relay_rate_matches_simulation(orc, streams, C, Bn, t0):
    Bp = 55e9
    model = orc.relay_rate(C, streams, Bp, Bn, t0)
    sim = simulate_relay(C, streams, Bp, Bn, t0)
    assert abs(model - sim) / model < 0.01, (model, sim)


@pytest.mark.parametrize("depth", [1, 2, 4])
@pytest.mark.parametrize("C", [256 << 10, 1 << 20, 5_000_000])
@pytest.mark.parametrize("t0", [0.0, 4e-6, 50e-6])
def test_direct_rate_matches_simulation(orc, depth, C, t0):
    B = 55e9
    model = orc.direct_rate(C, depth, B, t0)
    sim = simulate_direct(C, depth, B, t0)
    assert abs(model - sim) / model < 0.01, (model, sim)
