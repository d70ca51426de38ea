"""Topology probe: P2P matrix, NUMA node, copy engines and SMs per GPU as
the engine sees them, checked against torch's own view of the devices."""
import re

import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(120)]


def test_topology_matches_the_devices():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2512_16056_b200 as mma
    t = mma.get_topology()
    n = torch.cuda.device_count()
    assert t["ngpu"] == min(n, 16)
    for a in range(t["ngpu"]):
        pr = torch.cuda.get_device_properties(a)
        assert t["sms"][a] == pr.multi_processor_count
        assert t["copy_engines"][a] >= 1
        assert re.fullmatch(r"[0-9A-Fa-f]{4,8}:[0-9A-Fa-f]{2}:[0-9A-Fa-f]{2}\.[0-9]", t["bus_id"][a]), t["bus_id"][a]
        assert int(t["bus_id"][a].split(":")[1], 16) == pr.pci_bus_id
        assert t["p2p"][a][a] == 0
        for b in range(t["ngpu"]):
            if a != b:
                assert t["p2p"][a][b] == int(torch.cuda.can_device_access_peer(a, b))
        assert -1 <= t["numa_node"][a] < max(1, t["host_numa_nodes"])
    assert t["host_numa_nodes"] >= 1
