import os
import sys
from pathlib import Path

import pytest

# the engine raises the hardware queue count in its load constructor, which only takes
# effect if it runs before the process's first CUDA context; a test module that touches
# CUDA before importing the package would otherwise leave the whole session at 8 queues
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.lib()
    return oracle
