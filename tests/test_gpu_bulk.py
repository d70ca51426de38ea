"""The cp.async.bulk (TMA) forms. Relay kernels: the opt-in form (MMA_RELAY_BULK=1; SURVEY §8(a) a6 "or
stage through shared memory / cp.async.bulk"): the ring parity, forward-log and random-soak
modules run again with it in a fresh process (the knob is read at engine init), so every
check there -- bytes with guard bands, plan, delivery log, the flag each forward rested on --
covers the bulk form too."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(1500)]


def test_ring_modules_with_bulk_relay_kernels():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, MMA_RELAY_BULK="1", MMA_RANDOM_CASES="150", MMA_SPIN_TIMEOUT_MS="8000")
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_parity.py", "tests/test_gpu_forward_log.py", "tests/test_gpu_serialized.py",
                        "tests/test_gpu_random.py", "-k", "not test_gpu_bulk"],
                       cwd=str(ROOT), env=env, capture_output=True, text=True, timeout=1400)
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-2000:]
    assert " passed" in p.stdout


def test_zero_copy_modules_with_vector_kernel():
    """Direct zero-copy paths default to the cp.async.bulk kernel (zc_bulk_kernel); with
    MMA_ZC_BULK=0 they use the vector kernel (zc_copy_kernel, piece groups in registers). The
    segment modules (KV fetch / offload, irregular tables, small-piece groups, grid sizes) and
    the zero-copy parity cases run again with it in a fresh process."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, MMA_ZC_BULK="0", MMA_SPIN_TIMEOUT_MS="8000")
    p = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_segments.py", "tests/test_gpu_parity.py", "-k",
                        "not full_size and not mode_choice"],
                       cwd=str(ROOT), env=env, capture_output=True, text=True, timeout=1400)
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-2000:]
    assert " passed" in p.stdout
