"""C10: transparent injection with LD_PRELOAD (§4). An unmodified torch program's
host<->device copies are routed through the engine (here with one loopback relay so the
relay ring and kernel run on a single GPU) and stay bit-exact."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]

PROG = r"""
import json, sys, torch
sys.path.insert(0, {root!r})
torch.manual_seed(0)
n = 48 << 20
x = torch.randint(0, 256, (n,), dtype=torch.uint8).pin_memory()
y = x.to("cuda", non_blocking=True)          # cudaMemcpyAsync H2D -> engine
z = torch.empty_like(x).pin_memory()
z.copy_(y, non_blocking=True)                # cudaMemcpyAsync D2H -> engine
torch.cuda.synchronize()
w = y.cpu()                                  # pageable destination -> native
small = x[:1000].to("cuda")                  # below MMA_PRELOAD_MIN_BYTES -> native
import paper_2512_16056_b200 as m
st = m.get_stats(0)
print(json.dumps(dict(eq1=bool(torch.equal(x, z)), eq2=bool(torch.equal(x, w)),
                      eq3=bool(torch.equal(x[:1000], small.cpu())), calls=st["calls"],
                      kernels=st["kernels"], relay=st["relay_bytes"], err=m.get_last_error())))
"""


def test_preload_routes_torch_copies(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    lib = ROOT / "paper_2512_16056_b200" / "libmma_preload.so"
    assert lib.exists()
    script = tmp_path / "p.py"
    script.write_text(PROG.format(root=str(ROOT)))
    env = dict(os.environ, LD_PRELOAD=str(lib), MMA_LOOPBACK="1", MMA_FALLBACK_BYTES="0",
               MMA_PRELOAD_MIN_BYTES=str(1 << 20), MMA_HOP="1", MMA_CHUNK_BYTES=str(4 << 20))
    p = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True, timeout=280)
    assert p.returncode == 0, p.stderr[-3000:]
    r = json.loads(p.stdout.strip().splitlines()[-1])
    assert r["eq1"] and r["eq2"] and r["eq3"] and r["err"] == 0
    assert r["calls"] >= 2                    # the two pinned copies went through the engine
    assert r["kernels"] >= 2 and r["relay"] > 0   # relay kernels ran (loopback ring)


PIN_PROG = r"""
import json, sys, torch
sys.path.insert(0, {root!r})
import paper_2512_16056_b200 as m
n = 48 << 20
x = torch.randint(0, 256, (n,), dtype=torch.uint8).pin_memory()     # cudaHostAlloc -> mma_host_alloc
owned = m.host_alloc_size(x.data_ptr())
node = m.host_page_node(x.data_ptr())
small = torch.ones(1024, dtype=torch.uint8).pin_memory()            # below the size floor -> runtime
y = x.to("cuda", non_blocking=True)                                 # cudaMemcpyAsync -> engine, zero-copy
torch.cuda.synchronize()
st = m.get_stats(0)
ok = bool(torch.equal(x, y.cpu()))
freed = None
if hasattr(torch._C, "_host_emptyCache"):                           # cudaFreeHost -> mma_host_free
    ptr = x.data_ptr()
    del x
    torch._C._host_emptyCache()
    freed = m.host_alloc_size(ptr) is None
print(json.dumps(dict(owned=owned, node=node, small_owned=m.host_alloc_size(small.data_ptr()), ok=ok,
                      kernels=st["kernels"], calls=st["calls"], freed=freed, err=m.get_last_error())))
"""


def test_preload_pinned_allocations_are_engine_buffers(tmp_path):
    """NEXT-3 (§4, "transparent substitution for the native CUDA memory API"): torch's
    pin_memory() under the shim gets an mma_host_alloc buffer (NUMA-placed, mapped), which
    the engine's zero-copy kernel then reads; torch's cudaFreeHost returns it to the engine"""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    lib = ROOT / "paper_2512_16056_b200" / "libmma_preload.so"
    script = tmp_path / "pin.py"
    script.write_text(PIN_PROG.format(root=str(ROOT)))
    env = dict(os.environ, LD_PRELOAD=str(lib), MMA_FALLBACK_BYTES="0", MMA_PRELOAD_MIN_BYTES=str(1 << 20),
               MMA_HOP="2", MMA_CHUNK_BYTES=str(4 << 20))
    p = subprocess.run([sys.executable, str(script)], env=env, capture_output=True, text=True, timeout=280)
    assert p.returncode == 0, p.stderr[-3000:]
    r = json.loads(p.stdout.strip().splitlines()[-1])
    assert r["owned"] is not None and r["owned"] >= 48 << 20, r
    assert r["node"] >= 0, r                          # a real page with a real NUMA node
    assert r["small_owned"] is None, r
    assert r["ok"] and r["err"] == 0 and r["kernels"] >= 1, r   # the zero-copy kernel moved it
    assert r["freed"] in (None, True), r
