"""Build libmma.so in-tree with nvcc for sm_100a (no torch, no JIT cache).

    python -m paper_2512_16056_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libmma.so"
PRELOAD = PKG / "libmma_preload.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = [
    CSRC / "plane.cpp",
    CSRC / "api.cpp",
    CSRC / "tune.cpp",
    CSRC / "mp.cpp",
    CSRC / "trace.cpp",
    CSRC / "planner.cpp",
    CSRC / "hostmem.cpp",
    CSRC / "ledger_shm.cpp",
    CSRC / "kernels" / "relay.cu",
    CSRC / "kernels" / "zerocopy.cu",
    CSRC / "kernels" / "verify.cu",
]
HEADERS = [ROOT / "include" / "mma.h", CSRC / "engine.h", CSRC / "plane.h", CSRC / "kargs.h", CSRC / "planner.h",
           CSRC / "kernels" / "copy.cuh", CSRC / "preload.cpp", CSRC / "ranges.h"]

FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-Wall",
    "-Xptxas", "-v" if os.environ.get("MMA_PTXAS_V") else "-O3",
    "-I", str(ROOT / "include"),
    "--expt-relaxed-constexpr", "--extended-lambda",
] + (["-g"] if os.environ.get("MMA_HOST_DEBUG") else [])


def stale() -> bool:
    if not LIB.exists() or not PRELOAD.exists():
        return True
    t = LIB.stat().st_mtime
    return any(p.stat().st_mtime > t for p in SOURCES + HEADERS + [Path(__file__)])


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        return LIB
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    cmds = []
    for src in SOURCES:
        obj = objdir / (src.stem + ".o")
        cmd = [NVCC, *FLAGS, "-c", str(src), "-o", str(obj)]
        if src.suffix == ".cpp":
            cmd = [NVCC, *FLAGS, "-x", "cu", "-c", str(src), "-o", str(obj)]
        cmds.append((cmd, str(obj)))
    # the translation units compile independently: in parallel (nvcc is single-threaded)
    from concurrent.futures import ThreadPoolExecutor
    def run(c):
        if verbose:
            print(" ".join(c[0]))
        subprocess.check_call(c[0])
        return c[1]
    with ThreadPoolExecutor(max_workers=min(len(cmds), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(run, cmds))
    tmp = LIB.with_suffix(".so.tmp")
    subprocess.check_call([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-cudart", "static", "-o", str(tmp), *objs, "-ldl", "-lpthread", "-lrt"])
    os.replace(tmp, LIB)
    build_preload(verbose)
    return LIB


def build_preload(verbose: bool = False) -> Path:
    """libmma_preload.so: the LD_PRELOAD interceptor (C10), linked to libmma.so by rpath."""
    src = CSRC / "preload.cpp"
    tmp = PRELOAD.with_suffix(".so.tmp")
    cmd = ["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-Wall", "-I", str(ROOT / "include"),
           str(src), "-o", str(tmp), "-L", str(PKG), "-lmma", "-Wl,-rpath,$ORIGIN", "-ldl"]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(tmp, PRELOAD)
    return PRELOAD


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
