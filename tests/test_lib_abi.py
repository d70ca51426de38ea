"""CPU checks of the product library: it loads without a GPU, exports every entry point
include/mma.h declares, and its host-side planner (csrc/planner.cpp) assigns chunks to
paths bit-exactly like the oracle (independent implementations, SURVEY §4 tier T2)."""
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2512_16056_b200 as mma

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "mma.h").read_text()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(mma_\w+)\s*\(", text, re.M)))


def test_header_symbols_exported():
    import ctypes
    L = ctypes.CDLL(str(mma.mma.LIB_PATH))
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(mma.mma.SYMBOLS)


def test_no_cpu_fallback_without_library(tmp_path, monkeypatch):
    monkeypatch.setattr(mma.mma, "LIB_PATH", tmp_path / "missing.so")
    monkeypatch.setattr(mma.mma, "_lib", None)
    with pytest.raises(ImportError):
        mma.mma.lib()


def test_product_does_not_import_oracle():
    pat = re.compile(r"^\s*(#include\s*[<\"].*oracle|(from|import)\s+oracle)|liboracle|orc_\w+\(", re.M)
    for p in (ROOT / "paper_2512_16056_b200").rglob("*"):
        if p.suffix in (".py", ".cpp", ".cu", ".cuh", ".h"):
            assert not pat.search(p.read_text()), p
    import subprocess
    out = subprocess.run(["nm", "-D", str(mma.mma.LIB_PATH)], capture_output=True, text=True).stdout
    assert "orc_" not in out


def test_error_string():
    assert b"timed out" in mma.mma.lib().mma_error_string(2001)


@pytest.mark.parametrize("mode", [0, 1])
def test_planner_parity_random(orc, mode):
    rng = np.random.default_rng(1234 + mode)
    for case in range(5000):
        P = int(rng.integers(1, 9))
        mbps = [int(x) for x in rng.integers(0, 60001, P)]
        if rng.random() < 0.3:
            mbps = [int(x) for x in rng.choice([1, 2, 3, 55000], P)]
        if not any(mbps):
            mbps[0] = 1
        kinds = [0] + [1] * (P - 1) if rng.random() < 0.7 else [1] * P
        backlog = [int(x) for x in rng.integers(0, 1 << 30, P)] if rng.random() < 0.3 else None
        C = int(rng.choice([4096, 1 << 20, 4 << 20, 5_000_000 // 4096 * 4096]))
        B = int(rng.integers(0, 600)) * C + int(rng.integers(0, C))
        thr = int(rng.choice([0, 0, C, 2 * C, 11_300_000]))
        orc_rc, orc_path, _, orc_fb = orc.plan(mbps, B, C, thr, mode, kinds=kinds, backlog=backlog)
        rc, path, fb = mma.plan_chunks(mbps, kinds, B, C, thr, mode, backlog)
        assert (rc == 0) == (orc_rc == 0), (mbps, kinds, B, C)
        if rc == 0:
            assert fb == orc_fb
            assert path == orc_path.tobytes(), (case, mbps, kinds, B, C, thr)


def test_planner_parity_golden(orc):
    import json
    gold = json.loads((ROOT / "tests" / "golden" / "plan_examples.json").read_text())
    for ex in gold["examples"]:
        if ex["mode"] == "pull":
            continue
        mode = 1 if ex["mode"] == "interleaved" else 0
        rc, path, fb = mma.plan_chunks(ex["bw"], [0] + [1] * (len(ex["bw"]) - 1), ex["n"] * 4096, 4096, 0, mode)
        assert rc == 0 and not fb
        counts = [path.count(bytes([p])) for p in range(len(ex["bw"]))]
        assert counts == ex["counts"]
        if "path" in ex:
            assert list(path) == ex["path"]


def test_planner_rejects_bad_input():
    assert mma.plan_chunks([1, 1], [1, 0], 100, 10)[0] != 0        # direct not at index 0
    assert mma.plan_chunks([0, 0], [0, 1], 100, 10)[0] != 0        # no usable path
    assert mma.plan_chunks([1], [0], 100, 0)[0] != 0               # zero chunk
    rc, path, fb = mma.plan_chunks([1, 1], [0, 1], 0, 10)
    assert rc == 0 and path == b""


def test_header_is_plain_c(tmp_path):
    """include/mma.h is a C ABI: it compiles as strict C11 (no C++ types in the signatures)"""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if not gcc:
        pytest.skip("no gcc")
    src = tmp_path / "t.c"
    src.write_text('#include "mma.h"\nint main(void) { mma_config_t c; mma_stats_t s; mma_topology_t t;'
                   ' (void)c; (void)s; (void)t; return 0; }\n')
    r = subprocess.run([gcc, "-std=c11", "-Wall", "-Wextra", "-pedantic", "-Werror", "-I", str(ROOT / "include"),
                        "-c", str(src), "-o", str(tmp_path / "t.o")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.parametrize("mode", [0, 1], ids=["contiguous", "interleaved"])
def test_multi_planner_parity_random(orc, mode):
    """the engine's joint planner (mma_plan_multi, heap-based) vs the oracle's
    orc_plan_multi (linear scans), bit for bit on random link sets, carry matrices and
    transfer lists (NEXT-1)"""
    rng = np.random.default_rng(77 + mode)
    for case in range(3000):
        L = int(rng.integers(1, 10))
        bw = [int(x) for x in rng.integers(0, 60001, L)]
        if rng.random() < 0.4:
            bw = [int(x) for x in rng.choice([0, 1, 2, 3, 55000], L)]
        ok = (rng.random((L, L)) < rng.random()).astype(np.uint8)
        T = int(rng.integers(0, 7))
        targets = [int(x) for x in rng.integers(0, L, T)]
        nch = [int(x) for x in rng.integers(0, 300, T)]
        C = int(rng.choice([4096, 1 << 20, 8 << 20]))
        prefer = int(rng.integers(-1, L)) if rng.random() < 0.3 else -1
        orc_rc, orc_plans = orc.plan_multi(bw, ok, targets, nch, C, mode, prefer)
        rc, plans = mma.plan_multi(bw, ok, targets, nch, C, mode, prefer)
        assert (rc == 0) == (orc_rc == 0), (case, bw, ok.tolist(), targets, nch)
        if rc == 0:
            for a, b in zip(plans, orc_plans):
                assert a.tolist() == b.tolist(), (case, bw, ok.tolist(), targets, nch)
