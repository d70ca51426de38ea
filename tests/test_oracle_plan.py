"""Pins of the oracle's chunker and planner against things other than itself.

- chunking: SPEC.md's worked examples and the partition property;
- assignment: hand-derived worked examples (tests/golden/plan_examples.json), brute-force
  optimality over every assignment on tiny inputs, and the closed form
  T* = min{T : sum_p floor(T*bw_p/C) >= n} for the makespan;
- fallback: SPEC.md's examples and the strict boundary.
"""
import itertools
import json
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

GOLD = json.loads((Path(__file__).parent / "golden" / "plan_examples.json").read_text())
MODES = {"contiguous": 0, "interleaved": 1, "pull": 2}


@pytest.mark.parametrize("ex", GOLD["chunking"], ids=lambda e: f"{e['B']}/{e['C']}")
def test_chunking_examples(orc, ex):
    n = orc.nchunks(ex["B"], ex["C"])
    assert n == ex["n"]
    off, ln = orc.chunk_extent(n - 1, ex["B"], ex["C"])
    assert ln == ex["last"]
    assert off + ln == ex["B"]


@given(B=st.integers(0, 10**7), C=st.integers(1, 10**6))
@settings(max_examples=300, deadline=None)
def test_chunks_partition(orc, B, C):
    n = orc.nchunks(B, C)
    end = 0
    for i in ([] if n == 0 else [0, n // 2, n - 1]):
        off, ln = orc.chunk_extent(i, B, C)
        assert off == i * C and 0 < ln <= C
    if n:
        off, ln = orc.chunk_extent(n - 1, B, C)
        end = off + ln
    assert end == B
    assert n == (B + C - 1) // C


@pytest.mark.parametrize("ex", GOLD["examples"], ids=lambda e: f"{e['bw']}-{e['mode']}")
def test_worked_examples(orc, ex):
    rc, path, counts, fb = orc.plan(ex["bw"], ex["n"], 1, 0, MODES[ex["mode"]])
    assert rc == 0 and not fb
    assert counts == ex["counts"]
    if "path" in ex:
        assert path.tolist() == ex["path"]
    if "prefix" in ex:
        assert path[: len(ex["prefix"])].tolist() == ex["prefix"]


@pytest.mark.parametrize("ex", GOLD["fallback"], ids=lambda e: f"{e['B']}<{e['thr']}")
def test_fallback_examples(orc, ex):
    rc, path, counts, fb = orc.plan([55000, 55000], ex["B"], 5_000_000, ex["thr"], 0)
    assert rc == 0 and fb == ex["fallback"]
    if fb:
        assert path.tolist() == [0] and counts == [1, 0]


def test_relay_memory_formula():
    g = GOLD["relay_memory"]   # directions x pipelines x chunk
    assert g["directions"] * g["pipelines"] * g["chunk_bytes"] == g["bytes_per_gpu"]


def test_plan_edge_cases(orc):
    assert orc.plan([1, 1], 0, 4, 0)[0] == 0 and orc.plan([1, 1], 0, 4, 0)[1].size == 0
    # only the direct path usable -> native copy
    rc, path, counts, fb = orc.plan([55, 0, 0], 100, 4, 0)
    assert rc == 0 and fb and path.tolist() == [0]
    # relay-only set is planned normally (path 0 dropped)
    rc, path, counts, fb = orc.plan([0, 5, 5], 16, 4, 0, 1)
    assert rc == 0 and not fb and counts == [0, 2, 2] and path.tolist() == [1, 2, 1, 2]
    # no usable path / bad arguments
    assert orc.plan([0, 0], 16, 4, 0)[0] == orc.EINVAL
    assert orc.plan([1, 1], 16, 0, 0)[0] == orc.EINVAL
    assert orc.plan([1, 1], 16, 4, 0, 7)[0] == orc.EINVAL
    # a direct path anywhere but index 0 is illegal
    assert orc.plan([1, 1], 16, 4, 0, 0, kinds=[1, 0])[0] == orc.EINVAL
    # 256 paths is over the uint8 path index
    assert orc.plan([1] * 256, 16, 4, 0)[0] == orc.EINVAL


def test_direct_first_on_ties(orc):
    # equal bandwidth: the direct path (index 0) takes the first chunk and every tie
    rc, path, counts, _ = orc.plan([7, 7, 7], 3, 1, 0, 1)
    assert path.tolist() == [0, 1, 2]
    rc, path, counts, _ = orc.plan([7, 7, 7], 4, 1, 0, 1)
    assert path.tolist() == [0, 1, 2, 0]


def _opt_makespan(bw, backlog, n, C):
    """Exhaustive optimum over all count vectors of max_p (backlog_p + k_p C)/bw_p."""
    P = len(bw)
    best = None
    for ks in itertools.product(range(n + 1), repeat=P):
        if sum(ks) != n:
            continue
        if any(k and not bw[p] for p, k in enumerate(ks)):
            continue
        T = max((Fraction(backlog[p] + k * C, bw[p]) for p, k in enumerate(ks) if k), default=Fraction(0))
        best = T if best is None or T < best else best
    return best


def _plan_makespan(bw, backlog, counts, C):
    return max((Fraction(backlog[p] + k * C, bw[p]) for p, k in enumerate(counts) if k), default=Fraction(0))


def test_brute_force_optimal(orc):
    """EF greedy makespan == exhaustive optimum (equal chunks), P<=3, n<=7, with backlogs."""
    rng = np.random.default_rng(5)
    cases = 0
    for P in (1, 2, 3):
        for bw in itertools.product((1, 2, 3, 5), repeat=P):
            for n in range(1, 8):
                backlog = [0] * P if rng.random() < 0.5 else [int(x) for x in rng.integers(0, 9, P)]
                kinds = [1] * P           # relays only: no direct-only fallback
                rc, path, counts, fb = orc.plan(list(bw), n * 3, 3, 0, 1, kinds=kinds, backlog=backlog)
                assert rc == 0 and not fb
                assert sum(counts) == n
                assert _plan_makespan(bw, backlog, counts, 3) == _opt_makespan(bw, backlog, n, 3)
                cases += 1
    assert cases > 500


def _closed_form_T(bw, n, C):
    """T* = min{T : sum_p floor(T bw_p / C) >= n}; candidates are k C / bw_p."""
    cands = sorted({Fraction(k * C, b) for b in bw for k in range(1, n + 1)})
    for T in cands:
        if sum((T * b) // C for b in bw) >= n:
            return T
    raise AssertionError


@given(bw=st.lists(st.integers(1, 60000), min_size=1, max_size=8), n=st.integers(1, 400))
@settings(max_examples=200, deadline=None)
def test_closed_form_makespan_and_balance(orc, bw, n):
    C = 1 << 20
    kinds = [1] * len(bw)
    rc, path, counts, fb = orc.plan(bw, n * C, C, 0, 1, kinds=kinds)
    assert rc == 0
    T = _closed_form_T(bw, n, C)
    assert _plan_makespan(bw, [0] * len(bw), counts, C) == T
    # proportional split: T* <= (n+P)C/sum(bw) because sum floor(T bw/C) >= T sum(bw)/C - P,
    # so k_p <= T* bw_p / C < (n+P) bw_p / sum(bw), and |k_p - n bw_p/sum(bw)| < P.
    tot, P = sum(bw), len(bw)
    for p, b in enumerate(bw):
        assert counts[p] <= T * b / C
        assert abs(counts[p] - n * b / tot) < P


@given(bw=st.lists(st.integers(1, 100), min_size=1, max_size=6), n=st.integers(1, 200))
@settings(max_examples=200, deadline=None)
def test_contiguous_is_sorted_interleaved(orc, bw, n):
    kinds = [1] * len(bw)
    _, pi, ci, _ = orc.plan(bw, n, 1, 0, 1, kinds=kinds)
    _, pc, cc, _ = orc.plan(bw, n, 1, 0, 0, kinds=kinds)
    assert ci == cc
    assert pc.tolist() == sorted(pi.tolist())


def test_short_last_chunk_counts_as_full(orc):
    # B = 2.5 chunks on two equal paths: counts follow ceil(B/C) = 3 chunks
    rc, path, counts, fb = orc.plan([10, 10], 10, 4, 0, 1)
    assert counts == [2, 1] and path.tolist() == [0, 1, 0]


def test_predict(orc):
    T, g = orc.predict([1000, 1000], 2_000_000, 1_000_000, [0, 1])
    assert abs(T - 1e-3) < 1e-12 and abs(g - 2.0) < 1e-9
    # short last chunk counted with its real bytes
    T, g = orc.predict([1000, 1000], 1_500_000, 1_000_000, [0, 1])
    assert abs(T - 1e-3) < 1e-12
    # backlog delays a path
    T, g = orc.predict([1000, 1000], 2_000_000, 1_000_000, [0, 1], backlog=[0, 1_000_000])
    assert abs(T - 2e-3) < 1e-12
