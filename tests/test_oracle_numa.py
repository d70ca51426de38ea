"""Pins of the oracle's NUMA-affine order (orc_numa_order, reading R23; §5.1.1):
hand-worked examples (tests/golden/numa_regroup.json), the invariants that define the rule
(a permutation; group ranks non-decreasing in the reading's order; table order inside a
group; table order with fewer than two usable path nodes), and the locality property the
regrouping exists for, checked through the oracle's own planner."""
import json
from pathlib import Path

import numpy as np
from hypothesis import given, settings, strategies as st

import oracle

GOLD = json.loads((Path(__file__).parent / "golden" / "numa_regroup.json").read_text())


def test_golden_orders():
    for ex in GOLD["examples"]:
        got = oracle.numa_order(ex["seg_node"], ex["bw"], ex["path_node"])
        assert got.tolist() == ex["order"], ex["why"]


def test_golden_locality_through_the_planner():
    ex = GOLD["examples"][-1]
    n = len(ex["seg_node"])
    rc, path, _, fb = oracle.plan(ex["bw"], n, 1, 0, oracle.CONTIG)   # one unit per segment
    assert rc == 0 and path.tolist() == ex["plan_contiguous"]
    order = oracle.numa_order(ex["seg_node"], ex["bw"], ex["path_node"])
    seg_node = np.array(ex["seg_node"])
    path_node = np.array(ex["path_node"])
    local_re = int((seg_node[order] == path_node[path]).sum())
    local_tab = int((seg_node == path_node[path]).sum())
    assert (local_re, local_tab) == (ex["local_segments_regrouped"], ex["local_segments_table_order"])


def _rank(nd, groups):
    return groups.index(nd) if nd in groups else (len(groups) + nd if nd >= 0 else 1 << 30)


@settings(max_examples=300, deadline=None)
@given(st.lists(st.integers(-1, 5), min_size=0, max_size=40),
       st.lists(st.tuples(st.integers(-1, 5), st.integers(0, 3)), min_size=1, max_size=8))
def test_invariants(seg_node, paths):
    path_node = [p[0] for p in paths]
    bw = [p[1] for p in paths]
    order = oracle.numa_order(seg_node, bw, path_node).tolist()
    n = len(seg_node)
    assert sorted(order) == list(range(n))                       # a permutation
    groups = []
    for nd, b in zip(path_node, bw):
        if b > 0 and nd >= 0 and nd not in groups:
            groups.append(nd)
    if len(groups) < 2 or n < 2:
        assert order == list(range(n))                           # table order
        return
    ranks = [_rank(seg_node[k], groups) for k in order]
    assert ranks == sorted(ranks)                                # groups in the reading's order
    for a, b in zip(order, order[1:]):                           # table order inside a group
        if _rank(seg_node[a], groups) == _rank(seg_node[b], groups):
            assert a < b
