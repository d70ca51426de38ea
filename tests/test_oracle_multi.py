"""Pins of the oracle's joint plan of concurrent transfers (orc_plan_multi; SURVEY NEXT-1,
the paper's Path Selector under constant rates, §3.4.2; SPEC S:441-453
next_for_link): the SPEC's worked examples, a hand-worked two-target schedule, the
single-target case (which must be the paper's pull rule that orc_plan's PULL mode and the
golden examples already pin), and what any valid plan must satisfy."""
import numpy as np
from hypothesis import given, settings, strategies as st

import oracle

I, CT = oracle.INTERLEAVED, oracle.CONTIG


def test_spec_direct_first():
    """"own queue has 3 chunks, foreign queue has 100 -> own queue's head".
    Link 1 may relay for GPU 0 (100 chunks) but its own GPU 1 has 3: it drains those first."""
    rc, (a, b) = oracle.plan_multi([1, 1], [[0, 1], [1, 0]], [0, 1], [100, 3], 1, I)
    assert rc == 0
    assert b.tolist() == [1, 1, 1]                        # all of GPU 1's own chunks on its link
    assert a[:1].tolist() == [0] and (a[:4] == 0).sum() >= 3   # link 1 joins GPU 0 only after


def test_spec_longest_queue():
    """"own queue empty; foreign queues sized {A:4, B:9} -> head of B". Links 0
    and 1 pull their own heads at t = 0 (4 -> 3, 9 -> 8 left); link 2 (no queue of its own,
    1000x faster, free again long before t = 1) takes the longer queue's head each time:
    GPU 1's five times (8 -> 3), then the tie 3 : 3 goes to the lower GPU id, and the
    two queues alternate until both are empty."""
    ok = [[0, 0, 1], [0, 0, 1], [0, 0, 0]]
    rc, (a, b) = oracle.plan_multi([1, 1, 1000], ok, [0, 1], [4, 9], 1, I)
    assert rc == 0
    assert a.tolist() == [0, 2, 2, 2] and b.tolist() == [1, 2, 2, 2, 2, 2, 2, 2, 2]


def test_hand_worked_two_targets():
    """bw [1, 1], GPU 0: 6 chunks, GPU 1: 2 chunks, each link may relay for the other.
    free times (chunks taken): t=0 link0 own c0, link1 own d0; t=1 link0 own c1, link1 own
    d1; t=2 link0 own c2, link1 (own empty) takes GPU 0's c3; t=3 link0 own c4, link1 c5."""
    rc, (a, b) = oracle.plan_multi([1, 1], [[0, 1], [1, 0]], [0, 1], [6, 2], 1, I)
    assert rc == 0 and a.tolist() == [0, 0, 0, 1, 0, 1] and b.tolist() == [1, 1]
    rc, (a, b) = oracle.plan_multi([1, 1], [[0, 1], [1, 0]], [0, 1], [6, 2], 1, CT)
    assert rc == 0 and a.tolist() == [0, 0, 0, 0, 1, 1] and b.tolist() == [1, 1]


def test_queue_is_fifo_across_transfers_to_one_gpu():
    """two transfers to GPU 0 form one queue ("appended FIFO to the queue keyed by
    (direction, endpoint gpu)"): the second transfer's chunks follow the first's"""
    rc, (a, b) = oracle.plan_multi([3, 1], [[0, 1], [0, 0]], [0, 0], [5, 3], 1, I)
    assert rc == 0
    rc2, whole, _, _ = oracle.plan([3, 1], 8, 1, 0, oracle.PULL)
    assert np.concatenate([a, b]).tolist() == whole.tolist()


@settings(max_examples=200, deadline=None)
@given(st.lists(st.integers(1, 9), min_size=1, max_size=6), st.integers(0, 60), st.integers(1, 4))
def test_single_target_is_the_pull_rule(bw, n, C):
    """one target whose links are in ascending id order: the joint plan is orc_plan's PULL
    rule (golden pull examples: tests/golden/plan_examples.json)"""
    L = len(bw)
    ok = np.zeros((L, L), np.uint8)
    ok[0, :] = 1
    rc, (a,) = oracle.plan_multi(bw, ok, [0], [n], C, I)
    rc2, exp, _, fb = oracle.plan(bw, n * C, C, 0, oracle.PULL)
    assert rc == 0 and rc2 == 0
    if fb:                                   # one usable link: orc_plan reports the native piece
        exp = np.zeros(n, np.uint8)
    assert a.tolist() == (exp.tolist() if n else [])


@settings(max_examples=200, deadline=None)
@given(st.integers(1, 6), st.data())
def test_valid_plan(L, data):
    bw = data.draw(st.lists(st.integers(0, 9), min_size=L, max_size=L))
    ok = np.array(data.draw(st.lists(st.lists(st.integers(0, 1), min_size=L, max_size=L), min_size=L, max_size=L)),
                  np.uint8)
    T = data.draw(st.integers(0, 5))
    targets = data.draw(st.lists(st.integers(0, L - 1), min_size=T, max_size=T))
    nch = data.draw(st.lists(st.integers(0, 12), min_size=T, max_size=T))
    carriers = [[l for l in range(L) if bw[l] > 0 and (l == d or ok[d, l])] for d in range(L)]
    rc, plans = oracle.plan_multi(bw, ok, targets, nch, 1, I)
    if any(n and not carriers[d] for d, n in zip(targets, nch)):
        assert rc == oracle.EINVAL
        return
    assert rc == 0
    rc, cplans = oracle.plan_multi(bw, ok, targets, nch, 1, CT)
    for d, n, p, cp in zip(targets, nch, plans, cplans):
        assert len(p) == n and set(p.tolist()) <= set(carriers[d])     # exactly once, on a legal link
        assert sorted(p.tolist()) == sorted(cp.tolist())              # contiguous form: same counts
        if n:
            own = [d] if d in carriers[d] else []
            order = own + [l for l in range(L) if l != d]
            ranks = [order.index(x) for x in cp.tolist()]
            assert ranks == sorted(ranks)                               # own link first, then by id


def test_prefer_gpu():
    """P:569 "tasks can be preferentially fetched from the corresponding micro-task queue"
    (SPEC PreferGpu: the named queue when non-empty, then LongestQueueFirst). Same batch as
    test_spec_longest_queue, GPU 0 preferred: link 2 drains GPU 0's queue (3 left after link
    0's first pull) before it turns to the longer queue of GPU 1; the links' own queues still
    come first."""
    ok = [[0, 0, 1], [0, 0, 1], [0, 0, 0]]
    rc, (a, b) = oracle.plan_multi([1, 1, 1000], ok, [0, 1], [4, 9], 1, I, prefer=0)
    assert rc == 0
    assert a.tolist() == [0, 2, 2, 2] and b.tolist() == [1] + [2] * 8
    # preferring a GPU the link may not carry changes nothing
    rc, (a2, b2) = oracle.plan_multi([1, 1, 1000], [[0, 0, 0], [0, 0, 1], [0, 0, 0]], [0, 1], [4, 9], 1, I, prefer=0)
    rc3, (a3, b3) = oracle.plan_multi([1, 1, 1000], [[0, 0, 0], [0, 0, 1], [0, 0, 0]], [0, 1], [4, 9], 1, I)
    assert a2.tolist() == a3.tolist() and b2.tolist() == b3.tolist()
