"""Pins of the oracle's mover: the byte result has a plain definition (dst == src, nothing
outside dst written; §3.1 "preserving the semantics of existing transfer
APIs"), exactly-once delivery (per-byte write counters), and the relay-ring invariants on
the event log (forward only after staging completes; slot reuse only after forward).
Seeded protocol bugs must be caught.
"""
import itertools

import numpy as np
import pytest

import mma_inputs

GUARD = 64


def _buffers(B, seed=1):
    src = mma_inputs.pattern_bytes(seed, B) if B else np.zeros(0, np.uint8)
    dst = np.full(B + 2 * GUARD, 0xA5, dtype=np.uint8)
    return src, dst


def _run(orc, B, C, bw, path, S, exec_mode=0, base=None, fault=0, kinds=None):
    src, dstg = _buffers(B)
    dst = dstg[GUARD:GUARD + B]
    n = len(path)
    ev = np.zeros(max(n, 1) * orc.NEV, dtype=np.uint64)
    wc = np.zeros(max(B, 1), dtype=np.uint32)
    segs, ns = orc.segments_from_arrays([src.ctypes.data], [dst.ctypes.data], [B])
    rc = orc.move(segs, ns if B else 0, C, bw, path, S=S, base=base, exec_mode=exec_mode,
                  events=ev, write_count=wc, fault=fault, kinds=kinds)
    return rc, src, dstg, ev, wc


def _check_ok(orc, rc, src, dstg, ev, wc, B, bw, path, S, base=None, kinds=None):
    assert rc == 0
    assert np.array_equal(dstg[GUARD:GUARD + B], src)
    assert (dstg[:GUARD] == 0xA5).all() and (dstg[GUARD + B:] == 0xA5).all()
    if B:
        assert (wc[:B] == 1).all()          # every byte delivered exactly once
    assert orc.check_events(ev, bw, path, S, base=base, kinds=kinds) == 0


def test_brute_force_tiny(orc):
    """B in [0,64], C in [1,8], P <= 3, bw in {1,2,3,5}^P, S in {1,2,3}: planned moves."""
    cases = 0
    for P in (1, 2, 3):
        for bw in itertools.product((1, 2, 3, 5), repeat=P):
            for B in range(0, 65, 7 if P == 3 else 3):
                for C in range(1, 9, 1 if P < 3 else 3):
                    for mode in (0, 1):
                        kinds = [1] * P if (B + C) % 2 else None   # relay-only sets too
                        rc, path, counts, fb = orc.plan(list(bw), B, C, 0, mode, kinds=kinds)
                        assert rc == 0
                        S = 1 + (B + C + P) % 3
                        r = _run(orc, B, C, list(bw), path, S, kinds=kinds)
                        _check_ok(orc, *r, B, list(bw), path, S, kinds=kinds)
                        cases += 1
    assert cases > 3000


def test_arbitrary_assignments(orc):
    """Any assignment (not only planned ones) moves the bytes exactly once."""
    rng = np.random.default_rng(11)
    for _ in range(300):
        P = int(rng.integers(1, 6))
        C = int(rng.integers(1, 40))
        B = int(rng.integers(1, 900))
        n = (B + C - 1) // C
        path = rng.integers(0, P, n).astype(np.uint8)
        bw = [1] * P
        S = int(rng.integers(1, 5))
        base = rng.integers(0, 1 << 41, P).astype(np.uint64)
        for ex in (0, 1):
            r = _run(orc, B, C, bw, path, S, exec_mode=ex, base=base)
            _check_ok(orc, *r, B, bw, path, S, base=base)


@pytest.mark.parametrize("S", [1, 2, 4])
@pytest.mark.parametrize("base", [0, 3, 1 << 40])
def test_threaded_large(orc, S, base):
    B = (8 << 20) + 12345
    C = 1 << 18
    bw = [55, 54, 53, 56]
    rc, path, counts, fb = orc.plan(bw, B, C, 0, 1)
    b = [base] * 4
    r = _run(orc, B, C, bw, path, S, exec_mode=1, base=b)
    _check_ok(orc, *r, B, bw, path, S, base=b)


def test_fallback_plan_moves_whole_buffer(orc):
    B, C = 1000, 64
    rc, path, counts, fb = orc.plan([5, 5], B, C, thr=4096)
    assert fb and path.tolist() == [0]
    r = _run(orc, B, C, [5, 5], path, 2)
    _check_ok(orc, *r, B, [5, 5], path, 2)
    # a one-piece plan on a relay ring uses a slot as large as the piece
    r = _run(orc, B, C, [5, 5], np.array([0], np.uint8), 2, kinds=[1, 1])
    _check_ok(orc, *r, B, [5, 5], np.array([0], np.uint8), 2, kinds=[1, 1])


@pytest.mark.parametrize("fault", [1, 2])
def test_seeded_faults_detected(orc, fault):
    """Publishing before the staging write, or skipping the credit wait, must be caught by
    the byte compare or the event-log invariants (deterministic round-robin schedule).
    Skipping the credit wait only bites when the producer laps the consumer, which the
    lockstep schedule does at S = 1; test_oracle_ring.py catches it for every S by
    exhausting the interleavings."""
    caught = 0
    for S in ((1, 2) if fault == 1 else (1, 1)):
        for C in (4, 16):
            B = 40 * C
            bw = [1, 3]
            rc, path, counts, fb = orc.plan(bw, B, C, 0, 1)
            rc, src, dstg, ev, wc = _run(orc, B, C, bw, path, S, fault=fault)
            bad = rc != 0 or not np.array_equal(dstg[GUARD:GUARD + B], src) \
                or orc.check_events(ev, bw, path, S) > 0
            caught += bad
    assert caught == 4


def test_event_checker_catches_doctored_logs(orc):
    B, C, bw, S = 64, 4, [1, 1], 2
    rc, path, counts, fb = orc.plan(bw, B, C, 0, 1)
    r = _run(orc, B, C, bw, path, S)
    ev = r[3].reshape(-1, orc.NEV).copy()
    relay = [i for i in range(len(path)) if path[i] == 1]
    j = relay[3]
    d = ev.copy(); d[j, orc.EV_FWD_BEGIN] = d[j, orc.EV_STAGE_END] - 1   # forward before stage end
    assert orc.check_events(d.ravel(), bw, path, S) > 0
    d = ev.copy(); d[relay[2], orc.EV_STAGE_BEGIN] = ev[relay[0], orc.EV_CREDIT] - 1  # early reuse
    assert orc.check_events(d.ravel(), bw, path, S) > 0


def test_segments_scatter(orc):
    """Scattered variant: v = concatenation of segments in table order; chunk [a,b) of v
    copies each overlapping piece src_k+(x-v_k) -> dst_k+(x-v_k)."""
    rng = np.random.default_rng(3)
    pool = mma_inputs.pattern_bytes(9, 1 << 16)
    for trial in range(40):
        nseg = int(rng.integers(1, 40))
        lens = rng.integers(0, 700, nseg)
        src_off = rng.integers(0, pool.size - 700, nseg)          # sources may overlap
        dst = np.full(int(lens.sum()) * 2 + 64, 0xA5, np.uint8)
        perm = rng.permutation(nseg)
        dst_off = np.zeros(nseg, np.int64)
        pos = 0
        for k in perm:                                              # disjoint destinations
            dst_off[k] = pos
            pos += int(lens[k]) + int(rng.integers(0, 3))
        segs, ns = orc.segments_from_arrays(pool.ctypes.data + src_off, dst.ctypes.data + dst_off, lens)
        B = int(lens.sum())
        C = int(rng.integers(1, 300))
        bw = [int(x) for x in rng.integers(1, 9, 3)]
        rc, path, counts, fb = orc.plan(bw, B, C, 0, int(trial % 2))
        wc = np.zeros(max(B, 1), np.uint32)
        ev = np.zeros(max(len(path), 1) * orc.NEV, np.uint64)
        rc = orc.move(segs, ns, C, bw, path, S=2, exec_mode=trial % 2, events=ev, write_count=wc)
        assert rc == 0
        expect = np.full_like(dst, 0xA5)
        for k in range(nseg):
            expect[dst_off[k]:dst_off[k] + lens[k]] = pool[src_off[k]:src_off[k] + lens[k]]
        assert np.array_equal(dst, expect)
        if B:
            assert (wc[:B] == 1).all()
        assert orc.check_events(ev, bw, path, 2) == 0


def test_segments_overlapping_dst_rejected(orc):
    a = np.zeros(100, np.uint8)
    b = np.zeros(100, np.uint8)
    segs, ns = orc.segments_from_arrays([a.ctypes.data, a.ctypes.data], [b.ctypes.data, b.ctypes.data + 10], [20, 20])
    assert not orc.segments_disjoint(segs, ns)
    assert orc.move(segs, ns, 8, [1], np.zeros(5, np.uint8)) == orc.EINVAL
    segs, ns = orc.segments_from_arrays([a.ctypes.data, a.ctypes.data], [b.ctypes.data, b.ctypes.data + 20], [20, 20])
    assert orc.segments_disjoint(segs, ns)
    # empty segments never overlap anything
    segs, ns = orc.segments_from_arrays([a.ctypes.data] * 2, [b.ctypes.data, b.ctypes.data + 5], [20, 0])
    assert orc.segments_disjoint(segs, ns)


def test_bad_plans_rejected(orc):
    src, dstg = _buffers(100)
    segs, ns = orc.segments_from_arrays([src.ctypes.data], [dstg.ctypes.data], [100])
    assert orc.move(segs, ns, 10, [1, 1], np.zeros(9, np.uint8)) == orc.EINVAL     # wrong n
    assert orc.move(segs, ns, 10, [1, 1], np.full(10, 2, np.uint8)) == orc.EINVAL  # bad path
    assert orc.move(segs, ns, 10, [1, 1], np.zeros(10, np.uint8), S=0) == orc.EINVAL
