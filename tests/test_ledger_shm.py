"""The cross-process backlog ledger (SURVEY NEXT-4 "a shared-memory path ledger"): host-only
logic of libmma.so, run here on CPU. Two processes attach the same named ledger; bytes one
adds on a link (keyed by PCI bus id) are visible to the other, removals balance, and slots
are claimed per bus id, so processes with different device orderings agree."""
import multiprocessing as mp
import os

import pytest

H2D, D2H = 0, 1


def _lib():
    import paper_2512_16056_b200 as m
    m.mma.lib()
    return m


def _child(name, q_in, q_out):
    m = _lib()
    m.ledger_attach(name)
    q_out.put(("ready", None))
    while True:
        cmd, arg = q_in.get()
        if cmd == "add":
            bus, d, nb, own = arg
            m.ledger_shared_add(bus, d, nb, own)
            q_out.put(("ok", None))
        elif cmd == "get":
            bus, d = arg
            q_out.put(("val", m.ledger_shared_get(bus, d)))
        else:
            m.ledger_attach(None)
            q_out.put(("bye", None))
            return


@pytest.fixture()
def name():
    n = f"test{os.getpid()}"
    yield n
    _lib().ledger_unlink(n)


def test_two_processes_share_link_counters(name):
    m = _lib()
    m.ledger_attach(name)
    ctx = mp.get_context("spawn")
    q_in, q_out = ctx.Queue(), ctx.Queue()
    p = ctx.Process(target=_child, args=(name, q_in, q_out))
    p.start()
    try:
        assert q_out.get(timeout=120)[0] == "ready"
        busA, busB = "0000:1b:00.0", "0000:43:00.0"
        m.ledger_shared_add(busA, H2D, 24 << 20, 24 << 20)       # this process: a direct call on A
        q_in.put(("add", (busB, H2D, 8 << 20, 0)))               # the other: relay bytes on B
        assert q_out.get(timeout=60)[0] == "ok"
        assert m.ledger_shared_get(busB, H2D) == (8 << 20, 0)
        q_in.put(("get", (busA, H2D)))
        assert q_out.get(timeout=60) == ("val", (24 << 20, 24 << 20))
        q_in.put(("get", (busA, D2H)))                           # directions are separate
        assert q_out.get(timeout=60) == ("val", (0, 0))
        m.ledger_shared_add(busA, H2D, -(24 << 20), -(24 << 20))  # the call completed
        q_in.put(("add", (busB, H2D, -(8 << 20), 0)))
        assert q_out.get(timeout=60)[0] == "ok"
        q_in.put(("get", (busA, H2D)))
        assert q_out.get(timeout=60) == ("val", (0, 0))
        assert m.ledger_shared_get(busB, H2D) == (0, 0)
        q_in.put(("stop", None))
        assert q_out.get(timeout=60)[0] == "bye"
    finally:
        p.join(timeout=60)
        m.ledger_attach(None)
    assert p.exitcode == 0


def test_slots_by_bus_id_and_errors(name):
    m = _lib()
    with pytest.raises(Exception):
        m.ledger_shared_get("0000:01:00.0", H2D)                # not attached
    m.ledger_attach(name)
    try:
        buses = [f"0000:{k:02x}:00.0" for k in range(16)]
        for k, b in enumerate(buses):
            m.ledger_shared_add(b, D2H, k + 1, 0)
        for k, b in enumerate(buses):
            assert m.ledger_shared_get(b, D2H) == (k + 1, 0)
        with pytest.raises(Exception):
            m.ledger_shared_add("0000:ff:00.0", D2H, 1, 0)      # 16 slots, all taken
        with pytest.raises(Exception):
            m.ledger_shared_add(buses[0], 2, 1, 0)              # bad direction
        m.ledger_attach(None)
        m.ledger_attach(name)                                    # state persists in the object
        assert m.ledger_shared_get(buses[3], D2H) == (4, 0)
    finally:
        m.ledger_attach(None)
    with pytest.raises(Exception):
        m.ledger_attach("bad/name")


def _adder(name, bus, q_out):
    m = _lib()
    m.ledger_attach(name)
    m.ledger_process_add(bus, H2D, 8 << 20, 0)        # a call of this process, in flight
    q_out.put("added")
    import time
    time.sleep(600)                                   # killed before it completes


def test_dead_process_bytes_leave_the_ledger(name):
    """a process that dies with calls in flight must not pin its bytes in the
    ledger: entries belong to processes, readers skip a dead owner's, and a later attacher
    reclaims the entry"""
    import signal
    m = _lib()
    m.ledger_attach(name)
    bus = "0000:1b:00.0"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_adder, args=(name, bus, q))
    p.start()
    try:
        assert q.get(timeout=120) == "added"
        assert m.ledger_shared_get(bus, H2D) == (8 << 20, 0)
        m.ledger_process_add(bus, H2D, 1 << 20, 1 << 20)             # this process's own call
        assert m.ledger_shared_get(bus, H2D) == (9 << 20, 1 << 20)
    finally:
        os.kill(p.pid, signal.SIGKILL)
        p.join(timeout=60)
    assert m.ledger_shared_get(bus, H2D) == (1 << 20, 1 << 20)       # the dead process's bytes are gone
    m.ledger_process_add(bus, H2D, -(1 << 20), -(1 << 20))
    m.ledger_attach(name)                                             # re-attach: a fresh entry
    assert m.ledger_shared_get(bus, H2D) == (0, 0)
    m.ledger_attach(None)
