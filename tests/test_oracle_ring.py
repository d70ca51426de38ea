"""Exhaustive interleavings of the relay ring protocol.

The correct protocol must reach no violating state for every n <= 6, S <= 3 and several
ring bases (flags left by earlier calls, reading R18); each seeded bug must be caught.
"""
import pytest


@pytest.mark.parametrize("S", [1, 2, 3])
@pytest.mark.parametrize("base", [0, 1, 2, 5, 1 << 40])
def test_correct_protocol_has_no_violation(orc, S, base):
    for n in range(0, 7):
        rc, states, bad = orc.ring_explore(n, S, base)
        assert rc == 0 and bad == 0, (n, S, base)
        assert states >= 1


def test_state_space_is_nontrivial(orc):
    # with S >= 2 the producer runs ahead, so interleavings multiply
    _, s1, _ = orc.ring_explore(6, 1)
    _, s3, _ = orc.ring_explore(6, 3)
    assert s3 > s1 > 6 * 8


@pytest.mark.parametrize("fault", [1, 2], ids=["publish-early", "skip-credit"])
@pytest.mark.parametrize("S", [1, 2, 3])
def test_seeded_bugs_caught(orc, fault, S):
    n = S + 2          # enough chunks to reuse every slot
    for base in (0, 1 << 40):
        rc, states, bad = orc.ring_explore(n, S, base, fault)
        assert rc == 0 and bad > 0, (fault, S, base)


def test_explore_rejects_out_of_range(orc):
    assert orc.ring_explore(9, 2)[0] == orc.EINVAL
    assert orc.ring_explore(3, 0)[0] == orc.EINVAL
    assert orc.ring_explore(3, 5)[0] == orc.EINVAL


def test_oracle_cli():
    import json
    import subprocess
    import sys
    run = lambda *a: json.loads(subprocess.run([sys.executable, "-m", "oracle", *a], capture_output=True,
                                               text=True, check=True).stdout)
    p = run("plan", "--bw", "50,25", "--bytes", "6", "--chunk", "1", "--mode", "interleaved", "--relay-only")
    assert p["path"] == [0, 0, 1, 0, 0, 1] and p["counts"] == [4, 2]
    m = run("move", "--bw", "3,1", "--bytes", "1MiB", "--chunk", "64KiB", "--slots", "2", "--mode", "interleaved")
    assert m["bytes_equal"] and m["exactly_once"] and m["invariant_violations"] == 0
    r = run("ring", "--n", "4", "--slots", "2", "--fault", "publish-early")
    assert r["violations"] > 0
