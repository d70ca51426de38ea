"""Host-address issue order (reading R22): the engine's permutation must be the stable
ascending order of the addresses -- checked against numpy's stable argsort on the shapes the
engine sorts (a config-3 table of 32 KiB slots in an 8 GiB pool, duplicates, tiny and empty
inputs, both the radix path (>= 4096 keys) and the comparison path)."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def mma():
    import paper_2512_16056_b200 as m
    m.mma.lib()
    return m


@pytest.mark.parametrize("n", [0, 1, 2, 17, 4095, 4096, 131072])
def test_matches_stable_argsort(mma, n):
    rng = np.random.default_rng(n + 1)
    base = 0x7F0000000000
    slots = rng.permutation(262144)[:n].astype(np.uint64)
    addr = base + slots * np.uint64(32768) + rng.integers(0, 16, n, dtype=np.uint64) * np.uint64(16)
    got = mma.order_by_address(addr)
    assert np.array_equal(got, np.argsort(addr, kind="stable").astype(np.uint32))


def test_duplicates_and_same_page(mma):
    rng = np.random.default_rng(5)
    addr = (0x100000 + rng.integers(0, 64, 10000) * 64).astype(np.uint64)   # many keys share a page
    assert np.array_equal(mma.order_by_address(addr), np.argsort(addr, kind="stable").astype(np.uint32))
    wide = np.array([2**47 + 5, 3, 2**40, 3, 0], dtype=np.uint64)
    assert list(mma.order_by_address(wide)) == [4, 1, 3, 2, 0]


def test_radix_over_a_wide_range(mma):
    rng = np.random.default_rng(9)
    addr = rng.integers(0, 2**47, 6000, dtype=np.uint64)        # several radix digits
    assert np.array_equal(mma.order_by_address(addr), np.argsort(addr, kind="stable").astype(np.uint32))
