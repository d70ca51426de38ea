"""Seeded synthetic inputs shared by the oracle tests and the GPU tests/bench.

This module holds NONE of the method's arithmetic (no chunking, planning or movement):
only the byte pattern that fills source buffers, seeded permutations for scattered
layouts, and the workload shapes of BASELINE.json's configs (DESIGN.md §4 "Input recipe").

Pattern (SURVEY §8(c) "Input generator"): little-endian 64-bit word i of a buffer filled
with `seed` is splitmix64((seed << 40) ^ i). Words are offset-unique, so a misplaced,
stale or duplicated chunk is detected by a byte compare. The GPU side regenerates the same
counter-based words in its own verify kernel (paper_2512_16056_b200/csrc/kernels/verify.cu);
the two implementations share no code.
"""
from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
SEED_BASE = 0x4D4D41  # "MMA"; config k uses SEED_BASE + k


def splitmix64_scalar(x: int) -> int:
    """One splitmix64 output for state x (Steele, Lea, Flood 2014)."""
    z = (x + GOLDEN) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def pattern_words(seed: int, first_word: int, nwords: int) -> np.ndarray:
    """Words first_word .. first_word+nwords-1 of the pattern for `seed` (uint64)."""
    i = np.arange(first_word, first_word + nwords, dtype=np.uint64)
    x = np.uint64((seed << 40) & MASK64) ^ i
    with np.errstate(over="ignore"):
        z = x + np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return z


def pattern_bytes(seed: int, nbytes: int, offset: int = 0) -> np.ndarray:
    """Bytes [offset, offset+nbytes) of the pattern stream for `seed` (uint8)."""
    if nbytes <= 0:
        return np.zeros(0, dtype=np.uint8)
    w0 = offset // 8
    w1 = (offset + nbytes + 7) // 8
    words = pattern_words(seed, w0, w1 - w0)
    b = words.view(np.uint8)  # little-endian host
    s = offset - 8 * w0
    return b[s:s + nbytes].copy()


def fill_pattern(buf: np.ndarray, seed: int, offset: int = 0) -> None:
    """Fill a uint8 array in place with pattern bytes [offset, offset+len)."""
    n = buf.size
    step = 1 << 26
    for a in range(0, n, step):
        m = min(step, n - a)
        buf[a:a + m] = pattern_bytes(seed, m, offset + a)


def permutation(seed: int, n: int) -> np.ndarray:
    """A seeded permutation of range(n) (PCG64), used to scatter blocks."""
    return np.random.Generator(np.random.PCG64(seed)).permutation(n)


from . import workloads  # noqa: E402,F401
