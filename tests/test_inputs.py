"""The shared input generator (mma_inputs) against published splitmix64 values and the
workload arithmetic of SURVEY Appendix A."""
import numpy as np

import mma_inputs
from mma_inputs import workloads as W


def test_splitmix64_canonical():
    # splitmix64 from state 0: first output of the reference generator (Vigna's splitmix64.c)
    assert mma_inputs.splitmix64_scalar(0) == 0xE220A8397B1DCDAF


def test_pattern_words_pinned():
    w = mma_inputs.pattern_words(0x4D4D41, 0, 131072)
    assert int(w[0]) == 0x23C55927CEA1575D
    assert int(w[1]) == 0x58042E7674521C63
    assert int(w[2]) == 0xCF8F83A1E045AA25
    assert int(w[131071]) == 0x7C7A046CD1EBB40D
    for i in (0, 1, 77, 131071):
        assert int(w[i]) == mma_inputs.splitmix64_scalar((0x4D4D41 << 40) ^ i)


def test_pattern_bytes_offsets():
    full = mma_inputs.pattern_bytes(5, 1000)
    for off, n in [(0, 1), (3, 17), (8, 64), (13, 987)]:
        assert np.array_equal(mma_inputs.pattern_bytes(5, n, off), full[off:off + n])
    buf = np.zeros(333, np.uint8)
    mma_inputs.fill_pattern(buf, 5, 7)
    assert np.array_equal(buf, full[7:340])


def test_workload_arithmetic():
    kv = W.KVShape()
    assert kv.seg_bytes == 32768 and kv.nsegs == 131072 and kv.total_bytes == 4 << 30
    assert 2 * 32 * 8 * 128 * 2 == 131072            # bytes per token
    t = W.qwen25_14b_tensors()
    assert len(t) == 339 and sum(b for _, b in t) == 29_540_067_328


def test_kv_segments_layout():
    kv = W.scaled_kv(256)
    ho, do, sb, hpool, dbytes = W.kv_segments(kv)
    assert len(ho) == kv.nsegs and sb == 32768
    assert len(set(ho.tolist())) == kv.nsegs and len(set(do.tolist())) == kv.nsegs
    assert ho.max() + sb <= hpool and do.max() + sb <= dbytes
    assert (ho % sb == 0).all() and (do % sb == 0).all()
