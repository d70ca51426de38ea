"""Workload shapes of BASELINE.json's configs (SURVEY §8(d) "Concrete synthetic inputs").

Shapes only: byte counts, segment tables and tensor lists. No chunking, planning or copy
arithmetic lives here (that is the method, implemented separately by oracle/ and by the
CUDA path).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import permutation, SEED_BASE

MiB = 1 << 20
GiB = 1 << 30

# config 1: single 64 MiB host->GPU0 transfer, 1 MiB chunks, 2 paths
CONFIG1 = dict(bytes=64 * MiB, chunk=1 * MiB, paths=2)

# config 2: size sweep 4 MiB .. 16 GiB, 1/2/4/8 paths
CONFIG2_SIZES = [4 * MiB << j for j in range(13)]


@dataclass(frozen=True)
class KVShape:
    """Paged KV cache of one sequence (config 3): Llama-3-8B, bf16, 16-token blocks.

    32 layers x {K, V} x 8 KV heads x head_dim 128 x 2 B = 128 KiB per token; one segment
    is (layer, K|V, block) = 16 tokens x 8 x 128 x 2 B = 32 KiB.
    """
    layers: int = 32
    kv_heads: int = 8
    head_dim: int = 128
    dtype_bytes: int = 2
    block_tokens: int = 16
    tokens: int = 32768
    device_blocks: int = 8192       # device cache [8192, 16, 8, 128] per layer per K/V
    host_slot_factor: int = 2       # host pool = 2x the sequence's segments

    @property
    def seg_bytes(self) -> int:
        return self.block_tokens * self.kv_heads * self.head_dim * self.dtype_bytes

    @property
    def nblocks(self) -> int:
        return self.tokens // self.block_tokens

    @property
    def nsegs(self) -> int:
        return self.layers * 2 * self.nblocks

    @property
    def total_bytes(self) -> int:
        return self.nsegs * self.seg_bytes


def kv_segments(shape: KVShape, seed: int = SEED_BASE + 3, request: int = 0):
    """Segment table of one prefix-cache fetch (config 3), layer-major. `request` 1 gives a
    second sequence whose host slots and device blocks are disjoint from request 0's (for
    overlapping one request's fetch with another's offload).

    Returns (host_off, dev_off, seg_bytes, host_pool_bytes, dev_bytes) where host_off[k] /
    dev_off[k] are byte offsets of segment k inside one pinned host pool and one device
    region holding all layers' K and V caches. Host slots are a seeded permutation of a
    pool `host_slot_factor` times larger than the sequence; the sequence's block ids are
    one seeded sample shared by all layers and K/V (a vLLM block table).
    """
    sb = shape.seg_bytes
    nslots = shape.nsegs * shape.host_slot_factor
    r0, r1 = request * shape.nsegs, (request + 1) * shape.nsegs
    b0, b1 = request * shape.nblocks, (request + 1) * shape.nblocks
    assert r1 <= nslots and b1 <= shape.device_blocks
    host_slot = permutation(seed, nslots)[r0:r1].astype(np.int64)
    block_ids = np.sort(permutation(seed + 1, shape.device_blocks)[b0:b1]).astype(np.int64)
    # device layout: [layer][K|V][device_blocks] segments of sb bytes
    k = np.arange(shape.nsegs, dtype=np.int64)
    layer_kv = k // shape.nblocks           # (layer, K|V) index, layer-major
    blk = k % shape.nblocks
    dev_off = (layer_kv * shape.device_blocks + block_ids[blk]) * sb
    host_off = host_slot * sb
    return host_off, dev_off, sb, nslots * sb, shape.layers * 2 * shape.device_blocks * sb


def scaled_kv(tokens: int) -> KVShape:
    """The config-3 shape with a different token count (small parity cases)."""
    return KVShape(tokens=tokens, device_blocks=max(2 * (tokens // 16), 16))


def qwen25_14b_tensors():
    """Config 4: Qwen2.5-14B bf16 weights under vLLM's fused naming, module order.

    48 layers, hidden 5120, intermediate 13824, 40 Q / 8 KV heads (head_dim 128), vocab
    152064, untied embeddings -> 339 tensors, 29,540,067,328 bytes.
    """
    return qwen_like_tensors(layers=48, hidden=5120, inter=13824, q_heads=40, kv_heads=8,
                             head_dim=128, vocab=152064)


def qwen_like_tensors(layers, hidden, inter, q_heads, kv_heads, head_dim, vocab):
    """Tensor list (name, bytes) of a Qwen2-architecture bf16 model in module order."""
    h, v, L = hidden, vocab, layers
    q, kv = q_heads * head_dim, kv_heads * head_dim
    out = [("embed_tokens", v * h * 2)]
    for i in range(L):
        out += [
            (f"l{i}.input_layernorm", h * 2),
            (f"l{i}.qkv_proj.weight", (q + 2 * kv) * h * 2),
            (f"l{i}.qkv_proj.bias", (q + 2 * kv) * 2),
            (f"l{i}.o_proj", h * q * 2),
            (f"l{i}.post_attention_layernorm", h * 2),
            (f"l{i}.gate_up_proj", 2 * inter * h * 2),
            (f"l{i}.down_proj", h * inter * 2),
        ]
    out += [("norm", h * 2), ("lm_head", v * h * 2)]
    return out


def packed_layout(tensors, align=256):
    """Offsets of the tensors packed in module order at `align` bytes (the sleep-mode backup
    buffer and the device weights share this layout). Returns (offsets, sizes, total)."""
    offs, sizes, pos = [], [], 0
    for _, b in tensors:
        pos = (pos + align - 1) // align * align
        offs.append(pos)
        sizes.append(b)
        pos += b
    return offs, sizes, pos
