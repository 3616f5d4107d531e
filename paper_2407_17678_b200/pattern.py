"""Layout policy and per-head block layouts (host side, C++ builder via the C ABI).

Mirrors /root/reference/proj/include/shardattn/pattern.hpp and csr.hpp:
``StrideSegment``, ``PatternConfig`` (pattern.hpp:17-60), ``CsrMask``
(csr.hpp:15-24), ``build_head_mask`` / ``build_all_masks`` (pattern.cpp:127-166),
``to_csr`` / ``from_csr`` / ``nnz`` (csr.cpp:35-67), ``LayerSchedule`` /
``build_layer_masks`` (pattern.cpp:118-125,168-181) and the config factories
(pattern.cpp:190-236).  The CSR/CSC lists come from the analytic O(nnz)
builder in csrc/layout.cpp, bit-exact to the reference's O(B^2) scan.
Invalid inputs raise ``S2InvalidArgument`` (a ``ValueError``), the analogue of
the reference's ``std::invalid_argument``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Set

import numpy as np

from . import _abi
from ._abi import check, lib


@dataclass
class StrideSegment:
    start_block_distance: int = 0
    end_block_distance: int = 0
    stride: int = 1
    offsets: List[int] = field(default_factory=list)


@dataclass
class PatternConfig:
    seq_len: int = 0
    block_size: int = 1
    num_heads: int = 1
    num_kv_heads: int = 0
    local_blocks: int = 1
    local_stride: int = 1
    stride_segments: List[StrideSegment] = field(default_factory=list)

    # pattern.hpp:48-50
    def num_blocks(self) -> int:
        return -(-self.seq_len // self.block_size) if self.block_size > 0 else 0

    def kv_heads(self) -> int:
        return self.num_kv_heads if self.num_kv_heads > 0 else self.num_heads

    def heads_per_group(self) -> int:
        return self.num_heads // self.kv_heads()

    def group_of(self, head: int) -> int:
        return head // self.heads_per_group()

    def to_c(self):
        """(s2_pattern_config, keepalive) for a C call."""
        c = _abi.s2_pattern_config()
        c.seq_len, c.block_size = self.seq_len, self.block_size
        c.num_heads, c.num_kv_heads = self.num_heads, self.num_kv_heads
        c.local_blocks, c.local_stride = self.local_blocks, self.local_stride
        if len(self.stride_segments) > _abi.S2_MAX_SEGMENTS:
            raise _abi.S2InvalidArgument(1, "too many stride segments")
        c.num_segments = len(self.stride_segments)
        keep = []
        for i, s in enumerate(self.stride_segments):
            seg = c.segments[i]
            seg.start_block_distance = s.start_block_distance
            seg.end_block_distance = s.end_block_distance
            seg.stride = s.stride
            seg.num_offsets = len(s.offsets)
            if s.offsets:
                arr = (ctypes.c_int * len(s.offsets))(*s.offsets)
                keep.append(arr)
                seg.offsets = ctypes.cast(arr, ctypes.POINTER(ctypes.c_int))
        return c, keep

    def validate(self) -> None:
        c, keep = self.to_c()
        check(lib().s2_pattern_validate(ctypes.byref(c)))

    def offset_for(self, segment: int, head: int) -> int:
        c, keep = self.to_c()
        out = ctypes.c_int()
        check(lib().s2_pattern_offset_for(ctypes.byref(c), segment, head, ctypes.byref(out)))
        return out.value


@dataclass
class CsrMask:
    """csr.hpp:15-24: row i's key blocks are col_idx[row_ptr[i]:row_ptr[i+1]]."""
    head_index: int
    num_blocks: int
    row_ptr: np.ndarray
    col_idx: np.ndarray

    def validate(self) -> None:
        rp = np.ascontiguousarray(self.row_ptr, dtype=np.int32)
        ci = np.ascontiguousarray(self.col_idx, dtype=np.int32)
        if self.num_blocks >= 1 and rp.size != self.num_blocks + 1:
            raise _abi.S2InvalidArgument(1, "row_ptr must have num_blocks + 1 entries")
        if self.num_blocks >= 1 and rp[-1] != ci.size:
            raise _abi.S2InvalidArgument(1, "row_ptr[B] must equal col_idx length")
        check(lib().s2_csr_validate(self.num_blocks, _iptr(rp), _iptr(ci), ci.size))

    def nnz(self) -> int:
        return int(self.col_idx.size)

    def row(self, i: int) -> List[int]:
        return self.col_idx[self.row_ptr[i]:self.row_ptr[i + 1]].tolist()


def _iptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


def nnz(csr: CsrMask) -> int:
    return csr.nnz()


def build_csr(cfg: PatternConfig, head: int) -> CsrMask:
    """to_csr(build_head_mask(cfg, head)) without the B x B mask."""
    c, keep = cfg.to_c()
    n = ctypes.c_int64()
    check(lib().s2_layout_nnz(ctypes.byref(c), head, ctypes.byref(n)))
    B = cfg.num_blocks()
    rp = np.zeros(B + 1, np.int32)
    ci = np.zeros(max(n.value, 1), np.int32)
    check(lib().s2_layout_build_csr(ctypes.byref(c), head, _iptr(rp), _iptr(ci)))
    return CsrMask(head, B, rp, ci[: n.value])


def build_all_csr(cfg: PatternConfig) -> List[CsrMask]:
    """to_csr(build_all_masks(cfg)) (pattern.cpp:160-166, csr.cpp:49-54)."""
    cfg.validate()
    return [build_csr(cfg, h) for h in range(cfg.num_heads)]


def build_csc(cfg: PatternConfig, head: int) -> CsrMask:
    """Transposed layout (column j -> ascending attending rows) for backward."""
    c, keep = cfg.to_c()
    n = ctypes.c_int64()
    check(lib().s2_layout_nnz(ctypes.byref(c), head, ctypes.byref(n)))
    B = cfg.num_blocks()
    cp = np.zeros(B + 1, np.int32)
    ri = np.zeros(max(n.value, 1), np.int32)
    check(lib().s2_layout_build_csc(ctypes.byref(c), head, _iptr(cp), _iptr(ri)))
    return CsrMask(head, B, cp, ri[: n.value])


def evict_after(cfg: PatternConfig, head: int) -> np.ndarray:
    """HeadCacheSchedule::evict_after (analysis.cpp:76-82)."""
    c, keep = cfg.to_c()
    ev = np.zeros(cfg.num_blocks(), np.int32)
    check(lib().s2_layout_evict_after(ctypes.byref(c), head, _iptr(ev)))
    return ev


def kv_efficient(cfg: PatternConfig, head: int) -> bool:
    """check_kv_cache_efficiency (verify.cpp:53-72)."""
    c, keep = cfg.to_c()
    ok = ctypes.c_int()
    check(lib().s2_layout_kv_efficient(ctypes.byref(c), head, ctypes.byref(ok)))
    return bool(ok.value)


# --------------------------------------------------------------- block masks
class HeadBlockMask:
    """pattern.hpp:64-92: B x B uint8 bits, row = query block."""

    def __init__(self, head_index: int, num_blocks: int, bits: Optional[np.ndarray] = None):
        self.head_index = head_index
        self._b = num_blocks
        self.bits = bits if bits is not None else np.zeros((num_blocks, num_blocks), np.uint8)

    def num_blocks(self) -> int:
        return self._b

    def at(self, i: int, j: int) -> bool:
        return bool(self.bits[i, j])

    def set(self, i: int, j: int, v: bool) -> None:
        self.bits[i, j] = 1 if v else 0

    def row(self, i: int) -> List[int]:
        return np.nonzero(self.bits[i])[0].tolist()

    def popcount(self) -> int:
        return int(self.bits.sum())

    def is_causal(self) -> bool:
        return not np.triu(self.bits, 1).any()

    def has_full_diagonal(self) -> bool:
        return bool(np.all(np.diag(self.bits)))

    def __eq__(self, other) -> bool:
        return (self.head_index == other.head_index and self._b == other._b
                and np.array_equal(self.bits, other.bits))


def same_bits(a: HeadBlockMask, b: HeadBlockMask) -> bool:
    return a.num_blocks() == b.num_blocks() and np.array_equal(a.bits, b.bits)


def from_csr(csr: CsrMask, num_blocks: int) -> HeadBlockMask:
    """csr.cpp:56-65 (validates first)."""
    if csr.num_blocks != num_blocks:
        raise _abi.S2InvalidArgument(1, "csr block count does not match requested num_blocks")
    csr.validate()
    m = HeadBlockMask(csr.head_index, num_blocks)
    for i in range(num_blocks):
        m.bits[i, csr.col_idx[csr.row_ptr[i]:csr.row_ptr[i + 1]]] = 1
    return m


def to_csr(mask: HeadBlockMask) -> CsrMask:
    """csr.cpp:35-47."""
    B = mask.num_blocks()
    tri = np.tril(mask.bits)
    counts = tri.sum(axis=1)
    rp = np.zeros(B + 1, np.int32)
    rp[1:] = np.cumsum(counts)
    ci = np.nonzero(tri)[1].astype(np.int32)
    return CsrMask(mask.head_index, B, rp, ci)


def build_head_mask(cfg: PatternConfig, head: int) -> HeadBlockMask:
    return from_csr(build_csr(cfg, head), cfg.num_blocks())


def build_all_masks(cfg: PatternConfig) -> List[HeadBlockMask]:
    return [from_csr(c, cfg.num_blocks()) for c in build_all_csr(cfg)]


def dense_causal_mask(num_blocks: int, head_index: int = 0) -> HeadBlockMask:
    return HeadBlockMask(head_index, num_blocks, np.tril(np.ones((num_blocks, num_blocks), np.uint8)))


@dataclass
class LayerSchedule:
    """pattern.hpp:98-104."""
    num_layers: int = 0
    dense_layer_ids: Set[int] = field(default_factory=set)
    sparse_pattern: PatternConfig = field(default_factory=PatternConfig)

    def validate(self) -> None:
        if self.num_layers < 1:
            raise _abi.S2InvalidArgument(1, "num_layers must be positive")
        for i in self.dense_layer_ids:
            if i < 0 or i >= self.num_layers:
                raise _abi.S2InvalidArgument(1, f"dense layer id {i} outside [0, num_layers)")
        self.sparse_pattern.validate()

    def layer_config(self, layer: int) -> PatternConfig:
        """Dense layers use make_dense_config of the same shape (== dense_causal_mask)."""
        p = self.sparse_pattern
        if layer in self.dense_layer_ids:
            cfg = make_dense_config(p.seq_len, p.block_size, p.num_heads)
            cfg.num_kv_heads = p.num_kv_heads
            return cfg
        return p


def build_layer_masks(schedule: LayerSchedule) -> List[List[HeadBlockMask]]:
    """pattern.cpp:168-181."""
    schedule.validate()
    sparse = build_all_masks(schedule.sparse_pattern)
    B = schedule.sparse_pattern.num_blocks()
    dense = [dense_causal_mask(B, h) for h in range(len(sparse))]
    return [dense if l in schedule.dense_layer_ids else sparse for l in range(schedule.num_layers)]


# ------------------------------------------------------------------ factories
def make_single_stride_config(seq_len: int, block_size: int, num_heads: int, local_blocks: int,
                              remote_stride: int, local_stride: int = 1) -> PatternConfig:
    """pattern.cpp:190-204 (the vert_stride policy of DKernel)."""
    cfg = PatternConfig(seq_len, block_size, num_heads, num_heads, local_blocks, local_stride)
    if local_blocks < cfg.num_blocks():
        cfg.stride_segments.append(StrideSegment(local_blocks, cfg.num_blocks(), remote_stride))
    cfg.validate()
    return cfg


def make_multi_stride_config(seq_len, block_size, num_heads, local_blocks, mid_block_distance,
                             stride1, stride2) -> PatternConfig:
    """pattern.cpp:206-220."""
    cfg = PatternConfig(seq_len, block_size, num_heads, num_heads, local_blocks, 1)
    cfg.stride_segments.append(StrideSegment(local_blocks, mid_block_distance, stride1))
    cfg.stride_segments.append(StrideSegment(mid_block_distance, cfg.num_blocks(), stride2))
    cfg.validate()
    return cfg


def make_sliding_window_config(seq_len, block_size, num_heads, window_blocks) -> PatternConfig:
    """pattern.cpp:222-231."""
    cfg = PatternConfig(seq_len, block_size, num_heads, num_heads, window_blocks, 1)
    cfg.validate()
    return cfg


def make_dense_config(seq_len, block_size, num_heads) -> PatternConfig:
    """pattern.cpp:233-236."""
    return make_single_stride_config(seq_len, block_size, num_heads, 1, 1)


def make_s2_config(seq_len: int, num_heads: int, *, block_size: int = 64, local_blocks: int = 4,
                   vert_stride: int = 16, homo_head: bool = False, num_kv_heads: int = 0,
                   offsets: Optional[Sequence[int]] = None) -> PatternConfig:
    """north_star vocabulary: block_size / local_blocks / vert_stride / homo_head.

    homo_head=False -> HeadModStride offsets (o_h = group(h) mod v);
    homo_head=True  -> every head offset 0 (SURVEY §0 mapping)."""
    cfg = PatternConfig(seq_len, block_size, num_heads, num_kv_heads, local_blocks, 1)
    B = cfg.num_blocks()
    if local_blocks < B:
        offs = list(offsets) if offsets is not None else ([0] * num_heads if homo_head else [])
        cfg.stride_segments.append(StrideSegment(local_blocks, B, vert_stride, offs))
    cfg.validate()
    return cfg
