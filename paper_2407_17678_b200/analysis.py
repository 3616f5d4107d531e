"""Layout analysis: Python mirror of the reference's analysis.hpp
(/root/reference/proj/src/analysis.cpp) over the C ABI.  The decode-cache
simulation is computed from the CSC in O(B + T) per head instead of the
reference's O(B^2 + T*B) mask scans; results are identical
(tests/test_serialize.py pins them against the reference)."""
import ctypes
from dataclasses import dataclass, field
from typing import List

import numpy as np

from . import _abi
from ._abi import check, lib
from .pattern import LayerSchedule, PatternConfig


def _d(fn, *args) -> float:
    out = ctypes.c_double()
    check(fn(*args, ctypes.byref(out)))
    return out.value


def equivalent_context_length(seq_len: float, local_window: float, stride: float) -> float:
    """analysis.cpp:13-18."""
    return _d(lib().s2_equivalent_context_length, float(seq_len), float(local_window), float(stride))


def analytic_flops_reduction(seq_len: float, local_window: float, stride: float) -> float:
    """analysis.cpp:20-22."""
    return _d(lib().s2_analytic_flops_reduction, float(seq_len), float(local_window), float(stride))


def speedup_upper_bound(num_heads: int, seq_len: float, local_window: float) -> float:
    """analysis.cpp:24-27."""
    return _d(lib().s2_speedup_upper_bound, int(num_heads), float(seq_len), float(local_window))


def flops_per_block_pair(head_dim: int, block_size: int) -> float:
    """analysis.cpp:29-31: 4 * head_dim * block_size^2."""
    return 4.0 * head_dim * float(block_size) * block_size


@dataclass
class FlopsReport:
    """analysis.hpp:30-36."""
    dense_flops: float = 0.0
    sparse_flops: float = 0.0
    reduction_factor: float = 0.0
    equivalent_context: float = 0.0
    nnz_per_head: List[int] = field(default_factory=list)


def exact_flops(config: PatternConfig, head_dim: int) -> FlopsReport:
    """analysis.cpp:33-55."""
    c, keep = config.to_c()
    r = _abi.s2_flops_report()
    nph = np.zeros(max(1, config.num_heads), np.int64)
    check(lib().s2_exact_flops(ctypes.byref(c), head_dim, ctypes.byref(r),
                               nph.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
    return FlopsReport(r.dense_flops, r.sparse_flops, r.reduction_factor, r.equivalent_context,
                       nph[: config.num_heads].tolist())


@dataclass
class HeadCacheSchedule:
    """analysis.hpp:43-57."""
    head_index: int
    evict_after: np.ndarray
    occupancy: np.ndarray
    dead_blocks: np.ndarray
    peak_tokens: int
    mean_tokens: float


@dataclass
class CacheSchedule:
    """analysis.hpp:59-64."""
    block_size: int
    num_blocks: int
    total_tokens: int
    heads: List[HeadCacheSchedule]


def simulate_decode_cache(config: PatternConfig, total_tokens: int) -> CacheSchedule:
    """analysis.cpp:57-104."""
    c, keep = config.to_c()
    L = lib()
    B = config.num_blocks()
    heads = []
    for h in range(config.num_heads):
        ev = np.zeros(B, np.int32)
        occ = np.zeros(max(1, total_tokens), np.int64)
        dead = np.zeros(max(1, total_tokens), np.int32)
        pk, mean = ctypes.c_int64(), ctypes.c_double()
        ip = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))  # noqa: E731
        check(L.s2_simulate_decode_cache(ctypes.byref(c), total_tokens, h, ip(ev),
                                         occ.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ip(dead),
                                         ctypes.byref(pk), ctypes.byref(mean)))
        heads.append(HeadCacheSchedule(h, ev, occ, dead, pk.value, mean.value))
    return CacheSchedule(config.block_size, B, total_tokens, heads)


def kv_reduction(schedule: LayerSchedule) -> float:
    """analysis.cpp:106-121: percent of KV cache saved vs dense."""
    from .serialize import _schedule_to_c

    c, keep = _schedule_to_c(schedule)
    return _d(lib().s2_kv_reduction, ctypes.byref(c))
