"""Shared test helpers: golden fixtures, config (de)serialisation."""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
GOLDEN = os.path.join(HERE, "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)

from paper_2407_17678_b200.pattern import PatternConfig, StrideSegment  # noqa: E402


def cfg_from_dict(d) -> PatternConfig:
    return PatternConfig(d["seq_len"], d["block_size"], d["num_heads"], d["num_kv_heads"],
                         d["local_blocks"], d["local_stride"],
                         [StrideSegment(s["start_block_distance"], s["end_block_distance"],
                                        s["stride"], list(s.get("offsets", [])))
                          for s in d["stride_segments"]])


def single(N, S, H, local, v, local_stride=1, kv=0, offsets=None) -> PatternConfig:
    c = PatternConfig(N, S, H, kv if kv else H, local, local_stride)
    B = c.num_blocks()
    if local < B:
        c.stride_segments.append(StrideSegment(local, B, v, list(offsets or [])))
    return c


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def load_npz(name):
    return np.load(os.path.join(GOLDEN, name))


def fnv_fast(arr) -> str:
    """FNV-1a 64 over 32-bit words; must match oracle/make_golden.py::fnv_fast.
    Folded in C by the oracle library (s2o_fnv1a64_u32) so every head of a 128K
    layout is fingerprinted quickly; the Python fold below is its cross-check."""
    import oracle

    a = np.ascontiguousarray(arr, dtype=np.uint32)
    return f"{oracle.port().s2o_fnv1a64_u32(a.ctypes.data, a.size):016x}"


def fnv_py(arr) -> str:
    a = np.ascontiguousarray(arr, dtype=np.uint32).astype(np.uint64)
    h = 0xCBF29CE484222325
    prime = 0x100000001B3
    mask = 0xFFFFFFFFFFFFFFFF
    for w in a.tolist():
        h = ((h ^ w) * prime) & mask
    return f"{h:016x}"


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (RNE) -> fp32, exactly like torch's .to(bfloat16)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return (r & 0xFFFFFFFF).astype(np.uint32).view(np.float32)
