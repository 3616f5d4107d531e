"""JSON documents and config files: Python mirror of the reference's
serialize.hpp (/root/reference/proj/src/serialize.cpp) over the C ABI
(s2_pattern_to_json, s2_pattern_hash, s2_config_file_load, ...).

Documents are returned as parsed JSON values (dict / list), like
nlohmann::json in the reference; ``dumps`` gives the canonical text the
reference hashes (keys sorted, compact).  Errors: std::invalid_argument ->
S2InvalidArgument, load_config_file's std::runtime_error -> S2ConfigError.
"""
import ctypes
import json
from dataclasses import dataclass
from typing import Any, Optional

import numpy as np

from . import _abi
from ._abi import check, lib
from .pattern import CsrMask, LayerSchedule, PatternConfig, StrideSegment


def dumps(doc: Any) -> str:
    """nlohmann::json::dump() of a reference document (sorted keys, compact)."""
    return json.dumps(doc, sort_keys=True, separators=(",", ":"))


def _text(fn, *args) -> str:
    n = ctypes.c_size_t()
    check(fn(*args, None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value + 1)
    check(fn(*args, buf, n.value + 1, ctypes.byref(n)))
    return buf.value.decode()


def _pattern_from_c(c) -> PatternConfig:
    segs = []
    for i in range(c.num_segments):
        g = c.segments[i]
        offs = [g.offsets[k] for k in range(g.num_offsets)] if g.num_offsets > 0 else []
        segs.append(StrideSegment(g.start_block_distance, g.end_block_distance, g.stride, offs))
    return PatternConfig(c.seq_len, c.block_size, c.num_heads, c.num_kv_heads, c.local_blocks,
                         c.local_stride, segs)


def _schedule_to_c(s: LayerSchedule):
    c = _abi.s2_layer_schedule()
    ids = sorted(s.dense_layer_ids)
    arr = (ctypes.c_int * max(1, len(ids)))(*ids)
    c.num_layers, c.num_dense = s.num_layers, len(ids)
    c.dense_layer_ids = ctypes.cast(arr, ctypes.POINTER(ctypes.c_int))
    pc, keep = s.sparse_pattern.to_c()
    c.sparse_pattern = pc
    return c, (arr, keep)


def _schedule_from_c(c) -> LayerSchedule:
    return LayerSchedule(c.num_layers, {c.dense_layer_ids[i] for i in range(c.num_dense)},
                         _pattern_from_c(c.sparse_pattern))


def pattern_to_json(cfg: PatternConfig) -> dict:
    """to_json(const PatternConfig&) (serialize.cpp:30-47)."""
    c, keep = cfg.to_c()
    return json.loads(_text(lib().s2_pattern_to_json, ctypes.byref(c)))


def schedule_to_json(schedule: LayerSchedule) -> dict:
    """to_json(const LayerSchedule&) (serialize.cpp:49-53)."""
    c, keep = _schedule_to_c(schedule)
    return json.loads(_text(lib().s2_schedule_to_json, ctypes.byref(c)))


def csr_to_json(csr: CsrMask) -> dict:
    """to_json(const CsrMask&) (serialize.cpp:68-73)."""
    rp = np.ascontiguousarray(csr.row_ptr, dtype=np.int32)
    ci = np.ascontiguousarray(csr.col_idx, dtype=np.int32)
    ip = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))  # noqa: E731
    return json.loads(_text(lib().s2_csr_to_json, csr.head_index, csr.num_blocks, ip(rp), ip(ci)))


def to_json(obj) -> dict:
    """Overloads of the reference's to_json."""
    if isinstance(obj, PatternConfig):
        return pattern_to_json(obj)
    if isinstance(obj, LayerSchedule):
        return schedule_to_json(obj)
    if isinstance(obj, CsrMask):
        return csr_to_json(obj)
    raise TypeError(f"no to_json for {type(obj).__name__}")


def _as_text(j) -> bytes:
    return (j if isinstance(j, str) else dumps(j)).encode()


def pattern_config_from_json(j) -> PatternConfig:
    """pattern_config_from_json (serialize.cpp:75-95); validates."""
    c = _abi.s2_pattern_config()
    offs = (ctypes.c_int * 4096)()
    check(lib().s2_pattern_from_json(_as_text(j), ctypes.byref(c), offs, 4096))
    return _pattern_from_c(c)


def layer_schedule_from_json(j, default_pattern: PatternConfig) -> LayerSchedule:
    """layer_schedule_from_json (serialize.cpp:97-106)."""
    c = _abi.s2_layer_schedule()
    dense = (ctypes.c_int * 4096)()
    offs = (ctypes.c_int * 4096)()
    dc, keep = default_pattern.to_c()
    check(lib().s2_schedule_from_json(_as_text(j), ctypes.byref(dc), ctypes.byref(c), dense, 4096,
                                      offs, 4096))
    return _schedule_from_c(c)


def csr_from_json(j) -> CsrMask:
    """csr_from_json (serialize.cpp:108-116); validates (csr.cpp:11-33)."""
    t = _as_text(j)
    hi, nb, nnz = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
    L = lib()
    check(L.s2_csr_from_json(t, ctypes.byref(hi), ctypes.byref(nb), None, 0, None, 0,
                             ctypes.byref(nnz)))
    rp = np.zeros(nb.value + 1, np.int32)
    ci = np.zeros(max(1, nnz.value), np.int32)
    ip = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))  # noqa: E731
    check(L.s2_csr_from_json(t, ctypes.byref(hi), ctypes.byref(nb), ip(rp), rp.size, ip(ci),
                             ci.size, ctypes.byref(nnz)))
    return CsrMask(hi.value, nb.value, rp, ci[: nnz.value])


@dataclass
class CliConfigFile:
    """serialize.hpp:31-36."""
    pattern: PatternConfig
    schedule: Optional[LayerSchedule]
    out: str
    format: str


def load_config_file(path: str) -> CliConfigFile:
    """load_config_file (serialize.cpp:123-146): S2ConfigError names the file
    and the offending field."""
    f = _abi.s2_config_file()
    dense = (ctypes.c_int * 4096)()
    offs = (ctypes.c_int * 8192)()
    check(lib().s2_config_file_load(str(path).encode(), ctypes.byref(f), dense, 4096, offs, 8192))
    return CliConfigFile(_pattern_from_c(f.pattern),
                         _schedule_from_c(f.schedule) if f.has_schedule else None,
                         f.out.decode(), f.format.decode())


def config_hash(cfg: PatternConfig) -> int:
    """config_hash (serialize.cpp:148-156): FNV-1a 64 of the canonical document."""
    c, keep = cfg.to_c()
    h = ctypes.c_uint64()
    check(lib().s2_pattern_hash(ctypes.byref(c), ctypes.byref(h)))
    return h.value
