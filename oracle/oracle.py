"""ORACLE / TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke(), bench.py's
cpu_baseline and --impl reference legs).  Never imported by the product.

ctypes loaders for
  * ``port()``: oracle/lib/libs2oracle.so — the plain-C restatement
    (oracle/s2_oracle.c), built by ``make -C oracle port`` (gcc only, so it
    also builds on the GPU box);
  * ``ref()``: oracle/_ref/libshardattn_ref.so — the reference library compiled
    from /root/reference/proj/src (``make -C oracle ref``); None when absent.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "lib", "libs2oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libshardattn_ref.so")
REF_SRC = "/root/reference/proj/src"

_port = None
_ref = None

_F = ctypes.POINTER(ctypes.c_float)
_D = ctypes.POINTER(ctypes.c_double)
_IP = ctypes.POINTER(ctypes.c_int)
_I64P = ctypes.POINTER(ctypes.c_int64)


S2_MAX_SEGMENTS = 8  # include/s2attn.h


class _Segment(ctypes.Structure):
    """Mirror of include/s2attn.h's s2_stride_segment (POD), so the oracle needs
    nothing from the product package (bench.py's reference arm imports none of it)."""
    _fields_ = [("start_block_distance", ctypes.c_int), ("end_block_distance", ctypes.c_int),
                ("stride", ctypes.c_int), ("num_offsets", ctypes.c_int),
                ("offsets", ctypes.POINTER(ctypes.c_int))]


class PatternC(ctypes.Structure):
    """Mirror of include/s2attn.h's s2_pattern_config (the reference's PatternConfig
    as a POD, pattern.hpp:37-60)."""
    _fields_ = [("seq_len", ctypes.c_int), ("block_size", ctypes.c_int),
                ("num_heads", ctypes.c_int), ("num_kv_heads", ctypes.c_int),
                ("local_blocks", ctypes.c_int), ("local_stride", ctypes.c_int),
                ("num_segments", ctypes.c_int), ("segments", _Segment * S2_MAX_SEGMENTS)]


def single_stride(seq_len, block_size, num_heads, local_blocks, vert_stride, num_kv_heads=0):
    """make_single_stride_config (pattern.cpp:190-204) as the C struct: one segment
    {local_blocks, num_blocks, vert_stride} with the default head offsets."""
    c = PatternC()
    c.seq_len, c.block_size, c.num_heads = seq_len, block_size, num_heads
    c.num_kv_heads = num_kv_heads if num_kv_heads > 0 else num_heads
    c.local_blocks, c.local_stride = local_blocks, 1
    B = (seq_len + block_size - 1) // block_size
    if local_blocks < B:
        c.num_segments = 1
        c.segments[0].start_block_distance = local_blocks
        c.segments[0].end_block_distance = B
        c.segments[0].stride = vert_stride
    return c


def _cfg_type():
    # configs travel as pointers: the product's s2_pattern_config (tests) or PatternC
    # (same layout) both pass through ctypes.byref
    return ctypes.c_void_p


def build_port():
    src = os.path.join(HERE, "s2_oracle.c")
    if not os.path.exists(PORT_SO) or os.path.getmtime(PORT_SO) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", HERE, "port"])


def build_ref():
    if os.path.isdir(REF_SRC):
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"])


def port():
    global _port
    if _port is None:
        build_port()
        L = ctypes.CDLL(PORT_SO)
        C = _cfg_type()
        sig = {
            "s2o_num_blocks": (ctypes.c_int, [C]),
            "s2o_offset_for": (ctypes.c_int, [C, ctypes.c_int, ctypes.c_int]),
            "s2o_validate": (ctypes.c_int, [C, ctypes.c_char_p, ctypes.c_int]),
            "s2o_mask_bit": (ctypes.c_int, [C, ctypes.c_int, ctypes.c_int, ctypes.c_int]),
            "s2o_build_csr": (ctypes.c_int64, [C, ctypes.c_int, _IP, _IP]),
            "s2o_csc_from_csr": (None, [ctypes.c_int, _IP, _IP, _IP, _IP]),
            "s2o_evict_after": (None, [C, ctypes.c_int, _IP]),
            "s2o_kv_efficient": (ctypes.c_int, [C, ctypes.c_int]),
            "s2o_random_tensors": (None, [ctypes.c_int] * 3 + [ctypes.c_uint64, _F, _F, _F]),
            "s2o_attn_fwd": (None, [ctypes.c_int] * 6 + [ctypes.c_double, _F, _F, _F, _IP, _IP,
                                                         _F, _D]),
            "s2o_attn_bwd": (None, [ctypes.c_int] * 6 + [ctypes.c_double, _F, _F, _F, _F, _IP,
                                                         _IP, _F, _F, _F]),
            "s2o_attn_bwd_par": (None, [ctypes.c_int] * 6 + [ctypes.c_double, _F, _F, _F, _F, _IP,
                                                         _IP, _F, _F, _F]),
            "s2o_decode": (None, [ctypes.c_int] * 7 + [ctypes.c_double, _F, _F, _F,
                                                       _IP, _IP, ctypes.c_int, _F, _D]),
            "s2o_bwd_sample": (None, [ctypes.c_int] * 6 + [ctypes.c_double, _F, _F, _F, _F, _IP, _IP,
                                                           ctypes.c_int, _IP, _F, ctypes.c_int, _IP,
                                                           _F, _F]),
            "s2o_max_rel_f": (ctypes.c_double, [_F, _F, ctypes.c_int64]),
            "s2o_max_rel_d": (ctypes.c_double, [_D, _D, ctypes.c_int64]),
            "s2o_fnv1a64_u32": (ctypes.c_uint64, [ctypes.c_void_p, ctypes.c_int64]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        _port = L
    return _port


def ref():
    """The compiled reference, or None when it cannot be built/loaded here."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            try:
                build_ref()
            except Exception:
                return None
        if not os.path.exists(REF_SO):
            return None
        L = ctypes.CDLL(REF_SO)
        C = _cfg_type()
        sig = {
            "ref_last_error": (ctypes.c_char_p, []),
            "ref_validate": (ctypes.c_int, [C]),
            "ref_build_csr": (ctypes.c_int, [C, ctypes.c_int, _IP, _IP, _I64P]),
            "ref_build_all_csr": (ctypes.c_int, [C, _IP, _IP, _I64P]),
            "ref_csr_validate": (ctypes.c_int, [ctypes.c_int, _IP, _IP, ctypes.c_int64]),
            "ref_random_tensors": (ctypes.c_int, [ctypes.c_int] * 3 + [ctypes.c_uint64, _F, _F, _F]),
            "ref_streaming": (ctypes.c_int, [ctypes.c_int] * 4 + [ctypes.c_double, _F, _F, _F,
                                                                  ctypes.c_int, _IP, _IP,
                                                                  ctypes.c_int, _F, _D]),
            "ref_naive": (ctypes.c_int, [C, ctypes.c_int, ctypes.c_double, _F, _F, _F, _F, _D]),
            "ref_dense": (ctypes.c_int, [C, ctypes.c_int, ctypes.c_double, _F, _F, _F, _F, _D]),
            "ref_decode_cache": (ctypes.c_int, [C, ctypes.c_int, ctypes.c_int, _IP, _I64P, _IP]),
            "ref_kv_efficient": (ctypes.c_int, [C, ctypes.c_int, _IP]),
            "ref_exact_flops": (ctypes.c_int, [C, ctypes.c_int, _D, _D, _I64P]),
            "ref_config_json": (ctypes.c_int, [C, ctypes.c_char_p, ctypes.c_int]),
            "ref_config_hash": (ctypes.c_int, [C, ctypes.POINTER(ctypes.c_uint64)]),
            "ref_load_config": (ctypes.c_int, [ctypes.c_char_p] * 5 + [ctypes.c_int]),
            "ref_kv_reduction": (ctypes.c_int, [C, ctypes.c_int, _IP, ctypes.c_int, _D]),
            "ref_decode_cache_full": (ctypes.c_int, [C, ctypes.c_int, ctypes.c_int, _IP, _I64P, _IP,
                                                     _I64P, _D]),
            "ref_analytic": (ctypes.c_int, [ctypes.c_double] * 3 + [ctypes.c_int, _D, _D, _D]),
            "ref_max_relative_error_f": (ctypes.c_double, [_F, _F, ctypes.c_int64]),
            "ref_max_relative_error_d": (ctypes.c_double, [_D, _D, ctypes.c_int64]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        _ref = L
    return _ref


def fp(a):
    return a.ctypes.data_as(_F)


def dp(a):
    return a.ctypes.data_as(_D)


def ip(a):
    return a.ctypes.data_as(_IP)


# ------------------------------------------------------------ convenience
def csr_all(cfg):
    """Port: concatenated row_ptr [H*(B+1)] and col_idx for every head."""
    L = port()
    c, keep = cfg.to_c()
    B = cfg.num_blocks()
    rps, cis = [], []
    for h in range(cfg.num_heads):
        n = L.s2o_build_csr(ctypes.byref(c), h, None, None)
        rp = np.zeros(B + 1, np.int32)
        ci = np.zeros(max(n, 1), np.int32)
        L.s2o_build_csr(ctypes.byref(c), h, ip(rp), ip(ci))
        rps.append(rp)
        cis.append(ci[:n])
    return np.concatenate(rps), np.concatenate(cis) if cis else np.zeros(0, np.int32)


def csr_all_c(c):
    """Concatenated row_ptr [H*(B+1)] / col_idx of every head of a PatternC: the
    reference's own to_csr(build_all_masks) when oracle/_ref is built, else the
    port.  Returns (row_ptr, col_idx, kind)."""
    H = c.num_heads
    B = (c.seq_len + c.block_size - 1) // c.block_size
    R = ref()
    if R is not None:
        nnz = ctypes.c_int64()
        assert R.ref_build_all_csr(ctypes.byref(c), None, None, ctypes.byref(nnz)) == 0
        rp = np.zeros(H * (B + 1), np.int32)
        ci = np.zeros(max(nnz.value, 1), np.int32)
        assert R.ref_build_all_csr(ctypes.byref(c), ip(rp), ip(ci), ctypes.byref(nnz)) == 0
        return rp, ci[:nnz.value], "reference"
    L = port()
    rps, cis = [], []
    for h in range(H):
        n = L.s2o_build_csr(ctypes.byref(c), h, None, None)
        rp = np.zeros(B + 1, np.int32)
        ci = np.zeros(max(n, 1), np.int32)
        L.s2o_build_csr(ctypes.byref(c), h, ip(rp), ip(ci))
        rps.append(rp)
        cis.append(ci[:n])
    return np.concatenate(rps), np.concatenate(cis), "port"


def random_tensors(H, N, d, seed):
    """AttentionTensors::random's exact stream (mt19937_64 + libstdc++ mapping)."""
    n = H * N * d
    q = np.zeros(n, np.float32)
    k = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    port().s2o_random_tensors(H, N, d, seed, fp(q), fp(k), fp(v))
    return q, k, v


def attn_fwd(q, k, v, row_ptr, col_idx, batch, H, Hkv, N, D, S, scale=None):
    """Port streaming forward (fp64 accumulate).  Returns (out f32, lse f64)."""
    scale = 1.0 / np.sqrt(D) if scale is None else scale
    q = np.ascontiguousarray(q, np.float32)
    k = np.ascontiguousarray(k, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    out = np.zeros(batch * H * N * D, np.float32)
    lse = np.zeros(batch * H * N, np.float64)
    port().s2o_attn_fwd(batch, H, Hkv, N, D, S, scale, fp(q), fp(k), fp(v),
                        ip(np.ascontiguousarray(row_ptr, np.int32)),
                        ip(np.ascontiguousarray(col_idx, np.int32)), fp(out), dp(lse))
    return out, lse


def attn_bwd(q, k, v, dout, row_ptr, col_idx, batch, H, Hkv, N, D, S, scale=None):
    scale = 1.0 / np.sqrt(D) if scale is None else scale
    q, k, v, dout = (np.ascontiguousarray(x, np.float32) for x in (q, k, v, dout))
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    port().s2o_attn_bwd(batch, H, Hkv, N, D, S, scale, fp(q), fp(k), fp(v), fp(dout),
                        ip(np.ascontiguousarray(row_ptr, np.int32)),
                        ip(np.ascontiguousarray(col_idx, np.int32)), fp(dq), fp(dk), fp(dv))
    return dq, dk, dv


def attn_bwd_par(q, k, v, dout, row_ptr, col_idx, batch, H, Hkv, N, D, S, scale=None):
    """attn_bwd parallel inside a unit (s2o_attn_bwd_par): the same values, bit for
    bit; bench.py's CPU-baseline legs use it so that one head uses every core."""
    scale = 1.0 / np.sqrt(D) if scale is None else scale
    q, k, v, dout = (np.ascontiguousarray(x, np.float32) for x in (q, k, v, dout))
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    port().s2o_attn_bwd_par(batch, H, Hkv, N, D, S, scale, fp(q), fp(k), fp(v), fp(dout),
                            ip(np.ascontiguousarray(row_ptr, np.int32)),
                            ip(np.ascontiguousarray(col_idx, np.int32)), fp(dq), fp(dk), fp(dv))
    return dq, dk, dv


def decode(q, k, v, row_ptr, col_idx, batch, H, Hkv, T, D, S, t, B, scale=None):
    scale = 1.0 / np.sqrt(D) if scale is None else scale
    q, k, v = (np.ascontiguousarray(x, np.float32) for x in (q, k, v))
    out = np.zeros(batch * H * D, np.float32)
    lse = np.zeros(batch * H, np.float64)
    port().s2o_decode(batch, H, Hkv, T, D, S, t, scale, fp(q), fp(k), fp(v),
                      ip(np.ascontiguousarray(row_ptr, np.int32)),
                      ip(np.ascontiguousarray(col_idx, np.int32)), B, fp(out), dp(lse))
    return out, lse


def bwd_sample(q, k, v, dout, row_ptr, col_idx, batch, H, Hkv, N, D, S, q_rows, k_rows,
               scale=None):
    """s2o_attn_bwd's gradient at sampled rows (s2o_bwd_sample), for full-size
    parity: q_rows = [(b*H + h, i)] -> dq rows; k_rows = [(b*Hkv + g, j)] ->
    (dk, dv) rows.  q/dout [batch,H,N,D], k/v [batch,Hkv,N,D] fp32 (flat ok)."""
    scale = 1.0 / np.sqrt(D) if scale is None else scale
    q, k, v, dout = (np.ascontiguousarray(x, np.float32) for x in (q, k, v, dout))
    qs = np.ascontiguousarray(np.asarray(q_rows, np.int32).reshape(-1, 2))
    ks = np.ascontiguousarray(np.asarray(k_rows, np.int32).reshape(-1, 2))
    dq = np.zeros((len(qs), D), np.float32)
    dk = np.zeros((len(ks), D), np.float32)
    dv = np.zeros((len(ks), D), np.float32)
    port().s2o_bwd_sample(batch, H, Hkv, N, D, S, scale, fp(q), fp(k), fp(v), fp(dout),
                          ip(np.ascontiguousarray(row_ptr, np.int32)),
                          ip(np.ascontiguousarray(col_idx, np.int32)), len(qs), ip(qs), fp(dq),
                          len(ks), ip(ks), fp(dk), fp(dv))
    return dq, dk, dv


def max_rel(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    if a.dtype == np.float64:
        return port().s2o_max_rel_d(dp(a), dp(b.astype(np.float64)), a.size)
    return port().s2o_max_rel_f(fp(a.astype(np.float32)), fp(b.astype(np.float32)), a.size)
