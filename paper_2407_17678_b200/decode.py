"""Sparse decode over a per-(batch, kv-head) compacted KV cache (north_star item 4).

The cache stores, per kv head, only the key blocks its decode rows can still
attend (simulate_decode_cache semantics, /root/reference/proj/src/
analysis.cpp:57-104): stripe blocks stay, local-window blocks are evicted as
the window moves.  Requires a KV-efficient mask (verify.cpp:53-72).
"""
from __future__ import annotations

import ctypes
from typing import Optional

from ._abi import check, lib
from . import _abi


class KVCache:
    def __init__(self, plan, batch: int, head_dim: int):
        self.plan = plan
        self.batch = batch
        self.head_dim = head_dim
        h = ctypes.c_void_p()
        check(lib().s2_kvcache_create(plan.handle, batch, head_dim, _abi.S2_DTYPE_BF16,
                                      ctypes.byref(h)))
        self._h = h
        ws = ctypes.c_size_t()
        check(lib().s2_attn_decode_workspace_size(self._h, ctypes.byref(ws)))
        self._ws_bytes = ws.value
        self._ws = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().s2_kvcache_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def length(self) -> int:
        n = ctypes.c_int()
        check(lib().s2_kvcache_length(self._h, ctypes.byref(n)))
        return n.value

    def bytes(self):
        """(pool bytes, dense-cache bytes)."""
        a, b = ctypes.c_int64(), ctypes.c_int64()
        check(lib().s2_kvcache_bytes(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def retained_tokens(self, kv_head: int) -> int:
        n = ctypes.c_int64()
        check(lib().s2_kvcache_retained_tokens(self._h, kv_head, ctypes.byref(n)))
        return n.value

    def decode_bytes(self) -> int:
        n = ctypes.c_int64()
        check(lib().s2_attn_decode_bytes(self._h, ctypes.byref(n)))
        return n.value

    def _check(self, what, want_shape, *ts):
        """The C ABI reads these through raw pointers: shapes and dtype first."""
        import torch

        for t in ts:
            if t.dtype != torch.bfloat16:
                raise _abi.S2InvalidArgument(1, f"{what}: bfloat16 tensors required")
            if tuple(t.shape) != tuple(want_shape):
                raise _abi.S2InvalidArgument(1, f"{what}: expected shape {tuple(want_shape)}, got {tuple(t.shape)}")

    def prefill(self, k, v, stream=None):
        """k, v: [batch, Hkv, T, D] bf16 CUDA tensors (dense prefix)."""
        from .attention import _require_cuda, _stream_ptr

        _require_cuda(k, v)
        if k.dim() != 4:
            raise _abi.S2InvalidArgument(1, "prefill: k/v must be [batch, Hkv, T, D]")
        if k.shape[2] > self.plan.seq_len:
            raise _abi.S2InvalidArgument(1, "prefill: T exceeds the plan's seq_len (the cache capacity)")
        self._check("prefill", (self.batch, self.plan.num_kv_heads, k.shape[2], self.head_dim), k, v)
        check(lib().s2_kvcache_prefill(self._h, ctypes.c_void_p(k.data_ptr()),
                                       ctypes.c_void_p(v.data_ptr()), k.shape[2],
                                       _stream_ptr(stream)))

    def append(self, k, v, stream=None):
        """k, v: [batch, Hkv, D] bf16 — the token at position `length`."""
        from .attention import _require_cuda, _stream_ptr

        _require_cuda(k, v)
        self._check("append", (self.batch, self.plan.num_kv_heads, self.head_dim), k, v)
        check(lib().s2_kvcache_append(self._h, ctypes.c_void_p(k.data_ptr()),
                                      ctypes.c_void_p(v.data_ptr()), _stream_ptr(stream)))

    def decode(self, q, scale: Optional[float] = None, out=None, lse=None, stream=None):
        """q: [batch, H, D] bf16 at position length-1.  Returns (out [B,H,D], lse [B,H])."""
        import torch

        from .attention import _require_cuda, _stream_ptr

        _require_cuda(q)
        self._check("decode", (self.batch, self.plan.num_heads, self.head_dim), q)
        if out is None:
            out = torch.empty_like(q)
        if lse is None:
            lse = torch.empty(q.shape[:2], device=q.device, dtype=torch.float32)
        _require_cuda(out, lse)
        self._check("decode out", tuple(q.shape), out)
        if tuple(lse.shape) != tuple(q.shape[:2]) or lse.dtype != torch.float32:
            raise _abi.S2InvalidArgument(1, "decode: lse must be float32 [batch, H]")
        if self._ws is None:
            self._ws = torch.empty(max(self._ws_bytes, 16), dtype=torch.uint8, device=q.device)
        check(lib().s2_attn_decode(self._h, ctypes.c_void_p(q.data_ptr()),
                                   ctypes.c_void_p(out.data_ptr()),
                                   ctypes.c_void_p(lse.data_ptr()), 0.0 if scale is None else (-0.0 if scale == 0 else scale),
                                   ctypes.c_void_p(self._ws.data_ptr()), self._ws_bytes,
                                   _stream_ptr(stream)))
        return out, lse
