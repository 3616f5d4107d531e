"""S2 attention entry points over the C ABI (sm_100a kernels).

Two surfaces:

* the reference-shaped host API — ``AttentionTensors``,
  ``streaming_sharded_attention`` and ``dsplit_attention`` with the exact
  argument meaning and error behaviour of
  /root/reference/proj/include/shardattn/attention.hpp:17-66 (fp32 host arrays
  in, ``out``/``lse`` overwritten), executed on the GPU; and
* the device API — ``s2_attn_fwd`` / ``s2_attn_bwd`` on torch CUDA tensors
  ([batch, heads, seq, dim], bf16 or fp32) and the autograd op
  ``s2_attention``.

torch is used only for device memory and streams; all math runs in
libs2attn.so.  There is no CPU fallback: every call fails loudly when the
library or the GPU is missing.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _abi
from ._abi import check, lib
from .pattern import CsrMask, PatternConfig


class Plan:
    """Owns an s2_plan: per-head CSR + tile work lists, uploaded lazily."""

    def __init__(self, handle, num_heads, num_kv_heads, seq_len, block_size):
        self._h = handle
        self.num_heads = num_heads
        self.num_kv_heads = num_kv_heads
        self.seq_len = seq_len
        self.block_size = block_size

    @classmethod
    def from_config(cls, cfg: PatternConfig) -> "Plan":
        c, keep = cfg.to_c()
        h = ctypes.c_void_p()
        check(lib().s2_plan_create(ctypes.byref(c), ctypes.byref(h)))
        return cls(h, cfg.num_heads, cfg.kv_heads(), cfg.seq_len, cfg.block_size)

    @classmethod
    def from_csr(cls, csr: Sequence[CsrMask], seq_len: int, block_size: int,
                 num_kv_heads: int = 0) -> "Plan":
        H = len(csr)
        if H == 0:
            raise _abi.S2InvalidArgument(1, "csr list is empty")
        B = -(-seq_len // block_size) if block_size > 0 else 0
        rps, cis = [], []
        for c in csr:
            if c.num_blocks != csr[0].num_blocks:
                raise _abi.S2InvalidArgument(1, "csr masks differ in block count")
            rp = np.ascontiguousarray(c.row_ptr, dtype=np.int32)
            ci = np.ascontiguousarray(c.col_idx, dtype=np.int32)
            if rp.size != B + 1 or c.num_blocks != B:
                raise _abi.S2InvalidArgument(
                    1, "mask block count does not match ceil(seq_len/block_size)")
            if ci.size == 0:
                ci = np.zeros(1, np.int32)
            rps.append(rp)
            cis.append(ci)
        RP = (ctypes.POINTER(ctypes.c_int) * H)(
            *[r.ctypes.data_as(ctypes.POINTER(ctypes.c_int)) for r in rps])
        CI = (ctypes.POINTER(ctypes.c_int) * H)(
            *[c.ctypes.data_as(ctypes.POINTER(ctypes.c_int)) for c in cis])
        h = ctypes.c_void_p()
        check(lib().s2_plan_create_from_csr(H, num_kv_heads, seq_len, block_size, RP, CI,
                                            ctypes.byref(h)))
        return cls(h, H, num_kv_heads if num_kv_heads > 0 else H, seq_len, block_size)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().s2_plan_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    def stats(self) -> dict:
        st = _abi.s2_plan_stats()
        check(lib().s2_plan_get_stats(self._h, ctypes.byref(st)))
        return {name: getattr(st, name) for name, _ in st._fields_}

    def head_nnz(self, head: int) -> int:
        n = ctypes.c_int64()
        check(lib().s2_plan_head_nnz(self._h, head, ctypes.byref(n)))
        return n.value

    def fwd_flops(self, batch: int, head_dim: int):
        """(active-block FLOPs, dense-causal FLOPs), analysis.cpp:29-55 counting."""
        a, d = ctypes.c_double(), ctypes.c_double()
        check(lib().s2_plan_fwd_flops(self._h, batch, head_dim, ctypes.byref(a), ctypes.byref(d)))
        return a.value, d.value

    def unit_weights(self, batch: int) -> np.ndarray:
        w = np.zeros(batch * self.num_kv_heads, np.int64)
        check(lib().s2_plan_unit_weights(self._h, batch,
                                         w.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        return w


def _dtype_code(t):
    import torch

    if t.dtype == torch.bfloat16:
        return _abi.S2_DTYPE_BF16
    if t.dtype == torch.float32:
        return _abi.S2_DTYPE_F32
    raise _abi.S2InvalidArgument(1, f"unsupported dtype {t.dtype} (bf16 or float32)")


def _stream_ptr(stream):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _require_cuda(*ts):
    for t in ts:
        if not t.is_cuda:
            raise _abi.S2InvalidArgument(1, "tensors must live on a CUDA device (no CPU path)")
        if not t.is_contiguous():
            raise _abi.S2InvalidArgument(1, "tensors must be contiguous")


def _check_tensors(q, k, v, out=None, lse=None, dout=None, grads=(), unit_ids=None, plan=None):
    """Shapes / dtypes / devices the C ABI takes on trust (it receives pointers):
    mismatches raise here instead of reading out of bounds (kernel_common.hpp:20-32's
    size checks, for device tensors).  With the plan, the head counts are checked
    against it too (the kernels size their TMA maps and head lists from the plan)."""
    import torch

    def bad(msg):
        raise _abi.S2InvalidArgument(1, msg)

    if q.dtype not in (torch.bfloat16, torch.float32):
        bad("q must be bfloat16 or float32")
    if k.dtype != q.dtype or v.dtype != q.dtype:
        bad("q, k and v must share one dtype")
    if k.shape != v.shape:
        bad("k and v shapes differ")
    if unit_ids is None:
        if q.dim() != 4 or k.dim() != 4:
            bad("q must be [B, H, N, D] and k/v [B, Hkv, N, D]")
        if k.shape[0] != q.shape[0] or k.shape[2] != q.shape[2] or k.shape[3] != q.shape[3]:
            bad("q and k/v disagree in batch, seq_len or head_dim")
        if plan is not None and (q.shape[1] != plan.num_heads or k.shape[1] != plan.num_kv_heads):
            bad("q / k heads do not match the plan's num_heads / num_kv_heads")
    else:
        if q.dim() != 4 or k.dim() != 3:
            bad("with unit_ids, q must be [U, H/Hkv, N, D] and k/v [U, N, D]")
        if k.shape[0] != q.shape[0] or k.shape[1] != q.shape[2] or k.shape[2] != q.shape[3]:
            bad("q and k/v disagree in units, seq_len or head_dim")
        if len(unit_ids) != q.shape[0]:
            bad("len(unit_ids) must equal the packed unit dimension")
        if plan is not None and q.shape[1] != plan.num_heads // plan.num_kv_heads:
            bad("with unit_ids, q's second dimension must be the plan's num_heads / num_kv_heads")
    devs = {t.device for t in (q, k, v, out, lse, dout, *grads) if t is not None}
    if len(devs) != 1:
        bad("tensors live on different devices")
    if out is not None and (out.shape != q.shape or out.dtype != q.dtype):
        bad("out must have q's shape and dtype")
    if lse is not None and (tuple(lse.shape) != tuple(q.shape[:-1]) or lse.dtype != torch.float32):
        bad("lse must be float32 with q's shape without head_dim")
    if dout is not None and (dout.shape != q.shape or dout.dtype != q.dtype):
        bad("dout must have q's shape and dtype")
    for g, ref in zip(grads, (q, k, v)):
        if g is not None and (g.shape != ref.shape or g.dtype != ref.dtype):
            bad("dq/dk/dv must have the shapes and dtype of q/k/v")


def _fwd_args(plan, q, k, v, out, lse, scale, num_splits, unit_ids):
    if unit_ids is None:
        B, H, N, D = q.shape
        Hkv = k.shape[1]
        nu = 0
        uptr = None
        keep = None
    else:
        U, hpg, N, D = q.shape
        H = plan.num_heads
        Hkv = plan.num_kv_heads
        B = 0
        arr = np.ascontiguousarray(unit_ids, dtype=np.int32)
        B = int(arr.max()) // Hkv + 1 if arr.size else 1
        nu = int(arr.size)
        keep = arr
        uptr = arr.ctypes.data_as(ctypes.POINTER(ctypes.c_int))
    a = _abi.s2_attn_args()
    a.dtype = _dtype_code(q)
    a.batch, a.num_heads, a.num_kv_heads, a.seq_len, a.head_dim = B, H, Hkv, N, D
    # None: 1/sqrt(D) (+0.0 in the ABI); an explicit 0 is the reference's literal
    # zero scale (uniform weights), S2_SCALE_ZERO = -0.0
    a.scale = 0.0 if scale is None else (-0.0 if float(scale) == 0.0 else float(scale))
    a.num_splits = num_splits
    a.num_units = nu
    a.unit_ids = uptr
    a.q, a.k, a.v = q.data_ptr(), k.data_ptr(), v.data_ptr()
    a.out, a.lse = out.data_ptr(), lse.data_ptr()
    return a, keep


def s2_attn_fwd(plan: Plan, q, k, v, *, scale: Optional[float] = None, num_splits: int = 1,
                out=None, lse=None, unit_ids=None, stream=None):
    """Sparse forward on device tensors.  q [B,H,N,D], k/v [B,Hkv,N,D] (bf16 -> tcgen05
    kernel, fp32 -> reference-precision kernel).  Returns (out, lse[B,H,N] fp32)."""
    import torch

    _require_cuda(q, k, v)
    if out is None:
        out = torch.empty_like(q)
    if lse is None:
        lse = torch.empty(q.shape[:-1], device=q.device, dtype=torch.float32)
    _require_cuda(out, lse)
    _check_tensors(q, k, v, out, lse, unit_ids=unit_ids, plan=plan)
    a, keep = _fwd_args(plan, q, k, v, out, lse, scale, num_splits, unit_ids)
    check(lib().s2_attn_fwd(plan.handle, ctypes.byref(a), _stream_ptr(stream)))
    return out, lse


def s2_attn_fwd_peers(plan: Plan, q, k, v, *, unit_ids, peer_out, peer_lse, unit_global, total_units: int,
                      scale: Optional[float] = None, out=None, lse=None, stream=None):
    """Forward of this rank's packed units with the output exchange fused in
    (s2_attn_fwd_peers): every O tile also lands in each rank's full output
    (`peer_out[r]` [total_units, hpg, N, D], `peer_lse[r]` [total_units, hpg, N],
    device tensors mapped into this process), at the global unit
    `unit_global[i]` (int32 device tensor) of local unit i.  Returns the local
    (out, lse); the caller orders the ranks' completion before reading the
    full buffers."""
    import torch

    _require_cuda(q, k, v, unit_global, *peer_out, *peer_lse)
    if out is None:
        out = torch.empty_like(q)
    if lse is None:
        lse = torch.empty(q.shape[:-1], device=q.device, dtype=torch.float32)
    _require_cuda(out, lse)
    _check_tensors(q, k, v, out, lse, unit_ids=unit_ids, plan=plan)
    full = (int(total_units),) + tuple(q.shape[1:])
    for po_, pl_ in zip(peer_out, peer_lse):
        if tuple(po_.shape) != full or po_.dtype != q.dtype or tuple(pl_.shape) != full[:-1]:
            raise _abi.S2InvalidArgument(1, "peer buffers must be [total_units, H/Hkv, N, D] / [.., N]")
    if unit_global.numel() != q.shape[0]:
        raise _abi.S2InvalidArgument(1, "unit_global must list one global unit per local unit")
    a, keep = _fwd_args(plan, q, k, v, out, lse, scale, 1, unit_ids)
    n = len(peer_out)
    if len(peer_lse) != n:
        raise _abi.S2InvalidArgument(1, "peer_out and peer_lse differ in length")
    po = (ctypes.c_void_p * n)(*[t.data_ptr() for t in peer_out])
    pl = (ctypes.c_void_p * n)(*[t.data_ptr() for t in peer_lse])
    ug = unit_global.to(torch.int32).contiguous()
    check(lib().s2_attn_fwd_peers(plan.handle, ctypes.byref(a), n, po, pl, ctypes.c_void_p(ug.data_ptr()),
                                  int(total_units), _stream_ptr(stream)))
    return out, lse


def s2_attn_bwd(plan: Plan, q, k, v, out, lse, dout, *, scale: Optional[float] = None,
                dq=None, dk=None, dv=None, unit_ids=None, stream=None):
    """Sparse backward: (dq, dk, dv).  dK/dV tiles are owned by one CTA each (no atomics).
    bf16 with head_dim 64 / 128 and block_size % 16 == 0 -> tcgen05 kernels; fp32 (and
    other bf16 shapes) with head_dim <= 128 -> reference-precision FFMA kernels;
    head_dim > 128 otherwise raises S2Unsupported."""
    import torch

    _require_cuda(q, k, v, out, lse, dout)
    dq = torch.empty_like(q) if dq is None else dq
    dk = torch.empty_like(k) if dk is None else dk
    dv = torch.empty_like(v) if dv is None else dv
    _require_cuda(dq, dk, dv)
    _check_tensors(q, k, v, out, lse, dout, (dq, dk, dv), unit_ids=unit_ids, plan=plan)
    fa, keep = _fwd_args(plan, q, k, v, out, lse, scale, 1, unit_ids)
    a = _abi.s2_attn_bwd_args()
    a.fwd = fa
    a.dout, a.dq, a.dk, a.dv = dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr()
    ws = ctypes.c_size_t()
    check(lib().s2_attn_bwd_workspace_size(plan.handle, ctypes.byref(a), ctypes.byref(ws)))
    work = torch.empty(max(ws.value, 1), dtype=torch.uint8, device=q.device)
    check(lib().s2_attn_bwd(plan.handle, ctypes.byref(a), ctypes.c_void_p(work.data_ptr()),
                            ws.value, _stream_ptr(stream)))
    return dq, dk, dv


def s2_attn_fwd_bwd_host(plan: Plan, q, k, v, dout, out, lse, dq, dk, dv, *,
                         scale: Optional[float] = None, num_chunks: int = 4, stream=None,
                         workspace=None):
    """One layer's forward + backward on HOST tensors (pinned CPU torch tensors,
    bf16 or fp32; lse fp32): the reference API's host-resident data path.  The C ABI
    pipelines H2D copies, kernels and D2H copies over `num_chunks` chunks of
    (batch, kv-group) units (s2_attn_fwd_bwd_host).  Returns when the work is
    queued on `stream`; synchronize before reading the outputs."""
    import torch

    for t in (q, k, v, dout, out, lse, dq, dk, dv):
        if t.is_cuda:
            raise _abi.S2InvalidArgument(1, "s2_attn_fwd_bwd_host takes host tensors")
    a = _abi.s2_attn_bwd_args()
    B, H, N, D = q.shape
    f = a.fwd
    f.dtype = _dtype_code(q)
    f.batch, f.num_heads, f.num_kv_heads, f.seq_len, f.head_dim = B, H, k.shape[1], N, D
    f.scale = 0.0 if scale is None else float(scale)
    f.num_splits, f.num_units, f.unit_ids = 1, 0, None
    f.q, f.k, f.v, f.out, f.lse = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr()
    a.dout, a.dq, a.dk, a.dv = dout.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr()
    ws = ctypes.c_size_t()
    check(lib().s2_attn_fwd_bwd_host_workspace_size(plan.handle, ctypes.byref(a), num_chunks,
                                                     ctypes.byref(ws)))
    if workspace is None or workspace.numel() < ws.value:
        workspace = torch.empty(ws.value, dtype=torch.uint8, device="cuda")
    check(lib().s2_attn_fwd_bwd_host(plan.handle, ctypes.byref(a), num_chunks,
                                     ctypes.c_void_p(workspace.data_ptr()), ws.value,
                                     _stream_ptr(stream)))
    return workspace


def s2_attention(q, k, v, plan: Plan, scale: Optional[float] = None):
    """Differentiable S2 attention (DKernel's plug-in role): the
    `s2attn::fwd` torch.library op, whose registered autograd formula calls
    `s2attn::bwd` (torch_ops.py)."""
    from .torch_ops import s2_attention as op

    return op(q, k, v, plan, scale)


# ----------------------------------------------------- reference-shaped API
@dataclass
class AttentionTensors:
    """attention.hpp:17-37: q/k/v/out fp32 [H, N, d] flat, lse fp64 [H, N]."""
    num_heads: int = 0
    seq_len: int = 0
    head_dim: int = 0
    scale: float = 0.0
    q: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    k: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    v: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    out: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float32))
    lse: np.ndarray = field(default_factory=lambda: np.zeros(0, np.float64))

    @staticmethod
    def zeros(num_heads, seq_len, head_dim) -> "AttentionTensors":
        n = num_heads * seq_len * head_dim
        return AttentionTensors(num_heads, seq_len, head_dim, 1.0 / math.sqrt(head_dim),
                                np.zeros(n, np.float32), np.zeros(n, np.float32),
                                np.zeros(n, np.float32))

    @staticmethod
    def random(num_heads, seq_len, head_dim, seed) -> "AttentionTensors":
        """The reference's inputs for `seed` (attention.cpp:135-144): mt19937_64,
        U[-1,1] floats, q then k then v (s2_random_tensors: the same stream)."""
        t = AttentionTensors.zeros(num_heads, seq_len, head_dim)
        fp = ctypes.POINTER(ctypes.c_float)
        check(lib().s2_random_tensors(num_heads, seq_len, head_dim, int(seed) & (2**64 - 1),
                                      t.q.ctypes.data_as(fp), t.k.ctypes.data_as(fp), t.v.ctypes.data_as(fp)))
        return t

    def idx(self, head, token, component) -> int:
        return (head * self.seq_len + token) * self.head_dim + component

    def row_index(self, head, token) -> int:
        return head * self.seq_len + token

    def copy(self) -> "AttentionTensors":
        return AttentionTensors(self.num_heads, self.seq_len, self.head_dim, self.scale,
                                self.q.copy(), self.k.copy(), self.v.copy(), self.out.copy(),
                                self.lse.copy())


def _check_shapes(t: AttentionTensors, num_masks: int, mask_blocks: int, block_size: int):
    """kernel_common.hpp:20-32, same messages."""
    if t.num_heads < 1 or t.seq_len < 1 or t.head_dim < 1:
        raise _abi.S2InvalidArgument(1, "tensor dimensions must be positive")
    n = t.num_heads * t.seq_len * t.head_dim
    if t.q.size != n or t.k.size != n or t.v.size != n:
        raise _abi.S2InvalidArgument(1, "q/k/v sizes do not match [heads, seq, dim]")
    if num_masks != t.num_heads:
        raise _abi.S2InvalidArgument(1, "one mask per head required")
    if block_size < 1:
        raise _abi.S2InvalidArgument(1, "block_size must be positive")
    if mask_blocks != -(-t.seq_len // block_size):
        raise _abi.S2InvalidArgument(1, "mask block count does not match ceil(seq_len/block_size)")


def dsplit_attention(t: AttentionTensors, csr: List[CsrMask], block_size: int,
                     num_splits: int) -> None:
    """attention.cpp:100-118,195-198 on the GPU (fp32 kernel).  Writes t.out / t.lse."""
    import torch

    if not csr:
        raise _abi.S2InvalidArgument(1, "csr list is empty")
    _check_shapes(t, len(csr), csr[0].num_blocks, block_size)
    for c in csr:
        c.validate()
        if c.num_blocks != csr[0].num_blocks:
            raise _abi.S2InvalidArgument(1, "csr masks differ in block count")
    if num_splits < 1 or t.head_dim % num_splits != 0:
        raise _abi.S2InvalidArgument(1, "num_splits must divide head_dim")
    if not torch.cuda.is_available():
        raise _abi.S2Error(_abi.S2_ERR_NO_DEVICE, "no CUDA device: the S2 kernels need a B200")
    plan = Plan.from_csr(csr, t.seq_len, block_size)
    shape = (1, t.num_heads, t.seq_len, t.head_dim)
    dev = torch.device("cuda")
    q = torch.from_numpy(np.ascontiguousarray(t.q, np.float32)).reshape(shape).to(dev)
    k = torch.from_numpy(np.ascontiguousarray(t.k, np.float32)).reshape(shape).to(dev)
    v = torch.from_numpy(np.ascontiguousarray(t.v, np.float32)).reshape(shape).to(dev)
    out, lse = s2_attn_fwd(plan, q, k, v, scale=t.scale if t.scale else None,
                           num_splits=num_splits)
    torch.cuda.synchronize()
    t.out = out.reshape(-1).cpu().numpy().astype(np.float32)
    t.lse = lse.reshape(-1).cpu().numpy().astype(np.float64)


def streaming_sharded_attention(t: AttentionTensors, csr: List[CsrMask], block_size: int) -> None:
    """attention.cpp:190-193 on the GPU; bit-identical to dsplit_attention(..., 1)."""
    dsplit_attention(t, csr, block_size, 1)
