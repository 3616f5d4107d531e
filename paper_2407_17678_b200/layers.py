"""Hybrid dense / S2 layer stacks over the C ABI (s2_layers_*): the
reference's LayerSchedule / build_layer_masks (pattern.hpp:98-118,
pattern.cpp:168-181) made executable.  Dense layer ids run with the
dense-causal layout (make_dense_config of the same shape), every other layer
with the sparse pattern; both through the same tcgen05 kernels."""
import ctypes
from typing import Optional

from . import _abi
from ._abi import check, lib
from .attention import Plan, s2_attention, s2_attn_bwd, s2_attn_fwd
from .pattern import LayerSchedule


class _Borrowed(Plan):
    """A plan owned by its LayerStack (never destroyed on its own)."""

    def __del__(self):
        pass


class LayerStack:
    """One plan per distinct layer type of `schedule`."""

    def __init__(self, schedule: LayerSchedule):
        from .serialize import _schedule_to_c

        c, self._keep = _schedule_to_c(schedule)
        self._h = ctypes.c_void_p()
        check(lib().s2_layers_create(ctypes.byref(c), ctypes.byref(self._h)))
        self.schedule = schedule
        p = schedule.sparse_pattern
        self._plans = {}
        for layer in range(schedule.num_layers):
            h, d = ctypes.c_void_p(), ctypes.c_int()
            check(lib().s2_layers_plan(self._h, layer, ctypes.byref(h), ctypes.byref(d)))
            key = bool(d.value)
            if key not in self._plans:
                self._plans[key] = _Borrowed(h, p.num_heads, p.kv_heads(), p.seq_len, p.block_size)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                lib().s2_layers_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def num_layers(self) -> int:
        return self.schedule.num_layers

    def is_dense(self, layer: int) -> bool:
        if not 0 <= layer < self.schedule.num_layers:
            raise _abi.S2InvalidArgument(1, "layer outside [0, num_layers)")
        return layer in self.schedule.dense_layer_ids

    def plan(self, layer: int) -> Plan:
        return self._plans[self.is_dense(layer)]

    def forward(self, layer: int, q, k, v, **kw):
        """(out, lse) of `layer` (s2_attn_fwd with the layer's plan)."""
        return s2_attn_fwd(self.plan(layer), q, k, v, **kw)

    def backward(self, layer: int, q, k, v, out, lse, dout, **kw):
        return s2_attn_bwd(self.plan(layer), q, k, v, out, lse, dout, **kw)

    def attention(self, layer: int, q, k, v, scale: Optional[float] = None):
        """Differentiable attention of `layer` (torch autograd)."""
        return s2_attention(q, k, v, self.plan(layer), scale)
