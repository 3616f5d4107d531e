"""PyTorch operator registration of the S2 attention path (SURVEY §8(f) row 4:
DKernel's "plug-in replacement" role, PAPER.md:86,492 -- not in the C++ reference).

Two `torch.library` custom ops wrap the C ABI (include/s2attn.h):

    s2attn::fwd(q, k, v, plan_id, scale) -> (out, lse)
    s2attn::bwd(q, k, v, out, lse, dout, plan_id, scale) -> (dq, dk, dv)

* They are opaque to torch.compile / FX tracing: each has a fake (meta)
  implementation that gives output shapes without touching a device.
* `fwd` has an autograd formula registered (`register_autograd`) that calls
  `bwd`: `s2_attention` is differentiable through the dispatcher. No
  Python-level autograd.Function is involved.
* A plan (per-head CSR + work lists, a C handle) is not a tensor, so the ops
  take its registry id (`Plan.op_id`). The registry holds weak references, and
  an id whose plan was freed is an error.
* `scale` = 0.0 selects 1/sqrt(head_dim), as in the C ABI.

There is no CPU implementation: on a CPU tensor the op raises (the product
path has no CPU fallback)."""
import itertools
import math
import weakref
from typing import Tuple

import torch

from . import _abi

_PLANS: "weakref.WeakValueDictionary[int, object]" = weakref.WeakValueDictionary()
_NEXT = itertools.count(1)


def plan_id(plan) -> int:
    """Registry id of `plan` (assigned on first use, stable for the plan's life)."""
    pid = getattr(plan, "_op_id", None)
    if pid is None:
        pid = next(_NEXT)
        plan._op_id = pid
        _PLANS[pid] = plan
    return pid


def _plan(pid: int):
    p = _PLANS.get(pid)
    if p is None:
        raise _abi.S2InvalidArgument(1, f"s2attn op: no live plan with id {pid}")
    return p


def _opt_scale(scale: float):
    # +0.0 encodes "default 1/sqrt(D)"; -0.0 an explicit zero (S2_SCALE_ZERO)
    return None if (scale == 0.0 and math.copysign(1.0, scale) > 0) else scale


@torch.library.custom_op("s2attn::fwd", mutates_args=())
def s2attn_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, plan_id: int,
               scale: float) -> Tuple[torch.Tensor, torch.Tensor]:
    from .attention import s2_attn_fwd

    return s2_attn_fwd(_plan(plan_id), q.contiguous(), k.contiguous(), v.contiguous(),
                       scale=_opt_scale(scale))


@s2attn_fwd.register_fake
def _(q, k, v, plan_id, scale):
    return torch.empty_like(q), q.new_empty(q.shape[:-1], dtype=torch.float32)


@torch.library.custom_op("s2attn::bwd", mutates_args=())
def s2attn_bwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: torch.Tensor,
               lse: torch.Tensor, dout: torch.Tensor, plan_id: int,
               scale: float) -> Tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    from .attention import s2_attn_bwd

    return s2_attn_bwd(_plan(plan_id), q.contiguous(), k.contiguous(), v.contiguous(),
                       out.contiguous(), lse.contiguous(), dout.contiguous(),
                       scale=_opt_scale(scale))


@s2attn_bwd.register_fake
def _(q, k, v, out, lse, dout, plan_id, scale):
    return torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)


def _setup_context(ctx, inputs, output):
    q, k, v, pid, scale = inputs
    out, lse = output
    ctx.save_for_backward(q, k, v, out, lse)
    ctx.pid, ctx.scale = pid, scale
    # the registry holds plans weakly: keep this one alive as long as the graph
    # (s2_attention(q, k, v, Plan.from_config(cfg)) passes a temporary)
    ctx.plan = _plan(pid)
    ctx.set_materialize_grads(True)


def _backward(ctx, dout, dlse):
    # lse is an auxiliary output (the backward's softmax statistics): its
    # gradient is not propagated
    q, k, v, out, lse = ctx.saved_tensors
    dq, dk, dv = torch.ops.s2attn.bwd(q, k, v, out, lse, dout, ctx.pid, ctx.scale)
    return dq, dk, dv, None, None


s2attn_fwd.register_autograd(_backward, setup_context=_setup_context)


def s2_attention(q, k, v, plan, scale=None):
    """Differentiable S2 attention through the registered ops: out [B,H,N,D]."""
    return torch.ops.s2attn.fwd(q, k, v, plan_id(plan),
                                0.0 if scale is None else (float(scale) if scale != 0 else -0.0))[0]
