"""torch.library registration of the S2 path (torch_ops.py).
CPU: the fake (meta) kernels, the registered autograd formula driven on meta
tensors, the plan registry and the no-CPU-path rule.  GPU: opcheck, equality
with the direct C-ABI calls, and torch.compile(fullgraph) over the opaque op."""
import gc

import pytest
import torch

import paper_2407_17678_b200 as s2
from paper_2407_17678_b200 import torch_ops


def _plan(n=512, h=4):
    return s2.Plan.from_config(s2.make_s2_config(n, h, block_size=64, local_blocks=2, vert_stride=3))


def test_ops_are_registered():
    assert hasattr(torch.ops.s2attn, "fwd") and hasattr(torch.ops.s2attn, "bwd")
    sch = str(torch.ops.s2attn.fwd.default._schema)
    assert "SymInt plan_id" in sch or "int plan_id" in sch


def test_fake_kernels_give_shapes_and_autograd_is_registered():
    plan = _plan()
    q = torch.empty(2, 4, 512, 128, dtype=torch.bfloat16, device="meta", requires_grad=True)
    k = torch.empty(2, 2, 512, 128, dtype=torch.bfloat16, device="meta", requires_grad=True)
    v = torch.empty(2, 2, 512, 128, dtype=torch.bfloat16, device="meta", requires_grad=True)
    out, lse = torch.ops.s2attn.fwd(q, k, v, torch_ops.plan_id(plan), 0.0)
    assert out.shape == q.shape and out.dtype == torch.bfloat16
    assert lse.shape == (2, 4, 512) and lse.dtype == torch.float32
    out.sum().backward()  # runs the registered formula -> s2attn::bwd's fake kernel
    assert q.grad.shape == q.shape and k.grad.shape == k.shape and v.grad.shape == v.shape


def test_plan_ids_are_stable_and_weak():
    plan = _plan()
    pid = torch_ops.plan_id(plan)
    assert torch_ops.plan_id(plan) == pid
    assert torch_ops._plan(pid) is plan
    del plan
    gc.collect()
    with pytest.raises(s2.S2InvalidArgument, match="no live plan"):
        torch_ops._plan(pid)


def test_cpu_tensors_are_rejected():
    plan = _plan()
    x = torch.zeros(1, 4, 512, 128, dtype=torch.bfloat16)
    with pytest.raises(s2.S2InvalidArgument, match="CUDA"):
        torch.ops.s2attn.fwd(x, x, x, torch_ops.plan_id(plan), 0.0)


@pytest.mark.gpu
def test_opcheck_and_equality_with_direct_calls():
    plan = _plan()
    g = torch.Generator(device="cuda").manual_seed(3)
    mk = lambda *s: (torch.rand(*s, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)  # noqa
    q, k, v, do = mk(1, 4, 512, 128), mk(1, 4, 512, 128), mk(1, 4, 512, 128), mk(1, 4, 512, 128)
    pid = torch_ops.plan_id(plan)
    torch.library.opcheck(torch.ops.s2attn.fwd, (q, k, v, pid, 0.0))
    o_ref, l_ref = s2.s2_attn_fwd(plan, q, k, v)
    dq_ref, dk_ref, dv_ref = s2.s2_attn_bwd(plan, q, k, v, o_ref, l_ref, do)
    qa, ka, va = (t.clone().requires_grad_() for t in (q, k, v))
    o = s2.s2_attention(qa, ka, va, plan)
    o.backward(do)
    # same kernels, same inputs: identical bits
    assert torch.equal(o, o_ref)
    assert torch.equal(qa.grad, dq_ref) and torch.equal(ka.grad, dk_ref) and torch.equal(va.grad, dv_ref)


@pytest.mark.gpu
def test_compiles_fullgraph_as_an_opaque_op():
    plan = _plan()
    q = (torch.rand(1, 4, 512, 128, device="cuda") * 2 - 1).to(torch.bfloat16)

    def f(x):
        return s2.s2_attention(x * 0.5, x, x, plan).float().sum()

    want = f(q)
    got = torch.compile(f, fullgraph=True)(q)
    torch.testing.assert_close(got, want, rtol=1e-3, atol=1e-3)
