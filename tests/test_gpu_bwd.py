"""Backward parity on the B200 vs the oracle's fp64 gradient restatement.

The oracle backward (oracle/s2_oracle.c:s2o_attn_bwd) is itself pinned to
fp64 torch autograd and to central differences through the reference's own
forward (tests/test_oracle.py).  bf16 inputs, rtol=atol=1e-2 (north_star).
"""
import numpy as np
import pytest

import paper_2407_17678_b200 as s2
from helpers import bf16_round, single
import oracle

pytestmark = pytest.mark.gpu
TOL = dict(rtol=1e-2, atol=1e-2)


def run(cfg, batch, D, seed=0, unit_ids=None):
    import torch

    H, Hkv, N, S = cfg.num_heads, cfg.kv_heads(), cfg.seq_len, cfg.block_size
    rng = np.random.default_rng(seed)
    q = bf16_round(rng.uniform(-1, 1, batch * H * N * D).astype(np.float32))
    k = bf16_round(rng.uniform(-1, 1, batch * Hkv * N * D).astype(np.float32))
    v = bf16_round(rng.uniform(-1, 1, batch * Hkv * N * D).astype(np.float32))
    do = bf16_round(rng.uniform(-1, 1, batch * H * N * D).astype(np.float32))
    plan = s2.Plan.from_config(cfg)
    dev = torch.device("cuda")
    T = lambda x, h: torch.from_numpy(x).reshape(batch, h, N, D).to(dev, torch.bfloat16)  # noqa
    tq, tk, tv, tdo = T(q, H), T(k, Hkv), T(v, Hkv), T(do, H)
    out, lse = s2.s2_attn_fwd(plan, tq, tk, tv)
    dq, dk, dv = s2.s2_attn_bwd(plan, tq, tk, tv, out, lse, tdo)
    torch.cuda.synchronize()
    rp, ci = oracle.csr_all(cfg)
    rq, rk, rv = oracle.attn_bwd(q, k, v, do, rp, ci, batch, H, Hkv, N, D, S)
    f = lambda t: t.float().cpu().numpy().ravel()  # noqa
    return (f(dq), f(dk), f(dv)), (rq, rk, rv), (plan, tq, tk, tv, tdo, out, lse)


CASES = {
    "h4_n1000_ragged_d128": (single(1000, 64, 4, 2, 4), 1, 128),
    "cfg1_shape_d64": (single(2048, 64, 8, 4, 8), 1, 64),
    "batch2_h8_n2048": (single(2048, 64, 8, 4, 16), 2, 128),
    "gqa_16q4kv": (single(2048, 64, 16, 4, 4, kv=4), 1, 128),
    "gqa_8q2kv_d64_batch2": (single(1536, 64, 8, 3, 4, kv=2), 2, 64),
    "block128": (single(1024, 128, 2, 2, 3), 1, 128),
    "block32_ragged": (single(900, 32, 2, 3, 5), 1, 128),
    "single_tile": (single(100, 64, 2, 1, 2), 1, 128),
    "dense_causal": (s2.make_dense_config(768, 64, 2), 1, 128),
}


@pytest.mark.parametrize("name", list(CASES))
def test_bwd_matches_oracle(name):
    cfg, batch, D = CASES[name]
    got, ref, _ = run(cfg, batch, D)
    for nm, g, r in zip(("dq", "dk", "dv"), got, ref):
        print(f"{name} {nm}: max|d|={np.abs(g - r).max():.3e} max|ref|={np.abs(r).max():.3e}")
        np.testing.assert_allclose(g, r, **TOL, err_msg=nm)


def test_bwd_deterministic():
    import torch

    cfg = single(1024, 64, 4, 2, 4)
    got, ref, (plan, q, k, v, do, out, lse) = run(cfg, 1, 128)
    g2 = s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
    torch.cuda.synchronize()
    for a, b in zip(got, g2):
        assert np.array_equal(a, b.float().cpu().numpy().ravel())


def test_autograd_op():
    import torch

    cfg = single(512, 64, 2, 2, 3)
    plan = s2.Plan.from_config(cfg)
    torch.manual_seed(0)
    q = torch.randn(1, 2, 512, 128, device="cuda", dtype=torch.bfloat16, requires_grad=True)
    k = torch.randn(1, 2, 512, 128, device="cuda", dtype=torch.bfloat16, requires_grad=True)
    v = torch.randn(1, 2, 512, 128, device="cuda", dtype=torch.bfloat16, requires_grad=True)
    o = s2.s2_attention(q, k, v, plan)
    o.float().square().sum().backward()
    # token-mask reference in fp32 torch
    m = np.zeros((2, 512, 512), bool)
    for h in range(2):
        bits = s2.build_head_mask(cfg, h).bits
        m[h] = np.kron(bits, np.ones((64, 64), np.uint8)).astype(bool) & np.tril(np.ones((512, 512), bool))
    mask = torch.from_numpy(m).cuda()
    qf, kf, vf = (t.detach().float().requires_grad_() for t in (q, k, v))
    s = (qf @ kf.transpose(-1, -2)) / np.sqrt(128)
    of = torch.softmax(s.masked_fill(~mask, float("-inf")), -1) @ vf
    of.square().sum().backward()
    torch.testing.assert_close(o.float(), of, rtol=2e-2, atol=2e-2)
    for a, b in ((q, qf), (k, kf), (v, vf)):
        torch.testing.assert_close(a.grad.float(), b.grad, rtol=5e-2, atol=5e-2)


def test_hybrid_layer_stack_fwd_bwd():
    """A 4-layer hybrid stack (dense {0, 2}): each layer's fwd+bwd through
    LayerStack equals the oracle on that layer's layout (build_layer_masks)."""
    import torch

    from paper_2407_17678_b200.pattern import LayerSchedule

    pat = single(1024, 64, 4, 2, 3)
    sched = LayerSchedule(4, {0, 2}, pat)
    stack = s2.LayerStack(sched)
    H, N, D = 4, 1024, 128
    rng = np.random.default_rng(3)
    dev = torch.device("cuda")
    for layer in range(4):
        cfg = s2.make_dense_config(N, 64, H) if layer in (0, 2) else pat
        x = [bf16_round(rng.uniform(-1, 1, H * N * D).astype(np.float32)) for _ in range(4)]
        tq, tk, tv, tdo = (torch.from_numpy(a).reshape(1, H, N, D).to(dev, torch.bfloat16) for a in x)
        out, lse = stack.forward(layer, tq, tk, tv)
        dq, dk, dv = stack.backward(layer, tq, tk, tv, out, lse, tdo)
        torch.cuda.synchronize()
        rp, ci = oracle.csr_all(cfg)
        ro, rl = oracle.attn_fwd(*x[:3], rp, ci, 1, H, H, N, D, 64)
        rq, rk, rv = oracle.attn_bwd(*x, rp, ci, 1, H, H, N, D, 64)
        f = lambda t: t.float().cpu().numpy().ravel()  # noqa: E731
        np.testing.assert_allclose(f(out), ro, **TOL)
        for g, r in ((dq, rq), (dk, rk), (dv, rv)):
            np.testing.assert_allclose(f(g), r, **TOL)


@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_host_buffer_pipeline_matches_device_path(dt):
    """s2_attn_fwd_bwd_host (host tensors, chunked H2D / kernels / D2H on three
    streams) returns exactly what the device path returns -- on the tcgen05 kernels
    (bf16) and on the FFMA kernels (fp32, the reference API's precision)."""
    import torch

    if dt == "bf16":
        cfg, B, H, Hkv, N, D, tdt = single(2048, 64, 8, 4, 8, kv=4), 2, 8, 4, 2048, 128, torch.bfloat16
    else:
        cfg, B, H, Hkv, N, D, tdt = single(640, 32, 4, 3, 4, kv=2), 2, 4, 2, 640, 64, torch.float32
    plan = s2.Plan.from_config(cfg)
    g = torch.Generator().manual_seed(9)
    mk = lambda h: (torch.rand((B, h, N, D), generator=g) * 2 - 1).to(tdt).pin_memory()  # noqa
    q, k, v, do = mk(H), mk(Hkv), mk(Hkv), mk(H)
    outs = [torch.empty_like(q).pin_memory(), torch.empty((B, H, N), dtype=torch.float32).pin_memory(),
            torch.empty_like(q).pin_memory(), torch.empty_like(k).pin_memory(), torch.empty_like(v).pin_memory()]
    for chunks in (1, 3, 8):
        s2.s2_attn_fwd_bwd_host(plan, q, k, v, do, *outs, num_chunks=chunks)
        torch.cuda.synchronize()
        dev = [t.cuda() for t in (q, k, v, do)]
        o, l = s2.s2_attn_fwd(plan, *dev[:3])
        gq, gk, gv = s2.s2_attn_bwd(plan, *dev[:3], o, l, dev[3])
        for a, b in zip(outs, (o, l, gq, gk, gv)):
            assert torch.equal(a, b.cpu()), chunks
