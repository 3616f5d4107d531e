"""Backward on the reference-precision path (fp32-FFMA tile kernels,
csrc/kernels/bwd_simt.cu) vs the oracle's fp64 gradient (oracle/s2_oracle.c:
s2o_attn_bwd, itself pinned to fp64 autograd and to central differences through the
reference's forward in tests/test_oracle.py).

fp32 inputs: rtol=atol=1e-4 (north_star's fp32 tolerance).  bf16 inputs with a
head_dim / block_size the tcgen05 kernels do not tile: rtol=atol=1e-2.  The forward
feeding the backward is this repo's (its out / lse), as in tests/test_gpu_bwd.py.
"""
import numpy as np
import pytest

import paper_2407_17678_b200 as s2
from helpers import bf16_round, single
import oracle

pytestmark = pytest.mark.gpu
F32_TOL = dict(rtol=1e-4, atol=1e-4)
BF16_TOL = dict(rtol=1e-2, atol=1e-2)


def _inputs(cfg, batch, D, seed, bf16):
    H, Hkv, N = cfg.num_heads, cfg.kv_heads(), cfg.seq_len
    rng = np.random.default_rng(seed)
    mk = lambda n: rng.uniform(-1, 1, n).astype(np.float32)  # noqa: E731
    q, k, v, do = mk(batch * H * N * D), mk(batch * Hkv * N * D), mk(batch * Hkv * N * D), mk(batch * H * N * D)
    if bf16:
        q, k, v, do = (bf16_round(x) for x in (q, k, v, do))
    return q, k, v, do


def run(cfg, batch, D, seed=0, bf16=False):
    import torch

    H, Hkv, N, S = cfg.num_heads, cfg.kv_heads(), cfg.seq_len, cfg.block_size
    q, k, v, do = _inputs(cfg, batch, D, seed, bf16)
    dt = torch.bfloat16 if bf16 else torch.float32
    T = lambda x, h: torch.from_numpy(x).reshape(batch, h, N, D).to("cuda", dt)  # noqa: E731
    plan = s2.Plan.from_config(cfg)
    tq, tk, tv, tdo = T(q, H), T(k, Hkv), T(v, Hkv), T(do, H)
    out, lse = s2.s2_attn_fwd(plan, tq, tk, tv)
    dq, dk, dv = s2.s2_attn_bwd(plan, tq, tk, tv, out, lse, tdo)
    torch.cuda.synchronize()
    rp, ci = oracle.csr_all(cfg)
    ref = oracle.attn_bwd(q, k, v, do, rp, ci, batch, H, Hkv, N, D, S)
    f = lambda t: t.float().cpu().numpy().ravel()  # noqa: E731
    return (f(dq), f(dk), f(dv)), ref, (plan, tq, tk, tv, tdo, out, lse)


F32_CASES = {
    # BASELINE configs[0]'s shape (fp32, H=8, S=2048, D=64, block 64, local 4, stride 8)
    "cfg1_shape": (single(2048, 64, 8, 4, 8, offsets=[0, 1, 2, 3, 4, 5, 6, 7]), 1, 64),
    "ragged_n1000_d128": (single(1000, 64, 4, 2, 4), 1, 128),
    "gqa_8q2kv_batch2": (single(1536, 64, 8, 3, 4, kv=2), 2, 64),
    "block32_d96": (single(900, 32, 2, 3, 5), 1, 96),
    "block48_not_mult16": (single(700, 24, 2, 3, 4), 1, 64),
    "block128_d80": (single(1024, 128, 2, 2, 3), 1, 80),
    "single_tile": (single(50, 64, 2, 1, 2), 1, 32),
    "dense_causal": (s2.make_dense_config(640, 64, 2), 1, 64),
}


@pytest.mark.parametrize("name", list(F32_CASES))
def test_f32_bwd_matches_oracle(name):
    cfg, batch, D = F32_CASES[name]
    got, ref, _ = run(cfg, batch, D)
    for nm, g, r in zip(("dq", "dk", "dv"), got, ref):
        print(f"{name} {nm}: max|d|={np.abs(g - r).max():.3e} max|ref|={np.abs(r).max():.3e}")
        np.testing.assert_allclose(g, r, **F32_TOL, err_msg=nm)


@pytest.mark.parametrize("D", [32, 96])
def test_bf16_untiled_head_dims_bwd(D):
    """bf16 with head_dim outside {64, 128}: the forward and the backward both take
    the FFMA kernels (bf16 loads, fp32 arithmetic)."""
    cfg = single(700, 64, 4, 2, 3, kv=2)
    got, ref, _ = run(cfg, 1, D, seed=D, bf16=True)
    for nm, g, r in zip(("dq", "dk", "dv"), got, ref):
        np.testing.assert_allclose(g, r, **BF16_TOL, err_msg=nm)


def test_bf16_block_not_multiple_of_16_bwd():
    cfg = single(600, 40, 2, 2, 3)
    got, ref, _ = run(cfg, 1, 128, seed=3, bf16=True)
    for nm, g, r in zip(("dq", "dk", "dv"), got, ref):
        np.testing.assert_allclose(g, r, **BF16_TOL, err_msg=nm)


def test_f32_bwd_deterministic_and_unit_subset():
    """Repeat calls are bit-identical, and a unit_ids subset computes exactly the
    full call's rows for those (batch, kv-group) units."""
    import torch

    cfg = single(1024, 64, 8, 2, 4, kv=2)
    batch, D = 2, 64
    got, ref, (plan, q, k, v, do, out, lse) = run(cfg, batch, D, seed=5)
    g2 = s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
    torch.cuda.synchronize()
    for a, b in zip(got, g2):
        assert np.array_equal(a, b.cpu().numpy().ravel())
    H, kv, N = 8, 2, 1024
    hpg = H // kv
    units = np.array([3, 0], np.int32)  # (b=1, g=1), (b=0, g=0)
    idx = torch.as_tensor(units, dtype=torch.long)
    sel = lambda t, h: t.reshape(batch * kv, h, N, D)[idx].contiguous()  # noqa: E731
    qu, dou, ou = sel(q, hpg), sel(do, hpg), sel(out, hpg)
    lu = lse.reshape(batch * kv, hpg, N)[idx].contiguous()
    ku, vu = (t.reshape(batch * kv, N, D)[idx].contiguous() for t in (k, v))
    dqu, dku, dvu = s2.s2_attn_bwd(plan, qu, ku, vu, ou, lu, dou, unit_ids=units)
    torch.cuda.synchronize()
    assert torch.equal(dqu, g2[0].reshape(batch * kv, hpg, N, D)[idx])
    assert torch.equal(dku, g2[1].reshape(batch * kv, N, D)[idx])
    assert torch.equal(dvu, g2[2].reshape(batch * kv, N, D)[idx])


def test_head_dim_over_128_bwd_is_unsupported():
    import torch

    cfg = single(256, 64, 2, 2, 3)
    plan = s2.Plan.from_config(cfg)
    x = torch.zeros(1, 2, 256, 160, device="cuda", dtype=torch.float32)
    out, lse = s2.s2_attn_fwd(plan, x, x, x)
    with pytest.raises(s2.S2Unsupported):
        s2.s2_attn_bwd(plan, x, x, x, out, lse, x)


def test_f32_autograd_op_matches_torch_fp64_autograd():
    """s2_attention (torch.library op) on fp32 tensors: forward and the gradients of
    a random loss against torch fp64 autograd of the dense masked softmax built from
    the same block layout (the token mask of reference.cpp:28-36), at 1e-4."""
    import torch

    from paper_2407_17678_b200.torch_ops import s2_attention

    cfg = single(320, 32, 2, 2, 3)
    H, N, D, S = 2, 320, 48, 32
    rp, ci = oracle.csr_all(cfg)
    B = (N + S - 1) // S
    mask = np.zeros((H, N, N), bool)
    off = 0
    for h in range(H):
        r = rp[h * (B + 1):(h + 1) * (B + 1)] if len(rp) == H * (B + 1) else None
        assert r is not None
        for qb in range(B):
            for e in range(r[qb], r[qb + 1]):
                kb = ci[off + e]
                mask[h, qb * S:(qb + 1) * S, kb * S:(kb + 1) * S] = True
        off += r[B]
    mask &= np.tril(np.ones((N, N), bool))[None]
    g = torch.Generator().manual_seed(11)
    q, k, v, do = (torch.rand(1, H, N, D, generator=g, dtype=torch.float64) * 2 - 1 for _ in range(4))
    qc, kc, vc = (x.float().cuda().requires_grad_() for x in (q, k, v))
    out = s2_attention(qc, kc, vc, s2.Plan.from_config(cfg))
    out.backward(do.float().cuda())
    qr, kr, vr = (x.clone().requires_grad_() for x in (q, k, v))
    sc = (qr @ kr.transpose(-1, -2)) / np.sqrt(D)
    sc = sc.masked_fill(~torch.from_numpy(mask)[None], float("-inf"))
    ref = torch.softmax(sc, -1) @ vr
    ref.backward(do)
    tol = dict(rtol=1e-4, atol=1e-4)
    torch.testing.assert_close(out.detach().cpu().double(), ref.detach(), **tol)
    for got, want in ((qc.grad, qr.grad), (kc.grad, kr.grad), (vc.grad, vr.grad)):
        torch.testing.assert_close(got.cpu().double(), want, **tol)


@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("N", [1, 2, 7, 65])
def test_tiny_sequences_fwd_bwd(dt, N):
    """N below one block (test_attention.cpp:72-79,149-156's N=1 and N<S cases) through
    the forward and backward: N=1 gives out = v exactly, dq = dk = 0 and dv = dout up
    to rounding."""
    import torch

    H, D, S = 2, 64 if dt == "f32" else 128, 64
    cfg = single(N, S, H, 1, 1) if N <= S else single(N, S, H, 1, 2)
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    tol = dict(rtol=1e-4, atol=1e-4) if dt == "f32" else dict(rtol=1e-2, atol=1e-2)
    rng = np.random.default_rng(N)
    q, k, v, do = (rng.uniform(-1, 1, H * N * D).astype(np.float32) for _ in range(4))
    if dt == "bf16":
        q, k, v, do = (bf16_round(x) for x in (q, k, v, do))
    T = lambda x: torch.from_numpy(x).reshape(1, H, N, D).to("cuda", tdt)  # noqa: E731
    plan = s2.Plan.from_config(cfg)
    tq, tk, tv, tdo = T(q), T(k), T(v), T(do)
    out, lse = s2.s2_attn_fwd(plan, tq, tk, tv)
    dq, dk, dv = s2.s2_attn_bwd(plan, tq, tk, tv, out, lse, tdo)
    torch.cuda.synchronize()
    rp, ci = oracle.csr_all(cfg)
    ro, _ = oracle.attn_fwd(q, k, v, rp, ci, 1, H, H, N, D, S)
    ref = oracle.attn_bwd(q, k, v, do, rp, ci, 1, H, H, N, D, S)
    f = lambda t: t.float().cpu().numpy().ravel()  # noqa: E731
    np.testing.assert_allclose(f(out), ro, **tol)
    for nm, g_, r_ in zip(("dq", "dk", "dv"), (dq, dk, dv), ref):
        np.testing.assert_allclose(f(g_), np.ravel(r_), **tol, err_msg=nm)
    if N == 1:  # one admitted key: P = 1, so out = v exactly (the reference's pin);
        # dS = dP - Delta vanishes up to rounding, dv = dout up to the rounding of P
        assert torch.equal(out, tv)
        small = 1e-6 if dt == "f32" else 1e-2
        assert dq.float().abs().max() <= small and dk.float().abs().max() <= small
        torch.testing.assert_close(dv.float(), tdo.float(), **tol)
