"""Seeded random configurations through the bf16 tcgen05 forward AND backward vs
the oracle (rtol = atol = 1e-2).  The generator is the reference's own fuzz
(test_pattern.cpp:31-53, `random_config`: ragged N, GQA, 1-2 stride segments,
local_stride 1-3) with the block sizes the tensor-core path takes (16..128),
plus head_dim 64 / 128 and batch 1 / 2."""
import random

import numpy as np
import pytest

import paper_2407_17678_b200 as s2
import helpers  # noqa: F401  (puts oracle/ on sys.path)
from helpers import bf16_round
from paper_2407_17678_b200.pattern import PatternConfig, StrideSegment
import oracle

pytestmark = pytest.mark.gpu


def _fuzz_config(rng: random.Random) -> PatternConfig:
    blocks = rng.randint(2, 40)
    c = PatternConfig()
    c.block_size = rng.choice([16, 32, 64, 128])
    c.seq_len = blocks * c.block_size - rng.randrange(c.block_size)
    c.num_heads = 1 + rng.randrange(8)
    c.num_kv_heads = c.num_heads // 2 if (c.num_heads % 2 == 0 and rng.randrange(2)) else c.num_heads
    c.local_blocks = 1 + rng.randrange(min(4, blocks))
    c.local_stride = 1 + rng.randrange(3)
    if c.local_blocks < blocks:
        mid = c.local_blocks + rng.randrange(blocks - c.local_blocks)
        if mid > c.local_blocks and rng.randrange(2):
            c.stride_segments.append(StrideSegment(c.local_blocks, mid, rng.randint(1, 6)))
            c.stride_segments.append(StrideSegment(mid, blocks, rng.randint(1, 6)))
        else:
            c.stride_segments.append(StrideSegment(c.local_blocks, blocks, rng.randint(1, 6)))
    c.validate()
    return c


@pytest.mark.parametrize("seed", range(64))
def test_random_config_fwd_bwd_match_oracle(seed):
    import torch

    rng = random.Random(7000 + seed)
    cfg = _fuzz_config(rng)
    D = rng.choice([64, 128])
    batch = rng.choice([1, 2])
    H, Hkv, N, S = cfg.num_heads, cfg.kv_heads(), cfg.seq_len, cfg.block_size
    nrng = np.random.default_rng(seed)
    q, do = (bf16_round(nrng.uniform(-1, 1, batch * H * N * D).astype(np.float32)) for _ in range(2))
    k, v = (bf16_round(nrng.uniform(-1, 1, batch * Hkv * N * D).astype(np.float32)) for _ in range(2))
    T = lambda x, h: torch.from_numpy(x).reshape(batch, h, N, D).to("cuda", torch.bfloat16)  # noqa: E731
    tq, tk, tv, tdo = T(q, H), T(k, Hkv), T(v, Hkv), T(do, H)
    plan = s2.Plan.from_config(cfg)
    out, lse = s2.s2_attn_fwd(plan, tq, tk, tv)
    dq, dk, dv = s2.s2_attn_bwd(plan, tq, tk, tv, out, lse, tdo)
    torch.cuda.synchronize()
    rp, ci = oracle.csr_all(cfg)
    ro, rl = oracle.attn_fwd(q, k, v, rp, ci, batch, H, Hkv, N, D, S)
    rq, rk, rv = oracle.attn_bwd(q, k, v, do, rp, ci, batch, H, Hkv, N, D, S)
    f = lambda t: t.float().cpu().numpy().ravel()  # noqa: E731
    desc = f"cfg={cfg} D={D} batch={batch}"
    np.testing.assert_allclose(f(out), ro, rtol=1e-2, atol=1e-2, err_msg="out " + desc)
    np.testing.assert_allclose(lse.cpu().numpy().ravel(), rl, rtol=1e-2, atol=1e-2, err_msg="lse " + desc)
    for nm, g_, r_ in (("dq", dq, rq), ("dk", dk, rk), ("dv", dv, rv)):
        np.testing.assert_allclose(f(g_), r_, rtol=1e-2, atol=1e-2, err_msg=nm + " " + desc)


def _fuzz_config_any_block(rng: random.Random) -> PatternConfig:
    """random_config with any block size (the FFMA kernels take all of them)."""
    blocks = rng.randint(2, 30)
    c = PatternConfig()
    c.block_size = rng.choice([8, 16, 24, 40, 64, 100, 128])
    c.seq_len = blocks * c.block_size - rng.randrange(c.block_size)
    c.num_heads = 1 + rng.randrange(6)
    c.num_kv_heads = c.num_heads // 2 if (c.num_heads % 2 == 0 and rng.randrange(2)) else c.num_heads
    c.local_blocks = 1 + rng.randrange(min(4, blocks))
    c.local_stride = 1 + rng.randrange(3)
    if c.local_blocks < blocks:
        c.stride_segments.append(StrideSegment(c.local_blocks, blocks, rng.randint(1, 6)))
    c.validate()
    return c


@pytest.mark.parametrize("seed", range(24))
def test_random_config_f32_fwd_bwd_match_oracle(seed):
    """The reference-precision path: fp32 forward and backward (FFMA kernels) on
    random layouts, any block size, head_dim 16..128, at 1e-4 (north_star's fp32
    tolerance) against the oracle's fp64 forward and gradient."""
    import torch

    rng = random.Random(9100 + seed)
    cfg = _fuzz_config_any_block(rng)
    D = rng.choice([16, 32, 48, 64, 80, 96, 128])
    batch = rng.choice([1, 2])
    H, Hkv, N, S = cfg.num_heads, cfg.kv_heads(), cfg.seq_len, cfg.block_size
    nrng = np.random.default_rng(100 + seed)
    q, do = (nrng.uniform(-1, 1, batch * H * N * D).astype(np.float32) for _ in range(2))
    k, v = (nrng.uniform(-1, 1, batch * Hkv * N * D).astype(np.float32) for _ in range(2))
    T = lambda x, h: torch.from_numpy(x).reshape(batch, h, N, D).to("cuda")  # noqa: E731
    tq, tk, tv, tdo = T(q, H), T(k, Hkv), T(v, Hkv), T(do, H)
    plan = s2.Plan.from_config(cfg)
    out, lse = s2.s2_attn_fwd(plan, tq, tk, tv)
    dq, dk, dv = s2.s2_attn_bwd(plan, tq, tk, tv, out, lse, tdo)
    torch.cuda.synchronize()
    rp, ci = oracle.csr_all(cfg)
    ro, rl = oracle.attn_fwd(q, k, v, rp, ci, batch, H, Hkv, N, D, S)
    rq, rk, rv = oracle.attn_bwd(q, k, v, do, rp, ci, batch, H, Hkv, N, D, S)
    f = lambda t: t.float().cpu().numpy().ravel()  # noqa: E731
    desc = f"cfg={cfg} D={D} batch={batch}"
    tol = dict(rtol=1e-4, atol=1e-4)
    np.testing.assert_allclose(f(out), ro, **tol, err_msg="out " + desc)
    np.testing.assert_allclose(lse.cpu().numpy().ravel(), rl, **tol, err_msg="lse " + desc)
    for nm, g_, r_ in (("dq", dq, rq), ("dk", dk, rk), ("dv", dv, rv)):
        np.testing.assert_allclose(f(g_), r_, **tol, err_msg=nm + " " + desc)
