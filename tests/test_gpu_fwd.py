"""Forward parity on the B200: CUDA path (via the C ABI) vs the oracle.

bf16 (tcgen05) path: inputs rounded to bf16, oracle run on the same values,
out/lse within rtol=atol=1e-2 (north_star tolerance).  fp32 path: within
1e-4 of the reference's own fp32 outputs (golden fixtures) — north_star's
fp32 tolerance.  Plus the reference's exactness properties
(test_attention.cpp:124-132,196-257).
"""
import numpy as np
import pytest

import paper_2407_17678_b200 as s2
from helpers import bf16_round, cfg_from_dict, load_json, load_npz, single
import oracle

pytestmark = pytest.mark.gpu
FWD = load_json("fwd_cases.json")
FWD_ARR = load_npz("fwd_outputs.npz")

BF16_TOL = dict(rtol=1e-2, atol=1e-2)
F32_TOL = dict(rtol=1e-4, atol=1e-4)


def _torch():
    import torch

    return torch


def run_bf16(cfg, batch, D, seed=0, scale=None, dist="uniform"):
    torch = _torch()
    H, Hkv, N, S = cfg.num_heads, cfg.kv_heads(), cfg.seq_len, cfg.block_size
    rng = np.random.default_rng(seed)
    if dist == "uniform":
        gen = lambda n: rng.uniform(-1, 1, n)  # noqa: E731
    else:
        gen = lambda n: rng.standard_normal(n) * 3.0  # noqa: E731
    q = bf16_round(gen(batch * H * N * D).astype(np.float32))
    k = bf16_round(gen(batch * Hkv * N * D).astype(np.float32))
    v = bf16_round(gen(batch * Hkv * N * D).astype(np.float32))
    plan = s2.Plan.from_config(cfg)
    dev = torch.device("cuda")
    tq = torch.from_numpy(q).reshape(batch, H, N, D).to(dev, torch.bfloat16)
    tk = torch.from_numpy(k).reshape(batch, Hkv, N, D).to(dev, torch.bfloat16)
    tv = torch.from_numpy(v).reshape(batch, Hkv, N, D).to(dev, torch.bfloat16)
    out, lse = s2.s2_attn_fwd(plan, tq, tk, tv, scale=scale)
    torch.cuda.synchronize()
    rp, ci = oracle.csr_all(cfg)
    ro, rl = oracle.attn_fwd(q, k, v, rp, ci, batch, H, Hkv, N, D, S, scale)
    return (out.float().cpu().numpy().ravel(), lse.cpu().numpy().ravel(), ro, rl,
            (plan, tq, tk, tv))


BF16_CASES = {
    # name: (cfg, batch, D)
    "cfg1_shape_bf16": (single(2048, 64, 8, 4, 8), 1, 64),
    "h4_n1000_ragged_d128": (single(1000, 64, 4, 2, 4), 1, 128),
    "cfg2_like_batch2_n2048": (single(2048, 64, 32, 4, 16), 2, 128),
    "gqa_32q8kv": (single(2048, 64, 32, 4, 8, kv=8), 1, 128),
    "gqa_8q2kv_d64_batch2": (single(1536, 64, 8, 3, 4, kv=2), 2, 64),
    "block128": (single(2048, 128, 4, 2, 3), 1, 128),
    "block32": (single(1536, 32, 4, 3, 5), 1, 64),
    "block16_local_stride2": (single(700, 16, 2, 5, 4, local_stride=2), 1, 128),
    "single_qtile_n100": (single(100, 64, 2, 1, 2), 1, 128),
    "dense_causal": (s2.make_dense_config(1024, 64, 2), 1, 128),
    "homo_head": (single(2048, 64, 4, 2, 8, offsets=[0] * 4), 1, 128),
}


@pytest.mark.parametrize("name", list(BF16_CASES))
def test_bf16_forward_matches_oracle(name):
    cfg, batch, D = BF16_CASES[name]
    out, lse, ro, rl, _ = run_bf16(cfg, batch, D)
    err = oracle.max_rel(out, ro)
    print(f"{name}: max|d out|={np.abs(out - ro).max():.3e} max_rel={err:.3e} "
          f"max|d lse|={np.abs(lse - rl).max():.3e}")
    np.testing.assert_allclose(out, ro, **BF16_TOL)
    np.testing.assert_allclose(lse, rl, **BF16_TOL)


def test_bf16_forward_stress_distribution():
    """N(0,1)*3 inputs exercise the online-softmax rescale path."""
    cfg = single(2048, 64, 4, 4, 8)
    out, lse, ro, rl, _ = run_bf16(cfg, 1, 128, seed=3, dist="normal")
    np.testing.assert_allclose(out, ro, rtol=2e-2, atol=2e-2)
    np.testing.assert_allclose(lse, rl, rtol=1e-2, atol=1e-2)


def test_bf16_deterministic_and_head_permutation_exact():
    torch = _torch()
    cfg = single(1024, 64, 4, 2, 4)
    out, lse, ro, rl, (plan, q, k, v) = run_bf16(cfg, 1, 128)
    o2, l2 = s2.s2_attn_fwd(plan, q, k, v)
    torch.cuda.synchronize()
    assert np.array_equal(o2.float().cpu().numpy().ravel(), out)
    assert np.array_equal(l2.cpu().numpy().ravel(), lse)
    # permuting heads (and their masks) permutes outputs exactly (test_attention.cpp:217-240)
    perm = [2, 0, 3, 1]
    csr = [s2.build_csr(cfg, h) for h in range(4)]
    pplan = s2.Plan.from_csr([csr[p] for p in perm], cfg.seq_len, cfg.block_size)
    po, pl = s2.s2_attn_fwd(pplan, q[:, perm].contiguous(), k[:, perm].contiguous(),
                            v[:, perm].contiguous())
    torch.cuda.synchronize()
    o = torch.from_numpy(out).reshape(1, 4, 1024, 128)
    assert torch.equal(po.float().cpu(), o[:, perm])


def test_bf16_unattended_value_rows_change_nothing():
    """test_attention.cpp:196-215 at the kernel's 64-key chunk granularity."""
    torch = _torch()
    cfg = single(1024, 64, 2, 2, 5)
    out, lse, ro, rl, (plan, q, k, v) = run_bf16(cfg, 1, 128)
    mask = s2.build_head_mask(cfg, 0).bits
    i_block = 13
    unattended = [j for j in range(cfg.num_blocks()) if not mask[i_block, j]]
    v2 = v.clone()
    for j in unattended:
        v2[0, 0, j * 64:(j + 1) * 64] += 1000.0
    o2, _ = s2.s2_attn_fwd(plan, q, k, v2)
    torch.cuda.synchronize()
    rows = slice(i_block * 64, (i_block + 1) * 64)
    a = out.reshape(1, 2, 1024, 128)[0, 0, rows]
    b = o2.float().cpu().numpy()[0, 0, rows]
    assert np.array_equal(a, b)


def test_bf16_unit_subset_matches_full():
    torch = _torch()
    cfg = single(2048, 64, 8, 4, 8, kv=4)
    out, lse, ro, rl, (plan, q, k, v) = run_bf16(cfg, 2, 128)
    units = np.array([5, 0, 3], np.int32)  # (b, g) = (1,1), (0,0), (0,3)
    hpg = 2
    qu = q.reshape(8, hpg, 2048, 128)[torch.as_tensor(units, dtype=torch.long)].contiguous()
    ku = k.reshape(8, 2048, 128)[torch.as_tensor(units, dtype=torch.long)].contiguous()
    vu = v.reshape(8, 2048, 128)[torch.as_tensor(units, dtype=torch.long)].contiguous()
    ou, lu = s2.s2_attn_fwd(plan, qu, ku, vu, unit_ids=units)
    torch.cuda.synchronize()
    full = torch.from_numpy(out).reshape(8, hpg, 2048, 128)
    assert torch.equal(ou.float().cpu(), full[torch.as_tensor(units, dtype=torch.long)])


# ------------------------------------------------------------------- fp32 path
@pytest.mark.parametrize("name", list(FWD["cases"]))
def test_f32_forward_matches_reference_fixture(name):
    """fp32 kernel vs the reference's own fp32 streaming outputs at 1e-4."""
    p = FWD["cases"][name]
    cfg = cfg_from_dict(p["config"])
    q, k, v = oracle.random_tensors(p["H"], p["N"], p["d"], p["seed"])
    t = s2.AttentionTensors.zeros(p["H"], p["N"], p["d"])
    t.q, t.k, t.v = q, k, v
    s2.streaming_sharded_attention(t, s2.build_all_csr(cfg), p["S"])
    out, lse = t.out, t.lse
    if name + "__out_idx" in FWD_ARR:
        out = out[FWD_ARR[name + "__out_idx"]]
        lse = lse[FWD_ARR[name + "__lse_idx"]]
    ref_out, ref_lse = FWD_ARR[name + "__out"], FWD_ARR[name + "__lse"]
    print(f"{name}: max_rel out={oracle.max_rel(out, ref_out):.3e} "
          f"max|d|={np.abs(out - ref_out).max():.3e}")
    np.testing.assert_allclose(out, ref_out, **F32_TOL)
    np.testing.assert_allclose(lse, ref_lse, **F32_TOL)


def test_f32_reference_test_cases():
    """Restated test_attention.cpp:72-96,124-132,149-194,284-294 on the GPU path."""
    # N=1 -> out = v exactly
    cfg = s2.make_single_stride_config(1, 4, 2, 1, 1)
    t = s2.AttentionTensors.random(2, 1, 8, 3)
    s2.streaming_sharded_attention(t, s2.build_all_csr(cfg), 4)
    np.testing.assert_array_equal(t.out, t.v)
    # zero values -> zero output, finite lse
    cfg = s2.make_single_stride_config(32, 8, 2, 1, 2)
    t = s2.AttentionTensors.random(2, 32, 8, 5)
    t.v[:] = 0
    s2.streaming_sharded_attention(t, s2.build_all_csr(cfg), 8)
    assert np.all(t.out == 0) and np.all(np.isfinite(t.lse))
    # dsplit(1) == streaming bit for bit
    cfg = s2.make_single_stride_config(96, 16, 3, 1, 3)
    t = s2.AttentionTensors.random(3, 96, 16, 17)
    a = t.copy()
    b = t.copy()
    s2.streaming_sharded_attention(a, s2.build_all_csr(cfg), 16)
    s2.dsplit_attention(b, s2.build_all_csr(cfg), 16, 1)
    assert np.array_equal(a.out, b.out) and np.array_equal(a.lse, b.lse)
    # softmax weights recomputed from lse sum to one (1e-6)
    cfg = s2.make_single_stride_config(64, 8, 2, 1, 3)
    t = s2.AttentionTensors.random(2, 64, 16, 37)
    s2.streaming_sharded_attention(t, s2.build_all_csr(cfg), 8)
    masks = s2.build_all_masks(cfg)
    Q = t.q.reshape(2, 64, 16).astype(np.float64)
    K = t.k.reshape(2, 64, 16).astype(np.float64)
    for h in range(2):
        for i in range(64):
            js = [j for j in range(i + 1) if masks[h].at(i // 8, j // 8)]
            s = (K[h, js] @ Q[h, i]) * t.scale
            assert abs(np.exp(s - t.lse[h * 64 + i]).sum() - 1.0) < 1e-6


def test_f32_error_contract():
    """test_attention.cpp:143-147,259-282."""
    cfg = s2.make_single_stride_config(16, 8, 2, 1, 1)
    t = s2.AttentionTensors.random(2, 16, 6, 23)
    csr = s2.build_all_csr(cfg)
    with pytest.raises(s2.S2InvalidArgument):
        s2.dsplit_attention(t, csr, 8, 4)
    with pytest.raises(s2.S2InvalidArgument):
        s2.dsplit_attention(t, csr, 8, 0)
    with pytest.raises(s2.S2InvalidArgument):
        s2.streaming_sharded_attention(t, csr[:1], 8)
    with pytest.raises(s2.S2InvalidArgument):
        s2.streaming_sharded_attention(t, csr, 4)
    t.q = t.q[:-1]
    with pytest.raises(s2.S2InvalidArgument):
        s2.streaming_sharded_attention(t, csr, 8)


def test_f32_negative_control_corrupted_csr_fails_parity():
    """selftest.cpp:41-49: dropping one remote block must break parity."""
    p = FWD["cases"]["h2_n256_s64_d64"]
    cfg = cfg_from_dict(p["config"])
    q, k, v = oracle.random_tensors(p["H"], p["N"], p["d"], p["seed"])
    csr = s2.build_all_csr(cfg)
    c = csr[0]
    for i in range(c.num_blocks - 1, 0, -1):
        if c.row_ptr[i + 1] - c.row_ptr[i] >= 2:
            c.col_idx = np.delete(c.col_idx, c.row_ptr[i])
            c.row_ptr[i + 1:] -= 1
            break
    t = s2.AttentionTensors.zeros(p["H"], p["N"], p["d"])
    t.q, t.k, t.v = q, k, v
    s2.streaming_sharded_attention(t, csr, p["S"])
    name = "h2_n256_s64_d64"
    out = t.out[FWD_ARR[name + "__out_idx"]] if name + "__out_idx" in FWD_ARR else t.out
    assert not np.allclose(out, FWD_ARR[name + "__out"], **F32_TOL)
    # the uncorrupted CSR passes (so the failure is the corruption, not noise)
    t2 = s2.AttentionTensors.zeros(p["H"], p["N"], p["d"])
    t2.q, t2.k, t2.v = q, k, v
    s2.streaming_sharded_attention(t2, s2.build_all_csr(cfg), p["S"])
    out2 = t2.out[FWD_ARR[name + "__out_idx"]] if name + "__out_idx" in FWD_ARR else t2.out
    np.testing.assert_allclose(out2, FWD_ARR[name + "__out"], **F32_TOL)


@pytest.mark.parametrize("d", [3, 24, 40, 96, 200, 256, 300, 512, 1000])
def test_f32_any_head_dim_matches_oracle(d):
    """The reference takes any head dim (AttentionTensors d, attention.hpp:17-37); the
    fp32 kernel serves every d <= 2048.  Unusual sizes vs the oracle port (itself
    bit-identical to the reference's streaming forward), at the fp32 tolerance."""
    cfg = s2.make_single_stride_config(300, 16, 3, 2, 3)
    H, N = 3, 300
    q, k, v = oracle.random_tensors(H, N, d, 40 + d)
    t = s2.AttentionTensors.zeros(H, N, d)
    t.q, t.k, t.v = q, k, v
    s2.streaming_sharded_attention(t, s2.build_all_csr(cfg), 16)
    rp, ci = oracle.csr_all(cfg)
    ro, rl = oracle.attn_fwd(q, k, v, rp, ci, 1, H, H, N, d, 16)
    np.testing.assert_allclose(t.out, ro, **F32_TOL)
    np.testing.assert_allclose(t.lse, rl, **F32_TOL)


@pytest.mark.parametrize("N,S,d,rowwise", [(1000, 128, 64, False), (333, 8, 40, False), (777, 96, 128, False),
                                           (1000, 128, 64, True), (520, 64, 256, False), (65, 200, 17, False)])
def test_f32_tiled_kernel_blocks_and_tails(N, S, d, rowwise, monkeypatch):
    """The tiled fp32 kernel's 64-row sub-tiles of large blocks (S=128, 200), small
    blocks (S=8), ragged N and head dims that are not multiples of 4 -- and the same
    case on the row-wise kernel (S2_SIMT_ROWWISE=1) -- vs the oracle at 1e-4."""
    if rowwise:
        monkeypatch.setenv("S2_SIMT_ROWWISE", "1")
    cfg = s2.make_single_stride_config(N, S, 2, 2, 3)
    H = 2
    q, k, v = oracle.random_tensors(H, N, d, 7 + d + S)
    t = s2.AttentionTensors.zeros(H, N, d)
    t.q, t.k, t.v = q, k, v
    s2.streaming_sharded_attention(t, s2.build_all_csr(cfg), S)
    rp, ci = oracle.csr_all(cfg)
    ro, rl = oracle.attn_fwd(q, k, v, rp, ci, 1, H, H, N, d, S)
    np.testing.assert_allclose(t.out, ro, **F32_TOL)
    np.testing.assert_allclose(t.lse, rl, **F32_TOL)


@pytest.mark.parametrize("D,S,kv", [(64, 64, 2), (40, 32, 1), (128, 128, 4)])
def test_f32_tiled_kernel_gqa_batch_units(D, S, kv):
    """fp32 forward with GQA (query heads per kv head 2 / 4), batch 2 and a unit
    subset: every (batch, kv group) of the tiled kernel against the oracle at 1e-4,
    and the unit-subset call bit-identical to the full call."""
    torch = _torch()
    H, N, B = 4, 777, 2
    cfg = single(N, S, H, 2, 3, kv=kv)
    rng = np.random.default_rng(D + S)
    q = rng.uniform(-1, 1, B * H * N * D).astype(np.float32)
    k, v = (rng.uniform(-1, 1, B * kv * N * D).astype(np.float32) for _ in range(2))
    T = lambda x, h: torch.from_numpy(x).reshape(B, h, N, D).cuda()  # noqa: E731
    plan = s2.Plan.from_config(cfg)
    out, lse = s2.s2_attn_fwd(plan, T(q, H), T(k, kv), T(v, kv))
    torch.cuda.synchronize()
    rp, ci = oracle.csr_all(cfg)
    ro, rl = oracle.attn_fwd(q, k, v, rp, ci, B, H, kv, N, D, S)
    np.testing.assert_allclose(out.cpu().numpy().ravel(), ro, **F32_TOL)
    np.testing.assert_allclose(lse.cpu().numpy().ravel(), rl, **F32_TOL)
    hpg = H // kv
    units = np.array([2 * kv - 1, 0], np.int32)  # (b=1, g=kv-1), (b=0, g=0)
    idx = torch.as_tensor(units, dtype=torch.long)
    qu = T(q, H).reshape(B * kv, hpg, N, D)[idx].contiguous()
    ku = T(k, kv).reshape(B * kv, N, D)[idx].contiguous()
    vu = T(v, kv).reshape(B * kv, N, D)[idx].contiguous()
    ou, _ = s2.s2_attn_fwd(plan, qu, ku, vu, unit_ids=units)
    torch.cuda.synchronize()
    assert torch.equal(ou.cpu(), out.reshape(B * kv, hpg, N, D).cpu()[idx])


@pytest.mark.parametrize("d", [32, 96, 256])
def test_bf16_other_head_dims_take_the_simt_kernel_and_match_oracle(d):
    """bf16 with a head dim the tensor-core kernel does not take (not 64 / 128) runs
    the SIMT kernel on bf16 data: parity with the oracle at the bf16 tolerance."""
    import torch

    cfg = single(700, 64, 4, 2, 3, kv=2)
    H, Hkv, N, S = 4, 2, 700, 64
    rng = np.random.default_rng(d)
    q = bf16_round(rng.uniform(-1, 1, H * N * d).astype(np.float32))
    k, v = (bf16_round(rng.uniform(-1, 1, Hkv * N * d).astype(np.float32)) for _ in range(2))
    T = lambda x, h: torch.from_numpy(x).reshape(1, h, N, d).to("cuda", torch.bfloat16)  # noqa: E731
    out, lse = s2.s2_attn_fwd(s2.Plan.from_config(cfg), T(q, H), T(k, Hkv), T(v, Hkv))
    torch.cuda.synchronize()
    rp, ci = oracle.csr_all(cfg)
    ro, rl = oracle.attn_fwd(q, k, v, rp, ci, 1, H, Hkv, N, d, S)
    np.testing.assert_allclose(out.float().cpu().numpy().ravel(), ro, rtol=1e-2, atol=1e-2)
    np.testing.assert_allclose(lse.cpu().numpy().ravel(), rl, rtol=1e-2, atol=1e-2)
    # head_dim > 128 has no backward: an explicit error, never a silent fallback
    # (head_dim <= 128 runs the fp32-FFMA backward: tests/test_gpu_bwd_simt.py)
    if d > 128:
        with pytest.raises(s2.S2Unsupported):
            s2.s2_attn_bwd(s2.Plan.from_config(cfg), T(q, H), T(k, Hkv), T(v, Hkv), out, lse, out)
