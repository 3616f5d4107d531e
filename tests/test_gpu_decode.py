"""Decode over the compacted cache vs the oracle's single-row restatement.

Pins: decode at position t == row t of the forward (the
oracle's decode is itself checked against its forward in test_oracle.py);
the cache holds exactly the retained set of simulate_decode_cache.
"""
import numpy as np
import pytest

import paper_2407_17678_b200 as s2
from paper_2407_17678_b200.decode import KVCache
from helpers import bf16_round, single
import oracle

pytestmark = pytest.mark.gpu


def _dense(batch, Hkv, T, D, seed):
    rng = np.random.default_rng(seed)
    k = bf16_round(rng.uniform(-1, 1, batch * Hkv * T * D).astype(np.float32))
    v = bf16_round(rng.uniform(-1, 1, batch * Hkv * T * D).astype(np.float32))
    return k, v


@pytest.mark.parametrize("case", [
    # (N, H, Hkv, D, local, v, batch, prefill, steps)
    (4096, 8, 2, 128, 4, 2, 2, 1000, 70),
    (2048, 32, 8, 128, 4, 8, 2, 1, 40),
    (3000, 4, 4, 64, 2, 3, 3, 700, 20),
    (8192, 8, 1, 128, 1, 8, 1, 8000, 5),
])
def test_decode_matches_oracle(case):
    import torch

    N, H, Hkv, D, local, v, batch, T0, steps = case
    cfg = single(N, 64, H, local, v, kv=Hkv)
    plan = s2.Plan.from_config(cfg)
    cache = KVCache(plan, batch, D)
    T = T0 + steps
    k, vv = _dense(batch, Hkv, T, D, 1)
    dev = torch.device("cuda")
    tk = torch.from_numpy(k).reshape(batch, Hkv, T, D).to(dev, torch.bfloat16)
    tv = torch.from_numpy(vv).reshape(batch, Hkv, T, D).to(dev, torch.bfloat16)
    cache.prefill(tk[:, :, :T0].contiguous(), tv[:, :, :T0].contiguous())
    rp, ci = oracle.csr_all(cfg)
    rng = np.random.default_rng(2)
    checked = 0
    for t in range(T0 - 1, T):
        if t >= T0:
            cache.append(tk[:, :, t].contiguous(), tv[:, :, t].contiguous())
        assert cache.length == t + 1
        if t != T - 1 and (t - T0) % 7 != 0:
            continue
        q = bf16_round(rng.uniform(-1, 1, batch * H * D).astype(np.float32))
        tq = torch.from_numpy(q).reshape(batch, H, D).to(dev, torch.bfloat16)
        out, lse = cache.decode(tq)
        torch.cuda.synchronize()
        ro, rl = oracle.decode(q, k, vv, rp, ci, batch, H, Hkv, T, D, 64, t, cfg.num_blocks())
        np.testing.assert_allclose(out.float().cpu().numpy().ravel(), ro, rtol=1e-2, atol=1e-2)
        np.testing.assert_allclose(lse.cpu().numpy().ravel(), rl, rtol=1e-3, atol=1e-3)
        checked += 1
    assert checked >= 2


def test_cache_holds_exactly_the_retained_blocks():
    """Occupancy == simulate_decode_cache's retained tokens (analysis.cpp:84-99)."""
    import torch

    N, H, D = 4096, 4, 128
    cfg = single(N, 64, H, 2, 3)
    plan = s2.Plan.from_config(cfg)
    cache = KVCache(plan, 1, D)
    pool, dense = cache.bytes()
    assert pool < dense
    for T in (1, 64, 65, 1000, 4096):
        z = torch.zeros(1, H, T, D, device="cuda", dtype=torch.bfloat16)
        cache.prefill(z, z)
        for g in range(H):
            ev = s2.evict_after(cfg, g)
            bt = (T - 1) // 64
            want = sum((64 if j < bt else T - bt * 64) for j in range(bt + 1) if ev[j] >= bt)
            assert cache.retained_tokens(g) == want


def test_non_kv_efficient_mask_rejected():
    cfg = s2.make_single_stride_config(2048, 64, 4, 3, 3, local_stride=2)
    plan = s2.Plan.from_config(cfg)
    with pytest.raises(s2.S2Unsupported):
        KVCache(plan, 1, 128)


def test_cache_tensor_contract_errors_raise():
    import torch

    cfg = single(1024, 64, 8, 2, 2, kv=2)
    cache = KVCache(s2.Plan.from_config(cfg), 2, 128)
    z = lambda *sh, dt=torch.bfloat16: torch.zeros(*sh, device="cuda", dtype=dt)  # noqa: E731
    with pytest.raises(s2.S2InvalidArgument):
        cache.prefill(z(2, 8, 10, 128), z(2, 8, 10, 128))      # query heads, not kv heads
    with pytest.raises(s2.S2InvalidArgument):
        cache.prefill(z(2, 2, 2000, 128), z(2, 2, 2000, 128))  # past the capacity
    cache.prefill(z(2, 2, 10, 128), z(2, 2, 10, 128))
    with pytest.raises(s2.S2InvalidArgument):
        cache.append(z(2, 2, 64), z(2, 2, 64))                 # head_dim
    with pytest.raises(s2.S2InvalidArgument):
        cache.decode(z(2, 8, 128, dt=torch.float32))           # dtype
    out, lse = cache.decode(z(2, 8, 128))
    assert out.shape == (2, 8, 128) and lse.shape == (2, 8)


@pytest.mark.parametrize("seed", range(16))
def test_decode_fuzz_matches_oracle(seed):
    """Seeded random KV-efficient configs (local_stride 1; the decode cache's
    block 64 and 1/2/4/8 query heads per kv head): prefill, a few appended
    tokens, decode at the last position vs the oracle's single-row restatement."""
    import random

    import torch

    rng = random.Random(9000 + seed)
    Hkv = rng.choice([1, 2, 4])
    hpg = rng.choice([1, 2, 4, 8])
    H = Hkv * hpg
    D = rng.choice([64, 128])
    blocks = rng.randint(2, 48)
    N = blocks * 64 - rng.randrange(64)
    batch = rng.randint(1, 3)
    local = 1 + rng.randrange(min(4, blocks))
    vs = rng.randint(1, 8)
    cfg = single(N, 64, H, local, vs, kv=Hkv)
    plan = s2.Plan.from_config(cfg)
    cache = KVCache(plan, batch, D)
    T0 = rng.randint(1, N - 1)
    T = min(N, T0 + rng.randint(0, 5))
    k, vv = _dense(batch, Hkv, T, D, seed)
    dev = torch.device("cuda")
    tk = torch.from_numpy(k).reshape(batch, Hkv, T, D).to(dev, torch.bfloat16)
    tv = torch.from_numpy(vv).reshape(batch, Hkv, T, D).to(dev, torch.bfloat16)
    cache.prefill(tk[:, :, :T0].contiguous(), tv[:, :, :T0].contiguous())
    for t in range(T0, T):
        cache.append(tk[:, :, t].contiguous(), tv[:, :, t].contiguous())
    assert cache.length == T
    q = bf16_round(np.random.default_rng(seed).uniform(-1, 1, batch * H * D).astype(np.float32))
    out, lse = cache.decode(torch.from_numpy(q).reshape(batch, H, D).to(dev, torch.bfloat16))
    torch.cuda.synchronize()
    rp, ci = oracle.csr_all(cfg)
    ro, rl = oracle.decode(q, k, vv, rp, ci, batch, H, Hkv, T, D, 64, T - 1, cfg.num_blocks())
    np.testing.assert_allclose(out.float().cpu().numpy().ravel(), ro, rtol=1e-2, atol=1e-2)
    np.testing.assert_allclose(lse.cpu().numpy().ravel(), rl, rtol=1e-3, atol=1e-3)
