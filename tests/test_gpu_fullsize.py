"""Parity at BASELINE.json's full sizes: the CUDA path on the
real configs, checked against the oracle on sampled rows and through
size-independent identities (the oracle cannot run a whole 32K/128K layer in
a test's time).

* Forward rows: row t of the forward == the oracle's single-row restatement at
  position t (s2o_decode; decode-at-t == forward row t is pinned in
  test_oracle.py::test_port_decode_equals_forward_row).
* Backward rows: s2o_bwd_sample (pinned against the full oracle backward in
  test_oracle.py) at sampled query rows (dQ) and key rows (dK, dV), including
  vertical-stride keys that every later row attends.
* Identities over every head and key: each row of P sums to 1, so
  sum_j dV_j = sum_i dO_i; each row of dS sums to 0, so sum_j dK_j = 0.  A
  missing or doubled tile breaks them far beyond the bf16 rounding noise.
* Decode: cfg4 (B=64, 128K context, 32q/8kv) over the compacted cache, sampled
  (sequence, kv-group) rows.

Inputs: U[-1,1] bf16 (the reference's distribution), seeded on the device.
Tolerance: rtol = atol = 1e-2 (north_star, bf16)."""
import numpy as np
import pytest

import paper_2407_17678_b200 as s2
import helpers  # noqa: F401  (puts oracle/ on sys.path)
import oracle

pytestmark = pytest.mark.gpu
TOL = dict(rtol=1e-2, atol=1e-2)


def _torch():
    import torch

    return torch


def _uniform(shape, gen):
    torch = _torch()
    return (torch.rand(shape, device="cuda", generator=gen) * 2 - 1).to(torch.bfloat16)


def _csr_heads(rp, ci, B, heads):
    """The (row_ptr, col_idx) of a subset of heads, in the oracle's packing."""
    rps, cis, off = [], [], 0
    per = [rp[h * (B + 1):(h + 1) * (B + 1)] for h in range(len(rp) // (B + 1))]
    offs = np.concatenate([[0], np.cumsum([int(r[-1]) for r in per])])
    for h in heads:
        rps.append(per[h])
        cis.append(ci[offs[h]: offs[h] + int(per[h][-1])])
    return np.concatenate(rps), np.concatenate(cis)


def _host(t):
    return t.float().cpu().numpy()


def _cfg3():
    return s2.make_s2_config(32768, 32, block_size=64, local_blocks=4, vert_stride=16)


def test_cfg3_forward_rows_match_oracle():
    torch = _torch()
    cfg = _cfg3()
    N, H, D, S = cfg.seq_len, cfg.num_heads, 128, cfg.block_size
    g = torch.Generator(device="cuda").manual_seed(31)
    q, k, v = (_uniform((1, H, N, D), g) for _ in range(3))
    plan = s2.Plan.from_config(cfg)
    out, lse = s2.s2_attn_fwd(plan, q, k, v)
    torch.cuda.synchronize()
    rp, ci = oracle.csr_all(cfg)
    hk, hv = _host(k), _host(v)
    for t in (0, 1, 63, 64, 1023, 4096, 16383, 20011, 32766, 32767):
        ro, rl = oracle.decode(_host(q[:, :, t]), hk, hv, rp, ci, 1, H, H, N, D, S, t, cfg.num_blocks())
        np.testing.assert_allclose(_host(out[:, :, t]).ravel(), ro, **TOL, err_msg=f"out row {t}")
        np.testing.assert_allclose(lse[:, :, t].cpu().numpy().ravel(), rl, **TOL, err_msg=f"lse row {t}")


def test_cfg3_backward_rows_and_identities():
    torch = _torch()
    cfg = _cfg3()
    N, H, D, S = cfg.seq_len, cfg.num_heads, 128, cfg.block_size
    g = torch.Generator(device="cuda").manual_seed(32)
    q, k, v, do = (_uniform((1, H, N, D), g) for _ in range(4))
    plan = s2.Plan.from_config(cfg)
    out, lse = s2.s2_attn_fwd(plan, q, k, v)
    dq, dk, dv = s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
    torch.cuda.synchronize()

    # identities over every head (fp64 sums on the device)
    sum_dv = dv.double().sum(dim=2)
    sum_do = do.double().sum(dim=2)
    scale_v = dv.double().abs().sum(dim=2)
    assert torch.all((sum_dv - sum_do).abs() <= 1e-3 * scale_v + 1e-3), "sum_j dV_j != sum_i dO_i"
    sum_dk = dk.double().sum(dim=2)
    scale_k = dk.double().abs().sum(dim=2)
    assert torch.all(sum_dk.abs() <= 1e-3 * scale_k + 1e-3), "sum_j dK_j != 0"

    # sampled rows against the oracle, heads 0 and 29 (offsets 0 and 13)
    heads = [0, 29]
    rp, ci = oracle.csr_all(cfg)
    srp, sci = _csr_heads(rp, ci, cfg.num_blocks(), heads)
    sel = lambda t: np.ascontiguousarray(_host(t[:, heads]).ravel())  # noqa: E731
    hq, hk, hv, hdo = sel(q), sel(k), sel(v), sel(do)
    q_rows = [(u, i) for u in range(2) for i in (0, 64, 4095, 16383, 32767)]
    k_rows = []
    for u, h in enumerate(heads):
        o = h % 16  # HeadModStride offset: block o + 16m is this head's stripe
        k_rows += [(u, (o + 16 * 3) * S + 5),   # a stripe key: attended by every later row
                   (u, (o + 16 * 3 + 1) * S + 7),  # a local-only key
                   (u, N - 1)]
    rq, rk, rv = oracle.bwd_sample(hq, hk, hv, hdo, srp, sci, 1, 2, 2, N, D, S, q_rows, k_rows)
    gq, gk, gv = (_host(t[0, heads]) for t in (dq, dk, dv))
    for n, (u, i) in enumerate(q_rows):
        np.testing.assert_allclose(gq[u, i], rq[n], **TOL, err_msg=f"dq head {heads[u]} row {i}")
    for n, (u, j) in enumerate(k_rows):
        np.testing.assert_allclose(gk[u, j], rk[n], **TOL, err_msg=f"dk head {heads[u]} key {j}")
        np.testing.assert_allclose(gv[u, j], rv[n], **TOL, err_msg=f"dv head {heads[u]} key {j}")


def test_cfg5_128k_forward_rows_match_oracle():
    torch = _torch()
    cfg = s2.make_s2_config(131072, 32, block_size=64, local_blocks=4, vert_stride=16)
    N, H, D, S = cfg.seq_len, cfg.num_heads, 128, cfg.block_size
    g = torch.Generator(device="cuda").manual_seed(33)
    q, k, v = (_uniform((1, H, N, D), g) for _ in range(3))
    plan = s2.Plan.from_config(cfg)
    out, lse = s2.s2_attn_fwd(plan, q, k, v)
    torch.cuda.synchronize()
    heads = [3, 30]
    rp, ci = oracle.csr_all(cfg)
    srp, sci = _csr_heads(rp, ci, cfg.num_blocks(), heads)
    hk = np.ascontiguousarray(_host(k[:, heads]).ravel())
    hv = np.ascontiguousarray(_host(v[:, heads]).ravel())
    for t in (0, 65535, 100003, 131071):
        ro, rl = oracle.decode(_host(q[:, heads, t]).ravel(), hk, hv, srp, sci, 1, 2, 2, N, D, S, t,
                               cfg.num_blocks())
        np.testing.assert_allclose(_host(out[:, heads, t]).ravel(), ro, **TOL, err_msg=f"out row {t}")
        np.testing.assert_allclose(lse[:, heads, t].cpu().numpy().ravel(), rl, **TOL)


def test_cfg5_128k_backward_rows_and_identities():
    """cfg5 (S=128K, H=32) fwd+bwd: the dK/dV identities over every head and key,
    and sampled dQ rows and dK/dV key rows of two heads against the oracle.  The
    key rows sit in the last stripe period (a stripe key attended by every later
    row, a local-only key, the last key), so the oracle's row sums stay short."""
    torch = _torch()
    cfg = s2.make_s2_config(131072, 32, block_size=64, local_blocks=4, vert_stride=16)
    N, H, D, S = cfg.seq_len, cfg.num_heads, 128, cfg.block_size
    B = cfg.num_blocks()
    g = torch.Generator(device="cuda").manual_seed(37)
    q, k, v, do = (_uniform((1, H, N, D), g) for _ in range(4))
    plan = s2.Plan.from_config(cfg)
    out, lse = s2.s2_attn_fwd(plan, q, k, v)
    dq, dk, dv = s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
    torch.cuda.synchronize()
    for h in range(H):  # sum_j dV_j = sum_i dO_i ; sum_j dK_j = 0, per head
        sdv, sdo = dv[0, h].double().sum(0), do[0, h].double().sum(0)
        assert torch.all((sdv - sdo).abs() <= 1e-3 * dv[0, h].double().abs().sum(0) + 1e-3), f"dV sum head {h}"
        assert torch.all(dk[0, h].double().sum(0).abs() <= 1e-3 * dk[0, h].double().abs().sum(0) + 1e-3), \
            f"dK sum head {h}"
    heads = [5, 26]
    rp, ci = oracle.csr_all(cfg)
    srp, sci = _csr_heads(rp, ci, B, heads)
    sel = lambda t: np.ascontiguousarray(_host(t[:, heads]).ravel())  # noqa: E731
    hq, hk, hv, hdo = sel(q), sel(k), sel(v), sel(do)
    q_rows = [(u, i) for u in range(2) for i in (0, 64, 65535, 100003, N - 1)]
    k_rows = []
    for u, h in enumerate(heads):
        o = h % 16
        sb = o + 16 * ((B - 8 - o) // 16)  # the last stripe block with >= 4 later blocks
        k_rows += [(u, sb * S + 5), (u, (sb + 1) * S + 7), (u, N - 1)]
    rq, rk, rv = oracle.bwd_sample(hq, hk, hv, hdo, srp, sci, 1, 2, 2, N, D, S, q_rows, k_rows)
    gq, gk, gv = (_host(t[0, heads]) for t in (dq, dk, dv))
    for n, (u, i) in enumerate(q_rows):
        np.testing.assert_allclose(gq[u, i], rq[n], **TOL, err_msg=f"dq head {heads[u]} row {i}")
    for n, (u, j) in enumerate(k_rows):
        np.testing.assert_allclose(gk[u, j], rk[n], **TOL, err_msg=f"dk head {heads[u]} key {j}")
        np.testing.assert_allclose(gv[u, j], rv[n], **TOL, err_msg=f"dv head {heads[u]} key {j}")


def test_cfg4_decode_full_context_matches_oracle():
    torch = _torch()
    from paper_2407_17678_b200.decode import KVCache

    Bd, Hq, Hk, T, D, S = 64, 32, 8, 131072, 128, 64
    cfg = s2.make_s2_config(T, Hq, num_kv_heads=Hk, block_size=S, local_blocks=4, vert_stride=8)
    plan = s2.Plan.from_config(cfg)
    cache = KVCache(plan, Bd, D)
    g = torch.Generator(device="cuda").manual_seed(34)
    k = _uniform((Bd, Hk, T, D), g)
    v = _uniform((Bd, Hk, T, D), g)
    cache.prefill(k, v)
    q = _uniform((Bd, Hq, D), g)
    out, lse = cache.decode(q)
    torch.cuda.synchronize()
    hpg = Hq // Hk
    rp, ci = oracle.csr_all(cfg)
    for b, grp in ((0, 0), (17, 3), (63, 7)):
        heads = list(range(grp * hpg, (grp + 1) * hpg))
        srp, sci = _csr_heads(rp, ci, cfg.num_blocks(), heads)
        ro, rl = oracle.decode(_host(q[b, heads]).ravel(), _host(k[b, grp]).ravel(), _host(v[b, grp]).ravel(),
                               srp, sci, 1, hpg, 1, T, D, S, T - 1, cfg.num_blocks())
        np.testing.assert_allclose(_host(out[b, heads]).ravel(), ro, **TOL, err_msg=f"seq {b} group {grp}")
        np.testing.assert_allclose(lse[b, heads].cpu().numpy().ravel(), rl, rtol=1e-3, atol=1e-3)


def test_cfg2_batch4_fwd_bwd_rows_match_oracle():
    """cfg2 (Llama-2-7B-shaped layer: B=4, H=32, N=8K, D=128, vert_stride 16):
    forward rows and backward rows of several (batch, head) units."""
    torch = _torch()
    cfg = s2.make_s2_config(8192, 32, block_size=64, local_blocks=4, vert_stride=16)
    Bt, N, H, D, S = 4, cfg.seq_len, cfg.num_heads, 128, cfg.block_size
    g = torch.Generator(device="cuda").manual_seed(35)
    q, k, v, do = (_uniform((Bt, H, N, D), g) for _ in range(4))
    plan = s2.Plan.from_config(cfg)
    out, lse = s2.s2_attn_fwd(plan, q, k, v)
    dq, dk, dv = s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
    torch.cuda.synchronize()
    rp, ci = oracle.csr_all(cfg)
    hq, hk, hv, hdo = (np.ascontiguousarray(_host(t).ravel()) for t in (q, k, v, do))
    for t in (0, 4095, 8191):
        ro, rl = oracle.decode(_host(q[:, :, t]).ravel(), hk, hv, rp, ci, Bt, H, H, N, D, S, t,
                               cfg.num_blocks())
        np.testing.assert_allclose(_host(out[:, :, t]).ravel(), ro, **TOL, err_msg=f"out row {t}")
        np.testing.assert_allclose(lse[:, :, t].cpu().numpy().ravel(), rl, **TOL)
    units = [(0, 0), (1, 7), (3, 31)]  # (batch, head)
    q_rows = [(b * H + h, i) for b, h in units for i in (0, 1000, 8191)]
    k_rows = [(b * H + h, j) for b, h in units for j in ((h % 16) * S + 3, 4096 + 9, N - 1)]
    rq, rk, rv = oracle.bwd_sample(hq, hk, hv, hdo, rp, ci, Bt, H, H, N, D, S, q_rows, k_rows)
    gq, gk, gv = (_host(t).reshape(Bt * H, N, D) for t in (dq, dk, dv))
    for n, (u, i) in enumerate(q_rows):
        np.testing.assert_allclose(gq[u, i], rq[n], **TOL, err_msg=f"dq unit {u} row {i}")
    for n, (u, j) in enumerate(k_rows):
        np.testing.assert_allclose(gk[u, j], rk[n], **TOL, err_msg=f"dk unit {u} key {j}")
        np.testing.assert_allclose(gv[u, j], rv[n], **TOL, err_msg=f"dv unit {u} key {j}")


def test_512k_forward_backward_rows_match_oracle():
    """Past the largest BASELINE config (128K): a 512K-token layer (B=8192 blocks,
    32 heads) -- the plan's lists, the persistent schedules and 64-bit offsets at
    4 GB per tensor.  Sampled forward rows and the dK/dV identities."""
    torch = _torch()
    cfg = s2.make_s2_config(524288, 32, block_size=64, local_blocks=4, vert_stride=16)
    N, H, D, S = cfg.seq_len, cfg.num_heads, 128, cfg.block_size
    g = torch.Generator(device="cuda").manual_seed(36)
    q, k, v, do = (_uniform((1, H, N, D), g) for _ in range(4))
    plan = s2.Plan.from_config(cfg)
    out, lse = s2.s2_attn_fwd(plan, q, k, v)
    dq, dk, dv = s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
    torch.cuda.synchronize()
    heads = [1, 31]
    rp, ci = oracle.csr_all(cfg)
    srp, sci = _csr_heads(rp, ci, cfg.num_blocks(), heads)
    hk = np.ascontiguousarray(_host(k[:, heads]).ravel())
    hv = np.ascontiguousarray(_host(v[:, heads]).ravel())
    for t in (0, 300001, N - 1):
        ro, rl = oracle.decode(_host(q[:, heads, t]).ravel(), hk, hv, srp, sci, 1, 2, 2, N, D, S, t,
                               cfg.num_blocks())
        np.testing.assert_allclose(_host(out[:, heads, t]).ravel(), ro, **TOL, err_msg=f"out row {t}")
        np.testing.assert_allclose(lse[:, heads, t].cpu().numpy().ravel(), rl, **TOL)
    for h in heads:  # sum_j dV_j = sum_i dO_i ; sum_j dK_j = 0
        sdv, sdo = dv[0, h].double().sum(0), do[0, h].double().sum(0)
        assert torch.all((sdv - sdo).abs() <= 1e-3 * dv[0, h].double().abs().sum(0) + 1e-3)
        assert torch.all(dk[0, h].double().sum(0).abs() <= 1e-3 * dk[0, h].double().abs().sum(0) + 1e-3)
