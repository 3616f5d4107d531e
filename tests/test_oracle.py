"""Pins the C restatement (oracle/s2_oracle.c) to the reference.

Against the committed golden fixtures (made from the reference library by
oracle/make_golden.py) always, and live against oracle/_ref when the
reference sources exist (this container).
"""
import ctypes

import numpy as np
import pytest

from helpers import cfg_from_dict, fnv_fast, load_json, load_npz, single
import oracle

LAYOUTS = load_json("layouts.json")
FWD = load_json("fwd_cases.json")
FWD_ARR = load_npz("fwd_outputs.npz")


def port_csr(cfg):
    return oracle.csr_all(cfg)


def test_rng_stream_matches_reference_fixture():
    r = FWD["rng"]
    q, k, v = oracle.random_tensors(r["H"], r["N"], r["d"], r["seed"])
    assert q.tolist() == r["q"] and k.tolist() == r["k"] and v.tolist() == r["v"]


def test_product_random_tensors_is_the_reference_stream():
    """The Python mirror's AttentionTensors.random (s2_random_tensors in the
    library) reproduces the reference's mt19937_64 stream: the fixture made by
    the reference, and the port at a larger size."""
    import paper_2407_17678_b200 as s2

    r = FWD["rng"]
    t = s2.AttentionTensors.random(r["H"], r["N"], r["d"], r["seed"])
    assert t.q.tolist() == r["q"] and t.k.tolist() == r["k"] and t.v.tolist() == r["v"]
    t = s2.AttentionTensors.random(8, 2048, 64, 7)  # cfg1 with bench_attention.cpp:34's seed
    q, k, v = oracle.random_tensors(8, 2048, 64, 7)
    assert np.array_equal(t.q, q) and np.array_equal(t.k, k) and np.array_equal(t.v, v)


@pytest.mark.parametrize("name", list(LAYOUTS))
def test_port_layout_matches_reference_fixture(name):
    rec = LAYOUTS[name]
    cfg = cfg_from_dict(rec["config"])
    c, keep = cfg.to_c()
    msg = ctypes.create_string_buffer(256)
    rc = oracle.port().s2o_validate(ctypes.byref(c), msg, 256)
    if "invalid" in rec:
        assert rc == 1 and msg.value.decode() == rec["invalid"]
        return
    assert rc == 0
    rp, ci = port_csr(cfg)
    B = cfg.num_blocks()
    off = 0
    for h, e in enumerate(rec["heads"]):
        r = rp[h * (B + 1):(h + 1) * (B + 1)]
        col = ci[off: off + e["nnz"]]
        off += e["nnz"]
        assert int(r[-1]) == e["nnz"]
        if "row_ptr" in e:
            assert r.tolist() == e["row_ptr"] and col.tolist() == e["col_idx"]
        else:
            assert fnv_fast(r) == e["row_ptr_fnv"] and fnv_fast(col) == e["col_idx_fnv"]
        assert bool(oracle.port().s2o_kv_efficient(ctypes.byref(c), h)) == e["kv_efficient"]
        if "evict_after_fnv" in e:
            ev = np.zeros(B, np.int32)
            oracle.port().s2o_evict_after(ctypes.byref(c), h, oracle.ip(ev))
            assert fnv_fast(ev) == e["evict_after_fnv"]


def _case_inputs(p):
    return oracle.random_tensors(p["H"], p["N"], p["d"], p["seed"])


@pytest.mark.parametrize("name", list(FWD["cases"]))
def test_port_forward_matches_reference_fixture(name):
    p = FWD["cases"][name]
    cfg = cfg_from_dict(p["config"])
    q, k, v = _case_inputs(p)
    assert float(q.astype(np.float64).sum()) == p["q_sum"]
    rp, ci = port_csr(cfg)
    out, lse = oracle.attn_fwd(q, k, v, rp, ci, 1, p["H"], p["H"], p["N"], p["d"], p["S"])
    if name + "__out_idx" in FWD_ARR:
        out = out[FWD_ARR[name + "__out_idx"]]
        lse = lse[FWD_ARR[name + "__lse_idx"]]
    # same operation order as process_query_block -> bit-identical
    np.testing.assert_array_equal(out, FWD_ARR[name + "__out"])
    np.testing.assert_array_equal(lse, FWD_ARR[name + "__lse"])


# ---------------------------------------------------------------- live reference
ref = oracle.ref()
needs_ref = pytest.mark.skipif(ref is None, reason="reference sources not present")


@needs_ref
@pytest.mark.parametrize("seed", range(6))
def test_port_streaming_equals_reference_live(seed):
    rng = np.random.default_rng(seed)
    H = int(rng.integers(1, 5))
    N = int(rng.integers(8, 200))
    d = int(rng.choice([8, 16, 64]))
    S = int(rng.choice([4, 8, 16, 64]))
    v = int(rng.integers(1, 5))
    cfg = single(N, S, H, 1 + seed % 2 if -(-N // S) > 2 else 1, v)
    rp, ci = port_csr(cfg)
    q, k, vv = oracle.random_tensors(H, N, d, 1000 + seed)
    out, lse = oracle.attn_fwd(q, k, vv, rp, ci, 1, H, H, N, d, S)
    rout = np.zeros_like(out)
    rlse = np.zeros_like(lse)
    assert ref.ref_streaming(H, N, d, S, 0.0, oracle.fp(q), oracle.fp(k), oracle.fp(vv),
                             cfg.num_blocks(), oracle.ip(rp), oracle.ip(ci), 0, oracle.fp(rout),
                             oracle.dp(rlse)) == 0
    np.testing.assert_array_equal(out, rout)
    np.testing.assert_array_equal(lse, rlse)


@needs_ref
def test_port_random_equals_reference_live():
    for (H, N, d, seed) in [(2, 45, 8, 61), (3, 17, 5, 99)]:
        q, k, v = oracle.random_tensors(H, N, d, seed)
        n = H * N * d
        rq, rk, rv = (np.zeros(n, np.float32) for _ in range(3))
        ref.ref_random_tensors(H, N, d, seed, oracle.fp(rq), oracle.fp(rk), oracle.fp(rv))
        np.testing.assert_array_equal(q, rq)
        np.testing.assert_array_equal(k, rk)
        np.testing.assert_array_equal(v, rv)


# ------------------------------------------------------------------ backward pin
def _torch_token_mask(cfg, rp, ci, N):
    B = cfg.num_blocks()
    S = cfg.block_size
    H = cfg.num_heads
    m = np.zeros((H, N, N), bool)
    off = 0
    for h in range(H):
        r = rp[h * (B + 1):(h + 1) * (B + 1)]
        cols = ci[off: off + r[-1]]
        off += r[-1]
        for i in range(B):
            for j in cols[r[i]:r[i + 1]]:
                m[h, i * S:(i + 1) * S, j * S:(j + 1) * S] = True
    m &= np.tril(np.ones((N, N), bool))[None]
    return m


@pytest.mark.parametrize("case", [(2, 24, 8, 4, 1, 2), (3, 40, 16, 8, 2, 3), (2, 33, 8, 8, 1, 2)])
def test_port_backward_matches_torch_fp64_autograd(case):
    """backward restatement vs fp64 autograd on the token mask
    expanded from the layout (which itself matches the reference forward)."""
    torch = pytest.importorskip("torch")
    H, N, d, S, local, v = case
    cfg = single(N, S, H, local, v)
    rp, ci = port_csr(cfg)
    q, k, vv = oracle.random_tensors(H, N, d, 5)
    dout = np.random.default_rng(1).uniform(-1, 1, H * N * d).astype(np.float32)
    dq, dk, dv = oracle.attn_bwd(q, k, vv, dout, rp, ci, 1, H, H, N, d, S)
    mask = torch.from_numpy(_torch_token_mask(cfg, rp, ci, N))
    Q, K, V = (torch.from_numpy(x.astype(np.float64)).reshape(H, N, d).requires_grad_()
               for x in (q, k, vv))
    s = (Q @ K.transpose(-1, -2)) / np.sqrt(d)
    s = s.masked_fill(~mask, float("-inf"))
    o = torch.softmax(s, -1) @ V
    o.backward(torch.from_numpy(dout.astype(np.float64)).reshape(H, N, d))
    np.testing.assert_allclose(dq, Q.grad.numpy().ravel(), rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(dk, K.grad.numpy().ravel(), rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(dv, V.grad.numpy().ravel(), rtol=1e-5, atol=1e-6)


@needs_ref
def test_port_backward_matches_finite_differences_through_reference():
    """Central differences through the reference's own streaming forward."""
    H, N, d, S = 2, 24, 8, 4
    cfg = single(N, S, H, 1, 2)
    rp, ci = port_csr(cfg)
    q, k, v = oracle.random_tensors(H, N, d, 9)
    dout = np.random.default_rng(2).uniform(-1, 1, H * N * d).astype(np.float64)
    dq, dk, dv = oracle.attn_bwd(q, k, v, dout.astype(np.float32), rp, ci, 1, H, H, N, d, S)

    def loss(qq, kk, vv_):
        out = np.zeros(H * N * d, np.float32)
        lse = np.zeros(H * N, np.float64)
        assert ref.ref_streaming(H, N, d, S, 0.0, oracle.fp(qq), oracle.fp(kk), oracle.fp(vv_),
                                 cfg.num_blocks(), oracle.ip(rp), oracle.ip(ci), 0,
                                 oracle.fp(out), oracle.dp(lse)) == 0
        return float((out.astype(np.float64) * dout).sum())

    rng = np.random.default_rng(3)
    h = 1e-2
    for which, grad, base in (("q", dq, q), ("k", dk, k), ("v", dv, v)):
        for idx in rng.choice(base.size, 20, replace=False):
            args = {"q": q.copy(), "k": k.copy(), "v": v.copy()}
            args[which][idx] += h
            lp = loss(args["q"], args["k"], args["v"])
            args[which][idx] -= 2 * h
            lm = loss(args["q"], args["k"], args["v"])
            fd = (lp - lm) / (2 * h)
            assert abs(fd - grad[idx]) <= 5e-4 + 1e-3 * abs(fd), (which, idx, fd, grad[idx])


def test_port_decode_equals_forward_row():
    """Decode at position t == row t of the forward (SURVEY §8(c) decode pin)."""
    H, Hkv, N, d, S = 8, 2, 1000, 16, 64
    cfg = single(N, S, H, 2, 2, kv=Hkv)
    rp, ci = port_csr(cfg)
    rng = np.random.default_rng(4)
    q = rng.uniform(-1, 1, H * N * d).astype(np.float32)
    k = rng.uniform(-1, 1, Hkv * N * d).astype(np.float32)
    v = rng.uniform(-1, 1, Hkv * N * d).astype(np.float32)
    out, lse = oracle.attn_fwd(q, k, v, rp, ci, 1, H, Hkv, N, d, S)
    for t in (0, 63, 64, 500, 777, 999):
        qt = q.reshape(H, N, d)[:, t].copy()
        o, l = oracle.decode(qt, k, v, rp, ci, 1, H, Hkv, N, d, S, t, cfg.num_blocks())
        np.testing.assert_allclose(o, out.reshape(H, N, d)[:, t].ravel(), rtol=1e-6, atol=1e-7)
        np.testing.assert_allclose(l, lse.reshape(H, N)[:, t], rtol=1e-12)


@pytest.mark.parametrize("case", ["gqa_ragged", "batch2"])
def test_port_sampled_backward_rows_equal_full_backward(case):
    """s2o_bwd_sample (the full-size parity checker) restates s2o_attn_bwd at
    sampled rows: pinned against the full port backward on small cases."""
    if case == "gqa_ragged":
        cfg, batch, D = single(300, 16, 4, 2, 3, kv=2), 1, 32
    else:
        cfg, batch, D = single(256, 32, 2, 1, 2), 2, 16
    H, Hkv, N, S = cfg.num_heads, cfg.kv_heads(), cfg.seq_len, cfg.block_size
    rng = np.random.default_rng(11)
    q, do = (rng.uniform(-1, 1, batch * H * N * D).astype(np.float32) for _ in range(2))
    k, v = (rng.uniform(-1, 1, batch * Hkv * N * D).astype(np.float32) for _ in range(2))
    rp, ci = oracle.csr_all(cfg)
    dq, dk, dv = oracle.attn_bwd(q, k, v, do, rp, ci, batch, H, Hkv, N, D, S)
    q_rows = [(u, i) for u in range(batch * H) for i in (0, 1, S - 1, S, N // 2, N - 1)]
    k_rows = [(g, j) for g in range(batch * Hkv) for j in (0, S - 1, S, 2 * S + 3, N - 1)]
    sq, sk, sv = oracle.bwd_sample(q, k, v, do, rp, ci, batch, H, Hkv, N, D, S, q_rows, k_rows)
    dq, dk, dv = dq.reshape(-1, N, D), dk.reshape(-1, N, D), dv.reshape(-1, N, D)
    for n, (u, i) in enumerate(q_rows):
        np.testing.assert_allclose(sq[n], dq[u, i], rtol=1e-5, atol=1e-6)
    for n, (g, j) in enumerate(k_rows):
        np.testing.assert_allclose(sk[n], dk[g, j], rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(sv[n], dv[g, j], rtol=1e-5, atol=1e-6)


@pytest.mark.parametrize("case", ["gqa_ragged", "batch2", "local_stride"])
def test_parallel_port_backward_is_bit_identical(case):
    """s2o_attn_bwd_par (the CPU baseline's backward: parallel over rows, then over
    key blocks) equals s2o_attn_bwd bit for bit -- same expressions, same dK / dV
    accumulation order -- at any thread count."""
    import ctypes

    if case == "gqa_ragged":
        cfg, batch, D = single(300, 16, 4, 2, 3, kv=2), 1, 32
    elif case == "batch2":
        cfg, batch, D = single(256, 32, 2, 1, 2), 2, 16
    else:
        cfg, batch, D = single(500, 32, 4, 3, 2), 1, 16
        cfg.local_stride = 2
        cfg.validate()
    H, Hkv, N, S = cfg.num_heads, cfg.kv_heads(), cfg.seq_len, cfg.block_size
    rng = np.random.default_rng(12)
    q, do = (rng.uniform(-1, 1, batch * H * N * D).astype(np.float32) for _ in range(2))
    k, v = (rng.uniform(-1, 1, batch * Hkv * N * D).astype(np.float32) for _ in range(2))
    rp, ci = oracle.csr_all(cfg)
    ref = oracle.attn_bwd(q, k, v, do, rp, ci, batch, H, Hkv, N, D, S)
    gomp = ctypes.CDLL("libgomp.so.1")
    for threads in (1, 3, 8):
        gomp.omp_set_num_threads(threads)
        par = oracle.attn_bwd_par(q, k, v, do, rp, ci, batch, H, Hkv, N, D, S)
        for a, b in zip(par, ref):
            np.testing.assert_array_equal(a, b)
