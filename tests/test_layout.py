"""Product layout builder (csrc/layout.cpp via the C ABI) vs the reference.

Bit-exact CSR against the reference-generated fixtures for every BASELINE
config, the reference's proj/configs, explicit-offset / GQA / multi-stride
variants and 40 configs from the reference's own fuzz generator
(test_pattern.cpp:31-53); restated pins of test_pattern.cpp / test_csr.cpp.
"""
import ctypes

import numpy as np
import pytest

import paper_2407_17678_b200 as s2
from helpers import cfg_from_dict, fnv_fast, fnv_py, load_json, single
import oracle

LAYOUTS = load_json("layouts.json")


@pytest.mark.parametrize("name", list(LAYOUTS))
def test_csr_bit_exact_vs_reference(name):
    rec = LAYOUTS[name]
    cfg = cfg_from_dict(rec["config"])
    if "invalid" in rec:
        with pytest.raises(s2.S2InvalidArgument, match=rec["invalid"]):
            cfg.validate()
        return
    for h, e in enumerate(rec["heads"]):
        c = s2.build_csr(cfg, h)
        assert c.nnz() == e["nnz"]
        if "row_ptr" in e:
            assert c.row_ptr.tolist() == e["row_ptr"] and c.col_idx.tolist() == e["col_idx"]
        else:  # every head, 128K configs included (C-folded fingerprint)
            assert fnv_fast(c.row_ptr) == e["row_ptr_fnv"]
            assert fnv_fast(c.col_idx) == e["col_idx_fnv"]
        assert s2.kv_efficient(cfg, h) == e["kv_efficient"]
        if "evict_after_fnv" in e:
            assert fnv_fast(s2.evict_after(cfg, h)) == e["evict_after_fnv"]


def test_c_fingerprint_equals_the_python_fold():
    rng = np.random.default_rng(3)
    for n in (0, 1, 7, 1000):
        a = rng.integers(0, 2**31, n, dtype=np.int64).astype(np.uint32)
        assert fnv_fast(a) == fnv_py(a)


def test_plan_flops_match_reference_exact_flops():
    for name in ("cfg1_fp32_2k", "cfg2_llama7b_8k", "cfg3_32k", "refcfg_l1v16"):
        rec = LAYOUTS[name]
        cfg = cfg_from_dict(rec["config"])
        plan = s2.Plan.from_config(cfg)
        active, dense = plan.fwd_flops(1, 128)
        assert active == rec["exact_flops_d128"]["sparse"]
        assert dense == rec["exact_flops_d128"]["dense"]


def test_golden_file_of_the_reference():
    g = load_json("csr_figure_left_head1.json")
    c = s2.build_csr(s2.make_single_stride_config(8, 1, 4, 2, 3), 1)
    assert c.head_index == g["head_index"]
    assert c.row_ptr.tolist() == g["row_ptr"] and c.col_idx.tolist() == g["col_idx"]


def test_worked_rows():
    # test_pattern.cpp:65-79, test_csr.cpp:22-28
    m = s2.build_head_mask(s2.make_single_stride_config(8, 1, 4, 2, 3), 1)
    assert m.row(7) == [1, 4, 6, 7] and m.row(0) == [0] and m.row(2) == [1, 2]
    m = s2.build_head_mask(s2.make_single_stride_config(8, 1, 4, 3, 3, 2), 0)
    assert m.row(6) == [0, 3, 4, 6]


def test_dense_and_triangle():
    # test_csr.cpp:16-20, test_pattern.cpp:81-87
    c = s2.to_csr(s2.dense_causal_mask(3))
    assert c.row_ptr.tolist() == [0, 1, 3, 6] and c.col_idx.tolist() == [0, 0, 1, 0, 1, 2]
    cfg = s2.make_single_stride_config(16, 2, 3, 1, 1)
    for h in range(3):
        assert s2.same_bits(s2.build_head_mask(cfg, h), s2.dense_causal_mask(cfg.num_blocks()))


def test_gqa_homogeneous_and_heterogeneous():
    # test_pattern.cpp:105-113
    cfg = s2.make_single_stride_config(32, 1, 4, 1, 3)
    cfg.num_kv_heads = 2
    m = s2.build_all_masks(cfg)
    assert s2.same_bits(m[0], m[1]) and s2.same_bits(m[2], m[3])
    assert not s2.same_bits(m[0], m[2])


def test_offsets_normalised_modulo_stride():
    # test_pattern.cpp:169-180
    cfg = s2.make_single_stride_config(16, 1, 4, 1, 3)
    cfg.stride_segments[0].offsets = [0, 4, 8, 12]
    plain = s2.make_single_stride_config(16, 1, 4, 1, 3)
    plain.stride_segments[0].offsets = [0, 1, 2, 0]
    for a, b in zip(s2.build_all_masks(cfg), s2.build_all_masks(plain)):
        assert s2.same_bits(a, b)


def test_validation_errors_like_reference():
    # test_pattern.cpp:193-226
    base = s2.make_single_stride_config(8, 1, 4, 2, 3)
    with pytest.raises(s2.S2InvalidArgument):
        s2.build_csr(base, -1)
    with pytest.raises(s2.S2InvalidArgument):
        s2.build_csr(base, 4)

    def bad(mut):
        c = s2.make_single_stride_config(8, 1, 4, 2, 3)
        mut(c)
        with pytest.raises(s2.S2InvalidArgument):
            c.validate()

    bad(lambda c: setattr(c.stride_segments[0], "start_block_distance", 1))
    bad(lambda c: setattr(c.stride_segments[0], "end_block_distance", 9))
    bad(lambda c: setattr(c.stride_segments[0], "stride", 0))
    bad(lambda c: c.stride_segments.append(s2.StrideSegment(2, 8, 2)))
    bad(lambda c: setattr(c, "num_kv_heads", 3))
    bad(lambda c: setattr(c.stride_segments[0], "offsets", [0, -1, 0, 0]))

    def gqa_disagree(c):
        c.num_kv_heads = 2
        c.stride_segments[0].offsets = [0, 1, 0, 0]

    bad(gqa_disagree)


def test_ragged_block_count():
    cfg = s2.make_single_stride_config(100, 16, 2, 1, 2)
    assert cfg.num_blocks() == 7 and s2.build_head_mask(cfg, 0).num_blocks() == 7


def test_csc_is_transpose_and_roundtrip():
    # test_csr.cpp:75-102 + the CSC pin of SURVEY §8(c)
    rng = np.random.default_rng(17)
    for _ in range(20):
        blocks = int(rng.integers(2, 26))
        cfg = s2.make_single_stride_config(blocks, 1, int(rng.integers(1, 7)),
                                           int(rng.integers(1, min(3, blocks) + 1)),
                                           int(rng.integers(1, 6)))
        for h in range(cfg.num_heads):
            m = s2.build_head_mask(cfg, h)
            csr = s2.to_csr(m)
            assert s2.from_csr(csr, blocks) == m and csr.nnz() == m.popcount()
            csc = s2.build_csc(cfg, h)
            for j in range(blocks):
                assert csc.row(j) == np.nonzero(m.bits[:, j])[0].tolist()


def test_malformed_csr_rejected():
    # test_csr.cpp:66-102
    good = s2.to_csr(s2.dense_causal_mask(4))

    def bad(mut):
        c = s2.CsrMask(0, 4, good.row_ptr.copy(), good.col_idx.copy())
        mut(c)
        with pytest.raises(s2.S2InvalidArgument):
            c.validate()

    bad(lambda c: c.col_idx.__setitem__(-1, 4))
    bad(lambda c: c.row_ptr.__setitem__(0, 1))
    bad(lambda c: c.row_ptr.__setitem__(-1, 3))

    def desc(c):
        a, b = c.row_ptr[3], c.row_ptr[3] + 1
        c.col_idx[a], c.col_idx[b] = c.col_idx[b], c.col_idx[a]

    bad(desc)
    bad(lambda c: c.col_idx.__setitem__(c.row_ptr[2], 3))
    with pytest.raises(s2.S2InvalidArgument):
        s2.from_csr(good, 5)


@pytest.mark.parametrize("seed", range(30))
def test_product_equals_port_formula_on_fuzz(seed):
    """Every bit of random configs vs the formula restatement (test_pattern.cpp:145-160)."""
    import random

    from make_golden import random_config

    cfg = random_config(random.Random(1000 + seed))
    c, keep = cfg.to_c()
    P = oracle.port()
    B = cfg.num_blocks()
    for h in range(cfg.num_heads):
        m = s2.build_head_mask(cfg, h)
        for i in range(B):
            for j in range(B):
                assert m.bits[i, j] == P.s2o_mask_bit(ctypes.byref(c), h, i, j)


def test_layer_schedule():
    # test_pattern.cpp:115-143
    sched = s2.LayerSchedule(24, {0, 1}, s2.make_single_stride_config(8, 1, 4, 2, 3))
    layers = s2.build_layer_masks(sched)
    dense = s2.dense_causal_mask(8)
    assert all(s2.same_bits(layers[l][h], dense) for l in (0, 1) for h in range(4))
    assert all(layers[l][h] == s2.build_head_mask(sched.sparse_pattern, h)
               for l in range(2, 24) for h in range(4))


def test_partitioner_lpt_balance():
    plan = s2.Plan.from_config(single(32768, 64, 32, 4, 16))
    w = plan.unit_weights(1)
    from paper_2407_17678_b200.dist import partition_lpt

    for G in (1, 2, 4, 8):
        owner, load = partition_lpt(w, G)
        assert sorted(set(owner.tolist())) == list(range(G))
        assert load.sum() == w.sum()
        assert load.max() / (w.sum() / G) < 1.01  # 1.000 at cfg3


def test_tile_lists_cover_every_block_pair_exactly():
    """Fwd chunk lists and bwd (transposed) lists cover exactly the layout's
    token pairs at 16x16 granularity."""
    for cfg in (single(1000, 64, 4, 2, 3), single(777, 32, 2, 3, 5), single(4096, 128, 2, 1, 4),
                single(2048, 16, 2, 4, 7, kv=1)):
        plan = s2.Plan.from_config(cfg)
        st = plan.stats()
        assert st["fwd_tiles"] == cfg.num_heads * -(-cfg.seq_len // 128)
        assert st["fwd_chunk_visits"] > 0 and st["bwd_qtile_visits"] > 0


def _fwd_lists(plan):
    L = s2.lib()
    nq = ctypes.c_int()
    ne = ctypes.c_int64()
    s2._abi.check(L.s2_plan_fwd_tiles(plan.handle, ctypes.byref(nq), ctypes.byref(ne), None,
                                      None, None))
    off = np.zeros(plan.num_heads * nq.value + 1, np.int64)
    ch = np.zeros(max(ne.value, 1), np.int32)
    mk = np.zeros(max(ne.value, 1), np.uint32)
    s2._abi.check(L.s2_plan_fwd_tiles(
        plan.handle, ctypes.byref(nq), ctypes.byref(ne),
        off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
        ch.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
        mk.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))))
    return nq.value, off, ch[: ne.value], mk[: ne.value]


def _bwd_lists(plan):
    L = s2.lib()
    nt = ctypes.c_int64()
    ne = ctypes.c_int64()
    s2._abi.check(L.s2_plan_bwd_tiles(plan.handle, ctypes.byref(nt), ctypes.byref(ne), None, None))
    tiles = np.zeros(5 * nt.value, np.int64)
    ent = np.zeros(3 * max(ne.value, 1), np.int64)
    s2._abi.check(L.s2_plan_bwd_tiles(plan.handle, ctypes.byref(nt), ctypes.byref(ne),
                                      tiles.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                      ent.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
    return tiles.reshape(-1, 5), ent[: 3 * ne.value].reshape(-1, 3)


def _expected_bits(cfg, h):
    """Token-level (16x16 square) attend map of head h from the reference mask."""
    N, S = cfg.seq_len, cfg.block_size
    m = s2.build_head_mask(cfg, h).bits
    g = -(-N // 16)
    rows = np.arange(g) * 16 // S
    return m[np.ix_(rows, rows)].astype(bool)  # [row group, col group]


@pytest.mark.parametrize("cfg", [single(1000, 64, 4, 2, 3), single(777, 32, 2, 3, 5),
                                 single(4096, 128, 2, 1, 4), single(2048, 16, 4, 4, 7, kv=2),
                                 single(8192, 64, 2, 4, 16)])
def test_fwd_and_bwd_tile_lists_are_exact_covers(cfg):
    plan = s2.Plan.from_config(cfg)
    nq, off, ch, mk = _fwd_lists(plan)
    ngrp = -(-cfg.seq_len // 16)
    hpg = cfg.heads_per_group()
    tiles, ent = _bwd_lists(plan)
    for h in range(cfg.num_heads):
        want = _expected_bits(cfg, h)
        got = np.zeros_like(want)
        for t in range(nq):
            w = h * nq + t
            cs = ch[off[w]:off[w + 1]]
            assert np.all(np.diff(cs) > 0)  # ascending, unique
            for c, m in zip(cs, mk[off[w]:off[w + 1]]):
                for g in range(8):
                    for cg in range(4):
                        if (int(m) >> (g * 4 + cg)) & 1:
                            r, k = t * 8 + g, c * 4 + cg
                            assert r < ngrp and k < ngrp
                            got[r, k] = True
        np.testing.assert_array_equal(got, want)
        if h % hpg:
            continue
        # transposed list of this head's group: same bits again
        gotb = np.zeros_like(want)
        for grp, c0, c1, o, n in tiles[tiles[:, 0] == h // hpg]:
            qt = ent[o:o + n, 0]
            assert np.all(np.diff(qt) > 0)
            for (t, m0, m1) in ent[o:o + n]:
                for c, m in ((c0, m0), (c1, m1)):
                    if c < 0:
                        assert m == 0
                        continue
                    for g in range(8):
                        for cg in range(4):
                            if (int(m) >> (g * 4 + cg)) & 1:
                                gotb[t * 8 + g, c * 4 + cg] = True
        np.testing.assert_array_equal(gotb, want)
