"""JSON documents, config files, config_hash and the layout analysis
(SURVEY §8(f) row 1, and the analysis half of row 2) against fixtures the
reference library produced (oracle/make_golden.py serialize_fixtures:
to_json / config_hash / load_config_file / kv_reduction /
simulate_decode_cache / the analytic closed forms), plus the reference's own
test_serialize.cpp cases restated.  CPU only: no device is touched."""
import json
import os

import numpy as np
import pytest

import paper_2407_17678_b200 as s2
from paper_2407_17678_b200 import analysis, serialize
from paper_2407_17678_b200.pattern import LayerSchedule, make_multi_stride_config, make_single_stride_config
from helpers import cfg_from_dict, load_json

FIX = load_json("serialize.json")


@pytest.mark.parametrize("name", sorted(FIX["patterns"]))
def test_canonical_document_and_hash_match_reference(name):
    rec = FIX["patterns"][name]
    cfg = cfg_from_dict(rec["config"])
    doc = s2.to_json(cfg)
    assert serialize.dumps(doc) == rec["json"]
    assert s2.config_hash(cfg) == int(rec["hash"], 16)
    back = s2.pattern_config_from_json(rec["json"])  # serialize.cpp:75-95
    assert serialize.dumps(s2.to_json(back)) == rec["json"]
    assert s2.config_hash(back) == int(rec["hash"], 16)


@pytest.mark.parametrize("name", sorted(FIX["config_files"]))
def test_config_files_load_like_the_reference(name, tmp_path):
    rec = FIX["config_files"][name]
    path = tmp_path / f"{name}.json"
    path.write_text(rec["text"])
    if "error" in rec:
        with pytest.raises(s2.S2ConfigError) as ei:
            s2.load_config_file(str(path))
        msg = str(ei.value)
        assert f"config '{path}'" in msg
        # the reference's message after the path: same offending field / reason
        ref_reason = rec["error"].split("': ", 1)[1]
        key = {"missing_seq_len": "seq_len", "stride_zero": "stride", "unknown_scheme": "offset_scheme",
               "bad_dense_id": "dense layer id 7", "not_json": "parse error"}[name]
        assert key in ref_reason and key in msg
        return
    f = s2.load_config_file(str(path))
    assert serialize.dumps(s2.to_json(f.pattern)) == rec["pattern"]
    if rec["schedule"]:
        assert f.schedule is not None
        assert serialize.dumps(s2.to_json(f.schedule)) == rec["schedule"]
    else:
        assert f.schedule is None
    assert f.out == rec["out"] and f.format == rec["format"]


def test_missing_config_file_is_a_config_error():
    with pytest.raises(s2.S2ConfigError, match="cannot open config file"):
        s2.load_config_file("does_not_exist.json")


def test_pattern_round_trip_with_offsets_and_gqa():
    """test_serialize.cpp:30-49."""
    cfg = make_multi_stride_config(256, 16, 8, 2, 8, 3, 6)
    cfg.num_kv_heads = 4
    cfg.stride_segments[0].offsets = [0, 1, 2, 0]
    cfg.validate()
    doc = s2.to_json(cfg)
    for key in ("seq_len", "block_size", "num_heads", "num_kv_heads", "local_blocks", "local_stride",
                "stride_segments", "offset_scheme"):
        assert key in doc
    for key in ("start_block_distance", "end_block_distance", "stride"):
        assert key in doc["stride_segments"][0]
    back = s2.pattern_config_from_json(doc)
    assert s2.to_json(back) == doc
    assert s2.config_hash(back) == s2.config_hash(cfg)


def test_schedule_round_trip_and_inheritance():
    """test_serialize.cpp:51-67."""
    sched = LayerSchedule(24, {0, 1}, make_single_stride_config(512, 64, 4, 1, 4))
    doc = s2.to_json(sched)
    back = s2.layer_schedule_from_json(doc, sched.sparse_pattern)
    assert back.num_layers == 24 and back.dense_layer_ids == {0, 1}
    assert s2.to_json(back.sparse_pattern) == s2.to_json(sched.sparse_pattern)
    inherited = s2.layer_schedule_from_json({"num_layers": 8}, sched.sparse_pattern)
    assert inherited.dense_layer_ids == set()
    assert s2.to_json(inherited.sparse_pattern) == s2.to_json(sched.sparse_pattern)
    with pytest.raises(s2.S2InvalidArgument, match="outside"):
        s2.layer_schedule_from_json({"num_layers": 2, "dense_layer_ids": [2]}, sched.sparse_pattern)


def test_csr_documents_round_trip_and_golden():
    """test_serialize.cpp:88-94 and the reference's golden CSR file."""
    g = load_json("csr_figure_left_head1.json")
    csr = s2.csr_from_json(g)
    ours = s2.build_csr(make_single_stride_config(8, 1, 4, 2, 3), 1)
    assert csr.head_index == 1 and csr.num_blocks == 8
    assert csr.row_ptr.tolist() == ours.row_ptr.tolist() == g["row_ptr"]
    assert csr.col_idx.tolist() == ours.col_idx.tolist() == g["col_idx"]
    assert s2.to_json(csr) == {**g}
    bad = dict(g, col_idx=[0, 1] + g["col_idx"][2:])  # row 1 lists 0 then ... not ascending/causal
    bad["col_idx"][1] = 5
    with pytest.raises(s2.S2InvalidArgument):
        s2.csr_from_json(bad)


def test_config_hash_is_content_sensitive():
    """test_serialize.cpp:135-141."""
    a = make_single_stride_config(512, 64, 4, 1, 4)
    b = make_single_stride_config(512, 64, 4, 1, 4)
    assert s2.config_hash(a) == s2.config_hash(b)
    b.stride_segments[0].stride = 5
    assert s2.config_hash(a) != s2.config_hash(b)


@pytest.mark.parametrize("i", range(len(FIX["kv_reduction"])))
def test_kv_reduction_matches_reference(i):
    rec = FIX["kv_reduction"][i]
    pat = cfg_from_dict(FIX["patterns"][rec["pattern"]]["config"])
    got = s2.kv_reduction(LayerSchedule(rec["num_layers"], set(rec["dense"]), pat))
    assert got == pytest.approx(rec["percent"], rel=0, abs=1e-9)


@pytest.mark.parametrize("name", sorted(FIX["decode_cache"]))
def test_decode_cache_schedule_matches_reference(name):
    rec = FIX["decode_cache"][name]
    cfg = cfg_from_dict(rec["config"])
    cs = s2.simulate_decode_cache(cfg, rec["total_tokens"])
    for h, want in enumerate(rec["heads"]):
        got = cs.heads[h]
        assert got.evict_after.tolist() == want["evict_after"]
        assert got.occupancy.tolist() == want["occupancy"]
        assert got.dead_blocks.tolist() == want["dead"]
        assert got.peak_tokens == want["peak"]
        assert got.mean_tokens == pytest.approx(want["mean"], rel=1e-12)


@pytest.mark.parametrize("i", range(len(FIX["analytic"])))
def test_analytic_closed_forms(i):
    r = FIX["analytic"][i]
    assert analysis.equivalent_context_length(r["seq_len"], r["local_window"], r["stride"]) == r["equivalent_context"]
    assert analysis.analytic_flops_reduction(r["seq_len"], r["local_window"], r["stride"]) == r["reduction"]
    assert analysis.speedup_upper_bound(r["num_heads"], r["seq_len"], r["local_window"]) == r["upper"]
    with pytest.raises(s2.S2InvalidArgument):
        analysis.equivalent_context_length(100, 0, 2)
    with pytest.raises(s2.S2InvalidArgument):
        analysis.equivalent_context_length(100, 10, 0.5)


def test_exact_flops_matches_layout_fixture():
    lay = load_json("layouts.json")
    for name, rec in lay.items():
        if "invalid" in rec:
            continue
        cfg = cfg_from_dict(rec["config"])
        if cfg.num_blocks() > 4096:
            continue
        rep = s2.exact_flops(cfg, 128)
        assert rep.dense_flops == rec["exact_flops_d128"]["dense"]
        assert rep.sparse_flops == rec["exact_flops_d128"]["sparse"]
        assert rep.nnz_per_head == [h["nnz"] for h in rec["heads"]]
        assert rep.reduction_factor == rep.dense_flops / rep.sparse_flops
