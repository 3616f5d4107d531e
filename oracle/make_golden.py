"""ORACLE / TEST INFRASTRUCTURE ONLY.

Generates tests/golden/ from the reference itself (oracle/_ref, compiled from
/root/reference/proj/src).  Run here, where /root/reference exists:

    python oracle/make_golden.py

The fixtures let the GPU box (no /root/reference) pin both the C restatement
(oracle/s2_oracle.c) and the CUDA path to the reference's own outputs.
"""
import ctypes
import json
import os
import random
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import oracle  # noqa: E402
from paper_2407_17678_b200.pattern import PatternConfig, StrideSegment  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
REF_GOLDEN = "/root/reference/proj/tests/golden/csr_figure_left_head1.json"
REF_CONFIGS = "/root/reference/proj/configs"


def fnv1a64(arr: np.ndarray) -> str:
    h = 0xCBF29CE484222325
    for b in np.ascontiguousarray(arr, dtype="<i4").tobytes():
        h ^= b
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def fnv_fast(arr: np.ndarray) -> str:
    """FNV-1a over int32 words (vectorised-friendly variant used for big layouts)."""
    h = np.uint64(0xCBF29CE484222325)
    prime = np.uint64(0x100000001B3)
    with np.errstate(over="ignore"):
        for w in np.ascontiguousarray(arr, dtype=np.uint32).astype(np.uint64):
            h = (h ^ w) * prime
    return f"{int(h):016x}"


def cfg_to_dict(c: PatternConfig):
    return {"seq_len": c.seq_len, "block_size": c.block_size, "num_heads": c.num_heads,
            "num_kv_heads": c.num_kv_heads, "local_blocks": c.local_blocks,
            "local_stride": c.local_stride,
            "stride_segments": [{"start_block_distance": s.start_block_distance,
                                 "end_block_distance": s.end_block_distance, "stride": s.stride,
                                 "offsets": list(s.offsets)} for s in c.stride_segments]}


def single(N, S, H, local, v, local_stride=1, kv=0, offsets=None):
    c = PatternConfig(N, S, H, kv if kv else H, local, local_stride)
    B = c.num_blocks()
    if local < B:
        c.stride_segments.append(StrideSegment(local, B, v, list(offsets or [])))
    return c


def random_config(rng: random.Random) -> PatternConfig:
    """Python form of test_pattern.cpp:31-53 (ragged N, GQA, 1-2 segments)."""
    blocks = rng.randint(2, 32)
    c = PatternConfig()
    c.block_size = 1 + rng.randrange(16)
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
    return c


def layout_configs():
    cfgs = {
        "figure_left": single(8, 1, 4, 2, 3),
        "figure_right": single(8, 1, 4, 3, 3, local_stride=2),
        "cfg1_fp32_2k": single(2048, 64, 8, 4, 8),
        "cfg2_llama7b_8k": single(8192, 64, 32, 4, 16),
        "cfg3_32k": single(32768, 64, 32, 4, 16),
        "cfg4_decode_128k_gqa": single(131072, 64, 32, 4, 8, kv=8),
        "cfg5_128k": single(131072, 64, 32, 4, 16),
        "multi_stride": PatternConfig(4096, 64, 8, 8, 2, 1, [StrideSegment(2, 16, 3),
                                                             StrideSegment(16, 64, 7)]),
        "gqa_explicit_offsets": single(4096, 64, 8, 2, 4, kv=4, offsets=[1, 1, 3, 3, 0, 0, 2, 2]),
        "homo_head": single(4096, 64, 8, 2, 8, offsets=[0] * 8),
        "block128": single(8192, 128, 8, 2, 4),
        "block32_ragged": single(5000, 32, 4, 3, 5),
    }
    for name in sorted(os.listdir(REF_CONFIGS)) if os.path.isdir(REF_CONFIGS) else []:
        with open(os.path.join(REF_CONFIGS, name)) as f:
            p = json.load(f)["pattern"]
        cfgs["refcfg_" + name[:-5]] = PatternConfig(
            p["seq_len"], p["block_size"], p["num_heads"], p["num_kv_heads"], p["local_blocks"],
            p["local_stride"],
            [StrideSegment(s["start_block_distance"], s["end_block_distance"], s["stride"],
                           list(s.get("offsets", []))) for s in p["stride_segments"]])
    rng = random.Random(7)
    for i in range(40):
        cfgs[f"fuzz_{i:02d}"] = random_config(rng)
    return cfgs


def ref_csr_all(R, cfg):
    c, keep = cfg.to_c()
    n = ctypes.c_int64()
    assert R.ref_build_all_csr(ctypes.byref(c), None, None, ctypes.byref(n)) == 0, R.ref_last_error()
    B = cfg.num_blocks()
    rp = np.zeros(cfg.num_heads * (B + 1), np.int32)
    ci = np.zeros(max(n.value, 1), np.int32)
    assert R.ref_build_all_csr(ctypes.byref(c), oracle.ip(rp), oracle.ip(ci), ctypes.byref(n)) == 0
    return rp, ci[: n.value]


def main():
    R = oracle.ref()
    if R is None:
        sys.exit("reference library unavailable (needs /root/reference)")
    os.makedirs(GOLDEN, exist_ok=True)

    # 1. the reference's own golden CSR, reproduced through its library
    cfg = single(8, 1, 4, 2, 3)
    rp, ci = ref_csr_all(R, cfg)
    B = cfg.num_blocks()
    head1 = {"head_index": 1, "num_blocks": B, "row_ptr": rp[B + 1: 2 * (B + 1)].tolist(),
             "col_idx": ci[int(rp[B]): int(rp[B]) + int(rp[2 * (B + 1) - 1])].tolist()}
    if os.path.exists(REF_GOLDEN):
        with open(REF_GOLDEN) as f:
            g = json.load(f)
        assert g["row_ptr"] == head1["row_ptr"] and g["col_idx"] == head1["col_idx"]
    with open(os.path.join(GOLDEN, "csr_figure_left_head1.json"), "w") as f:
        json.dump(head1, f, indent=1)

    # 2. layouts: per head nnz + FNV-1a of row_ptr / col_idx, evict_after hash,
    #    kv-efficiency, exact_flops
    layouts = {}
    for name, cfg in layout_configs().items():
        c, keep = cfg.to_c()
        if R.ref_validate(ctypes.byref(c)) != 0:
            layouts[name] = {"config": cfg_to_dict(cfg), "invalid": R.ref_last_error().decode()}
            continue
        rp, ci = ref_csr_all(R, cfg)
        B = cfg.num_blocks()
        heads = []
        off = 0
        small = B <= 40
        for h in range(cfg.num_heads):
            r = rp[h * (B + 1):(h + 1) * (B + 1)]
            n = int(r[-1])
            col = ci[off: off + n]
            off += n
            entry = {"nnz": n, "row_ptr_fnv": fnv_fast(r), "col_idx_fnv": fnv_fast(col)}
            if small:
                entry["row_ptr"] = r.tolist()
                entry["col_idx"] = col.tolist()
            eff = ctypes.c_int()
            R.ref_kv_efficient(ctypes.byref(c), h, ctypes.byref(eff))
            entry["kv_efficient"] = bool(eff.value)
            if B <= 4096 and h < 2:
                ev = np.zeros(B, np.int32)
                occ = ctypes.c_int64()
                dead = ctypes.c_int()
                T = min(cfg.seq_len, 4096)
                assert R.ref_decode_cache(ctypes.byref(c), T, h, oracle.ip(ev), ctypes.byref(occ),
                                          ctypes.byref(dead)) == 0
                entry["evict_after_fnv"] = fnv_fast(ev)
                entry["decode_T"] = T
                entry["occupancy_last"] = int(occ.value)
                entry["dead_total"] = int(dead.value)
            heads.append(entry)
        dense = ctypes.c_double()
        sparse = ctypes.c_double()
        nph = np.zeros(cfg.num_heads, np.int64)
        R.ref_exact_flops(ctypes.byref(c), 128, ctypes.byref(dense), ctypes.byref(sparse),
                          nph.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)))
        layouts[name] = {"config": cfg_to_dict(cfg), "heads": heads,
                         "exact_flops_d128": {"dense": dense.value, "sparse": sparse.value}}
        print(f"layout {name}: B={B} nnz={sum(x['nnz'] for x in heads)}")
    with open(os.path.join(GOLDEN, "layouts.json"), "w") as f:
        json.dump(layouts, f, indent=0)

    # 3. RNG stream of AttentionTensors::random
    n = 2 * 3 * 4
    q = np.zeros(n, np.float32)
    k = np.zeros(n, np.float32)
    v = np.zeros(n, np.float32)
    R.ref_random_tensors(2, 3, 4, 7, oracle.fp(q), oracle.fp(k), oracle.fp(v))
    rng_fix = {"H": 2, "N": 3, "d": 4, "seed": 7, "q": q.tolist(), "k": k.tolist(),
               "v": v.tolist()}

    # 4. forward outputs of the reference streaming kernel
    fwd_cases = {
        "ragged_45_s8": dict(H=2, N=45, d=8, S=8, local=1, v=2, seed=61),
        "h3_n96_s16": dict(H=3, N=96, d=16, S=16, local=1, v=3, seed=17),
        "n1_single_token": dict(H=2, N=1, d=8, S=4, local=1, v=1, seed=3),
        "n6_lt_block": dict(H=2, N=6, d=8, S=8, local=1, v=1, seed=29),
        "h2_n256_s64_d64": dict(H=2, N=256, d=64, S=64, local=2, v=2, seed=5),
        "cfg1_fp32": dict(H=8, N=2048, d=64, S=64, local=4, v=8, seed=7),
        "h4_n1000_s64_d128": dict(H=4, N=1000, d=128, S=64, local=2, v=4, seed=11),
        "h2_n300_s16_d64_l3v5": dict(H=2, N=300, d=64, S=16, local=3, v=5, seed=13),
    }
    fwd = {}
    arrays = {}
    for name, p in fwd_cases.items():
        cfg = single(p["N"], p["S"], p["H"], p["local"], p["v"])
        rp, ci = ref_csr_all(R, cfg)
        nel = p["H"] * p["N"] * p["d"]
        q = np.zeros(nel, np.float32)
        k = np.zeros(nel, np.float32)
        v = np.zeros(nel, np.float32)
        R.ref_random_tensors(p["H"], p["N"], p["d"], p["seed"], oracle.fp(q), oracle.fp(k),
                             oracle.fp(v))
        out = np.zeros(nel, np.float32)
        lse = np.zeros(p["H"] * p["N"], np.float64)
        assert R.ref_streaming(p["H"], p["N"], p["d"], p["S"], 0.0, oracle.fp(q), oracle.fp(k),
                               oracle.fp(v), cfg.num_blocks(), oracle.ip(rp), oracle.ip(ci), 0,
                               oracle.fp(out), oracle.dp(lse)) == 0
        rec = dict(p)
        rec["config"] = cfg_to_dict(cfg)
        rec["q_sum"] = float(q.astype(np.float64).sum())
        rec["out_sum"] = float(out.astype(np.float64).sum())
        rec["lse_sum"] = float(lse.sum())
        if nel <= 20000:
            arrays[name + "__out"] = out
            arrays[name + "__lse"] = lse
        else:
            idx = np.arange(0, nel, 997)
            lidx = np.arange(0, lse.size, 97)
            arrays[name + "__out_idx"] = idx
            arrays[name + "__out"] = out[idx]
            arrays[name + "__lse_idx"] = lidx
            arrays[name + "__lse"] = lse[lidx]
        fwd[name] = rec
        print(f"fwd {name}: out_sum={rec['out_sum']:.6f}")
    np.savez_compressed(os.path.join(GOLDEN, "fwd_outputs.npz"), **arrays)
    with open(os.path.join(GOLDEN, "fwd_cases.json"), "w") as f:
        json.dump({"rng": rng_fix, "cases": fwd}, f, indent=1)


BAD_CONFIGS = {
    # test_serialize.cpp:113-133 cases (the reference's message must name the field)
    "missing_seq_len": '{"pattern": {"block_size": 64, "num_heads": 4}}',
    "stride_zero": '{"seq_len": 64, "block_size": 8, "num_heads": 4, "stride_segments": '
                   '[{"start_block_distance": 1, "end_block_distance": 8, "stride": 0}]}',
    "unknown_scheme": '{"seq_len": 64, "block_size": 8, "num_heads": 4, "offset_scheme": "mystery"}',
    "bad_dense_id": '{"seq_len": 512, "block_size": 64, "num_heads": 4, '
                    '"schedule": {"num_layers": 4, "dense_layer_ids": [7]}}',
    "not_json": '{"seq_len": 512, ',
}
GOOD_CONFIGS = {
    # test_serialize.cpp:96-111
    "with_schedule": '{"pattern": {"seq_len": 512, "block_size": 64, "num_heads": 4, "local_blocks": 1, '
                     '"stride_segments": [{"start_block_distance": 1, "end_block_distance": 8, '
                     '"stride": 2}]}, "schedule": {"num_layers": 12, "dense_layer_ids": [0]}, '
                     '"report": {"out": "r.csv", "format": "csv"}}',
    "bare": '{"seq_len": 64, "block_size": 8, "num_heads": 2}',
    "schedule_own_pattern": '{"seq_len": 512, "block_size": 64, "num_heads": 4, "schedule": '
                            '{"num_layers": 6, "dense_layer_ids": [5, 0], "sparse_pattern": '
                            '{"seq_len": 512, "block_size": 64, "num_heads": 4, "local_blocks": 2, '
                            '"stride_segments": [{"start_block_distance": 2, "end_block_distance": 8, '
                            '"stride": 3, "offsets": [0, 1, 2, 0]}]}}}',
}


def serialize_fixtures(R):
    """tests/golden/serialize.json: canonical documents, config hashes, config
    files, kv_reduction, decode-cache schedules and analytic closed forms,
    all produced by the reference library."""
    import tempfile

    out = {"patterns": {}, "config_files": {}, "kv_reduction": [], "decode_cache": {},
           "analytic": []}
    buf = ctypes.create_string_buffer(1 << 20)
    for name, cfg in layout_configs().items():
        c, keep = cfg.to_c()
        if R.ref_validate(ctypes.byref(c)) != 0:
            continue
        assert R.ref_config_json(ctypes.byref(c), buf, len(buf)) == 0
        h = ctypes.c_uint64()
        assert R.ref_config_hash(ctypes.byref(c), ctypes.byref(h)) == 0
        out["patterns"][name] = {"config": cfg_to_dict(cfg), "json": buf.value.decode(),
                                 "hash": f"{h.value:016x}"}
    texts = dict(GOOD_CONFIGS)
    texts.update(BAD_CONFIGS)
    for fn in sorted(os.listdir(REF_CONFIGS)) if os.path.isdir(REF_CONFIGS) else []:
        with open(os.path.join(REF_CONFIGS, fn)) as f:
            texts["refcfg_" + fn[:-5]] = f.read()
    bufs = [ctypes.create_string_buffer(1 << 16) for _ in range(4)]
    with tempfile.TemporaryDirectory() as d:
        for name, text in texts.items():
            path = os.path.join(d, name + ".json")
            with open(path, "w") as f:
                f.write(text)
            rc = R.ref_load_config(path.encode(), *bufs, 1 << 16)
            rec = {"text": text}
            if rc == 0:
                rec.update(pattern=bufs[0].value.decode(), schedule=bufs[1].value.decode(),
                           out=bufs[2].value.decode(), format=bufs[3].value.decode())
            else:
                rec["error"] = R.ref_last_error().decode().replace(path, "<path>")
            out["config_files"][name] = rec
    sched = [("cfg3_32k", 24, [0, 1]), ("cfg2_llama7b_8k", 32, []), ("cfg4_decode_128k_gqa", 32, [0, 31]),
             ("figure_left", 4, [1]), ("multi_stride", 12, [0, 5, 11]), ("refcfg_l1v15_dense01", 24, [0, 1]),
             ("refcfg_swa576_dense01", 24, [0, 1]), ("block32_ragged", 3, [])]
    cfgs = layout_configs()
    for name, L, dense in sched:
        c, keep = cfgs[name].to_c()
        ids = np.array(dense or [0], np.int32)
        pct = ctypes.c_double()
        assert R.ref_kv_reduction(ctypes.byref(c), L, oracle.ip(ids), len(dense), ctypes.byref(pct)) == 0
        out["kv_reduction"].append({"pattern": name, "num_layers": L, "dense": dense, "percent": pct.value})
    for name in ("figure_left", "figure_right", "cfg1_fp32_2k", "gqa_explicit_offsets", "block32_ragged",
                 "fuzz_03", "fuzz_11"):
        cfg = cfgs[name]
        c, keep = cfg.to_c()
        T = min(cfg.seq_len, 2048)
        heads = []
        for h in range(min(cfg.num_heads, 3)):
            ev = np.zeros(cfg.num_blocks(), np.int32)
            occ = np.zeros(T, np.int64)
            dead = np.zeros(T, np.int32)
            pk, mean = ctypes.c_int64(), ctypes.c_double()
            assert R.ref_decode_cache_full(ctypes.byref(c), T, h, oracle.ip(ev),
                                           occ.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                           oracle.ip(dead), ctypes.byref(pk), ctypes.byref(mean)) == 0
            heads.append({"evict_after": ev.tolist(), "occupancy": occ.tolist(), "dead": dead.tolist(),
                          "peak": int(pk.value), "mean": mean.value})
        out["decode_cache"][name] = {"config": cfg_to_dict(cfg), "total_tokens": T, "heads": heads}
    for seq, lw, st, hh in ((32768, 256, 16, 32), (131072, 256, 16, 32), (8192, 64, 15, 16), (4096, 4096, 1, 1)):
        eq, red, up = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        assert R.ref_analytic(seq, lw, st, hh, ctypes.byref(eq), ctypes.byref(red), ctypes.byref(up)) == 0
        out["analytic"].append({"seq_len": seq, "local_window": lw, "stride": st, "num_heads": hh,
                                "equivalent_context": eq.value, "reduction": red.value, "upper": up.value})
    with open(os.path.join(GOLDEN, "serialize.json"), "w") as f:
        json.dump(out, f, indent=0)
    print(f"serialize fixtures: {len(out['patterns'])} patterns, {len(out['config_files'])} files")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "serialize":
        serialize_fixtures(oracle.ref())
    else:
        main()
        serialize_fixtures(oracle.ref())
