#!/usr/bin/env python
"""GPU selftest verb: the reference's oracle-equivalence
matrix (`shardattn selftest`, main.cpp:144-164; run_selftest,
selftest.cpp:61-146) with the B200 kernels swapped in for the streaming and
D-split kernels.  TEST INFRASTRUCTURE: it lives under tests/ because its
checker is the oracle restatement (oracle/s2_oracle.c).

Grid (as the reference): seq_len in {16, 64, 128, 256} x block_size in
{8, 16, 64} x head_dim in {16, 64} x stride in {1, 3, 4, H}, plus a 2-head
variant for seq_len <= 64: 144 instances.  Inputs are
AttentionTensors::random(H, N, d, seed + instance) (bit-exact port).
Per instance:
  oracle_vs_streaming   fp32 reference-precision kernel (fwd_simt) vs the
                        oracle's streaming restatement; allclose ratio
                        max|a-b|/(1e-4 + 1e-4|b|) <= 1 (north_star fp32 tolerance)
  streaming_vs_dsplit2  num_splits = 2 (d even) on the GPU;            <= 1e-5
  streaming_vs_dsplit1  dsplit(1) and streaming are the same launch;   == 0 (1e-6 as the reference)
  oracle_vs_tcgen05     bf16 tcgen05 kernel on bf16-rounded inputs (block % 16 == 0,
                        head_dim 64): allclose ratio max|a-b|/(1e-2 + 1e-2|b|) <= 1
  oracle_vs_tcgen05_bwd bf16 backward (dQ, dK, dV) vs the oracle's gradient; same ratio
CSV (one row per comparison, the reference's columns):
  config,seq_len,block_size,head_dim,num_heads,stride,comparison,tolerance,max_rel_error,status
Exit codes as the reference CLI: 0 all pass, 1 a comparison failed, 2 bad
usage / environment (no GPU, missing library).

    python tests/selftest.py [--seed 42] [--seq-lens 16,64,128,256] [--csv out.csv]
                             [--inject-corruption]
"""
import argparse
import io
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def max_rel(a, b):
    """max_relative_error (selftest.cpp:19-30): skips 0/0."""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    sc = np.maximum(np.abs(a), np.abs(b))
    m = sc > 0
    return float((np.abs(a - b)[m] / sc[m]).max()) if m.any() else 0.0


def allclose_ratio(a, b, rtol=1e-2, atol=1e-2):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float((np.abs(a - b) / (atol + rtol * np.abs(b))).max()) if a.size else 0.0


def corrupt(rp, ci, B):
    """selftest.cpp:43-52 on head 0: drop the first key block of the last row
    holding >= 2 blocks (structurally valid, numerically wrong)."""
    rp = rp.copy()
    ci = ci.copy()
    for i in range(B - 1, 0, -1):
        if rp[i + 1] - rp[i] < 2:
            continue
        ci = np.delete(ci, rp[i])
        rp[i + 1:B + 1] -= 1  # per-head row_ptr are 0-based: only head 0 changes
        return rp, ci
    return rp, ci


def run_selftest(seed=42, seq_lens=(16, 64, 128, 256), inject_corruption=False, csv=None):
    import torch

    import oracle
    import paper_2407_17678_b200 as s2
    from paper_2407_17678_b200.pattern import CsrMask

    csv = csv if csv is not None else io.StringIO()
    csv.write("config,seq_len,block_size,head_dim,num_heads,stride,comparison,tolerance,"
              "max_rel_error,status\n")
    dev = torch.device("cuda")
    rep = {"instances": 0, "comparisons": 0, "failures": 0}
    first = True
    for n in seq_lens:
        for S in (8, 16, 64):
            for d in (16, 64):
                for v_code in (1, 3, 4, 0):
                    for heads in ((4, 2) if n <= 64 else (4,)):
                        v = heads if v_code == 0 else v_code
                        B = -(-n // S)
                        local = min(1 + rep["instances"] % 2, B)
                        cfg = s2.make_single_stride_config(n, S, heads, local, v)
                        rp, ci = oracle.csr_all(cfg)
                        g_rp, g_ci = (corrupt(rp, ci, B) if inject_corruption and first else (rp, ci))
                        first = False
                        q, k, vv = oracle.random_tensors(heads, n, d, seed + rep["instances"])
                        ro, rl = oracle.attn_fwd(q, k, vv, rp, ci, 1, heads, heads, n, d, S)
                        # GPU plan from the (possibly corrupted) shard lists
                        csr, off = [], 0
                        for h in range(heads):
                            r = g_rp[h * (B + 1):(h + 1) * (B + 1)]
                            csr.append(CsrMask(h, B, r, g_ci[off: off + int(r[-1])]))
                            off += int(r[-1])
                        plan = s2.Plan.from_csr(csr, n, S)
                        T = lambda x: torch.from_numpy(x).reshape(1, heads, n, d).to(dev)  # noqa: E731
                        tq, tk, tv = T(q), T(k), T(vv)
                        o1, l1 = s2.s2_attn_fwd(plan, tq, tk, tv)
                        o2, l2 = s2.s2_attn_fwd(plan, tq, tk, tv, num_splits=2 if d % 2 == 0 else 1)
                        o3, l3 = s2.s2_attn_fwd(plan, tq, tk, tv, num_splits=1)
                        f = lambda t: t.float().cpu().numpy().ravel()  # noqa: E731
                        # fp32 kernel vs the fp64-accumulating oracle: the north_star's
                        # rtol = atol = 1e-4 (max_relative_error is unbounded near zero)
                        a4 = lambda x, y: allclose_ratio(x, y, 1e-4, 1e-4)  # noqa: E731
                        rows = [("oracle_vs_streaming", 1.0, max(a4(f(o1), ro), a4(f(l1), rl))),
                                ("streaming_vs_dsplit2", 1e-5, max(max_rel(f(o1), f(o2)), max_rel(f(l1), f(l2)))),
                                ("streaming_vs_dsplit1", 1e-6, max(max_rel(f(o1), f(o3)), max_rel(f(l1), f(l3))))]
                        if S % 16 == 0 and d == 64:
                            bf = lambda x: torch.from_numpy(x).reshape(1, heads, n, d).to(dev, torch.bfloat16)  # noqa
                            qb, kb, vb = (bf(x) for x in (q, k, vv))
                            r = lambda t: t.float().cpu().numpy().ravel()  # noqa: E731
                            qr, kr, vr = r(qb), r(kb), r(vb)
                            ob, lb = s2.s2_attn_fwd(plan, qb, kb, vb)
                            rob, rlb = oracle.attn_fwd(qr, kr, vr, rp, ci, 1, heads, heads, n, d, S)
                            rows.append(("oracle_vs_tcgen05", 1.0,
                                         max(allclose_ratio(f(ob), rob), allclose_ratio(f(lb), rlb))))
                            rng = np.random.default_rng(seed + rep["instances"])
                            do = rng.uniform(-1, 1, q.size).astype(np.float32)
                            dob = bf(do)
                            gq, gk, gv = s2.s2_attn_bwd(plan, qb, kb, vb, ob, lb, dob)
                            rq, rk, rv = oracle.attn_bwd(qr, kr, vr, r(dob), rp, ci, 1, heads, heads, n, d, S)
                            rows.append(("oracle_vs_tcgen05_bwd", 1.0,
                                         max(allclose_ratio(f(gq), rq), allclose_ratio(f(gk), rk),
                                             allclose_ratio(f(gv), rv))))
                        h = f"{s2.config_hash(cfg):016x}"
                        for label, tol, err in rows:
                            ok = err <= tol
                            csv.write(f"{h},{n},{S},{d},{heads},{v},{label},{tol:g},{err:.3e},"
                                      f"{'pass' if ok else 'FAIL'}\n")
                            rep["comparisons"] += 1
                            rep["failures"] += 0 if ok else 1
                        rep["instances"] += 1
    rep["ok"] = rep["failures"] == 0
    return rep


def main(argv=None):
    ap = argparse.ArgumentParser(prog="selftest", description=__doc__.split("\n\n")[0])
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--seq-lens", default="16,64,128,256")
    ap.add_argument("--csv", default="-")
    ap.add_argument("--inject-corruption", action="store_true")
    try:
        a = ap.parse_args(argv)
        seq_lens = [int(x) for x in a.seq_lens.split(",") if x]
        if not seq_lens or min(seq_lens) < 1:
            raise ValueError("--seq-lens must list positive integers")
        import torch

        if not torch.cuda.is_available():
            raise RuntimeError("selftest needs a CUDA device")
    except SystemExit as e:
        return 2 if e.code else 0
    except Exception as ex:  # usage / environment: exit 2 (main.cpp:223-226)
        print(f"error: {ex}", file=sys.stderr)
        return 2
    out = sys.stdout if a.csv == "-" else open(a.csv, "w")
    try:
        rep = run_selftest(a.seed, seq_lens, a.inject_corruption, out)
    except Exception as ex:
        print(f"error: {ex}", file=sys.stderr)
        return 2
    finally:
        if out is not sys.stdout:
            out.close()
    print(f"selftest: {rep['instances']} instances, {rep['comparisons']} comparisons, "
          f"{rep['failures']} failures", file=sys.stderr)
    return 0 if rep["ok"] else 1


if __name__ == "__main__":
    sys.exit(main())
