"""Stress: repeated fwd+bwd must be bit-identical run to run (tools only).

A race in the mbarrier / TMEM pipelines shows up as an occasional wrong value or a
hang.  This runs the cfg3 layer (32K, H=32, D=128) and a set of seeded random
configurations many times, and compares every output with the first run, bit for bit:

    python tools/stress_determinism.py [cfg3_reps] [small_reps]
"""
import os
import random
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2407_17678_b200 as s2


def run(plan, q, k, v, do):
    out, lse = s2.s2_attn_fwd(plan, q, k, v)
    dq, dk, dv = s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
    return [out, lse, dq, dk, dv]


def check(name, plan, q, k, v, do, reps):
    ref = [t.clone() for t in run(plan, q, k, v, do)]
    bad = 0
    for _ in range(reps):
        got = run(plan, q, k, v, do)
        if not all(torch.equal(a, b) for a, b in zip(got, ref)):
            bad += 1
    torch.cuda.synchronize()
    print(f"{name}: {reps} repeats, {bad} mismatching", flush=True)
    return bad


def main():
    cfg3_reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    small_reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    g = torch.Generator(device="cuda").manual_seed(0)
    mk = lambda *sh: (torch.rand(*sh, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)  # noqa: E731
    bad = 0
    plan = s2.Plan.from_config(s2.make_s2_config(32768, 32, local_blocks=4, vert_stride=16))
    bad += check("cfg3", plan, mk(1, 32, 32768, 128), mk(1, 32, 32768, 128), mk(1, 32, 32768, 128),
                 mk(1, 32, 32768, 128), cfg3_reps)
    rng = random.Random(5)
    for i in range(24):
        N = rng.randint(100, 6000)
        H = rng.choice([2, 4, 8])
        Hkv = rng.choice([h for h in (1, 2, 4, 8) if H % h == 0])
        D = rng.choice([64, 128])
        B = rng.choice([1, 2])
        cfg = s2.make_s2_config(N, H, block_size=64, local_blocks=rng.randint(1, 4),
                                vert_stride=rng.randint(1, 8), num_kv_heads=Hkv)
        plan = s2.Plan.from_config(cfg)
        bad += check(f"rand{i} N={N} H={H}/{Hkv} D={D} B={B}", plan, mk(B, H, N, D), mk(B, Hkv, N, D),
                     mk(B, Hkv, N, D), mk(B, H, N, D), small_reps)
    print("TOTAL mismatching runs:", bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
