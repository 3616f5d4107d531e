"""Small calls through every CUDA kernel of the product path, for compute-sanitizer
(tools only):

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
    compute-sanitizer --tool synccheck python tools/sanitize_run.py

It covers the bf16 tcgen05 forward and backward (D = 64 / 128, MHA and GQA, a ragged
N, batch 2, a tile with no keys), the fp32 forwards (tiled and row-wise) and the fp32-FFMA backward, the CTA-pair forward when S2_FWD_2CTA=1,
the layout / compaction /
append kernels and the split-KV decode with its combine.  Results are not checked here:
the parity tests do that.  The process exits non-zero if a CUDA call fails.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2407_17678_b200 as s2
from paper_2407_17678_b200.decode import KVCache
from paper_2407_17678_b200.pattern import CsrMask


def rnd(*shape, dt=torch.bfloat16, g=None):
    return (torch.rand(*shape, device="cuda", generator=g) * 2 - 1).to(dt)


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    cases = [  # N, H, Hkv, D, local, v, batch
        (640, 4, 4, 128, 2, 3, 1),
        (1000, 4, 2, 64, 2, 2, 2),
        (200, 2, 2, 128, 1, 2, 1),
    ]
    if os.environ.get("S2_SAN_REVERSE"):  # attribute first-launch reports to a config
        cases.reverse()
    for N, H, Hkv, D, local, v, batch in cases:
        plan = s2.Plan.from_config(s2.make_s2_config(N, H, block_size=64, local_blocks=local, vert_stride=v,
                                                     num_kv_heads=Hkv))
        q, do = rnd(batch, H, N, D, g=g), rnd(batch, H, N, D, g=g)
        k, vv = rnd(batch, Hkv, N, D, g=g), rnd(batch, Hkv, N, D, g=g)
        out, lse = s2.s2_attn_fwd(plan, q, k, vv)
        s2.s2_attn_bwd(plan, q, k, vv, out, lse, do)
        torch.cuda.synchronize()
        print(f"bf16 fwd+bwd N={N} H={H}/{Hkv} D={D} batch={batch}: ok "
              f"(out {out.data_ptr():#x}+{out.nbytes}, dout {do.data_ptr():#x}+{do.nbytes})", flush=True)
    # fp32 paths: the tiled kernel (block 32 and block 128 sub-tiles, D 64 / 17) and the
    # row-wise kernel (D 300)
    for N, S, D in ((300, 32, 64), (333, 128, 17), (200, 16, 300)):
        plan = s2.Plan.from_config(s2.make_s2_config(N, 2, block_size=S, local_blocks=2, vert_stride=2))
        x = [rnd(1, 2, N, D, dt=torch.float32, g=g) for _ in range(3)]
        out, lse = s2.s2_attn_fwd(plan, *x)
        if D <= 128:  # the fp32-FFMA backward (bwd_simt.cu)
            s2.s2_attn_bwd(plan, *x, out, lse, rnd(1, 2, N, D, dt=torch.float32, g=g))
        torch.cuda.synchronize()
        print(f"fp32 fwd{'+bwd' if D <= 128 else ''} N={N} block={S} D={D}: ok", flush=True)
    # the FFMA backward with GQA, batch 2 and bf16 at an untiled head dim
    plan = s2.Plan.from_config(s2.make_s2_config(500, 4, block_size=48, local_blocks=2, vert_stride=3,
                                                 num_kv_heads=2))
    q, do = rnd(2, 4, 500, 96, g=g), rnd(2, 4, 500, 96, g=g)
    k, vv = rnd(2, 2, 500, 96, g=g), rnd(2, 2, 500, 96, g=g)
    out, lse = s2.s2_attn_fwd(plan, q, k, vv)
    s2.s2_attn_bwd(plan, q, k, vv, out, lse, do)
    torch.cuda.synchronize()
    print("bf16 D=96 block 48 GQA batch 2 fwd+bwd (FFMA kernels): ok", flush=True)
    # the opt-in CTA-pair forward (fwd_pair2.cu)
    if os.environ.get("S2_FWD_2CTA") == "1":
        plan = s2.Plan.from_config(s2.make_s2_config(1000, 4, block_size=64, local_blocks=2, vert_stride=3))
        q, k, vv = (rnd(1, 4, 1000, 128, g=g) for _ in range(3))
        s2.s2_attn_fwd(plan, q, k, vv)
        torch.cuda.synchronize()
        print("pair2 fwd: ok", flush=True)
    # a row block without keys and an uncovered key block (zero-filled dK / dV)
    B = 8
    rows = [[0], [0, 1], [], [0, 3], [], [], [0, 6], [6, 7]]
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int32)
    ci = np.concatenate([np.array(r, np.int32) for r in rows]).astype(np.int32)
    plan = s2.Plan.from_csr([CsrMask(h, B, rp, ci) for h in range(2)], 512, 64)
    q, k, vv, do = (rnd(1, 2, 512, 128, g=g) for _ in range(4))
    out, lse = s2.s2_attn_fwd(plan, q, k, vv)
    s2.s2_attn_bwd(plan, q, k, vv, out, lse, do)
    torch.cuda.synchronize()
    print("empty rows / uncovered keys: ok", flush=True)
    # decode: prefill (compaction) + appends + split-KV decode and combine
    cfg = s2.make_s2_config(2048, 8, block_size=64, local_blocks=2, vert_stride=2, num_kv_heads=2)
    plan = s2.Plan.from_config(cfg)
    cache = KVCache(plan, 2, 128)
    T0 = 1500
    k, vv = rnd(2, 2, T0 + 3, 128, g=g), rnd(2, 2, T0 + 3, 128, g=g)
    cache.prefill(k[:, :, :T0].contiguous(), vv[:, :, :T0].contiguous())
    for t in range(T0, T0 + 3):
        cache.append(k[:, :, t].contiguous(), vv[:, :, t].contiguous())
        cache.decode(rnd(2, 8, 128, g=g))
    torch.cuda.synchronize()
    print("decode: ok", flush=True)


if __name__ == "__main__":
    main()
