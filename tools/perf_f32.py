"""Quick cfg1 timing (fp32 forward, reference precision; CUDA events). Not the bench."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2407_17678_b200 as s2

for name, (N, H, D, S, v) in {"cfg1": (2048, 8, 64, 64, 8), "cfg1-d128": (2048, 8, 128, 64, 8),
                             "8k-h8-d64": (8192, 8, 64, 64, 16), "blk32-d96": (4096, 4, 96, 32, 8)}.items():
    cfg = s2.make_s2_config(N, H, block_size=S, local_blocks=4, vert_stride=v)
    plan = s2.Plan.from_config(cfg)
    q, k, vv = (torch.rand(1, H, N, D, device="cuda") * 2 - 1 for _ in range(3))
    out, lse = s2.s2_attn_fwd(plan, q, k, vv)
    for _ in range(3):
        s2.s2_attn_fwd(plan, q, k, vv, out=out, lse=lse)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        s2.s2_attn_fwd(plan, q, k, vv, out=out, lse=lse)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    act, _ = plan.fwd_flops(1, D)
    print(f"{name}: {ms:.3f} ms  {act / ms / 1e9:.2f} TFLOP/s")
