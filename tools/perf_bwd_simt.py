"""Time the fp32-FFMA backward (csrc/kernels/bwd_simt.cu) at BASELINE cfg1's shape
(fp32, H=8, S=2048, D=64, block 64, local 4, vert_stride 8) with CUDA events."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2407_17678_b200 as s2  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2048)
ap.add_argument("--h", type=int, default=8)
ap.add_argument("--d", type=int, default=64)
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
cfg = s2.make_s2_config(a.n, a.h, block_size=64, local_blocks=4, vert_stride=8)
plan = s2.Plan.from_config(cfg)
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda: torch.rand((1, a.h, a.n, a.d), device="cuda", generator=g) * 2 - 1  # noqa: E731
q, k, v, do = mk(), mk(), mk(), mk()
out, lse = s2.s2_attn_fwd(plan, q, k, v)
for _ in range(3):
    s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    s2.s2_attn_fwd(plan, q, k, v)
e1.record()
torch.cuda.synchronize()
fwd = e0.elapsed_time(e1) / a.iters
e0.record()
for _ in range(a.iters):
    s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
e1.record()
torch.cuda.synchronize()
bwd = e0.elapsed_time(e1) / a.iters
f = s2.exact_flops(cfg, a.d).sparse_flops  # forward, block granularity
print(f"fp32 N={a.n} H={a.h} D={a.d}: fwd {fwd:.3f} ms ({f / fwd / 1e9:.1f} TF/s)  "
      f"bwd {bwd:.3f} ms ({2.5 * f / bwd / 1e9:.1f} TF/s at 2.5x the forward's flops)")
