"""Quick forward timing (CUDA events) at a BASELINE config. Not the bench."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2407_17678_b200 as s2

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--h", type=int, default=32)
ap.add_argument("--b", type=int, default=1)
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--v", type=int, default=16)
ap.add_argument("--local", type=int, default=4)
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
cfg = s2.make_s2_config(a.n, a.h, local_blocks=a.local, vert_stride=a.v)
plan = s2.Plan.from_config(cfg)
q = torch.randn(a.b, a.h, a.n, a.d, device="cuda", dtype=torch.bfloat16)
k = torch.randn(a.b, a.h, a.n, a.d, device="cuda", dtype=torch.bfloat16)
v = torch.randn(a.b, a.h, a.n, a.d, device="cuda", dtype=torch.bfloat16)
out, lse = s2.s2_attn_fwd(plan, q, k, v)
for _ in range(3):
    s2.s2_attn_fwd(plan, q, k, v, out=out, lse=lse)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    s2.s2_attn_fwd(plan, q, k, v, out=out, lse=lse)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
act, dense = plan.fwd_flops(a.b, a.d)
st = plan.stats()
print(f"fwd N={a.n} H={a.h} B={a.b} D={a.d}: {ms:.3f} ms  active {act/ms/1e9:.1f} TFLOP/s "
      f"(dense-equiv {dense/ms/1e9:.1f})  chunk-visit eff {st['nnz_total']*1.0/(2*st['fwd_chunk_visits']):.3f}")
