"""Decode step timing at cfg4 (B=64, 128K context, 32q/8kv, v=8). Not the bench."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2407_17678_b200 as s2
from paper_2407_17678_b200.decode import KVCache

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=131072)
ap.add_argument("--b", type=int, default=64)
ap.add_argument("--h", type=int, default=32)
ap.add_argument("--hkv", type=int, default=8)
ap.add_argument("--v", type=int, default=8)
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
D = 128
plan = s2.Plan.from_config(s2.make_s2_config(a.n, a.h, num_kv_heads=a.hkv, local_blocks=4, vert_stride=a.v))
cache = KVCache(plan, a.b, D)
T = a.n
for b0 in range(0, a.b, 8):  # prefill in batch slices would need per-slice API; fill all at once
    pass
k = torch.randn(a.b, a.hkv, T, D, device="cuda", dtype=torch.bfloat16)
cache.prefill(k, k)
del k
torch.cuda.empty_cache()
q = torch.randn(a.b, a.h, D, device="cuda", dtype=torch.bfloat16)
out, lse = cache.decode(q)
for _ in range(3):
    cache.decode(q, out=out, lse=lse)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    cache.decode(q, out=out, lse=lse)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
by = cache.decode_bytes()
pool, dense = cache.bytes()
print(f"decode B={a.b} ctx={T} {a.h}q/{a.hkv}kv: {ms*1000:.1f} us/step  {a.b/ms*1000:.0f} tok/s  "
      f"{by/ms/1e6:.0f} GB/s  bytes/step {by/1e9:.3f} GB  pool {pool/1e9:.2f} GB vs dense {dense/1e9:.2f} GB")
