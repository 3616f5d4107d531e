"""Debug: forward time through the head-parallel unit list (bench.py's call) vs
the plain [1, H, N, D] call on the same data."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2407_17678_b200 as s2
from paper_2407_17678_b200.dist import HeadParallelPlan

N, H, D = 32768, 32, 128
plan = s2.Plan.from_config(s2.make_s2_config(N, H, block_size=64, local_blocks=4, vert_stride=16))
hp = HeadParallelPlan(plan, 1, 1)
units = hp.units[0]
print("units order", units[:8], "...")
U = len(units)
base = [(torch.rand(U, N, D, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(3)]


def run(tag, **kw):
    if "unit_ids" in kw:
        q, k, v = base[0].reshape(U, 1, N, D), base[1], base[2]
        out = torch.empty_like(q)
        lse = torch.empty(U, 1, N, device="cuda")
    else:
        q, k, v = (t.reshape(1, U, N, D) for t in base)
        out = torch.empty_like(q)
        lse = torch.empty(1, U, N, device="cuda")
    for _ in range(3):
        s2.s2_attn_fwd(plan, q, k, v, out=out, lse=lse, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        s2.s2_attn_fwd(plan, q, k, v, out=out, lse=lse, **kw)
    e1.record()
    torch.cuda.synchronize()
    print(tag, f"{e0.elapsed_time(e1) / 20:.3f} ms")


run("hp units", unit_ids=units)
run("iota units", unit_ids=list(range(U)))
run("plain [1,H,N,D]")
run("hp units again", unit_ids=units)
