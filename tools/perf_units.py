"""Same-process A/B: fwd+bwd through the full-layout call vs the unit_ids call (tools only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2407_17678_b200 as s2

N, H, D = 32768, 32, 128
plan = s2.Plan.from_config(s2.make_s2_config(N, H, local_blocks=4, vert_stride=16))
mk = lambda *s: (torch.rand(*s, device="cuda") * 2 - 1).to(torch.bfloat16)  # noqa
q, do = mk(1, H, N, D), mk(1, H, N, D)
k, v = mk(1, H, N, D), mk(1, H, N, D)
out, lse = s2.s2_attn_fwd(plan, q, k, v)
dq, dk, dv = s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
units = np.arange(H, dtype=np.int32)
qu, dou = q.reshape(H, 1, N, D), do.reshape(H, 1, N, D)
ku, vu = k.reshape(H, N, D), v.reshape(H, N, D)
ou, lu = out.reshape(H, 1, N, D), lse.reshape(H, 1, N)
dqu, dku, dvu = dq.reshape(H, 1, N, D), dk.reshape(H, N, D), dv.reshape(H, N, D)


def full():
    s2.s2_attn_fwd(plan, q, k, v, out=out, lse=lse)
    s2.s2_attn_bwd(plan, q, k, v, out, lse, do, dq=dq, dk=dk, dv=dv)


def unit():
    s2.s2_attn_fwd(plan, qu, ku, vu, out=ou, lse=lu, unit_ids=units)
    s2.s2_attn_bwd(plan, qu, ku, vu, ou, lu, dou, dq=dqu, dk=dku, dv=dvu, unit_ids=units)


for name, f in (("full", full), ("unit", unit), ("full", full), ("unit", unit)):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(30):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / 30:.3f} ms/step")
