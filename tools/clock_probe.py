"""Effective SM clock inside the forward kernel (tools only): CTA 0's clock64 span
over its globaltimer span, from the debug trace (first/last traced step and the
CTA start/end stamps), for an isolated launch and for launches 50 deep into a
back-to-back loop."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2407_17678_b200 as s2

L = s2.lib()
L.s2_debug_set_trace.argtypes = [ctypes.c_void_p]
plan = s2.Plan.from_config(s2.make_s2_config(32768, 32, local_blocks=4, vert_stride=16))
mk = lambda: (torch.rand(1, 32, 32768, 128, device="cuda") * 2 - 1).to(torch.bfloat16)  # noqa
q, k, v, do = mk(), mk(), mk(), mk()
out, lse = s2.s2_attn_fwd(plan, q, k, v)
dq, dk, dv = s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
tr = torch.zeros(24 * 2048, dtype=torch.int64, device="cuda")


def probe(tag, warm_steps):
    for _ in range(warm_steps):
        s2.s2_attn_fwd(plan, q, k, v, out=out, lse=lse)
        s2.s2_attn_bwd(plan, q, k, v, out, lse, do, dq=dq, dk=dk, dv=dv)
    tr.zero_()
    L.s2_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
    s2.s2_attn_fwd(plan, q, k, v, out=out, lse=lse)
    L.s2_debug_set_trace(None)
    torch.cuda.synchronize()
    t = tr.cpu().numpy().reshape(24, 2048)
    n = int((t[0] > 0).sum())
    clk = float(t[0, n - 1] - t[0, 0])
    ns_start, ns_end = t[15, 0], t[15, 1]
    # the traced steps span most of the CTA's lifetime; compare with the CTA's globaltimer span
    ns = float(ns_end - ns_start)
    print(f"{tag}: CTA0 traced steps {n}, clock64 span {clk:.0f} cyc over the CTA's {ns / 1e3:.1f} us "
          f"-> >= {clk / ns * 1e3:.0f} MHz effective (lower bound: steps span < CTA span)")


probe("isolated (after sync)", 0)
torch.cuda.synchronize()
probe("after 50 back-to-back fwd+bwd steps", 50)
