"""Debug: per-CTA start / end times (globaltimer) of the persistent kernels at
cfg3 -> how much of each launch is tail imbalance.
    idle = sum_c (last end - end_c) / (CTAs x span)"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2407_17678_b200 as s2

N = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
L = s2.lib()
L.s2_debug_set_trace.argtypes = [ctypes.c_void_p]
L.s2_debug_set_mode.argtypes = [ctypes.c_int]
plan = s2.Plan.from_config(s2.make_s2_config(N, 32, local_blocks=4, vert_stride=16))
mk = lambda: (torch.rand(1, 32, N, 128, device="cuda") * 2 - 1).to(torch.bfloat16)  # noqa
q, k, v, do = mk(), mk(), mk(), mk()
out, lse = s2.s2_attn_fwd(plan, q, k, v)
dq, dk, dv = s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
torch.cuda.synchronize()


def report(name, fn):
    tr = torch.zeros(16 * 2048, dtype=torch.int64, device="cuda")
    L.s2_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
    fn()
    torch.cuda.synchronize()
    L.s2_debug_set_trace(None)
    t = tr.cpu().numpy().reshape(16, 2048)[15]
    st, en = t[0::2], t[1::2]
    n = int((en > 0).sum())
    st, en = st[:n].astype(np.float64), en[:n].astype(np.float64)
    span = en.max() - st.min()
    idle_tail = (en.max() - en).sum() / (n * span)
    idle_head = (st - st.min()).sum() / (n * span)
    print(f"{name}: {n} CTAs, span {span / 1e3:.1f} us, tail idle {idle_tail:.1%}, start skew {idle_head:.1%}, "
          f"end spread p50/p90/max behind last: {np.percentile(en.max() - en, 50) / 1e3:.1f}/"
          f"{np.percentile(en.max() - en, 90) / 1e3:.1f}/{(en.max() - en.min()) / 1e3:.1f} us")


report("fwd", lambda: s2.s2_attn_fwd(plan, q, k, v, out=out, lse=lse))
L.s2_debug_set_mode(0)
report("dkv", lambda: s2.s2_attn_bwd(plan, q, k, v, out, lse, do, dq=dq, dk=dk, dv=dv))
L.s2_debug_set_mode(8)  # trace the dQ kernel instead
report("dq", lambda: s2.s2_attn_bwd(plan, q, k, v, out, lse, do, dq=dq, dk=dk, dv=dv))
L.s2_debug_set_mode(0)
