"""Debug: CTA-0 per-step timeline of the 128-key-step dQ kernel (s2_bwd_dq2_kernel)."""
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
s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
L.s2_debug_set_mode.argtypes = [ctypes.c_int]
L.s2_debug_set_mode(8 | (int(sys.argv[1]) if len(sys.argv) > 1 else 0))
tr = torch.zeros(16 * 2048, dtype=torch.int64, device="cuda")
L.s2_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
torch.cuda.synchronize()
L.s2_debug_set_trace(None)
L.s2_debug_set_mode(0)
t = tr.cpu().numpy().reshape(16, 2048).astype(np.float64)
n = int((t[2] > 0).sum())
sl = slice(4, n - 2)
med = lambda x: float(np.median(x[sl]))  # noqa
print(f"dq2 CTA0: {n} steps, median period {np.median(np.diff(t[2, :n])):.0f} cyc, total {t[2, n-1] - t[2, 0]:.0f}")
print(f"  MMA: wait K/V {med(t[8]-t[0]):.0f}  wait S-read {med(t[1]-t[8]):.0f}  S..dP issue (incl dQ prev) {med(t[2]-t[1]):.0f}")
nd = n - 1
print(f"  MMA: wait dS {float(np.median(t[4, 4:nd-2]-t[3, 4:nd-2])):.0f}")
print(f"  EW : wait S {med(t[6]-t[5]):.0f}  S-ready -> dS arrive {med(t[7]-t[6]):.0f}")
print(f"  S issue(t1) -> EW sees S {med(t[6]-t[1]):.0f};  EW dS arrive -> MMA sees dS {float(np.median(t[4, 4:nd-2]-t[7, 4:nd-2])):.0f}")
for i in range(8, 14):
    print(i, {k: int(t[j, i] - t[0, 8]) for k, j in (("w_kv", 0), ("kv_ok", 8), ("s_ok", 1), ("dp_iss", 2), ("w_ds", 3), ("ds_ok", 4), ("ew_ws", 5), ("ew_s", 6), ("ew_ds", 7))})
