"""Debug: CTA-0 per-step timeline of the 128-row-step dK/dV kernel (s2_bwd_dkv2_kernel)."""
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
L.s2_debug_set_mode(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
tr = torch.zeros(16 * 2048, dtype=torch.int64, device="cuda")
L.s2_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
torch.cuda.synchronize()
L.s2_debug_set_trace(None)
L.s2_debug_set_mode(0)
t = tr.cpu().numpy().reshape(16, 2048).astype(np.float64)
n = int((t[3] > 0).sum())
sl = slice(4, n - 2)
med = lambda x: float(np.median(x[sl]))  # noqa
per = np.diff(t[3, :n])
print(f"dkv2 CTA0: {n} steps, median period {np.median(per):.0f} cyc, mean {per.mean():.0f}, total {t[3, n-1] - t[3, 0]:.0f}")
print(f"  MMA: wait S-read {med(t[1]-t[0]):.0f}  issue S (incl Q/K wait) -> wait P {med(t[2]-t[1]):.0f} (incl pds wait)  dV,dK,dP issue {med(t[3]-t[2]):.0f}")
print(f"  EW : wait S {med(t[6]-t[5]):.0f}  S-ready -> P/dS arrive {med(t[7]-t[6]):.0f}")
print(f"  EW arrive -> MMA past pds {med(t[2]-t[7]):.0f}")
big = per > 2 * np.median(per)
print(f"  steps > 2x median: {big.sum()} carrying {per[big].sum() / per.sum():.1%} of the time")
for i in range(8, 14):
    print(i, {k: int(t[j, i] - t[0, 8]) for k, j in (("w_sfr", 0), ("iss_s", 1), ("pds_ok", 2), ("dp_done", 3), ("ew_ws", 5), ("ew_s", 6), ("ew_pds", 7))})
print(f"  EW detail: S read {med(t[9]-t[6]):.0f}  exp {med(t[10]-t[9]):.0f}  wait dP {med(t[11]-t[10]):.0f}  dP read {med(t[12]-t[11]):.0f}  dS+store {med(t[7]-t[12]):.0f}")
print(f"  MMA: S^T(n+1) issued at +{med(t[1]-t[0]):.0f}; pds(n) seen {med(t[2]-t[7]):.0f} after the EW arrive")
print(f"  issuer: Q/K wait {med(t[4]-t[0]):.0f}  S^T issue {med(t[1]-t[4]):.0f}  pds wait {med(t[2]-t[1]):.0f}  dV issue {med(t[8]-t[2]):.0f}  "
      f"sfr wait {med(t[13]-t[8]):.0f}  dP issue {med(t[14]-t[13]):.0f}  dK issue {med(t[3]-t[14]):.0f}")
