"""Debug: CTA-0 per-step timeline of the dK/dV kernel (s2_debug_set_trace)."""
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
mk = lambda: torch.randn(1, 32, 32768, 128, device="cuda", dtype=torch.bfloat16)  # noqa
q, k, v, do = mk(), mk(), mk(), mk()
out, lse = s2.s2_attn_fwd(plan, q, k, v)
s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
L.s2_debug_set_mode.argtypes = [ctypes.c_int]
L.s2_debug_set_mode(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
tr = torch.zeros(8 * 2048, dtype=torch.int64, device="cuda")
L.s2_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
torch.cuda.synchronize()
L.s2_debug_set_trace(None)
t = tr.cpu().numpy().reshape(8, 2048)
n = int((t[2] > 0).sum())
t0 = t[0, 0]
t = t - t0
names = ["mma_wait_sf", "mma_sf_ok", "mma_S_commit", "mma_wait_p(n)", "mma_p_ok(n)", "ew_wait_s", "ew_s_ok", "ew_arrive_p"]
print("steps traced", n)
for i in list(range(0, 12)) + list(range(200, 212)):
    print(i, " ".join(f"{names[s]}={t[s, i]}" for s in range(8)))
d = np.diff(t[2, 10:n])
print("median issue S/dP (sf_ok -> S commit):", np.median(t[2, 10:n] - t[1, 10:n]))
print("median dV/dK issue (p_ok -> next wait_sf):", np.median(t[0, 11:n] - t[4, 10:n - 1]))
print("median cycles/step (S commit to S commit):", np.median(d))
print("median EW compute (s_ok -> arrive):", np.median(t[7, 10:n] - t[6, 10:n]))
print("median EW wait for S:", np.median(t[6, 10:n] - t[5, 10:n]))
print("median MMA wait p:", np.median(t[4, 10:n - 1] - t[3, 10:n - 1]))
print("median MMA wait stage:", np.median(t[1, 10:n] - t[0, 10:n]))
print("median S issue->EW sees S:", np.median(t[6, 10:n] - t[2, 10:n]))
print("median EW arrive->MMA sees P:", np.median(t[4, 10:n - 1] - t[7, 10:n - 1]))
