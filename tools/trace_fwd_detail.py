import ctypes, os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2407_17678_b200 as s2
L = s2.lib(); L.s2_debug_set_trace.argtypes = [ctypes.c_void_p]
plan = s2.Plan.from_config(s2.make_s2_config(32768, 32, local_blocks=4, vert_stride=16))
mk = lambda: torch.randn(1, 32, 32768, 128, device="cuda", dtype=torch.bfloat16)
q, k, v = mk(), mk(), mk()
out, lse = s2.s2_attn_fwd(plan, q, k, v)
tr = torch.zeros(8 * 2048, dtype=torch.int64, device="cuda")
L.s2_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
s2.s2_attn_fwd(plan, q, k, v, out=out, lse=lse)
torch.cuda.synchronize(); L.s2_debug_set_trace(None)
t = tr.cpu().numpy().reshape(8, 2048).astype(np.int64)
n = int((t[0] > 0).sum()); lo, hi = 20, n - 2
m = lambda a: float(np.median(a))
names = ["S ok", "ld wait", "mask+max", "rescale", "exp+st issue", "st wait+arrive"]
for i in range(1, 6): print(names[i], m(t[i, lo:hi] - t[i - 1, lo:hi]))
print("arrive -> next wait", m(t[6, lo + 1:hi + 1] - t[5, lo:hi]), " wait S", m(t[0, lo:hi] - t[6, lo:hi]))
