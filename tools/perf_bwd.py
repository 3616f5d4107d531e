"""Quick fwd+bwd timing (CUDA events) at a BASELINE config. Not the bench."""
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
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--uniform", action="store_true", help="U[-1,1] inputs (bench.py's data) instead of N(0,1)")
a = ap.parse_args()
plan = s2.Plan.from_config(s2.make_s2_config(a.n, a.h, local_blocks=a.local, vert_stride=a.v))
if a.uniform:
    mk = lambda: (torch.rand(a.b, a.h, a.n, a.d, device="cuda") * 2 - 1).to(torch.bfloat16)  # noqa
else:
    mk = lambda: torch.randn(a.b, a.h, a.n, a.d, device="cuda", dtype=torch.bfloat16)  # noqa
q, k, v, do = mk(), mk(), mk(), mk()
out, lse = s2.s2_attn_fwd(plan, q, k, v)
dq, dk, dv = s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for _ in range(3):
    s2.s2_attn_fwd(plan, q, k, v, out=out, lse=lse)
    s2.s2_attn_bwd(plan, q, k, v, out, lse, do, dq=dq, dk=dk, dv=dv)
torch.cuda.synchronize()
import ctypes
L = s2.lib()
L.s2_debug_set_mode.argtypes = [ctypes.c_int]
L.s2_debug_set_mode(int(os.environ.get("S2_DEBUG", "0")))  # kernel ablations (results invalid when != 0)
L.s2_profile_enable(1)
tf = tb = 0.0
for _ in range(a.iters):
    ev[0].record()
    s2.s2_attn_fwd(plan, q, k, v, out=out, lse=lse)
    ev[1].record()
    s2.s2_attn_bwd(plan, q, k, v, out, lse, do, dq=dq, dk=dk, dv=dv)
    ev[2].record()
    torch.cuda.synchronize()
    tf += ev[0].elapsed_time(ev[1])
    tb += ev[1].elapsed_time(ev[2])
tf /= a.iters
tb /= a.iters
act, dense = plan.fwd_flops(a.b, a.d)
print(f"N={a.n} H={a.h} B={a.b}: fwd {tf:.3f} ms ({act/tf/1e9:.0f} TF/s)  bwd {tb:.3f} ms "
      f"({2.5*act/tb/1e9:.0f} TF/s)  fwd+bwd {tf+tb:.3f} ms ({3.5*act/(tf+tb)/1e9:.0f} TF/s active, "
      f"{3.5*dense/(tf+tb)/1e9:.0f} dense-equiv)")
names = ctypes.create_string_buffer(32 * 16)
tot = (ctypes.c_double * 16)()
cnt = (ctypes.c_int * 16)()
nk = ctypes.c_int()
L.s2_profile_collect(16, names, tot, cnt, ctypes.byref(nk))
L.s2_profile_enable(0)
print("  kernels: " + ", ".join(
    f"{names.raw[32*i:32*i+32].split(bytes(1))[0].decode()} {tot[i]/cnt[i]:.3f} ms" for i in range(nk.value)))
