"""Debug: per-step timeline of cluster 0 of the CTA-pair forward (fwd_pair2.cu)."""
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
q, k, v = mk(), mk(), mk()
out, lse = s2.s2_attn_fwd(plan, q, k, v)
tr = torch.zeros(48 * 2048, dtype=torch.int64, device="cuda")
L.s2_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
s2.s2_attn_fwd(plan, q, k, v, out=out, lse=lse)
torch.cuda.synchronize()
L.s2_debug_set_trace(None)
t = tr.cpu().numpy().reshape(48, 2048).astype(np.int64)
m = lambda a: float(np.median(a))  # noqa
n = int((t[2] > 0).sum())
lo, hi = 10, n - 2
print("steps traced", n)
print(f"S issuer: wait K {m(t[1, lo:hi] - t[0, lo:hi]):.0f}, wait buffer (P V k-3) {m(t[2, lo:hi] - t[1, lo:hi]):.0f}, "
      f"issue -> next {m(t[0, lo + 1:hi + 1] - t[2, lo:hi]):.0f}, period {m(np.diff(t[0, lo:hi])):.0f}")
print(f"PV issuer: wait P {m(t[4, lo:hi] - t[3, lo:hi]):.0f}, issue -> next {m(t[3, lo + 1:hi + 1] - t[11, lo:hi]):.0f}, "
      f"period {m(np.diff(t[3, lo:hi])):.0f}")
ns = int((t[6] > 0).sum())  # softmax rows are indexed per warpgroup step when the warpgroups alternate steps
slo, shi = (lo, hi) if ns > n * 3 // 4 else (5, ns - 2)
for rk, X in ((0, 0), (0, 1), (1, 0), (1, 1)):
    o = 24 * rk + 12 * X
    lo, hi = slo, shi
    print(f"softmax rank {rk} wg {X}: wait S {m(t[o + 6, lo:hi] - t[o + 5, lo:hi]):.0f}, ld+mask+max {m(t[o + 7, lo:hi] - t[o + 6, lo:hi]):.0f}, "
          f"exp+store+arrive {m(t[o + 8, lo:hi] - t[o + 7, lo:hi]):.0f}, arrive -> next wait {m(t[o + 5, lo + 1:hi + 1] - t[o + 8, lo:hi]):.0f}, "
          f"period {m(np.diff(t[o + 6, lo:hi])):.0f}")
lo, hi = 10, n - 2
for rk in (0, 1):
    o = 24 * rk
    print(f"producer rank {rk}: wait stage {m(t[o + 10, lo:hi] - t[o + 9, lo:hi]):.0f}, period {m(np.diff(t[o + 9, lo:hi])):.0f}")
# cross-CTA: P arrive (both ranks) vs PV issuer's wait end
print(f"P ready rank0 -> PV wait end {m(t[4, lo:hi] - t[8, lo:hi]):.0f}, rank1 -> PV wait end {m(t[4, lo:hi] - t[32, lo:hi]):.0f}")
print(f"S issue -> softmax S ready (rank0) {m(t[6, lo:hi] - t[2, lo:hi]):.0f}, (rank1) {m(t[30, lo:hi] - t[2, lo:hi]):.0f}")
print(f"PV issue -> S issue of k+3 {m(t[2, lo + 3:hi + 3] - t[11, lo:hi]):.0f}")
print(f"wg0 detail: S ready -> ld done {m(t[21, lo:hi] - t[6, lo:hi]):.0f}, mask+max+shfl {m(t[22, lo:hi] - t[21, lo:hi]):.0f}, "
      f"rescale check+arrive {m(t[7, lo:hi] - t[22, lo:hi]):.0f}")
