"""Debug: CTA-0 per-step timeline of the dK/dV kernel, or of the dQ kernel with
`dq` as the second argument (s2_debug_set_trace; the other kernel runs untraced)."""
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
tr = torch.zeros(16 * 2048, dtype=torch.int64, device="cuda")
L.s2_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
s2.s2_attn_bwd(plan, q, k, v, out, lse, do)
torch.cuda.synchronize()
L.s2_debug_set_trace(None)
t = tr.cpu().numpy().reshape(16, 2048)
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
dd = np.diff(t[2, 1:n]).astype(np.float64)
print(f"mean cycles/step {dd.mean():.0f}  (median {np.median(dd):.0f}); steps > 2x median: {(dd > 2 * np.median(dd)).sum()} "
      f"carrying {dd[dd > 2 * np.median(dd)].sum() / dd.sum():.1%} of the time")
long = np.where(dd > 2 * np.median(dd))[0] + 1  # index of the step whose S commit came late
ws = (t[1] - t[0]).astype(np.float64)
wp = (t[4] - t[3]).astype(np.float64)
iss = (t[2] - t[1]).astype(np.float64)
print("long steps: median wait_sf", np.median(ws[long]), " issue S", np.median(iss[long]),
      " wait_p(prev)", np.median(wp[long - 1]), " gap", np.median(dd[long - 1]))
ni = int((t[10] != -t0).sum())
if ni > 2:
    e = t[:, 1:ni - 1].astype(np.float64)
    print(f"items traced {ni}: EW wait af {np.median(e[9] - e[8]):.0f}, epilogue {np.median(e[10] - e[9]):.0f}; "
          f"MMA wait ae {np.median(e[12] - e[11]):.0f}")

ni2 = int((t[14] != -t0).sum())
if ni2 > 3:
    e = t[:, 1:ni2 - 1].astype(np.float64)
    print(f"dq items traced {ni2}: MMA wait for the next item's Q/dO (bar_qf) median {np.median(e[14] - e[13]):.0f} cycles")
    # where the dQ kernel's time goes: steady steps vs item boundaries
    sc = t[2, :n].astype(np.float64)
    starts = t[14, 1:ni2].astype(np.float64)  # issuer has the next item's Q/dO
    first = np.searchsorted(sc, starts)       # index of the first S commit of each item
    first = first[(first > 0) & (first < n)]
    st = np.diff(sc)
    med = np.median(st)
    bd = sc[first] - sc[first - 1]
    print(f"dq: {n} steps, median step {med:.0f} cyc, total {sc[-1] - sc[0]:.0f}; "
          f"{len(first)} item boundaries: median gap {np.median(bd):.0f} cyc, "
          f"boundary excess {np.sum(bd - med) / (sc[-1] - sc[0]):.1%} of the time; "
          f"non-boundary steps > 1.5x median carry {np.sum(st[st > 1.5 * med]) / st.sum():.1%}")
    print("EW compute median", np.median(t[7, :n] - t[6, :n]), " EW wait S median", np.median(t[6, :n] - t[5, :n]),
          " MMA wait P median", np.median(t[4, :n - 1] - t[3, :n - 1]))
