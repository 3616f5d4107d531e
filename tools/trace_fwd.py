"""Debug: CTA-0 per-step timeline of the forward kernel (s2_debug_set_trace)."""
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
tr = torch.zeros(24 * 2048, dtype=torch.int64, device="cuda")
L.s2_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
s2.s2_attn_fwd(plan, q, k, v, out=out, lse=lse)
torch.cuda.synchronize()
L.s2_debug_set_trace(None)
t = tr.cpu().numpy().reshape(24, 2048).astype(np.int64)
n = int((t[5] > 0).sum())
m = lambda a: float(np.median(a))  # noqa
lo, hi = 20, min(n, 1500)
print("tile-0 softmax steps traced", n)
print("softmax0: wait S", m(t[5, lo:hi] - t[4, lo:hi]), " step period", m(np.diff(t[5, lo:hi])))
print("softmax0: S ok -> next wait (compute+store+arrive)", m(t[4, lo + 1:hi + 1] - t[5, lo:hi]))
print("softmax1: wait S", m(t[7, lo:hi] - t[6, lo:hi]), " compute", m(t[6, lo + 1:hi + 1] - t[7, lo:hi]))
print("softmax0: S ok -> P arrive", m(t[8, lo:hi] - t[5, lo:hi]), " P arrive -> next wait", m(t[4, lo + 1:hi + 1] - t[8, lo:hi]))
nk = int((t[2] > 0).sum())
if nk > 40:
    a, b = 20, min(nk, 1500)
    print(f"MMA: chunks {nk}: wait K {m(t[1, a:b] - t[0, a:b]):.0f}, S issue {m(t[2, a:b] - t[1, a:b]):.0f}, "
          f"S issued -> next chunk {m(t[0, a + 1:b + 1] - t[2, a:b]):.0f}, chunk period {m(np.diff(t[0, a:b])):.0f}")
    print(f"MMA: wait P tile0 {m(t[12, a:b] - t[3, a:b]):.0f}, wait P tile1 {m(t[14, a:b] - t[13, a:b]):.0f}")
    wk = (t[1, a:b] - t[0, a:b]).astype(np.float64).sum()
    wp = ((t[12, a:b] - t[3, a:b]) + (t[14, a:b] - t[13, a:b])).astype(np.float64).sum()
    span = float(t[0, b] - t[0, a])
    print(f"MMA warp share: wait K {wk / span:.1%}, wait P {wp / span:.1%}")
ni = int((t[11] > 0).sum())
if ni > 3:
    e = slice(1, ni - 1)
    tot = float(t[11, ni - 1] - t[9, 0])
    ep = (t[11, e] - t[10, e]).astype(np.float64)
    wo = (t[10, e] - t[9, e]).astype(np.float64)
    print(f"items {ni}: epilogue median {np.median(ep):.0f} cycles, wait O {np.median(wo):.0f}; "
          f"epilogue+wait share of CTA-0 time {(ep.sum() + wo.sum()) / tot:.1%}")
    busy = (t[8, lo:hi] - t[5, lo:hi]).astype(np.float64).sum()
    waits = (t[5, lo:hi] - t[4, lo:hi]).astype(np.float64).sum()
    span = float(t[8, hi - 1] - t[4, lo])
    print(f"softmax0 over steps {lo}..{hi}: compute {busy / span:.1%}, wait S {waits / span:.1%}, other {1 - (busy + waits) / span:.1%}")
if (t[12] > 0).sum() > 10:  # built with -DS2_FWD_DETAIL_TRACE
    k = np.arange(lo, hi)
    names = ["S ok -> ld done", "mask + local max", "max exchange", "exp + P store", "rescale + st wait + arrive"]
    prev = t[5, k - 1]  # slot 5 uses the pre-increment count
    for i, nm in enumerate(names):
        cur = t[8 + i, k]
        print(f"  {nm}: {np.median(cur - prev):.0f}")
        prev = cur

if (t[16] > 0).sum() > 40:
    print(f"softmax0 gap split: P arrive -> next chunk's loop top {m(t[16, lo + 1:hi + 1] - t[8, lo:hi]):.0f}, "
          f"loop top -> wait {m(t[4, lo + 1:hi + 1] - t[16, lo + 1:hi + 1]):.0f}")

# period distribution of the S issuer's chunk starts (all traced chunks)
nk = int((t[0] > 0).sum())
if nk > 40:
    per = np.diff(t[0, :nk]).astype(np.float64)
    q = np.percentile(per, [10, 50, 75, 90, 99])
    print(f"chunk period: mean {per.mean():.0f}, p10/50/75/90/99 {q.round(0).tolist()}; "
          f"share of time in chunks > 1.5x median {per[per > 1.5 * np.median(per)].sum() / per.sum():.1%}")
    big = per > 1.5 * np.median(per)
    print(f"  chunks > 1.5x median: {big.sum()} of {len(per)}; their mean {per[big].mean():.0f}")
    # where the slow chunks spend their time (S issuer view): chunk k's period is
    # t0[k+1] - t0[k] = wait K(k) + issue S(k) (incl. the S-half waits) + gap to chunk k+1
    idx = np.where(big)[0]
    wk = (t[1] - t[0]).astype(np.float64)
    iss = (t[2] - t[1]).astype(np.float64)
    gap = (np.roll(t[0], -1) - t[2]).astype(np.float64)
    print(f"  slow chunks: wait K {np.median(wk[idx]):.0f}, S issue incl. half waits {np.median(iss[idx]):.0f}, "
          f"gap to next {np.median(gap[idx]):.0f}  (all chunks: {np.median(wk[:nk]):.0f} / {np.median(iss[:nk]):.0f} / "
          f"{np.median(gap[:nk - 1]):.0f})")

# softmax phases of tile 0 (slots 16-18 between S ready (5) and P arrive (8))
if (t[16] > 0).sum() > 40:
    a, b = 20, min(int((t[16] > 0).sum()), 1500)
    ph = {"S ready -> TMEM ld done": t[16, a:b] - t[5, a:b],
          "mask + max + rescale test": t[17, a:b] - t[16, a:b],
          "rescale + exp + P st issue": t[18, a:b] - t[17, a:b],
          "st wait + fence + arrive": t[8, a:b] - t[18, a:b],
          "arrive -> next S wait start": t[4, a + 1:b + 1] - t[8, a:b],
          "wait S": t[5, a + 1:b + 1] - t[4, a + 1:b + 1]}
    for k_, v_ in ph.items():
        print(f"  softmax0 {k_}: median {np.median(v_):.0f}, mean {np.mean(v_):.0f}")
