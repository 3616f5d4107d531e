"""Dense-causal cfg3-shaped layer (S=32K, H=32, D=128, bf16, block 64) through this
repo's kernels: forward, backward kernels and fwd+bwd, CUDA events (tools only).
The kernel choice follows the environment (S2_FWD_2CTA, ...), so variants A/B."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2407_17678_b200 as s2

N, H, D = int(os.environ.get("N", 32768)), 32, 128
B = N // 64
flops_f = 4 * D * 64 * 64 * (B * (B + 1) / 2) * H  # dense-causal block pairs, whole diagonal blocks
plan = s2.Plan.from_config(s2.make_dense_config(N, 64, H))
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda: (torch.rand(1, H, N, D, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)  # noqa
q, k, v, do = mk(), mk(), mk(), mk()
out, lse = s2.s2_attn_fwd(plan, q, k, v)
dq, dk, dv = s2.s2_attn_bwd(plan, q, k, v, out, lse, do)


def timeit(f, it=5):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


fw = timeit(lambda: s2.s2_attn_fwd(plan, q, k, v, out=out, lse=lse))
bw = timeit(lambda: s2.s2_attn_bwd(plan, q, k, v, out, lse, do, dq=dq, dk=dk, dv=dv))
print(f"dense N={N}: fwd {fw:.2f} ms = {flops_f / fw / 1e9:.0f} TF/s; bwd {bw:.2f} ms = "
      f"{2.5 * flops_f / bw / 1e9:.0f} TF/s; fwd+bwd {fw + bw:.2f} ms = {3.5 * flops_f / (fw + bw) / 1e9:.0f} TF/s")

import ctypes  # noqa: E402

lib = s2.lib()
lib.s2_profile_enable(1)
for _ in range(3):
    s2.s2_attn_bwd(plan, q, k, v, out, lse, do, dq=dq, dk=dk, dv=dv)
torch.cuda.synchronize()
names = ctypes.create_string_buffer(32 * 16)
tot = (ctypes.c_double * 16)()
cnt = (ctypes.c_int * 16)()
nk = ctypes.c_int()
lib.s2_profile_collect(16, names, tot, cnt, ctypes.byref(nk))
lib.s2_profile_enable(0)
print("  kernels: " + ", ".join(f"{names.raw[32 * i: 32 * i + 32].split(bytes(1))[0].decode()} "
                                f"{tot[i] / cnt[i]:.2f} ms" for i in range(nk.value)))
