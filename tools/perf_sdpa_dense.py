"""Context number (tools only): a dense-causal cfg3-shaped layer (S=32K, H=32, D=128,
bf16) fwd+bwd through torch's scaled_dot_product_attention (library backends: cuDNN /
flash), against this repo's dense layer through the S2 kernels (LayerStack path)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.nn.functional as F

import paper_2407_17678_b200 as s2

N, H, D = 32768, 32, 128
mk = lambda: (torch.rand(1, H, N, D, device="cuda") * 2 - 1).to(torch.bfloat16).requires_grad_()  # noqa
q, k, v = mk(), mk(), mk()
do = (torch.rand(1, H, N, D, device="cuda") * 2 - 1).to(torch.bfloat16)
flops = 3.5 * 4 * D * 64 * 64 * (512 * 513 / 2) * H  # dense-causal block pairs, whole diagonal blocks


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


from torch.nn.attention import SDPBackend, sdpa_kernel

for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION),
                 ("efficient", SDPBackend.EFFICIENT_ATTENTION)):
    try:
        def f():
            with sdpa_kernel([be]):
                o = F.scaled_dot_product_attention(q, k, v, is_causal=True)
            o.backward(do)
        ms = timeit(f)
        print(f"torch SDPA {name}: {ms:.2f} ms fwd+bwd = {flops / ms / 1e9:.0f} TFLOP/s (dense-causal count)")
    except Exception as ex:
        print(f"torch SDPA {name}: unavailable ({str(ex).splitlines()[0][:120]})")

plan = s2.Plan.from_config(s2.make_dense_config(N, 64, H))
qd, kd, vd, dod = (x.detach() for x in (q, k, v, do))
out, lse = s2.s2_attn_fwd(plan, qd, kd, vd)
dq, dk, dv = s2.s2_attn_bwd(plan, qd, kd, vd, out, lse, dod)


def g():
    s2.s2_attn_fwd(plan, qd, kd, vd, out=out, lse=lse)
    s2.s2_attn_bwd(plan, qd, kd, vd, out, lse, dod, dq=dq, dk=dk, dv=dv)


ms = timeit(g)
print(f"this repo (S2 kernels, dense-causal plan): {ms:.2f} ms fwd+bwd = {flops / ms / 1e9:.0f} TFLOP/s")

# forward only
with torch.no_grad():
    def ff():
        with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
            F.scaled_dot_product_attention(q, k, v, is_causal=True)
    try:
        ms = timeit(ff)
        print(f"torch SDPA cudnn forward only: {ms:.2f} ms = {flops / 3.5 / ms / 1e9:.0f} TFLOP/s")
    except Exception as ex:
        print("cudnn fwd-only unavailable", ex)
    ms = timeit(lambda: s2.s2_attn_fwd(plan, qd, kd, vd, out=out, lse=lse))
    print(f"this repo forward only: {ms:.2f} ms = {flops / 3.5 / ms / 1e9:.0f} TFLOP/s")
