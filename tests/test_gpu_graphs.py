"""CUDA-graph capture of the path (the brief's "CUDA streams and graphs instead of
a tracing compiler"): after one warm-up call has built and uploaded the plan's
lists and work items, a fwd + bwd step captures into a torch.cuda.CUDAGraph
and replays bit-identically to eager calls -- kernel launches, the dK/dV memset
and the workspace all being stream-ordered."""
import pytest

import paper_2407_17678_b200 as s2
from helpers import single

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", ["s2", "gqa_batch2", "f32_ffma"])
def test_fwd_bwd_step_captures_into_a_cuda_graph(case):
    import torch

    dt, D = torch.bfloat16, 128
    if case == "s2":
        cfg, B, H, Hkv = single(2048, 64, 4, 2, 4), 1, 4, 4
    elif case == "gqa_batch2":
        cfg, B, H, Hkv = single(1024, 64, 8, 2, 4, kv=2), 2, 8, 2
    else:  # the fp32-FFMA forward and backward (CSC uploaded by the warm-up call)
        cfg, B, H, Hkv = single(700, 48, 4, 2, 3, kv=2), 2, 4, 2
        dt, D = torch.float32, 64
    plan = s2.Plan.from_config(cfg)
    N = cfg.seq_len
    g = torch.Generator(device="cuda").manual_seed(11)
    mk = lambda h: (torch.rand(B, h, N, D, device="cuda", generator=g) * 2 - 1).to(dt)  # noqa
    q, k, v, do = mk(H), mk(Hkv), mk(Hkv), mk(H)
    out, lse = torch.empty_like(q), torch.empty(B, H, N, device="cuda")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)

    def step():
        s2.s2_attn_fwd(plan, q, k, v, out=out, lse=lse)
        s2.s2_attn_bwd(plan, q, k, v, out, lse, do, dq=dq, dk=dk, dv=dv)

    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        step()  # warm-up: lists / work items built and uploaded outside the capture
    torch.cuda.synchronize()
    ref = [t.clone() for t in (out, lse, dq, dk, dv)]
    for t in (out, lse, dq, dk, dv):
        t.zero_()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        step()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    for a, b in zip((out, lse, dq, dk, dv), ref):
        assert torch.equal(a, b)
