"""Multi-rank path with the real kernels on a one-GPU box.

Two processes share cuda:0 and talk over gloo (NCCL refuses two ranks on one
device; the driver's 8-GPU runs use NCCL). This covers with the sm_100a kernels
what tests/test_dist_gloo.py covers with the oracle:
  * head_parallel_forward's gathered O / lse are bit-identical to one process
    (head-permutation exactness, test_attention.cpp:217-240), and each rank's
    backward on its own units equals the single-process gradients of those units;
  * s2_attn_fwd_peers (the forward storing O into every rank's full output,
    peer memory mapped with CUDA IPC) leaves the whole O / lse on every rank,
    bit-identical to one process;
  * bench.py launched by torchrun at world size 2 prints one valid JSON line
    with either exchange (n_gpus 2, weak scaling, positive throughput) -- a
    code-path check, not a performance number (both ranks time-slice one GPU).
"""
import json
import os
import socket
import subprocess
import sys

import pytest

from helpers import single

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, batch, D, res_path, f32=False):
    import torch
    import torch.distributed as dist

    import paper_2407_17678_b200 as s2
    from paper_2407_17678_b200.dist import HeadParallelPlan, head_parallel_forward

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = s2.Plan.from_config(cfg)
    N, H, Hkv = cfg.seq_len, cfg.num_heads, cfg.kv_heads()
    g = torch.Generator(device="cuda").manual_seed(7)
    dt = torch.float32 if f32 else torch.bfloat16
    mk = lambda h: (torch.rand((batch, h, N, D), device="cuda", generator=g) * 2 - 1).to(dt)  # noqa
    q, k, v, do = mk(H), mk(Hkv), mk(Hkv), mk(H)
    hp = HeadParallelPlan(plan, batch, world)
    out, lse = head_parallel_forward(plan, q, k, v, rank, world, hp=hp)
    # this rank's backward on its own units (the gradients stay sharded)
    units = hp.units[rank]
    grads = None
    if len(units):
        ql, kl, vl, dol = hp.scatter_q(q, rank), hp.scatter_kv(k, rank), hp.scatter_kv(v, rank), hp.scatter_q(do, rank)
        ol, ll = s2.s2_attn_fwd(plan, ql, kl, vl, unit_ids=units)
        grads = s2.s2_attn_bwd(plan, ql, kl, vl, ol, ll, dol, unit_ids=units)
    torch.cuda.synchronize()
    if rank == 0:
        ref_out, ref_lse = s2.s2_attn_fwd(plan, q, k, v)
        rq, rk, rv = s2.s2_attn_bwd(plan, q, k, v, ref_out, ref_lse, do)
        ok = torch.equal(out, ref_out) and torch.equal(lse, ref_lse)
        if grads is not None:
            qu = torch.as_tensor(units, device="cuda")
            ok = ok and torch.equal(grads[0], rq.reshape(batch * Hkv, -1, N, D)[qu])
            ok = ok and torch.equal(grads[1], rk.reshape(batch * Hkv, N, D)[qu])
            ok = ok and torch.equal(grads[2], rv.reshape(batch * Hkv, N, D)[qu])
        with open(res_path, "w") as f:
            f.write("ok" if ok else "MISMATCH")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["mha_b2", "gqa", "f32_gqa_b2"])
def test_head_parallel_world2_on_one_gpu_is_bit_identical(case, tmp_path):
    import torch.multiprocessing as mp

    f32 = False
    if case == "mha_b2":
        cfg, batch, D = single(1024, 64, 4, 2, 4), 2, 128
    elif case == "gqa":
        cfg, batch, D = single(2048, 64, 8, 4, 4, kv=2), 1, 128
    else:  # the fp32-FFMA forward and backward on each rank's units
        cfg, batch, D, f32 = single(640, 32, 8, 3, 3, kv=4), 2, 64, True
    res = str(tmp_path / "res.txt")
    mp.spawn(_worker, args=(2, _free_port(), cfg, batch, D, res, f32), nprocs=2, join=True)
    assert open(res).read() == "ok"


@pytest.mark.parametrize("exchange", ["none", "allgather", "fused"])
def test_bench_world2_prints_one_valid_line(exchange):
    env = dict(os.environ, S2_BENCH_SHARE_GPU="1", S2_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu-baseline", "--no-decode",
           "--no-hybrid", "--exchange", exchange]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0 and d["steps"] == 3
    assert d["config"]["global_batch"] == 2
    assert ("fused" in d["config"]["parallelism"]) == (exchange == "fused")
    assert d["exchange"]["mode"] == exchange
    if exchange == "none":  # cfg3's default: one sequence per rank, nothing gathered
        assert "data-parallel" in d["config"]["parallelism"]
        assert d["exchange"]["all_gather_bytes_total"] == 0 and d["exchange"]["imbalance_max_over_ideal"] == 1.0


def test_bench_cfg5_strong_world2_prints_one_valid_line():
    """--workload cfg5: the 128K layer's 32 heads split over 2 ranks (strong scaling),
    with the exchange budget in the line."""
    env = dict(os.environ, S2_BENCH_SHARE_GPU="1", S2_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--workload", "cfg5", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-3000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["seq_len"] == 131072 and d["config"]["global_batch"] == 1
    ex = d["exchange"]
    assert len(ex["rank_active_blocks"]) == 2 and ex["imbalance_max_over_ideal"] < 1.01
    assert ex["all_gather_bytes_total"] == 32 * 131072 * 128 * 2


def _fused_worker(rank, world, port, cfg, batch, D, res_dir):
    import torch
    import torch.distributed as dist

    import paper_2407_17678_b200 as s2
    from paper_2407_17678_b200.dist import HeadParallelPlan, PeerOutputs

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = s2.Plan.from_config(cfg)
    N, H, Hkv = cfg.seq_len, cfg.num_heads, cfg.kv_heads()
    g = torch.Generator(device="cuda").manual_seed(9)
    mk = lambda h: (torch.rand((batch, h, N, D), device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)  # noqa
    q, k, v = mk(H), mk(Hkv), mk(Hkv)
    hp = HeadParallelPlan(plan, batch, world)
    peers = PeerOutputs(hp, N, D, torch.bfloat16, torch.device("cuda", 0), rank)
    peers.out.fill_(float("nan"))
    peers.lse.fill_(float("nan"))
    dist.barrier()
    ql, kl, vl = hp.scatter_q(q, rank), hp.scatter_kv(k, rank), hp.scatter_kv(v, rank)
    out_l, lse_l = hp.fused_forward(plan, ql, kl, vl, rank, peers)
    ref_out, ref_lse = s2.s2_attn_fwd(plan, q, k, v)
    ref_l, ref_ll = s2.s2_attn_fwd(plan, ql, kl, vl, unit_ids=hp.units[rank])
    torch.cuda.synchronize()
    ok = (torch.equal(peers.out.reshape(batch, H, N, D), ref_out)
          and torch.equal(peers.lse.reshape(batch, H, N), ref_lse)
          and torch.equal(out_l, ref_l) and torch.equal(lse_l, ref_ll))
    with open(os.path.join(res_dir, f"r{rank}.txt"), "w") as f:
        f.write("ok" if ok else "MISMATCH")
    dist.barrier()
    del peers
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["mha_b2", "gqa"])
def test_fused_forward_exchange_world2_on_one_gpu(case, tmp_path):
    """s2_attn_fwd_peers: each rank's forward stores its O tiles straight into both
    ranks' full outputs (peer memory mapped with CUDA IPC); afterwards every rank
    holds the whole O / lse, bit-identical to one process."""
    import torch.multiprocessing as mp

    if case == "mha_b2":
        cfg, batch, D = single(1024, 64, 4, 2, 4), 2, 128
    else:
        cfg, batch, D = single(2048, 64, 8, 4, 4, kv=2), 1, 128
    mp.spawn(_fused_worker, args=(2, _free_port(), cfg, batch, D, str(tmp_path)), nprocs=2, join=True)
    assert open(tmp_path / "r0.txt").read() == "ok"
    assert open(tmp_path / "r1.txt").read() == "ok"
