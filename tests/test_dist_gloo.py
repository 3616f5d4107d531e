"""Head-parallel multi-GPU path on CPU: world_size 2 over gloo.

Exercises the partitioner, unit scatter, the single all-gather and the
unpack of HeadParallelPlan exactly as bench.py / head_parallel_forward use
them, with the oracle standing in for the local kernel (test-only).  The
gathered output must be bit-identical to a single-process run
(head-permutation exactness, test_attention.cpp:217-240).
"""
import os
import socket

import numpy as np
import pytest

from helpers import single


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_local(cfg):
    import torch

    import oracle

    B = cfg.num_blocks()
    rp_all, ci_all = oracle.csr_all(cfg)
    H, Hkv = cfg.num_heads, cfg.kv_heads()
    hpg = H // Hkv
    offs = np.concatenate([[0], np.cumsum([rp_all[h * (B + 1) + B] for h in range(H)])])

    def fn(plan, ql, kl, vl, units):
        U, _, N, D = ql.shape
        outs, lses = [], []
        for i, u in enumerate(units):
            g = int(u) % Hkv
            heads = list(range(g * hpg, (g + 1) * hpg))
            rp = np.concatenate([rp_all[h * (B + 1):(h + 1) * (B + 1)] for h in heads])
            ci = np.concatenate([ci_all[offs[h]:offs[h + 1]] for h in heads])
            o, l = oracle.attn_fwd(ql[i].numpy().ravel(), kl[i].numpy().ravel(),
                                   vl[i].numpy().ravel(), rp, ci, 1, hpg, 1, N, D,
                                   cfg.block_size)
            outs.append(torch.from_numpy(o).reshape(1, hpg, N, D))
            lses.append(torch.from_numpy(l.astype(np.float32)).reshape(1, hpg, N))
        return torch.cat(outs), torch.cat(lses)

    return fn


def _worker(rank, world, port, cfg, batch, D, res_path):
    import torch
    import torch.distributed as dist

    import paper_2407_17678_b200 as s2
    from paper_2407_17678_b200.dist import HeadParallelPlan, head_parallel_forward

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    plan = s2.Plan.from_config(cfg)
    N, H, Hkv = cfg.seq_len, cfg.num_heads, cfg.kv_heads()
    g = torch.Generator().manual_seed(5)
    q = torch.rand((batch, H, N, D), generator=g) * 2 - 1
    k = torch.rand((batch, Hkv, N, D), generator=g) * 2 - 1
    v = torch.rand((batch, Hkv, N, D), generator=g) * 2 - 1
    hp = HeadParallelPlan(plan, batch, world)
    out, lse = head_parallel_forward(plan, q, k, v, rank, world, hp=hp,
                                     local_fn=_oracle_local(cfg))
    # bench.py's overlapped form: start the gather, do unrelated local work (the
    # backward there), finish: the same bytes
    ql = hp.scatter_q(q, rank)
    finish = hp.all_gather_async(ql)
    _ = (ql * 2).sum()  # work between start and finish
    gathered = finish()
    B_, H_, N_, D_ = q.shape
    assert torch.equal(gathered.reshape(B_, H_, N_, D_), q)
    if rank == 0:
        np.savez(res_path, out=out.numpy(), lse=lse.numpy(), q=q.numpy(), k=k.numpy(),
                 v=v.numpy(), load=hp.load, owner=hp.owner)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    (single(512, 64, 4, 2, 3), 2, 16),          # MHA, batch 2
    (single(640, 64, 8, 2, 4, kv=2), 3, 8),     # GQA 4:1, batch 3 (uneven units)
])
def test_head_parallel_world2_gloo_matches_single_process(case, tmp_path):
    import torch.multiprocessing as mp

    import oracle

    cfg, batch, D = case
    res = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(2, _free_port(), cfg, batch, D, res), nprocs=2, join=True)
    r = np.load(res)
    H, Hkv, N = cfg.num_heads, cfg.kv_heads(), cfg.seq_len
    rp, ci = oracle.csr_all(cfg)
    ro, rl = oracle.attn_fwd(r["q"].ravel(), r["k"].ravel(), r["v"].ravel(), rp, ci, batch, H,
                             Hkv, N, D, cfg.block_size)
    np.testing.assert_array_equal(r["out"].ravel(), ro)
    np.testing.assert_array_equal(r["lse"].ravel(), rl.astype(np.float32))
    # both ranks got work and LPT balanced it
    assert set(r["owner"].tolist()) == {0, 1}
    assert r["load"].max() <= r["load"].sum() / 2 * 1.5


def test_cfg5_shaped_split_32_heads_over_8_ranks_gloo(tmp_path):
    """bench.py --workload cfg5's split at world 8: one sequence's 32 heads
    (heterogeneous offsets) LPT-assigned by active blocks, 4 per rank, gathered
    output bit-identical to one process (small N: the oracle computes locally)."""
    import torch.multiprocessing as mp

    import oracle

    cfg, batch, D = single(1024, 64, 32, 4, 16), 1, 8
    res = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(8, _free_port(), cfg, batch, D, res), nprocs=8, join=True)
    r = np.load(res)
    rp, ci = oracle.csr_all(cfg)
    ro, rl = oracle.attn_fwd(r["q"].ravel(), r["k"].ravel(), r["v"].ravel(), rp, ci, batch, 32, 32, 1024, D, 64)
    np.testing.assert_array_equal(r["out"].ravel(), ro)
    np.testing.assert_array_equal(r["lse"].ravel(), rl.astype(np.float32))
    assert sorted(np.bincount(r["owner"], minlength=8).tolist()) == [4] * 8
    assert r["load"].max() / (r["load"].sum() / 8) < 1.05


def test_batch_mode_gives_each_rank_whole_sequences():
    """HeadParallelPlan(mode="batch"), bench.py's cfg3 default (data parallel): with
    world_size dividing the batch, rank r owns exactly the (batch, kv-group) units of
    sequences r*B/W .. (r+1)*B/W - 1, loads are equal (one layout for every sequence),
    and a batch the ranks do not divide falls back to the LPT split."""
    import numpy as np

    import paper_2407_17678_b200 as s2
    from paper_2407_17678_b200.dist import HeadParallelPlan

    plan = s2.Plan.from_config(s2.make_s2_config(4096, 8, local_blocks=2, vert_stride=4, num_kv_heads=4))
    hp = HeadParallelPlan(plan, 4, 2, mode="batch")
    assert [u.tolist() for u in hp.units] == [list(range(0, 8)), list(range(8, 16))]
    assert hp.load[0] == hp.load[1] and hp.imbalance() == 1.0
    lpt = HeadParallelPlan(plan, 4, 2)
    odd = HeadParallelPlan(plan, 3, 2, mode="batch")  # 3 sequences over 2 ranks: LPT
    ref = HeadParallelPlan(plan, 3, 2)
    assert np.array_equal(odd.owner, ref.owner)
    assert sorted(np.concatenate(lpt.units).tolist()) == list(range(16))
