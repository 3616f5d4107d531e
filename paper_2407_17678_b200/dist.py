"""Head-parallel multi-GPU execution (north_star subsystem 5).

Units are (batch, kv-group) pairs — a GQA group's query heads share one K/V
head and one mask, so they stay on one GPU.  Each unit's weight is its
active-block count (CSR nnz, identical for the CSC, so it balances backward
too).  ``partition_lpt`` (C++, s2_partition_lpt) assigns units longest-first
to the least-loaded rank.  Every rank runs the sparse kernels on its own
units only (no data-path collective); the single exchange is an all-gather
of the packed per-rank outputs (NCCL over NVLink via torch.distributed),
padded to the largest rank and unpacked by the unit map.

The reference has no multi-device path (OpenMP only, attention.cpp:114-117);
its head-permutation exactness (test_attention.cpp:217-240) is what makes the
gathered output bit-identical to the single-GPU output.
"""
from __future__ import annotations

import ctypes
from typing import List, Optional, Tuple

import numpy as np

from ._abi import check, lib


def partition_lpt(weights, num_ranks: int) -> Tuple[np.ndarray, np.ndarray]:
    """(owner[num_units], load[num_ranks]) — LPT, deterministic."""
    w = np.ascontiguousarray(weights, dtype=np.int64)
    owner = np.zeros(w.size, np.int32)
    load = np.zeros(num_ranks, np.int64)
    check(lib().s2_partition_lpt(int(w.size), w.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                 num_ranks, owner.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                 load.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
    return owner, load


class HeadParallelPlan:
    """Which (batch, kv-group) units each rank owns, and how to scatter / gather."""

    def __init__(self, plan, batch: int, world_size: int, mode: str = "lpt"):
        """mode "lpt": units (batch, kv-group) longest-first to the least-loaded rank
        (one sequence's heads spread over the ranks: the output exchange assembles
        it).  mode "batch": whole sequences per rank when world_size divides batch
        (data parallelism: every rank owns complete outputs, nothing to exchange;
        the loads are equal because every sequence has the same layout)."""
        self.plan = plan
        self.batch = batch
        self.world_size = world_size
        self.hpg = plan.num_heads // plan.num_kv_heads
        self.weights = plan.unit_weights(batch)
        if mode == "batch" and batch % world_size == 0:
            per = batch // world_size * plan.num_kv_heads
            self.owner = (np.arange(batch * plan.num_kv_heads) // per).astype(np.int32)
            self.load = np.array([self.weights[self.owner == r].sum() for r in range(world_size)], np.int64)
        elif mode in ("lpt", "batch"):
            self.owner, self.load = partition_lpt(self.weights, world_size)
        else:
            raise ValueError(f"unknown mode {mode!r}")
        self.units: List[np.ndarray] = [np.nonzero(self.owner == r)[0].astype(np.int32)
                                        for r in range(world_size)]
        self.max_units = max(1, max(len(u) for u in self.units))

    def imbalance(self) -> float:
        ideal = self.weights.sum() / self.world_size
        return float(self.load.max() / ideal) if ideal else 1.0

    # ---- data movement (torch tensors) --------------------------------
    def scatter_q(self, q, rank: int):
        """q [B,H,N,D] -> packed [U_r, hpg, N, D] for this rank's units."""
        B, H, N, D = q.shape
        Hkv = H // self.hpg
        qu = q.reshape(B * Hkv, self.hpg, N, D)
        return qu[self._index(rank, q.device)].contiguous()

    def scatter_kv(self, k, rank: int):
        """k [B,Hkv,N,D] -> packed [U_r, N, D]."""
        B, Hkv, N, D = k.shape
        return k.reshape(B * Hkv, N, D)[self._index(rank, k.device)].contiguous()

    def _index(self, rank, device):
        import torch

        return torch.as_tensor(self.units[rank], device=device, dtype=torch.long)

    def fused_forward(self, plan, ql, kl, vl, rank: int, peers: "PeerOutputs", *, scale=None, group=None,
                      sync: bool = True):
        """This rank's units through s2_attn_fwd_peers: the forward writes O / lse
        into every rank's full buffers (peers).  Returns the local (out, lse) and
        leaves the full result in peers.out / peers.lse once every rank's kernel
        is done (sync=True orders that with a device synchronize + barrier)."""
        import torch
        import torch.distributed as dist

        from .attention import s2_attn_fwd_peers

        units = self.units[rank]
        ug = torch.as_tensor(np.asarray(units, dtype=np.int32), device=ql.device)
        out, lse = s2_attn_fwd_peers(plan, ql, kl, vl, unit_ids=units, peer_out=peers.peer_out,
                                     peer_lse=peers.peer_lse, unit_global=ug,
                                     total_units=peers.total_units, scale=scale)
        if sync:
            torch.cuda.synchronize()
            dist.barrier(group=group)
        return out, lse

    def all_gather(self, local, group=None):
        """local [U_r, ...] on every rank -> full [B*Hkv, ...] in unit order.

        One all_gather of equal-sized (max-unit padded) buffers; no other
        collective on the data path."""
        return self.all_gather_async(local, group)()

    def all_gather_async(self, local, group=None):
        """Start the all-gather and return finish() -> full tensor.

        The collective runs on the communication stream of the process group
        (NCCL's own stream), so work issued between start and finish — the
        backward, which needs only this rank's output and lse — overlaps the
        NVLink transfer.  finish() makes the current stream wait and unpacks.
        Pair with s2_set_sm_reserve so the persistent kernels leave NCCL's CTAs
        their SMs."""
        import torch
        import torch.distributed as dist

        U = local.shape[0]
        pad = torch.zeros((self.max_units,) + tuple(local.shape[1:]), dtype=local.dtype,
                          device=local.device)
        pad[:U] = local
        bufs = [torch.empty_like(pad) for _ in range(self.world_size)]
        work = dist.all_gather(bufs, pad, group=group, async_op=True)

        def finish():
            work.wait()
            full = torch.empty((self.batch * self.plan.num_kv_heads,) + tuple(local.shape[1:]),
                               dtype=local.dtype, device=local.device)
            for r in range(self.world_size):
                n = len(self.units[r])
                if n:
                    full[self._index(r, local.device)] = bufs[r][:n]
            return full

        return finish


class PeerOutputs:
    """Every rank's full output buffers, mapped into this process: the targets of
    the fused forward + exchange (s2_attn_fwd_peers).

    Each rank allocates out [total_units, hpg, N, D] and lse [total_units, hpg, N]
    and shares them with CUDA IPC handles (torch's cross-process CUDA tensor
    reduction, exchanged with one object all-gather at setup).  On an NVLink /
    NVSwitch node the mapped peer buffers are P2P memory, so the forward's
    epilogue stores O straight into every rank's output -- no separate
    collective on the data path."""

    def __init__(self, hp: "HeadParallelPlan", seq_len: int, head_dim: int, dtype, device, rank: int,
                 group=None):
        import torch
        import torch.distributed as dist
        from torch.multiprocessing.reductions import reduce_tensor

        total = hp.batch * hp.plan.num_kv_heads
        self.total_units = total
        self.rank = rank
        self.out = torch.empty((total, hp.hpg, seq_len, head_dim), dtype=dtype, device=device)
        self.lse = torch.empty((total, hp.hpg, seq_len), dtype=torch.float32, device=device)
        mine = (reduce_tensor(self.out), reduce_tensor(self.lse))
        handles = [None] * hp.world_size
        dist.all_gather_object(handles, mine, group=group)
        self.peer_out, self.peer_lse = [], []
        for r, (ho, hl) in enumerate(handles):
            if r == rank:
                self.peer_out.append(self.out)
                self.peer_lse.append(self.lse)
            else:
                self.peer_out.append(ho[0](*ho[1]))
                self.peer_lse.append(hl[0](*hl[1]))


def head_parallel_forward(plan, q, k, v, rank: int, world_size: int, *, group=None,
                          scale: Optional[float] = None, hp: Optional[HeadParallelPlan] = None,
                          local_fn=None):
    """Shard units over ranks, run the local sparse forward, all-gather O and lse.

    q [B,H,N,D], k/v [B,Hkv,N,D] are the full tensors (each rank reads only its
    units).  Returns full (out [B,H,N,D], lse [B,H,N]).  local_fn(plan, q_units,
    k_units, v_units, unit_ids) -> (out_units, lse_units) defaults to the sm_100a
    kernel (s2_attn_fwd)."""
    from .attention import s2_attn_fwd

    B, H, N, D = q.shape
    hp = hp or HeadParallelPlan(plan, B, world_size)
    units = hp.units[rank]
    if len(units):
        ql = hp.scatter_q(q, rank)
        kl = hp.scatter_kv(k, rank)
        vl = hp.scatter_kv(v, rank)
        if local_fn is None:
            out_l, lse_l = s2_attn_fwd(plan, ql, kl, vl, scale=scale, unit_ids=units)
        else:
            out_l, lse_l = local_fn(plan, ql, kl, vl, units)
    else:
        import torch

        out_l = torch.zeros((0, hp.hpg, N, D), dtype=q.dtype, device=q.device)
        lse_l = torch.zeros((0, hp.hpg, N), dtype=torch.float32, device=q.device)
    out = hp.all_gather(out_l, group).reshape(B, H, N, D)
    lse = hp.all_gather(lse_l, group).reshape(B, H, N)
    return out, lse
