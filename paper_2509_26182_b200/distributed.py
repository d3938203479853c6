"""Multi-GPU host logic: one process per GPU, torch.distributed for plumbing.

* Phase-2 shards scenarios, Phase-1 shards pool variants: item i -> rank i mod world.
  No data-path collective; requests inside one scenario are serially dependent
  (router.py:256, perfmap.py:375-382) and never split.
* The exchanges: the Phase-1 global argmax -- each rank
  contributes (best objective total, variant id); an all-gather (NCCL over
  NVLink on B200, gloo on CPU) lets every rank pick max objective, ties ->
  lowest id -- and the gather of chosen chains: per-rank int16 host[L] +
  fp64 cost per selection collected on one rank in global scenario order
  (gather_chains), or only a wrap-around sum of chain hashes when the full
  chains are not needed (chain_checksum).
"""

from __future__ import annotations

import numpy as np


def shard(n_per_rank: int, rank: int, world: int) -> np.ndarray:
    """Global ids owned by `rank` under weak scaling: rank + world * i."""
    return rank + world * np.arange(n_per_rank, dtype=np.int64)


def global_argmax(best_total, best_id, group=None):
    """All-gather (total, id) pairs and return the global (total, id) on every rank.

    best_total / best_id are 0-d or 1-element tensors on the process group's
    device (cuda for NCCL, cpu for gloo).  best_id < 0 means "no feasible
    candidate on this rank".
    """
    import torch
    import torch.distributed as dist
    mine = torch.stack([best_total.reshape(()).to(torch.float64), best_id.reshape(()).to(torch.float64)])
    world = dist.get_world_size(group)
    out = torch.empty(2 * world, dtype=torch.float64, device=mine.device)
    dist.all_gather_into_tensor(out, mine, group=group)
    pairs = out.view(world, 2).cpu().numpy()
    best_t, best_v = -np.inf, -1
    for t, v in pairs:
        if v < 0:
            continue
        if best_v < 0 or t > best_t or (t == best_t and v < best_v):
            best_t, best_v = float(t), int(v)
    return best_t, best_v


def gather_chains(gpus, cost, dst: int = 0, group=None):
    """Collect every rank's replay outputs on rank ``dst`` in global scenario order.

    gpus [S_rank, R, L] int16 and cost [S_rank, R] float64 on the group's device; every rank owns the same
    number of scenarios (scenario s -> rank s mod world, :func:`shard`).  Returns (gpus [S, R, L],
    cost [S, R]) on ``dst`` (None elsewhere).  An all-gather moves the (small) per-selection records over
    NVLink; NCCL has no gather primitive.
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    S = gpus.shape[0]
    dtype = gpus.dtype
    gpus = gpus.to(torch.int32)                   # NCCL and gloo have no int16 collectives
    g_all = torch.empty((world * S,) + tuple(gpus.shape[1:]), dtype=gpus.dtype, device=gpus.device)
    c_all = torch.empty((world * S,) + tuple(cost.shape[1:]), dtype=cost.dtype, device=cost.device)
    dist.all_gather_into_tensor(g_all, gpus.contiguous(), group=group)
    dist.all_gather_into_tensor(c_all, cost.contiguous(), group=group)
    if rank != dst:
        return None, None
    # rank r's i-th scenario is global scenario r + world * i: interleave
    g_all = g_all.view((world, S) + tuple(gpus.shape[1:]))
    c_all = c_all.view((world, S) + tuple(cost.shape[1:]))
    order = g_all.transpose(0, 1).reshape((S * world,) + tuple(gpus.shape[1:]))
    corder = c_all.transpose(0, 1).reshape((S * world,) + tuple(cost.shape[1:]))
    return order.to(dtype), corder


def chain_checksum(hashes, group=None) -> int:
    """Wrap-around uint64 sum of every selection's chain hash over all ranks (all-reduce)."""
    import torch
    import torch.distributed as dist
    local = hashes.to(torch.int64).sum()          # int64 add wraps like uint64
    t = local.reshape(1).clone()
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item()) & ((1 << 64) - 1)
