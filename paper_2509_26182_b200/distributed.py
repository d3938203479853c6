"""Multi-GPU host logic: one process per GPU, torch.distributed for plumbing.

* Phase-2 shards scenarios, Phase-1 shards pool variants: item i -> rank i mod world.
  No data-path collective; requests inside one scenario are serially dependent
  (router.py:256, perfmap.py:375-382) and never split.
* The one real exchange is the Phase-1 global argmax: each rank contributes
  (best objective total, variant id); an all-gather (NCCL over NVLink on
  B200, gloo on CPU) lets every rank pick max objective, ties -> lowest id.
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
