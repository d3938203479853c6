"""Multi-GPU host logic: one process per GPU, torch.distributed for plumbing.

* Phase-2 shards scenarios, Phase-1 shards pool variants: item i -> rank i mod world.
  No data-path collective; requests inside one scenario are serially dependent
  (router.py:256, perfmap.py:375-382) and never split.
* On GPUs the two exchanges run through the C ABI of libswarmsched_b200_nccl.so (:class:`NcclExchange`:
  ``ss_argmax_allgather`` = ncclAllGather of 16-byte records + a pick kernel, ``ss_gather_chains`` = grouped
  ncclSend / ncclRecv to the root); torch.distributed only broadcasts the 128-byte NCCL unique id.  The
  functions below are the same exchanges over any torch process group (gloo on CPU tests).
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


class NcclExchange:
    """The path's two multi-GPU exchanges through ``libswarmsched_b200_nccl.so`` (include/swarmsched_b200_nccl.h).

    One NCCL communicator over the ranks of a torch process group (which only carries the 128-byte unique id);
    every call is ordered on the given CUDA stream.  No fallback: the library must load and CUDA must be up.
    """

    def __init__(self, group=None, stream=None):
        import ctypes as C
        import torch
        import torch.distributed as dist
        from . import _native as N
        self.lib = N.nccl_lib()
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.stream = stream
        uid = (C.c_uint8 * 128)()
        if self.rank == 0:
            N.check(self.lib.ss_nccl_unique_id(uid), "ss_nccl_unique_id")
        box = [bytes(uid) if self.rank == 0 else None]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        uid = (C.c_uint8 * 128).from_buffer_copy(box[0])
        self._comm = C.c_void_p()
        N.check(self.lib.ss_nccl_comm_init(uid, self.world, self.rank, C.byref(self._comm)), "ss_nccl_comm_init")
        dev = torch.device("cuda", torch.cuda.current_device())
        self._scratch = torch.empty(2 * self.world, dtype=torch.float64, device=dev)
        self._best = torch.empty(1, dtype=torch.float64, device=dev)
        self._best_id = torch.empty(1, dtype=torch.int64, device=dev)

    def _sh(self):
        from . import _native as N
        return N.stream_handle(self.stream)

    def argmax(self, best_total, best_id):
        """Global (objective, id): max objective, ties -> lowest id, id < 0 = nothing feasible on that rank."""
        import torch
        from . import _native as N
        t = best_total.reshape(1).to(torch.float64).contiguous()
        v = best_id.reshape(1).to(torch.int64).contiguous()
        N.check(self.lib.ss_argmax_allgather(self._comm, N.ptr(t), N.ptr(v), N.ptr(self._best), N.ptr(self._best_id),
                                             N.ptr(self._scratch), self._sh()), "ss_argmax_allgather")
        return self._best, self._best_id

    def gather_chains(self, gpus, cost, dst: int = 0):
        """Every rank's gpus [S, R, L] int16 / cost [S, R] fp64 on ``dst`` in global scenario order
        (scenario s on rank s mod world); (None, None) elsewhere."""
        import torch
        from . import _native as N
        S = gpus.shape[0]
        rest = tuple(gpus.shape[1:])
        L = int(gpus.shape[-1])
        n_sel = int(gpus.numel() // L)
        g = gpus.contiguous()
        c = cost.contiguous()
        go = co = None
        if self.rank == dst:
            go = torch.empty((self.world * S,) + rest, dtype=torch.int16, device=g.device)
            co = torch.empty((self.world * S,) + tuple(cost.shape[1:]), dtype=torch.float64, device=g.device)
        N.check(self.lib.ss_gather_chains(self._comm, N.ptr(g), N.ptr(c), n_sel, L, dst,
                                          N.ptr(go) if go is not None else None,
                                          N.ptr(co) if co is not None else None, self._sh()), "ss_gather_chains")
        if self.rank != dst:
            return None, None
        go = go.view((self.world, S) + rest).transpose(0, 1).reshape((self.world * S,) + rest)
        co = co.view((self.world, S) + tuple(cost.shape[1:])).transpose(0, 1).reshape(
            (self.world * S,) + tuple(cost.shape[1:]))
        return go, co

    def close(self):
        if self._comm:
            self.lib.ss_nccl_comm_destroy(self._comm)
            self._comm = None
