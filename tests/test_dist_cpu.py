"""World-size-2 gloo tests of the multi-GPU host logic (CPU, no GPU needed)."""

import os
import socket

import numpy as np
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, results):
    import torch.distributed as dist
    from paper_2509_26182_b200.distributed import global_argmax, shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ids = shard(5, rank, world)
        # per-variant totals known to every rank: pick the best inside the shard, then gather
        totals = {0: 1.5, 1: 2.0, 2: 0.5, 3: 2.0, 4: 1.0, 5: 1.9, 6: 0.1, 7: 1.2, 8: 2.0, 9: 0.3}
        mine = max(ids, key=lambda v: (totals[int(v)], -int(v)))
        t, v = global_argmax(torch.tensor(totals[int(mine)]), torch.tensor(float(mine)))
        # a rank with nothing feasible contributes id -1 and never wins
        t2, v2 = global_argmax(torch.tensor(9.0 if rank == 0 else 0.0),
                               torch.tensor(-1.0 if rank == 0 else float(rank)))
        results[rank] = (ids.tolist(), t, v, t2, v2)
    finally:
        dist.destroy_process_group()


def test_shard_and_global_argmax_gloo_world2():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.start_processes(_worker, args=(world, port, results), nprocs=world, join=True, start_method="fork")
    ids0, t, v, t2, v2 = results[0]
    ids1 = results[1][0]
    assert ids0 == [0, 2, 4, 6, 8] and ids1 == [1, 3, 5, 7, 9]
    assert sorted(ids0 + ids1) == list(range(10))
    # 2.0 appears at variants 1, 3 and 8: ties go to the lowest id on every rank
    assert (t, v) == (2.0, 1) and results[1][1:3] == (2.0, 1)
    assert (t2, v2) == (0.0, 1)


def _gather_worker(rank, world, port, results):
    import torch.distributed as dist
    from paper_2509_26182_b200.distributed import chain_checksum, gather_chains, shard
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ids = shard(3, rank, world)                     # global scenarios owned by this rank
        gpus = torch.tensor([[[int(s) * 10 + r, int(s)] for r in range(2)] for s in ids], dtype=torch.int16)
        cost = torch.tensor([[float(s) + 0.25 * r for r in range(2)] for s in ids], dtype=torch.float64)
        g, c = gather_chains(gpus, cost, dst=0)
        hashes = torch.tensor([int(s) for s in ids] + [-1], dtype=torch.int64)
        results[rank] = (None if g is None else g.tolist(), None if c is None else c.tolist(), chain_checksum(hashes))
    finally:
        dist.destroy_process_group()


def test_gather_chains_gloo_world2():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    results = mgr.dict()
    mp.start_processes(_gather_worker, args=(world, port, results), nprocs=world, join=True, start_method="fork")
    g, c, ck = results[0]
    assert results[1][0] is None
    assert [row[0][1] for row in g] == list(range(6))          # global scenario order 0..5
    assert g[3] == [[30, 3], [31, 3]] and c[4] == [4.0, 4.25]
    assert ck == results[1][2] == (sum(range(6)) - 2) & ((1 << 64) - 1)
