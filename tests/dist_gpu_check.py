"""Multi-GPU exchanges on real GPUs, one process per GPU over NCCL / NVLink:

    torchrun --standalone --local-addr 127.0.0.1 --nproc-per-node N tests/dist_gpu_check.py

* Phase-1: the bench's C3 variants sharded v -> rank v mod world; each rank's best (objective total, variant)
  goes through ``ss_argmax_allgather`` (and torch's all-gather, ``global_argmax``); rank 0 re-runs the whole
  sweep alone and must find the same winner.
* Phase-2: C4 churn + jitter scenarios sharded s -> rank s mod world, replayed on device (2 launches of R
  requests, W = 64, so releases run); the second launch's full chains (int16 host[L] + fp64 cost per
  selection) go to rank 0 through ``ss_gather_chains`` (grouped ncclSend / ncclRecv) and through
  ``gather_chains``; rank 0 replays every global scenario on its own GPU (the N = 1 run) and must get the
  identical chains, and two scenarios are checked against the oracle.
Rank 0 prints one JSON line; the exit code is non-zero on any mismatch.
"""

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch
    import torch.distributed as dist
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    from paper_2509_26182_b200 import allocate, scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer, VariantSweep
    from paper_2509_26182_b200.distributed import NcclExchange, gather_chains, global_argmax, shard
    stream = torch.cuda.current_stream()
    ex = NcclExchange(stream=stream)
    ok = True
    report = {"world": world}

    # ---- Phase-1 global argmax -------------------------------------------------
    V = 16 * world
    mine = shard(V // world, rank, world)
    packs = [scen.bench_variants(1, 256, 80, seed0=int(v))[0] for v in mine]

    def sweep_best(pack_list, ids):
        best_t, best_v = -np.inf, -1
        for pk, v in zip(pack_list, ids):
            sw = VariantSweep(pk, fill_all=True)
            sw.run()
            t = float(sw.total.cpu()[0])
            if t > best_t or (t == best_t and v < best_v):
                best_t, best_v = t, int(v)
        return best_t, best_v

    bt, bv = sweep_best(packs, mine)
    t_dev, v_dev = ex.argmax(torch.tensor([bt], dtype=torch.float64, device="cuda"),
                             torch.tensor([bv], dtype=torch.int64, device="cuda"))
    got_abi = (float(t_dev.cpu()[0]), int(v_dev.cpu()[0]))
    got_torch = global_argmax(torch.tensor(bt, dtype=torch.float64, device="cuda"),
                              torch.tensor(float(bv), dtype=torch.float64, device="cuda"))
    if rank == 0:
        all_ids = np.arange(V)
        want = sweep_best([scen.bench_variants(1, 256, 80, seed0=int(v))[0] for v in all_ids], all_ids)
        report["argmax"] = {"variants": V, "winner": got_abi[1], "objective": got_abi[0].hex(),
                            "single_gpu": [want[0].hex(), int(want[1])], "torch": [float(got_torch[0]).hex(),
                                                                                  int(got_torch[1])],
                            "abi_matches_single_gpu": got_abi == want, "torch_matches_single_gpu": got_torch == want}
        ok &= got_abi == want and got_torch == want

    # ---- Phase-2 chain gather ----------------------------------------------------
    S, R, W = 8, 64, 64
    cl, model = scen.synthetic_cluster(256, seed=0, model=scen.bench_model(64))
    plan = allocate(cl, model)
    seeds = shard(S, rank, world)
    ss = scen.build_scenarios(cl, model, plan, S, churn=0.05, jitter=True, seeds=seeds, host_events=False)
    rp = ScenarioReplayer(ss, window=W, mode="slots", max_requests=2 * R)
    rp.run(R)
    out = rp.run(R, gpus=True)
    rp.raise_first_failure()
    torch.cuda.synchronize()
    g_abi, c_abi = ex.gather_chains(out.gpus, out.cost, dst=0)
    g_t, c_t = gather_chains(out.gpus, out.cost, dst=0)
    torch.cuda.synchronize()
    if rank == 0:
        all_seeds = np.arange(S * world, dtype=np.int64)
        ss1 = scen.build_scenarios(cl, model, plan, len(all_seeds), churn=0.05, jitter=True, seeds=all_seeds,
                                   host_events=False)
        rp1 = ScenarioReplayer(ss1, window=W, mode="slots", max_requests=2 * R)
        rp1.run(R)
        o1 = rp1.run(R, gpus=True)
        rp1.raise_first_failure()
        want_g, want_c = o1.gpus.cpu().numpy(), o1.cost.cpu().numpy()
        same_abi = np.array_equal(g_abi.cpu().numpy(), want_g) and np.array_equal(c_abi.cpu().numpy(), want_c)
        same_t = np.array_equal(g_t.cpu().numpy(), want_g) and np.array_equal(c_t.cpu().numpy(), want_c)
        from oracle import chain_ref
        host = scen.build_scenarios(cl, model, plan, 2, churn=0.05, jitter=True, seeds=all_seeds[[1, S * world - 1]])
        oracle_ok = True
        for j, s in enumerate((1, S * world - 1)):
            wg, wc, _, _ = chain_ref.replay(host.columns(j), host.base_tau, host.scenario_rtt(j), 2 * R, W,
                                            chain_ref.occ_power_table(W + 2))
            oracle_ok &= g_abi.cpu().numpy()[s].tolist() == wg[R:] and c_abi.cpu().numpy()[s].tolist() == wc[R:]
        report["chain_gather"] = {"scenarios": int(S * world), "selections": int(S * world * R),
                                  "bytes": int(S * world * R * (2 * model.layer_count + 8)),
                                  "abi_matches_single_gpu": bool(same_abi), "torch_matches_single_gpu": bool(same_t),
                                  "oracle_sampled_match": bool(oracle_ok)}
        ok &= same_abi and same_t and oracle_ok
        report["ok"] = bool(ok)
        print(json.dumps(report), flush=True)
    ex.close()
    flag = torch.tensor([0 if ok else 1], device="cuda")
    dist.all_reduce(flag)
    dist.destroy_process_group()
    sys.exit(int(flag.item() != 0))


if __name__ == "__main__":
    main()
