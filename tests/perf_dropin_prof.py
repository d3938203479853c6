"""Ad-hoc probe: cProfile of the drop-in ChainRouter.route at C1 shape (host overhead split)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2509_26182_b200 import ChainRouter, PerfMap, allocate, scenarios as scen
    n, L = int(os.environ.get("PN", "8")), int(os.environ.get("PL", "32"))
    cl, model = scen.synthetic_cluster(n, seed=0, model=scen.bench_model(L))
    plan = allocate(cl, model)
    by = {g.id: g for g in cl.gpus}
    ids = sorted(by)
    pm = PerfMap(ttl_s=4.5, latency_fn=lambda g, l, occ: model.flops_per_layer_per_token / by[g].flops * (1 + occ))
    for g in ids:
        pm.register_gpu(g)
    pm.publish_link_rtts({(a, b): cl.rtt_s(a, b) for i, a in enumerate(ids) for b in ids[i + 1:]}, 0.0)
    for g, sl in plan.gpu_slices().items():
        pm.sync_gpu_layers(g, range(sl.start_layer, sl.end_layer + 1), 0.0)
    router = ChainRouter(pm, L)
    for _ in range(50):
        router.route(0.0)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(1000):
        router.route(0.0)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__":
    main()
