"""Ad-hoc probe: latency of the single-request drop-in ChainRouter.route/release at C4 scale (not a test)."""

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2509_26182_b200 import ChainRouter, PerfMap, allocate, scenarios as scen
    for n, L in [(64, 64), (256, 64)]:
        cl, model = scen.synthetic_cluster(n, seed=0, model=scen.bench_model(L))
        plan = allocate(cl, model)
        by = {g.id: g for g in cl.gpus}
        pm = PerfMap(ttl_s=4.5, latency_fn=lambda g, l, occ: model.flops_per_layer_per_token / by[g].flops * (1 + occ))
        ids = sorted(by)
        for g in ids:
            pm.register_gpu(g)
        pm.publish_link_rtts({(a, b): cl.rtt_s(a, b) for i, a in enumerate(ids) for b in ids[i + 1:]}, 0.0)
        for g, sl in plan.gpu_slices().items():
            pm.sync_gpu_layers(g, range(sl.start_layer, sl.end_layer + 1), 0.0)
        router = ChainRouter(pm, L)
        live = []
        for i in range(20):
            live.append(router.route(0.0))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        R = 200
        for i in range(R):
            router.release(live.pop(0), 0.0)
            live.append(router.route(0.0))
        t = time.perf_counter() - t0
        print(f"n={n} L={L} k={plan.replication_count}: {1e3 * t / R:.2f} ms per route+release "
              f"({R / t:.0f} routes/s), matrix rebuilds {router.stats.matrix_rebuilds}")


if __name__ == "__main__":
    main()
