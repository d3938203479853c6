"""Ad-hoc probe: latency of the single-call allocate() drop-in (not a test)."""

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2509_26182_b200 import allocate, scenarios as scen
    for n, L in [(4, 48), (8, 48), (16, 48), (32, 48), (64, 48), (128, 48), (256, 48), (8, 32), (64, 64), (256, 64),
                 (256, 80)]:
        cl, model = scen.synthetic_cluster(n, seed=0, model=scen.bench_model(L))
        allocate(cl, model)
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            t0 = time.perf_counter()
            plan = allocate(cl, model)
            ts.append(time.perf_counter() - t0)
        ts.sort()
        print(f"n={n} L={L}: allocate min {1e3 * ts[0]:.1f} / median {1e3 * ts[10]:.1f} / max {1e3 * ts[-1]:.1f} ms "
              f"(k={plan.replication_count})")


if __name__ == "__main__":
    main()
