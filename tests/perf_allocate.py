"""Ad-hoc probe: latency of the single-call allocate() drop-in (not a test)."""

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2509_26182_b200 import allocate, scenarios as scen
    for n, L in [(64, 64), (256, 64), (256, 80)]:
        cl, model = scen.synthetic_cluster(n, seed=0, model=scen.bench_model(L))
        allocate(cl, model)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            plan = allocate(cl, model)
        t = (time.perf_counter() - t0) / 5
        print(f"n={n} L={L}: allocate {1e3 * t:.1f} ms (k={plan.replication_count})")


if __name__ == "__main__":
    main()
