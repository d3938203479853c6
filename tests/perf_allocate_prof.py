"""Ad-hoc probe: where a single allocate() call spends its time (cProfile + per-kernel device times)."""

import cProfile
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2509_26182_b200 import allocate, scenarios as scen
    n = int(os.environ.get("PN", "256")); L = int(os.environ.get("PL", "64"))
    cl, model = scen.synthetic_cluster(n, seed=0, model=scen.bench_model(L))
    allocate(cl, model)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(200):
        allocate(cl, model)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(40)


if __name__ == "__main__":
    main()
