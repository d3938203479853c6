"""Ad-hoc probe: per-call allocate() wall times at N=256 / L=64 (parallel vs serial group-count search)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2509_26182_b200 import _native as N, allocate, scenarios as scen
    cl, model = scen.synthetic_cluster(256, seed=0, model=scen.bench_model(64))
    lib = N.lib()
    for limit in (2048, 0):
        lib.ss_set_cover_parallel_limit(limit)
        allocate(cl, model)
        torch.cuda.synchronize()
        ts = []
        for _ in range(30):
            t0 = time.perf_counter()
            allocate(cl, model)
            ts.append(round(1e3 * (time.perf_counter() - t0), 1))
        print(f"parallel limit {limit}: wall ms sorted {sorted(ts)}")


if __name__ == "__main__":
    main()
