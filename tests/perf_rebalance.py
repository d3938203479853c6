"""Ad-hoc probe of the rebalance loop at C4 scale (not a test): route -> device events -> triggers ->
device rebalance (Phase-1 over every churned pool) -> route.

    python tests/perf_rebalance.py [--scen 1184] [--req 64] [--thr 0.02]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scen", type=int, default=1184)
    ap.add_argument("--req", type=int, default=64)
    ap.add_argument("--thr", type=float, default=0.02)
    ap.add_argument("--joins", type=int, default=4)
    args = ap.parse_args()
    import torch
    from paper_2509_26182_b200 import allocate, scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    rc = scen.default_region_count(256)
    full, model = scen.synthetic_cluster(256 + 16, seed=0, model=scen.bench_model(64), region_count=rc)
    base, _ = scen.synthetic_cluster(256, seed=0, model=scen.bench_model(64), region_count=rc)
    plan = allocate(base, model)
    join_ids = [g.id for g in full.gpus[256:]]
    seeds = np.arange(args.scen)
    kw = dict(seeds=seeds, jitter=True, join_pool=join_ids)
    b = scen.build_scenarios(full, model, plan, args.scen, churn=0.0, **kw)
    e = scen.build_scenarios(full, model, plan, args.scen, churn=0.05, joins=args.joins, host_events=False, **kw)
    rp0 = ScenarioReplayer(b, window=64)
    rp1 = ScenarioReplayer(e, window=64)
    rp0.run(args.req)
    torch.cuda.synchronize()
    t = {}
    t0 = time.perf_counter()
    rp1.build()
    dep = rp1.leave.view(rp1.S, rp1.G).cpu().numpy().astype(bool) & e.present0
    rp0.abort_on(dep)
    rp1.adopt_state(rp0)
    torch.cuda.synchronize()
    t["events_ms"] = 1e3 * (time.perf_counter() - t0)
    t0 = time.perf_counter()
    dec = rp1.triggers(cov_threshold=args.thr)[0]
    torch.cuda.synchronize()
    t["triggers_ms"] = 1e3 * (time.perf_counter() - t0)
    t0 = time.perf_counter()
    rp2, info = rp1.rebalance(cov_threshold=args.thr)
    torch.cuda.synchronize()
    t["rebalance_ms"] = 1e3 * (time.perf_counter() - t0)
    t0 = time.perf_counter()
    rp2.run(args.req)
    torch.cuda.synchronize()
    t["route_ms"] = 1e3 * (time.perf_counter() - t0)
    rp2.raise_first_failure()
    print(json.dumps({"scen": args.scen, "rebalanced": int(info["rebalanced"].sum()),
                      "changed_mean": float(np.mean([len(c) for c in info["changed"]])),
                      "aborted_mean": float(info["aborted"].mean()), "mode_after": rp2.mode, **t}))


if __name__ == "__main__":
    if "--profile" in sys.argv:                      # host-side hot spots of the loop (cProfile)
        import cProfile
        import pstats
        sys.argv.remove("--profile")
        pr = cProfile.Profile()
        pr.enable()
        main()
        pr.disable()
        pstats.Stats(pr).sort_stats("cumulative").print_stats("paper_2509|_phase1|batched|method .to|cpu", 40)
    else:
        main()
