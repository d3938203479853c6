"""Ad-hoc C2 probe (one scenario, long request stream, on-device load update): latency-bound path.

    python tests/perf_c2.py [--req 20000] [--mode warp|slots|blocks] [--scenarios 1]
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--req", type=int, default=20000)
    ap.add_argument("--mode", default="slots")
    ap.add_argument("--window", type=int, default=64)
    ap.add_argument("--scenarios", type=int, default=1)
    args = ap.parse_args()
    import torch
    from paper_2509_26182_b200 import allocate, scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    cl, model = scen.synthetic_cluster(64, seed=0, model=scen.bench_model(64))
    plan = allocate(cl, model)
    ss = scen.build_scenarios(cl, model, plan, args.scenarios, churn=0.0, jitter=args.scenarios > 1)
    rp = ScenarioReplayer(ss, window=args.window, mode=args.mode)
    rp.run(64)
    torch.cuda.synchronize()
    rp.reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = rp.run(args.req)
    e1.record()
    torch.cuda.synchronize()
    rp.raise_first_failure()
    t = e0.elapsed_time(e1) / 1e3
    print(json.dumps({"mode": rp.mode, "k": plan.replication_count, "req": args.req, "time_s": t,
                      "scenarios": args.scenarios, "sel_per_s": args.scenarios * args.req / t,
                      "us_per_sel": 1e6 * t / args.req, "route": os.environ.get("SS_WARP_ROUTE", "default")}))


if __name__ == "__main__":
    main()
