"""Ad-hoc GPU throughput probe for the replay kernel (not a test; run by hand / gpurun).

    python tests/perf_probe.py [--scen 296] [--req 32] [--L 64] [--n 256] [--nbuf 3] [--budget 110]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scen", type=int, default=296)
    ap.add_argument("--req", type=int, default=32)
    ap.add_argument("--L", type=int, default=64)
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--window", type=int, default=64)
    ap.add_argument("--nbuf", type=int, default=0)
    ap.add_argument("--budget", type=int, default=0)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--nojitter", action="store_true")
    ap.add_argument("--mode", default="slots")
    ap.add_argument("--stage", type=int, default=0)
    ap.add_argument("--sbuf", type=int, default=0)
    ap.add_argument("--lib", default="", help="alternative libswarmsched_b200.so (A/B builds)")
    ap.add_argument("--c5", default="", help="C5 sub-pool (8b / 32b / 70b) instead of synthetic_cluster(--n)")
    args = ap.parse_args()
    import torch
    from paper_2509_26182_b200 import _native as N, scenarios as scen
    if args.lib:
        N.load_library(args.lib)
    from paper_2509_26182_b200.batched import ScenarioReplayer
    from helpers_golden import plan_from_golden
    from oracle import alloc_ref
    t0 = time.time()
    if args.c5:
        cl, model = {n: (c, m) for n, c, m in scen.c5_pools(0)}[args.c5]
        args.L, args.n = model.layer_count, len(cl.gpus)
    else:
        cl, model = scen.synthetic_cluster(args.n, seed=0, model=scen.bench_model(args.L))
    d = alloc_ref.allocate(cl, model)
    d["objective"] = d["objective"].hex()
    d["per_k"] = [dict(r, z=r["z"].hex()) for r in d["per_k"]]
    plan = plan_from_golden(d)
    ss = scen.build_scenarios(cl, model, plan, args.scen, seed0=1, churn=0.05, jitter=not args.nojitter,
                              host_events=False)
    print(f"prep {time.time()-t0:.1f}s k={plan.replication_count}", flush=True)
    lib = N.lib()
    if args.nbuf or args.budget:
        lib.ss_set_tiling(args.budget * 1024, args.nbuf, None, None)
    if args.stage or args.sbuf:
        lib.ss_set_slot_staging(args.stage * 1024, args.sbuf)
    rp = ScenarioReplayer(ss, window=args.window, mode=args.mode)
    torch.cuda.synchronize()
    t1 = time.time()
    rp.build()
    torch.cuda.synchronize()
    print(f"build {1e3*(time.time()-t1):.1f} ms", flush=True)
    out = rp.run(args.req)
    torch.cuda.synchronize()
    rp.raise_first_failure()
    b2 = rp.bytes_per_selection()
    times = []
    for _ in range(args.iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rp.run(args.req, out=out)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    t = float(np.median(times))
    sel = args.scen * args.req
    gbs = float(b2.mean()) * sel / t / 1e9
    print(json.dumps({"mode": rp.mode, "s_rows": getattr(rp, "s_rows", None), "scen": args.scen, "req": args.req, "L": args.L, "n": args.n, "k": plan.replication_count,
                      "time_ms": t * 1e3, "sel_per_s": sel / t, "B2_mean": float(b2.mean()),
                      "algo_GBps": gbs, "frac_hbm": gbs / 6538.9, "times": times}))


if __name__ == "__main__":
    main()
