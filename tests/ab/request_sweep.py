"""Selections/s of the region replay vs requests per launch R and scenarios per launch S (not a test; B200 via gpurun).

Per-launch set-up amortises over R (measured: it barely matters), the last wave's tail over S (2,368 scenarios per
launch run ~2.5% faster than the bench step's 1,184).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def main():
    import torch
    from paper_2509_26182_b200 import allocate, scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    cl, model = scen.synthetic_cluster(256, seed=0, model=scen.bench_model(64))
    plan = allocate(cl, model)
    for S in (1184, 2368):
        ss = scen.build_scenarios(cl, model, plan, S, churn=0.05, jitter=True, seeds=list(range(S)),
                                  host_events=False)
        for R in (32, 64, 128, 256):
            rp = ScenarioReplayer(ss, window=64, mode="regions", max_requests=64 + 4 * R + 8)
            rp.run(64)
            rp.run(R)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                rp.run(R)
            e1.record()
            torch.cuda.synchronize()
            print(json.dumps({"S": S, "R": R, "sel_per_s": S * R * 3 / (e0.elapsed_time(e1) / 1e3)}), flush=True)


if __name__ == "__main__":
    main()
