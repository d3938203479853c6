"""Ad-hoc ncu targets (not a test): one launch of a chosen kernel family at its bench shape.

    ncu --set full -k regex:<kernel> -c 1 python tests/ncu_targets.py <admission|sim|exact|cover|cover64|warp|slots|blocks|c5>

``slots`` / ``blocks``: bench.py's own headline launch (C4 pool, 1,184 device-churned scenarios, 64 requests, W=64),
launched twice -- profile the second (``-s 1 -c 1``), whose requests 64..127 run the steady state.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(what):
    import torch
    from paper_2509_26182_b200 import allocate, scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer, VariantSweep
    if what in ("admission", "sim", "warp"):
        cl, model = scen.synthetic_cluster(64, seed=0, model=scen.bench_model(64))
        plan = allocate(cl, model)
        S = 1184
        ss = scen.build_scenarios(cl, model, plan, S, seeds=list(range(S)), churn=0.0, jitter=True)
        if what == "admission":
            rp = ScenarioReplayer(ss, window=24, mode="warp")
            rp.admit(256, tok_lo=30000, tok_hi=90000)
        elif what == "sim":
            rp = ScenarioReplayer(ss, window=1, mode="warp")
            traces = [scen.generate_trace(150.0, 2.0, seed=s, prompt_tokens=(500, 20000), output_tokens=(8, 48))
                      for s in range(S)]
            rp.simulate(traces)
        else:
            rp = ScenarioReplayer(ss, window=64, mode="warp")
            rp.run(64)
    elif what in ("slots", "blocks", "cluster", "regions"):
        cl, model = scen.synthetic_cluster(256, seed=0, model=scen.bench_model(64))
        plan = allocate(cl, model)
        S = 1184
        ss = scen.build_scenarios(cl, model, plan, S, churn=0.05, jitter=True, seeds=list(range(S)), host_events=False)
        rp = ScenarioReplayer(ss, window=64, mode=what)
        out = rp.run(64)
        rp.run(64, out=out)
    elif what == "c5":
        pools = scen.c5_pools(0)
        name, cl, model = pools[2]                                   # 70B: L=80 over 384 GPUs
        plan = allocate(cl, model)
        S = 1184
        ss = scen.build_scenarios(cl, model, plan, S, churn=0.05, jitter=True, seeds=list(range(S)), host_events=False)
        rp = ScenarioReplayer(ss, window=64, mode=os.environ.get("SS_MODE", "auto"))
        out = rp.run(64)
        rp.run(64, out=out)
    elif what == "exact":
        packed, _ = scen.bench_variants(256, 64, 64, seed0=0)      # C2-shaped pools: 16 GPUs per region
        VariantSweep(packed, fill_all=True).run()
    elif what in ("cover", "cover64"):
        packed, _ = scen.bench_variants(1812, 256, 80 if what == "cover" else 64, seed0=0)
        VariantSweep(packed, fill_all=True).run()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(sys.argv[1])
