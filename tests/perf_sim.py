"""Ad-hoc probe: where ScenarioReplayer.simulate spends its wall time at the bench's C2 simulator shape."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2509_26182_b200 import allocate, scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    S = 1184
    cl, model = scen.synthetic_cluster(64, seed=0, model=scen.bench_model(64))
    plan = allocate(cl, model)
    ss = scen.build_scenarios(cl, model, plan, S, seeds=list(range(S)), churn=0.0, jitter=True)
    traces = [scen.generate_trace(150.0, 2.0, seed=s, prompt_tokens=(500, 20000), output_tokens=(8, 48))
              for s in range(S)]
    rp = ScenarioReplayer(ss, window=1, mode="warp")
    rp.build()
    rp.simulate(traces)
    torch.cuda.synchronize()
    pr = cProfile.Profile()
    t0 = time.perf_counter()
    pr.enable()
    rp.simulate(traces)
    pr.disable()
    print(f"simulate wall {1e3 * (time.perf_counter() - t0):.1f} ms")
    pstats.Stats(pr).sort_stats("tottime").print_stats(12)


if __name__ == "__main__":
    main()
