"""Parity at the bench's own size ("every 97th scenario in full plus 1% random others").

The headline workload exactly as bench.py builds it -- C4 pool (L64/N256, k=73), 1,184 scenarios with
device-drawn departures + jitter, W=64 -- through every throughput kernel (regions, slots, blocks, cluster), for 320 requests (5 x W): the timed
region's steady state, with a release before every route from request 64 on and up to 64 live chains.  Every 97th scenario
plus a seeded 1% random sample is replayed by the oracle on the same (host-drawn, identical) scenario states
and must match chain for chain, cost for cost, occupancy for occupancy.  The kernels must agree on all
1,184 scenarios.
"""

import numpy as np
import pytest

from oracle import chain_ref

pytestmark = pytest.mark.gpu

S, R, W = 1184, 320, 64


def test_c4_bench_size_sampled_scenarios_vs_oracle(cuda_ready):
    from paper_2509_26182_b200 import allocate, scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    from paper_2509_26182_b200.distributed import shard
    cl, model = scen.synthetic_cluster(256, seed=0, model=scen.bench_model(64))
    plan = allocate(cl, model)
    assert plan.replication_count == 73
    seeds = shard(S, 0, 1)
    dev = scen.build_scenarios(cl, model, plan, S, churn=0.05, jitter=True, seeds=seeds, host_events=False)
    outs = {}
    for mode in ("regions", "slots", "blocks", "cluster"):
        rp = ScenarioReplayer(dev, window=W, mode=mode, max_requests=R)
        out = rp.run(R, gpus=True)
        rp.raise_first_failure()
        outs[mode] = (out.gpus.cpu().numpy(), out.cost.cpu().numpy(), rp.occ.view(S, -1).cpu().numpy())
    for m in ("blocks", "cluster", "regions"):
        for a, b in zip(outs["slots"], outs[m]):
            assert np.array_equal(a, b), m
    rng = np.random.default_rng(97)
    sample = sorted(set(range(0, S, 97)) | set(rng.choice(S, size=S // 100, replace=False).tolist()))
    host = scen.build_scenarios(cl, model, plan, len(sample), churn=0.05, jitter=True, seeds=seeds[sample])
    gpus, cost, occ = outs["slots"]
    for k, s in enumerate(sample):
        want_g, want_c, want_occ, _ = chain_ref.replay(host.columns(k), host.base_tau, host.scenario_rtt(k), R, W,
                                                       chain_ref.occ_power_table(W + 2))
        assert gpus[s].tolist() == want_g, s
        assert cost[s].tolist() == want_c, s
        assert occ[s].tolist() == want_occ.tolist(), s
