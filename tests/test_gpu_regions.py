"""Region-tiled replay (ss_replay_regions, replay_regions.cu) vs the oracle, on pools built to defeat its bound test.

The kernel skips a cross-region block only when no candidate of it can reach -- or tie -- a destination minimum,
and relaxes every other block exactly (entries recomputed from the pool matrix and the scenario jitter).  The C4 /
C5 pools exercise the skip (> 99% of cross blocks); these pools exercise the relaxed path and its tie rule:

* cross-region RTT 1.1 ms against 1 ms inside a region (bound gap < 0: most cross blocks are relaxed);
* cross-region RTT == intra-region RTT with homogeneous flops and no jitter: exact cross-region ties, where the
  lexicographic (value, position) merge must reproduce numpy's first-index argmin;
* eight regions (the C5 tile count) and every release window of the op script.
Reference semantics: router.py:163-185 (_relax), router.py:247-260 (route/release).
"""

import numpy as np
import pytest

from helpers_golden import plan_from_golden
from oracle import alloc_ref, chain_ref

pytestmark = pytest.mark.gpu


def _plan_dict(d):
    d = dict(d)
    d["objective"] = d["objective"].hex()
    d["per_k"] = [dict(r, z=r["z"].hex()) for r in d["per_k"]]
    return d


def _pool(n, L, *, cross=None, region_count=None, homogeneous=None, seed=0):
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.topology import ClusterSnapshot
    cl, model = scen.synthetic_cluster(n, seed=seed, model=scen.bench_model(L), region_count=region_count,
                                       homogeneous_flops=homogeneous)
    if cross is not None:
        cl = ClusterSnapshot(gpus=cl.gpus, links=cl.links, default_cross_region_rtt_s=cross)
    plan = plan_from_golden(_plan_dict(alloc_ref.allocate(cl, model)))
    return cl, model, plan


def _check(ss, n_req, window, stats_min=None):
    from paper_2509_26182_b200.batched import ScenarioReplayer
    rp = ScenarioReplayer(ss, window=window, max_requests=n_req + 4, mode="regions")
    out = rp.run(n_req, gpus=True)
    rp.raise_first_failure()
    gpus, cost = out.gpus.cpu().numpy(), out.cost.cpu().numpy()
    W = None if window < 0 else window
    for s in range(ss.n_scenarios):
        want_g, want_c, want_occ, _ = chain_ref.replay(ss.columns(s), ss.base_tau, ss.scenario_rtt(s), n_req, W,
                                                       chain_ref.occ_power_table(n_req + 4))
        assert gpus[s].tolist() == want_g, s
        assert cost[s].tolist() == want_c, s
        assert rp.occ.view(ss.n_scenarios, -1)[s].cpu().numpy().tolist() == want_occ.tolist(), s
    return rp


@pytest.mark.parametrize("window", [64, 7, 0, -1])
def test_regions_small_gap_pool_vs_oracle(cuda_ready, window):
    """Cross-region 1.1 ms vs intra 1 ms: the bound test keeps most cross blocks, relaxed from the pool matrix."""
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import region_tiles
    cl, model, plan = _pool(128, 48, cross=0.0011, seed=3)
    ss = scen.build_scenarios(cl, model, plan, 16, seed0=500 + window, churn=0.05, jitter=True)
    assert region_tiles(ss).gap < 0
    _check(ss, 48, window)


def test_regions_cross_region_ties_vs_oracle(cuda_ready):
    """Homogeneous flops, cross == intra RTT, no jitter: exact ties across regions (first-index rule)."""
    from paper_2509_26182_b200 import scenarios as scen
    cl, model, plan = _pool(96, 40, cross=0.001, homogeneous=1e14, seed=5)
    ss = scen.build_scenarios(cl, model, plan, 8, seed0=77, churn=0.05, jitter=False)
    _check(ss, 60, 16)


@pytest.mark.parametrize("window", [64, 1])
def test_regions_eight_regions_vs_oracle(cuda_ready, window):
    """Eight regions (C5's tile count) on the bench pool law: eight consumer warps, seven bound tests each."""
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import region_tiles
    cl, model, plan = _pool(256, 64, region_count=8, seed=1)
    ss = scen.build_scenarios(cl, model, plan, 12, seed0=40 + window, churn=0.05, jitter=True)
    assert region_tiles(ss).n_tiles == 8
    _check(ss, 80, window)


def test_regions_matches_slots_on_c4_batch(cuda_ready):
    """C4 shape with device-drawn departures: regions == slots == blocks on every scenario, 200 requests."""
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer, replay_mode
    cl, model, plan = _pool(256, 64, seed=0)
    ss = scen.build_scenarios(cl, model, plan, 296, seed0=9000, churn=0.05, jitter=True, host_events=False)
    assert replay_mode(ss, window=64) == "regions"
    res = {}
    for mode in ("regions", "slots", "blocks"):
        rp = ScenarioReplayer(ss, window=64, mode=mode, max_requests=200)
        out = rp.run(200, gpus=True)
        rp.raise_first_failure()
        res[mode] = (out.gpus.cpu().numpy(), out.cost.cpu().numpy(), rp.occ.cpu().numpy())
    for m in ("slots", "blocks"):
        for a, b in zip(res["regions"], res[m]):
            assert np.array_equal(a, b), m


def test_regions_nonuniform_cross_links_vs_oracle(cuda_ready):
    """Explicit cross-region links of different RTTs (uni[S][D] = NaN): kept blocks read the pool matrix entry by
    entry instead of the per-tile-pair constant; many are kept (cross links 0.9-1.6 ms vs 1 ms inside)."""
    import random
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import region_tiles
    from paper_2509_26182_b200.topology import ClusterSnapshot
    cl, model, plan = _pool(96, 40, seed=7)
    rng = random.Random(7)
    ids = sorted(g.id for g in cl.gpus)
    links = dict(cl.links)
    for i in range(len(ids)):
        for j in range(i + 1, len(ids)):
            a, b = cl.gpu(ids[i]), cl.gpu(ids[j])
            if a.region != b.region and rng.random() < 0.5:
                links[(ids[i], ids[j])] = rng.uniform(0.0009, 0.0016)
    cl2 = ClusterSnapshot(gpus=cl.gpus, links=links, default_cross_region_rtt_s=0.0012)
    ss = scen.build_scenarios(cl2, model, plan, 10, seed0=300, churn=0.05, jitter=True)
    t = region_tiles(ss)
    T = t.n_tiles
    assert np.isnan(t.bounds[T * T + T:]).reshape(T, T)[~np.eye(T, dtype=bool)].all()
    _check(ss, 70, 16)


@pytest.mark.parametrize("region_count", [1, 2, 3, 5, 6, 7])
def test_regions_every_tile_count_vs_oracle(cuda_ready, region_count):
    """Every replay_regions_kernel<NTL> instantiation the C4 (4) / C5 (8) tests do not reach: 16 GPUs per region,
    L=32, churn + jitter, W=16 (releases from request 16 on); with three regions also a small-gap pool (cross
    1.1 ms) so kept cross blocks run on an odd tile count."""
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import region_tiles
    cl, model, plan = _pool(16 * region_count, 32, region_count=region_count, seed=2)
    ss = scen.build_scenarios(cl, model, plan, 6, seed0=5, churn=0.05, jitter=True)
    t = region_tiles(ss)
    assert t.n_tiles == region_count and t.fits()
    _check(ss, 96, 16)
    if region_count == 3:
        cl, model, plan = _pool(48, 32, region_count=3, cross=0.0011, seed=2)
        ss = scen.build_scenarios(cl, model, plan, 6, seed0=7, churn=0.05, jitter=True)
        assert region_tiles(ss).gap < 0
        _check(ss, 96, 16)
