"""Host side of the region-tiled replay (no GPU): the bound tables the kernel's skip test relies on.

ss_replay_regions skips a cross-region block S -> D when cmin_S + lb[S][D] > cmin_D + ub[D]; that is exact only if
lb[S][D] is <= every S -> D entry and ub[D] >= every D -> D entry of EVERY scenario's jittered matrix
(scenarios.ScenarioSet.scenario_rtt, the values the kernels relax).  Checked here on the C4 and C5 pools.
"""

import numpy as np


def _plan(cl, model):
    from helpers_golden import plan_from_golden
    from oracle import alloc_ref
    d = alloc_ref.allocate(cl, model)
    d["objective"] = d["objective"].hex()
    d["per_k"] = [dict(r, z=r["z"].hex()) for r in d["per_k"]]
    return plan_from_golden(d)


def _check_bounds(ss, n_scen):
    from paper_2509_26182_b200.batched import region_tiles
    t = region_tiles(ss)
    T = t.n_tiles
    lb = t.bounds[:T * T].reshape(T, T)
    ub = t.bounds[T * T:T * T + T]
    uni = t.bounds[T * T + T:].reshape(T, T)
    mem = [np.nonzero(t.tile_of == k)[0] for k in range(T)]
    base = np.asarray(ss.base_rtt)
    for a in range(T):                     # uni[S][D]: the common pool value the kernel multiplies by the jitter
        for b in range(T):
            if a != b and np.isfinite(uni[a, b]):
                assert np.all(base[np.ix_(mem[a], mem[b])] == uni[a, b])
    for s in range(n_scen):
        m = ss.scenario_rtt(s)
        for a in range(T):
            assert m[np.ix_(mem[a], mem[a])].max() <= ub[a]
            for b in range(T):
                if a != b:
                    assert m[np.ix_(mem[a], mem[b])].min() >= lb[a, b]
    return t


def test_region_bounds_hold_on_c4_scenarios():
    from paper_2509_26182_b200 import scenarios as scen
    cl, model = scen.synthetic_cluster(256, seed=0, model=scen.bench_model(64))
    ss = scen.build_scenarios(cl, model, _plan(cl, model), 24, seed0=3, churn=0.05, jitter=True)
    t = _check_bounds(ss, 24)
    assert t.n_tiles == 4 and t.fits() and t.gap > 0
    uni = t.bounds[20:].reshape(4, 4)
    assert np.all(uni[~np.eye(4, dtype=bool)] == 0.010)      # every cross pair at the default cross-region RTT


def test_region_bounds_hold_on_c5_scenarios():
    from paper_2509_26182_b200 import scenarios as scen
    name, cl, model = scen.c5_pools(0)[2]                     # 70B sub-pool: 384 GPUs, 8 regions
    ss = scen.build_scenarios(cl, model, _plan(cl, model), 6, seed0=11, churn=0.05, jitter=True)
    t = _check_bounds(ss, 6)
    assert t.n_tiles == 8 and t.fits() and t.gap > 0
    uni = t.bounds[72:].reshape(8, 8)
    assert np.isfinite(uni[~np.eye(8, dtype=bool)]).all()   # the explicit table is uniform per region pair


def test_region_tiles_without_jitter_are_the_pool_extremes():
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import region_tiles
    cl, model = scen.synthetic_cluster(64, seed=2, model=scen.bench_model(32))
    ss = scen.build_scenarios(cl, model, _plan(cl, model), 2, churn=0.0, jitter=False)
    t = region_tiles(ss)
    T = t.n_tiles
    assert np.all(t.bounds[:T * T].reshape(T, T)[~np.eye(T, dtype=bool)] == 0.010)   # default cross-region RTT
    assert np.all(t.bounds[T * T:T * T + T] == 0.001)                                 # intra-region links
