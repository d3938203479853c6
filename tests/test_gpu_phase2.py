"""Phase-2 parity on a B200: CUDA path vs reference golden vectors and the oracle.

Bar: bit-exact chains and fp64 costs (router.py returns float64 sums of the
same IEEE operations, so no tolerance is needed or allowed).
"""

import math

import numpy as np
import pytest

from conftest import hx
from helpers_golden import case_latencies, hops_from_gpus, plan_from_golden, replay_inputs
from oracle import chain_ref

pytestmark = pytest.mark.gpu


def _perf_map_from_case(case):
    from paper_2509_26182_b200.perfmap import PerfMap
    pm = PerfMap(ttl_s=1e9)
    lat = case_latencies(case)
    names = {g for g, _ in lat} | {g for a, b, _ in case["rtts"] for g in (a, b)}
    for g in sorted(names):
        pm.register_gpu(g)
    for (g, l), v in lat.items():
        pm.publish_layer_latency(g, l, v, now=0.0)
    rtts = {(a, b): hx(v) for a, b, v in case["rtts"]}
    if rtts:
        pm.publish_link_rtts(rtts, now=0.0)
    return pm


def test_select_chain_golden(cuda_ready, router_cases):
    from paper_2509_26182_b200 import router as R
    from paper_2509_26182_b200.errors import NoPath, UncoveredLayer
    for i, case in enumerate(router_cases):
        snap = _perf_map_from_case(case).snapshot(0.0)
        want = case["result"]
        try:
            dag = R.build_dag(snap, case["L"], exclude=frozenset(case["exclude"]))
            chain = R.select_chain(dag, snap)
            got = {"status": "ok", "hops": [[h.gpu_id, h.start_layer, h.end_layer] for h in chain.hops],
                   "cost": chain.cost_s.hex(), "edges": R.count_dag_edges(dag, snap)}
        except UncoveredLayer as exc:
            got = {"status": "uncovered", "layer": exc.layer}
        except NoPath:
            got = {"status": "no_path"}
        assert got == want, i


def _map_for_plan(ids, base, rtt, plan):
    from paper_2509_26182_b200.perfmap import PerfMap
    pm = PerfMap(ttl_s=4.5, latency_fn=lambda g, l, occ, _b=dict(zip(ids, base)): _b[g] * (1 + occ))
    for g in ids:
        pm.register_gpu(g)
    n = len(ids)
    pm.publish_link_rtts({(ids[a], ids[b]): float(rtt[a, b]) for a in range(n) for b in range(a + 1, n)}, 0.0)
    for g, sl in plan.gpu_slices().items():
        pm.sync_gpu_layers(g, range(sl.start_layer, sl.end_layer + 1), 0.0)
    return pm


@pytest.mark.parametrize("name,limit", [("c1", 250), ("c1_tie", 120), ("rt16", 20), ("c2", 80)])
def test_chain_router_golden(cuda_ready, router_replays, name, limit):
    """The drop-in ChainRouter (device DP + PerfMap feedback) replays the reference op script."""
    from paper_2509_26182_b200.router import ChainRouter
    rep = router_replays[name]
    _, base, rtt, ids = replay_inputs(rep, rep["plan"])
    plan = plan_from_golden(rep["plan"])
    pm = _map_for_plan(ids, base, rtt, plan)
    router = ChainRouter(pm, rep["L"])
    pos = {g: i for i, g in enumerate(ids)}
    W = rep["window"]
    live = []
    for i in range(limit):
        if W is not None and W > 0 and i >= W:
            router.release(live.pop(0), 0.0)
        chain = router.route(0.0)
        if W == 0:
            router.release(chain, 0.0)
        elif W is not None:
            live.append(chain)
        want = rep["routes"][i]
        assert [[pos[h.gpu_id], h.start_layer, h.end_layer] for h in chain.hops] == want["hops"], (name, i)
        assert chain.cost_s == hx(want["cost"]), (name, i)
    assert router.stats.matrix_rebuilds == 1


def _replayer_for_golden(rep, plan_dict, n_scen=1, seed0=None, mode="slots"):
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    L = rep["L"]
    flops = hx(rep["flops"]) if "flops" in rep else None
    cl, model = scen.synthetic_cluster(rep["n"], seed=rep["seed"], model=scen.bench_model(L), homogeneous_flops=flops)
    plan = plan_from_golden(plan_dict)
    if "scenario_seed" in rep:
        ss = scen.build_scenarios(cl, model, plan, n_scen, seed0=rep["scenario_seed"], churn=0.05, jitter=True)
    else:
        ss = scen.build_scenarios(cl, model, plan, n_scen, churn=0.0, jitter=False)
    W = rep["window"]
    if mode == "warp" and int(ss.slice_hi.max()) > 0:
        layers = np.arange(1, L + 1)
        hosts = ((ss.slice_lo[None, :] <= layers[:, None]) & (ss.slice_hi[None, :] >= layers[:, None])).sum(axis=1)
        if hosts.max() > 32:
            pytest.skip("warp replay needs <= 32 hosts per layer")
    return ss, ScenarioReplayer(ss, window=-1 if W is None else W, max_requests=len(rep["routes"]) + 4, mode=mode)


@pytest.mark.parametrize("mode", ["slots", "cluster", "blocks", "warp"])
@pytest.mark.parametrize("name", ["c1", "c1_tie", "n32_tie", "rt16", "c2", "c4_s11", "c4_s12"])
def test_replay_kernel_golden(cuda_ready, router_replays, name, mode):
    """ss_replay / ss_replay_slots (on-device load update) == reference ChainRouter op script, bit-exact."""
    rep = router_replays[name]
    plan = rep.get("plan", router_replays.get("c4_plan"))
    ss, rp = _replayer_for_golden(rep, plan, mode=mode)
    if "leave" in rep:
        assert sorted(np.nonzero(ss.leave[0])[0].tolist()) == rep["leave"]
    n = len(rep["routes"])
    # two chunks: state (occupancy, ring, request counter) must persist across launches
    first = n // 3
    a = rp.run(first, gpus=True)
    b = rp.run(n - first, gpus=True)
    rp.raise_first_failure()
    gpus = np.concatenate([a.gpus.cpu().numpy()[0], b.gpus.cpu().numpy()[0]])
    cost = np.concatenate([a.cost.cpu().numpy()[0], b.cost.cpu().numpy()[0]])
    for r in range(n):
        assert hops_from_gpus(gpus[r].tolist()) == rep["routes"][r]["hops"], (name, r)
        assert float(cost[r]) == hx(rep["routes"][r]["cost"]), (name, r)
    occ = rp.occ.cpu().numpy()
    gone = set(rep.get("leave", []))
    assert [int(occ[g]) if g not in gone else 0 for g in range(len(occ))] == rep["final_occ"]


def _hash(gpus_row):
    M = (1 << 64) - 1
    from paper_2509_26182_b200.scenarios import splitmix64
    return sum(splitmix64((l << 32) | int(g)) for l, g in enumerate(gpus_row)) & M


@pytest.mark.parametrize("mode", ["slots", "cluster", "blocks", "regions"])
@pytest.mark.parametrize("window", [64, 0, -1, 1, 7])
def test_replay_many_scenarios_vs_oracle(cuda_ready, window, mode):
    """C4-shaped batch (L64/N256 pool, churn + jitter) vs the oracle, every scenario."""
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    import json, os
    here = os.path.dirname(os.path.abspath(__file__))
    plan = plan_from_golden(json.load(open(os.path.join(here, "golden", "router_replays.json")))["c4_plan"])
    cl, model = scen.synthetic_cluster(256, seed=0, model=scen.bench_model(64))
    S, n_req = 12, 40
    ss = scen.build_scenarios(cl, model, plan, S, seed0=1000 + window, churn=0.05, jitter=True)
    rp = ScenarioReplayer(ss, window=window, max_requests=n_req + 4, mode=mode)
    out = rp.run(n_req, gpus=True)
    rp.raise_first_failure()
    gpus, cost, hashes = out.gpus.cpu().numpy(), out.cost.cpu().numpy(), out.chain_hash.cpu().numpy()
    W = None if window < 0 else window
    for s in range(S):
        cols = ss.columns(s)
        want_g, want_c, want_occ, _ = chain_ref.replay(cols, ss.base_tau, ss.scenario_rtt(s), n_req, W,
                                                       chain_ref.occ_power_table(n_req + 4))
        assert gpus[s].tolist() == want_g, s
        assert cost[s].tolist() == want_c, s
        assert rp.occ.view(S, -1)[s].cpu().numpy().tolist() == want_occ.tolist(), s
        for r in range(n_req):
            assert int(hashes[s, r]) & ((1 << 64) - 1) == _hash(want_g[r])


@pytest.mark.parametrize("mode", ["slots", "cluster", "blocks", "warp", "regions"])
def test_replay_tie_pool_vs_oracle(cuda_ready, mode):
    """Homogeneous flops => many exact ties (13-23% of columns): first-index rule must hold."""
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    from oracle import alloc_ref
    from helpers_golden import plan_from_golden
    cl, model = scen.synthetic_cluster(64, seed=5, model=scen.bench_model(48), homogeneous_flops=1e14)
    plan = plan_from_golden(_plan_dict(alloc_ref.allocate(cl, model)))
    ss = scen.build_scenarios(cl, model, plan, 4, seed0=77, churn=0.05, jitter=False)
    rp = ScenarioReplayer(ss, window=16, max_requests=64, mode=mode)
    out = rp.run(60, gpus=True)
    rp.raise_first_failure()
    for s in range(4):
        want_g, want_c, _, _ = chain_ref.replay(ss.columns(s), ss.base_tau, ss.scenario_rtt(s), 60, 16,
                                                chain_ref.occ_power_table(64))
        assert out.gpus.cpu().numpy()[s].tolist() == want_g
        assert out.cost.cpu().numpy()[s].tolist() == want_c


def _plan_dict(d):
    d = dict(d)
    d["objective"] = d["objective"].hex()
    d["per_k"] = [dict(r, z=r["z"].hex()) for r in d["per_k"]]
    return d


@pytest.mark.parametrize("mode", ["slots", "blocks", "warp"])
def test_uncovered_scenario_reports_status(cuda_ready, mode):
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    from paper_2509_26182_b200.errors import UncoveredLayer
    cl, model = scen.synthetic_cluster(8, seed=0, model=scen.bench_model(32))
    from oracle import alloc_ref
    plan = plan_from_golden(_plan_dict(alloc_ref.allocate(cl, model)))
    ss = scen.build_scenarios(cl, model, plan, 3, churn=0.0, jitter=False)
    first_gpu = min(g for g in range(ss.n_gpus) if ss.slice_lo[g] == 1)
    ss.leave[1, :] = False
    ss.leave[1, [g for g in range(ss.n_gpus) if ss.slice_lo[g] <= 1 <= ss.slice_hi[g]]] = True
    rp = ScenarioReplayer(ss, window=4, max_requests=16, mode=mode)
    rp.run(5)
    st = rp.status.cpu().numpy()
    assert st[0] == 0 and st[2] == 0 and st[1] == 1 and int(rp.aux.cpu()[1]) == 1
    with pytest.raises(UncoveredLayer):
        rp.raise_first_failure()
    assert first_gpu >= 0


@pytest.mark.parametrize("mode", ["slots", "blocks"])
def test_replay_wide_columns_vs_oracle(cuda_ready, mode):
    """k = 129 hosts per layer: every slot-replay warp owns > 32 source positions (multi-pass staging)."""
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    from oracle import alloc_ref
    cl, model = scen.synthetic_cluster(144, seed=0, model=scen.bench_model(10))
    plan = plan_from_golden(_plan_dict(alloc_ref.allocate(cl, model)))
    assert plan.replication_count == 129
    ss = scen.build_scenarios(cl, model, plan, 3, seed0=404, churn=0.05, jitter=True)
    rp = ScenarioReplayer(ss, window=8, max_requests=32, mode=mode)
    assert rp.mode == mode
    out = rp.run(24, gpus=True)
    rp.raise_first_failure()
    for s in range(3):
        want_g, want_c, want_occ, _ = chain_ref.replay(ss.columns(s), ss.base_tau, ss.scenario_rtt(s), 24, 8,
                                                       chain_ref.occ_power_table(32))
        assert out.gpus.cpu().numpy()[s].tolist() == want_g, s
        assert out.cost.cpu().numpy()[s].tolist() == want_c, s
        assert rp.occ.view(3, -1)[s].cpu().numpy().tolist() == want_occ.tolist(), s


def test_replay_auto_mode_picks_blocks_for_wide_frontiers(cuda_ready):
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    from oracle import alloc_ref
    cl, model = scen.synthetic_cluster(144, seed=0, model=scen.bench_model(10))
    plan = plan_from_golden(_plan_dict(alloc_ref.allocate(cl, model)))
    ss = scen.build_scenarios(cl, model, plan, 1, churn=0.0, jitter=False)
    assert ScenarioReplayer(ss, window=8).mode == "blocks"
    cl, model = scen.synthetic_cluster(64, seed=0, model=scen.bench_model(64))
    plan = plan_from_golden(_plan_dict(alloc_ref.allocate(cl, model)))
    ss = scen.build_scenarios(cl, model, plan, 1, churn=0.0, jitter=False)
    assert ScenarioReplayer(ss, window=8).mode == "warp"


@pytest.mark.parametrize("window", [64, 0, -1, 1, 7])
def test_warp_replay_c2_shape_vs_oracle(cuda_ready, window):
    """Warp-resident replay on C2-shaped scenarios (L64/N64 pool, k=17, churn + jitter) vs the oracle."""
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    from oracle import alloc_ref
    cl, model = scen.synthetic_cluster(64, seed=0, model=scen.bench_model(64))
    plan = plan_from_golden(_plan_dict(alloc_ref.allocate(cl, model)))
    S, n_req = 6, 40
    ss = scen.build_scenarios(cl, model, plan, S, seed0=300 + window, churn=0.05, jitter=True)
    rp = ScenarioReplayer(ss, window=window, max_requests=n_req + 4)
    assert rp.mode == "warp"
    a = rp.run(n_req // 2, gpus=True)
    b = rp.run(n_req - n_req // 2, gpus=True)
    rp.raise_first_failure()
    gpus = np.concatenate([a.gpus.cpu().numpy(), b.gpus.cpu().numpy()], axis=1)
    cost = np.concatenate([a.cost.cpu().numpy(), b.cost.cpu().numpy()], axis=1)
    hashes = np.concatenate([a.chain_hash.cpu().numpy(), b.chain_hash.cpu().numpy()], axis=1)
    W = None if window < 0 else window
    for s in range(S):
        want_g, want_c, want_occ, _ = chain_ref.replay(ss.columns(s), ss.base_tau, ss.scenario_rtt(s), n_req, W,
                                                       chain_ref.occ_power_table(n_req + 4))
        assert gpus[s].tolist() == want_g, s
        assert cost[s].tolist() == want_c, s
        assert rp.occ.view(S, -1)[s].cpu().numpy().tolist() == want_occ.tolist(), s
        for r in range(n_req):
            assert int(hashes[s, r]) & ((1 << 64) - 1) == _hash(want_g[r])


@pytest.mark.gpu
@pytest.mark.parametrize("n,L,nwd", [(16, 48, 1), (24, 32, 2), (36, 24, 3), (48, 24, 4)])
def test_warp_replay_destination_split_widths_vs_oracle(cuda_ready, n, L, nwd):
    """replay_warp_kernel<NWD> at every warp count (column widths 1-8, 9-16, 17-24, 25-32 hosts) vs the oracle."""
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    from oracle import alloc_ref
    cl, model = scen.synthetic_cluster(n, seed=0, model=scen.bench_model(L))
    plan = plan_from_golden(_plan_dict(alloc_ref.allocate(cl, model)))
    S, n_req, window = 4, 36, 16
    ss = scen.build_scenarios(cl, model, plan, S, seed0=900 + n, churn=0.05, jitter=True)
    widest = max(max(len(c) for c in ss.columns(s)) for s in range(S))
    assert (widest + 7) // 8 == nwd, widest
    rp = ScenarioReplayer(ss, window=window, max_requests=n_req + 4, mode="warp")
    out = rp.run(n_req, gpus=True)
    rp.raise_first_failure()
    gpus, cost = out.gpus.cpu().numpy(), out.cost.cpu().numpy()
    for s in range(S):
        want_g, want_c, want_occ, _ = chain_ref.replay(ss.columns(s), ss.base_tau, ss.scenario_rtt(s), n_req, window,
                                                       chain_ref.occ_power_table(n_req + 4))
        assert gpus[s].tolist() == want_g, s
        assert cost[s].tolist() == want_c, s
        assert rp.occ.view(S, -1)[s].cpu().numpy().tolist() == want_occ.tolist(), s


def test_warp_matrix_mode_many_scenarios_vs_oracle(cuda_ready):
    """More scenarios than SMs: the warp kernel stages each scenario's RTT matrix (ss_scenario_rtt) instead of its
    edge blocks and gathers E_b[i][j] = M[node_i][node_j].  Every 10th of 160 churned + jittered C2 scenarios vs
    the oracle, and all 160 against the edge-block run of the same scenarios in groups below the SM count."""
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    from oracle import alloc_ref
    cl, model = scen.synthetic_cluster(64, seed=0, model=scen.bench_model(64))
    plan = plan_from_golden(_plan_dict(alloc_ref.allocate(cl, model)))
    S, n_req, W = 160, 24, 8
    ss = scen.build_scenarios(cl, model, plan, S, seed0=2000, churn=0.05, jitter=True)
    rp = ScenarioReplayer(ss, window=W, max_requests=n_req + 4, mode="warp")
    assert rp._warp_mats() is not None                       # matrix mode offered and taken
    out = rp.run(n_req, gpus=True)
    rp.raise_first_failure()
    gpus, cost = out.gpus.cpu().numpy(), out.cost.cpu().numpy()
    for s in range(0, S, 10):
        want_g, want_c, want_occ, _ = chain_ref.replay(ss.columns(s), ss.base_tau, ss.scenario_rtt(s), n_req, W,
                                                       chain_ref.occ_power_table(n_req + 4))
        assert gpus[s].tolist() == want_g, s
        assert cost[s].tolist() == want_c, s
    half = scen.build_scenarios(cl, model, plan, 80, seed0=2000, churn=0.05, jitter=True)
    rp2 = ScenarioReplayer(half, window=W, max_requests=n_req + 4, mode="warp")
    assert rp2._warp_mats() is None                           # 80 <= SMs: edge blocks
    out2 = rp2.run(n_req, gpus=True)
    assert np.array_equal(out2.gpus.cpu().numpy(), gpus[:80]) and np.array_equal(out2.cost.cpu().numpy(), cost[:80])
