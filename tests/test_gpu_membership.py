"""Membership churn on device (ss_scenario_membership, ss_membership_triggers) vs the reference.

The device generator must reproduce the host generator's events (which tests/test_membership.py pins to the
reference MembershipManager), the replay on the device-generated states must route exactly like the reference
ChainRouter on the churned/joined perf map, and the device evaluate_triggers must return the reference's
decision, CoV and per-layer loads bit for bit.
"""

import json
import os

import numpy as np
import pytest

from conftest import hx
from helpers_membership import pool_for_case

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
CASES = ["c1j", "n64j", "n256j", "n64j_lowthr"]
DECISION = {0: ["local", "balanced"], 1: ["global", "uncovered_layers"], 2: ["global", "load_cov_exceeded"]}


@pytest.fixture(scope="module")
def membership_cases():
    with open(os.path.join(HERE, "golden", "membership_cases.json")) as fh:
        return json.load(fh)


def _sets(case, seeds):
    from paper_2509_26182_b200 import scenarios as scen
    full, model, plan, join_ids, _ = pool_for_case(case)
    kw = dict(seeds=seeds, churn=case["churn"], jitter=False, join_pool=join_ids, joins=case["joins"])
    host = scen.build_scenarios(full, model, plan, len(seeds), host_events=True, **kw)
    dev = scen.build_scenarios(full, model, plan, len(seeds), host_events=False, **kw)
    return host, dev


def _hops(row):
    out, start = [], 1
    for layer in range(2, len(row) + 1):
        if row[layer - 1] != row[layer - 2]:
            out.append([row[layer - 2], start, layer - 1])
            start = layer
    out.append([row[-1], start, len(row)])
    return out


@pytest.mark.parametrize("mode", ["auto", "blocks", "slots"])
@pytest.mark.parametrize("name", CASES)
def test_device_events_replay_and_triggers(cuda_ready, membership_cases, name, mode):
    from paper_2509_26182_b200.batched import ScenarioReplayer
    case = membership_cases[name]
    want = case["scenarios"]
    seeds = [w["seed"] for w in want]
    host, dev = _sets(case, seeds)
    R = case["routes"]
    rp = ScenarioReplayer(dev, window=-1, max_requests=R + 4, mode=mode)
    rp.build()
    S, G = dev.n_scenarios, dev.n_gpus
    leave = rp.leave.view(S, G).cpu().numpy().astype(bool)
    lo = rp.lo_s.view(S, G).cpu().numpy()
    hi = rp.hi_s.view(S, G).cpu().numpy()
    assert (leave == host.leave).all(), name
    assert (lo == host.slice_lo_s).all() and (hi == host.slice_hi_s).all(), name
    joined = rp.joined.view(S, -1).cpu().numpy()
    for s, w in enumerate(want):
        assert [int(g) for g in joined[s][:len(w["joined"])]] == w["joined"]
    out = rp.run(R, gpus=True)
    rp.raise_first_failure()
    gpus, cost = out.gpus.cpu().numpy(), out.cost.cpu().numpy()
    occ = rp.occ.view(S, G).cpu().numpy()
    dec, cov, hole, loads = rp.triggers(cov_threshold=case["cov_threshold"])
    dec, cov, hole, loads = dec.cpu().numpy(), cov.cpu().numpy(), hole.cpu().numpy(), loads.cpu().numpy()
    for s, w in enumerate(want):
        for r in range(R):
            assert _hops(gpus[s, r].tolist()) == w["chains"][r]["hops"], (name, s, r)
            assert float(cost[s, r]) == hx(w["chains"][r]["cost"]), (name, s, r)
        assert occ[s].tolist() == w["occ"], (name, s)
        assert DECISION[int(dec[s])] + [float(cov[s]).hex(), []] == w["decision"], (name, s)
        assert [float(v).hex() for v in loads[s]] == w["loads"], (name, s)
        assert int(hole[s]) == 0


def test_device_triggers_uncovered(cuda_ready, membership_cases):
    from paper_2509_26182_b200.batched import ScenarioReplayer
    case = membership_cases["n64j_hole"]
    w = case["scenarios"][0]
    host, _ = _sets(case, [w["seed"]])
    hole_gpus = [g for g in range(host.n_gpus)
                 if host.present0[g] and host.slice_lo[g] <= case["hole_layer"] <= host.slice_hi[g]]
    host.leave[0, hole_gpus] = True
    host.slice_lo_s = np.where(host.leave, 0, np.broadcast_to(host.slice_lo, host.leave.shape)).astype(np.int32)
    host.slice_hi_s = np.where(host.leave, -1, np.broadcast_to(host.slice_hi, host.leave.shape)).astype(np.int32)
    host.joins = 0
    rp = ScenarioReplayer(host, window=-1, max_requests=8, mode="blocks")
    rp.per_scenario = True
    rp.lo_s = rp.torch.from_numpy(host.slice_lo_s.reshape(-1)).to(rp.dev)
    rp.hi_s = rp.torch.from_numpy(host.slice_hi_s.reshape(-1)).to(rp.dev)
    rp.build()
    dec, cov, hole, _ = rp.triggers()
    assert DECISION[int(dec[0])] + [float(cov[0]).hex()] == w["decision"][:3]
    assert int(hole[0]) == w["decision"][3][0]
    st = rp.status.cpu().numpy()
    assert st[0] == 1 and int(rp.aux.cpu()[0]) == w["decision"][3][0]


def test_device_departures_equal_host_churn_c4(cuda_ready):
    """C4 (leave-only events): the device-drawn departures equal the host churn sets scenario for scenario."""
    import json
    from helpers_golden import plan_from_golden
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    plan = plan_from_golden(json.load(open(os.path.join(HERE, "golden", "router_replays.json")))["c4_plan"])
    cl, model = scen.synthetic_cluster(256, seed=0, model=scen.bench_model(64))
    seeds = np.arange(500, 564)
    host = scen.build_scenarios(cl, model, plan, 64, seeds=seeds, churn=0.05, jitter=True)
    dev = scen.build_scenarios(cl, model, plan, 64, seeds=seeds, churn=0.05, jitter=True, host_events=False)
    rp = ScenarioReplayer(dev, window=64)
    rp.build()
    leave = rp.leave.view(64, -1).cpu().numpy().astype(bool)
    assert (leave == host.leave).all()
    rph = ScenarioReplayer(host, window=64)
    a, b = rp.run(16), rph.run(16)
    assert (a.cost.cpu().numpy() == b.cost.cpu().numpy()).all()


@pytest.fixture(scope="module")
def rebalance_cases():
    with open(os.path.join(HERE, "golden", "rebalance_cases.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("name", ["n64_w8", "c1_w4", "n64_nochange"])
def test_device_rebalance_loop(cuda_ready, rebalance_cases, name):
    """route R1 -> device membership events (+ aborts on departing GPUs) -> device triggers -> device
    allocate() on the churned pools -> abort on changed GPUs -> route R2; == the reference, scenario batch."""
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    case = rebalance_cases[name]
    want = case["scenarios"]
    seeds = [w["seed"] for w in want]
    full, model, plan, join_ids, _ = pool_for_case(case)
    W, r1, r2 = case["window"], case["r1"], case["r2"]
    kw = dict(seeds=seeds, jitter=False, join_pool=join_ids)
    base = scen.build_scenarios(full, model, plan, len(seeds), churn=0.0, **kw)
    ev = scen.build_scenarios(full, model, plan, len(seeds), churn=case["churn"], joins=case["joins"],
                              host_events=False, **kw)
    rp0 = ScenarioReplayer(base, window=W, max_requests=r1 + r2 + 4)
    a = rp0.run(r1, gpus=True)
    rp1 = ScenarioReplayer(ev, window=W, max_requests=r1 + r2 + 4)
    rp1.build()                                                    # device membership events
    S, G = rp1.S, rp1.G
    departed = rp1.leave.view(S, G).cpu().numpy().astype(bool) & ev.present0
    ab_leave = rp0.abort_on(departed)
    rp1.adopt_state(rp0)
    rp2, info = rp1.rebalance(cov_threshold=case["cov_threshold"])
    b = rp2.run(r2, gpus=True)
    rp2.raise_first_failure()
    gpus = np.concatenate([a.gpus.cpu().numpy(), b.gpus.cpu().numpy()], axis=1)
    cost = np.concatenate([a.cost.cpu().numpy(), b.cost.cpu().numpy()], axis=1)
    occ = rp2.occ.view(S, G).cpu().numpy()
    lo = rp2.lo_s.view(S, G).cpu().numpy()
    hi = rp2.hi_s.view(S, G).cpu().numpy()
    absent = rp2.leave.view(S, G).cpu().numpy().astype(bool)
    for s, w in enumerate(want):
        for r in range(r1 + r2):
            assert _hops(gpus[s, r].tolist()) == w["chains"][r]["hops"], (name, s, r)
            assert float(cost[s, r]) == hx(w["chains"][r]["cost"]), (name, s, r)
        assert DECISION[int(info["decision"][s])] == w["decision"][:2]
        assert info["changed"][s] == w["changed"]
        assert int(ab_leave[s]) == len(w["aborted_leave"])
        assert int(info["aborted"][s]) == len(w["aborted_rebalance"])
        assert occ[s].tolist() == w["occ"]
        got = sorted([g, int(lo[s, g]), int(hi[s, g])] for g in range(G) if not absent[s, g] and lo[s, g] <= hi[s, g])
        assert got == w["slices"]
