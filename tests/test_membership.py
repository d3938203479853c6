"""Membership churn vs the reference's MembershipManager (tests/golden/membership_cases.json).

CPU: the scenario generator's on_leave / on_join (bottleneck_layer) slices, the oracle replay on the churned
state, and the oracle evaluate_triggers are bit-identical to the reference's.  GPU: ss_scenario_membership and
ss_membership_triggers (device) reproduce the same states and decisions, and the device replay routes them
exactly like the reference ChainRouter.
"""

import json
import os

import numpy as np
import pytest

from conftest import hx
from helpers_membership import pool_for_case, trigger_inputs
from oracle import chain_ref, membership_ref

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = ["c1j", "n64j", "n256j", "n64j_lowthr"]
ALL_ROUTED = CASES + ["n64j_hole_filled"]      # hole_filled adds departures the generator does not draw


@pytest.fixture(scope="module")
def membership_cases():
    with open(os.path.join(HERE, "golden", "membership_cases.json")) as fh:
        return json.load(fh)


def _scenarios(case, seeds, host_events=True):
    from paper_2509_26182_b200 import scenarios as scen
    full, model, plan, join_ids, order = pool_for_case(case)
    ss = scen.build_scenarios(full, model, plan, len(seeds), seeds=seeds, churn=case["churn"], jitter=False,
                              join_pool=join_ids, joins=case["joins"], host_events=host_events)
    return full, model, plan, order, ss


def _hops(cols, picks):
    out, start = [], 1
    for layer in range(2, len(picks) + 1):
        if picks[layer - 1] != picks[layer - 2]:
            out.append([picks[layer - 2], start, layer - 1])
            start = layer
    out.append([picks[-1], start, len(picks)])
    return out


@pytest.mark.parametrize("name", CASES)
def test_generator_events_match_reference(membership_cases, name):
    case = membership_cases[name]
    seeds = [s["seed"] for s in case["scenarios"]]
    _, _, _, _, ss = _scenarios(case, seeds)
    for s, want in enumerate(case["scenarios"]):
        lo, hi = ss.slices(s)
        got = sorted([g, int(lo[g]), int(hi[g])] for g in range(ss.n_gpus) if not ss.leave[s, g] and lo[g] <= hi[g])
        assert got == want["slices"], (name, s)
        assert sorted(np.nonzero(ss.leave[s] & ss.present0)[0].tolist()) == want["left"]
        assert [[g, int(lo[g]), int(hi[g])] for g in want["joined"]] == want["join_slices"]


def golden_state(ss, want):
    """Scenario state straight from the golden event lists (left, joined + their slices)."""
    absent = ~ss.present0.copy()
    lo, hi = ss.slice_lo.astype(np.int32).copy(), ss.slice_hi.astype(np.int32).copy()
    lo[absent], hi[absent] = 0, -1
    for g in want["left"]:
        absent[g] = True
        lo[g], hi[g] = 0, -1
    for g, a, b in want["join_slices"]:
        absent[g] = False
        lo[g], hi[g] = a, b
    return absent, lo, hi


@pytest.mark.parametrize("name", ALL_ROUTED)
def test_oracle_replay_and_triggers_on_churned_state(membership_cases, name):
    case = membership_cases[name]
    seeds = [s["seed"] for s in case["scenarios"]]
    full, model, plan, order, ss = _scenarios(case, seeds)
    R = case["routes"]
    thr = case["cov_threshold"]
    for s, want in enumerate(case["scenarios"]):
        absent, lo, hi = golden_state(ss, want)
        cols = [np.nonzero(~absent & (lo <= l) & (hi >= l))[0] for l in range(1, ss.layer_count + 1)]
        picks, costs, occ, _ = chain_ref.replay(cols, ss.base_tau, ss.scenario_rtt(s), R, None,
                                                chain_ref.occ_power_table(R + 4))
        for r in range(R):
            assert _hops(cols, picks[r]) == want["chains"][r]["hops"], (name, s, r)
            assert costs[r] == hx(want["chains"][r]["cost"]), (name, s, r)
        assert occ.tolist() == want["occ"]
        gpus, slices, kv, occupancy = trigger_inputs(full, ss.ids, order, want["left"], want["joined"], lo, hi, occ,
                                                     ss.present0)
        scope, reason, cov, unc, loads = membership_ref.evaluate_triggers(ss.layer_count, gpus, slices, kv,
                                                                          occupancy, cov_threshold=thr)
        assert [scope, reason, cov.hex(), list(unc)] == want["decision"]
        assert [v.hex() for v in loads] == want["loads"]


def test_uncovered_trigger(membership_cases):
    case = membership_cases["n64j_hole"]
    want = case["scenarios"][0]
    full, model, plan, order, ss = _scenarios(case, [want["seed"]])
    lo, hi = ss.slices(0)
    left = sorted(set(np.nonzero(ss.leave[0] & ss.present0)[0].tolist())
                  | {g for g in range(ss.n_gpus) if ss.present0[g] and lo[g] <= case["hole_layer"] <= hi[g]})
    lo, hi = lo.copy(), hi.copy()
    lo[left], hi[left] = 0, -1
    gpus, slices, kv, occupancy = trigger_inputs(full, ss.ids, order, left, want["joined"], lo, hi,
                                                 np.zeros(ss.n_gpus, dtype=np.int64), ss.present0)
    scope, reason, cov, unc, _ = membership_ref.evaluate_triggers(ss.layer_count, gpus, slices, kv, occupancy)
    assert [scope, reason, cov.hex(), list(unc)] == want["decision"]


@pytest.fixture(scope="module")
def rebalance_cases():
    with open(os.path.join(HERE, "golden", "rebalance_cases.json")) as fh:
        return json.load(fh)


def oracle_rebalance_flow(case, want):
    """The oracle's rebalance loop for one golden scenario (oracle/rebalance_ref.py)."""
    from oracle import alloc_ref, rebalance_ref
    from paper_2509_26182_b200 import scenarios as scen
    full, model, plan, join_ids, order = pool_for_case(case)
    ss = scen.build_scenarios(full, model, plan, 1, seeds=[want["seed"]], churn=case["churn"], jitter=False,
                              join_pool=join_ids, joins=case["joins"])
    L, W, r1, r2 = case["L"], case["window"], case["r1"], case["r2"]
    rtt = ss.scenario_rtt(0)
    occpow = chain_ref.occ_power_table(W + 4)
    absent0 = ~ss.present0
    cols = rebalance_ref.columns_of(absent0, ss.slice_lo, ss.slice_hi, L)
    picks1, costs1, occ, live = chain_ref.replay(cols, ss.base_tau, rtt, r1, W, occpow)
    first = r1 - len(live)
    absent, lo, hi = ss.leave[0].copy(), ss.slice_lo_s[0].copy(), ss.slice_hi_s[0].copy()
    left = np.nonzero(ss.leave[0] & ss.present0)[0].tolist()
    joined = want["joined"]
    ab_leave = []
    for g in sorted(left):
        ab_leave += [first + j for j in rebalance_ref.abort(live, occ, [g])]
    gpus, slices, kv, occupancy = trigger_inputs(full, ss.ids, order, left, joined, lo, hi, occ, ss.present0)
    scope, reason, cov, _, _ = membership_ref.evaluate_triggers(L, gpus, slices, kv, occupancy,
                                                                cov_threshold=case["cov_threshold"])
    changed, ab_reb = [], []
    if scope == "global":
        pos = {g: i for i, g in enumerate(ss.ids)}
        d = alloc_ref.allocate(rebalance_ref.churned_cluster(full, ss.ids, absent), model)
        lo1, hi1, _ = rebalance_ref.plan_slices(d, pos, ss.n_gpus)
        changed = rebalance_ref.changed_gpus(lo, hi, lo1, hi1)
        ab_reb = [first + j for j in rebalance_ref.abort(live, occ, changed)]
        lo, hi = lo1, hi1
    cols2 = rebalance_ref.columns_of(absent, lo, hi, L)
    picks2, costs2, occ, live = chain_ref.replay(cols2, ss.base_tau, rtt, r2, W, occpow, occ=occ, start=r1, live=live)
    return dict(picks=picks1 + picks2, costs=costs1 + costs2, occ=occ, decision=[scope, reason, cov.hex()],
                changed=changed, ab_leave=ab_leave, ab_reb=ab_reb, lo=lo, hi=hi, absent=absent)


@pytest.mark.parametrize("name", ["n64_w8", "c1_w4", "n64_nochange"])
def test_oracle_rebalance_loop_matches_reference(rebalance_cases, name):
    case = rebalance_cases[name]
    for want in case["scenarios"]:
        got = oracle_rebalance_flow(case, want)
        for r, row in enumerate(got["picks"]):
            assert _hops(None, row) == want["chains"][r]["hops"], (name, want["seed"], r)
            assert got["costs"][r] == hx(want["chains"][r]["cost"]), (name, want["seed"], r)
        assert got["decision"] == want["decision"]
        assert got["changed"] == want["changed"]
        assert sorted(got["ab_leave"]) == sorted(want["aborted_leave"])
        assert got["ab_reb"] == want["aborted_rebalance"]
        assert got["occ"].tolist() == want["occ"]
        slices = sorted([g, int(got["lo"][g]), int(got["hi"][g])] for g in range(len(got["lo"]))
                        if not got["absent"][g] and got["lo"][g] <= got["hi"][g])
        assert slices == want["slices"]
