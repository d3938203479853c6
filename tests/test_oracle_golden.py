"""Pin the CPU oracle against the reference's golden vectors (CPU only).

Every fixture under tests/golden was produced by the unmodified reference
(tests/golden/make_golden.py).  These tests prove the oracle restatement is
bit-identical to it, so the GPU parity tests can use the oracle on inputs the
fixtures do not cover.
"""

import math
import random

import numpy as np
import pytest

from conftest import hx, untag
from helpers_golden import (case_latencies, case_links, cluster_from_alloc_case, hops_from_gpus,
                            replay_inputs)
from oracle import alloc_ref, chain_ref, waterfill_ref


def test_router_cases_bit_exact(router_cases):
    n_ok = n_tie_cols = 0
    for i, case in enumerate(router_cases):
        got = chain_ref.select(case_latencies(case), case["L"], case_links(case), frozenset(case["exclude"]))
        want = case["result"]
        if want["status"] == "ok":
            assert got[0] == "ok", i
            assert [list(h) for h in got[1]] == want["hops"], i
            assert got[2] == hx(want["cost"]), i        # bit-exact
            n_ok += 1
        elif want["status"] == "uncovered":
            assert got == ("uncovered", want["layer"]), i
        else:
            assert got == ("no_path",), i
    assert n_ok > 600


@pytest.mark.parametrize("name", ["c1", "c1_tie", "n32_tie", "rt16", "c2", "c4_s11", "c4_s12"])
def test_replays_bit_exact(router_replays, name):
    rep = router_replays[name]
    plan = rep["plan"] if "plan" in rep else router_replays["c4_plan"]
    cols, base, rtt, ids = replay_inputs(rep, plan)
    n = len(rep["routes"])
    W = rep["window"]
    size = n + 2 if W is None else max(W, 1) + 2
    gpus, costs, occ, _ = chain_ref.replay(cols, base, rtt, n, W, chain_ref.occ_power_table(size))
    for r in range(n):
        assert hops_from_gpus(gpus[r]) == rep["routes"][r]["hops"], (name, r)
        assert costs[r] == hx(rep["routes"][r]["cost"]), (name, r)
    gone = set(rep.get("leave", []))
    want_occ = [o for g, o in enumerate(rep["final_occ"])]
    assert [int(occ[g]) if g not in gone else 0 for g in range(len(ids))] == want_occ


def test_demo_feedback_map(router_replays):
    rec = router_replays["demo_feedback"]
    ids = ["a-back", "a-front", "b-back", "b-front"]
    links = [("a-front", "a-back", 0.001), ("b-front", "b-back", 0.001),
             ("a-front", "b-back", 0.008), ("b-front", "a-back", 0.008)]
    rtt = chain_ref.dense_rtt(sorted(links), ids)
    cols = [np.array([1, 3])] * 3 + [np.array([0, 2])] * 3
    gpus, costs, occ, _ = chain_ref.replay(cols, np.full(4, 0.002), rtt, 6, None, chain_ref.occ_power_table(8))
    for r, want in enumerate(rec["routes"]):
        assert [[ids[g], a, b] for g, a, b in hops_from_gpus(gpus[r])] == want["hops"]
        assert costs[r] == hx(want["cost"])
    assert {ids[g]: int(occ[g]) for g in range(4)} == rec["occ"]


def test_stage_counts(phase1_cases):
    for i, case in enumerate(phase1_cases["stage_counts"]):
        got = alloc_ref.stage_counts(case["caps"], case["L"], case["kmax"])
        want = {int(k): (v[0], tuple(tuple(g) for g in v[1])) for k, v in case["sols"].items()}
        assert got == want, i


def _plan_floats(d):
    d = dict(d)
    d["objective"] = d["objective"].hex() if isinstance(d["objective"], float) else d["objective"]
    d["per_k"] = [dict(r, z=r["z"].hex() if isinstance(r["z"], float) else r["z"]) for r in d["per_k"]]
    return d


def test_allocate(phase1_cases):
    for rec in phase1_cases["allocate"]:
        cluster, model = cluster_from_alloc_case(rec)
        kw = {}
        if "alpha" in rec["kw"]:
            kw["alpha"] = hx(rec["kw"]["alpha"])
        if "params" in rec["kw"]:
            a, t, r = (hx(x) for x in rec["kw"]["params"])

            class P:
                alpha, t_comp_seconds, rtt_seconds = a, t, r
            kw["params"] = P
        try:
            got = _plan_floats(alloc_ref.allocate(cluster, model, **kw))
        except LookupError:
            got = None
        assert got == rec["plan"], rec["name"]


def test_objective(phase1_cases):
    from paper_2509_26182_b200 import scenarios as scen
    for rec in phase1_cases["objective"]:
        cl, m = scen.synthetic_cluster(rec["n"], seed=rec["seed"], model=scen.bench_model(rec["L"]))
        rg = cl.gpus_in_region(rec["region"])
        t, r = alloc_ref.objective([g.flops for g in rg], [g.id for g in rg], cl.rtt_s,
                                   m.flops_per_layer_per_token, m.layer_count, 128.0)
        assert (t, r) == (hx(rec["t_comp"]), hx(rec["rtt"]))


def test_waterfill(phase1_cases):
    for i, rec in enumerate(phase1_cases["waterfill"]):
        flops = [hx(f) for f in rec["flops"]]
        targets, level = waterfill_ref.water_level(flops, rec["caps"], rec["L"])
        want = [untag(t) for t in rec["targets"]]
        assert [type(t) for t in targets] == [type(t) for t in want], i
        assert list(targets) == want and level == hx(rec["level"]), i
        assert list(waterfill_ref.largest_remainder(targets, rec["caps"], rec["L"])) == rec["layers"], i


def test_rebalance(phase1_cases):
    for i, rec in enumerate(phase1_cases["rebalance"]):
        flops = [hx(f) for f in rec["flops"]]
        try:
            got = waterfill_ref.stage_lengths(flops, rec["caps"], rec["L"])
        except waterfill_ref.WaterfillError as exc:
            got = {"overflow": "RoundingOverflow", "infeasible": "InfeasibleCapacity"}[exc.kind]
        assert got == rec["lengths"], i


def test_cpython_sum_model_matches_builtin():
    """The explicit Neumaier model the CUDA kernels implement equals CPython's sum()."""
    rng = random.Random(4242)
    for case in range(20000):
        n = rng.randint(0, 12)
        items = []
        for _ in range(n):
            kind = rng.random()
            if kind < 0.3:
                items.append(rng.randint(0, 40))
            elif kind < 0.6:
                items.append(rng.uniform(0, 40))
            elif kind < 0.8:
                items.append(rng.uniform(1e-16, 1e-3) * rng.choice([1, 1e10]))
            else:
                items.append(rng.choice([0.1, 0.2, 0.3, 1e16, 1.0, 3.0]))
        want = sum(items)
        got = waterfill_ref.cpython_sum_model(items)
        assert type(got) is type(want) and (got == want or (math.isnan(got) and math.isnan(want))), (items, got, want)
