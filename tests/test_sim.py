"""Serving simulator (admission path with occupancy-dependent step time) vs the reference.

CPU: the oracle event loop reproduces the reference's MetricsReport and per-request latencies bit for bit.
GPU: ss_sim_warp (one warp per scenario, the same event order on device) does the same.
"""

import json
import os

import numpy as np
import pytest

from conftest import hx
from helpers_golden import plan_from_golden
from oracle import alloc_ref, sim_ref

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = ["c1_light", "c1_heavy", "c2_mid", "c2_amortized"]


@pytest.fixture(scope="module")
def sim_cases():
    with open(os.path.join(HERE, "golden", "sim_cases.json")) as fh:
        return json.load(fh)


def pool(case):
    from paper_2509_26182_b200 import scenarios as scen
    cl, model = scen.synthetic_cluster(case["n"], seed=0, model=scen.bench_model(case["L"]))
    d = alloc_ref.allocate(cl, model)
    d["objective"] = d["objective"].hex()
    d["per_k"] = [dict(r, z=r["z"].hex()) for r in d["per_k"]]
    plan = plan_from_golden(d)
    return scen.build_scenarios(cl, model, plan, 1, churn=0.0, jitter=False)


def trace_of(case):
    return [(hx(a), int(p), int(o)) for a, p, o in case["trace"]]


def report_hex(rep):
    return {k: (float(v).hex() if isinstance(v, float) else int(v)) for k, v in rep.items()}


@pytest.mark.parametrize("name", CASES)
def test_oracle_simulator_matches_reference(sim_cases, name):
    case = sim_cases[name]
    ss = pool(case)
    rep, lat, _ = sim_ref.simulate(ss.columns(0), ss.base_tau, ss.base_rtt, ss.token_cap, trace_of(case),
                                   amortize_rtt=case["amortize"], contention=case["contention"])
    assert report_hex(rep) == case["report"]
    assert [v.hex() for v in lat] == case["latencies"]
