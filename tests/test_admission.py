"""Admission path vs the reference (tests/golden/admission_cases.json).

CPU: the oracle (KV-headroom exclusion as +inf latency, strict FIFO drain) reproduces the reference
simulator's admission decisions, chains and costs bit for bit.  GPU: ss_admission_warp does the same on device.
"""

import json
import os

import numpy as np
import pytest

from conftest import hx
from helpers_golden import plan_from_golden
from oracle import admission_ref, alloc_ref, chain_ref

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = ["c1", "c1_tight", "c2", "c2_light", "c2_tight"]


@pytest.fixture(scope="module")
def admission_cases():
    with open(os.path.join(HERE, "golden", "admission_cases.json")) as fh:
        return json.load(fh)


def _hops(row):
    out, start = [], 1
    for layer in range(2, len(row) + 1):
        if row[layer - 1] != row[layer - 2]:
            out.append([row[layer - 2], start, layer - 1])
            start = layer
    out.append([row[-1], start, len(row)])
    return out


def scenario_set(case, seeds):
    from paper_2509_26182_b200 import scenarios as scen
    cl, model = scen.synthetic_cluster(case["n"], seed=0, model=scen.bench_model(case["L"]))
    d = alloc_ref.allocate(cl, model)
    d["objective"] = d["objective"].hex()
    d["per_k"] = [dict(r, z=r["z"].hex()) for r in d["per_k"]]
    plan = plan_from_golden(d)
    return scen.build_scenarios(cl, model, plan, len(seeds), seeds=seeds, churn=0.0, jitter=False)


def check(case, want, admitted, queue_left, kv, occ):
    for i, w in enumerate(want["admitted"]):
        got = admitted[i]
        if w is None:
            assert got is None, i
            continue
        step, gpus, cost = got
        assert step == w["step"], i
        assert _hops(gpus) == w["hops"], i
        assert cost == hx(w["cost"]), i
    assert list(queue_left) == want["queue_left"]
    assert [int(x) for x in kv] == want["kv"]
    assert [int(x) for x in occ] == want["occ"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_admission_matches_reference(admission_cases, name):
    from paper_2509_26182_b200 import scenarios as scen
    case = admission_cases[name]
    seeds = [w["seed"] for w in case["scenarios"]]
    ss = scenario_set(case, seeds)
    for s, want in enumerate(case["scenarios"]):
        toks = [scen.request_tokens(want["seed"], i, case["tok_lo"], case["tok_hi"]) for i in range(case["steps"])]
        got = admission_ref.admission_replay(ss.columns(s), ss.base_tau, ss.scenario_rtt(s), ss.token_cap, toks,
                                             case["steps"], case["window"],
                                             chain_ref.occ_power_table(case["steps"] + 4))
        check(case, want, *got)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_admission_matches_reference(cuda_ready, admission_cases, name):
    from paper_2509_26182_b200.batched import ScenarioReplayer
    case = admission_cases[name]
    seeds = [w["seed"] for w in case["scenarios"]]
    ss = scenario_set(case, seeds)
    rp = ScenarioReplayer(ss, window=case["window"], mode="warp")
    out = rp.admit(case["steps"], tok_lo=case["tok_lo"], tok_hi=case["tok_hi"], gpus=True)
    rp.raise_first_failure()
    step, cost, gpus = out["step"].cpu().numpy(), out["cost"].cpu().numpy(), out["gpus"].cpu().numpy()
    kv, occ = out["kv"].cpu().numpy(), out["occ"].cpu().numpy()
    for s, want in enumerate(case["scenarios"]):
        admitted = [None if step[s, i] < 0 else (int(step[s, i]), gpus[s, i].tolist(), float(cost[s, i]))
                    for i in range(case["steps"])]
        queue_left = [i for i in range(case["steps"]) if step[s, i] < 0]
        check(case, want, admitted, queue_left, kv[s], occ[s])


@pytest.mark.gpu
@pytest.mark.parametrize("n,L", [(24, 32), (36, 24), (48, 24)])
def test_device_admission_widths_vs_oracle(cuda_ready, n, L):
    """admission_warp_kernel at 2 / 3 / 4 warps (12, 23, 30 hosts per column) vs the oracle, under KV pressure."""
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    case = {"n": n, "L": L}
    seeds, steps, window, lo, hi = [3, 4], 64, 12, 30000, 90000
    ss = scenario_set(case, seeds)
    rp = ScenarioReplayer(ss, window=window, mode="warp")
    out = rp.admit(steps, tok_lo=lo, tok_hi=hi, gpus=True)
    rp.raise_first_failure()
    step, cost, gpus = out["step"].cpu().numpy(), out["cost"].cpu().numpy(), out["gpus"].cpu().numpy()
    kv, occ = out["kv"].cpu().numpy(), out["occ"].cpu().numpy()
    for s, seed in enumerate(seeds):
        toks = [scen.request_tokens(seed, i, lo, hi) for i in range(steps)]
        want_adm, want_q, want_kv, want_occ = admission_ref.admission_replay(
            ss.columns(s), ss.base_tau, ss.scenario_rtt(s), ss.token_cap, toks, steps, window,
            chain_ref.occ_power_table(steps + 4))
        got = [None if step[s, i] < 0 else (int(step[s, i]), gpus[s, i].tolist(), float(cost[s, i]))
               for i in range(steps)]
        assert got == want_adm, s
        assert [i for i in range(steps) if step[s, i] < 0] == list(want_q)
        assert [int(x) for x in kv[s]] == [int(x) for x in want_kv]
        assert [int(x) for x in occ[s]] == [int(x) for x in want_occ]


@pytest.mark.gpu
def test_device_admission_matrix_mode_vs_oracle(cuda_ready):
    """160 C2 scenarios (more than SMs -> matrix mode): a sample vs the oracle."""
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    seeds, steps, window, lo, hi = list(range(100, 260)), 48, 12, 30000, 90000
    ss = scenario_set({"n": 64, "L": 64}, seeds)
    rp = ScenarioReplayer(ss, window=window, mode="warp")
    out = rp.admit(steps, tok_lo=lo, tok_hi=hi, gpus=True)
    rp.raise_first_failure()
    step, cost, gpus = out["step"].cpu().numpy(), out["cost"].cpu().numpy(), out["gpus"].cpu().numpy()
    for s in range(0, len(seeds), 16):
        toks = [scen.request_tokens(seeds[s], i, lo, hi) for i in range(steps)]
        want_adm, want_q, _, _ = admission_ref.admission_replay(
            ss.columns(s), ss.base_tau, ss.scenario_rtt(s), ss.token_cap, toks, steps, window,
            chain_ref.occ_power_table(steps + 4))
        got = [None if step[s, i] < 0 else (int(step[s, i]), gpus[s, i].tolist(), float(cost[s, i]))
               for i in range(steps)]
        assert got == want_adm, s
