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
CASES = ["c1_light", "c1_heavy", "c2_mid", "c2_amortized", "c4_light", "n192_wide"]


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


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_device_simulator_matches_reference(cuda_ready, sim_cases, name):
    """ss_sim_warp (<= 32 hosts per layer) or ss_sim_cta (wide pools: C4's k = 73, k = 172) vs the reference."""
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer, replay_mode
    c = sim_cases[name]
    base = pool(c)
    # two copies of the scenario in one launch: both must reproduce the reference
    ss = scen.ScenarioSet(base.layer_count, base.ids, base.base_rtt, base.base_tau, base.slice_lo, base.slice_hi,
                          np.arange(2), np.zeros((2, base.n_gpus), dtype=bool), False, token_cap=base.token_cap)
    mode = "warp" if replay_mode(ss, window=1) == "warp" else "blocks"
    rp = ScenarioReplayer(ss, window=1, mode=mode)
    t = trace_of(c)
    tr = (np.array([x[0] for x in t]), np.array([x[1] for x in t], dtype=np.int32),
          np.array([x[2] for x in t], dtype=np.int32))
    reps = rp.simulate([tr, tr], amortize_rtt=c["amortize"], contention=c["contention"])
    for rep in reps:
        lat = rep.pop("latencies")
        rep.pop("events")
        assert report_hex(rep) == c["report"], mode
        assert [v.hex() for v in lat] == c["latencies"], mode


def test_generate_trace_matches_reference_draws(sim_cases):
    from paper_2509_26182_b200.scenarios import generate_trace
    for c in sim_cases.values():
        a, p, o = generate_trace(c["rate"], c["duration"], seed=c["seed"], prompt_tokens=tuple(c["prompt"]),
                                 output_tokens=tuple(c["output"]))
        assert [[x.hex(), int(y), int(z)] for x, y, z in zip(a.tolist(), p, o)] == c["trace"]


def test_dropin_trace_api_matches_reference_draws(sim_cases, tmp_path):
    """sim.py:62-159 drop-ins: generate_trace Requests (ids, draws), JSON-lines round trip, nearest-rank percentile."""
    from paper_2509_26182_b200 import EmptySample, Request, generate_trace, load_trace, percentile, save_trace
    c = sim_cases["c2_mid"]
    tr = generate_trace(c["rate"], c["duration"], seed=c["seed"], prompt_tokens=tuple(c["prompt"]),
                        output_tokens=tuple(c["output"]))
    assert [[r.arrival_s.hex(), r.prompt_tokens, r.output_tokens] for r in tr] == c["trace"]
    assert tr[0].id == "r00000" and tr[-1].id == f"r{len(tr) - 1:05d}"
    path = str(tmp_path / "trace.jsonl")
    save_trace(list(reversed(tr)), path)
    assert load_trace(path) == tr
    assert percentile([5.0, 1.0, 3.0], 50) == 3.0 and percentile([5.0, 1.0, 3.0], 100) == 5.0
    assert percentile([2.0], 0.1) == 2.0
    with pytest.raises(EmptySample):
        percentile([], 50)
    with pytest.raises(ValueError):
        Request("x", 0.0, 0, 1)


def test_membership_event_validation():
    """MembershipEvent (membership.py:55-70): joins carry a GPU record (their id becomes gpu_id), leaves an id."""
    from paper_2509_26182_b200 import MembershipEvent
    from paper_2509_26182_b200.topology import GpuNode
    g = GpuNode(id="x", region="r", vram_bytes=1e10, flops=1e14)
    assert MembershipEvent(at_s=1.0, kind="join", gpu=g).gpu_id == "x"
    assert MembershipEvent(at_s=1.0, kind="leave", gpu_id="y").gpu is None
    for bad in (dict(kind="join"), dict(kind="leave"), dict(kind="move", gpu_id="y")):
        with pytest.raises(ValueError):
            MembershipEvent(at_s=0.0, **bad)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_run_simulation_dropin_matches_reference(cuda_ready, sim_cases, name):
    """The public run_simulation (sim.py:478-510) on the device vs the reference's MetricsReport, bit for bit."""
    from paper_2509_26182_b200 import Request, run_simulation
    from paper_2509_26182_b200 import scenarios as scen
    c = sim_cases[name]
    cl, model = scen.synthetic_cluster(c["n"], seed=0, model=scen.bench_model(c["L"]))
    d = alloc_ref.allocate(cl, model)
    d["objective"] = d["objective"].hex()
    d["per_k"] = [dict(r, z=r["z"].hex()) for r in d["per_k"]]
    plan = plan_from_golden(d)
    trace = [Request(f"r{i:05d}", a, p, o) for i, (a, p, o) in enumerate(trace_of(c))]
    rep = run_simulation(cl, model, plan, trace[::-1], amortize_rtt=c["amortize"],
                         contention_exponent=c["contention"])
    assert report_hex(rep.to_dict()) == c["report"]


@pytest.mark.gpu
def test_device_simulator_on_jittered_scenarios(cuda_ready):
    """Jittered C2-shaped scenarios: the per-scenario RTT matrices come from ss_scenario_rtt on device; they must
    equal ScenarioSet.scenario_rtt bit for bit, and each scenario's MetricsReport must match the oracle event loop."""
    import torch
    from paper_2509_26182_b200 import _native as N, scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    cl, model = scen.synthetic_cluster(64, seed=0, model=scen.bench_model(64))
    d = alloc_ref.allocate(cl, model)
    d["objective"] = d["objective"].hex()
    d["per_k"] = [dict(r, z=r["z"].hex()) for r in d["per_k"]]
    plan = plan_from_golden(d)
    S = 3
    ss = scen.build_scenarios(cl, model, plan, S, seeds=[11, 12, 13], churn=0.0, jitter=True)
    rp = ScenarioReplayer(ss, window=1, mode="warp")
    G = ss.n_gpus
    out = torch.empty(S * G * G, dtype=torch.float64, device="cuda")
    N.check(N.lib().ss_scenario_rtt(S, G, N.ptr(rp.base_rtt), N.ptr(rp.seeds), N.ptr(out), None), "ss_scenario_rtt")
    got = out.cpu().numpy().reshape(S, G, G)
    for s in range(S):
        assert np.array_equal(got[s], ss.scenario_rtt(s))
    traces = [scen.generate_trace(120.0, 1.0, seed=s, prompt_tokens=(500, 20000), output_tokens=(8, 32))
              for s in (11, 12, 13)]
    reps = rp.simulate(traces)
    for s in range(S):
        tr = traces[s]
        rep, lat, _ = sim_ref.simulate(ss.columns(s), ss.base_tau, ss.scenario_rtt(s), ss.token_cap,
                                       list(zip(tr[0].tolist(), tr[1].tolist(), tr[2].tolist())))
        mine = dict(reps[s])
        assert [v.hex() for v in mine.pop("latencies")] == [v.hex() for v in lat], s
        mine.pop("events")
        assert report_hex(mine) == report_hex(rep), s


@pytest.mark.gpu
@pytest.mark.parametrize("n,L", [(24, 32), (36, 24), (48, 24)])
def test_multiwarp_simulator_widths_vs_oracle(cuda_ready, n, L):
    """sim_mw_kernel at 2 / 3 / 4 warps (12, 23, 30 hosts per column) vs the oracle event loop, report and
    per-request latencies bit for bit (jittered RTT, KV pressure from long prompts)."""
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    cl, model = scen.synthetic_cluster(n, seed=0, model=scen.bench_model(L))
    d = alloc_ref.allocate(cl, model)
    d["objective"] = d["objective"].hex()
    d["per_k"] = [dict(r, z=r["z"].hex()) for r in d["per_k"]]
    plan = plan_from_golden(d)
    ss = scen.build_scenarios(cl, model, plan, 2, seeds=[5, 6], churn=0.0, jitter=True)
    rp = ScenarioReplayer(ss, window=1, mode="warp")
    traces = [scen.generate_trace(200.0, 0.8, seed=s, prompt_tokens=(1000, 40000), output_tokens=(4, 24))
              for s in (5, 6)]
    reps = rp.simulate(traces)
    for s in range(2):
        tr = traces[s]
        rep, lat, _ = sim_ref.simulate(ss.columns(s), ss.base_tau, ss.scenario_rtt(s), ss.token_cap,
                                       list(zip(tr[0].tolist(), tr[1].tolist(), tr[2].tolist())))
        mine = dict(reps[s])
        assert [v.hex() for v in mine.pop("latencies")] == [v.hex() for v in lat], s
        mine.pop("events")
        assert report_hex(mine) == report_hex(rep), s


@pytest.mark.gpu
def test_device_simulator_matrix_mode_vs_oracle(cuda_ready):
    """160 jittered C2 scenarios (more than SMs -> the simulator stages each RTT matrix): a sample vs the oracle."""
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    cl, model = scen.synthetic_cluster(64, seed=0, model=scen.bench_model(64))
    d = alloc_ref.allocate(cl, model)
    d["objective"] = d["objective"].hex()
    d["per_k"] = [dict(r, z=r["z"].hex()) for r in d["per_k"]]
    plan = plan_from_golden(d)
    S = 160
    ss = scen.build_scenarios(cl, model, plan, S, seeds=list(range(S)), churn=0.0, jitter=True)
    rp = ScenarioReplayer(ss, window=1, mode="warp")
    traces = [scen.generate_trace(100.0, 0.6, seed=s, prompt_tokens=(500, 20000), output_tokens=(4, 24))
              for s in range(S)]
    reps = rp.simulate(traces)
    for s in range(0, S, 40):
        tr = traces[s]
        rep, lat, _ = sim_ref.simulate(ss.columns(s), ss.base_tau, ss.scenario_rtt(s), ss.token_cap,
                                       list(zip(tr[0].tolist(), tr[1].tolist(), tr[2].tolist())))
        mine = dict(reps[s])
        assert [v.hex() for v in mine.pop("latencies")] == [v.hex() for v in lat], s
        mine.pop("events")
        assert report_hex(mine) == report_hex(rep), s


@pytest.mark.gpu
def test_baseline_plan_matches_reference(cuda_ready):
    """sim.py:513-553 baseline_plan (water-fill and rounding on device) vs the reference's plans."""
    from paper_2509_26182_b200 import baseline_plan, plan_to_dict, scenarios as scen
    with open(os.path.join(HERE, "golden", "baseline_cases.json")) as fh:
        cases = json.load(fh)
    for name, c in cases.items():
        cl, model = scen.synthetic_cluster(c["n"], seed=c["seed"], model=scen.bench_model(c["L"]))
        d = plan_to_dict(baseline_plan(cl, model))
        d["objective"] = float(d["objective"]).hex()
        assert d == c["plan"], name


def test_latency_model_is_the_device_tau_law():
    """LatencyModel (sim.py:161-186) == the tau every device replay applies: base_tau[g] * occpow[occ]."""
    from paper_2509_26182_b200 import LatencyModel, scenarios as scen
    from paper_2509_26182_b200.batched import occ_power_table
    ss = pool({"n": 16, "L": 32})
    cl, model = scen.synthetic_cluster(16, seed=0, model=scen.bench_model(32))
    for e in (1.0, 0.5, 2.0):
        lm = LatencyModel(model, cl, contention_exponent=e)
        pw = occ_power_table(8, e)
        for g, gid in enumerate(ss.ids):
            assert lm.base_s(gid) == ss.base_tau[g]
            for o in range(8):
                assert lm.published(gid, 1, o) == ss.base_tau[g] * pw[o]
            assert lm.executing(gid, 0) == lm.executing(gid, 1) == ss.base_tau[g] * 1.0 ** e
