"""Wire formats against the reference's own JSON text (tests/golden/wire_cases.json).

CPU: plan JSON round trip (load -> save reproduces the reference text byte for byte).
GPU: device allocate -> save_plan text, and device replay -> chains_from_replay -> chains_to_json, equal to the
reference's ``swarmsched route --json`` output for the same pool.
"""

import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def wire_cases():
    with open(os.path.join(HERE, "golden", "wire_cases.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_plan_json_round_trip(tmp_path, wire_cases, name):
    from paper_2509_26182_b200.wire import load_plan, save_plan
    src = tmp_path / "ref.json"
    src.write_text(wire_cases[name]["plan_json"])
    plan = load_plan(str(src))
    dst = tmp_path / "ours.json"
    save_plan(plan, str(dst))
    assert dst.read_text() == wire_cases[name]["plan_json"]


def test_load_plan_rejects_malformed(tmp_path):
    from paper_2509_26182_b200.wire import load_plan
    p = tmp_path / "bad.json"
    p.write_text('{"k": 1}')
    with pytest.raises(ValueError, match="not a valid plan file"):
        load_plan(str(p))


def test_chains_from_replay_merges_hops():
    from paper_2509_26182_b200.wire import chains_from_replay, chains_to_json
    ids = ["a", "b", "c"]
    chains = chains_from_replay(ids, np.array([[0, 0, 1, 1, 0], [2, 2, 2, 2, 2]]), np.array([1.5, 0.25]))
    assert [(h.gpu_id, h.start_layer, h.end_layer) for h in chains[0].hops] == [("a", 1, 2), ("b", 3, 4), ("a", 5, 5)]
    assert [(h.gpu_id, h.start_layer, h.end_layer) for h in chains[1].hops] == [("c", 1, 5)]
    payload = json.loads(chains_to_json(chains))
    assert payload["chains"][0]["cost_s"] == 1.5 and payload["chains"][1]["hops"][0]["gpu_id"] == "c"


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_device_path_reproduces_reference_json(cuda_ready, tmp_path, wire_cases, name):
    from paper_2509_26182_b200 import allocate, scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    from paper_2509_26182_b200.wire import chains_from_replay, chains_to_json, save_plan
    c = wire_cases[name]
    cl, model = scen.synthetic_cluster(c["n"], seed=c["seed"], model=scen.bench_model(c["L"]))
    plan = allocate(cl, model)
    out = tmp_path / "plan.json"
    save_plan(plan, str(out))
    assert out.read_text() == c["plan_json"]
    ss = scen.build_scenarios(cl, model, plan, 1, churn=0.0, jitter=False)
    for mode in ("warp", "slots", "blocks"):
        rp = ScenarioReplayer(ss, window=-1, max_requests=c["requests"] + 4, mode=mode)
        res = rp.run(c["requests"], gpus=True)
        rp.raise_first_failure()
        chains = chains_from_replay(ss.ids, res.gpus.cpu().numpy()[0], res.cost.cpu().numpy()[0])
        assert chains_to_json(chains) + "\n" == c["route_json"], mode


def test_layer_load_helpers_known_values():
    """perfmap.py:73-114 exports: blend, zero denominators, population CoV (known answers)."""
    import math
    from paper_2509_26182_b200 import LayerLoad, layer_load, layer_load_cov
    assert layer_load(2.0, 1.0, 8.0, 4.0) == 0.5 * 0.25 + 0.5 * 0.25
    assert layer_load(2.0, 1.0, 0.0, 0.0, mix_alpha=0.3) == 0.0
    assert layer_load(2.0, 3.0, 4.0, 6.0, mix_alpha=1.0) == 0.5
    with pytest.raises(ValueError):
        layer_load(1.0, 1.0, 1.0, 1.0, mix_alpha=1.5)
    assert layer_load_cov([]) == 0.0 and layer_load_cov([0.0, 0.0]) == 0.0
    assert layer_load_cov([1.0, 3.0]) == 0.5
    assert layer_load_cov([2.0, 2.0, 2.0]) == 0.0
    assert math.isclose(layer_load_cov([1.0, 2.0, 3.0, 4.0]), math.sqrt(1.25) / 2.5, rel_tol=0, abs_tol=0)
    assert LayerLoad(3, 0.2, 0.6, 0.25).value == 0.25 * 0.2 + 0.75 * 0.6


@pytest.mark.parametrize("name,kind", [("io_cluster_bench16.json", "cluster"), ("io_cluster_hand.json", "cluster"),
                                       ("io_model_bench32.json", "model")])
def test_cluster_and_model_files_round_trip_reference_text(tmp_path, name, kind):
    """topology.py:180-288 file formats: reference-written files load through the drop-in and save back to the
    same text (ms on disk, s in memory; asymmetric links and a custom cross-region RTT included)."""
    from paper_2509_26182_b200 import load_cluster, load_model, save_cluster, save_model
    src = os.path.join(os.path.dirname(__file__), "golden", name)
    out = str(tmp_path / name)
    if kind == "cluster":
        snap = load_cluster(src)
        save_cluster(snap, out)
        if name == "io_cluster_hand.json":
            assert snap.rtt_s("a", "b") == 0.0015 and snap.rtt_s("b", "a") == 0.0025
            assert snap.rtt_s("c", "a") == 0.031 and snap.rtt_s("b", "c") == 0.042
            assert snap.gpu("a").ram_token_capacity == 50_000 and snap.regions == frozenset({"east", "west"})
    else:
        save_model(load_model(src), out)
    assert open(out).read() == open(src).read()
