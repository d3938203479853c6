"""C2 stream golden (L64/N64 seed 0, k=17, one scenario, W=64).

tests/golden/c2_stream.json holds per-1,000-op digests of the reference's own first 50,000 C2 ops
(tests/golden/make_c2_stream_golden.py).  Here the oracle restatement is pinned against the first two
blocks; tests/test_gpu_c2_stream.py checks every block on the device.
"""

import json
import os

import numpy as np
import pytest

from helpers_golden import stream_digests

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "c2_stream.json")


@pytest.fixture(scope="module")
def c2_stream():
    with open(GOLDEN) as f:
        return json.load(f)


def c2_scenario():
    from oracle import alloc_ref
    from paper_2509_26182_b200 import scenarios as scen
    from helpers_golden import plan_from_golden
    cl, model = scen.synthetic_cluster(64, seed=0, model=scen.bench_model(64))
    d = dict(alloc_ref.allocate(cl, model))
    d["objective"] = d["objective"].hex()
    d["per_k"] = [dict(r, z=r["z"].hex()) for r in d["per_k"]]
    plan = plan_from_golden(d)
    return cl, model, plan, scen.build_scenarios(cl, model, plan, 1, churn=0.0, jitter=False)


def test_c2_stream_fixture_shape(c2_stream):
    assert c2_stream["routes"] == 50_000 and c2_stream["block"] == 1_000
    assert len(c2_stream["digests"]) == 50 and c2_stream["k"] == 17
    assert sum(c2_stream["final_occ"]) > 0


def test_oracle_matches_reference_c2_stream_prefix(c2_stream):
    from oracle import chain_ref
    from paper_2509_26182_b200.scenarios import splitmix64
    _, _, plan, ss = c2_scenario()
    assert plan.replication_count == c2_stream["k"]
    n = 2 * c2_stream["block"]
    gpus, costs, _, _ = chain_ref.replay(ss.columns(0), ss.base_tau, ss.scenario_rtt(0), n, c2_stream["window"],
                                         chain_ref.occ_power_table(n + 4))
    M = (1 << 64) - 1
    hashes = [sum(splitmix64((l << 32) | g) for l, g in enumerate(row)) & M for row in gpus]
    hashes = np.array([h - (1 << 64) if h >= 1 << 63 else h for h in hashes], dtype=np.int64)
    assert stream_digests(hashes, costs, c2_stream["block"]) == c2_stream["digests"][:2]
