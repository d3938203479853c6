"""The drop-in MembershipManager (membership.py:129-421) on CPU vs the reference's, event for event.

tests/golden/membership_cases.json records the reference's manager after initialize(plan), on_leave / on_join of a
seeded event set and a few routes: the slices (and each join's bottleneck-layer slice), the uncovered layers, the
bottleneck layer, the per-layer loads, the CoV and the trigger decision.  The drop-in applies the same events to
the drop-in PerfMap, replays the reference's routed chains as select events (the routes themselves need the GPU
and are covered by tests/test_gpu_membership.py), and must reproduce every value bit for bit.
"""

import json
import os

import numpy as np
import pytest

from conftest import hx
from helpers_membership import pool_for_case

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = ["c1j", "n64j", "n256j", "n64j_lowthr", "n64j_hole", "n64j_hole_filled"]


@pytest.fixture(scope="module")
def membership_cases():
    with open(os.path.join(HERE, "golden", "membership_cases.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("name", CASES)
def test_dropin_manager_matches_reference(membership_cases, name):
    from paper_2509_26182_b200 import LatencyModel, MembershipManager, PerfMap, layer_capacity, scenarios as scen
    from paper_2509_26182_b200.router import PipelineChain
    from paper_2509_26182_b200.topology import ClusterSnapshot, LayerSlice
    case = membership_cases[name]
    full, model, plan, _, _ = pool_for_case(case)
    nb, L = case["n_base"], case["L"]
    base = ClusterSnapshot(gpus=tuple(full.gpus[:nb]), links=dict(full.links))
    ids = sorted(g.id for g in full.gpus)
    pos = {g: i for i, g in enumerate(ids)}
    by_id = {g.id: g for g in full.gpus}
    lo = np.zeros(len(ids), dtype=np.int32)
    hi = np.full(len(ids), -1, dtype=np.int32)
    for gid, sl in plan.gpu_slices().items():
        lo[pos[gid]], hi[pos[gid]] = sl.start_layer, sl.end_layer
    present = np.array([int(g[4:]) < nb for g in ids])
    token = np.array([by_id[g].ram_token_capacity for g in ids], dtype=np.int64)
    lcap = np.array([layer_capacity(by_id[g], model) for g in ids], dtype=np.int32)
    for want in case["scenarios"]:
        _, _, _, gen_left, joined, _ = scen.membership_events(want["seed"], lo, hi, present, token, lcap, L,
                                                              case["churn"], case["joins"])
        left = sorted(want["left"])                                 # + the hole cases' extra departures
        assert set(int(g) for g in gen_left) <= set(left)
        assert [int(g) for g in joined] == want["joined"]
        pm = PerfMap(ttl_s=4.5)
        mgr = MembershipManager(base, model, pm, cov_threshold=case["cov_threshold"])
        pm.latency_fn = LatencyModel(model, mgr, 1.0).published
        mgr.initialize(plan, 0.0)
        for g in left:
            mgr.on_leave(ids[g], 0.0)
        join_slices = []
        for g in joined:
            sl = mgr.on_join(by_id[ids[g]], 0.0)
            join_slices.append([int(g), sl.start_layer, sl.end_layer])
        assert join_slices == want["join_slices"]
        assert sorted([pos[gid], sl.start_layer, sl.end_layer] for gid, sl in mgr.slices.items()) == want["slices"]
        assert list(mgr.uncovered_layers()) == want["uncovered"]
        for ch in want["chains"]:                                   # the reference's routes as occupancy feedback
            hops = tuple(LayerSlice(ids[g], a, b) for g, a, b in ch["hops"])
            pm.on_chain_event(PipelineChain(hops, hx(ch["cost"])), "select", 0.0)
        assert [int(pm.occupancy(g)) if pm.is_registered(g) else 0 for g in ids] == want["occ"]
        loads = mgr.layer_loads()
        assert [v.hex() for v in loads] == want["loads"]
        dec = mgr.evaluate_triggers()
        assert [dec.scope, dec.reason, dec.load_cov.hex(), list(dec.uncovered)] == want["decision"]
        assert mgr.bottleneck_layer() == want["bottleneck_after"]
