#!/usr/bin/env python3
"""Membership-churn golden fixtures from the UNMODIFIED reference (build container only).

    python tests/golden/make_membership_golden.py

Per scenario, the event sequence is drawn by this repo's generator
(paper_2509_26182_b200.scenarios.membership_events: which plan GPUs leave, which
pool GPUs join, in which order); the reference's own MembershipManager then
applies it -- initialize(plan), on_leave(...), on_join(...) (membership.py:
270-357) -- and its ChainRouter routes on the resulting perf map
(router.py:247-257, W = inf), after which evaluate_triggers() / layer_loads()
(membership.py:359-396) read the occupancy.  Recorded: the slices after the
events, each join's slice, the chains (hops as pool indices + cost hex), final
occupancy, per-layer loads (hex), the CoV (hex) and the trigger decision.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, REPO)

import swarmsched as ref                                    # noqa: E402
from swarmsched.membership import MembershipManager          # noqa: E402
from swarmsched.sim import LatencyModel                      # noqa: E402

from paper_2509_26182_b200 import scenarios as scen          # noqa: E402  (event generator only)


def fx(v):
    return float(v).hex()


def case(n_base, n_join, L, seeds, churn, joins, routes, cov_threshold=0.5, hole_layer=None):
    model = ref.ModelSpec(f"bench-{L}l", L, 1.2e9, 2.8e10)
    full, model = ref.synthetic_cluster(n_base + n_join, seed=0, model=model,
                                        region_count=scen.default_region_count(n_base))
    base_gpus = full.gpus[:n_base]
    base = ref.ClusterSnapshot(gpus=base_gpus, links=dict(full.links))
    plan = ref.allocate(ref.ClusterSnapshot(gpus=base_gpus, links={p: v for p, v in full.links.items()
                                                                    if int(p[0][4:]) < n_base and
                                                                    int(p[1][4:]) < n_base}), model)
    ids = sorted(g.id for g in full.gpus)
    pos = {g: i for i, g in enumerate(ids)}
    by_id = {g.id: g for g in full.gpus}
    lo = np.zeros(len(ids), dtype=np.int32)
    hi = np.full(len(ids), -1, dtype=np.int32)
    for gid, sl in plan.gpu_slices().items():
        lo[pos[gid]], hi[pos[gid]] = sl.start_layer, sl.end_layer
    present = np.array([int(g[4:]) < n_base for g in ids])
    token = np.array([by_id[g].ram_token_capacity for g in ids], dtype=np.int64)
    lcap = np.array([ref.layer_capacity(by_id[g], model) for g in ids], dtype=np.int32)
    out = []
    for seed in seeds:
        _, _, _, left, joined, _ = scen.membership_events(seed, lo, hi, present, token, lcap, L, churn, joins)
        if hole_layer is not None:       # extra departures that empty one layer (uncovered trigger)
            left = sorted(set(left) | {g for g in range(len(ids)) if present[g] and lo[g] <= hole_layer <= hi[g]})
        pm = ref.PerfMap(ttl_s=4.5)
        mgr = MembershipManager(base, model, pm, cov_threshold=cov_threshold)
        pm.latency_fn = LatencyModel(model, mgr, 1.0).published
        mgr.initialize(plan, 0.0)
        for g in sorted(left):
            mgr.on_leave(ids[g], 0.0)
        join_slices = []
        for g in joined:
            sl = mgr.on_join(by_id[ids[g]], 0.0)
            join_slices.append([g, sl.start_layer, sl.end_layer])
        slices = {pos[gid]: [sl.start_layer, sl.end_layer] for gid, sl in mgr.slices.items()}
        router = ref.ChainRouter(pm, L)
        chains = []
        for _ in range(routes if not mgr.uncovered_layers() else 0):
            c = router.route(0.0)
            chains.append({"hops": [[pos[h.gpu_id], h.start_layer, h.end_layer] for h in c.hops], "cost": fx(c.cost_s)})
        occ = [int(pm.occupancy(g)) if pm.is_registered(g) else 0 for g in ids]
        dec = mgr.evaluate_triggers()
        loads = mgr.layer_loads()
        out.append({"seed": seed, "left": sorted(int(g) for g in left), "joined": [int(g) for g in joined],
                    "join_slices": join_slices, "slices": sorted([int(g), a, b] for g, (a, b) in slices.items()),
                    "uncovered": list(mgr.uncovered_layers()), "bottleneck_after": mgr.bottleneck_layer(),
                    "chains": chains, "occ": occ, "loads": [fx(v) for v in loads],
                    "cov": fx(ref.layer_load_cov(loads)),
                    "decision": [dec.scope, dec.reason, fx(dec.load_cov), list(dec.uncovered)]})
    return {"n_base": n_base, "n_join": n_join, "L": L, "churn": churn, "joins": joins, "routes": routes,
            "cov_threshold": cov_threshold, "hole_layer": hole_layer, "scenarios": out}


def main():
    fixtures = {
        "c1j": case(8, 2, 32, [1, 2, 3, 4], 0.25, 2, 40),
        "n64j": case(64, 8, 32, [11, 12, 13], 0.1, 4, 30),
        "n256j": case(256, 16, 64, [21, 22], 0.05, 6, 12),
        "n64j_lowthr": case(64, 8, 32, [11, 12, 14], 0.1, 4, 30, cov_threshold=0.06),
        "n64j_hole": case(64, 8, 32, [15], 0.1, 0, 0, hole_layer=5),
        "n64j_hole_filled": case(64, 8, 32, [15], 0.1, 2, 10, hole_layer=5),
    }
    path = os.path.join(HERE, "membership_cases.json")
    with open(path, "w") as fh:
        json.dump(fixtures, fh, sort_keys=True)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
