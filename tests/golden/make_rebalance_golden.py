#!/usr/bin/env python3
"""Global-rebalance golden fixtures from the UNMODIFIED reference (build container only).

    python tests/golden/make_rebalance_golden.py

Per scenario, driven with the reference's own objects:
  1. MembershipManager.initialize(plan); ChainRouter routes R1 requests, op script route(i) /
     release(i - W) (router.py:247-260);
  2. the scenario's membership events (drawn by this repo's generator) as the simulator applies them
     (sim.py:413-424): before each on_leave, every live chain on the departing GPU is aborted
     (released); then on_join for the joiners;
  3. evaluate_triggers(); on a global decision, global_rebalance() (membership.py:398-411) and the
     abort of every live chain on result.changed_gpus (sim.py:425-429), in request-id order;
  4. R2 more requests with the same op script; an aborted chain is not released again.
Recorded: chains of both phases, the decision, changed GPUs, final slices and occupancy.
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


def case(n_base, n_join, L, seeds, churn, joins, r1, r2, window, cov_threshold):
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
        pm = ref.PerfMap(ttl_s=4.5)
        mgr = MembershipManager(base, model, pm, cov_threshold=cov_threshold)
        pm.latency_fn = LatencyModel(model, mgr, 1.0).published
        mgr.initialize(plan, 0.0)
        router = ref.ChainRouter(pm, L)
        live = {}                                     # request index -> chain (not yet released)
        chains = []

        def route(i):
            if window > 0 and i >= window and (i - window) in live:
                router.release(live.pop(i - window), 0.0)
            c = router.route(0.0)
            live[i] = c
            chains.append({"hops": [[pos[h.gpu_id], h.start_layer, h.end_layer] for h in c.hops],
                           "cost": fx(c.cost_s)})

        def abort(gpu_ids):
            victims = sorted(i for i, c in live.items() if set(gpu_ids) & set(c.gpu_ids))
            for i in victims:
                router.release(live.pop(i), 0.0)
            return victims

        for i in range(r1):
            route(i)
        aborted_leave = []
        for g in sorted(left):
            aborted_leave += abort({ids[g]})
            mgr.on_leave(ids[g], 0.0)
        for g in joined:
            mgr.on_join(by_id[ids[g]], 0.0)
        dec = mgr.evaluate_triggers()
        changed, aborted_rebalance, degraded = [], [], None
        if dec.is_global:
            res = mgr.global_rebalance(0.0)
            degraded = res.degraded
            if not res.degraded:
                changed = sorted(pos[g] for g in res.changed_gpus)
                aborted_rebalance = abort(set(res.changed_gpus))
        for i in range(r1, r1 + r2):
            route(i)
        occ = [int(pm.occupancy(g)) if pm.is_registered(g) else 0 for g in ids]
        slices = sorted([pos[g], sl.start_layer, sl.end_layer] for g, sl in mgr.slices.items())
        out.append({"seed": seed, "left": sorted(int(g) for g in left), "joined": [int(g) for g in joined],
                    "decision": [dec.scope, dec.reason, fx(dec.load_cov)], "degraded": degraded,
                    "changed": changed, "aborted_leave": aborted_leave, "aborted_rebalance": aborted_rebalance,
                    "chains": chains, "occ": occ, "slices": slices})
    return {"n_base": n_base, "n_join": n_join, "L": L, "churn": churn, "joins": joins, "r1": r1, "r2": r2,
            "window": window, "cov_threshold": cov_threshold, "scenarios": out}


def main():
    fixtures = {
        "n64_w8": case(64, 8, 32, [11, 12, 13, 14], 0.1, 2, 24, 24, 8, 0.02),
        "c1_w4": case(8, 2, 32, [1, 2, 3], 0.25, 1, 12, 12, 4, 0.02),
        "n64_nochange": case(64, 8, 32, [15, 16], 0.1, 2, 16, 16, 8, 0.9),
    }
    path = os.path.join(HERE, "rebalance_cases.json")
    with open(path, "w") as fh:
        json.dump(fixtures, fh, sort_keys=True)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
