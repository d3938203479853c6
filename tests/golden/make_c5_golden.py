#!/usr/bin/env python3
"""C5 golden fixture (BASELINE configs[4]) from the UNMODIFIED reference (build container only).

    python tests/golden/make_c5_golden.py

For each C5 sub-pool of ``scenarios.c5_pools(0)`` (8B L=32 over 256 GPUs, 32B L=64 over 384, 70B L=80
over 384; 8 regions, explicit all-pairs region-RTT links):

* ``allocate``: the reference's plan (``allocator.py:541-618``), floats as ``float.hex``;
* ``replays``: the reference's ``MembershipManager`` + ``ChainRouter`` (``router.py:247-260``) driven through
  the bench's scenario semantics for two scenario seeds: ``on_leave`` of the seeded churn set
  (``scenarios.churn_set``, 5%), per-pair jitter folded into an explicit symmetric link table, then 320
  routes with W = 64 (release of chain i-64 before route i, so releases run from request 64 on).

The GPU test (tests/test_gpu_c5_parity.py) rebuilds the same states on the device (device-generated events)
and compares plan for plan and chain for chain.  /root/reference is read, never copied; the output is
committed as c5_cases.json.
"""

from __future__ import annotations

import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_golden import REPO, dump, plan_json, ref, replay_record  # noqa: E402

sys.path.insert(1, REPO)
from paper_2509_26182_b200 import scenarios as scen  # noqa: E402  (generator only)

SEEDS = (0, 97)
ROUTES, WINDOW = 320, 64


def to_ref(cl, model):
    gpus = tuple(ref.GpuNode(g.id, g.region, g.vram_bytes, g.flops, g.reserve_fraction, g.ram_token_capacity)
                 for g in cl.gpus)
    rcl = ref.ClusterSnapshot(gpus=gpus, links=dict(cl.links),
                              default_cross_region_rtt_s=cl.default_cross_region_rtt_s)
    rmodel = ref.ModelSpec(model.name, model.layer_count, model.bytes_per_layer, model.flops_per_layer_per_token)
    return rcl, rmodel


def main():
    out = {}
    for name, cl, model in scen.c5_pools(0):
        rcl, rm = to_ref(cl, model)
        t0 = time.perf_counter()
        plan = ref.allocate(rcl, rm)
        print(f"{name}: allocate k={plan.replication_count} in {time.perf_counter() - t0:.2f}s")
        rec = {"gpus": len(cl.gpus), "L": model.layer_count, "plan": plan_json(plan), "replays": {}}
        ids = sorted(g.id for g in rcl.gpus)
        pos = {g: i for i, g in enumerate(ids)}
        slices = {pos[g]: (s.start_layer, s.end_layer) for g, s in plan.gpu_slices().items()}
        for s in SEEDS:
            leave_idx = scen.churn_set(s, sorted(slices), slices, model.layer_count, 0.05)
            jit = scen.jitter_factor_matrix(s, len(ids))
            links = {(ids[i], ids[j]): rcl.rtt_s(ids[i], ids[j]) * jit[i, j]
                     for i in range(len(ids)) for j in range(i + 1, len(ids))}
            clj = ref.ClusterSnapshot(gpus=rcl.gpus, links=links)
            rec["replays"][str(s)] = replay_record(clj, rm, plan, ROUTES, WINDOW, leave=[ids[g] for g in leave_idx],
                                                   name=f"c5_{name}_s{s}")
        out[name] = rec
    dump("c5_cases.json", out)


if __name__ == "__main__":
    main()
