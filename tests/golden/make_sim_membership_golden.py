#!/usr/bin/env python3
"""Simulator-with-membership golden fixtures from the UNMODIFIED reference (build container only).

    python tests/golden/make_sim_membership_golden.py

Runs the reference's discrete-event simulator (sim.py:_Simulation) with membership events -- leaves of plan GPUs
(chain aborts, re-queues, uncovered-layer global rebalances), joins (bottleneck-layer slices, a zero-capacity
join), a low CoV threshold (load-triggered rebalances) -- and with a short TTL (entries expiring between publish
ticks).  Records the MetricsReport and the per-request latencies in completion order; the event specs are stored
so tests/test_sim_membership.py can rebuild the same events for the drop-in run_simulation.
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import swarmsched as ref                                    # noqa: E402
from swarmsched import sim as ref_sim                       # noqa: E402
from swarmsched.membership import MembershipEvent           # noqa: E402


def fx(v):
    return float(v).hex()


def gpu_spec(gid, region, capacity, flops, tokens=100_000):
    return {"id": gid, "region": region, "vram_bytes": fx(capacity * 1.2e9 / 0.8), "flops": fx(flops),
            "ram_token_capacity": tokens}


def ref_gpu(spec):
    return ref.GpuNode(id=spec["id"], region=spec["region"], vram_bytes=float.fromhex(spec["vram_bytes"]),
                       flops=float.fromhex(spec["flops"]), reserve_fraction=0.2,
                       ram_token_capacity=spec["ram_token_capacity"])


def case(n, L, seed, rate, duration, prompt, output, events, *, ttl=2.0, cov=0.5, tokens=None):
    model = ref.ModelSpec(f"bench-{L}l", L, 1.2e9, 2.8e10)
    cluster, model = ref.synthetic_cluster(n, seed=0, model=model)
    if tokens is not None:                                   # tighter KV capacity: admission actually blocks
        gpus = tuple(ref.GpuNode(id=g.id, region=g.region, vram_bytes=g.vram_bytes, flops=g.flops,
                                 reserve_fraction=g.reserve_fraction, ram_token_capacity=tokens) for g in cluster.gpus)
        cluster = ref.ClusterSnapshot(gpus=gpus, links=cluster.links)
    plan = ref.allocate(cluster, model)
    trace = ref_sim.generate_trace(rate, duration, seed=seed, prompt_tokens=prompt, output_tokens=output)
    evs = []
    for e in events:
        if e["kind"] == "leave":
            evs.append(MembershipEvent(at_s=float.fromhex(e["t"]), kind="leave", gpu_id=e["gpu_id"]))
        else:
            evs.append(MembershipEvent(at_s=float.fromhex(e["t"]), kind="join", gpu=ref_gpu(e["gpu"])))
    sim = ref_sim._Simulation(cluster, model, plan, trace, membership_events=evs, ttl_multiplier=ttl,
                              cov_threshold=cov)
    rep = sim.run()
    d = rep.to_dict()
    return {"n": n, "L": L, "seed": seed, "ttl": ttl, "cov": cov, "tokens": tokens, "events": events,
            "trace": [[fx(r.arrival_s), r.prompt_tokens, r.output_tokens] for r in trace],
            "report": {k: (fx(v) if isinstance(v, float) else v) for k, v in d.items()},
            "latencies": [fx(v) for v in sim._latencies]}


def leave(t, gid):
    return {"kind": "leave", "t": fx(t), "gpu_id": gid}


def join(t, spec):
    return {"kind": "join", "t": fx(t), "gpu": spec}


def main():
    plan8 = ref.allocate(*ref.synthetic_cluster(8, seed=0, model=ref.ModelSpec("bench-32l", 32, 1.2e9, 2.8e10)))
    g8 = sorted(plan8.gpu_slices())
    plan64 = ref.allocate(*ref.synthetic_cluster(64, seed=0, model=ref.ModelSpec("bench-64l", 64, 1.2e9, 2.8e10)))
    g64 = sorted(plan64.gpu_slices())
    fixtures = {
        # a plan GPU leaves mid-run (aborts + uncovered layers -> global rebalance), a new GPU joins later
        "c1_leave_join": case(8, 32, 11, 40.0, 3.0, (64, 2048), (8, 64),
                              [leave(0.8, g8[1]), join(1.6, gpu_spec("gpu-new-a", "region-a", 12, 1.7e14))]),
        # a zero-capacity join (stays registered, serves nothing) and a leave that keeps coverage
        "c1_zero_join": case(8, 32, 12, 40.0, 2.0, (64, 2048), (8, 64),
                             [join(0.5, gpu_spec("gpu-tiny", "region-b", 0, 9e13)), leave(1.1, g8[-1])]),
        # C2 pool: several departures and arrivals under load, KV capacity low enough to gate admission
        "c2_churn": case(64, 64, 13, 120.0, 2.0, (500, 8000), (8, 40),
                         [leave(0.3, g64[5]), leave(0.7, g64[20]), join(0.9, gpu_spec("gpu-new-b", "region-c", 20, 2.1e14)),
                          leave(1.2, g64[33]), join(1.5, gpu_spec("gpu-new-c", "region-a", 9, 8e13))],
                         tokens=60_000),
        # load-CoV trigger: a tiny threshold turns every membership event into a global rebalance
        "c2_cov_rebalance": case(64, 64, 14, 100.0, 1.5, (500, 8000), (8, 40),
                                 [join(0.4, gpu_spec("gpu-new-d", "region-b", 16, 1.5e14)), leave(0.9, g64[40])],
                                 cov=0.01),
        # short TTL: latency / link entries expire between publish ticks (no membership events)
        "c1_short_ttl": case(8, 32, 15, 60.0, 2.0, (64, 2048), (8, 64), [], ttl=0.5),
    }
    path = os.path.join(HERE, "sim_membership_cases.json")
    with open(path, "w") as fh:
        json.dump(fixtures, fh, sort_keys=True)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")
    for k, v in fixtures.items():
        r = v["report"]
        print(k, "submitted", r["submitted"], "completed", r["completed"], "aborted", r["aborted"],
              "unserved", r["unserved"], "queue_peak", r["queue_peak"], "duration", float.fromhex(r["duration_s"]))


if __name__ == "__main__":
    main()
