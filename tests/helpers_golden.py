"""Rebuild golden-fixture inputs as package value objects (shared by CPU and GPU tests)."""

from __future__ import annotations

import numpy as np

from conftest import hx
from paper_2509_26182_b200 import scenarios as scen
from paper_2509_26182_b200.plan import AllocationPlan, PerKEntry, Pipeline
from paper_2509_26182_b200.topology import ClusterSnapshot, GpuNode, LayerSlice, ModelSpec


def case_latencies(case):
    return {(g, l): hx(v) for g, l, v in case["hosting"]}


def case_links(case):
    return [(a, b, hx(v)) for a, b, v in case["rtts"]]


def plan_from_golden(d) -> AllocationPlan:
    pipes = tuple(Pipeline(stages=tuple(LayerSlice(s["gpu_id"], s["start_layer"], s["end_layer"])
                                        for s in p["stages"]), region=p["region"]) for p in d["pipelines"])
    rows = tuple(PerKEntry(r["region"], r["k"], r["s_star"], hx(r["z"])) for r in d["per_k"])
    return AllocationPlan(d["k"], pipes, sum(p.stage_count for p in pipes), hx(d["objective"]), rows)


def cluster_from_alloc_case(rec):
    model = ModelSpec("golden", rec["L"], hx(rec["bpl"]), hx(rec["fpl"]))
    gpus = tuple(GpuNode(i, r, hx(v), hx(f), hx(res)) for i, r, v, f, res in rec["gpus"])
    links = {(a, b): hx(v) for a, b, v in rec["links"]}
    return ClusterSnapshot(gpus=gpus, links=links, default_cross_region_rtt_s=hx(rec["default_rtt"])), model


def replay_inputs(rep, plan_dict, *, tie=False):
    """(columns, base_tau, rtt, ids) of a golden replay record, scenario jitter/churn applied."""
    L = rep["L"]
    flops = hx(rep["flops"]) if "flops" in rep else None
    cl, model = scen.synthetic_cluster(rep["n"], seed=rep["seed"], model=scen.bench_model(L),
                                       homogeneous_flops=flops)
    ids = sorted(g.id for g in cl.gpus)
    by = {g.id: g for g in cl.gpus}
    base = np.array([model.flops_per_layer_per_token / by[g].flops for g in ids])
    rtt = scen.base_rtt_matrix(cl, ids)
    if "scenario_seed" in rep:
        rtt = rtt * scen.jitter_factor_matrix(rep["scenario_seed"], len(ids))
    plan = plan_from_golden(plan_dict)
    pos = {g: i for i, g in enumerate(ids)}
    gone = set(rep.get("leave", []))
    cols = []
    for l in range(1, L + 1):
        hosts = sorted(pos[g] for g, s in plan.gpu_slices().items() if s.covers(l) and pos[g] not in gone)
        cols.append(np.array(hosts, dtype=np.int64))
    return cols, base, rtt, ids


def hops_from_gpus(gpus):
    hops, start = [], 1
    for l in range(2, len(gpus) + 1):
        if gpus[l - 1] != gpus[l - 2]:
            hops.append([gpus[l - 2], start, l - 1])
            start = l
    hops.append([gpus[-1], start, len(gpus)])
    return hops


def stream_digests(hashes, costs, block):
    """Per-block digests of (chain hash, cost bits), as tests/golden/make_c2_stream_golden.py writes them."""
    import hashlib
    h = np.asarray(hashes, dtype=np.int64).astype("<u8", copy=False)
    c = np.asarray(costs, dtype="<f8").view("<u8")
    rec = np.stack([h, c], axis=1)
    return [hashlib.sha256(rec[i:i + block].tobytes()).hexdigest()[:16] for i in range(0, len(rec), block)]
