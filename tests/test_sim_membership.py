"""run_simulation with membership events and a short TTL (sim.py:226-475, membership.py:129-421) vs the reference.

The fixtures (tests/golden/make_sim_membership_golden.py) come from the unmodified reference: plan-GPU leaves that
abort and re-queue chains and uncover layers (global rebalance), joins onto the bottleneck layer, a zero-capacity
join, a CoV threshold low enough that every event re-places the pool, KV capacity that gates admission, and
latency entries expiring between publish ticks.  The drop-in replays the same timeline on the host with every
route on the device ChainRouter and every rebalance through the device allocate(): the MetricsReport and every
request's latency (completion order) must match bit for bit.
"""

import json
import os

import pytest

from conftest import hx

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
CASES = ["c1_leave_join", "c1_zero_join", "c2_churn", "c2_cov_rebalance", "c1_short_ttl"]


@pytest.fixture(scope="module")
def cases():
    with open(os.path.join(HERE, "golden", "sim_membership_cases.json")) as fh:
        return json.load(fh)


def _gpu(spec):
    from paper_2509_26182_b200.topology import GpuNode
    return GpuNode(id=spec["id"], region=spec["region"], vram_bytes=hx(spec["vram_bytes"]), flops=hx(spec["flops"]),
                   reserve_fraction=0.2, ram_token_capacity=spec["ram_token_capacity"])


def _run(case, sim_fn):
    from paper_2509_26182_b200 import allocate, scenarios as scen
    from paper_2509_26182_b200.membership import MembershipEvent
    from paper_2509_26182_b200.sim import Request
    from paper_2509_26182_b200.topology import ClusterSnapshot, GpuNode
    cl, model = scen.synthetic_cluster(case["n"], seed=0, model=scen.bench_model(case["L"]))
    if case["tokens"] is not None:
        cl = ClusterSnapshot(gpus=tuple(GpuNode(id=g.id, region=g.region, vram_bytes=g.vram_bytes, flops=g.flops,
                                                reserve_fraction=g.reserve_fraction,
                                                ram_token_capacity=case["tokens"]) for g in cl.gpus),
                             links=cl.links)
    plan = allocate(cl, model)
    trace = [Request(f"r{i:05d}", hx(a), int(p), int(o)) for i, (a, p, o) in enumerate(case["trace"])]
    events = [MembershipEvent(at_s=hx(e["t"]), kind="leave", gpu_id=e["gpu_id"]) if e["kind"] == "leave"
              else MembershipEvent(at_s=hx(e["t"]), kind="join", gpu=_gpu(e["gpu"])) for e in case["events"]]
    return sim_fn(cl, model, plan, trace, events, case)


@pytest.mark.parametrize("name", CASES)
def test_run_simulation_with_membership_matches_reference(cuda_ready, cases, name):
    from paper_2509_26182_b200 import run_simulation
    c = cases[name]
    rep = _run(c, lambda cl, m, p, t, ev, cc: run_simulation(cl, m, p, t, membership_events=ev,
                                                             ttl_multiplier=cc["ttl"], cov_threshold=cc["cov"]))
    got = {k: (float(v).hex() if isinstance(v, float) else v) for k, v in rep.to_dict().items()}
    assert got == c["report"]


@pytest.mark.parametrize("name", CASES)
def test_host_timeline_latencies_match_reference(cuda_ready, cases, name):
    from paper_2509_26182_b200.perfmap import DEFAULT_PUBLISH_INTERVAL_S
    from paper_2509_26182_b200.sim import _HostTimeline
    c = cases[name]

    def go(cl, m, p, t, ev, cc):
        tl = _HostTimeline(cl, m, p, t, ev, DEFAULT_PUBLISH_INTERVAL_S, cc["ttl"], 1.0, False, 0.5, cc["cov"],
                           1.0, 128.0)
        tl.run()
        return tl
    tl = _run(c, go)
    assert [float(v).hex() for v in tl.latencies] == c["latencies"]
    assert tl.aborted == c["report"]["aborted"]
