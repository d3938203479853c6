#!/usr/bin/env python3
"""Admission-path golden fixtures from the UNMODIFIED reference (build container only).

    python tests/golden/make_admission_golden.py

The simulator's per-request caller of route() (sim.py:319-366) on a time-free
step schedule: at step t, every chain admitted at step t - W completes (sim._release: router.release +
release_kv on its distinct GPUs, sim.py:353-357), request t arrives at the back of the queue
(sim.py:361-366), and the queue drains strictly FIFO (sim.py:345-351): the head is routed with
exclude = {GPUs whose kv_headroom < its tokens} (sim.py:319-327), reserves its tokens on the chain's
distinct GPUs (sim.py:330-331), and the drain stops at the first head that raises UncoveredLayer or
NoPath.  Request tokens come from scenarios.request_tokens (this repo's generator).
"""

from __future__ import annotations

import collections
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, REPO)

import swarmsched as ref                                    # noqa: E402
from swarmsched.errors import NoPath, UncoveredLayer          # noqa: E402
from swarmsched.membership import MembershipManager          # noqa: E402
from swarmsched.sim import LatencyModel                      # noqa: E402

from paper_2509_26182_b200 import scenarios as scen          # noqa: E402  (token generator only)


def fx(v):
    return float(v).hex()


def case(n, L, seeds, steps, window, tok_lo, tok_hi):
    model = ref.ModelSpec(f"bench-{L}l", L, 1.2e9, 2.8e10)
    cluster, model = ref.synthetic_cluster(n, seed=0, model=model)
    plan = ref.allocate(cluster, model)
    ids = sorted(g.id for g in cluster.gpus)
    pos = {g: i for i, g in enumerate(ids)}
    out = []
    for seed in seeds:
        pm = ref.PerfMap(ttl_s=4.5)
        mgr = MembershipManager(cluster, model, pm)
        pm.latency_fn = LatencyModel(model, mgr, 1.0).published
        mgr.initialize(plan, 0.0)
        router = ref.ChainRouter(pm, L)
        queue = collections.deque()
        live = collections.deque()                   # (admitted step, chain, tokens) in admission order
        admitted = [None] * steps
        for t in range(steps):
            while live and live[0][0] == t - window:
                _, chain, tok = live.popleft()
                router.release(chain, 0.0)
                for g in set(chain.gpu_ids):
                    mgr.release_kv(g, tok)
            queue.append(t)
            while queue:
                i = queue[0]
                tok = scen.request_tokens(seed, i, tok_lo, tok_hi)
                blocked = {g for g in mgr.gpu_ids() if mgr.kv_headroom(g) < tok}
                try:
                    chain = router.route(0.0, exclude=blocked)
                except (UncoveredLayer, NoPath):
                    break
                for g in set(chain.gpu_ids):
                    mgr.reserve_kv(g, tok)
                live.append((t, chain, tok))
                queue.popleft()
                admitted[i] = {"step": t, "hops": [[pos[h.gpu_id], h.start_layer, h.end_layer] for h in chain.hops],
                               "cost": fx(chain.cost_s)}
        kv = [int(mgr.kv_reserved(g)) for g in ids]
        occ = [int(pm.occupancy(g)) for g in ids]
        out.append({"seed": seed, "admitted": admitted, "queue_left": list(queue), "kv": kv, "occ": occ})
    return {"n": n, "L": L, "steps": steps, "window": window, "tok_lo": tok_lo, "tok_hi": tok_hi,
            "scenarios": out}


def main():
    fixtures = {
        "c1": case(8, 32, [1, 2, 3], 60, 6, 20000, 60000),
        "c1_tight": case(8, 32, [7, 8], 60, 6, 50000, 95000),
        "c2": case(64, 64, [4, 5], 80, 12, 30000, 90000),
        "c2_tight": case(64, 64, [9], 80, 24, 60000, 99000),
        "c2_light": case(64, 64, [6], 40, 8, 1000, 5000),
    }
    path = os.path.join(HERE, "admission_cases.json")
    with open(path, "w") as fh:
        json.dump(fixtures, fh, sort_keys=True)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
