#!/usr/bin/env python3
"""Simulator golden fixtures from the UNMODIFIED reference (build container only).

    python tests/golden/make_sim_golden.py

Runs the reference's discrete-event simulator (sim.py:_Simulation / run_simulation) on bench pools and
generate_trace traces (no membership events), and records the MetricsReport plus the per-request latencies in
completion order.  tests/test_sim.py replays the same traces through the device simulator.
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import swarmsched as ref                                    # noqa: E402
from swarmsched import sim as ref_sim                       # noqa: E402


def fx(v):
    return float(v).hex()


def case(n, L, seed, rate, duration, prompt, output, amortize=False, contention=1.0):
    model = ref.ModelSpec(f"bench-{L}l", L, 1.2e9, 2.8e10)
    cluster, model = ref.synthetic_cluster(n, seed=0, model=model)
    plan = ref.allocate(cluster, model)
    trace = ref_sim.generate_trace(rate, duration, seed=seed, prompt_tokens=prompt, output_tokens=output)
    sim = ref_sim._Simulation(cluster, model, plan, trace, amortize_rtt=amortize, contention_exponent=contention)
    rep = sim.run()
    d = rep.to_dict()
    return {"n": n, "L": L, "seed": seed, "rate": rate, "duration": duration, "prompt": list(prompt),
            "output": list(output), "amortize": amortize, "contention": contention,
            "trace": [[fx(r.arrival_s), r.prompt_tokens, r.output_tokens] for r in trace],
            "report": {k: (fx(v) if isinstance(v, float) else v) for k, v in d.items()},
            "latencies": [fx(v) for v in sim._latencies]}


def main():
    fixtures = {
        "c1_light": case(8, 32, 1, 20.0, 3.0, (32, 256), (16, 128)),
        "c1_heavy": case(8, 32, 2, 400.0, 1.0, (1000, 40000), (16, 64)),
        "c2_mid": case(64, 64, 3, 150.0, 2.0, (500, 20000), (8, 48)),
        "c2_amortized": case(64, 64, 4, 150.0, 1.0, (500, 20000), (8, 48), amortize=True),
        "c4_light": case(256, 64, 5, 60.0, 1.5, (500, 40000), (8, 32)),
        "n192_wide": case(192, 10, 6, 300.0, 1.0, (1000, 60000), (4, 24)),
    }
    path = os.path.join(HERE, "sim_cases.json")
    with open(path, "w") as fh:
        json.dump(fixtures, fh, sort_keys=True)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")
    for k, v in fixtures.items():
        r = v["report"]
        print(k, "submitted", r["submitted"], "completed", r["completed"], "unserved", r["unserved"],
              "queue_peak", r["queue_peak"], "duration", float.fromhex(r["duration_s"]))


if __name__ == "__main__":
    main()
