#!/usr/bin/env python3
"""Golden wire-format fixtures from the UNMODIFIED reference (build container only).

    python tests/golden/make_wire_golden.py

For bench pools C1 (L32/N8) and C2 (L64/N64) this runs the reference's own
``swarmsched route --json`` pipeline in-process (cli.py:152-161: allocate ->
_bootstrap_map -> ChainRouter.route(0.0) x n -> _print_json) and its
``save_plan`` text (plan.py:190-193), and stores both texts verbatim in
wire_cases.json.  tests/test_gpu_wire.py diffs the device path's output
against them character for character.
"""

from __future__ import annotations

import contextlib
import io
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import swarmsched as ref                                    # noqa: E402
from swarmsched import cli as ref_cli                       # noqa: E402
from swarmsched.config import resolve_config                # noqa: E402


def case(n, seed, L, requests):
    model = ref.ModelSpec(f"bench-{L}l", L, 1.2e9, 2.8e10)
    cluster, model = ref.synthetic_cluster(n, seed=seed, model=model)
    config = resolve_config(None)
    plan = ref.allocate(cluster, model, alpha=config.alpha, mean_tokens_per_request=config.mean_tokens_per_request)
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        perf_map, _ = ref_cli._bootstrap_map(cluster, model, plan, config)
        router = ref.ChainRouter(perf_map, model.layer_count)
        chains = [router.route(0.0) for _ in range(requests)]
        ref_cli._print_json({"chains": [ref_cli._chain_to_dict(c) for c in chains]})
    plan_text = json.dumps(ref.plan_to_dict(plan), indent=2, sort_keys=True) + "\n"
    return {"n": n, "seed": seed, "L": L, "requests": requests, "plan_json": plan_text, "route_json": buf.getvalue()}


def main():
    out = {"c1": case(8, 0, 32, 40), "c2": case(64, 0, 64, 20)}
    path = os.path.join(HERE, "wire_cases.json")
    with open(path, "w") as fh:
        json.dump(out, fh, sort_keys=True)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


if __name__ == "__main__":
    main()
