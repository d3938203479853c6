#!/usr/bin/env python3
"""baseline_plan fixtures from the UNMODIFIED reference (build container only).

    python tests/golden/make_baseline_golden.py

sim.py:513-553 baseline_plan (capacity-sorted first fit, equal-speed water-fill) on bench pools; plans are
stored as plan_to_dict with floats as float.hex.  tests/test_sim.py rebuilds them through the drop-in.
"""

from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import swarmsched as ref                                    # noqa: E402
from swarmsched import sim as ref_sim                       # noqa: E402


def main():
    out = {}
    for n, seed, L in [(8, 0, 32), (16, 1, 48), (64, 0, 64), (256, 0, 64), (256, 3, 80), (40, 7, 24)]:
        model = ref.ModelSpec(f"bench-{L}l", L, 1.2e9, 2.8e10)
        cluster, model = ref.synthetic_cluster(n, seed=seed, model=model)
        d = ref.plan_to_dict(ref_sim.baseline_plan(cluster, model))
        d["objective"] = float(d["objective"]).hex()
        out[f"n{n}_s{seed}_L{L}"] = {"n": n, "seed": seed, "L": L, "plan": d}
    path = os.path.join(HERE, "baseline_cases.json")
    with open(path, "w") as fh:
        json.dump(out, fh, sort_keys=True)
    print(f"wrote {path}: {len(out)} plans")


if __name__ == "__main__":
    main()
