#!/usr/bin/env python3
"""SweepStats fixtures from the UNMODIFIED reference (build container only).

    python tests/golden/make_sweep_stats_golden.py

For random exact-path pools (<= 16 usable GPUs, allocator.py:473-504 -> _sweep 138-225) records the reference's
SweepStats (levels, states_expanded, peak_frontier, pruned_dominated, allocator.py:87-94) and s*(k) per k.
tests/test_gpu_phase1.py compares the device sweep's counters field for field.
"""

from __future__ import annotations

import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from swarmsched import allocator as ref_alloc              # noqa: E402


def main():
    rng = random.Random(20261018)
    cases = []
    while len(cases) < 240:
        n = rng.randint(1, 16)
        L = rng.choice([8, 10, 12, 16, 24, 32, 48, 64, 80])
        lo = rng.choice([1, 2, 4, L // 4 or 1])
        caps = sorted((rng.randint(lo, L + 4) for _ in range(n)), reverse=True)
        if rng.random() < 0.2:
            caps += [0] * rng.randint(1, 3)
        kmax = rng.choice([ref_alloc.k_max(caps, L), rng.randint(1, 16)])
        if kmax < 1:
            continue
        st = ref_alloc.SweepStats()
        sols = ref_alloc.solve_stage_counts(caps, L, kmax, stats=st)
        cases.append({"caps": caps, "L": L, "kmax": kmax,
                      "stats": [st.levels, st.states_expanded, st.peak_frontier, st.pruned_dominated],
                      "s_star": {str(k): v.stages for k, v in sols.items()}})
    # hard shapes (N=16, L=80, caps U[4, 32] reach ~1.5k frontier / ~5k expansions)
    for q in range(40):
        n = rng.randint(12, 16)
        L = rng.choice([48, 64, 80])
        caps = sorted((rng.randint(4, 32) for _ in range(n)), reverse=True)
        kmax = ref_alloc.k_max(caps, L)
        if kmax < 1:
            continue
        st = ref_alloc.SweepStats()
        sols = ref_alloc.solve_stage_counts(caps, L, kmax, stats=st)
        cases.append({"caps": caps, "L": L, "kmax": kmax,
                      "stats": [st.levels, st.states_expanded, st.peak_frontier, st.pruned_dominated],
                      "s_star": {str(k): v.stages for k, v in sols.items()}})
    path = os.path.join(HERE, "sweep_stats_cases.json")
    with open(path, "w") as fh:
        json.dump(cases, fh)
    print(f"wrote {path}: {len(cases)} cases, max states_expanded {max(c['stats'][1] for c in cases)}")


if __name__ == "__main__":
    main()
