"""CPU baseline legs for bench.py -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Times the oracle port of the reference's CPU path (numpy / CPython restatement
of router.py + perfmap.py and allocator.py + waterfill.py, pinned bit-exact to
the reference by tests/test_oracle_golden.py) on the host cores, sharded over
independent scenarios / variants with multiprocessing, exactly as BASELINE.md
section 3 prescribes.  Only the routing loop (Phase-2) or the per-candidate
stage-count + score + water-fill section (Phase-1) is inside the timer.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from . import alloc_ref, chain_ref, waterfill_ref


def _replay_job(args):
    cols, base, rtt, n_req, window = args
    t0 = time.perf_counter()
    chain_ref.replay(cols, base, rtt, n_req, window, chain_ref.occ_power_table((window or n_req) + 4))
    return time.perf_counter() - t0, n_req


def phase2_rate(scen_set, scenarios, n_req, window, cores=None):
    """Selections/s of the oracle replay over `scenarios` (indices), n_req each."""
    cores = cores or len(os.sched_getaffinity(0))
    jobs = [(scen_set.columns(s), scen_set.base_tau, scen_set.scenario_rtt(s), n_req,
             None if window < 0 else window) for s in scenarios]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(cores) as pool:
        res = pool.map(_replay_job, jobs, chunksize=1)
    wall = time.perf_counter() - t0
    sel = sum(r[1] for r in res)
    return sel / wall, cores, sel, wall


def _candidate_job(args):
    pool_caps, pool_flops, L, kmax, t, r, alpha = args
    t0 = time.perf_counter()
    sols = alloc_ref.stage_counts(pool_caps, L, kmax)
    for k, (s, groups) in sols.items():
        alloc_ref.score(k, s, alpha, t, r)
        for grp in groups:
            waterfill_ref.stage_lengths([pool_flops[i] for i in grp], [pool_caps[i] for i in grp], L)
    return time.perf_counter() - t0, kmax


def phase1_rate(packed, n_pools, cores=None):
    """Candidates/s of the oracle per-(region, k) evaluation over the first n_pools pools."""
    cores = cores or len(os.sched_getaffinity(0))
    jobs = []
    for p in range(min(n_pools, len(packed.pools))):
        pool = packed.pools[p]
        ids = [str(i) for i in range(len(packed.obj_flops[p]))]
        m = packed.obj_rtt[p]
        t, r = alloc_ref.objective([float(x) for x in packed.obj_flops[p]], ids,
                                   lambda a, b, _m=m: float(_m[int(a), int(b)]), packed.fpl, packed.layers,
                                   packed.tokens)
        jobs.append((list(pool.caps), [float(f) for f in pool.flops], pool.layers, pool.kmax, t, r, packed.alpha))
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(cores) as pool:
        res = pool.map(_candidate_job, jobs, chunksize=1)
    wall = time.perf_counter() - t0
    cand = sum(r[1] for r in res)
    return cand / wall, cores, cand, wall
