"""Shared setup for the membership-churn parity tests (tests/golden/membership_cases.json)."""

import numpy as np

from conftest import hx
from helpers_golden import plan_from_golden


def pool_for_case(case):
    """(ScenarioSet inputs) for a golden case: full pool = base + join pool, plan on the base pool."""
    from oracle import alloc_ref
    from paper_2509_26182_b200 import scenarios as scen
    nb, nj, L = case["n_base"], case["n_join"], case["L"]
    rc = scen.default_region_count(nb)
    full, model = scen.synthetic_cluster(nb + nj, seed=0, model=scen.bench_model(L), region_count=rc)
    base, _ = scen.synthetic_cluster(nb, seed=0, model=scen.bench_model(L), region_count=rc)
    d = alloc_ref.allocate(base, model)
    order = [s["gpu_id"] for p in d["pipelines"] for s in p["stages"]]       # plan.gpu_slices() order
    d["objective"] = d["objective"].hex()
    d["per_k"] = [dict(r, z=r["z"].hex()) for r in d["per_k"]]
    plan = plan_from_golden(d)
    join_ids = [g.id for g in full.gpus[nb:]]
    return full, model, plan, join_ids, order


def trigger_inputs(full, ids, plan_order, left, joined, lo_s, hi_s, occ, present0):
    """_gpus / slices lists in the reference's dict orders (membership.py:150-154, apply_plan, on_join)."""
    by_id = {g.id: g for g in full.gpus}
    pos = {g: i for i, g in enumerate(ids)}
    gone = set(left)
    base_order = [pos[g.id] for g in full.gpus if present0[pos[g.id]]]        # cluster order of the base pool
    reg = [g for g in base_order if g not in gone] + list(joined)
    gpus = [(by_id[ids[g]].vram_bytes, by_id[ids[g]].reserve_fraction, by_id[ids[g]].flops,
             by_id[ids[g]].ram_token_capacity) for g in reg]
    at = {g: i for i, g in enumerate(reg)}
    sl_order = [pos[g] for g in plan_order if pos[g] not in gone] + [g for g in joined if lo_s[g] <= hi_s[g]]
    slices = [(at[g], int(lo_s[g]), int(hi_s[g])) for g in sl_order]
    occupancy = [int(occ[g]) for g in reg]
    return gpus, slices, [0] * len(reg), occupancy


def golden_occ(case_scn):
    return np.array(case_scn["occ"])


__all__ = ["pool_for_case", "trigger_inputs", "golden_occ", "hx"]
