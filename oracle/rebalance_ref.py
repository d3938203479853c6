"""CPU restatement of the rebalance loop (TEST INFRASTRUCTURE ONLY -- the checker, never the product path).

One scenario of SURVEY.md 8(f) row 2, in the reference's semantics:
  route R1 requests (router.py:247-260 op script with window W)
  -> membership events, aborting live chains on each departing GPU first (sim.py:413-418)
  -> evaluate_triggers (membership.py:389-396; oracle.membership_ref)
  -> on a global decision: allocate() on the churned pool (membership.py:398-411; oracle.alloc_ref),
     apply_plan's changed_gpus (membership.py:280-294), abort of the live chains on them (sim.py:425-429)
  -> route R2 more requests.
Pinned by tests/golden/rebalance_cases.json (the reference's MembershipManager + ChainRouter).
"""

from __future__ import annotations

from typing import Dict, List, Sequence, Tuple

import numpy as np

from . import alloc_ref, chain_ref, membership_ref


def columns_of(absent: np.ndarray, lo: np.ndarray, hi: np.ndarray, layer_count: int) -> List[np.ndarray]:
    return [np.nonzero(~absent & (lo <= l) & (hi >= l))[0] for l in range(1, layer_count + 1)]


def abort(live: List[list], occ: np.ndarray, gpus) -> List[int]:
    """Release every live chain touching ``gpus``; returns the aborted positions in ``live`` order."""
    gs = set(int(g) for g in gpus)
    hit = []
    for j, chain in enumerate(live):
        if chain and gs.intersection(chain):
            occ[chain] -= 1
            live[j] = []
            hit.append(j)
    return hit


def plan_slices(plan_dict, pos: Dict[str, int], n: int) -> Tuple[np.ndarray, np.ndarray, List[int]]:
    """Slices of an alloc_ref plan as index arrays, plus the plan.gpu_slices() order."""
    lo = np.zeros(n, dtype=np.int32)
    hi = np.full(n, -1, dtype=np.int32)
    order = []
    for p in plan_dict["pipelines"]:
        for st in p["stages"]:
            g = pos[st["gpu_id"]]
            lo[g], hi[g] = st["start_layer"], st["end_layer"]
            order.append(g)
    return lo, hi, order


def churned_cluster(cluster, ids: Sequence[str], absent: np.ndarray):
    """MembershipManager.cluster_snapshot() (membership.py:157-167): present GPUs in id order, their links."""
    from paper_2509_26182_b200.topology import ClusterSnapshot
    by_id = {g.id: g for g in cluster.gpus}
    keep = [ids[g] for g in range(len(ids)) if not absent[g]]
    alive = set(keep)
    links = {p: v for p, v in cluster.links.items() if p[0] in alive and p[1] in alive}
    return ClusterSnapshot(gpus=tuple(by_id[g] for g in sorted(keep)), links=links,
                           default_cross_region_rtt_s=cluster.default_cross_region_rtt_s)


def changed_gpus(lo0, hi0, lo1, hi1) -> List[int]:
    """apply_plan's changed set: GPUs whose (start, end) slice differs, either side may be absent."""
    a = np.where(lo0 <= hi0, lo0 * 100000 + hi0, -1)
    b = np.where(lo1 <= hi1, lo1 * 100000 + hi1, -1)
    return np.nonzero(a != b)[0].tolist()
