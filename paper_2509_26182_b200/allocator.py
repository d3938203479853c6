"""Phase-1 drop-in: layer allocation backed by the sm_100a kernels.

Same public names, signatures and return types as
``pkg/src/swarmsched/allocator.py`` (``ObjectiveParams`` 61-73,
``StageSolution`` 76-84, ``SweepStats`` 87-94, ``k_max`` 97-101, ``score``
104-111, ``solve_stage_counts`` 473-504, ``min_stages`` 507-513,
``estimate_objective_params`` 516-538, ``allocate`` 541-618).

Device work per ``allocate`` call (one stream, one host sync at the end):
    ss_rtt_fill + ss_objective           region objective inputs (CPython-sum exact)
    ss_stage_counts_{validate,exact,cover}  s*(k) and witness groups for every k
    ss_phase1_score + ss_phase1_best     Z(k), argmax by (Z, k), water-fill of the
                                         chosen groups (waterfill.py semantics)
    ss_variant_reduce                    objective_total as the reference's left fold
The host packs regions (sorted region names, GPUs sorted by (-cap, id) --
string order is Python's, so it is resolved here) and assembles the returned
``AllocationPlan`` from device outputs.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from ._phase1 import PoolBatch, PoolSpec, objective_device, objective_launch, objective_pack
from .errors import DegenerateObjective, NoFeasiblePipeline, SS_OK, raise_for_status
from .plan import AllocationPlan, PerKEntry, Pipeline
from .topology import ClusterSnapshot, GpuNode, LayerSlice, ModelSpec, layer_capacity

EXACT_SWEEP_LIMIT = 16


@dataclass(frozen=True)
class ObjectiveParams:
    alpha: float = 1.0
    t_comp_seconds: float = 0.0
    rtt_seconds: float = 0.0

    def __post_init__(self) -> None:
        if self.alpha <= 0:
            raise ValueError(f"alpha must be positive, got {self.alpha}")
        if self.t_comp_seconds < 0 or self.rtt_seconds < 0:
            raise ValueError("objective times must be >= 0")


@dataclass(frozen=True)
class StageSolution:
    stages: int
    groups: Tuple[Tuple[int, ...], ...]


@dataclass
class SweepStats:
    levels: int = 0
    states_expanded: int = 0
    peak_frontier: int = 0
    pruned_dominated: int = 0


def k_max(capacities: Sequence[int], layer_count: int) -> int:
    """min(#GPUs, floor(total capacity / L)) -- allocator.py:97-101 (zero-capacity GPUs count)."""
    if layer_count < 1:
        raise ValueError("layer_count must be >= 1")
    return min(len(capacities), sum(capacities) // layer_count)


def _kpow_table(kmax: int, alpha: float) -> np.ndarray:
    # k ** alpha is evaluated by CPython (glibc pow) and shipped to the device
    return np.array([0.0] + [float(k ** alpha) for k in range(1, kmax + 1)], dtype=np.float64)


def score(k: int, s_star: int, params: ObjectiveParams) -> float:
    import torch
    lib = N.lib()
    dev = torch.device("cuda")
    ints = torch.tensor([k, s_star], dtype=torch.int32, device=dev)
    kp = float(k ** params.alpha) if k >= 1 else 0.0
    dbl = torch.tensor([kp, params.t_comp_seconds, params.rtt_seconds], dtype=torch.float64, device=dev)
    z = torch.empty(1, dtype=torch.float64, device=dev)
    st = torch.empty(1, dtype=torch.int32, device=dev)
    N.check(lib.ss_score(1, N.ptr(ints[0:1]), N.ptr(ints[1:2]), N.ptr(dbl[0:1]), N.ptr(dbl[1:2]), N.ptr(dbl[2:3]),
                         N.ptr(z), N.ptr(st), N.stream_handle()), "ss_score")
    status = int(st.cpu()[0])
    if status == 8:
        raise ValueError(f"need k >= 1 and s_star >= k, got k={k} s_star={s_star}")
    if status == 7:
        raise DegenerateObjective("both t_comp and rtt are zero; the score is undefined")
    raise_for_status(status)
    return float(z.cpu()[0])


def _solve_pools(pools: List[PoolSpec]):
    batch = PoolBatch(pools)
    batch.stage_counts()
    return batch


def solve_stage_counts(capacities: Sequence[int], layer_count: int, max_replicas: int,
                       stats: Optional[SweepStats] = None) -> Dict[int, StageSolution]:
    caps = [int(c) for c in capacities]
    if any(caps[j] < caps[j + 1] for j in range(len(caps) - 1)):
        raise ValueError("capacities must be sorted non-increasing")
    if max_replicas < 1 or not any(c > 0 for c in caps):
        return {}
    batch = _solve_pools([PoolSpec(caps, [1.0] * len(caps), layer_count, max_replicas)])
    res = batch.fetch()
    st = int(res.status[0])
    if st == 8:
        raise ValueError("stage-count input outside the device limits or unsorted")
    res.raise_pool(0)
    if stats is not None and batch.exact.size:
        lv, ex, pk, pr = (int(x) for x in res.sweep_stats[0])
        stats.levels = lv
        stats.states_expanded += ex
        stats.peak_frontier = max(stats.peak_frontier, pk)
        stats.pruned_dominated += pr
    return {k: StageSolution(stages=s, groups=g) for k, (s, g) in res.solutions(0).items()}


def min_stages(capacities: Sequence[int], layer_count: int, k: int) -> Optional[StageSolution]:
    if k < 1:
        raise ValueError(f"k must be >= 1, got {k}")
    return solve_stage_counts(capacities, layer_count, k).get(k)


def _region_items(cluster: ClusterSnapshot, regions_gpus: List[Sequence[GpuNode]]):
    """(flops, links) per region in cluster order; links resolved direct>reverse on device."""
    where = {}                                   # gpu id -> (region item, position); one pass over the links
    for ri, rg in enumerate(regions_gpus):
        for i, g in enumerate(rg):
            where[g.id] = (ri, i)
    links = [[] for _ in regions_gpus]
    for (a, b), v in cluster.links.items():
        wa, wb = where.get(a), where.get(b)
        if wa is not None and wb is not None and wa[0] == wb[0] and wa[1] != wb[1]:
            links[wa[0]].append((wa[1], wb[1], float(v)))
    return [([g.flops for g in rg], lk) for rg, lk in zip(regions_gpus, links)]


def estimate_objective_params(region_gpus: Sequence[GpuNode], cluster: ClusterSnapshot, model: ModelSpec,
                              alpha: float, mean_tokens_per_request: float) -> ObjectiveParams:
    items = _region_items(cluster, [list(region_gpus)])
    t, r = objective_device(items, cluster.default_cross_region_rtt_s, model.flops_per_layer_per_token,
                            [model.layer_count], mean_tokens_per_request)
    return ObjectiveParams(alpha=alpha, t_comp_seconds=float(t.cpu()[0]), rtt_seconds=float(r.cpu()[0]))


def allocate(cluster: ClusterSnapshot, model: ModelSpec, *, alpha: float = 1.0,
             params: Optional[ObjectiveParams] = None, mean_tokens_per_request: float = 128.0) -> AllocationPlan:
    import torch
    L = model.layer_count
    packed = []     # (region, region_gpus, ordered_gpus, ordered_caps, kmax)
    for region in sorted(cluster.regions):
        rg = cluster.gpus_in_region(region)
        if not rg:
            continue
        caps = [layer_capacity(g, model) for g in rg]
        limit = k_max(caps, L)
        if limit < 1:
            continue
        order = sorted(range(len(rg)), key=lambda i: (-caps[i], rg[i].id))
        packed.append((region, rg, [rg[i] for i in order], [caps[i] for i in order], limit))
    if not packed:
        raise NoFeasiblePipeline(f"no region can host all {L} layers of {model.name!r}")
    pools = [PoolSpec(oc, [g.flops for g in og], L, km) for _, _, og, oc, km in packed]
    a = params.alpha if params is not None else alpha
    # k ** alpha table, the variant pointer and the objective inputs ride along in the batch's single H2D copy
    extra = {"kpow": _kpow_table(max(p.kmax for p in pools), a), "var_ptr": np.array([0, len(pools)], dtype=np.int32)}
    if params is not None:
        extra["tr"] = np.concatenate([np.full(len(pools), params.t_comp_seconds),
                                      np.full(len(pools), params.rtt_seconds)])
    else:
        obj_arrays, obj_meta = objective_pack(_region_items(cluster, [p[1] for p in packed]), [L] * len(pools))
        extra.update(obj_arrays)
    batch = PoolBatch(pools, extra=extra, defer_workspace_check=True)
    batch.stage_counts()
    if params is not None:
        t, r = batch.extra["tr"][:len(pools)], batch.extra["tr"][len(pools):]
    else:
        t, r = objective_launch(batch.extra, obj_meta, cluster.default_cross_region_rtt_s,
                                model.flops_per_layer_per_token, mean_tokens_per_request)
    batch.score_and_best(t, r, batch.extra["kpow"])
    # objective_total: the reference's left fold over regions (allocator.py:588), on device
    lib = N.lib()

    def reduce():
        N.check(lib.ss_variant_reduce(1, N.ptr(batch.extra["var_ptr"]), N.ptr(batch.koff), N.ptr(batch.best_k),
                                      N.ptr(batch.z), N.ptr(batch.status), N.ptr(batch.total), N.ptr(batch.feasible),
                                      None, None, N.stream_handle()), "ss_variant_reduce")
    batch.log_op(reduce)
    res = batch.fetch()
    pipelines: List[Pipeline] = []
    per_k: List[PerKEntry] = []
    for p, (region, _, og, oc, km) in enumerate(packed):
        res.raise_pool(p)
        sols = res.solutions(p)
        if not sols:
            continue
        for k in sorted(sols):
            per_k.append(PerKEntry(region=region, k=k, s_star=sols[k][0], z=res.z_of(p, k)))
        best = int(res.best_k[p])
        counts = res.counts_of(p, best)
        pos = 0
        for grp in sols[best][1]:
            slices, cursor = [], 1
            for idx in grp:
                n_layers = counts[pos]
                pos += 1
                slices.append(LayerSlice(og[idx].id, cursor, cursor + n_layers - 1))
                cursor += n_layers
            pipelines.append(Pipeline(stages=tuple(slices), region=region))
    if not pipelines:
        raise NoFeasiblePipeline(f"no region can host all {L} layers of {model.name!r}")
    return AllocationPlan(replication_count=len(pipelines), pipelines=tuple(pipelines),
                          stage_total=sum(pp.stage_count for pp in pipelines), objective_score=res.total,
                          per_k_table=tuple(per_k))
