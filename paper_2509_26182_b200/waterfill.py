"""Water-filling drop-in (``pkg/src/swarmsched/waterfill.py``) backed by ``ss_waterfill`` / ``ss_hamilton``.

``solve_lambda`` (47-88), ``hamilton_round`` (91-128) and
``rebalance_pipeline`` (142-183) keep their signatures and return types.
``FractionalAllocation.targets`` keeps the reference's item typing: a target
is the Python ``int`` capacity where ``min(c, level * f)`` returned ``c``,
else a float -- the device reports that as ``tflag``.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Mapping, Sequence, Union

import numpy as np

from . import _native as N
from .errors import InfeasibleCapacity, RoundingOverflow, ZeroCapacityGpu, raise_for_status
from .plan import Pipeline
from .topology import ClusterSnapshot, GpuNode, LayerSlice, ModelSpec, layer_capacity


@dataclass(frozen=True)
class FractionalAllocation:
    targets: tuple
    water_level: float


@dataclass(frozen=True)
class IntegerAllocation:
    layers: tuple


# one device water-fill group holds at most this many entries (phase1.cu NMAX: per-thread arrays); the reference
# accepts any length, but a pipeline never has more stages than its region has usable GPUs (<= 256 on the device
# path's constructive cover as well) -- documented in DESIGN.md "Limits of the device path"
MAX_ENTRIES = 256


def _check_len(n, what):
    if n > MAX_ENTRIES:
        raise ValueError(f"{what}: the device water-fill takes at most {MAX_ENTRIES} entries per call, got {n}")


def _dev():
    import torch
    return torch, torch.device("cuda")


def _run_waterfill(flops, caps, layer_count, mode):
    torch, dev = _dev()
    n = len(caps)
    _check_len(n, ("solve_lambda", "", "rebalance_pipeline")[mode] or "water-fill")
    ints = torch.tensor([0, n, layer_count] + [int(c) for c in caps], dtype=torch.int32, device=dev)
    fl = torch.tensor([float(f) for f in flops], dtype=torch.float64, device=dev)
    targets = torch.zeros(n, dtype=torch.float64, device=dev)
    tflag = torch.zeros(n, dtype=torch.int32, device=dev)
    level = torch.zeros(1, dtype=torch.float64, device=dev)
    counts = torch.zeros(n, dtype=torch.int32, device=dev)
    st = torch.zeros(2, dtype=torch.int32, device=dev)
    N.check(N.lib().ss_waterfill(1, N.ptr(ints[0:2]), N.ptr(fl), N.ptr(ints[3:]), N.ptr(ints[2:3]), mode,
                                 N.ptr(targets), N.ptr(tflag), N.ptr(level), N.ptr(counts), N.ptr(st[0:1]),
                                 N.ptr(st[1:2]), N.stream_handle()), "ss_waterfill")
    status, aux = st.cpu().tolist()
    return status, aux, targets.cpu().numpy(), tflag.cpu().numpy(), float(level.cpu()[0]), counts.cpu().tolist()


def _raise(status, aux, layer_count, what):
    if status == 8:
        raise ValueError(f"{what}: invalid input")
    if status == 5:
        raise InfeasibleCapacity(aux, layer_count)
    if status == 6:
        raise RoundingOverflow(f"{what}: rounding overflow")
    raise_for_status(status, aux)


def _typed_targets(values, flags):
    return tuple(int(v) if f else float(v) for v, f in zip(values, flags))


def solve_lambda(flops: Sequence[float], capacities: Sequence[int], layer_count: int) -> FractionalAllocation:
    if len(flops) != len(capacities) or not flops:
        raise ValueError("flops and capacities must be equal-length and non-empty")
    if any(f <= 0 for f in flops):
        raise ValueError("flops must be positive")
    if layer_count < 1:
        raise ValueError("layer_count must be >= 1")
    status, aux, t, tf, level, _ = _run_waterfill(flops, capacities, layer_count, 0)
    if status:
        _raise(status, aux, layer_count, "solve_lambda")
    return FractionalAllocation(targets=_typed_targets(t, tf), water_level=level)


def hamilton_round(frac: FractionalAllocation, capacities: Sequence[int], total: int = None) -> IntegerAllocation:
    targets = frac.targets
    if len(targets) != len(capacities):
        raise ValueError("targets and capacities must be equal-length")
    torch, dev = _dev()
    n = len(targets)
    _check_len(n, "hamilton_round")
    ints = torch.tensor([0, n, -1 if total is None else int(total)] + [int(c) for c in capacities] +
                        [1 if isinstance(t, int) else 0 for t in targets], dtype=torch.int32, device=dev)
    tv = torch.tensor([float(t) for t in targets], dtype=torch.float64, device=dev)
    counts = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    N.check(N.lib().ss_hamilton(1, N.ptr(ints[0:2]), N.ptr(tv), N.ptr(ints[3 + n:]), N.ptr(ints[3:3 + n]),
                                N.ptr(ints[2:3]), N.ptr(counts), N.ptr(st), N.stream_handle()), "ss_hamilton")
    status = int(st.cpu()[0])
    if status:
        _raise(status, 0, total, "hamilton_round")
    return IntegerAllocation(layers=tuple(counts.cpu().tolist()[:n]))


GpuLookup = Union[ClusterSnapshot, Mapping[str, GpuNode], Iterable[GpuNode]]


def _as_gpu_map(gpus: GpuLookup) -> Mapping[str, GpuNode]:
    if isinstance(gpus, ClusterSnapshot):
        return {g.id: g for g in gpus.gpus}
    if isinstance(gpus, Mapping):
        return gpus
    return {g.id: g for g in gpus}


def rebalance_pipeline(pipeline: Pipeline, gpus: GpuLookup, model: ModelSpec) -> Pipeline:
    by_id = _as_gpu_map(gpus)
    nodes = [by_id[s.gpu_id] for s in pipeline.stages]
    caps = [layer_capacity(n, model) for n in nodes]
    for node, cap in zip(nodes, caps):
        if cap < 1:
            raise ZeroCapacityGpu(node.id)
    status, aux, _, _, _, counts = _run_waterfill([n.flops for n in nodes], caps, model.layer_count, 2)
    if status:
        _raise(status, aux, model.layer_count, "rebalance_pipeline")
    slices, cursor = [], 1
    for node, n_layers in zip(nodes, counts):
        slices.append(LayerSlice(node.id, cursor, cursor + n_layers - 1))
        cursor += n_layers
    return Pipeline(stages=tuple(slices), region=pipeline.region)
