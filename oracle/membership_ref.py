"""CPU restatement of the membership triggers (TEST INFRASTRUCTURE ONLY -- the checker, never the product path).

Follows pkg/src/swarmsched/membership.py:359-396 (``layer_loads``, ``evaluate_triggers``) and
perfmap.py:86-114 (``layer_load``, ``layer_load_cov``) operation for operation, so every float is
bit-identical to the reference under CPython 3.12:

* ``sum(...)`` over floats is CPython 3.12's compensated ``sum`` (:func:`cpython_sum_model`):
  ``total_memory`` and ``total_flops`` (membership.py:366-369) in ``_gpus`` order, and the mean and
  variance of ``layer_load_cov`` (perfmap.py:110-113);
* the per-layer ``kv_bytes`` / ``compute`` accumulators are plain ``+=`` folds in ``slices`` order
  (membership.py:374-381); ``min(1, occ)`` is an int, so ``flops * min(1, occ)`` is one rounding;
* ``(v - mean) ** 2`` is ``pow(x, 2.0)``, correctly rounded == ``x * x``; ``math.sqrt`` is correctly rounded.

Pinned by tests/golden/membership_cases.json (the reference's MembershipManager on the same events).
"""

from __future__ import annotations

import math
from typing import List, Sequence, Tuple

from .waterfill_ref import cpython_sum_model

DEFAULT_COV_THRESHOLD = 0.5    # membership.py:48
DEFAULT_MIX_ALPHA = 0.5        # membership.py:49


def layer_load(kv_bytes: float, compute: float, total_memory: float, total_flops: float, mix_alpha: float) -> float:
    """perfmap.py:86-102."""
    kv_fraction = kv_bytes / total_memory if total_memory > 0 else 0.0
    compute_fraction = compute / total_flops if total_flops > 0 else 0.0
    return mix_alpha * kv_fraction + (1.0 - mix_alpha) * compute_fraction


def layer_load_cov(loads: Sequence[float]) -> float:
    """perfmap.py:105-114."""
    values = list(loads)
    if not values:
        return 0.0
    mean = cpython_sum_model(values) / len(values)
    if mean == 0.0:
        return 0.0
    variance = cpython_sum_model([(v - mean) ** 2 for v in values]) / len(values)
    return math.sqrt(variance) / mean


def layer_loads(layer_count: int, gpus: Sequence[Tuple[float, float, float, int]], slices: Sequence[Tuple[int, int, int]],
                kv_reserved: Sequence[int], occupancy: Sequence[int], mix_alpha: float = DEFAULT_MIX_ALPHA) -> List[float]:
    """membership.py:359-387.

    gpus: per registered GPU in ``_gpus`` order, (vram_bytes, reserve_fraction, flops, ram_token_capacity);
    slices: (gpu position in ``gpus``, start, end) in ``slices`` order; kv_reserved / occupancy per ``gpus`` entry.
    """
    total_memory = cpython_sum_model([v * r for v, r, _, _ in gpus])
    total_flops = cpython_sum_model([f for _, _, f, _ in gpus])
    loads = []
    for layer in range(1, layer_count + 1):
        kv_bytes = 0.0
        compute = 0.0
        for g, a, b in slices:
            if not a <= layer <= b:
                continue
            vram, reserve, flops, cap = gpus[g]
            if cap > 0:
                used_fraction = kv_reserved[g] / cap
                kv_bytes += used_fraction * vram * reserve
            compute += flops * min(1, occupancy[g])
        loads.append(layer_load(kv_bytes, compute, total_memory, total_flops, mix_alpha))
    return loads


def evaluate_triggers(layer_count: int, gpus, slices, kv_reserved, occupancy, *, mix_alpha: float = DEFAULT_MIX_ALPHA,
                      cov_threshold: float = DEFAULT_COV_THRESHOLD):
    """membership.py:389-396 -> (scope, reason, cov, uncovered layers, loads)."""
    covered = set()
    for _, a, b in slices:
        covered.update(range(a, b + 1))
    uncovered = tuple(layer for layer in range(1, layer_count + 1) if layer not in covered)
    loads = layer_loads(layer_count, gpus, slices, kv_reserved, occupancy, mix_alpha)
    cov = layer_load_cov(loads)
    if uncovered:
        return "global", "uncovered_layers", cov, uncovered, loads
    if cov > cov_threshold:
        return "global", "load_cov_exceeded", cov, (), loads
    return "local", "balanced", cov, (), loads
