"""Water-filling oracle -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates ``pkg/src/swarmsched/waterfill.py``:
* ``solve_lambda``       47-88   -> :func:`water_level`
* ``hamilton_round``     91-128  -> :func:`largest_remainder`
* ``rebalance_pipeline`` 142-183 -> :func:`stage_lengths`

The fill is evaluated with the interpreter's built-in ``sum`` over the same
int/float item mix as the reference (``min(c, level*f)`` yields the int ``c``
when ``level*f >= c``), so under CPython 3.12 it inherits the Neumaier-
compensated summation the device code must reproduce.
:func:`cpython_sum_model` is the explicit model of that built-in which the CUDA
kernels implement; ``tests/test_oracle_golden.py`` checks it against ``sum``.
"""

from __future__ import annotations

import math
from typing import List, Optional, Sequence, Tuple

TOL_SCALE = 1e-9     # waterfill.py:28
MAX_STEPS = 200      # waterfill.py:29


class WaterfillError(Exception):
    def __init__(self, kind: str, detail=None):
        super().__init__(kind)
        self.kind = kind          # "infeasible" | "overflow" | "zero_capacity" | "value"
        self.detail = detail


def cpython_sum_model(items) -> float:
    """Bit-level model of CPython 3.12 ``sum(items)`` over ints and floats, start 0.

    ints accumulate exactly until the first float; that float is added plainly
    (``float(acc) + x``) and Neumaier compensation starts; later ints are added
    uncompensated; the compensation is folded in at the end when non-zero and
    finite.  Returns an int when every item was an int.
    """
    it = iter(items)
    acc = 0
    for x in it:
        if isinstance(x, int):
            acc += x
            continue
        f = float(acc) + x
        c = 0.0
        for y in it:
            if isinstance(y, float):
                t = f + y
                if abs(f) >= abs(y):
                    c += (f - t) + y
                else:
                    c += (y - t) + f
                f = t
            else:
                f += float(y)
        if c != 0.0 and math.isfinite(c):
            f += c
        return f
    return acc


def water_level(flops: Sequence[float], caps: Sequence[int], layer_count: int):
    """(targets, level) with sum(min(c_i, level*F_i)) == L by bisection (waterfill.py:57-88)."""
    if len(flops) != len(caps) or not flops:
        raise WaterfillError("value")
    if any(f <= 0 for f in flops) or layer_count < 1:
        raise WaterfillError("value")
    have = sum(caps)
    if have < layer_count:
        raise WaterfillError("infeasible", have)

    def fill(level: float):
        return sum(min(c, level * f) for c, f in zip(caps, flops))

    lo = 0.0
    hi = layer_count / min(flops) + 1.0
    tol = TOL_SCALE * layer_count
    steps = 0
    while steps < MAX_STEPS:
        if abs(fill(hi) - layer_count) <= tol:
            break
        mid = 0.5 * (lo + hi)
        if fill(mid) >= layer_count:
            hi = mid
        else:
            lo = mid
        steps += 1
    if abs(fill(hi) - layer_count) > 2.0 * tol:
        raise WaterfillError("overflow")
    return tuple(min(c, hi * f) for c, f in zip(caps, flops)), hi


def largest_remainder(targets: Sequence, caps: Sequence[int], total: Optional[int] = None) -> Tuple[int, ...]:
    """Floor, then +1 by descending remainder (ties: lower index), then spill (waterfill.py:104-128)."""
    if len(targets) != len(caps):
        raise WaterfillError("value")
    if total is None:
        total = round(sum(targets))
    base = [min(math.floor(t), c) for t, c in zip(targets, caps)]
    spare = total - sum(base)
    if spare < 0:
        raise WaterfillError("overflow")
    order = sorted(range(len(targets)), key=lambda i: (-(targets[i] - base[i]), i))
    for i in order:
        if spare == 0:
            break
        if base[i] < caps[i]:
            base[i] += 1
            spare -= 1
    for i in range(len(base)):
        while spare > 0 and base[i] < caps[i]:
            base[i] += 1
            spare -= 1
    if spare > 0:
        raise WaterfillError("overflow")
    return tuple(base)


def stage_lengths(flops: Sequence[float], caps: Sequence[int], layer_count: int) -> List[int]:
    """Whole-layer stage lengths of one pipeline, GPU order kept (waterfill.py:152-176)."""
    for c in caps:
        if c < 1:
            raise WaterfillError("zero_capacity")
    targets, _ = water_level(flops, caps, layer_count)
    counts = list(largest_remainder(targets, caps, layer_count))
    while 0 in counts:
        hole = counts.index(0)
        donor = max(range(len(counts)), key=lambda i: (counts[i], -i))
        if counts[donor] < 2:
            raise WaterfillError("overflow")
        counts[donor] -= 1
        counts[hole] += 1
    return counts
