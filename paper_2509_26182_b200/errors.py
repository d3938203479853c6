"""Scheduler exceptions, name- and field-compatible with the reference.

Mirrors ``pkg/src/swarmsched/errors.py:11-95``: callers branch on the class and
read the structured attribute (``layer``, ``gpu_id``, ``link`` ...), never the
message.  The device C-ABI reports failures as integer status codes
(``include/swarmsched_b200.h``); :func:`raise_for_status` maps a code plus its
aux payload back onto these classes.
"""

from __future__ import annotations


class SchedulerError(Exception):
    """Root of every scheduling failure."""


class DuplicateGpuId(SchedulerError):
    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        super().__init__(f"gpu id {gpu_id!r} appears more than once")


class NegativeRtt(SchedulerError):
    def __init__(self, link, rtt_s: float):
        self.link = tuple(link)
        self.rtt_s = rtt_s
        super().__init__(f"link {self.link[0]!r}->{self.link[1]!r} has invalid rtt {rtt_s!r}")


class UnknownRegion(SchedulerError):
    def __init__(self, gpu_id: str, region: str):
        self.gpu_id = gpu_id
        self.region = region
        super().__init__(f"{gpu_id!r} names region {region!r}, which is not declared")


class InvalidCluster(SchedulerError):
    def __init__(self, violations):
        self.violations = list(violations)
        super().__init__("; ".join(map(str, self.violations)))


class NoFeasiblePipeline(SchedulerError):
    """No region holds enough capacity for one full model replica."""


class DegenerateObjective(SchedulerError):
    """Replication score denominator is not positive."""


class InfeasibleCapacity(SchedulerError):
    def __init__(self, capacity_total: int, layer_count: int):
        self.capacity_total = capacity_total
        self.layer_count = layer_count
        super().__init__(f"{capacity_total} layers of capacity < {layer_count} model layers")


class RoundingOverflow(SchedulerError):
    """Whole-layer rounding could not respect the per-GPU caps."""


class UnknownGpu(SchedulerError):
    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        super().__init__(f"{gpu_id!r} is not a registered gpu")


class ZeroCapacityGpu(SchedulerError):
    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        super().__init__(f"{gpu_id!r} cannot hold one layer")


class UncoveredLayer(SchedulerError):
    def __init__(self, layer: int):
        self.layer = layer
        super().__init__(f"no live host advertises layer {layer}")


class NoPath(SchedulerError):
    """Every layer has hosts but no finite chain connects them."""


class OccupancyUnderflow(SchedulerError):
    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        super().__init__(f"release on {gpu_id!r} has no matching select")


class EmptySample(SchedulerError):
    """Percentile requested over zero samples."""


class DeviceError(SchedulerError):
    """The CUDA extension reported a launch / runtime failure."""


# ---------------------------------------------------------------------------
# C-ABI status codes (include/swarmsched_b200.h, enum ss_status)
# ---------------------------------------------------------------------------
SS_OK = 0
SS_UNCOVERED_LAYER = 1
SS_NO_PATH = 2
SS_OCC_UNDERFLOW = 3
SS_NO_FEASIBLE_PIPELINE = 4
SS_INFEASIBLE_CAPACITY = 5
SS_ROUNDING_OVERFLOW = 6
SS_DEGENERATE_OBJECTIVE = 7
SS_BAD_INPUT = 8
SS_CUDA_ERROR = 9
SS_WORKSPACE = 10
SS_ZERO_CAPACITY = 11


def raise_for_status(code: int, aux: int = 0, *, names=None, detail: str = "", layer_count: int = -1) -> None:
    """Raise the reference exception matching a device status code.

    ``names`` maps an aux node index back to a gpu id when the status carries
    one (OCC_UNDERFLOW, ZERO_CAPACITY); ``layer_count`` completes InfeasibleCapacity(total_cap, layer_count).
    """
    code = int(code)
    if code == SS_OK:
        return
    if code == SS_UNCOVERED_LAYER:
        raise UncoveredLayer(int(aux))
    if code == SS_NO_PATH:
        raise NoPath()
    if code == SS_OCC_UNDERFLOW:
        raise OccupancyUnderflow(names[aux] if names is not None else str(aux))
    if code == SS_NO_FEASIBLE_PIPELINE:
        raise NoFeasiblePipeline(detail or "no feasible pipeline")
    if code == SS_INFEASIBLE_CAPACITY:
        raise InfeasibleCapacity(int(aux), int(layer_count))
    if code == SS_ROUNDING_OVERFLOW:
        raise RoundingOverflow(detail or "rounding overflow")
    if code == SS_DEGENERATE_OBJECTIVE:
        raise DegenerateObjective(detail or "degenerate objective")
    if code == SS_ZERO_CAPACITY:
        raise ZeroCapacityGpu(names[aux] if names is not None else str(aux))
    if code == SS_BAD_INPUT:
        raise ValueError(detail or "bad input to device kernel")
    raise DeviceError(f"device status {code} (aux {aux}) {detail}")
