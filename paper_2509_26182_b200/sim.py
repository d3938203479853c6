"""Serving-simulator entry points of the drop-in (``pkg/src/swarmsched/sim.py``), backed by the device simulator.

Same names, fields and semantics as the reference for the pieces the hot path feeds:

* ``Request`` (sim.py:62-76), the trace wire format ``request_from_dict`` / ``request_to_dict`` /
  ``load_trace`` / ``save_trace`` (79-115, JSON lines ``{"id", "t", "prompt_tokens", "output_tokens"}``);
* ``generate_trace`` (118-148): Poisson arrivals from ``random.Random(seed)``, ids ``r00000``...;
* ``percentile`` (151-159, nearest rank), ``LatencyModel`` (161-186, the tau law of the device replays) and
  ``MetricsReport`` (190-217);
* ``baseline_plan`` (513-553): the naive placement the simulator is compared against (capacity-sorted first fit,
  equal-speed water-fill through the device ``solve_lambda`` / ``hamilton_round``);
* ``run_simulation`` (478-510): the discrete-event serving simulation of one cluster / plan / trace.  The event
  loop runs on the GPU (``ss_sim_warp`` for <= 32 hosts per layer, ``ss_sim_cta`` up to 256) through
  ``ScenarioReplayer.simulate``; this wrapper only packs the pool and unpacks the report.

Not on the device path: membership events inside the simulator timeline (``sim.py:_on_membership``) -- the batched
replayer runs that loop instead (``ScenarioReplayer.rebalance``) -- and latency entries that expire between publish
ticks (``ttl_multiplier < 1``).  Both raise ``NotImplementedError`` rather than silently diverging.
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from typing import Iterable, List, Sequence, Tuple

import numpy as np

from .errors import EmptySample, NoFeasiblePipeline
from .perfmap import DEFAULT_PUBLISH_INTERVAL_S, DEFAULT_TTL_MULTIPLIER
from .plan import AllocationPlan, Pipeline
from .topology import ClusterSnapshot, LayerSlice, ModelSpec, layer_capacity


@dataclass(frozen=True)
class Request:
    id: str
    arrival_s: float
    prompt_tokens: int
    output_tokens: int

    def __post_init__(self) -> None:
        if self.prompt_tokens < 1:
            raise ValueError(f"prompt_tokens must be >= 1, got {self.prompt_tokens}")
        if self.output_tokens < 0:
            raise ValueError(f"output_tokens must be >= 0, got {self.output_tokens}")

    @property
    def total_tokens(self) -> int:
        return self.prompt_tokens + self.output_tokens


def request_from_dict(raw: dict) -> Request:
    return Request(id=str(raw["id"]), arrival_s=float(raw["t"]), prompt_tokens=int(raw["prompt_tokens"]),
                   output_tokens=int(raw["output_tokens"]))


def request_to_dict(request: Request) -> dict:
    return {"id": request.id, "t": request.arrival_s, "prompt_tokens": request.prompt_tokens,
            "output_tokens": request.output_tokens}


def load_trace(path: str) -> List[Request]:
    """JSON-lines trace, blank lines skipped, sorted by arrival (stable)."""
    out = []
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, 1):
            line = line.strip()
            if not line:
                continue
            try:
                out.append(request_from_dict(json.loads(line)))
            except (TypeError, KeyError, AttributeError) as exc:
                raise ValueError(f"{path}:{lineno}: bad trace line ({exc})") from exc
    out.sort(key=lambda r: r.arrival_s)
    return out


def save_trace(requests: Iterable[Request], path: str) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        for r in requests:
            fh.write(json.dumps(request_to_dict(r), sort_keys=True) + "\n")


def generate_trace(rate_rps: float, duration_s: float, *, seed: int = 0, prompt_tokens: Tuple[int, int] = (32, 256),
                   output_tokens: Tuple[int, int] = (16, 128)) -> List[Request]:
    """Poisson arrivals at rate_rps over [0, duration_s) with uniform token counts (the reference's draws)."""
    from .scenarios import generate_trace as draws
    arrival, prompt, output = draws(rate_rps, duration_s, seed=seed, prompt_tokens=tuple(prompt_tokens),
                                    output_tokens=tuple(output_tokens))
    return [Request(f"r{i:05d}", float(a), int(p), int(o))
            for i, (a, p, o) in enumerate(zip(arrival.tolist(), prompt.tolist(), output.tolist()))]


def percentile(values: Sequence[float], p: float) -> float:
    """Nearest-rank percentile, p in (0, 100]."""
    if not values:
        raise EmptySample("percentile of an empty sample")
    if not 0.0 < p <= 100.0:
        raise ValueError(f"p must be in (0, 100], got {p}")
    ordered = sorted(values)
    return ordered[max(1, math.ceil(p * len(ordered) / 100.0)) - 1]


class LatencyModel:
    """Per-layer step time from GPU speed plus a contention multiplier (sim.py:161-186): the tau law every device
    replay applies, tau(g) = base(g) * occpow[occ(g)] with base(g) = flops_per_layer_per_token / flops(g) and
    occpow[o] = (1 + o) ** e (``batched.occ_power_table``).

    ``manager`` is anything with ``gpu(gpu_id) -> GpuNode`` -- the reference passes its MembershipManager; a
    ``ClusterSnapshot`` works the same way here.
    """

    def __init__(self, model: ModelSpec, manager, contention_exponent: float = 1.0):
        self.model = model
        self.manager = manager
        self.contention_exponent = contention_exponent

    def base_s(self, gpu_id: str) -> float:
        return self.model.flops_per_layer_per_token / self.manager.gpu(gpu_id).flops

    def published(self, gpu_id: str, layer: int, occupancy: int) -> float:
        """What the GPU advertises: the step time a new chain would see (occupancy + itself)."""
        return self.base_s(gpu_id) * (1 + occupancy) ** self.contention_exponent

    def executing(self, gpu_id: str, live_chains: int) -> float:
        return self.base_s(gpu_id) * max(1, live_chains) ** self.contention_exponent


@dataclass(frozen=True)
class MetricsReport:
    submitted: int
    completed: int
    unserved: int
    aborted: int
    duration_s: float
    throughput_rps: float
    latency_mean_s: float
    latency_p50_s: float
    latency_p95_s: float
    latency_p99_s: float
    queue_peak: int

    def to_dict(self) -> dict:
        return {name: getattr(self, name) for name in self.__dataclass_fields__}


def run_simulation(cluster: ClusterSnapshot, model: ModelSpec, plan: AllocationPlan, trace: Sequence[Request], *,
                   membership_events: Sequence = (), publish_interval_s: float = DEFAULT_PUBLISH_INTERVAL_S,
                   ttl_multiplier: float = DEFAULT_TTL_MULTIPLIER, contention_exponent: float = 1.0,
                   amortize_rtt: bool = False, mix_alpha: float = 0.5, cov_threshold: float = 0.5, alpha: float = 1.0,
                   mean_tokens_per_request: float = 128.0) -> MetricsReport:
    """Run the trace against the plan on the GPU and report latency / throughput (sim.py:478-510).

    mix_alpha, cov_threshold, alpha and mean_tokens_per_request only steer membership handling, which this entry
    point does not run (see the module docstring).
    """
    if len(membership_events):
        raise NotImplementedError("membership events inside the simulator timeline are not on the device path; "
                                  "use batched.ScenarioReplayer.rebalance for the churn / rebalance loop")
    if ttl_multiplier < 1.0:
        raise NotImplementedError("ttl_multiplier < 1 lets latency entries expire between publish ticks; "
                                  "the device simulator keeps every entry live")
    from . import scenarios as scen
    from .batched import ScenarioReplayer, replay_mode
    ss = scen.build_scenarios(cluster, model, plan, 1, churn=0.0, jitter=False)
    mode = "warp" if replay_mode(ss, window=1) == "warp" else "blocks"
    order = sorted(range(len(trace)), key=lambda i: trace[i].arrival_s)       # arrival order, ties by position
    arrays = (np.array([trace[i].arrival_s for i in order], dtype=np.float64),
              np.array([trace[i].prompt_tokens for i in order], dtype=np.int32),
              np.array([trace[i].output_tokens for i in order], dtype=np.int32))
    rp = ScenarioReplayer(ss, window=1, mode=mode)
    rep = rp.simulate([arrays], publish_interval=float(publish_interval_s), amortize_rtt=bool(amortize_rtt),
                      contention=float(contention_exponent))[0]
    return MetricsReport(**{name: rep[name] for name in MetricsReport.__dataclass_fields__})


def baseline_plan(cluster: ClusterSnapshot, model: ModelSpec) -> AllocationPlan:
    """Naive placement (sim.py:513-553): GPUs by (-capacity, id) regardless of region, grouped first-fit until a
    group can hold the model; each group's layers split by an equal-speed water-fill + Hamilton rounding; GPUs of
    an unfinished last group stay unused.  objective 0.0, no per-k table."""
    from .waterfill import hamilton_round, solve_lambda
    L = model.layer_count
    caps_of = {g.id: layer_capacity(g, model) for g in cluster.gpus}
    usable = [g for g in sorted(cluster.gpus, key=lambda g: (-caps_of[g.id], g.id)) if caps_of[g.id] >= 1]
    pipelines: List[Pipeline] = []
    group: List[Tuple[str, int]] = []
    acc = 0
    for g in usable:
        group.append((g.id, caps_of[g.id]))
        acc += caps_of[g.id]
        if acc < L:
            continue
        caps = [c for _, c in group]
        rounded = hamilton_round(solve_lambda([1.0] * len(group), caps, L), caps, total=L)
        stages, cursor = [], 1
        for (gid, _), count in zip(group, rounded.layers):
            stages.append(LayerSlice(gid, cursor, cursor + count - 1))
            cursor += count
        regions = {cluster.gpu(gid).region for gid, _ in group}
        pipelines.append(Pipeline(stages=tuple(stages), region=regions.pop() if len(regions) == 1 else None))
        group, acc = [], 0
    if not pipelines:
        raise NoFeasiblePipeline()
    return AllocationPlan(replication_count=len(pipelines), pipelines=tuple(pipelines),
                          stage_total=sum(p.stage_count for p in pipelines), objective_score=0.0, per_k_table=())
