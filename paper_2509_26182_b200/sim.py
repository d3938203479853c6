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

Membership events inside the simulator timeline (``sim.py:_on_membership``, 401-430) and latency entries that
expire between publish ticks (``ttl_multiplier < 1``) change the serving DAG between admissions: those runs use
``_HostTimeline`` -- the reference's event order on the host, every route on the device ``ChainRouter``, every
global rebalance through the device ``allocate()``, the drop-in ``MembershipManager`` (membership.py).
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
    """Run the trace against the plan and report latency / throughput (sim.py:478-510).

    Without membership events (and with ttl_multiplier >= 1) the whole event loop runs on the GPU
    (``ScenarioReplayer.simulate``).  With them, ``_HostTimeline`` replays the reference timeline on the host with
    every route on the device (``ChainRouter``) and every global rebalance through the device ``allocate()``;
    mix_alpha, cov_threshold, alpha and mean_tokens_per_request steer that membership handling.
    """
    if len(membership_events) or ttl_multiplier < 1.0:
        # membership changes the serving DAG mid-timeline (and a short TTL lets entries expire between ticks):
        # the host timeline below routes every admission through the device ChainRouter instead
        return _HostTimeline(cluster, model, plan, trace, membership_events, publish_interval_s, ttl_multiplier,
                             contention_exponent, amortize_rtt, mix_alpha, cov_threshold, alpha,
                             mean_tokens_per_request).run()
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


class _HostTimeline:
    """The serving simulation of sim.py:226-475 with membership events: a host event heap ordered by (time, push
    sequence) like the reference's, over the drop-in PerfMap / MembershipManager / LatencyModel, routing on the
    device (``ChainRouter.route``, KV-blocked GPUs excluded) and re-placing the pool with the device ``allocate()``.

    Per request: admission reserves total_tokens on the chain's distinct GPUs and schedules the prefill at
    now + sum(base_s * hop.length) * prompt + chain RTT; each later step lasts the sum over hops of
    executing(gpu, occupancy) * hop.length (+ the chain RTT unless amortized); a chain aborted by a leave or a
    rebalance is released and re-queued under its original arrival time with a new generation, so its stale
    prefill / step events are dropped.  The queue drains strictly FIFO by (arrival, enqueue order).
    """

    ARRIVAL, PREFILL, STEP, MEMBER, PUBLISH = range(5)

    def __init__(self, cluster, model, plan, trace, events, publish_interval_s, ttl_multiplier, contention_exponent,
                 amortize_rtt, mix_alpha, cov_threshold, alpha, mean_tokens_per_request):
        import heapq
        from .membership import MembershipManager
        from .perfmap import PerfMap
        from .router import ChainRouter
        self._heapq = heapq
        self.publish_interval_s = publish_interval_s
        self.amortize_rtt = amortize_rtt
        self.pm = PerfMap(ttl_s=publish_interval_s * ttl_multiplier)
        self.mgr = MembershipManager(cluster, model, self.pm, mix_alpha=mix_alpha, cov_threshold=cov_threshold,
                                     alpha=alpha, mean_tokens_per_request=mean_tokens_per_request)
        self.lat = LatencyModel(model, self.mgr, contention_exponent)
        self.pm.latency_fn = self.lat.published
        self.mgr.initialize(plan, 0.0)
        self.router = ChainRouter(self.pm, model.layer_count)
        self.heap: list = []
        self.seq = 0
        self.live: dict = {}            # request id -> [request, chain, remaining steps, generation]
        self.gen: dict = {}
        self.queue: list = []           # (arrival_s, enqueue order, request)
        self.qseq = 0
        self.qpeak = 0
        self.latencies: List[float] = []
        self.submitted = len(trace)
        self.completed = self.aborted = 0
        self.arrivals_left = len(trace)
        self.members_left = len(events)
        self.now = 0.0
        for req in sorted(trace, key=lambda r: r.arrival_s):
            self._push(req.arrival_s, self.ARRIVAL, req)
        for ev in sorted(events, key=lambda e: e.at_s):
            self._push(ev.at_s, self.MEMBER, ev)
        if self._work_remains():
            self._push(publish_interval_s, self.PUBLISH, None)

    def _push(self, at_s: float, kind: int, payload) -> None:
        self._heapq.heappush(self.heap, (at_s, self.seq, kind, payload))
        self.seq += 1

    def _work_remains(self) -> bool:
        return bool(self.live) or self.arrivals_left > 0 or self.members_left > 0

    def _chain_rtt(self, chain) -> float:
        t = 0.0
        for a, b in zip(chain.hops, chain.hops[1:]):
            if a.gpu_id != b.gpu_id:
                t += self.mgr.rtt_s(a.gpu_id, b.gpu_id)
        return t

    def _step_time(self, chain) -> float:
        t = 0.0
        for hop in chain.hops:
            t += self.lat.executing(hop.gpu_id, self.pm.occupancy(hop.gpu_id)) * hop.length
        return t if self.amortize_rtt else t + self._chain_rtt(chain)

    def _enqueue(self, req) -> None:
        self._heapq.heappush(self.queue, (req.arrival_s, self.qseq, req))
        self.qseq += 1
        self.qpeak = max(self.qpeak, len(self.queue))

    def _admit(self, req, now: float) -> bool:
        from .errors import NoPath, UncoveredLayer
        tokens = req.total_tokens
        blocked = {g for g in self.mgr.gpu_ids() if self.mgr.kv_headroom(g) < tokens}
        try:
            chain = self.router.route(now, exclude=blocked)
        except (UncoveredLayer, NoPath):
            return False
        for g in set(chain.gpu_ids):
            self.mgr.reserve_kv(g, tokens)
        gen = self.gen.get(req.id, 0) + 1
        self.gen[req.id] = gen
        self.live[req.id] = [req, chain, req.output_tokens, gen]
        compute = sum(self.lat.base_s(h.gpu_id) * h.length for h in chain.hops)
        self._push(now + (compute * req.prompt_tokens + self._chain_rtt(chain)), self.PREFILL, (req.id, gen))
        return True

    def _drain(self, now: float) -> None:
        while self.queue and self._admit(self.queue[0][2], now):
            self._heapq.heappop(self.queue)

    def _release(self, entry, now: float) -> None:
        req, chain = entry[0], entry[1]
        self.router.release(chain, now)
        for g in set(chain.gpu_ids):
            self.mgr.release_kv(g, req.total_tokens)

    def _fresh(self, payload):
        rid, gen = payload
        entry = self.live.get(rid)
        return entry if entry is not None and entry[3] == gen else None

    def _advance(self, payload, now: float, first: bool) -> None:
        entry = self._fresh(payload)
        if entry is None:
            return                                  # aborted since this event was scheduled
        if not first:
            entry[2] -= 1
        if entry[2] == 0:
            self._release(entry, now)
            del self.live[entry[0].id]
            self.latencies.append(now - entry[0].arrival_s)
            self.completed += 1
            self._drain(now)
        else:
            self._push(now + self._step_time(entry[1]), self.STEP, payload)

    def _abort_on(self, gpu_ids, now: float) -> None:
        hit = [e for e in self.live.values() if gpu_ids.intersection(e[1].gpu_ids)]
        for e in sorted(hit, key=lambda e: e[0].id):
            self._release(e, now)
            del self.live[e[0].id]
            self.aborted += 1
            self._enqueue(e[0])                     # restarts from prefill, arrival time kept

    def _membership(self, ev, now: float) -> None:
        from .errors import ZeroCapacityGpu
        from .membership import LEAVE
        self.members_left -= 1
        if ev.kind == LEAVE:
            self._abort_on({ev.gpu_id}, now)        # release first: the GPU must still be registered
            self.mgr.on_leave(ev.gpu_id, now)
        else:
            try:
                self.mgr.on_join(ev.gpu, now)
            except ZeroCapacityGpu:
                pass
        if self.mgr.evaluate_triggers().is_global:
            res = self.mgr.global_rebalance(now)
            if not res.degraded:
                self._abort_on(set(res.changed_gpus), now)
        self._drain(now)

    def run(self) -> MetricsReport:
        heap = self.heap
        while heap:
            at_s, _, kind, payload = self._heapq.heappop(heap)
            self.now = at_s
            if kind == self.ARRIVAL:
                self.arrivals_left -= 1
                if self.queue or not self._admit(payload, at_s):
                    self._enqueue(payload)
            elif kind == self.PREFILL:
                self._advance(payload, at_s, True)
            elif kind == self.STEP:
                self._advance(payload, at_s, False)
            elif kind == self.MEMBER:
                self._membership(payload, at_s)
            elif self._work_remains():                 # publish tick
                self.mgr.republish_all(at_s)
                self._push(at_s + self.publish_interval_s, self.PUBLISH, None)
        lat = self.latencies
        dur = self.now
        if lat:
            stats = (sum(lat) / len(lat), percentile(lat, 50), percentile(lat, 95), percentile(lat, 99))
        else:
            stats = (0.0, 0.0, 0.0, 0.0)
        return MetricsReport(submitted=self.submitted, completed=self.completed,
                             unserved=self.submitted - self.completed, aborted=self.aborted, duration_s=dur,
                             throughput_rps=self.completed / dur if dur > 0 else 0.0, latency_mean_s=stats[0],
                             latency_p50_s=stats[1], latency_p95_s=stats[2], latency_p99_s=stats[3],
                             queue_peak=self.qpeak)


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
