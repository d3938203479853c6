"""CPU restatement of the serving simulator (TEST INFRASTRUCTURE ONLY -- the checker, never the product path).

pkg/src/swarmsched/sim.py:_Simulation without membership events, operation for operation:
* one event heap keyed (time, seq); arrivals pushed first in trace order, then the publish tick
  (sim.py:260-265); a tick re-arms itself while work remains and changes nothing else the router reads
  (republish_all refreshes TTLs with unchanged values), but it advances the clock, so duration_s is the
  time of the last tick (sim.py:432-436, 454);
* admission (sim.py:319-338): KV-blocked GPUs excluded (+inf latency here -- the same chain), reserve
  total_tokens on the chain's distinct GPUs, occupancy +1, prefill event at now + _prefill_s;
* _prefill_s = sum(base_s * hop.length) [CPython compensated sum] * prompt_tokens + chain RTT;
  _step_s = sum over hops of (base_s * max(1, occ) ** e) * hop.length [plain fold] + chain RTT unless
  amortized (sim.py:298-317), occupancy read when the step starts;
* completion (sim.py:394-399): release, latency = now - arrival, then the strict FIFO drain.
Pinned by tests/golden/sim_cases.json.
"""

from __future__ import annotations

import heapq
import math
from typing import List, Sequence, Tuple

import numpy as np

from . import chain_ref
from .waterfill_ref import cpython_sum_model

ARRIVAL, PREFILL, STEP, PUBLISH = 0, 1, 2, 3


def hops_of(gpus: Sequence[int]) -> List[Tuple[int, int]]:
    """(gpu, length) per merged hop (router.py:188-194)."""
    out = []
    for g in gpus:
        if out and out[-1][0] == g:
            out[-1] = (g, out[-1][1] + 1)
        else:
            out.append((g, 1))
    return out


def chain_rtt(hops, rtt) -> float:
    total = 0.0
    for (a, _), (b, _) in zip(hops, hops[1:]):
        if a != b:
            total += rtt[a, b]
    return total


def simulate(columns, base: np.ndarray, rtt: np.ndarray, token_cap: np.ndarray, trace, *, amortize_rtt=False,
             contention=1.0, publish_interval=1.5):
    """trace: [(arrival_s, prompt_tokens, output_tokens)] in arrival order.  Returns (report dict, latencies in
    completion order, completion time per request or None)."""
    n = base.shape[0]
    occ = np.zeros(n, dtype=np.int64)
    kv = np.zeros(n, dtype=np.int64)
    pw_pub = lambda o: float((1 + o) ** contention)
    pw_exec = lambda o: float(max(1, o) ** contention)
    heap, seq = [], 0

    def push(t, kind, payload):
        nonlocal seq
        heapq.heappush(heap, (t, seq, kind, payload))
        seq += 1

    order = sorted(range(len(trace)), key=lambda i: trace[i][0])
    for i in order:
        push(trace[i][0], ARRIVAL, i)
    live = {}
    queue, qseq, peak = [], 0, 0
    arrivals_left = len(trace)
    if live or arrivals_left:
        push(publish_interval, PUBLISH, None)
    latencies, done_at = [], [None] * len(trace)
    completed, now = 0, 0.0

    def try_admit(i, t):
        arr, prompt, out = trace[i]
        tok = prompt + out
        tau = np.array([base[g] * pw_pub(occ[g]) for g in range(n)])
        tau = np.where(token_cap - kv < tok, np.inf, tau)
        picks, cost = chain_ref.relax(columns, [tau[c] for c in columns], rtt)
        if picks is None:
            return False
        gpus = [int(columns[l][p]) for l, p in enumerate(picks)]
        d = list(dict.fromkeys(gpus))
        occ[d] += 1
        kv[d] += tok
        hops = hops_of(gpus)
        compute = cpython_sum_model([base[g] * ln for g, ln in hops])
        pre = compute * prompt + chain_rtt(hops, rtt)
        live[i] = [d, hops, out, tok]
        push(t + pre, PREFILL, i)
        return True

    def step_s(hops):
        total = 0.0
        for g, ln in hops:
            total += (base[g] * pw_exec(occ[g])) * ln
        if not amortize_rtt:
            total += chain_rtt(hops, rtt)
        return total

    def complete(i, t):
        nonlocal completed
        d, _, _, tok = live.pop(i)
        occ[d] -= 1
        kv[d] -= tok
        latencies.append(t - trace[i][0])
        done_at[i] = t
        completed += 1
        while queue:
            j = queue[0][2]
            if not try_admit(j, t):
                break
            heapq.heappop(queue)

    while heap:
        t, _, kind, p = heapq.heappop(heap)
        now = t
        if kind == ARRIVAL:
            arrivals_left -= 1
            if queue or not try_admit(p, t):
                heapq.heappush(queue, (trace[p][0], qseq, p))
                qseq += 1
                peak = max(peak, len(queue))
        elif kind == PREFILL or kind == STEP:
            entry = live[p]
            if kind == STEP:
                entry[2] -= 1
            if entry[2] == 0:
                complete(p, t)
            else:
                push(t + step_s(entry[1]), STEP, p)
        else:
            if live or arrivals_left:
                push(t + publish_interval, PUBLISH, None)
    duration = now
    mean = p50 = p95 = p99 = 0.0
    if latencies:
        mean = cpython_sum_model(latencies) / len(latencies)
        srt = sorted(latencies)
        rank = lambda q: srt[max(1, math.ceil(q * len(srt) / 100.0)) - 1]
        p50, p95, p99 = rank(50), rank(95), rank(99)
    report = {"submitted": len(trace), "completed": completed, "unserved": len(trace) - completed, "aborted": 0,
              "duration_s": duration, "throughput_rps": completed / duration if duration > 0 else 0.0,
              "latency_mean_s": mean, "latency_p50_s": p50, "latency_p95_s": p95, "latency_p99_s": p99,
              "queue_peak": peak}
    return report, latencies, done_at
