"""Phase-2 oracle: chain DP over the layer DAG, with occupancy replay.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates:

* ``pkg/src/swarmsched/router.py:87-115``  build_dag  -> :func:`dag_columns`
* ``pkg/src/swarmsched/router.py:118-143`` rtt_matrix -> :func:`dense_rtt`
* ``pkg/src/swarmsched/router.py:157-197`` _relax     -> :func:`relax`
* ``pkg/src/swarmsched/perfmap.py:353-382`` on_chain_event +
  ``sim.py:182-183`` / ``bench.py:150-151`` latency law -> :func:`replay`

Arithmetic is numpy fp64 exactly as the reference: one broadcast add
``cost[:, None] + E`` per boundary, first-occurrence ``argmin`` per column,
then ``+ tau`` -- i.e. the association ``(c_i + r_ij) + tau_j``.
"""

from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

NO_PATH = "no_path"


def dag_columns(latencies: Dict[Tuple[str, int], float], layer_count: int, exclude=frozenset()):
    """Sorted host columns per layer (router.py:99-110).

    Returns (columns, uncovered_layer) where uncovered_layer is the lowest
    1-based layer with no host (columns is then None), else 0.
    """
    per = {}
    for (gpu, layer) in latencies:
        if gpu in exclude or not (1 <= layer <= layer_count):
            continue
        per.setdefault(layer, []).append(gpu)
    cols = []
    for layer in range(1, layer_count + 1):
        hosts = per.get(layer)
        if not hosts:
            return None, layer
        cols.append(tuple(sorted(hosts)))
    return cols, 0


def dense_rtt(entries: Sequence[Tuple[str, str, float]], ids: Sequence[str]) -> np.ndarray:
    """inf off-diagonal, 0 diagonal; direct entry wins over mirrored reverse (router.py:128-143)."""
    pos = {g: i for i, g in enumerate(ids)}
    out = np.full((len(ids), len(ids)), np.inf)
    np.fill_diagonal(out, 0.0)
    pending = []
    for a, b, v in entries:
        ia, ib = pos.get(a), pos.get(b)
        if ia is None or ib is None or ia == ib:
            continue
        out[ia, ib] = v
        pending.append((ib, ia, v))
    for r, c, v in pending:
        if not np.isfinite(out[r, c]):
            out[r, c] = v
    return out


def relax(col_idx: List[np.ndarray], col_tau: List[np.ndarray], rtt: np.ndarray):
    """Min-plus DP over the columns (router.py:163-185).

    col_idx[l]: dense matrix indices of layer l's hosts in sorted order;
    col_tau[l]: their tau.  Returns (picks, cost) with picks[l] the position
    inside column l, or (None, NO_PATH).
    """
    cost = np.asarray(col_tau[0], dtype=np.float64).copy()
    backs = []
    for l in range(1, len(col_idx)):
        cand = cost[:, None] + rtt[np.ix_(col_idx[l - 1], col_idx[l])]
        arg = np.argmin(cand, axis=0)
        cost = cand[arg, np.arange(cand.shape[1])] + col_tau[l]
        backs.append(arg)
    last = int(np.argmin(cost))
    total = float(cost[last])
    if not np.isfinite(total):
        return None, NO_PATH
    picks = [last]
    for arg in reversed(backs):
        picks.append(int(arg[picks[-1]]))
    picks.reverse()
    return picks, total


def merge_hops(assignment: Sequence[str]) -> List[Tuple[str, int, int]]:
    """Consecutive equal hosts collapse into one (gpu, start, end) slice (router.py:188-194)."""
    hops = []
    start = 1
    for layer in range(2, len(assignment) + 1):
        if assignment[layer - 1] != assignment[layer - 2]:
            hops.append((assignment[layer - 2], start, layer - 1))
            start = layer
    hops.append((assignment[-1], start, len(assignment)))
    return hops


def select(latencies, layer_count, link_entries, exclude=frozenset()):
    """select_chain(build_dag(snapshot), snapshot) restated (router.py:200-205).

    Returns ("ok", hops, cost) / ("uncovered", layer) / ("no_path",).
    """
    cols, missing = dag_columns(latencies, layer_count, exclude)
    if cols is None:
        return ("uncovered", missing)
    ids = sorted({g for c in cols for g in c})
    pos = {g: i for i, g in enumerate(ids)}
    rtt = dense_rtt(link_entries, ids)
    col_idx = [np.array([pos[g] for g in c]) for c in cols]
    col_tau = [np.array([latencies[(g, l + 1)] for g in c]) for l, c in enumerate(cols)]
    picks, cost = relax(col_idx, col_tau, rtt)
    if picks is None:
        return ("no_path",)
    assign = [cols[l][p] for l, p in enumerate(picks)]
    return ("ok", merge_hops(assign), cost)


# ---------------------------------------------------------------------------
# Replay with on-device-equivalent load update
# ---------------------------------------------------------------------------

def occ_power_table(size: int, exponent: float = 1.0) -> np.ndarray:
    """occpow[o] = (1 + o) ** e evaluated with Python's ``**`` (sim.py:183)."""
    return np.array([float((1 + o) ** exponent) for o in range(size)], dtype=np.float64)


def replay(columns: List[np.ndarray], base: np.ndarray, rtt: np.ndarray, n_requests: int,
           window: Optional[int], occpow: np.ndarray, occ: Optional[np.ndarray] = None,
           start: int = 0, live: Optional[list] = None):
    """Route ``n_requests`` requests through one scenario with feedback.

    columns[l]: sorted GPU indices hosting layer l+1 (index order = sorted id
    order); base[g] = flops_per_layer_per_token / flops_g; rtt: dense matrix
    over the same GPU indices.  tau(g) = base[g] * occpow[occ[g]] is what
    ``on_chain_event`` republishes for every hosted layer (perfmap.py:375-382
    with the layer-independent law of sim.py:182-183 / bench.py:150-151), so
    the per-(gpu, layer) table collapses to a per-GPU vector.

    Op script: before request i, release chain i-W if i >= W
    (window None = never release, window 0 = release right after select).
    Returns (picks[list], costs[list], occ, live) so calls can be chained.
    """
    n_gpu = base.shape[0]
    occ = np.zeros(n_gpu, dtype=np.int64) if occ is None else occ.copy()
    live = [] if live is None else list(live)
    all_picks, costs = [], []
    for i in range(start, start + n_requests):
        if window is not None and window > 0 and i >= window:
            gone = live.pop(0)
            occ[gone] -= 1
        tau = base * occpow[occ]
        picks, cost = relax(columns, [tau[c] for c in columns], rtt)
        if picks is None:
            raise RuntimeError(f"NoPath at request {i}")
        gpus = [int(columns[l][p]) for l, p in enumerate(picks)]
        distinct = list(dict.fromkeys(gpus))
        occ[distinct] += 1
        if window == 0:
            occ[distinct] -= 1
        elif window is not None:
            live.append(distinct)
        all_picks.append(gpus)
        costs.append(cost)
    return all_picks, costs, occ, live
