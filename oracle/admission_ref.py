"""CPU restatement of the admission path (TEST INFRASTRUCTURE ONLY -- the checker, never the product path).

sim.py:319-366 on the time-free step schedule of tests/golden/make_admission_golden.py: at step t the chains
admitted at step t - W complete (router.release + release_kv, sim.py:353-357), request t joins the back of
the queue, and the queue drains strictly FIFO (sim.py:345-351).  Admission (sim.py:319-338) routes with
exclude = {g : ram_token_capacity - kv_reserved < tokens}; here exclusion is a +inf latency on the excluded
GPUs instead of removing them from the columns, which selects the same chain: an excluded host only ever
carries +inf candidates, finite candidates keep their relative (sorted-id) order, and a head with no finite
chain (UncoveredLayer or NoPath in the reference) fails either way.
"""

from __future__ import annotations

import collections
from typing import List, Optional, Sequence

import numpy as np

from . import chain_ref


def admission_replay(columns: List[np.ndarray], base: np.ndarray, rtt: np.ndarray, token_cap: np.ndarray,
                     tokens: Sequence[int], steps: int, window: int, occpow: np.ndarray):
    """Returns (admitted[i] = (step, gpus per layer, cost) or None, queue left, kv_reserved, occupancy)."""
    n = base.shape[0]
    occ = np.zeros(n, dtype=np.int64)
    kv = np.zeros(n, dtype=np.int64)
    queue = collections.deque()
    live = collections.deque()                    # (step, distinct gpus, tokens)
    admitted: List[Optional[tuple]] = [None] * steps
    for t in range(steps):
        while live and live[0][0] == t - window:
            _, d, tok = live.popleft()
            occ[d] -= 1
            kv[d] -= tok
        queue.append(t)
        while queue:
            i = queue[0]
            tok = int(tokens[i])
            tau = base * occpow[occ]
            tau = np.where(token_cap - kv < tok, np.inf, tau)
            picks, cost = chain_ref.relax(columns, [tau[c] for c in columns], rtt)
            if picks is None:
                break
            gpus = [int(columns[l][p]) for l, p in enumerate(picks)]
            d = list(dict.fromkeys(gpus))
            occ[d] += 1
            kv[d] += tok
            live.append((t, d, tok))
            queue.popleft()
            admitted[i] = (t, gpus, cost)
    return admitted, list(queue), kv, occ
