"""Phase-1 oracle -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates ``pkg/src/swarmsched/allocator.py``:
* ``k_max`` 97-101, ``score`` 104-111
* ``_prune_dominated`` 114-135 + ``_sweep`` 138-225   -> :func:`exact_sweep`
* ``_replay`` 228-264                                  -> :func:`sweep_groups`
* ``_best_fit_groups`` 267-350                         -> :func:`best_fit`
* ``_peel_groups`` 353-423                             -> :func:`peel`
* ``_cover_construct`` 426-470                         -> :func:`cover`
* ``solve_stage_counts`` 473-504                       -> :func:`stage_counts`
* ``estimate_objective_params`` 516-538                -> :func:`objective`
* ``allocate`` 541-618                                 -> :func:`allocate`

Results are plain tuples / dicts: ``stage_counts`` -> {k: (stages, groups)};
``allocate`` -> the ``plan_to_dict`` (plan.py:132-154) shape.
"""

from __future__ import annotations

import math
from bisect import bisect_left
from typing import Dict, List, Optional, Sequence, Tuple

from .waterfill_ref import stage_lengths

EXACT_LIMIT = 16   # allocator.py:54


def kmax(caps: Sequence[int], layer_count: int) -> int:
    if layer_count < 1:
        raise ValueError("layer_count must be >= 1")
    return min(len(caps), sum(caps) // layer_count)


def score(k: int, stages: int, alpha: float, t_comp: float, rtt: float) -> float:
    if k < 1 or stages < k:
        raise ValueError("need k >= 1 and stages >= k")
    denom = t_comp + (stages / k) * rtt
    if denom <= 0.0:
        raise ZeroDivisionError("degenerate objective")
    return k ** alpha / denom


# ---------------------------------------------------------------------------
# exact path (<= 16 usable GPUs)
# ---------------------------------------------------------------------------

def _child(res: tuple, slot: Optional[int], cap: int, layer_count: int, done: int):
    if slot is None:                       # start a pipeline
        rem, rest = layer_count - cap, res
    else:                                  # extend the pipeline in slot
        rem, rest = res[slot] - cap, res[:slot] + res[slot + 1:]
    if rem <= 0:
        return (rest, done + 1)
    return (tuple(sorted(rest + (rem,))), done)


def _undominated(tuples: List[tuple]) -> List[tuple]:
    keep: List[tuple] = []
    for cand in sorted(tuples):
        if not any(all(o <= c for o, c in zip(other, cand)) for other in keep):
            keep.append(cand)
    return keep


def exact_sweep(caps: Sequence[int], layer_count: int, max_replicas: int):
    """Level-synchronous stage DP; returns (found{k: level}, parent tables)."""
    n = len(caps)
    tail = [0] * (n + 1)
    for i in range(n - 1, -1, -1):
        tail[i] = tail[i + 1] + caps[i]
    tables = [{((), 0): (((), -1), ())}]
    found: Dict[int, int] = {}
    for i, cap in enumerate(caps):
        children: dict = {}
        for state in sorted(tables[-1]):
            res, done = state
            for slot in range(len(res)):
                if slot and res[slot] == res[slot - 1]:
                    continue
                children.setdefault(_child(res, slot, cap, layer_count, done), (state, ("extend", slot)))
            if done + len(res) < max_replicas:
                children.setdefault(_child(res, None, cap, layer_count, done), (state, ("start",)))
        left = n - i - 1
        classes: Dict[Tuple[int, int], List[tuple]] = {}
        for res, done in children:
            if len(res) <= left and sum(res) <= tail[i + 1]:
                classes.setdefault((done, len(res)), []).append(res)
        level = {}
        for (done, _), group in classes.items():
            for res in _undominated(group):
                level[(res, done)] = children[(res, done)]
        tables.append(level)
        for res, done in level:
            if not res and done >= 1 and done not in found:
                found[done] = i + 1
        if len(found) == max_replicas or not level:
            break
    return found, tables


def sweep_groups(tables, k: int, level: int, caps: Sequence[int], layer_count: int):
    acts = []
    state = ((), k)
    for lv in range(level, 0, -1):
        state, act = tables[lv][state][0], tables[lv][state][1]
        acts.append(act)
    acts.reverse()
    opened: List[Tuple[int, List[int]]] = []
    closed: List[List[int]] = []
    for idx, act in enumerate(acts):
        if act[0] == "start":
            rem, members = layer_count - caps[idx], [idx]
        else:
            rem, members = opened.pop(act[1])
            members.append(idx)
            rem -= caps[idx]
        if rem <= 0:
            closed.append(members)
        else:
            opened.append((rem, members))
            opened.sort(key=lambda item: item[0])
    assert not opened
    return tuple(tuple(g) for g in closed)


# ---------------------------------------------------------------------------
# constructive path (> 16 usable GPUs)
# ---------------------------------------------------------------------------

def best_fit(vals: Sequence[int], m: int, k: int, L: int):
    tot = list(vals[:k])
    grp = [[g] for g in range(k)]
    for i in range(k, m):
        tgt = -1
        for g in range(k):
            if tot[g] < L and (tgt < 0 or tot[g] > tot[tgt]):
                tgt = g
        if tgt < 0:
            break
        tot[tgt] += vals[i]
        grp[tgt].append(i)
    for _ in range(4):
        needy = [g for g in range(k) if tot[g] < L]
        if not needy:
            break
        changed = False
        for u in needy:
            if tot[u] >= L:
                continue
            pick, pick_key = None, None
            for g in range(k):
                if g == u:
                    continue
                for pos, it in enumerate(grp[g]):
                    if len(grp[g]) == 1 or tot[g] - vals[it] < L:
                        continue
                    closes = tot[u] + vals[it] >= L
                    key = (closes, -vals[it] if closes else vals[it])
                    if pick_key is None or key > pick_key:
                        pick_key, pick = key, (g, pos)
            if pick is not None:
                g, pos = pick
                it = grp[g].pop(pos)
                tot[g] -= vals[it]
                tot[u] += vals[it]
                grp[u].append(it)
                changed = True
                continue
            swap, best_gain = None, 0
            for g in range(k):
                if g == u or tot[g] < L:
                    continue
                for gp, b in enumerate(grp[g]):
                    for up, a in enumerate(grp[u]):
                        gain = vals[b] - vals[a]
                        if gain > best_gain and tot[g] - gain >= L:
                            best_gain, swap = gain, (g, gp, up)
            if swap is not None:
                g, gp, up = swap
                grp[g][gp], grp[u][up] = grp[u][up], grp[g][gp]
                tot[g] -= best_gain
                tot[u] += best_gain
                changed = True
        if not changed:
            break
    if any(t < L for t in tot):
        return None
    for g in range(k):
        for it in sorted(grp[g], key=lambda i: vals[i]):
            if len(grp[g]) > 1 and tot[g] - vals[it] >= L:
                grp[g].remove(it)
                tot[g] -= vals[it]
    return grp


def peel(vals: Sequence[int], m: int, k: int, L: int):
    mask = (1 << (2 * L)) - 1
    budget = [300 if m <= 24 else 80]

    def rec(pool: List[int], total: int, need: int):
        if need == 0:
            return []
        if budget[0] <= 0:
            return None
        budget[0] -= 1
        if total < need * L or len(pool) < need:
            return None
        if need == 1:
            short, took = L, []
            for i in pool:
                took.append(i)
                short -= vals[i]
                if short <= 0:
                    return [took]
            return None
        reach = [1]
        for i in pool:
            reach.append(reach[-1] | ((reach[-1] << vals[i]) & mask))
        hi = reach[-1] >> L
        targets, off = [], L
        while hi and len(targets) < 4:
            low = (hi & -hi).bit_length() - 1
            targets.append(off + low)
            hi >>= low + 1
            off += low + 1
        for tgt in targets:
            rem, took = tgt, []
            for pos in range(len(pool) - 1, -1, -1):
                if (reach[pos] >> rem) & 1:
                    continue
                took.append(pool[pos])
                rem -= vals[pool[pos]]
            used = set(took)
            tail = rec([i for i in pool if i not in used], total - tgt, need - 1)
            if tail is not None:
                return [took[::-1]] + tail
        return None

    return rec(list(range(m)), sum(vals[:m]), k)


def cover(caps: Sequence[int], layer_count: int, max_replicas: int):
    n = len(caps)
    vals = [min(c, layer_count) for c in caps]
    prefix = [0]
    for v in vals:
        prefix.append(prefix[-1] + v)
    per_group = -(-layer_count // vals[0])
    out = {}
    for k in range(1, max_replicas + 1):
        need = k * layer_count
        if prefix[n] < need:
            break
        m0 = max(k * per_group, bisect_left(prefix, need))
        groups = None
        for m in range(m0, n + 1):
            groups = best_fit(vals, m, k, layer_count)
            if groups is None:
                groups = peel(vals, m, k, layer_count)
            if groups is not None:
                break
        if groups is None:
            break
        out[k] = (sum(len(g) for g in groups), tuple(tuple(g) for g in groups))
    return out


def stage_counts(caps: Sequence[int], layer_count: int, max_replicas: int):
    caps = tuple(caps)
    if any(a < b for a, b in zip(caps, caps[1:])):
        raise ValueError("capacities must be sorted non-increasing")
    if max_replicas < 1:
        return {}
    usable = tuple(c for c in caps if c > 0)
    if not usable:
        return {}
    if len(usable) > EXACT_LIMIT:
        return cover(usable, layer_count, max_replicas)
    found, tables = exact_sweep(usable, layer_count, max_replicas)
    return {k: (found[k], sweep_groups(tables, k, found[k], usable, layer_count)) for k in sorted(found)}


# ---------------------------------------------------------------------------
# objective and full placement
# ---------------------------------------------------------------------------

def capacity(vram: float, reserve: float, bytes_per_layer: float) -> int:
    """topology.py:148-151."""
    return max(0, math.floor(vram * (1.0 - reserve) / bytes_per_layer + 1e-9))


def objective(flops: Sequence[float], ids: Sequence[str], rtt_fn, fpl: float, layer_count: int,
              tokens: float):
    """(t_comp, rtt) of a region, cluster order (allocator.py:524-537)."""
    inv = sum(1.0 / f for f in flops)
    harmonic = len(flops) / inv
    t_comp = fpl * layer_count * tokens / harmonic
    pairs = [rtt_fn(a, b) for a in ids for b in ids if a != b]
    rtt = sum(pairs) / len(pairs) if pairs else 0.0
    return t_comp, rtt


def allocate(cluster, model, *, alpha: float = 1.0, params=None, mean_tokens_per_request: float = 128.0):
    """Full placement (allocator.py:556-618) -> plan_to_dict-shaped dict, or raises."""
    L = model.layer_count
    pipes, per_k, total = [], [], 0.0
    for region in sorted(cluster.regions):
        members = [g for g in cluster.gpus if g.region == region]
        if not members:
            continue
        tagged = [(capacity(g.vram_bytes, g.reserve_fraction, model.bytes_per_layer), g) for g in members]
        limit = kmax([c for c, _ in tagged], L)
        if limit < 1:
            continue
        tagged.sort(key=lambda cg: (-cg[0], cg[1].id))
        caps = tuple(c for c, _ in tagged)
        order = [g for _, g in tagged]
        sols = stage_counts(caps, L, limit)
        if not sols:
            continue
        if params is not None:
            a, t, r = params.alpha, params.t_comp_seconds, params.rtt_seconds
        else:
            t, r = objective([g.flops for g in members], [g.id for g in members], cluster.rtt_s,
                             model.flops_per_layer_per_token, L, mean_tokens_per_request)
            a = alpha
        z = {k: score(k, s[0], a, t, r) for k, s in sols.items()}
        best = max(z, key=lambda k: (z[k], k))
        for k in sorted(sols):
            per_k.append({"region": region, "k": k, "s_star": sols[k][0], "z": z[k]})
        total += z[best]
        for grp in sols[best][1]:
            nodes = [order[i] for i in grp]
            lens = stage_lengths([g.flops for g in nodes], [caps[i] for i in grp], L)
            stages, cur = [], 1
            for g, n in zip(nodes, lens):
                stages.append({"gpu_id": g.id, "start_layer": cur, "end_layer": cur + n - 1})
                cur += n
            pipes.append({"region": region, "stages": stages})
    if not pipes:
        raise LookupError("no feasible pipeline")
    return {"k": len(pipes), "objective": total, "pipelines": pipes, "per_k": per_k}
