"""Synthetic pools and replay scenarios for the SURVEY.md 8(d) configs C1-C5.

* :func:`synthetic_cluster` reproduces ``pkg/src/swarmsched/bench.py:91-130``
  draw for draw (``random.Random(seed)``: capacity ``randint(4, 32)``, flops
  ``uniform(6e13, 2.4e14)``, round-robin regions, 1 ms intra-region links,
  10 ms default across), so a pool built here is the reference's pool.
* Scenario states (C4/C5) are the base pool after churn (a seeded set of plan
  GPUs leaves, as ``MembershipManager.on_leave`` would, no rebalance) and with
  a seeded per-pair RTT jitter: one LogNormal(0, 0.2) factor per unordered GPU
  pair, quantile ``jitter_index(seed, i, j)`` (a 32-bit pair
  hash, top 10 bits) of the 1024-point float32 grid in ``csrc/jitter_lognormal.inc``.  Kernels and
  host read the same committed table, so the device generators
  (``ss_scenario_rtt``, the edge / unit writers) and the host/oracle produce
  bit-identical RTTs: ``rtt_ab * Q[jitter_index(seed, a, b)]``.
"""

from __future__ import annotations

import os
import random
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from .topology import ClusterSnapshot, GpuNode, ModelSpec

CAPACITY_RANGE = (4, 32)
FLOPS_RANGE = (6e13, 2.4e14)
INTRA_REGION_RTT_S = 0.001
MASK64 = (1 << 64) - 1


def bench_model(layer_count: int = 48, name: Optional[str] = None) -> ModelSpec:
    """The bench's model shape (bench.py:116-121) at a given depth."""
    return ModelSpec(name or f"bench-{layer_count}l", layer_count, 1.2e9, 2.8e10)


def default_region_count(gpu_count: int) -> int:
    return max(1, min(4, gpu_count // 8))


def synthetic_cluster(gpu_count: int, *, seed: int = 0, region_count: Optional[int] = None,
                      model: Optional[ModelSpec] = None, homogeneous_flops: Optional[float] = None,
                      id_prefix: str = "gpu-", links: Optional[Dict] = None) -> Tuple[ClusterSnapshot, ModelSpec]:
    """Pool drawn exactly like the reference bench (bench.py:114-138).

    ``homogeneous_flops`` overrides every GPU's flops after the draw (the
    tie-heavy fixture of SURVEY.md 8(d)); the random stream is unchanged.
    ``links`` replaces the intra-region link table (used for jittered pools).
    """
    model = model or bench_model()
    rc = default_region_count(gpu_count) if region_count is None else region_count
    rng = random.Random(seed)
    names = [f"region-{chr(ord('a') + i)}" for i in range(rc)]
    nodes = []
    for i in range(gpu_count):
        cap = rng.randint(*CAPACITY_RANGE)
        flops = rng.uniform(*FLOPS_RANGE)
        nodes.append(GpuNode(id=f"{id_prefix}{i:04d}", region=names[i % rc],
                             vram_bytes=cap * model.bytes_per_layer / 0.8,
                             flops=homogeneous_flops if homogeneous_flops else flops,
                             reserve_fraction=0.2))
    if links is None:
        links = {}
        for i, a in enumerate(nodes):
            for b in nodes[i + 1:]:
                if a.region == b.region:
                    links[(a.id, b.id)] = INTRA_REGION_RTT_S
    return ClusterSnapshot(gpus=tuple(nodes), links=links), model


C5_SPLIT = ((256, 32, "8b"), (384, 64, "32b"), (384, 80, "70b"))


def region_rtt_matrix(region_count: int, seed: int, intra: float = INTRA_REGION_RTT_S,
                      inter: Tuple[float, float] = (0.005, 0.080)) -> np.ndarray:
    """Seeded symmetric region x region one-way RTT matrix: intra 1 ms, inter U(5, 80) ms."""
    rng = random.Random(seed)
    m = np.full((region_count, region_count), intra)
    for a in range(region_count):
        for b in range(a + 1, region_count):
            m[a, b] = m[b, a] = rng.uniform(*inter)
    return m


def c5_pools(seed: int = 0, region_count: int = 8):
    """C5: 1,024 bench-drawn GPUs in 8 regions with an explicit all-pairs link table from a
    seeded region RTT matrix, split 256 / 384 / 384 into 8B (L=32) / 32B (L=64) / 70B (L=80) sub-pools.
    Returns [(name, ClusterSnapshot, ModelSpec)], one per sub-pool (its GPUs and their links only)."""
    total = sum(n for n, _, _ in C5_SPLIT)
    rng = random.Random(seed)
    names = [f"region-{chr(ord('a') + i)}" for i in range(region_count)]
    reg = region_rtt_matrix(region_count, seed ^ 0x5EED)
    draws = [(rng.randint(*CAPACITY_RANGE), rng.uniform(*FLOPS_RANGE)) for _ in range(total)]
    out, start = [], 0
    for n, layers, name in C5_SPLIT:
        model = bench_model(layers, f"c5-{name}")
        nodes = tuple(GpuNode(id=f"gpu-{i:04d}", region=names[i % region_count],
                              vram_bytes=draws[i][0] * model.bytes_per_layer / 0.8, flops=draws[i][1],
                              reserve_fraction=0.2) for i in range(start, start + n))
        links = {}
        for a in range(n):
            ra = (start + a) % region_count
            for b in range(a + 1, n):
                links[(nodes[a].id, nodes[b].id)] = float(reg[ra, (start + b) % region_count])
        out.append((name, ClusterSnapshot(gpus=nodes, links=links), model))
        start += n
    return out


# ---------------------------------------------------------------------------
# deterministic hashing shared with the device generator
# ---------------------------------------------------------------------------

def splitmix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def _jitter_table() -> np.ndarray:
    """The 1024 LogNormal(0, 0.2) float32 quantiles of csrc/jitter_lognormal.inc (the kernels include the same file)."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "csrc", "jitter_lognormal.inc")
    with open(path) as fh:
        vals = [float.fromhex(t) for line in fh if not line.startswith("//")
                for t in line.replace(",", " ").split()]
    if len(vals) != 1024:
        raise RuntimeError(f"{path}: expected 1024 quantiles, found {len(vals)}")
    return np.array(vals, dtype=np.float64)


JITTER_Q = _jitter_table()


def jitter_index(seed: int, i: int, j: int) -> int:
    """Quantile index of the unordered pair (i, j): ss_jitter_index (ss_common.cuh) in Python integers."""
    if i > j:
        i, j = j, i
    mix = splitmix64(seed & MASK64)
    x = (i * 0x9E3779B1 + j * 0x85EBCA77 + ((mix ^ (mix >> 32)) & 0xFFFFFFFF)) & 0xFFFFFFFF
    x ^= x >> 16
    x = (x * 0x7FEB352D) & 0xFFFFFFFF
    x ^= x >> 15
    x = (x * 0x846CA68B) & 0xFFFFFFFF
    x ^= x >> 16
    return x >> 22


def jitter_factor(seed: int, i: int, j: int) -> float:
    """One LogNormal(0, 0.2) factor per unordered GPU pair: quantile jitter_index of JITTER_Q."""
    return float(JITTER_Q[jitter_index(seed, i, j)])


def jitter_factor_matrix(seed: int, n: int) -> np.ndarray:
    """Vectorised jitter_factor over all pairs (diagonal 1.0) -- numpy uint32 arithmetic."""
    i, j = np.triu_indices(n, 1)
    mix = splitmix64(seed & MASK64)
    h0 = np.uint32((mix ^ (mix >> 32)) & 0xFFFFFFFF)
    with np.errstate(over="ignore"):
        x = i.astype(np.uint32) * np.uint32(0x9E3779B1) + j.astype(np.uint32) * np.uint32(0x85EBCA77) + h0
        x ^= x >> np.uint32(16)
        x *= np.uint32(0x7FEB352D)
        x ^= x >> np.uint32(15)
        x *= np.uint32(0x846CA68B)
        x ^= x >> np.uint32(16)
    f = JITTER_Q[(x >> np.uint32(22)).astype(np.int64)]
    out = np.ones((n, n))
    out[i, j] = f
    out[j, i] = f
    return out


def churn_set(seed: int, plan_gpus: Sequence[int], slices: Dict[int, Tuple[int, int]], layer_count: int,
              fraction: float = 0.05) -> List[int]:
    """Seeded leave set: up to ``fraction`` of the plan GPUs, never uncovering a layer.

    Candidates are visited in ascending splitmix64(seed, gpu) order; one is
    accepted when every layer keeps at least one host afterwards.
    """
    want = int(len(plan_gpus) * fraction)
    cover = np.zeros(layer_count + 2, dtype=np.int64)
    for g in plan_gpus:
        a, b = slices[g]
        cover[a:b + 1] += 1
    order = sorted(plan_gpus, key=lambda g: (splitmix64((splitmix64(seed) ^ (0xC4 << 40) ^ g) & MASK64), g))
    out = []
    for g in order:
        if len(out) >= want:
            break
        a, b = slices[g]
        if np.all(cover[a:b + 1] >= 2):
            cover[a:b + 1] -= 1
            out.append(g)
    return sorted(out)


def generate_trace(rate_rps: float, duration_s: float, *, seed: int = 0, prompt_tokens=(32, 256),
                   output_tokens=(16, 128)):
    """Poisson arrivals with uniform token counts, draw for draw as sim.py:121-150 (random.Random(seed)).

    Returns (arrival_s float64[n], prompt int32[n], output int32[n]) in arrival order.
    """
    if rate_rps <= 0:
        raise ValueError(f"rate_rps must be positive, got {rate_rps}")
    if duration_s <= 0:
        raise ValueError(f"duration_s must be positive, got {duration_s}")
    rng = random.Random(seed)
    arr, pr, out = [], [], []
    t = 0.0
    while True:
        t += rng.expovariate(rate_rps)
        if t >= duration_s:
            break
        arr.append(t)
        pr.append(rng.randint(*prompt_tokens))
        out.append(rng.randint(*output_tokens))
    return np.array(arr, dtype=np.float64), np.array(pr, dtype=np.int32), np.array(out, dtype=np.int32)


TOKEN_SALT = 0x70 << 40


def request_tokens(seed: int, i: int, lo: int, hi: int) -> int:
    """Total tokens (prompt + output) of request i of a scenario: uniform in [lo, hi] from splitmix64."""
    return lo + splitmix64((splitmix64(seed & MASK64) ^ TOKEN_SALT ^ i) & MASK64) % (hi - lo + 1)


LEAVE_SALT = 0xC4 << 40
JOIN_SALT = 0x4A << 40


def join_order(seed: int, candidates: Sequence[int]) -> List[int]:
    """Seeded order in which absent pool GPUs join (ascending splitmix64 key, then index)."""
    return sorted(candidates, key=lambda g: (splitmix64((splitmix64(seed) ^ JOIN_SALT ^ g) & MASK64), g))


def membership_events(seed: int, lo: np.ndarray, hi: np.ndarray, present: np.ndarray, token_cap: np.ndarray,
                      layer_cap: np.ndarray, layer_count: int, fraction: float, n_join: int):
    """One scenario's membership history, in the reference's semantics.

    1. ``on_leave`` (membership.py:340-357) of the seeded churn set of the plan GPUs that are present
       (:func:`churn_set`: never uncovers a layer).
    2. ``on_join`` (membership.py:317-338) of the first ``n_join`` absent pool GPUs in :func:`join_order`:
       the GPU starts at ``bottleneck_layer()`` (membership.py:303-315: the layer with the least summed
       ``ram_token_capacity`` over its current hosts, first such layer; holes count as 0) and takes
       ``min(start + layer_capacity - 1, L)``; a GPU below one layer joins without a slice (ZeroCapacityGpu).

    Returns (absent[N] bool, lo_s[N], hi_s[N], left, joined, bottlenecks) -- slices 0/-1 when none.
    """
    n = lo.shape[0]
    lo_s, hi_s = lo.astype(np.int32).copy(), hi.astype(np.int32).copy()
    absent = ~present.astype(bool)
    lo_s[absent] = 0
    hi_s[absent] = -1
    plan = [g for g in range(n) if not absent[g] and lo_s[g] <= hi_s[g]]
    slices = {g: (int(lo_s[g]), int(hi_s[g])) for g in plan}
    want = int(len(plan) * fraction)
    left = churn_set(seed, plan, slices, layer_count, fraction) if want > 0 else []
    for g in left:
        absent[g] = True
        lo_s[g], hi_s[g] = 0, -1
    tot = np.zeros(layer_count + 2, dtype=np.int64)
    for g in range(n):
        if not absent[g] and lo_s[g] <= hi_s[g]:
            tot[lo_s[g]:hi_s[g] + 1] += int(token_cap[g])
    joined, bottlenecks = [], []
    candidates = [g for g in range(n) if not present[g]]
    for g in join_order(seed, candidates)[:n_join]:
        start = int(np.argmin(tot[1:layer_count + 1])) + 1          # first least-capacity layer
        bottlenecks.append(start)
        absent[g] = False
        joined.append(g)
        cap = int(layer_cap[g])
        if cap < 1:
            continue                                                   # registered, serves nothing
        end = min(start + cap - 1, layer_count)
        lo_s[g], hi_s[g] = start, end
        tot[start:end + 1] += int(token_cap[g])
    return absent, lo_s, hi_s, left, joined, bottlenecks


# ---------------------------------------------------------------------------
# scenario description (what the replay consumes)
# ---------------------------------------------------------------------------

@dataclass
class ScenarioSet:
    """Scenario batch over one base pool (GPU index = position in sorted-id order).

    base_rtt[N, N]   ground-truth rtt_s over all pool GPUs (diag 0)
    base_tau[N]      flops_per_layer_per_token / flops
    slice_lo/hi[N]   1-based inclusive layer range per GPU in the base plan, 0/-1 when not serving
    seeds[S]         per-scenario jitter / churn seed
    leave[S, N]      bool, GPU absent in scenario s (departed, or a join-pool GPU that did not join)
    present0[N]      bool, GPU in the pool before the scenario's events (False: join pool)
    slice_lo_s/hi_s  [S, N] per-scenario slices when the scenarios have joins, else None
    churn/joins      the event counts the device generator reproduces (ss_scenario_membership)
    """

    layer_count: int
    ids: List[str]
    base_rtt: np.ndarray
    base_tau: np.ndarray
    slice_lo: np.ndarray
    slice_hi: np.ndarray
    seeds: np.ndarray
    leave: np.ndarray
    jitter: bool = True
    present0: Optional[np.ndarray] = None
    slice_lo_s: Optional[np.ndarray] = None
    slice_hi_s: Optional[np.ndarray] = None
    churn: float = 0.0
    joins: int = 0
    token_cap: Optional[np.ndarray] = None
    layer_cap: Optional[np.ndarray] = None
    device_events: bool = False        # leave / slices are generated by ss_scenario_membership
    want_leave: int = 0
    cluster_order: Optional[np.ndarray] = None   # base pool GPUs in cluster (MembershipManager._gpus) order
    plan_order: Optional[np.ndarray] = None      # plan GPUs in plan.gpu_slices() order
    vram: Optional[np.ndarray] = None
    reserve: Optional[np.ndarray] = None
    flops: Optional[np.ndarray] = None
    region_idx: Optional[np.ndarray] = None      # per GPU, index into region_names (sorted)
    region_names: Tuple[str, ...] = ()
    fpl: float = 0.0                             # model.flops_per_layer_per_token
    slice_order_s: Optional[np.ndarray] = None   # [S, n] per-scenario plan.gpu_slices() order (-1 padded)
    joined_s: Optional[np.ndarray] = None        # [S, joins] join sequence per scenario (-1 padded)

    @property
    def n_scenarios(self) -> int:
        return int(self.seeds.shape[0])

    @property
    def n_gpus(self) -> int:
        return len(self.ids)

    def scenario_rtt(self, s: int) -> np.ndarray:
        if not self.jitter:
            return self.base_rtt.copy()
        return self.base_rtt * jitter_factor_matrix(int(self.seeds[s]), self.n_gpus)

    def slices(self, s: int) -> Tuple[np.ndarray, np.ndarray]:
        if self.slice_lo_s is not None:
            return self.slice_lo_s[s], self.slice_hi_s[s]
        return self.slice_lo, self.slice_hi

    def columns(self, s: int) -> List[np.ndarray]:
        alive = ~self.leave[s]
        lo, hi = self.slices(s)
        return [np.nonzero(alive & (lo <= l) & (hi >= l))[0] for l in range(1, self.layer_count + 1)]


def base_rtt_matrix(cluster: ClusterSnapshot, ids: Sequence[str]) -> np.ndarray:
    n = len(ids)
    out = np.empty((n, n))
    for a in range(n):
        for b in range(n):
            out[a, b] = cluster.rtt_s(ids[a], ids[b])
    return out


def build_scenarios(cluster: ClusterSnapshot, model: ModelSpec, plan, n_scenarios: int, *,
                    seed0: int = 0, churn: float = 0.05, jitter: bool = True, seeds=None,
                    join_pool: Sequence[str] = (), joins: int = 0, host_events: bool = True) -> ScenarioSet:
    """C4-style scenario batch over a placed pool.

    ``cluster`` holds every GPU a scenario can see; ``join_pool`` names the ones absent at the start
    (not in the plan's pool), ``joins`` of which join each scenario after its leaves
    (:func:`membership_events`).  With ``host_events=False`` the events are left to the device generator
    (``ss_scenario_membership``, run by ScenarioReplayer.build) and ``leave`` / per-scenario slices stay
    unset on the host.
    """
    ids = sorted(g.id for g in cluster.gpus)
    pos = {g: i for i, g in enumerate(ids)}
    n = len(ids)
    by_id = {g.id: g for g in cluster.gpus}
    base_tau = np.array([model.flops_per_layer_per_token / by_id[g].flops for g in ids])
    lo = np.zeros(n, dtype=np.int32)
    hi = np.full(n, -1, dtype=np.int32)
    slices = {}
    for gid, sl in plan.gpu_slices().items():
        lo[pos[gid]] = sl.start_layer
        hi[pos[gid]] = sl.end_layer
        slices[pos[gid]] = (sl.start_layer, sl.end_layer)
    rtt = base_rtt_matrix(cluster, ids)
    seeds = (np.arange(seed0, seed0 + n_scenarios, dtype=np.int64) if seeds is None
             else np.asarray(seeds, dtype=np.int64))
    leave = np.zeros((n_scenarios, n), dtype=bool)
    plan_gpus = sorted(slices)
    pool_absent = set(join_pool)
    present0 = np.array([g not in pool_absent for g in ids], dtype=bool)
    token_cap = np.array([by_id[g].ram_token_capacity for g in ids], dtype=np.int64)
    from .topology import layer_capacity
    layer_cap = np.array([layer_capacity(by_id[g], model) for g in ids], dtype=np.int32)
    if joins and not pool_absent:
        raise ValueError("joins need a join_pool of absent GPUs")
    lo_s = hi_s = None
    if not host_events:
        leave[:, ~present0] = True
        if joins:
            lo_s = np.zeros((n_scenarios, n), dtype=np.int32)
            hi_s = np.full((n_scenarios, n), -1, dtype=np.int32)
    elif joins:
        lo_s = np.zeros((n_scenarios, n), dtype=np.int32)
        hi_s = np.full((n_scenarios, n), -1, dtype=np.int32)
        for s in range(n_scenarios):
            absent, l_s, h_s, _, _, _ = membership_events(int(seeds[s]), lo, hi, present0, token_cap, layer_cap,
                                                          model.layer_count, churn, joins)
            leave[s], lo_s[s], hi_s[s] = absent, l_s, h_s
    else:
        leave[:, ~present0] = True
        if churn > 0:
            plan_now = [g for g in plan_gpus if present0[g]]
            for s in range(n_scenarios):
                leave[s, churn_set(int(seeds[s]), plan_now, slices, model.layer_count, churn)] = True
    want = int(len([g for g in plan_gpus if present0[g]]) * churn) if churn > 0 else 0
    cluster_order = np.array([pos[g.id] for g in cluster.gpus if present0[pos[g.id]]], dtype=np.int32)
    plan_order = np.array([pos[g] for g in plan.gpu_slices()], dtype=np.int32)
    vram = np.array([by_id[g].vram_bytes for g in ids], dtype=np.float64)
    reserve = np.array([by_id[g].reserve_fraction for g in ids], dtype=np.float64)
    flops = np.array([by_id[g].flops for g in ids], dtype=np.float64)
    region_names = tuple(sorted({g.region for g in cluster.gpus}))
    rpos = {r: i for i, r in enumerate(region_names)}
    region_idx = np.array([rpos[by_id[g].region] for g in ids], dtype=np.int32)
    return ScenarioSet(model.layer_count, ids, rtt, base_tau, lo, hi, seeds, leave, jitter, present0, lo_s, hi_s,
                       churn, joins, token_cap, layer_cap, not host_events, want, cluster_order, plan_order, vram,
                       reserve, flops, region_idx, region_names, model.flops_per_layer_per_token)


# ---------------------------------------------------------------------------
# C3 / C5 Phase-1 variants, packed straight into device order
# ---------------------------------------------------------------------------

def pack_variants(clusters_models, *, alpha: float = 1.0, tokens: float = 128.0):
    """allocate()-equivalent packing of many (cluster, model) pairs (allocator.py:561-581).

    Regions in sorted() order; per region GPUs sorted by (-capacity, id);
    objective inputs in cluster order with the dense rtt_s matrix.
    Returns (PackedVariants, meta) where meta[p] = (variant, region, ordered gpu ids).
    """
    from .batched import PackedVariants
    from ._phase1 import PoolSpec
    from .topology import layer_capacity
    pools, of, orr, meta, var_ptr = [], [], [], [], [0]
    L = fpl = None
    for v, (cluster, model) in enumerate(clusters_models):
        L, fpl = model.layer_count, model.flops_per_layer_per_token
        for region in sorted(cluster.regions):
            rg = cluster.gpus_in_region(region)
            if not rg:
                continue
            caps = [layer_capacity(g, model) for g in rg]
            limit = min(len(caps), sum(caps) // L)
            if limit < 1:
                continue
            order = sorted(range(len(rg)), key=lambda i: (-caps[i], rg[i].id))
            pools.append(PoolSpec([caps[i] for i in order], [rg[i].flops for i in order], L, limit))
            of.append(np.array([g.flops for g in rg]))
            ids = [g.id for g in rg]
            m = np.empty((len(rg), len(rg)))
            for a in range(len(rg)):
                for b in range(len(rg)):
                    m[a, b] = cluster.rtt_s(ids[a], ids[b])
            orr.append(m)
            meta.append((v, region, [rg[i].id for i in order]))
        var_ptr.append(len(pools))
    return PackedVariants(pools, of, orr, np.array(var_ptr), fpl, L, tokens, alpha), meta


def bench_variants(n_variants: int, gpu_count: int = 256, layer_count: int = 80, seed0: int = 0):
    """C3 sweep inputs: synthetic_cluster(gpu_count, seed=v) for v in [seed0, seed0+n) packed
    without building per-pair link dicts (bench pools: 1 ms inside a region, 10 ms across)."""
    from .batched import PackedVariants
    from ._phase1 import PoolSpec
    model = bench_model(layer_count)
    rc = default_region_count(gpu_count)
    pools, of, orr, meta, var_ptr = [], [], [], [], [0]
    for v in range(seed0, seed0 + n_variants):
        rng = random.Random(v)
        caps_all, flops_all = [], []
        for _ in range(gpu_count):
            c = rng.randint(*CAPACITY_RANGE)
            f = rng.uniform(*FLOPS_RANGE)
            vram = c * model.bytes_per_layer / 0.8
            caps_all.append(max(0, int(np.floor(vram * (1.0 - 0.2) / model.bytes_per_layer + 1e-9))))
            flops_all.append(f)
        for r in range(rc):             # region names region-a.. sort like r
            idx = list(range(r, gpu_count, rc))
            caps = [caps_all[i] for i in idx]
            limit = min(len(caps), sum(caps) // layer_count)
            if limit < 1:
                continue
            order = sorted(range(len(idx)), key=lambda q: (-caps[q], idx[q]))
            pools.append(PoolSpec([caps[q] for q in order], [flops_all[idx[q]] for q in order], layer_count, limit))
            of.append(np.array([flops_all[i] for i in idx]))
            m = np.full((len(idx), len(idx)), INTRA_REGION_RTT_S)
            np.fill_diagonal(m, 0.0)
            orr.append(m)
            meta.append((v, f"region-{chr(ord('a') + r)}", [f"gpu-{idx[q]:04d}" for q in order]))
        var_ptr.append(len(pools))
    return PackedVariants(pools, of, orr, np.array(var_ptr), model.flops_per_layer_per_token, layer_count), meta
