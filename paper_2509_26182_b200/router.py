"""Phase-2 drop-in: per-request chain selection backed by the sm_100a kernels.

Same public names, signatures and return types as
``pkg/src/swarmsched/router.py`` (``PipelineChain`` 37-58, ``LayerDag`` 61-75,
``RouteStats`` 78-84, ``build_dag`` 87-115, ``rtt_matrix`` 118-143,
``count_dag_edges`` 146-154, ``select_chain`` 200-205, ``ChainRouter`` 208-260,
``route_request`` / ``release_request`` 263-273).

What runs where:
* ``build_dag``      -> ``ss_dag_columns`` (device compaction of the live tau
                        table into sorted host columns, UncoveredLayer status)
* ``rtt_matrix``     -> ``ss_rtt_fill`` (direct > mirrored > inf, diag 0)
* ``select_chain``   -> ``ss_dag_edges`` + ``ss_select`` (the min-plus DP)
* ``ChainRouter``    -> the same, with the RTT matrix cached ON DEVICE under
                        the reference's (rtt_version, gpu_ids, ttl) rule; the
                        select/release feedback is applied to the caller's
                        PerfMap (a host store owned by the caller).
Host code only packs dict-shaped snapshots into flat arrays and turns device
picks back into ``LayerSlice`` hops.  No CPU fallback exists.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import AbstractSet, Dict, FrozenSet, List, Mapping, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from .errors import NoPath, UncoveredLayer, raise_for_status, SS_OK
from .perfmap import PerfMap, PerfSnapshot
from .topology import LayerSlice

_EMPTY: FrozenSet[str] = frozenset()


@dataclass(frozen=True)
class PipelineChain:
    hops: Tuple[LayerSlice, ...]
    cost_s: float

    @property
    def gpu_ids(self) -> Tuple[str, ...]:
        return tuple(h.gpu_id for h in self.hops)

    @property
    def layer_count(self) -> int:
        return self.hops[-1].end_layer if self.hops else 0

    @property
    def cross_gpu_edges(self) -> int:
        return sum(1 for a, b in zip(self.hops, self.hops[1:]) if a.gpu_id != b.gpu_id)


@dataclass(frozen=True)
class LayerDag:
    layer_count: int
    hosts: Tuple[Tuple[str, ...], ...]
    latencies: Mapping[Tuple[str, int], float]

    @property
    def node_count(self) -> int:
        return sum(len(c) for c in self.hosts)

    def gpu_ids(self) -> Tuple[str, ...]:
        return tuple(sorted({g for c in self.hosts for g in c}))


@dataclass
class RouteStats:
    dags_built: int = 0
    chains_selected: int = 0
    edges_relaxed: int = 0
    matrix_rebuilds: int = 0
    matrix_reuses: int = 0


# ---------------------------------------------------------------------------
# device helpers
# ---------------------------------------------------------------------------

def _torch():
    import torch
    return torch


def _dev():
    return _torch().device("cuda")


def _rtt_device(entries: Sequence[Tuple[str, str, float]], ids: Sequence[str]):
    """Dense RTT matrix on device via ss_rtt_fill (router.py:118-143 semantics)."""
    torch = _torch()
    lib = N.lib()
    pos = {g: i for i, g in enumerate(ids)}
    a_idx, b_idx, vals = [], [], []
    for a, b, v in entries:
        ia, ib = pos.get(a), pos.get(b)
        if ia is None or ib is None or ia == ib:
            continue
        a_idx.append(ia)
        b_idx.append(ib)
        vals.append(v)
    n = len(ids)
    dev = _dev()
    out = torch.empty(n * n, dtype=torch.float64, device=dev)
    meta = torch.tensor([0, n], dtype=torch.int64).to(dev, non_blocking=True)
    dim = torch.tensor([n], dtype=torch.int32).to(dev, non_blocking=True)
    la = torch.tensor(a_idx, dtype=torch.int32).to(dev, non_blocking=True) if a_idx else None
    lb = torch.tensor(b_idx, dtype=torch.int32).to(dev, non_blocking=True) if b_idx else None
    lv = torch.tensor(vals, dtype=torch.float64).to(dev, non_blocking=True) if vals else None
    N.check(lib.ss_rtt_fill(1, N.ptr(meta), N.ptr(dim), N.ptr(out), math.inf, len(vals), None,
                            N.ptr(la), N.ptr(lb), N.ptr(lv), N.stream_handle()), "ss_rtt_fill")
    return out, {g: i for i, g in enumerate(ids)}


class _DeviceDag:
    """One DAG resident on device: columns, tau, edge blocks."""

    def __init__(self, col_len: List[int], node_gpu: Sequence[int], node_tau: Sequence[float]):
        torch = _torch()
        L = len(col_len)
        self.L = L
        self.col_len_h = list(col_len)
        col_off = np.zeros(L, dtype=np.int64)
        np.cumsum(col_len[:-1], out=col_off[1:]) if L > 1 else None
        edge_off = np.zeros(L, dtype=np.int64)
        acc = 0
        for l in range(L - 1):
            edge_off[l] = acc
            blk = col_len[l] * col_len[l + 1]
            acc += blk + (blk & 1)
        self.edge_used = acc
        self.edge_total = max(acc, 2)
        dev = _dev()
        ints = np.concatenate([[0, L], col_off, np.asarray(col_len, dtype=np.int64),
                               np.asarray(node_gpu, dtype=np.int64)]).astype(np.int32)
        self.ints = torch.from_numpy(ints).to(dev, non_blocking=True)
        self.edge_off = torch.from_numpy(edge_off).to(dev, non_blocking=True)
        self.node_tau = torch.from_numpy(np.asarray(node_tau, dtype=np.float64)).to(dev, non_blocking=True)
        self.edge_val = torch.empty(self.edge_total, dtype=torch.float64, device=dev)
        i = self.ints
        self.layer_ptr, self.col_off = i[0:2], i[2:2 + L]
        self.col_len, self.node_gpu = i[2 + L:2 + 2 * L], i[2 + 2 * L:]
        self.max_hosts = max(col_len)

    def dag_set(self, n_gpus: int) -> N.DagSet:
        return N.DagSet(1, self.max_hosts, self.L, n_gpus, N.ptr(self.layer_ptr), N.ptr(self.col_off),
                        N.ptr(self.col_len), N.ptr(self.node_gpu), N.ptr(self.node_tau), N.ptr(self.edge_off),
                        N.ptr(self.edge_val))


def _select_on_device(ddag: _DeviceDag, rtt_dev, n_gpus: int, count_edges: bool = True):
    """ss_dag_edges (once per DAG) + ss_select; returns (picks, cost, status, finite edge count)."""
    torch = _torch()
    lib = N.lib()
    dev = _dev()
    ds = ddag.dag_set(n_gpus)
    st = N.stream_handle()
    if not getattr(ddag, "edges_built", False):
        rmeta = torch.tensor([0], dtype=torch.int64).to(dev, non_blocking=True)
        rdim = torch.tensor([n_gpus], dtype=torch.int32).to(dev, non_blocking=True)
        N.check(lib.ss_dag_edges(ds, N.ptr(rmeta), N.ptr(rdim), N.ptr(rtt_dev), None, 0, N.ptr(ddag.edge_val), st),
                "ss_dag_edges")
        ddag.edges_built = True
    if not hasattr(ddag, "out"):
        ddag.out = torch.empty(ddag.L + 4, dtype=torch.float64, device=dev)   # picks (as int32 pairs), cost, status
    out = ddag.out
    picks = out[:(ddag.L + 1) // 2 + 1].view(torch.int32)[:ddag.L]
    cost = out[ddag.L // 2 + 2: ddag.L // 2 + 3]
    status = out[ddag.L // 2 + 3: ddag.L // 2 + 4].view(torch.int32)[:1]
    N.check(lib.ss_select(ds, N.ptr(picks), N.ptr(cost), N.ptr(status), st), "ss_select")
    edges = 0
    if count_edges and ddag.L > 1:
        # finite edge count (router.py:176-177); block pads are +inf
        edges = int(torch.isfinite(ddag.edge_val[:ddag.edge_used]).sum())
    host = out.cpu()                                                          # one D2H for picks + cost + status
    picks_h = host[:(ddag.L + 1) // 2 + 1].view(torch.int32)[:ddag.L].tolist()
    cost_h = float(host[ddag.L // 2 + 2])
    status_h = int(host[ddag.L // 2 + 3:ddag.L // 2 + 4].view(torch.int32)[0])
    return picks_h, cost_h, status_h, edges


def _chain_from_picks(hosts: Sequence[Sequence[str]], picks: Sequence[int], cost: float) -> PipelineChain:
    assign = [hosts[l][p] for l, p in enumerate(picks)]
    hops: List[LayerSlice] = []
    start = 1
    for layer in range(2, len(assign) + 1):
        if assign[layer - 1] != assign[layer - 2]:
            hops.append(LayerSlice(assign[layer - 2], start, layer - 1))
            start = layer
    hops.append(LayerSlice(assign[-1], start, len(assign)))
    return PipelineChain(hops=tuple(hops), cost_s=cost)


def _columns_on_device(snapshot: PerfSnapshot, layer_count: int, exclude: AbstractSet[str]):
    """Device build_dag: tau table [L x G] (NaN = absent) -> sorted columns."""
    torch = _torch()
    lib = N.lib()
    lat = snapshot.layer_latencies
    ids = sorted({g for (g, l) in lat if 1 <= l <= layer_count})
    G = max(len(ids), 1)
    pos = {g: i for i, g in enumerate(ids)}
    table = np.full((layer_count, G), np.nan)
    for (g, l), v in lat.items():
        if 1 <= l <= layer_count:
            table[l - 1, pos[g]] = v
    excl = np.zeros(G, dtype=np.uint8)
    for g in exclude:
        if g in pos:
            excl[pos[g]] = 1
    dev = _dev()
    L = layer_count
    ints = np.concatenate([[0, L, 0, G], np.arange(L) * G]).astype(np.int32)
    ints_d = torch.from_numpy(ints).to(dev, non_blocking=True)
    tau_d = torch.from_numpy(table.reshape(-1)).to(dev, non_blocking=True)
    excl_d = torch.from_numpy(excl).to(dev, non_blocking=True)
    tau_off = torch.zeros(1, dtype=torch.int64, device=dev)
    col_len = torch.empty(L, dtype=torch.int32, device=dev)
    node_gpu = torch.empty(L * G, dtype=torch.int32, device=dev)
    node_tau = torch.empty(L * G, dtype=torch.float64, device=dev)
    status = torch.empty(2, dtype=torch.int32, device=dev)
    N.check(lib.ss_dag_columns(1, N.ptr(ints_d[0:2]), N.ptr(ints_d[2:4]), N.ptr(tau_off), N.ptr(tau_d),
                               N.ptr(excl_d), N.ptr(ints_d[4:]), N.ptr(col_len), N.ptr(node_gpu), N.ptr(node_tau),
                               N.ptr(status[0:1]), N.ptr(status[1:2]), N.stream_handle()), "ss_dag_columns")
    st, aux = status.cpu().tolist()
    if st != SS_OK:
        raise_for_status(st, aux)
    lens = col_len.cpu().tolist()
    ng = node_gpu.cpu().numpy().reshape(L, G)
    nt = node_tau.cpu().numpy().reshape(L, G)
    cols = [tuple(ids[g] for g in ng[l, :lens[l]]) for l in range(L)]
    flat_gpu = np.concatenate([ng[l, :lens[l]] for l in range(L)])
    flat_tau = np.concatenate([nt[l, :lens[l]] for l in range(L)])
    return cols, lens, flat_gpu, flat_tau


# ---------------------------------------------------------------------------
# public API (router.py names)
# ---------------------------------------------------------------------------

def build_dag(snapshot: PerfSnapshot, layer_count: int, *, exclude: AbstractSet[str] = _EMPTY) -> LayerDag:
    if layer_count < 1:
        raise ValueError(f"layer_count must be >= 1, got {layer_count}")
    cols, _, _, _ = _columns_on_device(snapshot, layer_count, exclude)
    return LayerDag(layer_count=layer_count, hosts=tuple(cols), latencies=snapshot.layer_latencies)


def rtt_matrix(snapshot: PerfSnapshot, gpu_ids: Sequence[str]) -> Tuple[np.ndarray, Dict[str, int]]:
    out, index = _rtt_device(snapshot.link_rtt_entries(), list(gpu_ids))
    n = len(gpu_ids)
    return out.cpu().numpy().reshape(n, n), index


def _pack_dag(dag: LayerDag, index: Mapping[str, int]):
    lens = [len(c) for c in dag.hosts]
    gpus = [index[g] for c in dag.hosts for g in c]
    taus = [dag.latencies[(g, l + 1)] for l, c in enumerate(dag.hosts) for g in c]
    return _DeviceDag(lens, gpus, taus)


def count_dag_edges(dag: LayerDag, snapshot: PerfSnapshot) -> int:
    torch = _torch()
    ids = dag.gpu_ids()
    rtt_dev, index = _rtt_device(snapshot.link_rtt_entries(), ids)
    ddag = _pack_dag(dag, index)
    lib = N.lib()
    dev = _dev()
    rmeta = torch.tensor([0], dtype=torch.int64).to(dev)
    rdim = torch.tensor([len(ids)], dtype=torch.int32).to(dev)
    N.check(lib.ss_dag_edges(ddag.dag_set(len(ids)), N.ptr(rmeta), N.ptr(rdim), N.ptr(rtt_dev), None, 0,
                             N.ptr(ddag.edge_val), N.stream_handle()), "ss_dag_edges")
    if ddag.L < 2:
        return 0
    return int(torch.isfinite(ddag.edge_val[:ddag.edge_used]).sum())


def select_chain(dag: LayerDag, snapshot: PerfSnapshot, stats: Optional[RouteStats] = None) -> PipelineChain:
    ids = dag.gpu_ids()
    rtt_dev, index = _rtt_device(snapshot.link_rtt_entries(), ids)
    return _select_with_matrix(dag, rtt_dev, index, len(ids), stats)


def _select_with_matrix(dag: LayerDag, rtt_dev, index, n_gpus, stats) -> PipelineChain:
    ddag = _pack_dag(dag, index)
    picks, cost, status, edges = _select_on_device(ddag, rtt_dev, n_gpus)
    if stats is not None:
        stats.edges_relaxed += edges
    if status == 2:
        raise NoPath()
    raise_for_status(status)
    if stats is not None:
        stats.chains_selected += 1
    return _chain_from_picks(dag.hosts, picks, cost)


class _RouteCache:
    """A device DAG kept across routes while the perf map's tau key set, the exclude set and the RTT table are
    unchanged and no entry can have expired: only republished tau values move, host mirror -> device."""

    def __init__(self, keys_version, exclude, rtt_key, min_pub, dag, ddag, index, edges, tau_h, nodes_of, hidden):
        self.keys_version = keys_version
        self.exclude = exclude
        self.rtt_key = rtt_key
        self.min_pub = min_pub          # oldest tau publish time when built; entries only get newer
        self.dag = dag
        self.ddag = ddag
        self.index = index
        self.edges = edges
        self.tau_h = tau_h              # host mirror of ddag.node_tau
        self.nodes_of = nodes_of        # gpu -> [(node position, layer)]
        self.hidden = hidden            # GPUs with a tau entry (layers 1..L) left out of the DAG as expired


class ChainRouter:
    """Snapshot -> device DAG -> device DP -> occupancy feedback on the PerfMap.

    Between membership / placement changes consecutive routes differ only in the latencies that the previous
    select / release republished, so the router keeps its device DAG (columns, edge blocks) and uploads just the
    tau column of the republished GPUs: the chain is the one router.py:247-257 would select from a fresh snapshot
    (same live keys -- none can have expired while now - oldest publish <= ttl --, same exclude set, same RTT
    table, current values).
    """

    def __init__(self, perf_map: PerfMap, layer_count: int):
        self.perf_map = perf_map
        self.layer_count = layer_count
        self.stats = RouteStats()
        self._key = None
        self._matrix = None
        self._index: Dict[str, int] = {}
        self._valid_until = -math.inf
        self._cache: Optional[_RouteCache] = None
        self._tau_seen = 0              # this router's read position in the perf map's tau write log

    def _matrix_for(self, snapshot: PerfSnapshot, gpu_ids: Tuple[str, ...]):
        key = (snapshot.rtt_version, gpu_ids)
        if self._matrix is not None and key == self._key and snapshot.now <= self._valid_until:
            self.stats.matrix_reuses += 1
            return self._matrix, self._index
        self._matrix, self._index = _rtt_device(snapshot.link_rtt_entries(), gpu_ids)
        self._key = key
        self._valid_until = snapshot.rtt_oldest_publish + self.perf_map.ttl_s
        self.stats.matrix_rebuilds += 1
        return self._matrix, self._index

    def route(self, now: float, *, exclude: AbstractSet[str] = _EMPTY) -> PipelineChain:
        pm = self.perf_map
        keys_version, seq, dirty = pm._tau_updates_since(self._tau_seen)
        self._tau_seen = seq
        c = self._cache
        excl = frozenset(exclude)
        # an entry that was expired when the DAG was built and has since been republished under the same key
        # changes the live key set without changing the key-set version: rebuild
        if (c is not None and dirty is not None and c.keys_version == keys_version and c.exclude == excl
                and c.rtt_key[0] == pm._rtt_version and now <= self._valid_until   # the cached DAG fixes the ids
                and now - c.min_pub <= pm.ttl_s and not (c.hidden and dirty & c.hidden)):
            return self._route_cached(c, dirty, now)
        snapshot = pm.snapshot(now)
        dag = build_dag(snapshot, self.layer_count, exclude=exclude)
        self.stats.dags_built += 1
        ids = dag.gpu_ids()
        matrix, index = self._matrix_for(snapshot, ids)
        ddag = _pack_dag(dag, index)
        picks, cost, status, edges = _select_on_device(ddag, matrix, len(ids))
        chain = self._finish(dag, picks, cost, status, edges)
        L = self.layer_count
        with pm._lock:
            min_pub = min((pm._tau[(g, l + 1)].published_at for l, col in enumerate(dag.hosts) for g in col),
                          default=math.inf)
            hidden = {g for (g, l), e in pm._tau.items() if 1 <= l <= L and e.expired(now)}
        nodes_of: Dict[str, list] = {}
        pos = 0
        for l, col in enumerate(dag.hosts):
            for g in col:
                nodes_of.setdefault(g, []).append((pos, l + 1))
                pos += 1
        tau_h = np.array([dag.latencies[(g, l + 1)] for l, col in enumerate(dag.hosts) for g in col],
                         dtype=np.float64)
        self._cache = _RouteCache(keys_version, excl, (pm._rtt_version, ids), min_pub, dag, ddag, index, edges,
                                  tau_h, nodes_of, frozenset(hidden))
        pm.on_chain_event(chain, "select", now)
        return chain

    def _route_cached(self, c: _RouteCache, dirty, now: float) -> PipelineChain:
        pm = self.perf_map
        torch = _torch()
        if dirty:
            with pm._lock:
                for g in dirty:
                    for p, layer in c.nodes_of.get(g, ()):
                        c.tau_h[p] = pm._tau[(g, layer)].value
            c.ddag.node_tau.copy_(torch.from_numpy(c.tau_h), non_blocking=False)
        self.stats.dags_built += 1
        self.stats.matrix_reuses += 1
        picks, cost, status, _ = _select_on_device(c.ddag, self._matrix, len(c.index), count_edges=False)
        chain = self._finish(c.dag, picks, cost, status, c.edges)
        pm.on_chain_event(chain, "select", now)
        return chain

    def _finish(self, dag, picks, cost, status, edges) -> PipelineChain:
        self.stats.edges_relaxed += edges
        if status == 2:
            raise NoPath()
        raise_for_status(status)
        self.stats.chains_selected += 1
        return _chain_from_picks(dag.hosts, picks, cost)

    def release(self, chain: PipelineChain, now: float) -> None:
        self.perf_map.on_chain_event(chain, "release", now)


def route_request(perf_map: PerfMap, layer_count: int, now: float) -> PipelineChain:
    snapshot = perf_map.snapshot(now)
    chain = select_chain(build_dag(snapshot, layer_count), snapshot)
    perf_map.on_chain_event(chain, "select", now)
    return chain


def release_request(perf_map: PerfMap, chain: PipelineChain, now: float) -> None:
    perf_map.on_chain_event(chain, "release", now)
