"""Device pool batches for Phase-1 (packing + launch sequencing; no arithmetic).

A *pool* is one region of one ``allocate`` call: its GPUs sorted by
``(-capacity, id)`` (allocator.py:570), their unclamped capacities and flops,
the model depth and ``k_max``.  :class:`PoolBatch` uploads many pools at once
and drives the C-ABI launches

    ss_stage_counts_validate -> ss_stage_counts_exact -> ss_stage_counts_cover
    -> ss_phase1_score -> ss_phase1_best [-> ss_variant_reduce]

stream-ordered with a single host sync when results are fetched.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

import os

import numpy as np

from . import _native as N
from .errors import SS_OK, SS_WORKSPACE, raise_for_status

EXACT_LIMIT = 16


@dataclass
class PoolSpec:
    caps: Sequence[int]          # sorted non-increasing
    flops: Sequence[float]       # same order
    layers: int
    kmax: int


def _torch():
    import torch
    return torch


@dataclass
class PoolArrays:
    """Many pools as flat arrays (the vectorised alternative to a list of PoolSpec)."""
    n: np.ndarray                # GPUs per pool
    caps: np.ndarray             # concatenated, each pool sorted non-increasing
    flops: np.ndarray            # same order
    layers: np.ndarray           # per pool
    kmax: np.ndarray             # per pool

    @staticmethod
    def from_specs(pools: List[PoolSpec]) -> "PoolArrays":
        P = len(pools)
        return PoolArrays(np.array([len(p.caps) for p in pools], dtype=np.int64),
                          np.concatenate([np.asarray(p.caps, dtype=np.int64) for p in pools]) if P else np.zeros(0, np.int64),
                          np.concatenate([np.asarray(p.flops, dtype=np.float64) for p in pools]) if P else np.zeros(0),
                          np.array([p.layers for p in pools], dtype=np.int64),
                          np.array([max(int(p.kmax), 0) for p in pools], dtype=np.int64))


def _ramp(counts: np.ndarray) -> np.ndarray:
    """1..c for every count c, concatenated."""
    total = int(counts.sum())
    if total == 0:
        return np.zeros(0, dtype=np.int64)
    starts = np.repeat(np.cumsum(counts) - counts, counts)
    return np.arange(total, dtype=np.int64) - starts + 1


class Upload:
    """Host arrays packed into ONE pinned staging buffer and copied with ONE H2D (stream-ordered, non-blocking);
    device views by name.  Small single calls (allocate() on a handful of GPUs) are launch/copy-latency bound,
    so every input of the call travels together."""

    def __init__(self):
        self.parts = []
        self.size = 0

    def add(self, name: str, arr) -> None:
        arr = np.ascontiguousarray(arr)
        off = (self.size + 15) // 16 * 16
        self.parts.append((name, off, arr))
        self.size = off + arr.nbytes

    def upload(self, dev, stream=None) -> dict:
        torch = _torch()
        host = torch.empty(max(self.size, 16), dtype=torch.uint8, pin_memory=True)   # caching host allocator
        hv = host.numpy()
        for _, off, arr in self.parts:
            hv[off:off + arr.nbytes] = arr.view(np.uint8).reshape(-1)
        if stream is not None:
            with torch.cuda.stream(stream):
                dbuf = host.to(dev, non_blocking=True)
        else:
            dbuf = host.to(dev, non_blocking=True)
        tmap = {np.dtype(np.int32): torch.int32, np.dtype(np.int64): torch.int64,
                np.dtype(np.float64): torch.float64, np.dtype(np.uint8): torch.uint8}
        return {name: dbuf[off:off + arr.nbytes].view(tmap[arr.dtype]) for name, off, arr in self.parts}


class PoolBatch:
    def __init__(self, pools=None, *, arrays: Optional[PoolArrays] = None, stream=None, extra: Optional[dict] = None,
                 defer_workspace_check: bool = False):
        """``extra``: further host arrays (name -> ndarray) that ride along in the batch's single H2D copy; their
        device views are ``self.extra[name]``.  ``defer_workspace_check``: the exact sweep's workspace overflow
        (SS_WORKSPACE) is detected by fetch(), which grows the caps and replays the logged launches -- no host
        sync inside stage_counts(); only for callers that always fetch() (allocate())."""
        self.defer = defer_workspace_check
        torch = _torch()
        A = arrays if arrays is not None else PoolArrays.from_specs(pools)
        self.stream = stream
        dev = torch.device("cuda")
        self.dev = dev
        P = int(A.n.size)
        self.P = P
        n = A.n.astype(np.int64)
        km = np.maximum(A.kmax.astype(np.int64), 0)
        self.n, self.km = n, km
        pool_ptr = np.concatenate([[0], np.cumsum(n)])
        koff = np.concatenate([[0], np.cumsum(km)])
        memb = np.concatenate([[0], np.cumsum(km * n)])
        gsz = np.concatenate([[0], np.cumsum(km * km)])
        self.koff_h, self.memb_h, self.gsz_h, self.pool_ptr_h = koff, memb, gsz, pool_ptr
        caps = A.caps.astype(np.int64)
        flops = A.flops.astype(np.float64)
        cpos = np.concatenate([[0], np.cumsum(caps > 0)])
        usable = cpos[pool_ptr[1:]] - cpos[pool_ptr[:-1]]
        self.usable = usable
        exact = np.nonzero((usable <= EXACT_LIMIT) & (usable > 0) & (km > 0))[0]
        cover_p = np.nonzero(usable > EXACT_LIMIT)[0]
        cand_pool = np.repeat(cover_p, km[cover_p])
        cand_k = _ramp(km[cover_p])
        all_pool = np.repeat(np.arange(P), km)
        all_k = _ramp(km)
        # one thread per candidate: order by (k, pool) so a warp's 32 candidates share k (and hence loop
        # trip counts) -- outputs are addressed by (pool, k), so the order is free
        order_mode = os.environ.get("SS_COVER_ORDER", "k")
        if order_mode in ("m0", "km0") and cand_pool.size:
            # group candidates by their first group count m0 = max(k * ceil(L / cap0), bisect(prefix, k * L))
            # (cover_setup), then k: a warp's candidates start their m loops together
            Lp = A.layers.astype(np.int64)[cand_pool]
            cl = np.minimum(caps, np.repeat(A.layers.astype(np.int64), n))       # clamped caps, pool-major
            pref = np.cumsum(cl)
            base = np.concatenate([[0], pref])[pool_ptr[:-1]]
            target = cand_k * Lp
            m_cap = np.searchsorted(pref, base[cand_pool] + target, side="left") - pool_ptr[:-1][cand_pool] + 1
            m_cap = np.minimum(m_cap, usable[cand_pool])
            c0 = np.maximum(cl[pool_ptr[:-1][cand_pool]], 1)
            m0 = np.maximum(cand_k * ((Lp + c0 - 1) // c0), m_cap)
            o = np.lexsort((cand_pool, cand_k, m0)) if order_mode == "m0" else np.lexsort((cand_pool, m0, cand_k))
        else:
            o = np.lexsort((cand_pool, cand_k))
        cand_pool, cand_k = cand_pool[o], cand_k[o]
        o = np.lexsort((all_pool, all_k))
        all_pool, all_k = all_pool[o], all_k[o]
        self.exact = exact
        self.n_cover = int(cand_pool.size)
        self.max_layers = int(A.layers.max()) if A.layers.size else 0
        self.n_cand = int(all_pool.size)
        ints = np.concatenate([pool_ptr, caps, A.layers, km, exact, cand_pool, cand_k, all_pool,
                               all_k])
        if ints.size and (int(ints.max()) > np.iinfo(np.int32).max or int(ints.min()) < np.iinfo(np.int32).min):
            raise ValueError("layer capacities, k_max or pool sizes exceed the device path's int32 range "
                             f"(max {int(ints.max())}); a capacity this large means bytes_per_layer is tiny")
        ints = ints.astype(np.int32)
        up = Upload()
        up.add("ints", ints)
        up.add("i64", np.concatenate([koff[:-1], memb[:-1], gsz[:-1]]).astype(np.int64))
        up.add("flops", flops)
        for name, arr in (extra or {}).items():
            up.add(name, arr)
        dv = up.upload(dev, stream)
        self.extra = {name: dv[name] for name in (extra or {})}
        self._ints = dv["ints"]
        o = 0

        def take(cnt):
            nonlocal o
            t = self._ints[o:o + cnt]
            o += cnt
            return t

        self.pool_ptr = take(P + 1)
        self.caps = take(caps.size)
        self.layers = take(P)
        self.kmax = take(P)
        self.exact_list = take(exact.size)
        self.cand_pool = take(cand_pool.size)
        self.cand_k = take(cand_k.size)
        self.all_pool = take(all_pool.size)
        self.all_k = take(all_k.size)
        i64 = dv["i64"]
        self.koff, self.memb_off, self.gsz_off = i64[:P], i64[P:2 * P], i64[2 * P:]
        self.flops = dv["flops"]
        K, M, G = int(koff[-1]), int(memb[-1]), int(gsz[-1])
        # outputs: ONE zeroed allocation -- an fp64 block then an int32 block -- read back by ONE D2H in fetch()
        sizes = [("stages", max(K, 1)), ("stall", max(K, 1)), ("kstatus", max(K, 1)), ("fstatus", max(K, 1)),
                 ("members", max(M, 1)), ("counts", max(M, 1)), ("gsize", max(G, 1)), ("status", max(P, 1)),
                 ("aux", max(P, 1)), ("best_k", max(P, 1)), ("sweep_stats", max(exact.size, 1) * 4),
                 ("feasible", 1)]
        nf = max(K, 1) + 1
        ni = sum(c for _, c in sizes)
        self._oblock = torch.zeros(nf * 8 + ni * 4, dtype=torch.uint8, device=dev)
        self._fblock = self._oblock[:nf * 8].view(torch.float64)
        self._iblock = self._oblock[nf * 8:].view(torch.int32)
        o = 0
        for name, cnt in sizes:
            setattr(self, name, self._iblock[o:o + cnt])
            o += cnt
        self.z = self._fblock[:max(K, 1)]
        self.total = self._fblock[max(K, 1):]              # spare slot: allocate()'s objective_total
        self._ops = []                                     # launch log: replayed when the exact sweep needs more room
        self.fcap, self.ccap = 4096, 65536

    def pool_set(self) -> N.PoolSet:
        return N.PoolSet(self.P, N.ptr(self.pool_ptr), N.ptr(self.caps), N.ptr(self.flops),
                         N.ptr(self.layers), N.ptr(self.kmax), N.ptr(self.memb_off), N.ptr(self.gsz_off))

    # -- stage counts ------------------------------------------------------
    def stage_counts(self) -> None:
        self._ops = [self._stage_counts]                   # a new launch sequence starts here
        self._stage_counts()

    def _stage_counts(self) -> None:
        lib = N.lib()
        st = N.stream_handle(self.stream)
        ps = self.pool_set()
        N.check(lib.ss_stage_counts_validate(ps, N.ptr(self.koff), N.ptr(self.stages), N.ptr(self.status),
                                             N.ptr(self.aux), st), "ss_stage_counts_validate")
        if self.exact.size:
            self._run_exact(lib, ps, st)
        N.check(lib.ss_stage_counts_cover(ps, N.ptr(self.koff), N.ptr(self.stages), N.ptr(self.members),
                                          N.ptr(self.gsize), N.ptr(self.status), N.ptr(self.cand_pool),
                                          N.ptr(self.cand_k), self.n_cover, N.ptr(self.stall), self.max_layers, st),
                "ss_stage_counts_cover")

    def _run_exact(self, lib, ps, st) -> None:
        # a pool whose frontier outgrows the workspace reports SS_WORKSPACE (aux = the size it needed): grow and
        # rerun here (one host sync), or -- deferred -- in fetch(), which replays the whole launch log
        torch = _torch()
        while True:
            per = int(lib.ss_stage_counts_workspace(self.fcap, self.ccap, 17))
            per = (per + 255) // 256 * 256
            self._ws = torch.empty(per * self.exact.size, dtype=torch.uint8, device=self.dev)
            N.check(lib.ss_stage_counts_exact(ps, N.ptr(self.koff), N.ptr(self.stages), N.ptr(self.members),
                                              N.ptr(self.gsize), N.ptr(self.status), N.ptr(self.aux),
                                              N.ptr(self.exact_list), int(self.exact.size), N.ptr(self._ws), per,
                                              self.fcap, self.ccap, N.ptr(self.sweep_stats), st),
                    "ss_stage_counts_exact")
            if self.defer:
                return
            status = self.status.cpu().numpy()[self.exact]
            if not (status == SS_WORKSPACE).any():
                return
            need = int(self.aux.cpu().numpy()[self.exact].max())
            self._grow(need)
            bad = self.exact[status == SS_WORKSPACE]
            self.status[torch.from_numpy(bad).to(self.dev)] = SS_OK

    def _grow(self, need: int) -> None:
        self.fcap = max(self.fcap * 4, need * 2)
        self.ccap = max(self.ccap * 4, need * 2)
        if self.ccap > 1 << 24:
            raise MemoryError("exact sweep frontier exceeds 16M children")

    # -- objective + score + best -----------------------------------------
    def score_and_best(self, t_comp, rtt, kpow, fill_all: bool = False) -> None:
        torch = _torch()
        self._t = t_comp if torch.is_tensor(t_comp) else torch.as_tensor(np.asarray(t_comp, dtype=np.float64)).to(self.dev)
        self._r = rtt if torch.is_tensor(rtt) else torch.as_tensor(np.asarray(rtt, dtype=np.float64)).to(self.dev)
        self._kpow = kpow if torch.is_tensor(kpow) else torch.from_numpy(np.asarray(kpow, dtype=np.float64)).to(self.dev)
        self._fill_all = fill_all
        self._ops.append(self._score_and_best)
        self._score_and_best()

    def log_op(self, fn) -> None:
        """Run a further launch on this batch's outputs and record it for fetch()'s replay."""
        self._ops.append(fn)
        fn()

    def _score_and_best(self) -> None:
        lib = N.lib()
        st = N.stream_handle(self.stream)
        ps = self.pool_set()
        fill_all = self._fill_all
        N.check(lib.ss_phase1_score(ps, N.ptr(self.koff), N.ptr(self.stages), N.ptr(self.members), N.ptr(self.gsize),
                                    N.ptr(self._t), N.ptr(self._r), N.ptr(self._kpow), int(self._kpow.numel()),
                                    int(fill_all), N.ptr(self.z), N.ptr(self.counts), N.ptr(self.kstatus),
                                    N.ptr(self.fstatus), N.ptr(self.all_pool), N.ptr(self.all_k), self.n_cand, st),
                "ss_phase1_score")
        N.check(lib.ss_phase1_best(ps, N.ptr(self.koff), N.ptr(self.stages), N.ptr(self.members), N.ptr(self.gsize),
                                   N.ptr(self.z), N.ptr(self.kstatus), N.ptr(self.fstatus), int(fill_all),
                                   N.ptr(self.best_k), N.ptr(self.counts), N.ptr(self.status), st), "ss_phase1_best")

    # -- host views ---------------------------------------------------------
    def fetch(self) -> "PoolResults":
        res = PoolResults(self)
        while self.exact.size:
            st = res.status[self.exact]
            if not (st == SS_WORKSPACE).any():
                break
            self._grow(int(res.aux[self.exact].max()))
            for op in self._ops:                           # validate resets status / aux / stages
                op()
            res = PoolResults(self)
        return res


class PoolResults:
    """Host copy of a PoolBatch's outputs with reference-shaped accessors."""

    def __init__(self, b: PoolBatch):
        self.b = b
        ob = b._oblock.cpu().numpy()                       # the one D2H of the call
        nf = b._fblock.numel()
        fb = ob[:nf * 8].view(np.float64)
        ib = ob[nf * 8:].view(np.int32)
        ibase = b._iblock.storage_offset()             # in int32 elements
        view = lambda t: ib[t.storage_offset() - ibase: t.storage_offset() - ibase + t.numel()]
        self.stages = view(b.stages)
        self.members = view(b.members)
        self.gsize = view(b.gsize)
        self.status = view(b.status)
        self.aux = view(b.aux)
        self.counts = view(b.counts)
        self.best_k = view(b.best_k)
        self.sweep_stats = view(b.sweep_stats).reshape(-1, 4)
        self.z = fb[:b.z.numel()]
        self.total = float(fb[-1])
        self.feasible = int(view(b.feasible)[0])

    def raise_pool(self, p: int) -> None:
        st = int(self.status[p])
        if st != SS_OK:
            raise_for_status(st, int(self.aux[p]), detail=f"pool {p}")

    def solutions(self, p: int):
        """{k: (stages, groups)} in increasing k (allocator.py:499-504 shape)."""
        b = self.b
        n, km = int(b.n[p]), int(b.km[p])
        out = {}
        for k in range(1, km + 1):
            s = int(self.stages[b.koff_h[p] + k - 1])
            if s == 0:
                continue
            base = int(b.memb_h[p] + (k - 1) * n)
            gbase = int(b.gsz_h[p] + (k - 1) * km)
            groups, pos = [], 0
            for g in range(k):
                sz = int(self.gsize[gbase + g])
                groups.append(tuple(int(x) for x in self.members[base + pos: base + pos + sz]))
                pos += sz
            out[k] = (s, tuple(groups))
        return out

    def best_groups(self, p: int):
        """(member arrays of the groups of the best k, water-filled layer counts in the same order) or None."""
        b = self.b
        k = int(self.best_k[p])
        if k < 1 or int(self.stages[b.koff_h[p] + k - 1]) == 0:
            return None
        n, km = int(b.n[p]), int(b.km[p])
        base = int(b.memb_h[p] + (k - 1) * n)
        total = int(self.stages[b.koff_h[p] + k - 1])
        sizes = self.gsize[int(b.gsz_h[p] + (k - 1) * km): int(b.gsz_h[p] + (k - 1) * km) + k]
        return self.members[base: base + total], sizes, self.counts[base: base + total]

    def z_of(self, p: int, k: int) -> float:
        return float(self.z[self.b.koff_h[p] + k - 1])

    def counts_of(self, p: int, k: int):
        b = self.b
        base = int(b.memb_h[p] + (k - 1) * int(b.n[p]))
        total = int(self.stages[b.koff_h[p] + k - 1])
        return [int(x) for x in self.counts[base: base + total]]


def objective_pack(items, layers: Sequence[int]):
    """Host arrays of estimate_objective_params for many regions (see objective_device): name -> ndarray for one
    Upload, plus (regions, link count, total matrix entries)."""
    n = np.array([len(f) for f, _ in items], dtype=np.int64)
    item_ptr = np.concatenate([[0], np.cumsum(n)])
    mat_off = np.concatenate([[0], np.cumsum(n * n)])
    flops = np.concatenate([np.asarray(f, dtype=np.float64) for f, _ in items])
    li, la, lb, lv = [], [], [], []
    for i, (_, links) in enumerate(items):
        for a, b, v in links:
            li.append(i)
            la.append(a)
            lb.append(b)
            lv.append(v)
    I, nl = len(items), len(li)
    if I > 65535:
        raise ValueError("at most 65535 objective regions per call")
    arrays = {"obj_ints": np.concatenate([item_ptr, n, layers, li, la, lb]).astype(np.int32),
              "obj_off": mat_off[:-1].astype(np.int64),
              "obj_lv": np.asarray(lv if nl else [0.0], dtype=np.float64),
              "obj_flops": flops}
    return arrays, (I, nl, int(mat_off[-1]))


def objective_launch(dv, meta, default_rtt: float, fpl: float, tokens: float, stream=None):
    """Launch ss_rtt_fill + ss_objective on uploaded objective_pack arrays; returns device (t_comp, rtt)."""
    torch = _torch()
    lib = N.lib()
    dev = dv["obj_flops"].device
    I, nl, mat_total = meta
    ints = dv["obj_ints"]
    item_ptr_d, dim_d = ints[:I + 1], ints[I + 1:2 * I + 1]
    layers_d = ints[2 * I + 1:3 * I + 1]
    li_d, la_d, lb_d = ints[3 * I + 1:3 * I + 1 + nl], ints[3 * I + 1 + nl:3 * I + 1 + 2 * nl], ints[3 * I + 1 + 2 * nl:]
    off_d, flops_d = dv["obj_off"], dv["obj_flops"]
    lv_d = dv["obj_lv"] if nl else None
    st = N.stream_handle(stream)
    rtt = torch.empty(max(mat_total, 1), dtype=torch.float64, device=dev)
    N.check(lib.ss_rtt_fill(I, N.ptr(off_d), N.ptr(dim_d), N.ptr(rtt), float(default_rtt), nl,
                            N.ptr(li_d) if nl else None, N.ptr(la_d) if nl else None, N.ptr(lb_d) if nl else None,
                            N.ptr(lv_d), st), "ss_rtt_fill")
    tr = torch.empty(2 * I, dtype=torch.float64, device=dev)
    t, r = tr[:I], tr[I:]
    N.check(lib.ss_objective(I, N.ptr(item_ptr_d), N.ptr(flops_d), N.ptr(off_d), N.ptr(rtt), float(fpl),
                             N.ptr(layers_d), float(tokens), N.ptr(t), N.ptr(r), st), "ss_objective")
    return t, r


def objective_device(items, default_rtt: float, fpl: float, layers: Sequence[int], tokens: float, stream=None):
    """estimate_objective_params for many regions on device.

    items: list of (flops_in_cluster_order, links) where links is a list of
    (a_idx, b_idx, rtt) with region-local cluster-order indices.  Returns
    device tensors (t_comp, rtt).
    """
    torch = _torch()
    arrays, meta = objective_pack(items, layers)
    up = Upload()                                          # one H2D for every input of the call
    for name, arr in arrays.items():
        up.add(name, arr)
    return objective_launch(up.upload(torch.device("cuda"), stream), meta, default_rtt, fpl, tokens, stream)


def objective_dense(flops_cluster_order, rtt_mats, fpl: float, layers: int, tokens: float, stream=None):
    """estimate_objective_params for many regions given dense rtt_s matrices (cluster order) -> (t_comp, rtt)."""
    torch = _torch()
    lib = N.lib()
    dev = torch.device("cuda")
    n = np.array([len(f) for f in flops_cluster_order], dtype=np.int64)
    item_ptr = np.concatenate([[0], np.cumsum(n)]).astype(np.int32)
    mat_off = np.concatenate([[0], np.cumsum(n * n)[:-1]]).astype(np.int64)
    I = len(n)
    flops = torch.from_numpy(np.concatenate([np.asarray(f, dtype=np.float64) for f in flops_cluster_order])).to(dev)
    rtt = torch.from_numpy(np.concatenate([np.asarray(m, dtype=np.float64).reshape(-1) for m in rtt_mats])).to(dev)
    ip = torch.from_numpy(item_ptr).to(dev)
    mo = torch.from_numpy(mat_off).to(dev)
    lay = torch.full((I,), int(layers), dtype=torch.int32, device=dev)
    t = torch.empty(I, dtype=torch.float64, device=dev)
    r = torch.empty(I, dtype=torch.float64, device=dev)
    N.check(lib.ss_objective(I, N.ptr(ip), N.ptr(flops), N.ptr(mo), N.ptr(rtt), float(fpl), N.ptr(lay), float(tokens),
                             N.ptr(t), N.ptr(r), N.stream_handle(stream)), "ss_objective")
    return t, r
