"""Batched device APIs (additive; no reference equivalent).

:class:`ScenarioReplayer` is the Phase-2 throughput path: many independent
cluster states (C4/C5) or one long stream (C2), each replaying
``route`` / ``release(i - W)`` op scripts with occupancy feedback entirely on
the device.  It is defined to be element-wise equal to looping the
reference's ``ChainRouter.route`` / ``release`` (router.py:247-260) on a
``PerfMap`` whose latency law is ``base_s(g) * (1 + occ) ** e``
(sim.py:182-183; bench.py:150-151) -- tests/test_gpu_parity.py checks that
against the oracle and the reference's golden replays.

Device layout per scenario s (capacity layout, no host sync needed):
  * layer columns at node slots ``s * cap_nodes + prefix(cap)[l]`` where cap_l
    = hosts of layer l in the base plan (churn only removes hosts);
  * edge block l -> l+1 at ``s * edge_stride + prefix(cap_l * cap_{l+1})``,
    actual R_l(s) x R_{l+1}(s) doubles row-major;
  * per-gpu arrays (base tau, occupancy) at ``s * N``.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native as N
from . import scenarios as _scen
from .errors import raise_for_status
from .scenarios import ScenarioSet


def occ_power_table(size: int, exponent: float = 1.0) -> np.ndarray:
    """occpow[o] = (1 + o) ** e with Python semantics (sim.py:183); exact for e = 1."""
    return np.array([float((1 + o) ** exponent) for o in range(size)], dtype=np.float64)


@dataclass
class ReplayResult:
    cost: Optional[object]        # torch float64 [S, n_req] (device)
    chain_hash: Optional[object]  # torch uint64 as int64 [S, n_req]
    gpus: Optional[object]        # torch int16 [S, n_req, L]
    status: object                # torch int32 [S]


def _replay_geometry(scen: ScenarioSet, window: int, max_requests: Optional[int], mode: str):
    """(kernel mode, hosts per layer of the base plan, slot capacity, occpow table length)."""
    L = scen.layer_count
    lo, hi = scen.slice_lo.astype(np.int64), scen.slice_hi.astype(np.int64)
    layers = np.arange(1, L + 1)
    cap = ((lo[None, :] <= layers[:, None]) & (hi[None, :] >= layers[:, None])).sum(axis=1)
    if (cap == 0).any():
        raise ValueError("base plan leaves a layer uncovered")
    # frontier |col_b U col_{b+1}| of the base plan, plus the slots held one boundary longer
    # (delayed reuse, replay_slots.cu), bounds the slots; departures only remove hosts, each join adds
    # at most one host per layer and one slot per boundary
    held = ((lo[None, :] <= layers[:-1, None] + 1) & (hi[None, :] >= layers[:-1, None] - 1)).sum(axis=1) \
        if L > 1 else np.zeros(1, dtype=np.int64)
    cap = cap + scen.joins
    held = held + scen.joins
    if scen.slice_lo_s is not None and not scen.device_events and scen.joins == 0:
        # explicit per-scenario placements (e.g. after a rebalance): the widest scenario bounds the layout
        cap, held = _explicit_widths(scen)
    s_cap = int(max(32, -(-int(held.max()) // 32) * 32))
    occ_len = window + 2 if window > 0 else (max_requests or 1 << 16) + 2
    probe = N.DagSet(scen.n_scenarios, int(cap.max()), L, scen.n_gpus, None, None, None, None, None, None, None)
    warp_ok = int(cap.max()) <= 32 and int(N.load_library().ss_replay_warp_smem(probe, window, occ_len,
                                                                                scen.n_gpus)) > 0
    tiles = region_tiles(scen) if mode in ("auto", "regions") else None
    if mode == "auto":
        if warp_ok:
            mode = "warp"
        elif tiles is not None and tiles.fits() and tiles.gap > 0 and int(cap.max()) <= 256:
            mode = "regions"
        else:
            mode = "slots" if s_cap <= 96 else "blocks"
    if mode == "warp" and not warp_ok:
        raise ValueError("warp mode needs <= 32 hosts per layer and edges + ring within 227 KB of shared memory")
    if mode == "regions" and (tiles is None or not tiles.fits() or int(cap.max()) > 256):
        raise ValueError("regions mode needs region indices, <= 8 regions and <= 32 frontier slots per region")
    if L < 2 and mode in ("slots", "cluster", "regions"):
        mode = "blocks"                      # no boundaries: nothing to tile
    return mode, cap, s_cap, occ_len


def _explicit_widths(scen: ScenarioSet):
    """Max over scenarios of hosts per layer and of frontier slots (+ the zombie boundary) per boundary."""
    L = scen.layer_count
    lo, hi = scen.slice_lo_s.astype(np.int64), scen.slice_hi_s.astype(np.int64)
    ok = ~scen.leave & (lo <= hi)
    s_idx, g_idx = np.nonzero(ok)
    a, b = lo[s_idx, g_idx], hi[s_idx, g_idx]
    d = np.zeros((scen.n_scenarios, L + 3), dtype=np.int64)
    np.add.at(d, (s_idx, a), 1)
    np.add.at(d, (s_idx, b + 1), -1)
    cap = np.cumsum(d, axis=1)[:, 1:L + 1].max(axis=0)
    # frontier interval of a host in boundaries [max(a-2, 0), b] (incl. the zombie boundary), b < L-1
    h = np.zeros((scen.n_scenarios, L + 2), dtype=np.int64)
    np.add.at(h, (s_idx, np.maximum(a - 2, 0)), 1)
    np.add.at(h, (s_idx, np.minimum(b, L - 2) + 1), -1)
    held = np.cumsum(h, axis=1)[:, :max(L - 1, 1)].max(axis=0)
    return cap, held


JITTER_MIN = float(_scen.JITTER_Q[0])     # ss_jitter / scenarios.jitter_factor: LogNormal(0, 0.2) quantile grid
JITTER_MAX = float(_scen.JITTER_Q[-1])
REGION_MAX_TILES = 8


class RegionTiles:
    """Region tiling of a scenario batch for ss_replay_regions (replay_regions.cu).

    tile_of[g]: the tile (a region of the pool that has GPUs) of pool GPU g; bounds = lb[T][T] ++ ub[T] ++ uni[T][T]
    (uni[S][D]: the common value of every S x D pool entry, NaN when they differ):
    lb[S][D] = min over S x D pool pairs of fl(rtt * JITTER_MIN) (<= every jittered entry: fl is monotone),
    ub[D] = max over D x D pairs of fl(rtt * JITTER_MAX).  held[t] = slots tile t needs (frontier + the zombie
    boundary + one per join), gap = min_{S != D} lb - max ub (> 0: cross-region blocks are expected to be
    skipped by the bound test)."""

    def __init__(self, scen: ScenarioSet):
        reg = np.asarray(scen.region_idx, dtype=np.int64)
        used = np.unique(reg)
        remap = np.full(int(reg.max()) + 1, -1, dtype=np.int64)
        remap[used] = np.arange(used.size)
        self.tile_of = remap[reg].astype(np.int32)
        self.n_tiles = int(used.size)
        T = self.n_tiles
        rtt = np.asarray(scen.base_rtt, dtype=np.float64)
        jmin, jmax = (JITTER_MIN, JITTER_MAX) if scen.jitter else (1.0, 1.0)
        lb = np.full((T, T), np.inf)
        ub = np.zeros(T)
        uni = np.full((T, T), np.nan)
        members = [np.nonzero(self.tile_of == t)[0] for t in range(T)]
        for a in range(T):
            ub[a] = float((rtt[np.ix_(members[a], members[a])] * jmax).max())
            for b in range(T):
                if a != b:
                    blk = rtt[np.ix_(members[a], members[b])]
                    lb[a, b] = float((blk * jmin).min())
                    if blk.size and np.isfinite(blk.flat[0]) and (blk == blk.flat[0]).all():
                        uni[a, b] = float(blk.flat[0])      # e.g. every pair at the default cross-region RTT
        self.bounds = np.concatenate([lb.reshape(-1), ub, uni.reshape(-1)])
        off = lb[~np.eye(T, dtype=bool)]
        self.gap = float(off.min() - ub.max()) if T > 1 else -np.inf
        # slots per tile: GPUs held at each boundary (interval [max(lo-2,0), hi] incl. the zombie boundary)
        L = scen.layer_count
        if scen.slice_lo_s is not None and not scen.device_events and scen.joins == 0:
            lo, hi = scen.slice_lo_s.astype(np.int64), scen.slice_hi_s.astype(np.int64)
            ok = ~scen.leave & (lo <= hi) & (hi >= 1)
        else:
            lo, hi = scen.slice_lo[None, :].astype(np.int64), scen.slice_hi[None, :].astype(np.int64)
            ok = (lo <= hi) & (hi >= 1)
        # per (scenario, tile) a difference array over the boundaries -> running counts -> the peak per tile
        nb = max(L - 1, 1)
        start = np.maximum(lo - 2, 0)
        end = np.minimum(hi, nb - 1)
        valid = ok & (start <= end)
        si, gi = np.nonzero(valid)
        held = np.zeros(T, dtype=np.int64)
        if si.size:
            n_rows = valid.shape[0]
            row = si * T + self.tile_of[gi]
            width = nb + 1
            delta = (np.bincount(row * width + start[si, gi], minlength=n_rows * T * width)
                     - np.bincount(row * width + end[si, gi] + 1, minlength=n_rows * T * width))
            counts = np.cumsum(delta.reshape(n_rows, T, width), axis=2)[:, :, :nb]
            held = counts.max(axis=(0, 2)).astype(np.int64)
        self.held = held + scen.joins

    def fits(self) -> bool:
        return 1 <= self.n_tiles <= REGION_MAX_TILES and int(self.held.max()) <= 32


def region_tiles(scen: ScenarioSet) -> Optional[RegionTiles]:
    if getattr(scen, "region_idx", None) is None or scen.layer_count < 2:
        return None
    cached = getattr(scen, "_region_tiles", None)             # a ScenarioSet is not mutated after it is built
    if cached is None:
        cached = RegionTiles(scen)
        try:
            scen._region_tiles = cached
        except AttributeError:
            pass
    return cached


def replay_mode(scen: ScenarioSet, *, window: int = 64, max_requests: Optional[int] = None,
                mode: str = "auto") -> str:
    """The replay kernel ScenarioReplayer would use for these scenarios (no GPU needed)."""
    return _replay_geometry(scen, int(window), max_requests, mode)[0]


class ScenarioReplayer:
    def __init__(self, scen: ScenarioSet, *, window: int = 64, exponent: float = 1.0,
                 max_requests: Optional[int] = None, stream=None, mode: str = "auto"):
        """mode "regions": one SM-resident slot tile per region of the pool, cross-region blocks relaxed only
        where an exact bound test cannot exclude them (ss_region_program + ss_replay_regions); "slots": SM-resident slot tile (ss_slot_program + ss_replay_slots, ~10x fewer HBM
        bytes); "cluster": the same tile split by destination slots over a thread-block cluster of CTAs
        (ss_replay_slots_cluster; wide frontiers); "blocks": streamed edge blocks (ss_dag_edges + ss_replay); "warp": one warp per scenario
        with its edge blocks resident in shared memory (ss_replay_warp; columns <= 32 hosts); "auto":
        warp when it qualifies, else slots while the tile leaves room for two CTAs per SM (<= 96 slots),
        else blocks.  All modes give bit-identical results."""
        import torch
        if mode not in ("slots", "cluster", "blocks", "warp", "regions", "auto"):
            raise ValueError(f"mode must be 'slots', 'cluster', 'blocks', 'warp', 'regions' or 'auto', got {mode!r}")
        self.torch = torch
        self.scen = scen
        self.window = int(window)
        self.stream = stream
        dev = torch.device("cuda")
        self.dev = dev
        S, G, L = scen.n_scenarios, scen.n_gpus, scen.layer_count
        self.S, self.G, self.L = S, G, L
        lo, hi = scen.slice_lo.astype(np.int64), scen.slice_hi.astype(np.int64)
        layers = np.arange(1, L + 1)
        mode, cap, s_cap, occ_len = _replay_geometry(scen, self.window, max_requests, mode)
        self.mode = mode
        self.cap = cap
        cap_nodes = int(cap.sum())
        node_pre = np.concatenate([[0], np.cumsum(cap)[:-1]])
        blk = cap[:-1] * cap[1:]
        blk = blk + (blk & 1)
        edge_pre = np.concatenate([[0], np.cumsum(blk)]) if L > 1 else np.zeros(1, dtype=np.int64)
        edge_stride = int(edge_pre[-1]) if L > 1 else 2
        self.edge_stride = edge_stride
        s_idx = np.arange(S, dtype=np.int64)
        col_off = (s_idx[:, None] * cap_nodes + node_pre[None, :]).reshape(-1)
        edge_off = (s_idx[:, None] * edge_stride + edge_pre[None, :L]).reshape(-1)
        layer_ptr = np.arange(S + 1, dtype=np.int64) * L
        gpu_ptr = np.arange(S + 1, dtype=np.int64) * G

        def up(a, dt):
            return torch.from_numpy(np.ascontiguousarray(a)).to(device=dev, dtype=dt)

        t32, t64, f64 = torch.int32, torch.int64, torch.float64
        self.layer_ptr = up(layer_ptr, t32)
        self.col_off = up(col_off, t32)
        self.edge_off = up(edge_off, t64)
        self.gpu_ptr = up(gpu_ptr, t32)
        self.col_len = torch.empty(S * L, dtype=t32, device=dev)
        self.node_gpu = torch.empty(S * cap_nodes, dtype=t32, device=dev)
        if mode in ("blocks", "warp"):
            self.edge_val = torch.empty(S * edge_stride, dtype=f64, device=dev)
        elif mode == "regions":
            self.edge_val = None
            tiles = region_tiles(scen)
            self.tiles = tiles
            self.pos_cap = int(min(256, -(-int(cap.max()) // 4) * 4))
            n_plan = int(((hi >= lo) & (hi >= 1)).sum()) + scen.joins
            lib = N.load_library()
            self.meta_stride = int(lib.ss_region_meta_bytes(L, G, tiles.n_tiles, self.pos_cap))
            self.stream_stride = 2 * max(n_plan, 1) * 32
            self.meta = torch.empty(S * self.meta_stride, dtype=torch.uint8, device=dev)
            self.stream_buf = torch.empty(max(S * self.stream_stride, 2), dtype=f64, device=dev)
            self.s_used = torch.zeros(S, dtype=t32, device=dev)
            self.prog_status = torch.zeros(S, dtype=t32, device=dev)
            self.tile_of = up(tiles.tile_of, t32)
            self.bounds = up(tiles.bounds, f64)
            self.s_rows = 32
        else:
            self.edge_val = None
            if s_cap > 256:
                raise ValueError(f"slot mode supports <= 256 frontier slots, this plan needs {s_cap}")
            self.s_cap = s_cap
            n_plan = int(((hi >= lo) & (hi >= 1)).sum())
            lib = N.load_library()
            self.meta_stride = int(lib.ss_slot_meta_bytes(L, G, self.s_cap))
            self.stream_stride = 2 * n_plan * self.s_cap
            self.meta = torch.empty(S * self.meta_stride, dtype=torch.uint8, device=dev)
            self.stream_buf = torch.empty(max(S * self.stream_stride, 2), dtype=f64, device=dev)
            self.s_used = torch.zeros(S, dtype=t32, device=dev)
            self.prog_status = torch.zeros(S, dtype=t32, device=dev)
            self.s_rows = self.s_cap
        self.base_tau = up(np.tile(scen.base_tau, S), f64)
        self.slice_lo = up(lo, t32)
        self.slice_hi = up(hi, t32)
        self.leave = up(scen.leave.astype(np.uint8), torch.uint8)
        # per-scenario slices (joins): host-made, or written by ss_scenario_membership in build()
        self.per_scenario = scen.joins > 0 or scen.device_events or scen.slice_lo_s is not None
        if self.per_scenario:
            if scen.slice_lo_s is not None and not scen.device_events:
                self.lo_s, self.hi_s = up(scen.slice_lo_s, t32), up(scen.slice_hi_s, t32)
            else:
                self.lo_s = torch.zeros(S * G, dtype=t32, device=dev)
                self.hi_s = torch.zeros(S * G, dtype=t32, device=dev)
            self.joined = torch.full((S * max(scen.joins, 1),), -1, dtype=t32, device=dev)
            if scen.joined_s is not None and scen.joins > 0:
                self.joined.copy_(torch.from_numpy(np.ascontiguousarray(scen.joined_s.reshape(-1))))
        if scen.device_events:
            self.present0 = up(scen.present0.astype(np.uint8), torch.uint8)
            self.token_cap = up(scen.token_cap, t64)
            self.layer_cap = up(scen.layer_cap, t32)
        self.seeds = up(scen.seeds.astype(np.int64), t64)
        self.base_rtt = up(scen.base_rtt.reshape(-1), f64)
        self.occ = torch.zeros(S * G, dtype=t32, device=dev)
        self.ring = torch.zeros(S * max(self.window, 1) * (L + 1), dtype=t32, device=dev)
        self.next_req = torch.zeros(S, dtype=t64, device=dev)
        self.status = torch.zeros(S, dtype=t32, device=dev)
        self.aux = torch.zeros(S, dtype=t32, device=dev)
        size = occ_len
        self.occpow_len = size
        self.occpow = up(occ_power_table(size, exponent), f64)
        self.max_hosts = int(cap.max())
        self.built = False

    # ------------------------------------------------------------------
    def dag_set(self) -> N.DagSet:
        return N.DagSet(self.S, self.max_hosts, self.L, self.G, N.ptr(self.layer_ptr), N.ptr(self.col_off),
                        N.ptr(self.col_len), N.ptr(self.node_gpu), None, N.ptr(self.edge_off),
                        N.ptr(self.edge_val) if self.edge_val is not None else None)

    def build(self) -> None:
        """Scenario columns + jittered edge blocks, fully on device (ss_scenario_columns, ss_dag_edges)."""
        lib = N.lib()
        st = N.stream_handle(self.stream)
        if self.scen.device_events:
            # membership churn on device: leaves + joins from the scenario seeds (no host prep)
            N.check(lib.ss_scenario_membership(self.S, self.L, self.G, N.ptr(self.slice_lo), N.ptr(self.slice_hi),
                                               N.ptr(self.present0), N.ptr(self.token_cap), N.ptr(self.layer_cap),
                                               N.ptr(self.seeds), self.scen.want_leave, self.scen.joins,
                                               N.ptr(self.leave), N.ptr(self.lo_s), N.ptr(self.hi_s),
                                               N.ptr(self.joined), N.ptr(self.status), N.ptr(self.aux), st),
                    "ss_scenario_membership")
        lo_p, hi_p, stride = ((self.lo_s, self.hi_s, self.G) if self.per_scenario
                              else (self.slice_lo, self.slice_hi, 0))
        N.check(lib.ss_scenario_columns(self.S, self.L, self.G, N.ptr(lo_p), N.ptr(hi_p), stride,
                                        N.ptr(self.leave), N.ptr(self.col_off), N.ptr(self.col_len),
                                        N.ptr(self.node_gpu), N.ptr(self.status), N.ptr(self.aux), st),
                "ss_scenario_columns")
        if self.mode in ("slots", "cluster"):
            N.check(lib.ss_slot_program(self.S, self.L, self.G, N.ptr(lo_p), N.ptr(hi_p), stride,
                                        N.ptr(self.leave), N.ptr(self.base_rtt),
                                        N.ptr(self.seeds) if self.scen.jitter else None, self.s_cap, self.meta_stride,
                                        self.stream_stride, N.ptr(self.meta), N.ptr(self.stream_buf),
                                        N.ptr(self.s_used), N.ptr(self.prog_status), st), "ss_slot_program")
            # one small D2H: the tile is sized by the slots actually used (two CTAs per SM at C4)
            used = self.s_used.cpu().numpy()
            bad = np.nonzero(self.prog_status.cpu().numpy())[0]
            if bad.size:
                raise ValueError(f"slot program failed for scenario {int(bad[0])} (slots > {self.s_cap})")
            self.s_rows = int(max(1, used.max()))
        elif self.mode == "regions":
            N.check(lib.ss_region_program(self.S, self.L, self.G, N.ptr(lo_p), N.ptr(hi_p), stride,
                                          N.ptr(self.leave), N.ptr(self.base_rtt),
                                          N.ptr(self.seeds) if self.scen.jitter else None, N.ptr(self.tile_of),
                                          self.tiles.n_tiles, self.pos_cap, self.meta_stride, self.stream_stride,
                                          N.ptr(self.meta), N.ptr(self.stream_buf), N.ptr(self.s_used),
                                          N.ptr(self.prog_status), st), "ss_region_program")
            used = self.s_used.cpu().numpy()
            bad = np.nonzero(self.prog_status.cpu().numpy())[0]
            if bad.size:
                raise ValueError(f"region program failed for scenario {int(bad[0])} (a region needs > 32 slots)")
            self.s_rows = int(max(1, used.max()))
        elif self.scen.jitter:
            N.check(lib.ss_dag_edges(self.dag_set(), None, None, N.ptr(self.base_rtt), N.ptr(self.seeds), self.G,
                                     N.ptr(self.edge_val), st), "ss_dag_edges")
        else:
            torch = self.torch
            if not hasattr(self, "_rtt_off"):
                self._rtt_off = torch.zeros(self.S, dtype=torch.int64, device=self.dev)
                self._rtt_dim = torch.full((self.S,), self.G, dtype=torch.int32, device=self.dev)
            N.check(lib.ss_dag_edges(self.dag_set(), N.ptr(self._rtt_off), N.ptr(self._rtt_dim), N.ptr(self.base_rtt),
                                     None, 0, N.ptr(self.edge_val), st), "ss_dag_edges")
        self.built = True

    def reset(self) -> None:
        self.occ.zero_()
        self.ring.zero_()
        self.next_req.zero_()

    def _scenario_mats(self):
        """Per-scenario RTT matrices [S, G, G] on device (ScenarioSet.scenario_rtt), built once."""
        torch = self.torch
        if getattr(self, "_mats", None) is None:
            S, G = self.S, self.G
            if self.scen.jitter:
                self._mats = torch.empty(S * G * G, dtype=torch.float64, device=self.dev)
                N.check(N.lib().ss_scenario_rtt(S, G, N.ptr(self.base_rtt), N.ptr(self.seeds), N.ptr(self._mats),
                                                N.stream_handle(self.stream)), "ss_scenario_rtt")
            else:
                self._mats = self.base_rtt.reshape(-1).repeat(S)
        return self._mats

    def _warp_mats(self):
        """The matrices for the warp kernels' matrix mode, or None when the edge blocks are smaller."""
        if self.G * self.G >= (self.L - 1) * self.max_hosts * self.max_hosts or self.S <= 148:
            return None                                  # warp_layout would stage the edge blocks anyway
        return self._scenario_mats()

    def run(self, n_req: int, *, cost: bool = True, hashes: bool = True, gpus: bool = False,
            out: Optional[ReplayResult] = None) -> ReplayResult:
        torch = self.torch
        if not self.built:
            self.build()
        S, L = self.S, self.L
        if out is None:
            out = ReplayResult(
                torch.empty((S, n_req), dtype=torch.float64, device=self.dev) if cost else None,
                torch.empty((S, n_req), dtype=torch.int64, device=self.dev) if hashes else None,
                torch.empty((S, n_req, L), dtype=torch.int16, device=self.dev) if gpus else None,
                self.status)
        st = N.ReplayState(N.ptr(self.gpu_ptr), N.ptr(self.base_tau), N.ptr(self.occ), N.ptr(self.ring),
                           N.ptr(self.next_req), N.ptr(self.status), N.ptr(self.aux))
        ro = N.ReplayOut(N.ptr(out.cost), N.ptr(out.chain_hash), N.ptr(out.gpus))
        if self.mode == "slots":
            N.check(N.lib().ss_replay_slots(self.dag_set(), N.ptr(self.meta), self.meta_stride, N.ptr(self.stream_buf),
                                            self.stream_stride, self.s_cap, self.s_rows, st, N.ptr(self.occpow),
                                            self.occpow_len, self.window, n_req, ro, N.stream_handle(self.stream)),
                    "ss_replay_slots")
        elif self.mode == "regions":
            N.check(N.lib().ss_replay_regions(self.dag_set(), N.ptr(self.meta), self.meta_stride,
                                              N.ptr(self.stream_buf), self.stream_stride, self.tiles.n_tiles,
                                              self.pos_cap, self.s_rows, N.ptr(self.bounds), N.ptr(self.base_rtt),
                                              N.ptr(self.seeds) if self.scen.jitter else None, st,
                                              N.ptr(self.occpow), self.occpow_len, self.window, n_req, ro,
                                              N.stream_handle(self.stream)), "ss_replay_regions")
        elif self.mode == "cluster":
            N.check(N.lib().ss_replay_slots_cluster(self.dag_set(), N.ptr(self.meta), self.meta_stride,
                                                    N.ptr(self.stream_buf), self.stream_stride, self.s_cap,
                                                    self.s_rows, st, N.ptr(self.occpow), self.occpow_len, self.window,
                                                    n_req, ro, 0, N.stream_handle(self.stream)),
                    "ss_replay_slots_cluster")
        elif self.mode == "warp":
            mat = self._warp_mats()
            N.check(N.lib().ss_replay_warp(self.dag_set(), st, N.ptr(self.occpow), self.occpow_len, self.window,
                                           n_req, ro, N.ptr(mat), self.G, N.stream_handle(self.stream)),
                    "ss_replay_warp")
        else:
            N.check(N.lib().ss_replay(self.dag_set(), st, N.ptr(self.occpow), self.occpow_len, self.window, n_req,
                                      ro, N.stream_handle(self.stream)), "ss_replay")
        return out

    def run_from_host(self, leave_h, seeds_h, n_req: int, cost_h, hash_h, gpus_h=None) -> ReplayResult:
        """End-to-end call: host scenario descriptors in, host per-request results out.

        leave_h [S, N] uint8 (None when the scenario events are generated on
        the device) and seeds_h [S] int64 (pinned) are copied to the device,
        the replay state is reset inside the C ABI (ss_replay_reset:
        cudaMemsetAsync, no kernel), the scenario DAGs are rebuilt (membership
        events, columns, edge blocks or slot program), n_req requests are
        routed per scenario and the costs / chain hashes -- and with gpus_h
        [S, n_req, L] int16 the chains themselves -- come back into pinned
        host buffers.  Stream-ordered; the caller synchronises.
        """
        if leave_h is not None:
            self.leave.copy_(leave_h, non_blocking=True)
        self.seeds.copy_(seeds_h, non_blocking=True)
        st = N.ReplayState(N.ptr(self.gpu_ptr), N.ptr(self.base_tau), N.ptr(self.occ), N.ptr(self.ring),
                           N.ptr(self.next_req), N.ptr(self.status), N.ptr(self.aux))
        N.check(N.lib().ss_replay_reset(st, self.S, self.occ.numel(), self.ring.numel(), N.stream_handle(self.stream)),
                "ss_replay_reset")
        self.build()
        out = self.run(n_req, gpus=gpus_h is not None)
        cost_h.copy_(out.cost, non_blocking=True)
        hash_h.copy_(out.chain_hash, non_blocking=True)
        if gpus_h is not None:
            gpus_h.copy_(out.gpus, non_blocking=True)
        return out

    def triggers(self, *, cov_threshold: float = 0.5, mix_alpha: float = 0.5, kv_reserved=None):
        """evaluate_triggers of every scenario on the current occupancy (membership.py:389-396).

        Returns (decision int32 [S]: 0 local, 1 global/uncovered_layers, 2 global/load_cov_exceeded;
        cov float64 [S]; first uncovered layer int32 [S]; loads float64 [S, L]) as device tensors.
        """
        torch = self.torch
        sc = self.scen
        if not hasattr(self, "_trig"):
            up = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(device=self.dev, dtype=dt)
            self._trig = dict(order=up(sc.cluster_order, torch.int32), sorder=up(sc.plan_order, torch.int32),
                              vram=up(sc.vram, torch.float64), reserve=up(sc.reserve, torch.float64),
                              flops=up(sc.flops, torch.float64), token=up(sc.token_cap, torch.int64))
            if not self.per_scenario:
                self._trig["lo"] = self.slice_lo
                self._trig["hi"] = self.slice_hi
        t = self._trig
        lo, hi, stride = ((self.lo_s, self.hi_s, self.G) if self.per_scenario else (t["lo"], t["hi"], 0))
        S, L = self.S, self.L
        dec = torch.empty(S, dtype=torch.int32, device=self.dev)
        cov = torch.empty(S, dtype=torch.float64, device=self.dev)
        hole = torch.empty(S, dtype=torch.int32, device=self.dev)
        loads = torch.empty((S, L), dtype=torch.float64, device=self.dev)
        n_join = self.scen.joins if self.per_scenario else 0
        if sc.slice_order_s is not None:
            if "sorder_s" not in t:
                t["sorder_s"] = torch.from_numpy(np.ascontiguousarray(sc.slice_order_s)).to(self.dev,
                                                                                          dtype=torch.int32)
                t["joined_s"] = torch.from_numpy(np.ascontiguousarray(sc.joined_s)).to(self.dev, dtype=torch.int32)
            sorder, n_sorder, ostride = t["sorder_s"], sc.slice_order_s.shape[1], sc.slice_order_s.shape[1]
            jn, n_join = t["joined_s"], sc.joined_s.shape[1]
        else:
            sorder, n_sorder, ostride = t["sorder"], len(sc.plan_order), 0
            jn = self.joined if n_join else None
        N.check(N.lib().ss_membership_triggers(
            S, L, self.G, N.ptr(self.leave), N.ptr(lo), N.ptr(hi), stride, N.ptr(t["order"]), len(sc.cluster_order),
            N.ptr(sorder), n_sorder, ostride, N.ptr(jn) if jn is not None else None, n_join,
            N.ptr(t["vram"]), N.ptr(t["reserve"]), N.ptr(t["flops"]), N.ptr(t["token"]),
            N.ptr(kv_reserved) if kv_reserved is not None else None, N.ptr(self.occ), self.G, float(mix_alpha),
            float(cov_threshold), N.ptr(loads), N.ptr(cov), N.ptr(dec), N.ptr(hole), N.stream_handle(self.stream)),
            "ss_membership_triggers")
        return dec, cov, hole, loads

    def rebalance(self, *, cov_threshold: float = 0.5, mix_alpha: float = 0.5, alpha: float = 1.0,
                  tokens: float = 128.0, force=None):
        """Global rebalance of the scenarios whose evaluate_triggers() says "global" (or of ``force``).

        Per scenario, as MembershipManager.global_rebalance (membership.py:398-411) and the simulator
        (sim.py:425-429): allocate() on the churned pool -- all selected scenarios' regions in ONE device
        Phase-1 batch (stage counts, objective, score, best k, water-fill) -- then apply_plan (new slices,
        changed_gpus) and the abort of every live chain on a changed GPU (ss_ring_abort).  A scenario whose
        pool has no feasible pipeline keeps its placement (degraded).

        Returns (replayer for the new placements carrying occupancy / ring / request counters, info) where
        info has per-scenario "decision", "rebalanced", "degraded", "changed" (GPU indices), "aborted".
        """
        import dataclasses
        from ._phase1 import PoolArrays, PoolBatch, _ramp
        from .errors import SS_OK as SS_OK_STATUS
        torch = self.torch
        sc = self.scen
        S, G, L = self.S, self.G, self.L
        dec = self.triggers(cov_threshold=cov_threshold, mix_alpha=mix_alpha)[0].cpu().numpy()
        sel = np.nonzero(dec != 0)[0] if force is None else np.asarray(force, dtype=np.int64)
        absent = self.leave.view(S, G).cpu().numpy().astype(bool)
        if self.per_scenario:
            lo = self.lo_s.view(S, G).cpu().numpy().copy()
            hi = self.hi_s.view(S, G).cpu().numpy().copy()
        else:
            lo = np.broadcast_to(sc.slice_lo, (S, G)).astype(np.int32).copy()
            hi = np.broadcast_to(sc.slice_hi, (S, G)).astype(np.int32).copy()
        if sc.joins > 0:
            joined = self.joined.view(S, -1).cpu().numpy().copy()
        else:
            joined = np.full((S, 1), -1, dtype=np.int32) if sc.joined_s is None else sc.joined_s.copy()
        # current slices order per scenario: the plan's then the joins (or the last rebalance's plan order)
        if sc.slice_order_s is not None:
            order = sc.slice_order_s.copy()
        else:
            po = np.asarray(sc.plan_order, dtype=np.int64)
            jn = joined.astype(np.int64)
            jv = np.where(jn >= 0, jn, 0)
            rows = np.arange(S)[:, None]
            cand = np.concatenate([np.broadcast_to(po, (S, po.size)), jn], axis=1)
            keep = np.concatenate([~absent[:, po], (jn >= 0) & (lo[rows, jv] <= hi[rows, jv])], axis=1)
            first = np.argsort(~keep, axis=1, kind="stable")          # kept entries first, in list order
            order = np.full((S, G), -1, dtype=np.int32)
            packed_o = np.take_along_axis(cand, first, axis=1)[:, :G]
            cnt = keep.sum(axis=1)
            order[:, :packed_o.shape[1]] = np.where(np.arange(packed_o.shape[1])[None, :] < cnt[:, None], packed_o, -1)
        # the churned pools, vectorised over scenarios: region by region (sorted names), the present GPUs of each
        # selected scenario in (-capacity, id) order (allocator.py:570); id order for the objective items
        sel = np.asarray(sel, dtype=np.int64)
        pres = ~absent[sel]
        P_n, P_caps, P_flops, P_km, P_scen, P_owner, I_gpu = [], [], [], [], [], [], []
        for r in range(len(sc.region_names)):
            gr = np.nonzero(sc.region_idx == r)[0]
            if gr.size == 0 or sel.size == 0:
                continue
            capr = sc.layer_cap[gr].astype(np.int64)
            o_r = np.lexsort((gr, -capr))
            pr_id = pres[:, gr]
            cnt = pr_id.sum(axis=1)
            limit = np.minimum(cnt, (pr_id * capr).sum(axis=1) // L)
            ok = (cnt > 0) & (limit >= 1)
            rows = np.nonzero(ok)[0]
            if rows.size == 0:
                continue
            pr_o = pr_id[rows][:, o_r]
            P_n.append(cnt[rows])
            P_km.append(limit[rows])
            P_scen.append(sel[rows])
            P_caps.append(np.broadcast_to(capr[o_r], pr_o.shape)[pr_o])
            P_flops.append(np.broadcast_to(sc.flops[gr][o_r], pr_o.shape)[pr_o])
            P_owner.append(np.broadcast_to(gr[o_r], pr_o.shape)[pr_o])
            I_gpu.append(np.broadcast_to(gr, (rows.size, gr.size))[pr_id[rows]])
        info = {"decision": dec, "rebalanced": np.zeros(S, dtype=bool), "degraded": np.zeros(S, dtype=bool),
                "changed": [[] for _ in range(S)], "aborted": np.zeros(S, dtype=np.int32)}
        new_lo, new_hi = lo.copy(), hi.copy()
        if P_n:
            # pools in (scenario, region) order, as the per-scenario allocate() calls would see them
            cat = lambda xs: np.concatenate(xs)
            pn, pkm, pscen = cat(P_n), cat(P_km), cat(P_scen)
            ptr0 = np.concatenate([[0], np.cumsum(pn)])
            perm = np.argsort(pscen, kind="stable")
            pn, pkm, pscen = pn[perm], pkm[perm], pscen[perm]
            gath = np.repeat(ptr0[perm], pn) + _ramp(pn) - 1                # pool-major gather in the new order
            caps_f, flops_f, owner_f = cat(P_caps)[gath], cat(P_flops)[gath], cat(P_owner)[gath]
            igpu_f = cat(I_gpu)[gath]                       # objective items: id order, same pool sizes
            n_it = int(pn.size)
            batch = PoolBatch(arrays=PoolArrays(pn, caps_f, flops_f, np.full(n_it, L, dtype=np.int64), pkm),
                              stream=self.stream)
            batch.stage_counts()
            # estimate_objective_params per churned region, gathered from the pool on device (no dense copies)
            iptr = np.concatenate([[0], np.cumsum(pn)]).astype(np.int32)
            up = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(device=self.dev, dtype=dt)
            if not hasattr(self, "_pool_flops"):
                self._pool_flops = up(sc.flops, torch.float64)
            t = torch.empty(n_it, dtype=torch.float64, device=self.dev)
            r = torch.empty(n_it, dtype=torch.float64, device=self.dev)
            ip_d, g_d = up(iptr, torch.int32), up(igpu_f, torch.int32)
            lay_d = torch.full((n_it,), L, dtype=torch.int32, device=self.dev)
            seed_d = up(sc.seeds[pscen].astype(np.int64), torch.int64) if sc.jitter else None
            N.check(N.lib().ss_objective_pool(n_it, N.ptr(ip_d), N.ptr(g_d), N.ptr(self._pool_flops),
                                              N.ptr(self.base_rtt), G, N.ptr(seed_d) if seed_d is not None else None,
                                              float(sc.fpl), N.ptr(lay_d), float(tokens), N.ptr(t), N.ptr(r),
                                              N.stream_handle(self.stream)), "ss_objective_pool")
            km = int(batch.km.max())
            batch.score_and_best(t, r, np.array([0.0] + [float(k ** alpha) for k in range(1, km + 1)]))
            res = batch.fetch()
            bad = np.nonzero(res.status != SS_OK_STATUS)[0]
            if bad.size:
                res.raise_pool(int(bad[0]))
            # best-k groups of every pool, flattened: member -> (pool, group, layer count)
            bk = res.best_k.astype(np.int64)
            kidx = batch.koff_h[:-1] + np.maximum(bk, 1) - 1
            total = np.where(bk >= 1, res.stages[kidx], 0).astype(np.int64)
            mbase = batch.memb_h[:-1] + (np.maximum(bk, 1) - 1) * pn
            midx = np.repeat(mbase, total) + _ramp(total) - 1
            members, counts = res.members[midx].astype(np.int64), res.counts[midx].astype(np.int64)
            kk = np.where(total > 0, bk, 0)
            gidx = np.repeat(batch.gsz_h[:-1] + (np.maximum(bk, 1) - 1) * pkm, kk) + _ramp(kk) - 1
            sizes = res.gsize[gidx].astype(np.int64)
            # contiguous slices from layer 1 inside every group (allocator.py:595-606)
            ends_all = np.cumsum(counts)
            gstart = np.repeat(np.cumsum(sizes) - sizes, sizes)            # first member of each member's group
            before = np.concatenate([[0], ends_all])[gstart]
            e = ends_all - before
            mpool = np.repeat(np.arange(n_it), total)
            g_all = owner_f[np.repeat(np.concatenate([[0], np.cumsum(pn)])[:-1], total) + members]
            m_scen = pscen[mpool]
            ok_s = np.zeros(S, dtype=bool)
            ok_s[m_scen] = True
            for s_ in sel[~ok_s[sel]]:                                   # NoFeasiblePipeline: keep the slices
                info["degraded"][int(s_)] = True
            done_s = np.nonzero(ok_s)[0]
            new_lo[done_s], new_hi[done_s] = 0, -1
            new_lo[m_scen, g_all] = e - counts + 1
            new_hi[m_scen, g_all] = e
            order[done_s] = -1
            rank = np.arange(m_scen.size) - np.searchsorted(m_scen, m_scen, side="left")
            order[m_scen, rank] = g_all
            info["rebalanced"][done_s] = True
        key0 = np.where(lo <= hi, lo.astype(np.int64) * 100000 + hi, -1)
        key1 = np.where(new_lo <= new_hi, new_lo.astype(np.int64) * 100000 + new_hi, -1)
        changed = key0 != key1
        for s in range(S):
            info["changed"][s] = np.nonzero(changed[s])[0].tolist()
        if self.window != 0 and changed.any():
            if self.window < 0:
                raise ValueError("aborting live chains needs a release window (W > 0)")
            mark = torch.from_numpy(changed.astype(np.uint8).reshape(-1)).to(self.dev)
            n_ab = torch.zeros(S, dtype=torch.int32, device=self.dev)
            N.check(N.lib().ss_ring_abort(S, G, L, self.window, N.ptr(mark), N.ptr(self.occ), N.ptr(self.ring),
                                          N.ptr(self.next_req), N.ptr(n_ab), None, N.stream_handle(self.stream)),
                    "ss_ring_abort")
            info["aborted"] = n_ab.cpu().numpy()
        new_set = dataclasses.replace(sc, leave=absent, slice_lo_s=new_lo.astype(np.int32),
                                      slice_hi_s=new_hi.astype(np.int32), device_events=False, joins=0,
                                      slice_order_s=order, joined_s=joined)
        rp = ScenarioReplayer(new_set, window=self.window, max_requests=self.occpow_len - 2, stream=self.stream)
        rp.adopt_state(self)
        rp.build()
        return rp, info

    def admit(self, steps: int, *, tok_lo: int, tok_hi: int, gpus: bool = False):
        """The simulator's admission path (sim.py:319-366) for every scenario on device (ss_admission_warp):
        step t completes the admissions of step t - W, enqueues request t and drains the queue strictly FIFO,
        each head routed with the KV-blocked GPUs excluded.  Needs mode "warp" (<= 32 hosts per layer); starts
        from zero occupancy / reservations.  Returns dict of device tensors: step [S, steps] (-1 = still
        queued), cost [S, steps], gpus [S, steps, L] (optional), kv [S, N], occ [S, N].
        """
        torch = self.torch
        if self.mode != "warp":
            raise ValueError("admission replay runs on the warp-resident kernel (<= 32 hosts per layer)")
        if self.window < 1:
            raise ValueError("admission needs a completion window W >= 1")
        if not self.built:
            self.build()
        S, G, L = self.S, self.G, self.L
        if not hasattr(self, "_tokcap"):
            self._tokcap = torch.from_numpy(np.tile(self.scen.token_cap, S)).to(self.dev)
        occpow = torch.from_numpy(occ_power_table(steps + 2)).to(self.dev)
        adm = torch.empty(S * steps * (L + 1), dtype=torch.int32, device=self.dev)
        out = {"step": torch.empty((S, steps), dtype=torch.int32, device=self.dev),
               "cost": torch.empty((S, steps), dtype=torch.float64, device=self.dev),
               "gpus": torch.empty((S, steps, L), dtype=torch.int16, device=self.dev) if gpus else None,
               "kv": torch.empty((S, G), dtype=torch.int64, device=self.dev),
               "occ": torch.empty((S, G), dtype=torch.int32, device=self.dev)}
        N.check(N.lib().ss_admission_warp(self.dag_set(), N.ptr(self.gpu_ptr), N.ptr(self.base_tau),
                                          N.ptr(self._tokcap), N.ptr(occpow), steps + 2, N.ptr(self.seeds),
                                          int(tok_lo), int(tok_hi), int(steps), self.window, N.ptr(adm),
                                          N.ptr(out["step"]), N.ptr(out["cost"]), N.ptr(out["gpus"]), N.ptr(out["kv"]),
                                          N.ptr(out["occ"]), N.ptr(self.status), N.ptr(self.aux),
                                          N.ptr(self._warp_mats()), self.G, N.stream_handle(self.stream)),
                "ss_admission_warp")
        return out

    def simulate(self, traces, *, publish_interval: float = 1.5, amortize_rtt: bool = False,
                 contention: float = 1.0, max_live: Optional[int] = None):
        """The serving simulator (sim.py:_Simulation, no membership events) for every scenario on device.

        traces: one (arrival_s, prompt_tokens, output_tokens) array triple per scenario, sorted by arrival (e.g.
        scenarios.generate_trace).  Each scenario starts idle.  Returns a list of per-scenario dicts with the
        MetricsReport fields (sim.py:190-224, latency mean over completion order with Python's sum(), nearest-
        rank percentiles) plus per-request completion times and the event count.  Needs mode "warp".
        """
        import math
        torch = self.torch
        if self.mode not in ("warp", "blocks"):
            raise ValueError("the simulator runs with mode 'warp' (<= 32 hosts per layer) or 'blocks' (<= 256)")
        if len(traces) != self.S:
            raise ValueError("one trace per scenario")
        if not self.built:
            self.build()
        S, G = self.S, self.G
        n = np.array([len(t[0]) for t in traces], dtype=np.int64)
        ptr = np.concatenate([[0], np.cumsum(n)]).astype(np.int32)
        arr = np.concatenate([np.asarray(t[0], dtype=np.float64) for t in traces]) if n.sum() else np.zeros(1)
        pr = np.concatenate([np.asarray(t[1], dtype=np.int32) for t in traces]) if n.sum() else np.zeros(1, np.int32)
        ou = np.concatenate([np.asarray(t[2], dtype=np.int32) for t in traces]) if n.sum() else np.zeros(1, np.int32)
        if max_live is None:
            max_live = max(1, int(n.max()) if n.size else 1)         # every request live at once, at most
        pow_len = max_live + 2
        pub = np.array([float((1 + o) ** contention) for o in range(pow_len)])
        exe = np.array([float(max(1, o) ** contention) for o in range(pow_len)])
        up = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(device=self.dev, dtype=dt)
        if not hasattr(self, "_tokcap"):
            self._tokcap = torch.from_numpy(np.tile(self.scen.token_cap, S)).to(self.dev)
        total = max(int(n.sum()), 1)
        done_t = torch.full((total,), float("nan"), dtype=torch.float64, device=self.dev)
        done_r = torch.full((total,), -1, dtype=torch.int32, device=self.dev)
        dur = torch.zeros(S, dtype=torch.float64, device=self.dev)
        comp = torch.zeros(S, dtype=torch.int32, device=self.dev)
        peak = torch.zeros(S, dtype=torch.int32, device=self.dev)
        nev = torch.zeros(S, dtype=torch.int64, device=self.dev)
        ptr_d, arr_d, pr_d, ou_d = up(ptr, torch.int32), up(arr, torch.float64), up(pr, torch.int32), up(ou, torch.int32)
        pub_d, exe_d = up(pub, torch.float64), up(exe, torch.float64)
        # per-scenario RTT matrices (scenario_rtt) built on device from the pool matrix and the jitter seeds
        rtt_d = self._scenario_mats()
        fn = N.lib().ss_sim_warp if self.mode == "warp" else N.lib().ss_sim_cta
        N.check(fn(self.dag_set(), N.ptr(self.gpu_ptr), N.ptr(self.base_tau), N.ptr(self._tokcap),
                                    N.ptr(rtt_d), N.ptr(pub_d), N.ptr(exe_d), pow_len, N.ptr(ptr_d), N.ptr(arr_d),
                                    N.ptr(pr_d), N.ptr(ou_d), float(publish_interval), int(amortize_rtt),
                                    int(max_live), N.ptr(done_t), N.ptr(done_r), N.ptr(dur), N.ptr(comp),
                                    N.ptr(peak), N.ptr(nev), N.ptr(self.status), N.ptr(self.aux),
                                    N.stream_handle(self.stream)), "ss_sim_" + self.mode)
        st = self.status.cpu().numpy()
        if (st == 8).any():
            raise ValueError("a scenario had more concurrent chains than the simulator's shared-memory table holds, "
                             "or a chain with more than 32 hops")
        self.raise_first_failure()
        done_t, done_r = done_t.cpu().numpy(), done_r.cpu().numpy()
        dur, comp, peak, nev = dur.cpu().numpy(), comp.cpu().numpy(), peak.cpu().numpy(), nev.cpu().numpy()
        # latencies in completion order per scenario (sim.py:397), vectorised: sort completed requests by
        # (scenario, completion rank); float64 subtraction is the reference's float subtraction
        total_n = int(ptr[-1])
        scen_of = np.repeat(np.arange(S), n)
        lat_all = done_t[:total_n] - arr[:total_n]
        fin = np.nonzero(done_r[:total_n] >= 0)[0]
        fin = fin[np.lexsort((done_r[fin], scen_of[fin]))]
        cut = np.searchsorted(scen_of[fin], np.arange(S + 1))
        lat_sorted = lat_all[fin]
        by_value = lat_sorted.copy()
        for s_ in range(S):                                          # per-scenario ascending copy for percentiles
            by_value[cut[s_]:cut[s_ + 1]].sort()
        reports = []
        for s in range(S):
            a, b = int(ptr[s]), int(ptr[s + 1])
            lat = lat_sorted[cut[s]:cut[s + 1]].tolist()
            mean = p50 = p95 = p99 = 0.0
            if lat:
                mean = sum(lat) / len(lat)                                     # CPython 3.12 sum, as sim.py:457
                srt = by_value[cut[s]:cut[s + 1]]
                rank = lambda q: float(srt[max(1, math.ceil(q * len(lat) / 100.0)) - 1])
                p50, p95, p99 = rank(50), rank(95), rank(99)
            d = float(dur[s])
            reports.append({"submitted": b - a, "completed": int(comp[s]), "unserved": b - a - int(comp[s]),
                            "aborted": 0, "duration_s": d, "throughput_rps": int(comp[s]) / d if d > 0 else 0.0,
                            "latency_mean_s": mean, "latency_p50_s": p50, "latency_p95_s": p95, "latency_p99_s": p99,
                            "queue_peak": int(peak[s]), "latencies": lat, "events": int(nev[s])})
        return reports

    def adopt_state(self, other: "ScenarioReplayer") -> None:
        """Continue another replayer's request stream (same scenarios, pool and window): occupancy, release
        ring and request counters move over, the placement stays this replayer's."""
        if (other.S, other.G, other.L, other.window) != (self.S, self.G, self.L, self.window):
            raise ValueError("adopt_state needs the same scenarios, pool, depth and window")
        self.occ.copy_(other.occ)
        self.ring.copy_(other.ring)
        self.next_req.copy_(other.next_req)

    def abort_on(self, mark) -> np.ndarray:
        """Release the live chains touching the marked GPUs ([S, N] bool); returns aborts per scenario."""
        torch = self.torch
        m = torch.from_numpy(np.ascontiguousarray(np.asarray(mark, dtype=np.uint8).reshape(-1))).to(self.dev)
        n_ab = torch.zeros(self.S, dtype=torch.int32, device=self.dev)
        N.check(N.lib().ss_ring_abort(self.S, self.G, self.L, self.window, N.ptr(m), N.ptr(self.occ),
                                      N.ptr(self.ring), N.ptr(self.next_req), N.ptr(n_ab), None,
                                      N.stream_handle(self.stream)), "ss_ring_abort")
        return n_ab.cpu().numpy()

    def raise_first_failure(self) -> None:
        st = self.status.cpu().numpy()
        bad = np.nonzero(st)[0]
        if bad.size:
            raise_for_status(int(st[bad[0]]), int(self.aux.cpu()[bad[0]]))

    def stream_bytes_per_selection(self) -> float:
        """Slot mode: bytes read from L2/HBM per selection (row/column units of every boundary)."""
        if self.mode not in ("slots", "cluster", "regions"):
            raise ValueError("stream bytes are defined for the slot and region modes")
        meta = self.meta.view(self.S, -1)[:, :16].cpu().numpy().view(np.int32)   # hdr: used, Wp, units, inserts
        return float((meta[:, 2].astype(np.int64) * meta[:, 1] * 8).mean())

    # algorithmic bytes: B2 = 8*sum R_l R_{l+1} + 8*sum R_l + 4*L per selection
    def bytes_per_selection(self) -> np.ndarray:
        cl = self.col_len.view(self.S, self.L).cpu().numpy().astype(np.int64)
        return 8 * (cl[:, :-1] * cl[:, 1:]).sum(axis=1) + 8 * cl.sum(axis=1) + 4 * self.L


# ---------------------------------------------------------------------------
# Phase-1 candidate sweep (C3 / C5): allocate() over many pool variants
# ---------------------------------------------------------------------------

@dataclass
class PackedVariants:
    """Pools of many allocate() calls, already in device order.

    pools[p] = (caps sorted by (-cap, id), flops in that order, L, kmax);
    obj_flops[p] = flops in CLUSTER order, obj_rtt[p] = dense rtt_s matrix in
    cluster order (the objective's inputs); var_ptr[v] = first pool of variant v;
    region names / gpu ids are kept host-side only for plan assembly.
    """

    pools: list
    obj_flops: list
    obj_rtt: list
    var_ptr: np.ndarray
    fpl: float
    layers: int
    tokens: float = 128.0
    alpha: float = 1.0

    @property
    def n_variants(self) -> int:
        return int(self.var_ptr.size - 1)

    @property
    def n_candidates(self) -> int:
        return int(sum(p.kmax for p in self.pools))


class VariantSweep:
    """Device Phase-1 over PackedVariants: stage counts, objective, Z(k), water-fill of
    every candidate's groups (fill_all), best k per region, objective fold per
    variant, global argmax (ties -> lowest variant)."""

    def __init__(self, packed: PackedVariants, *, fill_all: bool = True, stream=None):
        import torch
        from ._phase1 import PoolBatch
        self.torch = torch
        self.packed = packed
        self.fill_all = fill_all
        self.stream = stream
        self.batch = PoolBatch(packed.pools, stream=stream)
        dev = self.batch.dev
        n = np.array([len(f) for f in packed.obj_flops], dtype=np.int64)
        self.item_ptr = torch.from_numpy(np.concatenate([[0], np.cumsum(n)]).astype(np.int32)).to(dev)
        self.mat_off = torch.from_numpy(np.concatenate([[0], np.cumsum(n * n)[:-1]]).astype(np.int64)).to(dev)
        self.obj_flops = torch.from_numpy(np.concatenate(packed.obj_flops).astype(np.float64)).to(dev)
        self.obj_rtt = torch.from_numpy(np.concatenate([m.reshape(-1) for m in packed.obj_rtt])).to(dev)
        self.layers = torch.full((len(packed.pools),), packed.layers, dtype=torch.int32, device=dev)
        self.var_ptr = torch.from_numpy(packed.var_ptr.astype(np.int32)).to(dev)
        V = packed.n_variants
        self.t = torch.empty(len(packed.pools), dtype=torch.float64, device=dev)
        self.r = torch.empty(len(packed.pools), dtype=torch.float64, device=dev)
        self.total = torch.empty(V, dtype=torch.float64, device=dev)
        self.feasible = torch.empty(V, dtype=torch.int32, device=dev)
        self.best_variant = torch.empty(1, dtype=torch.int32, device=dev)
        self.best_total = torch.empty(1, dtype=torch.float64, device=dev)
        km = max(int(self.batch.km.max()), 1)
        self.kpow = np.array([0.0] + [float(k ** packed.alpha) for k in range(1, km + 1)])

    def run(self) -> None:
        lib = N.lib()
        st = N.stream_handle(self.stream)
        b = self.batch
        b.stage_counts()
        N.check(lib.ss_objective(len(self.packed.pools), N.ptr(self.item_ptr), N.ptr(self.obj_flops),
                                 N.ptr(self.mat_off), N.ptr(self.obj_rtt), float(self.packed.fpl), N.ptr(self.layers),
                                 float(self.packed.tokens), N.ptr(self.t), N.ptr(self.r), st), "ss_objective")
        b.score_and_best(self.t, self.r, self.kpow, fill_all=self.fill_all)
        N.check(lib.ss_variant_reduce(self.packed.n_variants, N.ptr(self.var_ptr), N.ptr(b.koff), N.ptr(b.best_k),
                                      N.ptr(b.z), N.ptr(b.status), N.ptr(self.total), N.ptr(self.feasible),
                                      N.ptr(self.best_variant), N.ptr(self.best_total), st), "ss_variant_reduce")
