"""CPU baseline of the UNMODIFIED reference -- TEST / BENCH INFRASTRUCTURE ONLY (see oracle/__init__.py).

Times the reference package itself (``swarmsched`` from ``/root/reference/pkg``, installed unmodified into the
git-ignored ``baseline/_ref`` with ``pip install --no-index --no-deps --target baseline/_ref``; that directory
travels to the GPU box with the snapshot) on the host cores, as BASELINE.md section 3 prescribes:

* Phase-2: per C4 scenario, the reference's own ``MembershipManager.initialize`` + ``on_leave`` of the scenario's
  churn set on a jittered explicit link table (set-up, not timed), then the op script of
  ``ChainRouter.route`` / ``ChainRouter.release`` (router.py:247-260) with window W: only that loop is inside
  ``perf_counter``.
* Phase-1: per C3 pool, the reference's ``solve_stage_counts`` + ``score`` + ``rebalance_pipeline`` of every k's
  groups' draft pipelines (allocator.py:473-504, 104-111, 597-606; waterfill.py:142-183) -- the per-candidate
  section, timed alone (``estimate_objective_params`` is per region, outside the timer).

Jobs run on ``multiprocessing`` fork pools (one process per host core); the pool start-up and the set-up are
outside the timers.  The aggregate rate is sum(selections) / sum(job seconds) x processes, i.e. the per-process
rate measured while every process is busy, times the number of processes.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

REF_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


def available() -> bool:
    return os.path.isdir(os.path.join(REF_DIR, "swarmsched"))


def _ref():
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import swarmsched
    if not os.path.abspath(swarmsched.__file__).startswith(REF_DIR):
        raise RuntimeError(f"swarmsched imported from {swarmsched.__file__}, not {REF_DIR}")
    return swarmsched


def _to_ref(ref, cl, model, links=None):
    gpus = tuple(ref.GpuNode(g.id, g.region, g.vram_bytes, g.flops, g.reserve_fraction, g.ram_token_capacity)
                 for g in cl.gpus)
    rcl = ref.ClusterSnapshot(gpus=gpus, links=dict(cl.links) if links is None else links,
                              default_cross_region_rtt_s=cl.default_cross_region_rtt_s)
    rm = ref.ModelSpec(model.name, model.layer_count, model.bytes_per_layer, model.flops_per_layer_per_token)
    return rcl, rm


# ---------------------------------------------------------------------------
# Phase-2: ChainRouter.route / release
# ---------------------------------------------------------------------------

_P2 = {}


def _p2_init(n_gpus, seed, layers):
    """Fork-time state shared by the workers: the base pool and the reference plan (computed once)."""
    if _P2.get("key") == (n_gpus, seed, layers):
        return
    from paper_2509_26182_b200 import scenarios as scen
    ref = _ref()
    cl, model = scen.synthetic_cluster(n_gpus, seed=seed, model=scen.bench_model(layers))
    rcl, rm = _to_ref(ref, cl, model)
    plan = ref.allocate(rcl, rm)
    _P2.update(ref=ref, cl=rcl, model=rm, plan=plan, key=(n_gpus, seed, layers))


def _route_job(args):
    s, n_req, window, churn = args
    from paper_2509_26182_b200 import scenarios as scen
    from swarmsched.membership import MembershipManager
    ref, cl, model, plan = _P2["ref"], _P2["cl"], _P2["model"], _P2["plan"]
    ids = sorted(g.id for g in cl.gpus)
    pos = {g: i for i, g in enumerate(ids)}
    slices = {pos[g]: (sl.start_layer, sl.end_layer) for g, sl in plan.gpu_slices().items()}
    leave = scen.churn_set(s, sorted(slices), slices, model.layer_count, churn) if churn > 0 else []
    jit = scen.jitter_factor_matrix(s, len(ids))
    links = {(ids[i], ids[j]): cl.rtt_s(ids[i], ids[j]) * jit[i, j]
             for i in range(len(ids)) for j in range(i + 1, len(ids))}
    clj = ref.ClusterSnapshot(gpus=cl.gpus, links=links)
    pm = ref.PerfMap(ttl_s=4.5)
    mgr = MembershipManager(clj, model, pm)
    base = {g.id: model.flops_per_layer_per_token / g.flops for g in clj.gpus}
    pm.latency_fn = lambda gpu_id, layer, occ: base[gpu_id] * (1 + occ)          # bench.py:150-151
    mgr.initialize(plan, 0.0)
    for g in leave:
        mgr.on_leave(ids[g], 0.0)
    router = ref.ChainRouter(pm, model.layer_count)
    live = []
    h = 0
    t0 = time.perf_counter()
    for i in range(n_req):
        if window > 0 and i >= window:
            router.release(live.pop(0), 0.0)
        chain = router.route(0.0)
        live.append(chain)
        h ^= hash((chain.cost_s, len(chain.hops)))
    return time.perf_counter() - t0, n_req, h


def phase2_rate(seeds, n_req, window, *, n_gpus=256, seed=0, layers=64, churn=0.05, cores=None):
    """Reference ChainRouter selections/s over C4 scenario states (one job per scenario seed)."""
    cores = cores or len(os.sched_getaffinity(0))
    _p2_init(n_gpus, seed, layers)
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(abs, range(cores))                       # workers up before any timing
        t0 = time.perf_counter()
        res = pool.map(_route_job, [(int(s), n_req, window, churn) for s in seeds], chunksize=1)
        wall = time.perf_counter() - t0
    busy = sum(r[0] for r in res)
    sel = sum(r[1] for r in res)
    procs = min(cores, len(seeds))
    return {"value": sel / busy * procs, "per_core": sel / busy, "cores": procs, "selections": sel,
            "route_seconds": busy, "wall_seconds": wall, "k": _P2["plan"].replication_count}


# ---------------------------------------------------------------------------
# Phase-1: solve_stage_counts + score + rebalance_pipeline per (region, k)
# ---------------------------------------------------------------------------

def _cand_job(args):
    v, layers = args
    from paper_2509_26182_b200 import scenarios as scen
    ref = _ref()
    from swarmsched import allocator as ra
    from swarmsched import waterfill as rw
    cl, model = scen.synthetic_cluster(256, seed=v, model=scen.bench_model(layers))
    rcl, rm = _to_ref(ref, cl, model)
    pools = []
    for region in sorted(rcl.regions):
        rg = rcl.gpus_in_region(region)
        caps = [ref.layer_capacity(g, rm) for g in rg]
        order = sorted(range(len(rg)), key=lambda i: (-caps[i], rg[i].id))
        caps_o = [caps[i] for i in order]
        km = ra.k_max(caps_o, layers)
        if km < 1:
            continue
        params = ra.estimate_objective_params(rg, rcl, rm, 1.0, 128.0)
        pools.append(([rg[i] for i in order], caps_o, km, params))
    t0 = time.perf_counter()
    cand = 0
    for gpus, caps, km, params in pools:
        gpu_map = {g.id: g for g in gpus}
        sols = ra.solve_stage_counts(caps, layers, km)
        for k, sol in sols.items():
            ra.score(k, sol.stages, params)
            for grp in sol.groups:                         # the draft pipeline of allocator.py:597-606
                cursor, stages = 1, []
                for i in grp:
                    span = min(caps[i], layers - cursor + 1)
                    stages.append(ref.LayerSlice(gpus[i].id, cursor, cursor + span - 1))
                    cursor += span
                rw.rebalance_pipeline(ref.Pipeline(stages=tuple(stages), region=gpus[0].region), gpu_map, rm)
            cand += 1
    return time.perf_counter() - t0, cand


def phase1_rate(variants, layers=80, cores=None):
    """Reference per-candidate Phase-1 evaluations/s over C3 variants (synthetic_cluster(256, seed=v))."""
    cores = cores or len(os.sched_getaffinity(0))
    ctx = mp.get_context("fork")
    with ctx.Pool(cores) as pool:
        pool.map(abs, range(cores))
        t0 = time.perf_counter()
        res = pool.map(_cand_job, [(int(v), layers) for v in variants], chunksize=1)
        wall = time.perf_counter() - t0
    busy = sum(r[0] for r in res)
    cand = sum(r[1] for r in res)
    procs = min(cores, len(variants))
    return {"value": cand / busy * procs, "per_core": cand / busy, "cores": procs, "candidates": cand,
            "eval_seconds": busy, "wall_seconds": wall}
