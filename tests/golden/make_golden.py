#!/usr/bin/env python3
"""Generate golden fixtures by running the UNMODIFIED reference (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference is read from /root/reference (never copied); it does not exist on
the GPU box, so the outputs are committed as small JSON files next to this
script.  Floats are stored as ``float.hex`` strings so comparisons are
bit-exact; ints stay ints; a value that the reference produced as a Python int
where a float could also appear is tagged ``["i", v]`` vs ``["f", hex]``.

Fixtures
  router_cases.json    select_chain on random DAGs (test_router.py:136-172 and
                       test_acceptance.py:112-158 generators, larger sizes too),
                       UncoveredLayer / NoPath cases
  router_replays.json  ChainRouter.route/release op scripts on bench pools:
                       C1 (L32/N8, W=inf), C1 tie pool (flops=1e14), C2 prefix
                       (L64/N64, W=64), bench round trips (W=0), the
                       routing_feedback demo map, C4-mini churn+jitter scenarios
  phase1_cases.json    solve_stage_counts (exact + constructive), allocate on
                       bench/desk/random pools, estimate_objective_params,
                       solve_lambda / hamilton_round / rebalance_pipeline
"""

from __future__ import annotations

import json
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, REPO)

import swarmsched as ref                                    # noqa: E402
from swarmsched import allocator as ref_alloc               # noqa: E402
from swarmsched import waterfill as ref_wf                  # noqa: E402
from swarmsched.membership import MembershipManager          # noqa: E402

from paper_2509_26182_b200 import scenarios as scen          # noqa: E402  (generator only)


def fx(v: float) -> str:
    return float(v).hex()


def tag(v):
    return ["i", v] if isinstance(v, int) else ["f", fx(v)]


def dump(name, obj):
    path = os.path.join(HERE, name)
    with open(path, "w") as fh:
        json.dump(obj, fh, separators=(",", ":"), sort_keys=True)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def ref_cluster(n, seed, L, *, flops=None, rc=None):
    """The reference's own synthetic_cluster, optionally homogenised."""
    model = ref.ModelSpec(f"bench-{L}l", L, 1.2e9, 2.8e10)
    cluster, model = ref.synthetic_cluster(n, seed=seed, region_count=rc, model=model)
    if flops is not None:
        gpus = tuple(ref.GpuNode(g.id, g.region, g.vram_bytes, flops, g.reserve_fraction,
                                 g.ram_token_capacity) for g in cluster.gpus)
        cluster = ref.ClusterSnapshot(gpus=gpus, links=dict(cluster.links))
    return cluster, model


def chain_json(chain, ids_pos):
    return {"hops": [[ids_pos[h.gpu_id], h.start_layer, h.end_layer] for h in chain.hops],
            "cost": fx(chain.cost_s)}


# ---------------------------------------------------------------------------
# Phase-2
# ---------------------------------------------------------------------------

def random_router_case(rng, n_gpu, n_layer, p_link, p_rtt_lo, p_rtt_hi, tau_lo, tau_hi):
    gpus = [f"g{i}" for i in range(n_gpu)]
    hosting, cols = {}, []
    for layer in range(1, n_layer + 1):
        col = rng.sample(gpus, rng.randint(1, n_gpu))
        cols.append(sorted(col))
        for g in col:
            hosting[(g, layer)] = rng.uniform(tau_lo, tau_hi)
    spine = [rng.choice(c) for c in cols]
    rtts = {}
    for a, b in zip(spine, spine[1:]):
        if a != b:
            rtts[(a, b)] = rng.uniform(p_rtt_lo, p_rtt_hi)
    for a in gpus:
        for b in gpus:
            if a != b and rng.random() < p_link and (a, b) not in rtts:
                rtts[(a, b)] = rng.uniform(p_rtt_lo, p_rtt_hi)
    return gpus, hosting, rtts


def run_select(hosting, rtts, L, exclude=()):
    pm = ref.PerfMap(ttl_s=1e9)
    names = {g for g, _ in hosting} | {g for p in rtts for g in p}
    for g in sorted(names):
        pm.register_gpu(g)
    for (g, l), v in hosting.items():
        pm.publish_layer_latency(g, l, v, now=0.0)
    if rtts:
        pm.publish_link_rtts(rtts, now=0.0)
    snap = pm.snapshot(0.0)
    case = {"L": L,
            "hosting": [[g, l, fx(v)] for (g, l), v in sorted(hosting.items())],
            "rtts": [[a, b, fx(v)] for (a, b), v in sorted(rtts.items())],
            "exclude": sorted(exclude)}
    try:
        dag = ref.build_dag(snap, L, exclude=frozenset(exclude))
        chain = ref.select_chain(dag, snap)
        case["result"] = {"status": "ok", "hops": [[h.gpu_id, h.start_layer, h.end_layer] for h in chain.hops],
                          "cost": fx(chain.cost_s), "edges": ref.count_dag_edges(dag, snap)}
    except ref.UncoveredLayer as exc:
        case["result"] = {"status": "uncovered", "layer": exc.layer}
    except ref.NoPath:
        case["result"] = {"status": "no_path"}
    return case


def router_cases():
    cases = []
    rng = random.Random(5001)                      # test_router.py:136-172 shape
    for _ in range(300):
        _, h, r = random_router_case(rng, rng.randint(1, 4), rng.randint(1, 6), 0.4, 0.001, 0.05, 0.001, 0.2)
        cases.append(run_select(h, r, max(l for _, l in h)))
    rng = random.Random(90003)                     # test_acceptance.py:112-158 shape
    for _ in range(200):
        _, h, r = random_router_case(rng, rng.randint(1, 4), rng.randint(1, 6), 0.8, 0.0005, 0.05, 0.0005, 0.25)
        cases.append(run_select(h, r, max(l for _, l in h)))
    rng = random.Random(777)                       # wider DAGs: many hosts, deep
    for _ in range(60):
        n = rng.randint(5, 40)
        _, h, r = random_router_case(rng, n, rng.randint(2, 24), 0.7, 0.0005, 0.02, 0.0005, 0.05)
        cases.append(run_select(h, r, max(l for _, l in h)))
    rng = random.Random(778)                       # tie-heavy: quantised values
    for _ in range(120):
        n = rng.randint(2, 12)
        gpus = [f"t{i:02d}" for i in range(n)]
        L = rng.randint(2, 10)
        h = {}
        for l in range(1, L + 1):
            for g in rng.sample(gpus, rng.randint(1, n)):
                h[(g, l)] = rng.choice([0.25, 0.5, 0.75, 1.0])
        r = {(a, b): rng.choice([0.125, 0.25, 0.5]) for a in gpus for b in gpus if a < b and rng.random() < 0.9}
        cases.append(run_select(h, r, L))
    rng = random.Random(779)                       # exclusion + uncovered / no-path edge cases
    for _ in range(40):
        _, h, r = random_router_case(rng, rng.randint(2, 6), rng.randint(2, 8), 0.3, 0.001, 0.05, 0.001, 0.2)
        L = max(l for _, l in h)
        hosts = sorted({g for g, _ in h})
        ex = rng.sample(hosts, min(len(hosts), rng.randint(0, 2)))
        cases.append(run_select(h, r, L + rng.randint(0, 1), ex))
    cases.append(run_select({("a", 1): 1.0, ("b", 2): 1.0}, {}, 2))                       # no path
    cases.append(run_select({("a", 1): 0.1, ("a", 3): 0.1}, {}, 3))                       # uncovered 2
    cases.append(run_select({("a", 1): 1.0, ("b", 1): 1.0, ("c", 2): 1.0},
                            {("a", "c"): 2.0, ("b", "c"): 2.0}, 2))                       # tie -> a
    cases.append(run_select({("a", 1): 2.0, ("a", 2): 9.0, ("b", 1): 5.0, ("b", 2): 3.0},
                            {("a", "b"): 1.0}, 2))
    cases.append(run_select({("a", 1): 1.0, ("a", 2): 1.0, ("b", 2): 0.5}, {("a", "b"): 10.0}, 2))
    cases.append(run_select({("a", 1): 0.1, ("b", 1): 0.1}, {("a", "b"): 0.004, ("b", "a"): 0.009}, 1))
    cases.append(run_select({("a", 1): 0.1, ("b", 2): 0.1, ("a", 2): 0.3},
                            {("a", "b"): 0.004, ("b", "a"): 0.009}, 2))
    return cases


def replay_record(cluster, model, plan, n_routes, window, *, leave=(), name=""):
    pm = ref.PerfMap(ttl_s=4.5)
    mgr = MembershipManager(cluster, model, pm)
    base = {g.id: model.flops_per_layer_per_token / g.flops for g in cluster.gpus}
    pm.latency_fn = lambda gpu_id, layer, occ: base[gpu_id] * (1 + occ)
    mgr.initialize(plan, 0.0)
    for g in leave:
        mgr.on_leave(g, 0.0)
    router = ref.ChainRouter(pm, model.layer_count)
    ids = sorted(g.id for g in cluster.gpus)
    pos = {g: i for i, g in enumerate(ids)}
    live, out = [], []
    t0 = time.perf_counter()
    for i in range(n_routes):
        if window is not None and window > 0 and i >= window:
            router.release(live.pop(0), 0.0)
        chain = router.route(0.0)
        if window == 0:
            router.release(chain, 0.0)
        elif window is not None:
            live.append(chain)
        out.append(chain_json(chain, pos))
    dt = time.perf_counter() - t0
    occ = [pm.occupancy(g) for g in ids]
    print(f"  replay {name}: {n_routes} routes in {dt:.2f}s")
    return {"routes": out, "final_occ": occ, "window": window, "leave": sorted(pos[g] for g in leave)}


def plan_json(plan):
    d = ref.plan_to_dict(plan)
    d["objective"] = fx(d["objective"])
    for row in d["per_k"]:
        row["z"] = fx(row["z"])
    return d


def router_replays():
    out = {}
    # C1: L32/N8 seed 0, accumulate (cli route semantics)
    cl, m = ref_cluster(8, 0, 32)
    plan = ref.allocate(cl, m)
    out["c1"] = {"n": 8, "seed": 0, "L": 32, "plan": plan_json(plan),
                 **replay_record(cl, m, plan, 1000, None, name="c1")}
    # C1 tie pool
    cl, m = ref_cluster(8, 0, 32, flops=1e14)
    plan = ref.allocate(cl, m)
    out["c1_tie"] = {"n": 8, "seed": 0, "L": 32, "flops": fx(1e14), "plan": plan_json(plan),
                     **replay_record(cl, m, plan, 300, None, name="c1_tie")}
    # tie pool, larger, windowed
    cl, m = ref_cluster(32, 3, 24, flops=1e14)
    plan = ref.allocate(cl, m)
    out["n32_tie"] = {"n": 32, "seed": 3, "L": 24, "flops": fx(1e14), "plan": plan_json(plan),
                      **replay_record(cl, m, plan, 200, 16, name="n32_tie")}
    # bench round trips (W = 0)
    cl, m = ref_cluster(16, 16, 48)
    plan = ref.allocate(cl, m)
    out["rt16"] = {"n": 16, "seed": 16, "L": 48, "plan": plan_json(plan),
                   **replay_record(cl, m, plan, 20, 0, name="rt16")}
    # C2 prefix: L64/N64 seed 0, W=64
    cl, m = ref_cluster(64, 0, 64)
    plan = ref.allocate(cl, m)
    out["c2"] = {"n": 64, "seed": 0, "L": 64, "plan": plan_json(plan),
                 **replay_record(cl, m, plan, 300, 64, name="c2")}
    # C4-mini: L64/N256 seed 0 base plan, 2 churn+jitter scenarios, W=64
    cl, m = ref_cluster(256, 0, 64)
    plan = ref.allocate(cl, m)
    out["c4_plan"] = plan_json(plan)
    ids = sorted(g.id for g in cl.gpus)
    pos = {g: i for i, g in enumerate(ids)}
    slices = {pos[g]: (s.start_layer, s.end_layer) for g, s in plan.gpu_slices().items()}
    for s in (11, 12):
        leave_idx = scen.churn_set(s, sorted(slices), slices, 64, 0.05)
        jit = scen.jitter_factor_matrix(s, len(ids))
        links = {}
        for i in range(len(ids)):
            for j in range(i + 1, len(ids)):
                links[(ids[i], ids[j])] = cl.rtt_s(ids[i], ids[j]) * jit[i, j]
        clj = ref.ClusterSnapshot(gpus=cl.gpus, links=links)
        rec = replay_record(clj, m, plan, 120, 64, leave=[ids[g] for g in leave_idx], name=f"c4_s{s}")
        out[f"c4_s{s}"] = {"n": 256, "seed": 0, "L": 64, "scenario_seed": s, **rec}
    # routing_feedback demo map (pkg/demos/routing_feedback.py:17-65)
    pm = ref.PerfMap(ttl_s=60.0, latency_fn=lambda g, l, o: 0.002 * (1 + o))
    hosting = {"a-front": range(1, 4), "a-back": range(4, 7), "b-front": range(1, 4), "b-back": range(4, 7)}
    for g, hosted in hosting.items():
        pm.register_gpu(g)
        for l in hosted:
            pm.publish_layer_latency(g, l, 0.002, now=0.0)
    pm.publish_link_rtts({("a-front", "a-back"): 0.001, ("b-front", "b-back"): 0.001,
                          ("a-front", "b-back"): 0.008, ("b-front", "a-back"): 0.008}, now=0.0)
    router = ref.ChainRouter(pm, 6)
    chains = [router.route(now=0.1 * i) for i in range(6)]
    out["demo_feedback"] = {"routes": [{"hops": [[h.gpu_id, h.start_layer, h.end_layer] for h in c.hops],
                                        "cost": fx(c.cost_s)} for c in chains],
                            "occ": {g: pm.occupancy(g) for g in hosting}}
    return out


# ---------------------------------------------------------------------------
# Phase-1
# ---------------------------------------------------------------------------

def sc_json(sols):
    return {str(k): [s.stages, [list(g) for g in s.groups]] for k, s in sorted(sols.items())}


def phase1_cases():
    out = {"stage_counts": [], "allocate": [], "objective": [], "waterfill": [], "rebalance": []}
    rng = random.Random(3001)
    for _ in range(250):                                     # exact path, small
        n, L = rng.randint(1, 7), rng.randint(1, 12)
        caps = sorted((rng.randint(0, L) for _ in range(n)), reverse=True)
        km = max(ref.k_max(caps, L), 1)
        out["stage_counts"].append({"caps": caps, "L": L, "kmax": km,
                                    "sols": sc_json(ref.solve_stage_counts(caps, L, km))})
    rng = random.Random(3011)
    for _ in range(40):                                      # exact path, up to the limit
        n, L = rng.randint(8, 16), rng.randint(8, 48)
        caps = sorted((rng.randint(1, 32) for _ in range(n)), reverse=True)
        km = ref.k_max(caps, L)
        if km < 1:
            continue
        out["stage_counts"].append({"caps": caps, "L": L, "kmax": km,
                                    "sols": sc_json(ref.solve_stage_counts(caps, L, km))})
    rng = random.Random(3012)
    for _ in range(60):                                      # constructive path
        n = rng.choice([17, 18, 20, 24, 25, 32, 48, 64])
        L = rng.choice([8, 12, 24, 48, 64, 80])
        caps = sorted((rng.randint(1, min(32, L)) for _ in range(n)), reverse=True)
        km = ref.k_max(caps, L)
        if km < 1:
            continue
        out["stage_counts"].append({"caps": caps, "L": L, "kmax": km,
                                    "sols": sc_json(ref.solve_stage_counts(caps, L, km))})
    caps = [32] * 32 + [16] * 32                             # test_allocator.py:154-165
    out["stage_counts"].append({"caps": caps, "L": 48, "kmax": ref.k_max(caps, 48),
                                "sols": sc_json(ref.solve_stage_counts(caps, 48, ref.k_max(caps, 48)))})

    def alloc_case(name, cl, m, **kw):
        rec = {"name": name, "L": m.layer_count, "bpl": fx(m.bytes_per_layer),
               "fpl": fx(m.flops_per_layer_per_token),
               "gpus": [[g.id, g.region, fx(g.vram_bytes), fx(g.flops), fx(g.reserve_fraction)] for g in cl.gpus],
               "links": [[a, b, fx(v)] for (a, b), v in sorted(cl.links.items())],
               "default_rtt": fx(cl.default_cross_region_rtt_s), "kw": {}}
        if "params" in kw:
            p = kw["params"]
            rec["kw"]["params"] = [fx(p.alpha), fx(p.t_comp_seconds), fx(p.rtt_seconds)]
        if "alpha" in kw:
            rec["kw"]["alpha"] = fx(kw["alpha"])
        try:
            rec["plan"] = plan_json(ref.allocate(cl, m, **kw))
        except ref.NoFeasiblePipeline:
            rec["plan"] = None
        out["allocate"].append(rec)

    for (n, seed, L) in [(8, 0, 32), (64, 0, 64), (256, 0, 80), (256, 0, 64), (16, 16, 48), (32, 5, 48),
                         (128, 1, 80)]:
        cl, m = ref_cluster(n, seed, L)
        alloc_case(f"bench_n{n}_s{seed}_L{L}", cl, m)
    cl, m = ref_cluster(64, 2, 64, flops=1e14)
    alloc_case("tie_n64", cl, m)
    # jittered links: exercises the compensated-sum path of the objective
    cl, m = ref_cluster(96, 4, 48)
    ids = sorted(g.id for g in cl.gpus)
    jit = scen.jitter_factor_matrix(4, len(ids))
    links = {(ids[i], ids[j]): cl.rtt_s(ids[i], ids[j]) * jit[i, j]
             for i in range(len(ids)) for j in range(i + 1, len(ids))}
    alloc_case("jitter_n96", ref.ClusterSnapshot(gpus=cl.gpus, links=links), m)
    sys.path.insert(0, "/root/reference/pkg/tests")
    from helpers import DESK_MODEL, TEST_MODEL, desk_cluster, gpu_with_capacity, linked_cluster  # noqa: E402

    alloc_case("desk", desk_cluster(), DESK_MODEL)
    gpus = [gpu_with_capacity(n, c) for n, c in (("a1", 6), ("a2", 5), ("a3", 5), ("a4", 4))]
    alloc_case("desk_example", linked_cluster(gpus), TEST_MODEL)
    gpus = [gpu_with_capacity("big", 10)] + [gpu_with_capacity(f"s{i}", 2) for i in range(5)]
    alloc_case("equal_scores", linked_cluster(gpus), TEST_MODEL,
               params=ref_alloc.ObjectiveParams(alpha=1.0, t_comp_seconds=0.5, rtt_seconds=0.5))
    gpus = [gpu_with_capacity("fast", 6, flops=3.0e14), gpu_with_capacity("slow", 6, flops=1.0e14)]
    alloc_case("fast_slow", linked_cluster(gpus), ref.ModelSpec("m8", 8, 1.0e9, 2.0e10))
    gpus = [gpu_with_capacity("a", 3), gpu_with_capacity("b", 3)]
    alloc_case("infeasible", linked_cluster(gpus), TEST_MODEL)
    rng = random.Random(3005)                               # test_allocator.py:315-343 shape
    for case in range(120):
        n, L = rng.randint(1, 6), rng.randint(2, 12)
        model = ref.ModelSpec("m", L, 1.0e9, 2.0e10)
        gpus = [gpu_with_capacity(f"g{i}", rng.randint(0, L), region=rng.choice(["east", "west"]),
                                  flops=rng.uniform(5e13, 3e14), model=model) for i in range(n)]
        alloc_case(f"rand{case}", linked_cluster(gpus), model, alpha=rng.choice([1.0, 0.5, 1.5]))
    rng = random.Random(3007)
    gpus = [gpu_with_capacity(f"g{i:02d}", rng.randint(2, 8), flops=rng.uniform(5e13, 2e14)) for i in range(40)]
    alloc_case("large_region_40", linked_cluster(gpus), TEST_MODEL)

    # estimate_objective_params on bench regions (+ jittered)
    for (n, seed, L) in [(64, 0, 64), (256, 0, 80), (96, 4, 48)]:
        cl, m = ref_cluster(n, seed, L)
        for region in sorted(cl.regions):
            rg = cl.gpus_in_region(region)
            p = ref_alloc.estimate_objective_params(rg, cl, m, 1.0, 128.0)
            out["objective"].append({"n": n, "seed": seed, "L": L, "region": region,
                                     "t_comp": fx(p.t_comp_seconds), "rtt": fx(p.rtt_seconds)})

    # water-fill primitives (test_waterfill.py generators + bench-scale flops)
    rng = random.Random(2002)
    for case in range(400):
        n, L = rng.randint(1, 6), rng.randint(1, 24)
        caps = [rng.randint(0, L) for _ in range(n)]
        if sum(caps) < L:
            caps[rng.randrange(n)] += L - sum(caps)
        flops = [rng.uniform(0.1, 10.0) if case % 2 else rng.uniform(6e13, 2.4e14) for _ in range(n)]
        frac = ref_wf.solve_lambda(flops, caps, L)
        layers = ref_wf.hamilton_round(frac, caps, total=L).layers
        out["waterfill"].append({"flops": [fx(f) for f in flops], "caps": caps, "L": L,
                                 "targets": [tag(t) for t in frac.targets], "level": fx(frac.water_level),
                                 "layers": list(layers)})
    rng = random.Random(2005)
    for case in range(300):
        n = rng.randint(1, 6)
        L = rng.randint(n, 40)
        caps = [rng.randint(1, L) for _ in range(n)]
        if sum(caps) < L:
            caps[rng.randrange(n)] += L - sum(caps)
        model = ref.ModelSpec("m", L, 1.0e9, 2.0e10)
        gpus = [gpu_with_capacity(f"g{i}", caps[i], flops=rng.uniform(5e13, 3e14) if case % 3 else
                                  rng.choice([1e12, 5e14]), model=model) for i in range(n)]
        stages = []
        cur = 1
        for g in gpus[:-1]:
            stages.append(ref.LayerSlice(g.id, cur, cur))
            cur += 1
        stages.append(ref.LayerSlice(gpus[-1].id, cur, L))
        pipe = ref.Pipeline(stages=tuple(stages), region="east")
        try:
            res = ref_wf.rebalance_pipeline(pipe, {g.id: g for g in gpus}, model)
            lens = [s.length for s in res.stages]
        except (ref.RoundingOverflow, ref.InfeasibleCapacity) as exc:
            lens = type(exc).__name__
        out["rebalance"].append({"flops": [fx(g.flops) for g in gpus], "caps": caps, "L": L, "lengths": lens})
    return out


if __name__ == "__main__":
    t = time.time()
    dump("router_cases.json", router_cases())
    dump("router_replays.json", router_replays())
    dump("phase1_cases.json", phase1_cases())
    print(f"done in {time.time() - t:.1f}s")
