"""Phase-1 parity on a B200: CUDA allocator / water-fill vs reference golden vectors and the oracle.

Bar: bit-exact integer outputs (stage counts, groups, layer counts, chosen k)
and bit-exact fp64 objective values (the reference's CPython arithmetic is
replayed operation by operation, including 3.12's compensated sum()).
"""

import random

import numpy as np
import pytest

from conftest import hx, untag
from helpers_golden import cluster_from_alloc_case
from oracle import alloc_ref, waterfill_ref

pytestmark = pytest.mark.gpu


def _plan_hex(plan):
    from paper_2509_26182_b200.plan import plan_to_dict
    d = plan_to_dict(plan)
    d["objective"] = d["objective"].hex()
    for row in d["per_k"]:
        row["z"] = row["z"].hex()
    return d


def test_stage_counts_golden(cuda_ready, phase1_cases):
    from paper_2509_26182_b200 import solve_stage_counts
    for i, case in enumerate(phase1_cases["stage_counts"]):
        got = solve_stage_counts(case["caps"], case["L"], case["kmax"])
        want = {int(k): (v[0], tuple(tuple(g) for g in v[1])) for k, v in case["sols"].items()}
        assert {k: (s.stages, s.groups) for k, s in got.items()} == want, (i, case["caps"], case["L"])


def test_stage_counts_random_vs_oracle(cuda_ready):
    """Exact path at the 16-GPU limit and constructive pools up to 128 GPUs, L up to 80."""
    from paper_2509_26182_b200._phase1 import PoolBatch, PoolSpec
    rng = random.Random(6001)
    specs, cases = [], []
    for _ in range(120):
        n = rng.choice([3, 8, 12, 16, 17, 24, 40, 64, 96, 128])
        L = rng.choice([6, 16, 32, 48, 64, 80])
        caps = sorted((rng.randint(0 if rng.random() < 0.1 else 1, min(32, L)) for _ in range(n)), reverse=True)
        km = alloc_ref.kmax(caps, L)
        if km < 1 or (sum(c > 0 for c in caps) <= 16 and L > 64 and n > 14):
            continue
        specs.append(PoolSpec(caps, [1.0] * n, L, km))
        cases.append((caps, L, km))
    batch = PoolBatch(specs)
    batch.stage_counts()
    res = batch.fetch()
    for p, (caps, L, km) in enumerate(cases):
        res.raise_pool(p)
        assert res.solutions(p) == alloc_ref.stage_counts(caps, L, km), (caps, L, km)


def test_allocate_golden(cuda_ready, phase1_cases):
    from paper_2509_26182_b200 import NoFeasiblePipeline, ObjectiveParams, allocate
    for rec in phase1_cases["allocate"]:
        cluster, model = cluster_from_alloc_case(rec)
        kw = {}
        if "alpha" in rec["kw"]:
            kw["alpha"] = hx(rec["kw"]["alpha"])
        if "params" in rec["kw"]:
            a, t, r = (hx(x) for x in rec["kw"]["params"])
            kw["params"] = ObjectiveParams(alpha=a, t_comp_seconds=t, rtt_seconds=r)
        try:
            got = _plan_hex(allocate(cluster, model, **kw))
        except NoFeasiblePipeline:
            got = None
        assert got == rec["plan"], rec["name"]


def test_objective_golden(cuda_ready, phase1_cases):
    from paper_2509_26182_b200 import estimate_objective_params, scenarios as scen
    for rec in phase1_cases["objective"]:
        cl, m = scen.synthetic_cluster(rec["n"], seed=rec["seed"], model=scen.bench_model(rec["L"]))
        p = estimate_objective_params(cl.gpus_in_region(rec["region"]), cl, m, 1.0, 128.0)
        assert (p.t_comp_seconds.hex(), p.rtt_seconds.hex()) == (rec["t_comp"], rec["rtt"])


def test_waterfill_golden(cuda_ready, phase1_cases):
    from paper_2509_26182_b200 import hamilton_round, solve_lambda
    for i, rec in enumerate(phase1_cases["waterfill"][:120]):
        flops = [hx(f) for f in rec["flops"]]
        frac = solve_lambda(flops, rec["caps"], rec["L"])
        want = [untag(t) for t in rec["targets"]]
        assert list(frac.targets) == want and [type(t) for t in frac.targets] == [type(t) for t in want], i
        assert frac.water_level == hx(rec["level"]), i
        assert list(hamilton_round(frac, rec["caps"], rec["L"]).layers) == rec["layers"], i
        assert list(hamilton_round(frac, rec["caps"]).layers) == list(
            waterfill_ref.largest_remainder(frac.targets, rec["caps"])), i


def test_waterfill_golden_all_batched(cuda_ready, phase1_cases):
    """All 400 golden solve_lambda + hamilton_round cases (total = L and total = None) in batched launches."""
    import torch
    from paper_2509_26182_b200 import _native as N
    recs = phase1_cases["waterfill"]
    sizes = [len(r["caps"]) for r in recs]
    ptr = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    dev = torch.device("cuda")
    n = int(ptr[-1])
    fl = torch.tensor([hx(f) for r in recs for f in r["flops"]], dtype=torch.float64, device=dev)
    caps = torch.tensor([c for r in recs for c in r["caps"]], dtype=torch.int32, device=dev)
    layers = torch.tensor([r["L"] for r in recs], dtype=torch.int32, device=dev)
    gp = torch.from_numpy(ptr).to(dev)
    targets = torch.zeros(n, dtype=torch.float64, device=dev)
    tflag = torch.zeros(n, dtype=torch.int32, device=dev)
    level = torch.zeros(len(recs), dtype=torch.float64, device=dev)
    st = torch.zeros(len(recs), dtype=torch.int32, device=dev)
    aux = torch.zeros(len(recs), dtype=torch.int32, device=dev)
    N.check(N.lib().ss_waterfill(len(recs), N.ptr(gp), N.ptr(fl), N.ptr(caps), N.ptr(layers), 0, N.ptr(targets),
                                 N.ptr(tflag), N.ptr(level), None, N.ptr(st), N.ptr(aux), N.stream_handle()),
            "ss_waterfill")
    assert not st.any().item()
    tv, tf, lv = targets.cpu().numpy(), tflag.cpu().numpy(), level.cpu().numpy()
    for i, rec in enumerate(recs):
        got = [int(v) if f else float(v) for v, f in zip(tv[ptr[i]:ptr[i + 1]], tf[ptr[i]:ptr[i + 1]])]
        want = [untag(t) for t in rec["targets"]]
        assert got == want and [type(t) for t in got] == [type(t) for t in want], i
        assert float(lv[i]) == hx(rec["level"]), i
    for total_of in (lambda r: r["L"], lambda r: -1):
        total = torch.tensor([total_of(r) for r in recs], dtype=torch.int32, device=dev)
        counts = torch.zeros(n, dtype=torch.int32, device=dev)
        hs = torch.zeros(len(recs), dtype=torch.int32, device=dev)
        N.check(N.lib().ss_hamilton(len(recs), N.ptr(gp), N.ptr(targets), N.ptr(tflag), N.ptr(caps), N.ptr(total),
                                    N.ptr(counts), N.ptr(hs), N.stream_handle()), "ss_hamilton")
        assert not hs.any().item()
        cv = counts.cpu().numpy()
        for i, rec in enumerate(recs):
            got = cv[ptr[i]:ptr[i + 1]].tolist()
            if total_of(rec) >= 0:
                assert got == rec["layers"], i
            else:
                tg = [untag(t) for t in rec["targets"]]
                assert got == list(waterfill_ref.largest_remainder(tg, rec["caps"])), i


def test_waterfill_batched_vs_oracle(cuda_ready, phase1_cases):
    """All golden rebalance cases in ONE batched ss_waterfill launch (mode 2)."""
    import torch
    from paper_2509_26182_b200 import _native as N
    recs = phase1_cases["rebalance"]
    sizes = [len(r["caps"]) for r in recs]
    ptr = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
    dev = torch.device("cuda")
    fl = torch.tensor([hx(f) for r in recs for f in r["flops"]], dtype=torch.float64, device=dev)
    caps = torch.tensor([c for r in recs for c in r["caps"]], dtype=torch.int32, device=dev)
    layers = torch.tensor([r["L"] for r in recs], dtype=torch.int32, device=dev)
    gp = torch.from_numpy(ptr).to(dev)
    n = int(ptr[-1])
    counts = torch.zeros(n, dtype=torch.int32, device=dev)
    st = torch.zeros(len(recs), dtype=torch.int32, device=dev)
    aux = torch.zeros(len(recs), dtype=torch.int32, device=dev)
    N.check(N.lib().ss_waterfill(len(recs), N.ptr(gp), N.ptr(fl), N.ptr(caps), N.ptr(layers), 2, None, None, None,
                                 N.ptr(counts), N.ptr(st), N.ptr(aux), N.stream_handle()), "ss_waterfill")
    counts, st = counts.cpu().numpy(), st.cpu().numpy()
    names = {6: "RoundingOverflow", 5: "InfeasibleCapacity"}
    for i, rec in enumerate(recs):
        got = names[int(st[i])] if st[i] else counts[ptr[i]:ptr[i + 1]].tolist()
        assert got == rec["lengths"], i


def test_rebalance_pipeline_dropin(cuda_ready):
    from paper_2509_26182_b200 import LayerSlice, ModelSpec, Pipeline, rebalance_pipeline, GpuNode
    model = ModelSpec("m8", 8, 1e9, 2e10)
    gpus = [GpuNode("fast", "east", 6 * 1e9 / 0.8, 3e14), GpuNode("slow", "east", 6 * 1e9 / 0.8, 1e14)]
    pipe = Pipeline((LayerSlice("fast", 1, 4), LayerSlice("slow", 5, 8)), "east")
    out = rebalance_pipeline(pipe, {g.id: g for g in gpus}, model)
    assert [s.length for s in out.stages] == [6, 2]


def test_score_and_errors(cuda_ready):
    from paper_2509_26182_b200 import DegenerateObjective, ObjectiveParams, score, min_stages, k_max
    p = ObjectiveParams(alpha=1.0, t_comp_seconds=0.5, rtt_seconds=0.25)
    assert score(1, 2, p) == alloc_ref.score(1, 2, 1.0, 0.5, 0.25)
    assert score(2, 4, p) == 2.0
    with pytest.raises(DegenerateObjective):
        score(1, 1, ObjectiveParams(1.0, 0.0, 0.0))
    with pytest.raises(ValueError):
        score(2, 1, p)
    assert min_stages([6, 5, 5, 4], 10, 2).stages == 4
    assert min_stages([6, 5, 5, 4], 10, 3) is None
    assert k_max([6, 4, 5, 5], 10) == 2
    from paper_2509_26182_b200 import solve_stage_counts, SweepStats
    with pytest.raises(ValueError):
        solve_stage_counts([4, 6], 10, 1)
    st = SweepStats()
    solve_stage_counts([8, 7, 6, 5, 5, 4, 3, 2], 12, 3, stats=st)
    assert st.pruned_dominated > 0 and st.states_expanded > 0


def test_allocate_bench_pools_vs_oracle(cuda_ready):
    """C1/C2/C3-shaped bench pools and a homogeneous tie pool, plan for plan."""
    from paper_2509_26182_b200 import allocate, scenarios as scen
    for n, seed, L, fl in [(8, 3, 32, None), (64, 7, 64, None), (256, 9, 80, None), (48, 2, 48, 1e14),
                           (1024, 1, 80, None)]:
        cl, m = scen.synthetic_cluster(n, seed=seed, model=scen.bench_model(L), homogeneous_flops=fl)
        got = _plan_hex(allocate(cl, m))
        want = alloc_ref.allocate(cl, m)
        want["objective"] = want["objective"].hex()
        want["per_k"] = [dict(r, z=r["z"].hex()) for r in want["per_k"]]
        assert got == want, (n, seed, L)


def test_variant_sweep_vs_oracle(cuda_ready):
    """C3-shaped candidate sweep (fill_all): every (variant, region, k) candidate vs the oracle."""
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import VariantSweep
    packed, meta = scen.bench_variants(6, 256, 80, seed0=40)
    sw = VariantSweep(packed, fill_all=True)
    sw.run()
    res = sw.batch.fetch()
    totals = sw.total.cpu().numpy()
    for v in range(6):
        cl, m = scen.synthetic_cluster(256, seed=40 + v, model=scen.bench_model(80))
        want = alloc_ref.allocate(cl, m)
        assert totals[v] == want["objective"], v
        for p in range(packed.var_ptr[v], packed.var_ptr[v + 1]):
            pool = packed.pools[p]
            sols = res.solutions(p)
            assert sols == alloc_ref.stage_counts(pool.caps, 80, pool.kmax)
            t, r = alloc_ref.objective([float(x) for x in packed.obj_flops[p]],  # exact floats: CPython sum compensates only PyFloat
                                        [str(i) for i in range(len(packed.obj_flops[p]))],
                                       lambda a, b: 0.0 if a == b else 0.001, m.flops_per_layer_per_token, 80, 128.0)
            for k, (s, groups) in sols.items():
                assert res.z_of(p, k) == alloc_ref.score(k, s, 1.0, t, r)
                counts = res.counts_of(p, k)
                pos = 0
                for grp in groups:
                    want_len = waterfill_ref.stage_lengths([pool.flops[i] for i in grp], [pool.caps[i] for i in grp], 80)
                    assert counts[pos:pos + len(grp)] == want_len
                    pos += len(grp)
    bv = int(sw.best_variant.cpu()[0])
    assert bv == int(np.argmax(totals)) and float(sw.best_total.cpu()[0]) == totals.max()


def test_sweep_stats_and_s_star_vs_reference(cuda_ready):
    """exact_sweep_cta_kernel counters (SweepStats, allocator.py:87-94) and s*(k) vs the reference's own sweep on
    280 exact-path pools, including N=16 / L=80 shapes with ~2k expanded states (tests/golden/sweep_stats_cases.json)."""
    import json
    import os
    from paper_2509_26182_b200 import SweepStats, solve_stage_counts
    with open(os.path.join(os.path.dirname(__file__), "golden", "sweep_stats_cases.json")) as fh:
        cases = json.load(fh)
    for c in cases:
        st = SweepStats()
        sols = solve_stage_counts(c["caps"], c["L"], c["kmax"], stats=st)
        assert [st.levels, st.states_expanded, st.peak_frontier, st.pruned_dominated] == c["stats"], c
        assert {str(k): v.stages for k, v in sols.items()} == c["s_star"], c


@pytest.mark.parametrize("L", [64, 80])
def test_cover_serial_and_parallel_m_paths_agree(cuda_ready, L):
    """ss_stage_counts_cover has two schedules -- the serial group-count loop (large batches) and the parallel
    group-count search with cancellation (small batches).  Forced through each on the same C3-shaped pools, the
    stage totals, groups, water-fill counts and scores must be identical, and the serial run must match the
    oracle (the parallel one is what allocate() and the golden tests exercise)."""
    from paper_2509_26182_b200 import _native as N
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import VariantSweep
    lib = N.lib()
    packed, _ = scen.bench_variants(8, 256, L, seed0=70)
    out = []
    old = lib.ss_set_cover_parallel_limit(-1)
    try:
        for limit in (0, 1 << 30):
            lib.ss_set_cover_parallel_limit(limit)
            sw = VariantSweep(packed, fill_all=True)
            sw.run()
            res = sw.batch.fetch()
            out.append((res.stages.copy(), res.members.copy(), res.gsize.copy(), res.counts.copy(), res.z.copy(),
                        sw.total.cpu().numpy().copy()))
    finally:
        lib.ss_set_cover_parallel_limit(old)
    for a, b in zip(*out):
        assert np.array_equal(a, b)
    stages, koff = out[0][0], sw.batch.koff_h
    for p in range(0, len(packed.pools), 3):
        pool = packed.pools[p]
        want = alloc_ref.stage_counts(pool.caps, L, pool.kmax)
        got = {k: int(stages[koff[p] + k - 1]) for k in range(1, pool.kmax + 1) if int(stages[koff[p] + k - 1]) > 0}
        assert {k: s for k, (s, _) in want.items()} == got, p


@pytest.mark.parametrize("L", [80, 64])
def test_bench_sweep_every_97th_variant_vs_oracle(cuda_ready, L):
    """The bench's whole C3 sweep (synthetic_cluster(256, seed=v), v = 0..1811, one launch set) at L=80 (configs[2])
    and at the north star's L=64: every 97th variant's objective total, stage counts, groups' water-filled layer
    counts and Z(k) vs the oracle's allocate (allocator.py:541-618), and the sweep's argmax vs the totals."""
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import VariantSweep
    V = 1812
    packed, meta = scen.bench_variants(V, 256, L, seed0=0)
    sw = VariantSweep(packed, fill_all=True)
    sw.run()
    res = sw.batch.fetch()
    totals = sw.total.cpu().numpy()
    for v in range(0, V, 97):
        cl, m = scen.synthetic_cluster(256, seed=v, model=scen.bench_model(L))
        want = alloc_ref.allocate(cl, m)
        assert totals[v] == want["objective"], v
        rows = {(r["region"], r["k"]): (r["s_star"], r["z"]) for r in want["per_k"]}
        for p in range(packed.var_ptr[v], packed.var_ptr[v + 1]):
            pool = packed.pools[p]
            region = meta[p][1]
            sols = res.solutions(p)
            assert sols == alloc_ref.stage_counts(pool.caps, L, pool.kmax), (v, region)
            for k, (s, groups) in sols.items():
                assert (s, res.z_of(p, k)) == rows[(region, k)], (v, region, k)
                counts = res.counts_of(p, k)
                pos = 0
                for grp in groups:
                    want_len = waterfill_ref.stage_lengths([pool.flops[i] for i in grp], [pool.caps[i] for i in grp], L)
                    assert counts[pos:pos + len(grp)] == want_len, (v, region, k)
                    pos += len(grp)
    assert int(sw.best_variant.cpu()[0]) == int(np.argmax(totals))
