"""The single-request ChainRouter keeps its device DAG across routes; every route must still equal a fresh
select_chain on that instant's snapshot (router.py:247-257) -- across feedback, exclude-set changes, placement
changes, RTT republication and TTL expiry."""

import pytest

from oracle import chain_ref

pytestmark = pytest.mark.gpu


def _expected(pm, now, L, exclude):
    snap = pm.snapshot(now)
    got = chain_ref.select(snap.layer_latencies, L, snap.link_rtt_entries(), frozenset(exclude))
    return got


def _as_tuple(chain):
    return ("ok", [(h.gpu_id, h.start_layer, h.end_layer) for h in chain.hops], chain.cost_s)


def test_cached_routes_equal_fresh_selection(cuda_ready):
    from paper_2509_26182_b200 import ChainRouter, NoPath, PerfMap, UncoveredLayer
    flops = {"a": 1.0, "b": 1.3, "c": 0.8, "d": 1.1, "e": 0.9, "f": 1.2}
    pm = PerfMap(ttl_s=2.0, latency_fn=lambda g, l, occ: 1e-3 / flops[g] * (1 + occ))
    for g in flops:
        pm.register_gpu(g)
    ids = sorted(flops)
    rtt = {(x, y): 0.001 * (1 + (ord(x) * 7 + ord(y) * 3) % 5) for i, x in enumerate(ids) for y in ids[i + 1:]}
    pm.publish_link_rtts(rtt, 0.0)
    slices = {"a": (1, 3), "b": (4, 6), "c": (1, 2), "d": (3, 6), "e": (1, 4), "f": (5, 6)}
    for g, (s, e) in slices.items():
        pm.sync_gpu_layers(g, range(s, e + 1), 0.0)
    L = 6
    router = ChainRouter(pm, L)
    live = []

    def route(now, exclude=frozenset()):
        want = _expected(pm, now, L, exclude)
        try:
            chain = router.route(now, exclude=exclude)
        except UncoveredLayer as exc:
            assert want == ("uncovered", exc.layer)
            return None
        except NoPath:
            assert want == ("no_path",)
            return None
        assert _as_tuple(chain) == (want[0], [tuple(h) for h in want[1]], want[2])
        live.append(chain)
        return chain

    for _ in range(5):                                  # feedback only: cached path
        route(0.1)
    router.release(live.pop(0), 0.2)
    route(0.2)
    route(0.3, exclude={"a", "e"})                       # exclude-set change
    route(0.3)
    pm.sync_gpu_layers("f", range(2, 7), 0.4)            # placement change: key set grows
    route(0.4)
    pm.sync_gpu_layers("c", range(1, 2), 0.5)            # key set shrinks
    route(0.5)
    pm.publish_link_rtts({("a", "b"): 0.0001}, 0.6)      # RTT table republished
    route(0.6)
    for g in ("a", "b", "c", "d"):                       # only some latencies refreshed ...
        pm.sync_gpu_layers(g, range(slices[g][0] if g != "c" else 1, (slices[g][1] if g != "c" else 1) + 1), 2.3)
    pm.publish_link_rtts(rtt, 2.3)
    route(2.45)                                          # ... e, f expired (ttl 2.0): dropped from the DAG
    route(2.45, exclude={"d"})
    pm.sync_gpu_layers("e", range(1, 5), 2.5)           # expired entries republished under the SAME keys:
    pm.sync_gpu_layers("f", range(2, 7), 2.5)           # the key-set version does not move, the DAG must
    route(2.55)
    route(2.6)
    assert router.stats.matrix_reuses > 0 and router.stats.dags_built == router.stats.matrix_reuses + \
        router.stats.matrix_rebuilds


def test_routers_sharing_one_perf_map(cuda_ready):
    """Two routers on one PerfMap: each must see every republication (no destructive drain of the changes)."""
    from paper_2509_26182_b200 import ChainRouter, PerfMap
    flops = {"a": 1.0, "b": 2.0, "c": 1.5, "d": 0.7}
    pm = PerfMap(ttl_s=10.0, latency_fn=lambda g, l, occ: 1e-3 / flops[g] * (1 + occ))
    for g in flops:
        pm.register_gpu(g)
    ids = sorted(flops)
    pm.publish_link_rtts({(x, y): 0.0005 * (1 + (i + j) % 3) for i, x in enumerate(ids)
                          for j, y in enumerate(ids) if i < j}, 0.0)
    for g, (s, e) in {"a": (1, 4), "b": (1, 2), "c": (3, 4), "d": (1, 4)}.items():
        pm.sync_gpu_layers(g, range(s, e + 1), 0.0)
    L = 4
    r1, r2 = ChainRouter(pm, L), ChainRouter(pm, L)
    for step in range(12):
        for r in ((r1, r2) if step % 3 else (r2, r1)):
            want = _expected(pm, 0.1, L, frozenset())
            chain = r.route(0.1)
            assert _as_tuple(chain) == (want[0], [tuple(h) for h in want[1]], want[2])
