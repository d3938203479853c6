"""Edge cases of the replay kernels on hand-built scenario sets, checked against the oracle.

Single-layer and two-layer models, a single pipeline, the widest columns each kernel accepts (32 hosts for the
warp-resident kernel, 256 for the streamed one), disconnected layers (NoPath), and the drop-in router's
OccupancyUnderflow.
"""

import numpy as np
import pytest

from oracle import chain_ref

pytestmark = pytest.mark.gpu


def manual_set(L, lo, hi, rtt, tau, S=2, jitter=False, seed0=3):
    from paper_2509_26182_b200.scenarios import ScenarioSet
    n = len(lo)
    ids = [f"gpu-{i:04d}" for i in range(n)]
    return ScenarioSet(L, ids, np.asarray(rtt, dtype=np.float64), np.asarray(tau, dtype=np.float64),
                       np.asarray(lo, dtype=np.int32), np.asarray(hi, dtype=np.int32),
                       np.arange(seed0, seed0 + S, dtype=np.int64), np.zeros((S, n), dtype=bool), jitter)


def random_pool(rng, n):
    rtt = rng.uniform(0.001, 0.02, size=(n, n))
    rtt = (rtt + rtt.T) / 2
    np.fill_diagonal(rtt, 0.0)
    tau = rng.uniform(1e-4, 5e-4, size=n)
    return rtt, tau


def check_vs_oracle(ss, mode, n_req=12, window=4):
    from paper_2509_26182_b200.batched import ScenarioReplayer
    rp = ScenarioReplayer(ss, window=window, max_requests=n_req + 4, mode=mode)
    assert rp.mode == mode
    out = rp.run(n_req, gpus=True)
    rp.raise_first_failure()
    for s in range(ss.n_scenarios):
        want_g, want_c, want_occ, _ = chain_ref.replay(ss.columns(s), ss.base_tau, ss.scenario_rtt(s), n_req,
                                                       window, chain_ref.occ_power_table(n_req + 4))
        assert out.gpus.cpu().numpy()[s].tolist() == want_g, (mode, s)
        assert out.cost.cpu().numpy()[s].tolist() == want_c, (mode, s)
        assert rp.occ.view(ss.n_scenarios, -1)[s].cpu().numpy().tolist() == want_occ.tolist()


@pytest.mark.parametrize("mode", ["warp", "blocks"])
def test_single_layer_model(cuda_ready, mode):
    rng = np.random.default_rng(1)
    rtt, tau = random_pool(rng, 6)
    check_vs_oracle(manual_set(1, [1] * 6, [1] * 6, rtt, tau), mode)


@pytest.mark.parametrize("mode", ["warp", "blocks", "slots"])
def test_two_layer_model_and_single_pipeline(cuda_ready, mode):
    rng = np.random.default_rng(2)
    rtt, tau = random_pool(rng, 5)
    # hosts 0-2 serve both layers, 3 serves layer 1, 4 serves layer 2
    check_vs_oracle(manual_set(2, [1, 1, 1, 1, 2], [2, 2, 2, 1, 2], rtt, tau, jitter=True), mode)
    # one pipeline of 3 GPUs: no choice at all
    check_vs_oracle(manual_set(6, [1, 3, 5], [2, 4, 6], rtt[:3, :3], tau[:3]), mode)


@pytest.mark.parametrize("mode", ["warp", "blocks"])
def test_widest_warp_column(cuda_ready, mode):
    rng = np.random.default_rng(3)
    rtt, tau = random_pool(rng, 40)
    lo = np.r_[np.ones(32, dtype=int), np.full(8, 9)]
    hi = np.r_[np.full(32, 8), np.full(8, 12)]          # 32 hosts on layers 1-8, 8 on 9-12
    check_vs_oracle(manual_set(12, lo, hi, rtt, tau, jitter=True), mode, n_req=10, window=3)


def test_widest_streamed_column(cuda_ready):
    rng = np.random.default_rng(4)
    rtt, tau = random_pool(rng, 256)
    check_vs_oracle(manual_set(3, [1] * 256, [3] * 256, rtt, tau, S=1), "blocks", n_req=6, window=2)


@pytest.mark.parametrize("mode", ["warp", "blocks", "slots"])
def test_disconnected_layers_report_no_path(cuda_ready, mode):
    from paper_2509_26182_b200.batched import ScenarioReplayer
    from paper_2509_26182_b200.errors import NoPath
    rng = np.random.default_rng(5)
    rtt, tau = random_pool(rng, 4)
    rtt[np.ix_([0, 1], [2, 3])] = np.inf                 # layer-1 hosts cannot reach layer-2 hosts
    rtt[np.ix_([2, 3], [0, 1])] = np.inf
    ss = manual_set(2, [1, 1, 2, 2], [1, 1, 2, 2], rtt, tau)
    rp = ScenarioReplayer(ss, window=2, max_requests=8, mode=mode)
    out = rp.run(3)
    assert (rp.status.cpu().numpy() == 2).all()
    assert np.isinf(out.cost.cpu().numpy()[:, 0]).all()
    with pytest.raises(NoPath):
        rp.raise_first_failure()


def test_dropin_release_without_select_underflows(cuda_ready):
    from paper_2509_26182_b200 import ChainRouter, OccupancyUnderflow, PerfMap, PipelineChain
    from paper_2509_26182_b200.topology import LayerSlice
    pm = PerfMap(ttl_s=10.0, latency_fn=lambda g, l, occ: 1e-3 * (1 + occ))
    for g in ("a", "b"):
        pm.register_gpu(g)
    pm.publish_link_rtts({("a", "b"): 0.002}, 0.0)
    pm.sync_gpu_layers("a", [1], 0.0)
    pm.sync_gpu_layers("b", [2], 0.0)
    router = ChainRouter(pm, 2)
    chain = router.route(0.0)
    assert [h.gpu_id for h in chain.hops] == ["a", "b"] and chain.cost_s == (1e-3 + 0.002) + 1e-3
    router.release(chain, 0.0)
    with pytest.raises(OccupancyUnderflow):
        router.release(PipelineChain(hops=(LayerSlice("a", 1, 1), LayerSlice("b", 2, 2)), cost_s=0.0), 0.0)
    assert pm.occupancy("a") == 0 and pm.occupancy("b") == 0


@pytest.mark.parametrize("n", [12, 20, 29])
def test_multiwarp_route_single_layer_and_ties(cuda_ready, n):
    """replay_warp_kernel<NWD> (NWD = 2, 3, 4 for 12 / 20 / 29 hosts): a one-layer model (no boundary: only the
    final first-index argmin) and a tie-quantised 6-layer pool where equal candidates meet across the four source
    phases and warps -- both vs the oracle's strict-< numpy argmin."""
    rng = np.random.default_rng(50 + n)
    rtt, tau = random_pool(rng, n)
    check_vs_oracle(manual_set(1, [1] * n, [1] * n, rtt, np.full(n, 2e-4)), "warp")
    q = rng.choice([0.001, 0.002], size=(n, n))
    q = np.triu(q, 1) + np.triu(q, 1).T
    lo = rng.integers(1, 4, size=n)
    hi = np.minimum(lo + rng.integers(2, 5, size=n), 6)
    lo[:3], hi[:3] = 1, 6                                      # every layer covered
    check_vs_oracle(manual_set(6, lo, hi, q, np.full(n, 1e-4)), "warp", n_req=16, window=5)
