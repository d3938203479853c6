"""The e2e (host-in, host-out) call of the replay: ScenarioReplayer.run_from_host resets the state inside the C ABI
(ss_replay_reset), rebuilds the device scenario states from host seeds and returns every selection's cost, chain
hash and chain into pinned host buffers -- identical to the device-resident run, call after call."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["slots", "blocks"])
def test_run_from_host_returns_the_device_run(cuda_ready, mode):
    import torch
    from paper_2509_26182_b200 import allocate, scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer
    cl, model = scen.synthetic_cluster(256, seed=0, model=scen.bench_model(64))
    plan = allocate(cl, model)
    S, R, W = 48, 96, 64
    ss = scen.build_scenarios(cl, model, plan, S, churn=0.05, jitter=True, seeds=np.arange(S), host_events=False)
    ref = ScenarioReplayer(ss, window=W, mode=mode, max_requests=R)
    want = ref.run(R, gpus=True)
    want_g, want_c, want_h = want.gpus.cpu().numpy(), want.cost.cpu().numpy(), want.chain_hash.cpu().numpy()
    rp = ScenarioReplayer(ss, window=W, mode=mode, max_requests=R)
    seeds_h = torch.from_numpy(ss.seeds.copy()).pin_memory()
    cost_h = torch.empty((S, R), dtype=torch.float64).pin_memory()
    hash_h = torch.empty((S, R), dtype=torch.int64).pin_memory()
    gpus_h = torch.empty((S, R, 64), dtype=torch.int16).pin_memory()
    for _ in range(3):                                    # state is reset every call: same answer each time
        rp.run_from_host(None, seeds_h, R, cost_h, hash_h, gpus_h)
        torch.cuda.synchronize()
        assert np.array_equal(gpus_h.numpy(), want_g)
        assert np.array_equal(cost_h.numpy(), want_c)
        assert np.array_equal(hash_h.numpy(), want_h)
