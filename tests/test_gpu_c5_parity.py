"""C5 (BASELINE configs[4]) parity on a B200: the mixed 1,024-GPU pool exactly as bench.py runs it.

* Phase-1: device ``allocate()`` of each sub-pool (8B L=32 / 32B L=64 / 70B L=80; k = 126 / 103 / 82) equals the
  reference's plan bit for bit (tests/golden/c5_cases.json, from ``allocator.py:541-618``).
* Phase-2: the bench's scenario states (device-generated churn + jitter, ``host_events=False``) replayed for 320
  requests with W = 64 -- releases from request 64 on -- through every kernel that takes the width:
  * against the reference's ``ChainRouter`` (``router.py:247-260``) for the golden seeds, chain for chain,
    cost for cost, final occupancy;
  * against the golden-pinned oracle for a further seeded sample of the bench's 4,096 scenario seeds;
  * the kernels agree with each other on every scenario of the batch.
"""

import numpy as np
import pytest

from conftest import golden, hx
from helpers_golden import hops_from_gpus, plan_from_golden
from oracle import chain_ref

pytestmark = pytest.mark.gpu

R, W = 320, 64
ORACLE_SEEDS = (1067, 2037, 4074)


@pytest.fixture(scope="module")
def c5_cases():
    return golden("c5_cases.json")


def _plan_hex(plan):
    from paper_2509_26182_b200.plan import plan_to_dict
    d = plan_to_dict(plan)
    d["objective"] = d["objective"].hex()
    for row in d["per_k"]:
        row["z"] = row["z"].hex()
    return d


@pytest.mark.parametrize("name", ["8b", "32b", "70b"])
def test_c5_sub_pool(cuda_ready, c5_cases, name):
    from paper_2509_26182_b200 import allocate, scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer, replay_mode
    rec = c5_cases[name]
    pools = {n: (cl, m) for n, cl, m in scen.c5_pools(0)}
    cl, model = pools[name]
    plan = allocate(cl, model)
    assert _plan_hex(plan) == rec["plan"], name
    gold_seeds = sorted(int(s) for s in rec["replays"])
    seeds = np.array(sorted(set(range(0, 4096, 97)) | set(gold_seeds) | set(ORACLE_SEEDS)), dtype=np.int64)
    ss = scen.build_scenarios(cl, model, plan, len(seeds), seeds=seeds, churn=0.05, jitter=True, host_events=False)
    from paper_2509_26182_b200.errors import DeviceError
    outs = {}
    for mode in ("blocks", "slots", "cluster", "regions"):
        rp = ScenarioReplayer(ss, window=W, mode=mode, max_requests=R)
        try:
            out = rp.run(R, gpus=True)
        except DeviceError:
            assert mode == "slots" and name == "8b"          # k = 126: the slot tile exceeds 227 KB
            continue
        rp.raise_first_failure()
        outs[mode] = (out.gpus.cpu().numpy(), out.cost.cpu().numpy(), rp.occ.view(len(seeds), -1).cpu().numpy())
    for mode in outs:
        for a, b in zip(outs["blocks"], outs[mode]):
            assert np.array_equal(a, b), mode
    assert replay_mode(ss, window=W, max_requests=R) in outs
    gpus, cost, occ = outs["blocks"]
    L = model.layer_count
    # the reference's ChainRouter on the same states
    for s in gold_seeds:
        k = int(np.nonzero(seeds == s)[0][0])
        want = rec["replays"][str(s)]
        for i, route in enumerate(want["routes"]):
            assert hops_from_gpus(gpus[k, i, :L].tolist()) == route["hops"], (name, s, i)
            assert cost[k, i] == hx(route["cost"]), (name, s, i)
        assert occ[k].tolist() == want["final_occ"], (name, s)
    # the oracle on further bench seeds (host-drawn states, identical to the device-drawn ones)
    host = scen.build_scenarios(cl, model, plan, len(ORACLE_SEEDS), seeds=np.array(ORACLE_SEEDS), churn=0.05,
                                jitter=True)
    for j, s in enumerate(ORACLE_SEEDS):
        k = int(np.nonzero(seeds == s)[0][0])
        want_g, want_c, want_occ, _ = chain_ref.replay(host.columns(j), host.base_tau, host.scenario_rtt(j), R, W,
                                                       chain_ref.occ_power_table(W + 2))
        assert gpus[k, :, :L].tolist() == want_g, (name, s)
        assert cost[k].tolist() == want_c, (name, s)
        assert occ[k].tolist() == want_occ.tolist(), (name, s)
