"""C2 stream parity on a B200: 50,000 consecutive ops of one scenario (L64/N64, k=17, W=64) through every
replay kernel, block digests vs the reference's own run (tests/golden/c2_stream.json), final occupancy vs
the reference's PerfMap."""

import pytest

from helpers_golden import stream_digests
from test_c2_stream import c2_scenario, c2_stream  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["warp", "slots", "blocks"])
def test_c2_stream_50k_ops_vs_reference(cuda_ready, c2_stream, mode):  # noqa: F811
    import numpy as np
    from paper_2509_26182_b200.batched import ScenarioReplayer
    _, _, _, ss = c2_scenario()
    rp = ScenarioReplayer(ss, window=c2_stream["window"], mode=mode)
    assert rp.mode == mode
    hashes, costs = [], []
    chunk = 10_000
    for _ in range(c2_stream["routes"] // chunk):
        out = rp.run(chunk)
        hashes.append(out.chain_hash.cpu().numpy()[0])
        costs.append(out.cost.cpu().numpy()[0])
    rp.raise_first_failure()
    got = stream_digests(np.concatenate(hashes), np.concatenate(costs), c2_stream["block"])
    bad = [i for i, (a, b) in enumerate(zip(got, c2_stream["digests"])) if a != b]
    assert not bad, f"first differing block: ops {bad[0] * c2_stream['block']}..+{c2_stream['block']}"
    assert rp.occ.cpu().numpy().tolist() == c2_stream["final_occ"]
