"""Generate tests/golden/c2_stream.json: the first 50,000 C2 ops through the reference itself.

SURVEY.md 8(d) C2: L=64, N=64, seed 0 (k=17), one scenario, W=64 -- the reference's own
`ChainRouter.route/release` (router.py:247-260) over `MembershipManager.initialize` (membership.py:270-278)
with the bench latency law base_s(g)*(1+occ) (bench.py:150-151).  Storing 50k chains verbatim would be
several MB, so each block of 1,000 ops is stored as a digest of (chain hash, cost bits) per op:

    chain hash = sum_l splitmix64((l << 32) | g_l)  mod 2^64   (g_l = sorted-id index of layer l's GPU)
    digest     = sha256(b"".join(pack("<QQ", hash, cost_bits)))[:16] (hex)

-- the same hash the replay kernels emit, so the GPU test compares digests block by block.  The first
differing block localises a mismatch; tests/golden/router_replays.json["c2"] holds the first 300 chains
in full.  Runs only in the build container (needs /root/reference); ~3 minutes at ~330 routes/s.

    python tests/golden/make_c2_stream_golden.py [--routes 50000]
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import struct
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, REPO)

import swarmsched as ref                                    # noqa: E402
from swarmsched.membership import MembershipManager          # noqa: E402

from paper_2509_26182_b200.scenarios import splitmix64       # noqa: E402  (hash definition only)

M64 = (1 << 64) - 1


def chain_hash(chain, pos, L):
    per_layer = [0] * L
    for h in chain.hops:
        for layer in range(h.start_layer, h.end_layer + 1):
            per_layer[layer - 1] = pos[h.gpu_id]
    return sum(splitmix64((l << 32) | g) for l, g in enumerate(per_layer)) & M64


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--routes", type=int, default=50_000)
    ap.add_argument("--block", type=int, default=1_000)
    args = ap.parse_args()
    n, seed, L, W = 64, 0, 64, 64
    model = ref.ModelSpec(f"bench-{L}l", L, 1.2e9, 2.8e10)
    cluster, model = ref.synthetic_cluster(n, seed=seed, model=model)
    plan = ref.allocate(cluster, model)
    pm = ref.PerfMap(ttl_s=4.5)
    mgr = MembershipManager(cluster, model, pm)
    base = {g.id: model.flops_per_layer_per_token / g.flops for g in cluster.gpus}
    pm.latency_fn = lambda gpu_id, layer, occ: base[gpu_id] * (1 + occ)
    mgr.initialize(plan, 0.0)
    router = ref.ChainRouter(pm, L)
    ids = sorted(g.id for g in cluster.gpus)
    pos = {g: i for i, g in enumerate(ids)}
    live, digests, buf = [], [], []
    t0 = time.perf_counter()
    for i in range(args.routes):
        if i >= W:
            router.release(live.pop(0), 0.0)
        chain = router.route(0.0)
        live.append(chain)
        cost_bits = struct.unpack("<Q", struct.pack("<d", chain.cost_s))[0]
        buf.append(struct.pack("<QQ", chain_hash(chain, pos, L), cost_bits))
        if len(buf) == args.block:
            digests.append(hashlib.sha256(b"".join(buf)).hexdigest()[:16])
            buf = []
        if (i + 1) % 10_000 == 0:
            print(f"  {i + 1} routes, {time.perf_counter() - t0:.1f}s", flush=True)
    assert not buf, "routes must be a multiple of block"
    out = {"n": n, "seed": seed, "L": L, "window": W, "k": plan.replication_count, "routes": args.routes,
           "block": args.block, "digests": digests, "final_occ": [pm.occupancy(g) for g in ids],
           "generator": "swarmsched ChainRouter (reference), CPython " + sys.version.split()[0]}
    with open(os.path.join(HERE, "c2_stream.json"), "w") as f:
        json.dump(out, f, indent=0)
    print(f"wrote c2_stream.json: {len(digests)} blocks in {time.perf_counter() - t0:.1f}s")


if __name__ == "__main__":
    main()
