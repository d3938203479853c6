"""Same-box A/B of region-replay library builds (not a test; run on a B200 through gpurun).

    python tests/ab/region_ab.py variants/a.so variants/b.so [...]

Per library: C4 (1,184 scenarios x 64 steady-state requests, the bench's launch shape) and the three C5 sub-pools
(2,048 scenarios each) in selections/s, plus a checksum of the C4 chains, which must agree across builds (every
experiment listed in DESIGN.md as "measured and dropped" was bit-identical by this checksum and the parity tests).
Each library runs in its own process (one CUDA context, one .so), twice in alternation to expose box drift.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def one(lib):
    sys.path.insert(0, ROOT)
    import torch
    from paper_2509_26182_b200 import _native as N
    N.load_library(lib)
    from paper_2509_26182_b200 import allocate, scenarios as scen
    from paper_2509_26182_b200.batched import ScenarioReplayer

    def rate(ss, R, reps):
        rp = ScenarioReplayer(ss, window=64, mode="regions")
        out = rp.run(R)
        rp.run(R, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            rp.run(R, out=out)
        e1.record()
        torch.cuda.synchronize()
        return ss.n_scenarios * R * reps / (e0.elapsed_time(e1) / 1e3), out

    cl, model = scen.synthetic_cluster(256, seed=0, model=scen.bench_model(64))
    ss = scen.build_scenarios(cl, model, allocate(cl, model), 1184, churn=0.05, jitter=True,
                              seeds=list(range(1184)), host_events=False)
    c4, out = rate(ss, 64, 6)
    res = {"lib": lib, "c4": c4, "c4_chain_checksum": int(out.chain_hash.to(torch.int64).sum().item()) & 0xffffffff}
    for name, pcl, pmodel in scen.c5_pools(0):
        pss = scen.build_scenarios(pcl, pmodel, allocate(pcl, pmodel), 2048, churn=0.05, jitter=True,
                                   seeds=list(range(2048)), host_events=False)
        res["c5_" + name] = rate(pss, 64, 3)[0]
    print(json.dumps(res))


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--one":
        return one(sys.argv[2])
    libs = sys.argv[1:]
    for _ in range(2):
        for lib in libs:
            subprocess.run([sys.executable, os.path.abspath(__file__), "--one", lib], check=True)


if __name__ == "__main__":
    main()
