"""Same-box A/B of Phase-1 library builds (not a test; run on a B200 through gpurun).

    python tests/ab/phase1_ab.py variants/a.so variants/b.so [...]

Per library: the bench's C3 sweep (1,812 variants, L=80) and the north-star shape (L=64) in candidates/s, plus a
hash of the sweep's stage counts, best k, Z(k), totals and argmax, which must agree across builds.  Each library
runs in its own process, twice in alternation.
"""
import hashlib
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
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import VariantSweep
    import bench
    res = {"lib": lib}
    for L in (80, 64):
        packed, _ = bench._variants_for_rank(scen, 1812, 0, 1, layers=L)
        sw = VariantSweep(packed, fill_all=True)
        sw.run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            sw.run()
        e1.record()
        torch.cuda.synchronize()
        b = sw.batch
        h = hashlib.sha1()
        for t in (b.stages, b.best_k, b.z, sw.total, sw.feasible, sw.best_variant):
            h.update(t.cpu().numpy().tobytes())
        res[f"l{L}"] = packed.n_candidates / (e0.elapsed_time(e1) / 5 / 1e3)
        res[f"l{L}_hash"] = h.hexdigest()[:12]
    print(json.dumps(res))


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--one":
        return one(sys.argv[2])
    for _ in range(2):
        for lib in sys.argv[1:]:
            subprocess.run([sys.executable, os.path.abspath(__file__), "--one", lib], check=True)


if __name__ == "__main__":
    main()
