"""Ad-hoc probe: C3 Phase-1 sweep throughput (VariantSweep over 1,812 variants), optionally with an A/B library.

    python tests/perf_phase1.py [--lib variants/lib_x.so] [--variants 1812]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default="")
    ap.add_argument("--variants", type=int, default=1812)
    ap.add_argument("--L", type=int, default=80)
    args = ap.parse_args()
    import torch
    from paper_2509_26182_b200 import _native as N, scenarios as scen
    from paper_2509_26182_b200.batched import VariantSweep
    if args.lib:
        N.load_library(args.lib)
    packed, _ = scen.bench_variants(args.variants, 256, args.L, seed0=0)
    sw = VariantSweep(packed, fill_all=True)
    sw.run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sw.run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    n = sw.batch.n_cand
    print(f"lib={args.lib or 'default'} L={args.L}: {n} candidates, median {ts[2]:.2f} ms -> {n / ts[2] * 1e3:.3e} cand/s "
          f"(total {float(sw.total.cpu().sum()):.6e})")


if __name__ == "__main__":
    main()
