#!/usr/bin/env python3
"""Cluster / model files written by the UNMODIFIED reference (build container only).

    python tests/golden/make_io_golden.py

topology.py save_cluster / save_model on a bench pool (explicit intra-region links) and on a hand-made pool with an
asymmetric link and a non-default cross-region RTT.  tests/test_wire.py loads them with the drop-in and must
write the same text back.
"""

from __future__ import annotations

import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import swarmsched as ref                                    # noqa: E402


def main():
    model = ref.ModelSpec("bench-32l", 32, 1.2e9, 2.8e10)
    cluster, model = ref.synthetic_cluster(16, seed=4, model=model)
    ref.save_cluster(cluster, os.path.join(HERE, "io_cluster_bench16.json"))
    ref.save_model(model, os.path.join(HERE, "io_model_bench32.json"))
    gpus = (ref.GpuNode("b", "east", 24e9, 1.5e14), ref.GpuNode("a", "east", 40e9, 2e14, 0.1, 50_000),
            ref.GpuNode("c", "west", 80e9, 3e14))
    hand = ref.ClusterSnapshot(gpus=gpus, links={("a", "b"): 0.0015, ("b", "a"): 0.0025, ("a", "c"): 0.031},
                               default_cross_region_rtt_s=0.042)
    ref.save_cluster(hand, os.path.join(HERE, "io_cluster_hand.json"))
    print("wrote io_cluster_bench16.json, io_model_bench32.json, io_cluster_hand.json")


if __name__ == "__main__":
    main()
