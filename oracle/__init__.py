"""CPU oracle for the Parallax scheduling hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, on the CPU, the reference's algorithms for the path
named by BASELINE.json's north star:

* ``oracle.chain_ref``    Phase-2 chain DP, DAG columns, RTT matrix, replay
                          with occupancy feedback (router.py / perfmap.py).
* ``oracle.alloc_ref``    Phase-1 stage-count sweep, constructive cover,
                          objective, score and allocate (allocator.py).
* ``oracle.waterfill_ref`` water level bisection, Hamilton rounding, stage
                          rebalance (waterfill.py).

Every function cites the reference file:line it follows.  The oracle is pinned
against golden vectors produced by importing the unmodified reference in the
build container (``tests/golden/make_golden.py``) -- see
``tests/test_oracle_golden.py``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg (``--impl reference`` / ``cpu_baseline``) may import this package.  The
product package ``paper_2509_26182_b200`` never imports it; its compute path
is the CUDA extension and fails loudly when that is missing.
"""
