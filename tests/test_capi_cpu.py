"""CPU-only checks of the C-ABI boundary and the host-side generators."""

import ctypes
import os
import re

import pytest

from conftest import hx

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols(name="swarmsched_b200.h"):
    text = open(os.path.join(ROOT, "include", name)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ss_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_and_exports_every_header_symbol():
    from paper_2509_26182_b200 import _build, _native
    _build.build()
    lib = _native.load_library()
    declared = _header_symbols()
    assert declared, "header parse failed"
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) <= set(_native.exported_symbols()) | {"ss_status_str"}
    assert lib.ss_version() >= 100
    assert lib.ss_status_str(1) == b"uncovered layer"
    h, l, g = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    assert lib.ss_limits(ctypes.byref(h), ctypes.byref(l), ctypes.byref(g)) == 0
    assert h.value == 256


def test_nccl_library_builds_and_exports_every_header_symbol():
    from paper_2509_26182_b200 import _build, _native
    _build.build_nccl()
    lib = _native.load_nccl_library()
    declared = _header_symbols("swarmsched_b200_nccl.h")
    assert set(declared) == set(_native._SIGS_NCCL), declared
    for name in declared:
        assert hasattr(lib, name), name


def test_compute_entry_points_refuse_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2509_26182_b200 import _native
    with pytest.raises(_native.NativeUnavailable):
        _native.lib()


def test_synthetic_cluster_matches_reference_pools(phase1_cases):
    from paper_2509_26182_b200 import scenarios as scen
    for rec in phase1_cases["allocate"]:
        m = re.match(r"bench_n(\d+)_s(\d+)_L(\d+)", rec["name"])
        if not m:
            continue
        n, seed, L = map(int, m.groups())
        cl, _ = scen.synthetic_cluster(n, seed=seed, model=scen.bench_model(L))
        got = [[g.id, g.region, g.vram_bytes.hex(), g.flops.hex(), g.reserve_fraction.hex()] for g in cl.gpus]
        assert got == rec["gpus"], rec["name"]
        assert [[a, b, v.hex()] for (a, b), v in sorted(cl.links.items())] == rec["links"]


def test_jitter_vectorised_equals_scalar():
    from paper_2509_26182_b200 import scenarios as scen
    m = scen.jitter_factor_matrix(12345, 40)
    for i in range(40):
        for j in range(40):
            if i != j:
                assert m[i, j] == scen.jitter_factor(12345, i, j)


def test_replay_mode_selection():
    """Kernel choice is a pure function of the plan geometry (no GPU needed)."""
    import sys, os
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from helpers_golden import plan_from_golden
    from oracle import alloc_ref
    from paper_2509_26182_b200 import scenarios as scen
    from paper_2509_26182_b200.batched import replay_mode

    def plan_for(n, L):
        cl, model = scen.synthetic_cluster(n, seed=0, model=scen.bench_model(L))
        d = alloc_ref.allocate(cl, model)
        d["objective"] = d["objective"].hex()
        d["per_k"] = [dict(r, z=r["z"].hex()) for r in d["per_k"]]
        return cl, model, plan_from_golden(d)

    cl, model, plan = plan_for(64, 64)                  # C2: k = 17
    ss = scen.build_scenarios(cl, model, plan, 2, churn=0.0, jitter=False)
    assert replay_mode(ss, window=64) == "warp"
    assert replay_mode(ss, window=64, mode="blocks") == "blocks"
    cl, model, plan = plan_for(256, 64)                 # C4: k = 73
    ss = scen.build_scenarios(cl, model, plan, 2, churn=0.0, jitter=False)
    assert replay_mode(ss, window=64) == "regions"       # 4 regions, <= 25 slots each, bound gap 6.25 ms
    assert replay_mode(ss, window=64, mode="slots") == "slots"
    with pytest.raises(ValueError):
        replay_mode(ss, window=64, mode="warp")
    cl, model, plan = plan_for(144, 10)                 # k = 129: tile too wide for 2 CTAs/SM
    ss = scen.build_scenarios(cl, model, plan, 2, churn=0.0, jitter=False)
    assert replay_mode(ss, window=64) == "blocks"
