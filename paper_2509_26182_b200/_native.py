"""ctypes binding of ``libswarmsched_b200.so`` (declared in include/swarmsched_b200.h).

This is the only place Python touches the C ABI.  There is no fallback: if the
library is missing or no CUDA device is present, every compute entry point
raises :class:`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import DeviceError, SS_OK

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libswarmsched_b200.so")

i32p = C.POINTER(C.c_int32)


class NativeUnavailable(RuntimeError):
    """The CUDA extension is not built / no B200 is visible.  No CPU fallback exists."""


class DagSet(C.Structure):
    _fields_ = [
        ("n_dags", C.c_int32), ("max_hosts", C.c_int32), ("max_layers", C.c_int32), ("max_gpus", C.c_int32),
        ("layer_ptr", C.c_void_p), ("col_off", C.c_void_p), ("col_len", C.c_void_p), ("node_gpu", C.c_void_p),
        ("node_tau", C.c_void_p), ("edge_off", C.c_void_p), ("edge_val", C.c_void_p),
    ]


class ReplayState(C.Structure):
    _fields_ = [
        ("gpu_ptr", C.c_void_p), ("base_tau", C.c_void_p), ("occ", C.c_void_p), ("ring", C.c_void_p),
        ("next_req", C.c_void_p), ("status", C.c_void_p), ("aux", C.c_void_p),
    ]


class ReplayOut(C.Structure):
    _fields_ = [("cost", C.c_void_p), ("chain_hash", C.c_void_p), ("gpus", C.c_void_p)]


_SIGS = {
    "ss_status_str": (C.c_char_p, [C.c_int]),
    "ss_version": (C.c_int, []),
    "ss_limits": (C.c_int, [i32p, i32p, i32p]),
    "ss_scenario_rtt": (C.c_int, [C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ss_rtt_fill": (C.c_int, [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_int32,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ss_dag_columns": (C.c_int, [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p]),
    "ss_scenario_columns": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p]),
    "ss_dag_edges": (C.c_int, [C.POINTER(DagSet), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                               C.c_void_p, C.c_void_p]),
    "ss_select": (C.c_int, [C.POINTER(DagSet), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ss_replay": (C.c_int, [C.POINTER(DagSet), C.POINTER(ReplayState), C.c_void_p, C.c_int32, C.c_int32,
                            C.c_int32, C.POINTER(ReplayOut), C.c_void_p]),
    "ss_replay_reset": (C.c_int, [C.POINTER(ReplayState), C.c_int32, C.c_int64, C.c_int64, C.c_void_p]),
    "ss_set_tiling": (C.c_int, [C.c_int32, C.c_int32, i32p, i32p]),
    "ss_slot_meta_bytes": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32]),
    "ss_slot_program": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                  C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p]),
    "ss_replay_slots": (C.c_int, [C.POINTER(DagSet), C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32,
                                  C.c_int32, C.POINTER(ReplayState), C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                  C.POINTER(ReplayOut), C.c_void_p]),
    "ss_replay_slots_cluster": (C.c_int, [C.POINTER(DagSet), C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32,
                                          C.c_int32, C.POINTER(ReplayState), C.c_void_p, C.c_int32, C.c_int32,
                                          C.c_int32, C.POINTER(ReplayOut), C.c_int32, C.c_void_p]),
    "ss_set_slot_staging": (C.c_int, [C.c_int32, C.c_int32]),
    "ss_region_meta_bytes": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32, C.c_int32]),
    "ss_region_program": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int64, C.c_int64,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ss_replay_regions": (C.c_int, [C.POINTER(DagSet), C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32,
                                    C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(ReplayState),
                                    C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(ReplayOut), C.c_void_p]),
    "ss_set_region_staging": (C.c_int, [C.c_int32, C.c_int32]),
    "ss_set_cover_parallel_limit": (C.c_int32, [C.c_int32]),
    "ss_replay_warp_smem": (C.c_int64, [C.POINTER(DagSet), C.c_int32, C.c_int32, C.c_int32]),
    "ss_sim_warp": (C.c_int, [C.POINTER(DagSet), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                              C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ss_sim_cta": (C.c_int, [C.POINTER(DagSet), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                              C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                              C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ss_admission_warp": (C.c_int, [C.POINTER(DagSet), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                                    C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_int32, C.c_void_p]),
    "ss_objective_pool": (C.c_int, [C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p,
                                    C.c_double, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ss_ring_abort": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ss_scenario_membership": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ss_membership_triggers": (C.c_int, [C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_int64, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32, C.c_int64, C.c_void_p,
                                         C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_int64, C.c_double, C.c_double, C.c_void_p, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p]),
    "ss_replay_warp": (C.c_int, [C.POINTER(DagSet), C.POINTER(ReplayState), C.c_void_p, C.c_int32, C.c_int32,
                                 C.c_int32, C.POINTER(ReplayOut), C.c_void_p, C.c_int32, C.c_void_p]),
}

class PoolSet(C.Structure):
    _fields_ = [
        ("n_pools", C.c_int32), ("pool_ptr", C.c_void_p), ("caps", C.c_void_p), ("flops", C.c_void_p),
        ("layers", C.c_void_p), ("kmax", C.c_void_p), ("memb_off", C.c_void_p), ("gsz_off", C.c_void_p),
    ]


_V = C.c_void_p
_SIGS_P1 = {
    "ss_stage_counts_workspace": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32]),
    "ss_stage_counts_validate": (C.c_int, [C.POINTER(PoolSet), _V, _V, _V, _V, _V]),
    "ss_stage_counts_exact": (C.c_int, [C.POINTER(PoolSet), _V, _V, _V, _V, _V, _V, _V, C.c_int32, _V, C.c_int64,
                                        C.c_int32, C.c_int32, _V, _V]),
    "ss_stage_counts_cover": (C.c_int, [C.POINTER(PoolSet), _V, _V, _V, _V, _V, _V, _V, C.c_int32, _V, C.c_int32,
                                        _V]),
    "ss_objective": (C.c_int, [C.c_int32, _V, _V, _V, _V, C.c_double, _V, C.c_double, _V, _V, _V]),
    "ss_phase1_score": (C.c_int, [C.POINTER(PoolSet), _V, _V, _V, _V, _V, _V, _V, C.c_int32, C.c_int32, _V, _V,
                                  _V, _V, _V, _V, C.c_int32, _V]),
    "ss_phase1_best": (C.c_int, [C.POINTER(PoolSet), _V, _V, _V, _V, _V, _V, _V, C.c_int32, _V, _V, _V, _V]),
    "ss_variant_reduce": (C.c_int, [C.c_int32, _V, _V, _V, _V, _V, _V, _V, _V, _V, _V]),
    "ss_waterfill": (C.c_int, [C.c_int32, _V, _V, _V, _V, C.c_int32, _V, _V, _V, _V, _V, _V, _V]),
    "ss_hamilton": (C.c_int, [C.c_int32, _V, _V, _V, _V, _V, _V, _V, _V]),
    "ss_score": (C.c_int, [C.c_int32, _V, _V, _V, _V, _V, _V, _V, _V]),
}

_lib = None
_lock = threading.Lock()


def exported_symbols():
    return sorted(set(_SIGS) | set(_SIGS_P1))


def load_library(path: str = LIB_PATH):
    """dlopen the library and attach signatures (works without a GPU)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(f"{path} is missing; run __graft_entry__.build() (nvcc, sm_100a)")
        lib = C.CDLL(path)
        for name, (res, args) in {**_SIGS, **_SIGS_P1}.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


_device_checked = False


LIB_NCCL_PATH = os.path.join(HERE, "libswarmsched_b200_nccl.so")
_nccl_lib = None

_SIGS_NCCL = {
    "ss_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "ss_nccl_comm_init": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "ss_nccl_comm_destroy": (C.c_int, [C.c_void_p]),
    "ss_argmax_allgather": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_void_p]),
    "ss_gather_chains": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_void_p,
                                   C.c_void_p, C.c_void_p]),
}


def load_nccl_library(path: str = LIB_NCCL_PATH):
    """dlopen the exchange library (include/swarmsched_b200_nccl.h); torch is imported first so the process
    shares torch's libnccl.so.2."""
    global _nccl_lib
    with _lock:
        if _nccl_lib is not None:
            return _nccl_lib
        if not os.path.exists(path):
            raise NativeUnavailable(f"{path} is missing; run __graft_entry__.build() (nvcc, sm_100a, NCCL)")
        import torch  # noqa: F401  (loads libnccl.so.2)
        lib = C.CDLL(path)
        for name, (res, args) in _SIGS_NCCL.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _nccl_lib = lib
        return lib


def nccl_lib():
    lib()                                   # device check
    return load_nccl_library()


def lib():
    """The loaded library, after checking (once) that a CUDA device is usable."""
    global _device_checked
    if not _device_checked:
        import torch
        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device visible: the scheduler kernels need a B200 (sm_100a)")
        _device_checked = True
    return load_library()


def check(status: int, what: str) -> None:
    if status != SS_OK:
        msg = "NCCL error" if status == 12 else load_library().ss_status_str(status).decode()
        raise DeviceError(f"{what}: {msg} (status {status})")


def ptr(t) -> C.c_void_p:
    """Device pointer of a torch tensor (None -> NULL)."""
    return C.c_void_p(0 if t is None else t.data_ptr())


def stream_handle(stream=None) -> C.c_void_p:
    import torch
    if stream is not None:
        return C.c_void_p(stream.cuda_stream)
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)    # the current stream without a Stream object
    if raw is not None:
        return C.c_void_p(raw(torch._C._cuda_getDevice()))
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)
