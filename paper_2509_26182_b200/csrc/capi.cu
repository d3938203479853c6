// Misc C-ABI exports: status strings, version, limits.
#include "ss_common.cuh"

extern "C" const char* ss_status_str(int status) {
    switch (status) {
        case SS_OK: return "ok";
        case SS_UNCOVERED_LAYER: return "uncovered layer";
        case SS_NO_PATH: return "no path";
        case SS_OCC_UNDERFLOW: return "occupancy underflow";
        case SS_NO_FEASIBLE_PIPELINE: return "no feasible pipeline";
        case SS_INFEASIBLE_CAPACITY: return "infeasible capacity";
        case SS_ROUNDING_OVERFLOW: return "rounding overflow";
        case SS_DEGENERATE_OBJECTIVE: return "degenerate objective";
        case SS_BAD_INPUT: return "bad input";
        case SS_CUDA_ERROR: return "cuda error";
        case SS_WORKSPACE: return "workspace too small";
        case SS_ZERO_CAPACITY: return "zero capacity gpu";
        default: return "unknown status";
    }
}

extern "C" int ss_version(void) { return 100; }

extern "C" int ss_limits(int32_t* max_hosts_h, int32_t* max_layers_h, int32_t* max_gpus_h) {
    if (max_hosts_h) *max_hosts_h = SS_MAX_HOSTS;
    if (max_layers_h) *max_layers_h = SS_MAX_LAYERS;
    if (max_gpus_h) *max_gpus_h = SS_MAX_GPUS;
    return SS_OK;
}

extern "C" int ss_replay_reset(const ss_replay_state* st, int32_t n_dags, int64_t n_gpus_total, int64_t ring_ints,
                               void* stream_h) {
    if (!st || n_dags < 0 || n_gpus_total < 0 || ring_ints < 0) return SS_BAD_INPUT;
    cudaStream_t s = ss_stream(stream_h);
    if ((n_gpus_total && cudaMemsetAsync(st->occ, 0, sizeof(int32_t) * (size_t)n_gpus_total, s) != cudaSuccess) ||
        (ring_ints && cudaMemsetAsync(st->ring, 0, sizeof(int32_t) * (size_t)ring_ints, s) != cudaSuccess) ||
        (n_dags && (cudaMemsetAsync(st->next_req, 0, sizeof(int64_t) * (size_t)n_dags, s) != cudaSuccess ||
                    cudaMemsetAsync(st->status, 0, sizeof(int32_t) * (size_t)n_dags, s) != cudaSuccess ||
                    (st->aux && cudaMemsetAsync(st->aux, 0, sizeof(int32_t) * (size_t)n_dags, s) != cudaSuccess))))
        return SS_CUDA_ERROR;
    return SS_OK;
}
