// Multi-GPU exchanges of the scheduling path over NCCL (NVLink 5 / NVSwitch on a B200 box): the Phase-1 global
// argmax and the chain gather.  Declared in include/swarmsched_b200_nccl.h.
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

#include "../../include/swarmsched_b200_nccl.h"

namespace {

constexpr int kOk = 0, kBadInput = 8, kCudaError = 9;

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// records [nranks][2]: (objective, id as double -- exact for |id| < 2^53); max objective, ties -> lowest id
__global__ void argmax_pick_kernel(const double* rec, int nranks, const double* obj, const int64_t* id,
                                   double* best_obj, int64_t* best_id) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double bt = 0.0;
    long long bv = -1;
    for (int r = 0; r < nranks; ++r) {
        const double t = rec[2 * r];
        const long long v = (long long)rec[2 * r + 1];
        if (v < 0) continue;
        if (bv < 0 || t > bt || (t == bt && v < bv)) { bt = t; bv = v; }
    }
    best_obj[0] = bt;
    best_id[0] = bv;
}

__global__ void pack_record_kernel(const double* obj, const int64_t* id, double* rec) {
    if (threadIdx.x == 0) { rec[0] = obj[0]; rec[1] = (double)id[0]; }
}

}  // namespace

extern "C" int ss_nccl_unique_id(uint8_t* uid_out) {
    if (!uid_out) return kBadInput;
    ncclUniqueId uid;
    if (ncclGetUniqueId(&uid) != ncclSuccess) return SS_NCCL_ERROR;
    static_assert(sizeof(uid) == SS_NCCL_UID_BYTES, "ncclUniqueId size");
    memcpy(uid_out, &uid, sizeof(uid));
    return kOk;
}

extern "C" int ss_nccl_comm_init(const uint8_t* uid, int32_t nranks, int32_t rank, void** comm_out) {
    if (!uid || !comm_out || nranks < 1 || rank < 0 || rank >= nranks) return kBadInput;
    ncclUniqueId u;
    memcpy(&u, uid, sizeof(u));
    ncclComm_t comm;
    if (ncclCommInitRank(&comm, nranks, u, rank) != ncclSuccess) return SS_NCCL_ERROR;
    *comm_out = comm;
    return kOk;
}

extern "C" int ss_nccl_comm_destroy(void* comm) {
    if (!comm) return kOk;
    return ncclCommDestroy(reinterpret_cast<ncclComm_t>(comm)) == ncclSuccess ? kOk : SS_NCCL_ERROR;
}

extern "C" int ss_argmax_allgather(void* comm, const double* obj, const int64_t* id, double* best_obj,
                                   int64_t* best_id, double* scratch, void* stream) {
    if (!comm || !obj || !id || !best_obj || !best_id || !scratch) return kBadInput;
    ncclComm_t c = reinterpret_cast<ncclComm_t>(comm);
    int nranks = 0, rank = 0;
    if (ncclCommCount(c, &nranks) != ncclSuccess || ncclCommUserRank(c, &rank) != ncclSuccess) return SS_NCCL_ERROR;
    cudaStream_t s = as_stream(stream);
    double* mine = scratch + 2 * rank;                       // in-place all-gather: own slot of the output
    pack_record_kernel<<<1, 32, 0, s>>>(obj, id, mine);
    if (cudaGetLastError() != cudaSuccess) return kCudaError;
    if (ncclAllGather(mine, scratch, 2, ncclFloat64, c, s) != ncclSuccess) return SS_NCCL_ERROR;
    argmax_pick_kernel<<<1, 32, 0, s>>>(scratch, nranks, obj, id, best_obj, best_id);
    return cudaGetLastError() == cudaSuccess ? kOk : kCudaError;
}

extern "C" int ss_gather_chains(void* comm, const int16_t* gpus, const double* cost, int64_t n_sel, int32_t L,
                                int32_t root, int16_t* gpus_out, double* cost_out, void* stream) {
    if (!comm || n_sel < 0 || L < 1 || (n_sel > 0 && (!gpus || !cost))) return kBadInput;
    ncclComm_t c = reinterpret_cast<ncclComm_t>(comm);
    int nranks = 0, rank = 0;
    if (ncclCommCount(c, &nranks) != ncclSuccess || ncclCommUserRank(c, &rank) != ncclSuccess) return SS_NCCL_ERROR;
    if (root < 0 || root >= nranks) return kBadInput;
    if (rank == root && n_sel > 0 && (!gpus_out || !cost_out)) return kBadInput;
    if (n_sel == 0) return kOk;
    cudaStream_t s = as_stream(stream);
    const size_t gbytes = (size_t)n_sel * L * sizeof(int16_t);   // int16 records travel as bytes
    if (ncclGroupStart() != ncclSuccess) return SS_NCCL_ERROR;
    if (rank == root) {
        for (int r = 0; r < nranks; ++r) {
            int16_t* gdst = gpus_out + (size_t)r * n_sel * L;
            double* cdst = cost_out + (size_t)r * n_sel;
            if (r == root) {
                cudaMemcpyAsync(gdst, gpus, gbytes, cudaMemcpyDeviceToDevice, s);
                cudaMemcpyAsync(cdst, cost, (size_t)n_sel * sizeof(double), cudaMemcpyDeviceToDevice, s);
                continue;
            }
            if (ncclRecv(gdst, gbytes, ncclInt8, r, c, s) != ncclSuccess ||
                ncclRecv(cdst, (size_t)n_sel, ncclFloat64, r, c, s) != ncclSuccess) {
                ncclGroupEnd();
                return SS_NCCL_ERROR;
            }
        }
    } else {
        if (ncclSend(gpus, gbytes, ncclInt8, root, c, s) != ncclSuccess ||
            ncclSend(cost, (size_t)n_sel, ncclFloat64, root, c, s) != ncclSuccess) {
            ncclGroupEnd();
            return SS_NCCL_ERROR;
        }
    }
    if (ncclGroupEnd() != ncclSuccess) return SS_NCCL_ERROR;
    return cudaGetLastError() == cudaSuccess ? kOk : kCudaError;
}
