/* swarmsched_b200_nccl.h -- C ABI of the multi-GPU exchanges.
 *
 * Separate library (libswarmsched_b200_nccl.so) so the single-GPU hot path has no NCCL dependency.
 * One process per GPU; the scenario / variant shards run with no data-path collective, and these are the
 * only two exchanges of the path:
 *   - the Phase-1 global argmax over variants (replaces the reference's single-process
 *     max(scored, key=(Z, k)) / left fold over regions, allocator.py:583-588, lifted to "best objective total
 *     over variants, ties -> lowest variant id");
 *   - the gather of chosen chains to one rank (the reference returns PipelineChain objects in-process,
 *     router.py:247-257; here int16 host[L] + fp64 cost records per selection).
 * Every call is stream-ordered on the caller's cudaStream_t; pointers are device pointers; int status
 * (0 OK, 8 BAD_INPUT, 9 CUDA_ERROR, 12 NCCL_ERROR). */
#ifndef SWARMSCHED_B200_NCCL_H
#define SWARMSCHED_B200_NCCL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SS_NCCL_ERROR 12
#define SS_NCCL_UID_BYTES 128

/* ncclGetUniqueId on the root rank; the caller broadcasts the 128 bytes (torch.distributed). */
int ss_nccl_unique_id(uint8_t* uid_out);

/* ncclCommInitRank over `nranks` ranks; *comm_out receives the opaque ncclComm_t. */
int ss_nccl_comm_init(const uint8_t* uid, int32_t nranks, int32_t rank, void** comm_out);

int ss_nccl_comm_destroy(void* comm);

/* Global argmax: every rank contributes (obj, id), id < 0 = no feasible candidate.  ncclAllGather of the
 * 16-byte records into scratch[2 * nranks] (doubles), then one thread picks max obj, ties -> lowest id.
 * Every rank receives the winner in best_obj[0] / best_id[0] (device memory). */
int ss_argmax_allgather(void* comm, const double* obj, const int64_t* id, double* best_obj, int64_t* best_id,
                        double* scratch, void* stream);

/* Gather n_sel selections of every rank on `root`: gpus int16[n_sel * L] and cost fp64[n_sel] per rank (every
 * rank holds the same n_sel).  Grouped ncclSend / ncclRecv (NCCL has no gather); on the root the records land
 * rank-major in gpus_out[nranks * n_sel * L] / cost_out[nranks * n_sel]; other ranks may pass NULL outputs. */
int ss_gather_chains(void* comm, const int16_t* gpus, const double* cost, int64_t n_sel, int32_t L, int32_t root,
                     int16_t* gpus_out, double* cost_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif
