/*
 * swarmsched_b200.h -- C ABI of the B200 scheduling hot path.
 *
 * The reference (arxiv/paper_2509_26182, package `swarmsched`) is pure Python
 * and has no FFI; these entry points are what its Python entry points bind
 * through ctypes.  Each export cites the reference
 * function(s) whose arithmetic it replaces.
 *
 * Conventions
 *   - every function returns an ss_status (int); per-item status arrays carry
 *     item-level failures so one bad scenario never aborts a batch
 *     (sim.py:326-329 records rejections rather than aborting);
 *   - all array pointers are DEVICE pointers unless the name ends in _h;
 *     structs are passed by host pointer and copied into kernel parameters;
 *   - every launch is stream-ordered on the `stream` argument (a cudaStream_t,
 *     NULL = legacy default stream); nothing allocates persistent memory;
 *   - GPU indices are dense positions in Python sorted() order of gpu ids, so
 *     index order == tie-break order (router.py:74,110);
 *   - floating point is IEEE fp64 with no FMA contraction (built -fmad=false),
 *     so results are bit-identical to CPython/numpy.
 */
#ifndef SWARMSCHED_B200_H
#define SWARMSCHED_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the Python shim maps them onto errors.py (errors.py:11-95). */
enum ss_status {
    SS_OK = 0,
    SS_UNCOVERED_LAYER = 1,      /* aux = lowest uncovered 1-based layer (router.py:106-109) */
    SS_NO_PATH = 2,              /* router.py:180-181 */
    SS_OCC_UNDERFLOW = 3,        /* aux = gpu index (perfmap.py:370-374) */
    SS_NO_FEASIBLE_PIPELINE = 4, /* allocator.py:608-611 */
    SS_INFEASIBLE_CAPACITY = 5,  /* waterfill.py:64-65 ; aux = capacity total */
    SS_ROUNDING_OVERFLOW = 6,    /* waterfill.py:86,112,127,167 */
    SS_DEGENERATE_OBJECTIVE = 7, /* allocator.py:109-110 */
    SS_BAD_INPUT = 8,
    SS_CUDA_ERROR = 9,
    SS_WORKSPACE = 10,           /* caller-provided scratch too small; aux = needed units */
    SS_ZERO_CAPACITY = 11        /* waterfill.py:155-157 ; aux = member position */
};

const char* ss_status_str(int status);
int ss_version(void);
/* Hard limits of the device kernels (hosts per DAG column, layers, gpus per DAG). */
int ss_limits(int32_t* max_hosts_h, int32_t* max_layers_h, int32_t* max_gpus_h);

/* ------------------------------------------------------------------------ */
/* Phase-2 layout: a set of layer DAGs           */
/* ------------------------------------------------------------------------ */
typedef struct ss_dag_set {
    int32_t n_dags;
    int32_t max_hosts;          /* max col_len over the set (<= 256) */
    int32_t max_layers;         /* max layers of one DAG (<= 1024) */
    int32_t max_gpus;           /* max DAG-local gpu count (replay; <= 4096) */
    const int32_t* layer_ptr;   /* [n_dags+1]  DAG d owns flat layers [layer_ptr[d], layer_ptr[d+1]) */
    const int32_t* col_off;     /* [total_layers] first node slot of the layer's host column */
    const int32_t* col_len;     /* [total_layers] hosts in the column, sorted-id order */
    const int32_t* node_gpu;    /* [node slots] DAG-local gpu index of each host */
    const double*  node_tau;    /* [node slots] tau(gpu, layer) (select) or NULL (replay) */
    const int64_t* edge_off;    /* [total_layers] offset (doubles, even) of block l -> l+1 */
    const double*  edge_val;    /* row-major R_l x R_{l+1}: row = source host, col = destination */
} ss_dag_set;

/* Per-scenario RTT matrices on device: out[s] = base_rtt (n_gpus x n_gpus, row-major) times the pair jitter of
 * seed s (one IEEE product by a LogNormal(0, 0.2) quantile from a 1,024-entry float32 table) (replaces scenarios.py ScenarioSet.scenario_rtt + an H2D copy of S x N x N doubles). */
int ss_scenario_rtt(int32_t n_scen, int32_t n_gpus, const double* base_rtt, const int64_t* seeds, double* out,
                    void* stream);
/* Dense RTT matrices, one per item (router.py:118-143 rtt_matrix and
 * topology.py:133-142 rtt_s share one rule): out[a][b] = direct (a,b) entry if
 * given, else the (b,a) entry, else `default_value`; diagonal 0; self-links
 * ignored.  Link keys must be unique per item (they come from a dict). */
int ss_rtt_fill(int32_t n_items, const int64_t* mat_off, const int32_t* mat_dim, double* out,
                double default_value, int32_t n_links, const int32_t* link_item,
                const int32_t* link_a, const int32_t* link_b, const double* link_v, void* stream);

/* build_dag (router.py:87-115) on device: host columns from a dense
 * per-DAG tau table (layer-major [L_d x G_d], NaN = no live entry) and an
 * optional exclude mask.  Writes col_len / node_gpu / node_tau into the slots
 * given by col_off (capacity G_d per layer is always enough); status[d] =
 * SS_UNCOVERED_LAYER with aux[d] = lowest empty layer. */
int ss_dag_columns(int32_t n_dags, const int32_t* layer_ptr, const int32_t* gpu_ptr,
                   const int64_t* tau_off, const double* tau_table, const uint8_t* exclude,
                   const int32_t* col_off, int32_t* col_len, int32_t* node_gpu, double* node_tau,
                   int32_t* status, int32_t* aux, void* stream);

/* Scenario columns (C4/C5 replay states): host set of layer l in scenario s =
 * gpus g (pool order) with !leave[s][g] and slice_lo[g] <= l <= slice_hi[g];
 * scenario s owns flat layers [s*L, (s+1)*L).  slice_stride = 0: one shared
 * plan; = n_gpus: per-scenario slices (after joins, ss_scenario_membership). */
int ss_scenario_columns(int32_t n_scen, int32_t layers, int32_t n_gpus, const int32_t* slice_lo,
                        const int32_t* slice_hi, int64_t slice_stride, const uint8_t* leave, const int32_t* col_off,
                        int32_t* col_len, int32_t* node_gpu, int32_t* status, int32_t* aux, void* stream);

/* Edge blocks E_l = RTT[col_l, col_{l+1}] (router.py:169 gather).  RTT source:
 * per-DAG dense matrices at rtt + rtt_off[d] (dim = gpu count of the DAG), or,
 * when jitter_seed != NULL, one shared pool matrix `rtt` (dim n_pool_gpus)
 * scaled per scenario by the splitmix64 pair factor of scenarios.py. */
int ss_dag_edges(const ss_dag_set* dags, const int64_t* rtt_off, const int32_t* rtt_dim, const double* rtt,
                 const int64_t* jitter_seed, int32_t n_pool_gpus, double* edge_val, void* stream);

/* Batched no-feedback chain DP (router.py:157-197 _relax, used by
 * select_chain 200-205): one CTA per DAG.  pick_out[flat layer] = position of
 * the chosen host in the column; cost_out[d] = chain cost; status_out[d]. */
int ss_select(const ss_dag_set* dags, int32_t* pick_out, double* cost_out, int32_t* status_out, void* stream);

/* Replay with on-device load update (router.py:247-260 route/release +
 * perfmap.py:353-382 on_chain_event + sim.py:182-183 latency law).
 * tau(g) = base_tau[g] * occpow[occ[g]].  Op script per scenario: before
 * request i, release chain i-W when W > 0 and i >= W; W == 0 releases right
 * after select; W < 0 never releases.  State (occ, ring, next_req) persists
 * across calls so long replays can be chunked. */
typedef struct ss_replay_state {
    const int32_t* gpu_ptr;     /* [n_dags+1] offsets of per-scenario gpu arrays */
    const double*  base_tau;    /* [sum G] flops_per_layer_per_token / flops */
    int32_t*       occ;         /* [sum G] occupancy, in/out */
    int32_t*       ring;        /* [n_dags * max(W,1) * (max_layers+1)] live chains' distinct gpus */
    int64_t*       next_req;    /* [n_dags] requests routed so far, in/out */
    int32_t*       status;      /* [n_dags] sticky per-scenario status */
    int32_t*       aux;         /* [n_dags] */
} ss_replay_state;

typedef struct ss_replay_out {
    double*   cost;             /* [n_dags * n_req] or NULL */
    uint64_t* chain_hash;       /* [n_dags * n_req] or NULL: sum_l splitmix64(l<<32 | gpu_l) */
    int16_t*  gpus;             /* [n_dags * n_req * max_layers] or NULL: chosen gpu per layer */
} ss_replay_out;

int ss_replay(const ss_dag_set* dags, const ss_replay_state* st, const double* occpow, int32_t occpow_len,
              int32_t window, int32_t n_req, const ss_replay_out* out, void* stream);

/* Fresh replay state (stream-ordered cudaMemsetAsync, no kernel): occupancy [n_gpus_total], release ring
 * [ring_ints], next_req / status / aux [n_dags] -- what a new batch of scenario states starts from (the e2e call
 * of the reference-facing path re-uses one allocation for every batch). */
int ss_replay_reset(const ss_replay_state* st, int32_t n_dags, int64_t n_gpus_total, int64_t ring_ints, void* stream);

/* Membership churn on device (membership.py:303-357).
 * One CTA per scenario replays the scenario's events on the base placement:
 *   1. on_leave of want_leave plan GPUs present at the start, visited in
 *      ascending splitmix64(splitmix64(seed) ^ 0xC4<<40 ^ g) order, each taken
 *      only if every layer of its slice keeps another host (never uncovers);
 *   2. on_join of the first n_join absent GPUs (present0 == 0) in ascending
 *      splitmix64(splitmix64(seed) ^ 0x4A<<40 ^ g) order: slice starts at
 *      bottleneck_layer() (least summed token_cap over current hosts, first
 *      such layer, holes = 0) and spans min(layer_cap, L - start + 1) layers;
 *      layer_cap < 1 joins without a slice (ZeroCapacityGpu).
 * Outputs per scenario row (stride n_gpus): absent (left or never joined),
 * lo_s / hi_s (0 / -1 when no slice), joined[s * n_join + j] (-1 past the
 * pool), status SS_UNCOVERED_LAYER + aux = first hole.  Bit-identical to
 * scenarios.membership_events (pinned to the reference MembershipManager). */
int ss_scenario_membership(int32_t n_scen, int32_t layers, int32_t n_gpus, const int32_t* slice_lo,
                           const int32_t* slice_hi, const uint8_t* present0, const int64_t* token_cap,
                           const int32_t* layer_cap, const int64_t* seeds, int32_t want_leave, int32_t n_join,
                           uint8_t* absent, int32_t* lo_s, int32_t* hi_s, int32_t* joined, int32_t* status,
                           int32_t* aux, void* stream);

/* evaluate_triggers per scenario (membership.py:359-396, perfmap.py:86-114),
 * bit-identical under CPython 3.12 semantics: total memory / flops and the CoV
 * mean / variance are compensated sum()s; per-layer kv / compute are plain
 * folds in slices order.  gpu_order lists the base pool in _gpus (cluster)
 * order, slice_order the plan GPUs in plan.gpu_slices() order; joined GPUs
 * (joined[s * n_join + j], -1 = none) are appended to both.  order_stride > 0:
 * per-scenario slice orders (after a rebalance: the new plan's order, joins
 * included), joined GPUs are then appended to the _gpus order only.  State rows
 * (kv_reserved int64, occ int32; either may be NULL = 0) use state_stride.
 * decision: 0 local/balanced, 1 global/uncovered_layers, 2 global/load_cov_exceeded;
 * first_uncovered = 0 when covered; loads may be NULL. */
int ss_membership_triggers(int32_t n_scen, int32_t layers, int32_t n_gpus, const uint8_t* absent,
                           const int32_t* lo_s, const int32_t* hi_s, int64_t slice_stride, const int32_t* gpu_order,
                           int32_t n_order, const int32_t* slice_order, int32_t n_slice_order, int64_t order_stride,
                           const int32_t* joined,
                           int32_t n_join, const double* vram, const double* reserve, const double* flops,
                           const int64_t* token_cap, const int64_t* kv_reserved, const int32_t* occ,
                           int64_t state_stride, double mix_alpha, double cov_threshold, double* loads, double* cov,
                           int32_t* decision, int32_t* first_uncovered, void* stream);

/* Abort of live chains (sim.py:401-411 _abort_chains_on): for every scenario, each
 * chain of requests [next_req - W, next_req) whose distinct GPUs (ring slot)
 * include a marked GPU (mark[s * n_gpus + g] != 0) is released now -- occ -1
 * on each of its GPUs -- and its ring slot emptied, so release(i - W) later is
 * a no-op.  n_aborted[s] / aborted[s * W + i % W] (optional) report them.
 * W = 0 is a no-op; W < 0 (no window) keeps no ring and is rejected. */
int ss_ring_abort(int32_t n_scen, int32_t n_gpus, int32_t max_layers, int32_t window, const uint8_t* mark,
                  int32_t* occ, int32_t* ring, const int64_t* next_req, int32_t* n_aborted, uint8_t* aborted,
                  void* stream);

/* Admission path (sim.py:319-366) per scenario on a time-free step schedule,
 * for DAGs with <= 32 hosts per layer (one CTA of 1-4 warps per scenario, edges
 * or the scenario's RTT matrix resident; matrix mode as for ss_replay_warp):
 * at step t the requests admitted at step t - W complete (occupancy -1 and
 * tokens released on their distinct GPUs), request t joins the queue, and the
 * queue drains strictly FIFO: the head (tokens uniform in [tok_lo, tok_hi]
 * from its scenario seed, scenarios.request_tokens) is routed with every GPU
 * whose token_cap - reserved < tokens excluded, reserves its tokens and +1
 * occupancy on the chain's distinct GPUs, and the drain stops at the first
 * head with no finite chain.  Occupancy and reservations start at 0.
 * Outputs per request (stride steps): step_out (admission step, -1 = still
 * queued), cost_out, gpus_out (optional); per GPU: kv_out, occ_out.
 * adm_gpus is scratch of n_dags * steps * (max_layers + 1) int32. */
int ss_admission_warp(const ss_dag_set* dags, const int32_t* gpu_ptr, const double* base_tau, const int64_t* token_cap,
                      const double* occpow, int32_t occpow_len, const int64_t* seeds, int32_t tok_lo, int32_t tok_hi,
                      int32_t steps, int32_t window, int32_t* adm_gpus, int32_t* step_out, double* cost_out,
                      int16_t* gpus_out, int64_t* kv_out, int32_t* occ_out, int32_t* status, int32_t* aux,
                      const double* mat, int32_t mat_dim, void* stream);

/* Serving simulator on device (sim.py:_Simulation without membership events):
 * one warp (<= 8 hosts) or a lockstep CTA of up to 4 warps (<= 32 hosts) per
 * scenario runs the discrete-event loop -- arrivals, KV-gated
 * strict-FIFO admission (route with KV-blocked GPUs excluded), prefill and
 * decode steps with occupancy-dependent duration, completions, publish ticks --
 * in the reference's (time, seq) order, on a warp-resident DAG (<= 32 hosts per
 * layer).  Scenario s simulates requests [trace_ptr[s], trace_ptr[s+1]) sorted
 * by arrival; rtt is the scenario's dense one-way RTT matrix (stride
 * max_gpus^2), pub_pow[o] = (1+o)^e and exec_pow[o] = max(1,o)^e for o <
 * pow_len (>= max_live + 2; the first 256 entries are cached in shared memory).
 * max_live is clamped to the live-chain table that fits in shared memory.
 * Per request: done_time / done_rank (completion
 * order), left untouched when unserved (callers pre-fill NaN / -1); per
 * scenario: duration (time of the last event, ticks included), completed,
 * queue_peak, n_events, status (SS_BAD_INPUT: more than max_live concurrent
 * chains, or a chain with more than 32 hops). */
int ss_sim_warp(const ss_dag_set* dags, const int32_t* gpu_ptr, const double* base_tau, const int64_t* token_cap,
                const double* rtt, const double* pub_pow, const double* exec_pow, int32_t pow_len,
                const int32_t* trace_ptr, const double* arrival, const int32_t* prompt, const int32_t* output,
                double publish_interval, int32_t amortize_rtt, int32_t max_live, double* done_time,
                int32_t* done_rank, double* duration, int32_t* completed, int32_t* queue_peak, int64_t* n_events,
                int32_t* status, int32_t* aux, void* stream);

/* ss_sim_warp for wide pools (columns of up to 256 hosts): one CTA of 128
 * threads per scenario, edge blocks (ss_dag_edges layout) read from global
 * memory by the chain DP.  Same arguments, semantics and outputs. */
int ss_sim_cta(const ss_dag_set* dags, const int32_t* gpu_ptr, const double* base_tau, const int64_t* token_cap,
               const double* rtt, const double* pub_pow, const double* exec_pow, int32_t pow_len,
               const int32_t* trace_ptr, const double* arrival, const int32_t* prompt, const int32_t* output,
               double publish_interval, int32_t amortize_rtt, int32_t max_live, double* done_time, int32_t* done_rank,
               double* duration, int32_t* completed, int32_t* queue_peak, int64_t* n_events, int32_t* status,
               int32_t* aux, void* stream);

/* Warp-resident replay for DAGs whose columns hold <= 32 hosts (C1/C2 shapes):
 * one CTA of 1-4 warps per scenario with its edge blocks (the ss_dag_edges
 * layout), ring and state staged in shared memory once per launch; one CTA
 * barrier per layer boundary when the destinations span warps (none for one warp) on the
 * request path.  Same state / outputs / op script as ss_replay (ring entries
 * of a chain are stored in layer order).  ss_replay_warp_smem returns the
 * dynamic shared memory one scenario needs, or -1 when the DAG set does not
 * qualify (hosts > 32, or edges + ring exceed 227 KB).
 * Matrix mode (ss_replay_warp, ss_admission_warp; mat may be NULL): mat holds
 * each scenario's RTT matrix [n_dags][mat_dim][mat_dim] over its pool GPUs
 * (ss_scenario_rtt); when mat_dim^2 is smaller than the edge blocks the kernel
 * stages the matrix instead and gathers E_b[i][j] = M[node_i][node_j] -- the
 * same fp64 values in less shared memory, so more scenarios fit per SM.
 * ss_sim_warp always offers its rtt input this way. */
int64_t ss_replay_warp_smem(const ss_dag_set* dags, int32_t window, int32_t occpow_len, int32_t mat_dim);
int ss_replay_warp(const ss_dag_set* dags, const ss_replay_state* st, const double* occpow, int32_t occpow_len,
                   int32_t window, int32_t n_req, const ss_replay_out* out, const double* mat, int32_t mat_dim,
                   void* stream);

/* ------------------------------------------------------------------------ */
/* Phase-1                                      */
/* ------------------------------------------------------------------------ */
/* A pool = one region of one allocate() call: GPUs sorted by (-capacity, id)
 * (allocator.py:570).  caps are unclamped layer capacities (topology.py:148). */
typedef struct ss_pool_set {
    int32_t n_pools;
    const int32_t* pool_ptr;    /* [n_pools+1] offsets into caps / flops */
    const int32_t* caps;        /* non-increasing within a pool */
    const double*  flops;       /* same order */
    const int32_t* layers;      /* [n_pools] model layer count L */
    const int32_t* kmax;        /* [n_pools] k_max (allocator.py:97-101) */
    const int64_t* memb_off;    /* [n_pools] offset of the pool's (k, member) output block: kmax*n ints */
    const int64_t* gsz_off;     /* [n_pools] offset of the pool's (k, group) size block: kmax*kmax ints */
} ss_pool_set;

/* solve_stage_counts (allocator.py:473-504) for every k <= kmax[p], in
 * three stream-ordered launches the packer issues back to back:
 *   _validate: non-increasing caps (ValueError, 488-489), device limits;
 *              zeroes stages; pool_status[p] = SS_OK / SS_BAD_INPUT.
 *   _exact:    pools with <= 16 usable GPUs (listed in exact_list): level sweep
 *              + dominance pruning + parent replay (138-264), one thread per
 *              pool over a global workspace (ss_stage_counts_workspace bytes
 *              each); SS_WORKSPACE with aux = entries needed when too small.
 *   _cover:    every (pool, k) candidate of the > 16 pools: constructive cover
 *              (267-470), one thread per candidate, then the "first stalled k
 *              drops every larger k" rule per pool (456-458).
 * Output: stages[koff[p] + k-1] = s*(k) or 0 when k is absent;
 * members[memb_off[p] + (k-1)*n + ...] = the k groups concatenated (indices
 * into the pool's sorted caps), gsize[gsz_off[p] + (k-1)*kmax + g] = sizes. */
int64_t ss_stage_counts_workspace(int32_t frontier_cap, int32_t children_cap, int32_t max_levels);
int ss_stage_counts_validate(const ss_pool_set* pools, const int64_t* koff, int32_t* stages, int32_t* pool_status,
                             int32_t* pool_aux, void* stream);
int ss_stage_counts_exact(const ss_pool_set* pools, const int64_t* koff, int32_t* stages, int32_t* members,
                          int32_t* gsize, int32_t* pool_status, int32_t* pool_aux, const int32_t* exact_list,
                          int32_t n_exact, void* workspace, int64_t ws_bytes_per, int32_t frontier_cap,
                          int32_t children_cap, int32_t* sweep_stats /* [n_exact*4] or NULL */, void* stream);
/* max_layers: the largest L among the batch's pools (0 = unknown); it only picks the serial kernel's register
 * budget (<= 64: sized for 12 blocks of 64 per SM), never the result. */
int ss_stage_counts_cover(const ss_pool_set* pools, const int64_t* koff, int32_t* stages, int32_t* members,
                          int32_t* gsize, int32_t* pool_status, const int32_t* cand_pool, const int32_t* cand_k,
                          int32_t n_cand, int32_t* stall, int32_t max_layers, void* stream);

/* estimate_objective_params (allocator.py:516-538): per item, flops and a
 * dense rtt_s matrix in CLUSTER order; CPython 3.12 sum() semantics
 * (Neumaier) reproduced bit-exactly.  out_t[i] = t_comp, out_r[i] = rtt. */
int ss_objective(int32_t n_items, const int32_t* item_ptr, const double* flops, const int64_t* rtt_off,
                 const double* rtt, double fpl, const int32_t* layers, double tokens, double* out_t,
                 double* out_r, void* stream);

/* estimate_objective_params of regions gathered from one pool: region item i =
 * pool GPUs gpu[item_ptr[i] .. item_ptr[i+1]) in cluster order, flops from
 * pool_flops, rtt_s(a, b) = base_rtt[a * n_pool + b] times the scenarios.py
 * pair jitter of seeds[i] when seeds != NULL.  Same arithmetic as ss_objective. */
int ss_objective_pool(int32_t n_items, const int32_t* item_ptr, const int32_t* gpu, const double* pool_flops,
                      const double* base_rtt, int32_t n_pool, const int64_t* seeds, double fpl, const int32_t* layers,
                      double tokens, double* out_t, double* out_r, void* stream);

/* score (allocator.py:104-111) of every (pool, k) candidate, z[koff[p]+k-1] =
 * kpow[k] / (t + (s/k) * r) with kpow[k] = k**alpha from the host; with
 * fill_all != 0 every present k's groups are also water-filled
 * (rebalance_pipeline, waterfill.py:142-183) into counts[memb_off[p] +
 * (k-1)*n + pos].  kstatus = score status, fstatus = fill status per k. */
int ss_phase1_score(const ss_pool_set* pools, const int64_t* koff, const int32_t* stages, const int32_t* members,
                    const int32_t* gsize, const double* t_comp, const double* rtt, const double* kpow,
                    int32_t kpow_len, int32_t fill_all, double* z, int32_t* counts, int32_t* kstatus,
                    int32_t* fstatus, const int32_t* cand_pool, const int32_t* cand_k, int32_t n_cand, void* stream);

/* best_k[p] = argmax over present k by (z, k) (allocator.py:583); then the
 * best k's groups are water-filled (597-606) unless fill_all already did.
 * pool_status takes the first failing score / fill status. */
int ss_phase1_best(const ss_pool_set* pools, const int64_t* koff, const int32_t* stages, const int32_t* members,
                   const int32_t* gsize, const double* z, const int32_t* kstatus, const int32_t* fstatus,
                   int32_t fill_all, int32_t* best_k, int32_t* counts, int32_t* pool_status, void* stream);

/* Objective fold + global argmax over variants (allocator.py:588):
 * variant v owns pools [var_ptr[v], var_ptr[v+1]) in sorted region order;
 * total[v] = left fold of z at each usable pool's best k; feasible[v] = 1 if
 * any pipeline, 0 if none (NoFeasiblePipeline), -status on a pool error;
 * best_variant[0] = argmax total over feasible variants (ties -> lowest v),
 * -1 if none. */
int ss_variant_reduce(int32_t n_var, const int32_t* var_ptr, const int64_t* koff, const int32_t* best_k,
                      const double* z, const int32_t* pool_status, double* total, int32_t* feasible,
                      int32_t* best_variant, double* best_total, void* stream);

/* Water-fill primitives, batched over independent groups (waterfill.py):
 * mode 0 = solve_lambda (targets + level, tflag = 1 where the target is the
 * int cap), 1 = solve_lambda + hamilton_round(total = L), 2 = rebalance
 * (zero promotion).  Per group status; aux = capacity total for INFEASIBLE. */
int ss_waterfill(int32_t n_groups, const int32_t* grp_ptr, const double* flops, const int32_t* caps,
                 const int32_t* layers, int32_t mode, double* targets, int32_t* tflag, double* level,
                 int32_t* counts, int32_t* status, int32_t* aux, void* stream);

/* hamilton_round on given targets (waterfill.py:91-128); total < 0 -> round(sum(targets)). */
int ss_hamilton(int32_t n_groups, const int32_t* grp_ptr, const double* targets, const int32_t* tflag,
                const int32_t* caps, const int32_t* total, int32_t* counts, int32_t* status, void* stream);

/* score() batched (allocator.py:104-111). */
int ss_score(int32_t n, const int32_t* k, const int32_t* s_star, const double* kpow, const double* t_comp,
             const double* rtt, double* z, int32_t* status, void* stream);

/* Slot-tile replay for interval-slice scenario sets (every GPU hosts one
 * contiguous layer slice: allocate() plans and their churned states).  Each
 * GPU gets one shared-memory slot for its whole frontier interval
 * [max(lo-2,0), hi-1] (interval partitioning); the CTA keeps T[slot][slot] =
 * rtt and streams only the rows/columns of GPUs entering the frontier.  The DP
 * reads the same fp64 values as ss_replay -> bit-identical results with ~10x
 * fewer HBM bytes per selection.
 *   ss_slot_program: builds meta (meta_stride bytes per scenario, >=
 *     ss_slot_meta_bytes) and row/column units (stream_stride doubles per
 *     scenario, even) from slices + leave masks + the pool rtt matrix (x the
 *     scenarios.py jitter when jitter_seed != NULL); s_used[s] = slots needed
 *     (<= s_cap, a multiple of 32 <= 256), status[s] = SS_BAD_INPUT if not.
 *   ss_replay_slots: same state / outputs / op script as ss_replay; dags
 *     must be the matching ss_scenario_columns set; s_rows >= max s_used. */
int64_t ss_slot_meta_bytes(int32_t layers, int32_t n_gpus, int32_t s_cap);
int ss_slot_program(int32_t n_scen, int32_t layers, int32_t n_gpus, const int32_t* slice_lo, const int32_t* slice_hi,
                    int64_t slice_stride, const uint8_t* leave, const double* rtt, const int64_t* jitter_seed, int32_t s_cap,
                    int64_t meta_stride, int64_t stream_stride, uint8_t* meta, double* stream, int32_t* s_used,
                    int32_t* status, void* stream_h);
int ss_replay_slots(const ss_dag_set* dags, const uint8_t* meta, int64_t meta_stride, const double* stream,
                    int64_t stream_stride, int32_t s_cap, int32_t s_rows, const ss_replay_state* st,
                    const double* occpow, int32_t occpow_len, int32_t window, int32_t n_req,
                    const ss_replay_out* out, void* stream_h);
int ss_set_slot_staging(int32_t stage_bytes, int32_t n_buffers);

/* Cluster slot replay: the same program (ss_slot_program), state, outputs and op script as ss_replay_slots,
 * for frontiers too wide for two single-CTA tiles per SM.  A thread-block cluster of
 * ceil(s_rows / (32 * dplc)) <= 8 CTAs shares each scenario: CTA q keeps every source row of the tile but only
 * its own 32 * dplc destination slots, so it owns complete destination minima; each boundary's costs are
 * broadcast to the cluster through distributed shared memory (one barrier.cluster per boundary) and CTA 0
 * holds the backpointers and runs the request epilogue.  dplc = 1 or 2 (0: default 1, env SS_CLUSTER_DPL). */
int ss_replay_slots_cluster(const ss_dag_set* dags, const uint8_t* meta, int64_t meta_stride, const double* stream,
                            int64_t stream_stride, int32_t s_cap, int32_t s_rows, const ss_replay_state* st,
                            const double* occpow, int32_t occpow_len, int32_t window, int32_t n_req,
                            const ss_replay_out* out, int32_t dplc, void* stream_h);

/* Region-tiled replay (replaces router.py:247-260 route/release over router.py:163-185 _relax for pools whose
 * GPUs fall into regions: the reference bench pool, bench.py:114-138 + topology.py:133-142, and C5).
 * Same state, outputs and op script as ss_replay; results bit-identical for any input.
 *   tile_of[g]  region ("tile") of pool GPU g, 0..n_tiles-1 (<= 8 tiles); every tile's frontier must fit 32
 *               slots (status[s] = SS_BAD_INPUT otherwise);
 *   bounds      lb[n_tiles][n_tiles], ub[n_tiles], then uni[n_tiles][n_tiles]: lb[S][D] <= every (jittered)
 *               S->D entry of the pool matrix, ub[D] >= every D->D entry, uni[S][D] = the value of every S->D
 *               pool entry when they are all equal (e.g. the default cross-region RTT), else NaN.  A cross-tile
 *               block S->D of a boundary is skipped only when cmin_S + lb[S][D] > cmin_D + ub[D], or exceeds the
 *               largest intra-tile destination minimum (no S candidate can reach, or tie, a D minimum); the
 *               others are relaxed exactly with entries recomputed from uni[S][D] or base_rtt (x the jitter of
 *               jitter_seed);
 *   ss_region_program: per-scenario program (meta_stride bytes >= ss_region_meta_bytes, units of stream_stride
 *               doubles), rt_used[s] = slots needed by the widest tile;
 *   ss_replay_regions: rt_rows >= max rt_used, pos_cap >= the widest column (<= 256). */
int64_t ss_region_meta_bytes(int32_t layers, int32_t n_gpus, int32_t n_tiles, int32_t pos_cap);
int ss_region_program(int32_t n_scen, int32_t layers, int32_t n_gpus, const int32_t* slice_lo,
                      const int32_t* slice_hi, int64_t slice_stride, const uint8_t* leave, const double* rtt,
                      const int64_t* jitter_seed, const int32_t* tile_of, int32_t n_tiles, int32_t pos_cap,
                      int64_t meta_stride, int64_t stream_stride, uint8_t* meta, double* stream, int32_t* rt_used,
                      int32_t* status, void* stream_h);
int ss_replay_regions(const ss_dag_set* dags, const uint8_t* meta, int64_t meta_stride, const double* stream,
                      int64_t stream_stride, int32_t n_tiles, int32_t pos_cap, int32_t rt_rows,
                      const double* bounds, const double* base_rtt, const int64_t* jitter_seed,
                      const ss_replay_state* st, const double* occpow, int32_t occpow_len, int32_t window,
                      int32_t n_req, const ss_replay_out* out, void* stream_h);
int ss_set_region_staging(int32_t stage_bytes, int32_t n_buffers);

/* Kernel tuning knobs (0 = default); returns previous values via *_h. */
int ss_set_tiling(int32_t smem_budget_bytes, int32_t n_buffers, int32_t* old_budget_h, int32_t* old_buffers_h);
/* Constructive stage counts: batches of at most max_candidates (pool, k) candidates try every group count in
 * parallel (cover_try_kernel), larger ones keep the serial m loop (cover_kernel); both give the same result.
 * < 0 leaves the limit unchanged; returns the previous limit (default 2048). */
int32_t ss_set_cover_parallel_limit(int32_t max_candidates);

#ifdef __cplusplus
}
#endif
#endif /* SWARMSCHED_B200_H */
