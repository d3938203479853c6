// Warp-resident replay: Phase-2 route / release(i - W) for DAGs whose layer
// columns hold <= 32 hosts (C1 / C2 shapes).
//
// One CTA owns one scenario for the whole launch.  Its edge blocks, host
// columns, occupancy, release ring and backpointers are copied into shared
// memory once; every request then runs the chain DP on NWD warps:
//   * <= 8 hosts (NWD = 1, warp_route): lane j forms the candidates c_i + E_b[i][j]
//     eight sources at a time, then a tournament whose left operand always holds the
//     lower source index and loses only to a strictly smaller right value == numpy
//     first-index argmin (router.py:171); no CTA barrier;
//   * 9..32 hosts (NWD = ceil(hosts / 8), mw_route in warp_dag.cuh): warps own eight
//     destinations each, lanes split the sources four ways, one CTA barrier per boundary;
//   * cost = (c_i + r_ij) + tau_j exactly (router.py:170-174);
//   * load update as perfmap.py:353-382 with tau = base(g) * (1 + occ)^e
//     (sim.py:182-183) and the distinct GPUs of each chain kept in the ring.
#include <float.h>
#include <stdio.h>
#include <stdlib.h>

#include "warp_dag.cuh"

namespace {

using namespace ssw;

struct WarpReplay {
    ss_replay_state st;
    ss_replay_out out;
    const double* occpow;
    int32_t occpow_len;
    int32_t window;
    int32_t n_req;
    unsigned long long* prof;   // diagnostics (env SS_WARP_PROF=1): cycles per phase, else NULL
    const double* mat;          // matrix mode (A.mat_dim > 0): per-scenario RTT matrices [n_dags][dim][dim]
};

// NWD = 1: one warp owns the scenario (<= 8 hosts per column, warp_route).  NWD = 2..4: the destinations of
// every boundary are spread over NWD warps (mw_route); the rest of the request stays on warp 0.
// LPD > 0: pad_route over padded edge blocks (LPD lanes per destination, SPL sources per lane, NWD warps).
template <int NWD, int SPL, bool MAT = false, int LPD = 0>
__global__ void __launch_bounds__(NWD * 32) replay_warp_kernel(ss_dag_set D, WarpLayout A, WarpReplay R) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int NT = NWD * 32;
    const int dag = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    if (R.st.status[dag] != SS_OK) return;                      // sticky failure: skip
    const int l0 = D.layer_ptr[dag];
    const int nl = D.layer_ptr[dag + 1] - l0;
    const int nblk = nl - 1;
    double* E = reinterpret_cast<double*>(smem + A.off_E);
    int* node = reinterpret_cast<int*>(smem + A.off_node);
    int* cl = reinterpret_cast<int*>(smem + A.off_cl);
    int* noff = reinterpret_cast<int*>(smem + A.off_noff);
    int* eoff = reinterpret_cast<int*>(smem + A.off_eoff);
    uint8_t* bp = smem + A.off_bp;
    int* picks = reinterpret_cast<int*>(smem + A.off_picks);
    double* tau = reinterpret_cast<double*>(smem + A.off_tau);
    double* base = reinterpret_cast<double*>(smem + A.off_base);
    int* occ = reinterpret_cast<int*>(smem + A.off_occ);
    int* stamp = reinterpret_cast<int*>(smem + A.off_stamp);
    int* ring = reinterpret_cast<int*>(smem + A.off_ring);
    double* pw = reinterpret_cast<double*>(smem + A.off_pow);
    double* costs = reinterpret_cast<double*>(smem + A.off_cost);   // [2][40] column costs (32 hosts + 8 pad)
    __shared__ double vshare;
    __shared__ int flag[3];
    __shared__ int ishare[16];
    int* pdst = reinterpret_cast<int*>(smem + A.off_dst);
    uint8_t* path = smem + A.off_path;

    // ---- one-time staging: columns, edges, per-GPU state, ring --------------
    if (warp == 0) {
        flag[0] = stage_dag(D, A, l0, nl, E, node, cl, noff, eoff, lane,
                            A.mat_dim ? R.mat + (int64_t)dag * A.mat_dim * A.mat_dim : nullptr) ? 0 : 1;
        if (LPD > 0 && !flag[0]) stage_pad_dst(node, cl, noff, nblk, A.pad, D.max_gpus, pdst, lane);
        if (lane == 0) tau[D.max_gpus] = INF;                       // pad_route's sentinel slot
    }
    __syncthreads();
    if (flag[0]) {
        if (tid == 0) R.st.status[dag] = SS_BAD_INPUT;
        return;
    }
    const int gbase = R.st.gpu_ptr[dag];
    const int ng = R.st.gpu_ptr[dag + 1] - gbase;
    const int window = R.window;
    const int ring_stride = D.max_layers + 1;
    int* ring_g = R.st.ring + (int64_t)dag * (window > 0 ? window : 1) * ring_stride;
    for (int g = tid; g < ng; g += NT) {
        occ[g] = R.st.occ[gbase + g];
        base[g] = R.st.base_tau[gbase + g];
        stamp[g] = 0;
    }
    for (int o = tid; o < A.pow_len; o += NT) pw[o] = R.occpow[o];
    for (int q = tid; q < A.ring_len; q += NT) ring[q] = ring_g[q];
    if (tid < 8) { costs[32 + tid] = INF; costs[72 + tid] = INF; }
    __syncthreads();

    const int n_req = R.n_req;
    const int64_t req0 = R.st.next_req[dag];
    int status = SS_OK, aux = 0, done = 0;
    unsigned long long pacc[3] = {0, 0, 0};
    long long tp = clock64();
    auto mark = [&](int k) {
        if (R.prof) {
            const long long t = clock64();
            pacc[k] += (unsigned long long)(t - tp);
            tp = t;
        }
    };
    for (int r = 0; r < n_req; ++r) {
        const int64_t req = req0 + r;
        mark(2);
        // ---- release chain req - W, refresh tau(g) ----------------------------
        if (window > 0 && req >= window) {
            const int* slot = ring + (int)(req % window) * ring_stride;
            const int cnt = slot[0];
            for (int k = tid; k < cnt; k += NT) occ[slot[1 + k]] -= 1;   // distinct GPUs: no collisions
        }
        if (tid == 0) flag[1] = 0;
        __syncthreads();
        for (int g = tid; g < ng; g += NT) {
            const int o = occ[g];
            if (o < 0 || o >= R.occpow_len) {
                flag[1] = o < 0 ? SS_OCC_UNDERFLOW : SS_BAD_INPUT;
                flag[2] = g;
            }
            const int oc = o < 0 ? 0 : (o >= R.occpow_len ? R.occpow_len - 1 : o);
            tau[g] = base[g] * (oc < A.pow_len ? pw[oc] : R.occpow[oc]);
        }
        __syncthreads();
        if (flag[1]) {
            status = flag[1];
            aux = flag[2];
            break;
        }
        mark(0);
        // ---- DP over the layer columns + final argmin / backtrack ------------------
        double v;
        if constexpr (LPD > 0)
            v = pad_route<LPD, SPL, NWD>(E, pdst, node, cl, nblk, tau, costs, bp, picks, path, D.max_layers, &vshare,
                                         ishare, tid);
        else if constexpr (NWD == 1) v = warp_route<MAT>(E, node, cl, noff, eoff, nblk, tau, costs, bp, picks, lane, A.mat_pitch);
        else v = mw_route<NWD, SPL, MAT>(E, node, cl, noff, eoff, nblk, tau, costs, bp, picks, &vshare, tid, A.mat_pitch);
        mark(1);
        if (tid == 0 && R.out.cost) R.out.cost[(int64_t)dag * n_req + r] = v;
        if (!(v <= DBL_MAX)) {
            status = SS_NO_PATH;
            break;
        }
        __syncthreads();
        // ---- load update: +1 per distinct GPU of the chain, ring, outputs ---------
        const int tag = (int)(req & 0x3fffffff) + 1;
        int* slot = window > 0 ? ring + (int)(req % window) * ring_stride : nullptr;
        uint64_t h = 0;
        int cnt = 0;
        if (warp == 0) {
        for (int l0c = 0; l0c < nl; l0c += 32) {
            const int l = l0c + lane;
            int g = 0;
            bool first = false;
            if (l < nl) {
                g = node[noff[l] + picks[l]];
                h += ss_splitmix64(((uint64_t)l << 32) | (uint64_t)g);
                if (R.out.gpus) R.out.gpus[((int64_t)dag * n_req + r) * D.max_layers + l] = (int16_t)g;
                first = atomicExch(&stamp[g], tag) != tag && window != 0;
            }
            const unsigned m = __ballot_sync(FULL, first);
            if (first) {
                occ[g] += 1;
                if (slot) slot[1 + cnt + __popc(m & ((1u << lane) - 1u))] = g;
            }
            cnt += __popc(m);
        }
        if (R.out.chain_hash) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(FULL, h, o);
            if (lane == 0) R.out.chain_hash[(int64_t)dag * n_req + r] = h;
        }
        if (lane == 0 && slot) slot[0] = cnt;
        }
        __syncthreads();
        ++done;
    }
    __syncthreads();
    mark(2);
    if (R.prof && tid == 0)
        for (int k = 0; k < 3; ++k) atomicAdd(&R.prof[k], pacc[k]);
    for (int g = tid; g < ng; g += NT) R.st.occ[gbase + g] = occ[g];
    for (int q = tid; q < A.ring_len; q += NT) ring_g[q] = ring[q];
    if (tid == 0) {
        R.st.next_req[dag] = req0 + done;
        if (status != SS_OK) { R.st.status[dag] = status; R.st.aux[dag] = aux; }
    }
}

// ---------------------------------------------------------------------------
// Admission path (sim.py:319-366) on the step schedule of tests/golden/make_admission_golden.py:
// at step t the chains admitted at step t - W complete (release + release_kv), request t joins the
// queue, and the queue drains strictly FIFO -- the head is routed with every GPU whose KV headroom
// (ram_token_capacity - reserved) is below its tokens excluded (+inf latency: the same chain as
// removing it from the columns), reserves its tokens on the chain's distinct GPUs, and the drain stops
// at the first head without a finite chain.  Strict FIFO admits in arrival order, so request i's
// admission record lives at index i.
// ---------------------------------------------------------------------------
struct AdmissionArgs {
    const int32_t* gpu_ptr;
    const double* base_tau;
    const int64_t* token_cap;
    const double* occpow;
    int32_t occpow_len;
    const int64_t* seeds;
    int32_t tok_lo, tok_hi, steps, window;
    int32_t* adm_gpus;
    int32_t* step_out;
    double* cost_out;
    int16_t* gpus_out;
    int64_t* kv_out;
    int32_t* occ_out;
    int32_t* status;
    int32_t* aux;
    const double* mat;          // matrix mode (A.mat_dim > 0): per-scenario RTT matrices
};

__device__ __forceinline__ long long request_tokens(uint64_t mix, int i, int lo, int hi) {
    return (long long)lo +
           (long long)(ss_splitmix64(mix ^ (0x70ull << 40) ^ (uint64_t)i) % (uint64_t)(hi - lo + 1));
}

// NWD as in replay_warp_kernel: the chain DP of every admission attempt spreads its destinations over NWD warps
template <int NWD, int SPL, bool MAT = false>
__global__ void __launch_bounds__(NWD * 32) admission_warp_kernel(ss_dag_set D, WarpLayout A, AdmissionArgs Q) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int NT = NWD * 32;
    const int dag = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ double vshare;
    __shared__ int flag[3];
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    const int l0 = D.layer_ptr[dag];
    const int nl = D.layer_ptr[dag + 1] - l0;
    const int nblk = nl - 1;
    double* E = reinterpret_cast<double*>(smem + A.off_E);
    int* node = reinterpret_cast<int*>(smem + A.off_node);
    int* cl = reinterpret_cast<int*>(smem + A.off_cl);
    int* noff = reinterpret_cast<int*>(smem + A.off_noff);
    int* eoff = reinterpret_cast<int*>(smem + A.off_eoff);
    uint8_t* bp = smem + A.off_bp;
    int* picks = reinterpret_cast<int*>(smem + A.off_picks);
    double* tau = reinterpret_cast<double*>(smem + A.off_tau);
    double* base = reinterpret_cast<double*>(smem + A.off_base);
    int* occ = reinterpret_cast<int*>(smem + A.off_occ);
    int* stamp = reinterpret_cast<int*>(smem + A.off_stamp);
    double* pw = reinterpret_cast<double*>(smem + A.off_pow);
    double* costs = reinterpret_cast<double*>(smem + A.off_cost);
    long long* kv = reinterpret_cast<long long*>(smem + A.off_kv);
    long long* tcap = reinterpret_cast<long long*>(smem + A.off_tcap);
    if (warp == 0)
        flag[0] = stage_dag(D, A, l0, nl, E, node, cl, noff, eoff, lane,
                            A.mat_dim ? Q.mat + (int64_t)dag * A.mat_dim * A.mat_dim : nullptr) ? 0 : 1;
    __syncthreads();
    if (flag[0]) {
        if (tid == 0) Q.status[dag] = SS_BAD_INPUT;
        return;
    }
    const int gbase = Q.gpu_ptr[dag];
    const int ng = Q.gpu_ptr[dag + 1] - gbase;
    for (int g = tid; g < ng; g += NT) {
        occ[g] = 0;
        kv[g] = 0;
        stamp[g] = 0;
        base[g] = Q.base_tau[gbase + g];
        tcap[g] = Q.token_cap[gbase + g];
    }
    for (int o = tid; o < A.pow_len; o += NT) pw[o] = Q.occpow[o];
    if (tid < 8) { costs[32 + tid] = INF; costs[72 + tid] = INF; }
    __syncthreads();
    const uint64_t mix = ss_splitmix64((uint64_t)Q.seeds[dag]);
    const int steps = Q.steps, W = Q.window;
    const int stride = D.max_layers + 1;
    int32_t* adm = Q.adm_gpus + (int64_t)dag * steps * stride;
    int32_t* step_out = Q.step_out + (int64_t)dag * steps;
    int head = 0, done_head = 0, status = SS_OK, aux = 0;
    for (int t = 0; t < steps && status == SS_OK; ++t) {
        // completions: admissions of step t - W, in admission order (sim.py:353-357)
        while (done_head < head && step_out[done_head] == t - W) {
            const int32_t* slot = adm + (int64_t)done_head * stride;
            const int cnt = slot[0];
            const long long tok = request_tokens(mix, done_head, Q.tok_lo, Q.tok_hi);
            for (int k = tid; k < cnt; k += NT) {
                occ[slot[1 + k]] -= 1;
                kv[slot[1 + k]] -= tok;
            }
            __syncthreads();
            ++done_head;
        }
        // request t arrived: drain the queue [head, t] strictly FIFO (sim.py:345-351, 361-366)
        while (head <= t) {
            const long long tok = request_tokens(mix, head, Q.tok_lo, Q.tok_hi);
            if (tid == 0) flag[1] = 0;
            __syncthreads();
            for (int g = tid; g < ng; g += NT) {
                const int o = occ[g];
                if (o >= Q.occpow_len) { flag[1] = SS_BAD_INPUT; flag[2] = g; }
                const int oc = o >= Q.occpow_len ? Q.occpow_len - 1 : o;
                const double live = base[g] * (oc < A.pow_len ? pw[oc] : Q.occpow[oc]);
                tau[g] = tcap[g] - kv[g] < tok ? INF : live;      // KV-blocked GPUs are excluded (sim.py:321-325)
            }
            __syncthreads();
            if (flag[1]) {
                status = flag[1];
                aux = flag[2];
                break;
            }
            double v;
            if constexpr (NWD == 1) v = warp_route<MAT>(E, node, cl, noff, eoff, nblk, tau, costs, bp, picks, lane, A.mat_pitch);
            else v = mw_route<NWD, SPL, MAT>(E, node, cl, noff, eoff, nblk, tau, costs, bp, picks, &vshare, tid, A.mat_pitch);
            if (!(v <= DBL_MAX)) break;                          // UncoveredLayer / NoPath: the head waits
            __syncthreads();
            // admit: reserve the tokens and +1 occupancy on the chain's distinct GPUs (sim.py:330-331)
            int32_t* slot = adm + (int64_t)head * stride;
            const int tag = head + 1;
            int cnt = 0;
            if (warp == 0) {
            for (int c0 = 0; c0 < nl; c0 += 32) {
                const int l = c0 + lane;
                int g = 0;
                bool first = false;
                if (l < nl) {
                    g = node[noff[l] + picks[l]];
                    if (Q.gpus_out) Q.gpus_out[((int64_t)dag * steps + head) * D.max_layers + l] = (int16_t)g;
                    first = atomicExch(&stamp[g], tag) != tag;
                }
                const unsigned m = __ballot_sync(FULL, first);
                if (first) {
                    occ[g] += 1;
                    kv[g] += tok;
                    slot[1 + cnt + __popc(m & ((1u << lane) - 1u))] = g;
                }
                cnt += __popc(m);
            }
            if (lane == 0) {
                slot[0] = cnt;
                step_out[head] = t;
                Q.cost_out[(int64_t)dag * steps + head] = v;
            }
            }
            __syncthreads();
            ++head;
        }
    }
    __syncthreads();
    for (int i = head + tid; i < steps; i += NT) {               // still queued at the end
        step_out[i] = -1;
        Q.cost_out[(int64_t)dag * steps + i] = INF;
    }
    for (int g = tid; g < ng; g += NT) {
        Q.kv_out[gbase + g] = kv[g];
        Q.occ_out[gbase + g] = occ[g];
    }
    if (tid == 0) {
        Q.status[dag] = status;
        Q.aux[dag] = aux;
    }
}

}  // namespace

// Latency path (a batch that fits on the SMs, 9..32 hosts, edge-block mode): pad_route with LPD lanes per
// destination over padded edge blocks.  Returns LPD (1, 2, 4) or 0 for mw_route.  Env SS_WARP_ROUTE=mw|pad1|pad2|pad4.
static int warp_pad_lpd(const ss_dag_set& D, bool mat) {
    if (D.max_hosts <= 8 || D.max_hosts > 32 || mat) return 0;
    int lpd = D.n_dags <= sm_count() ? 2 : 0;
    if (const char* e = getenv("SS_WARP_ROUTE")) {
        if (e[0] == 'm') lpd = 0;
        else if (e[0] == 'p') lpd = atoi(e + 3);
    }
    return (lpd == 1 || lpd == 2 || lpd == 4) ? lpd : 0;
}

// padded width P = LPD * HS for the instantiated shapes (HS rounded up), 0 if none fits
static int warp_pad_width(int lpd, int hosts) {
    static const int hs1[] = {12, 18, 24, 32}, hs2[] = {6, 9, 12, 16}, hs4[] = {3, 5, 6, 8};
    const int* hs = lpd == 1 ? hs1 : (lpd == 2 ? hs2 : hs4);
    for (int k = 0; k < 4; ++k)
        if (lpd * hs[k] >= hosts) return lpd * hs[k];
    return 0;
}

extern "C" int64_t ss_replay_warp_smem(const ss_dag_set* dags, int32_t window, int32_t occpow_len, int32_t mat_dim) {
    if (!dags) return -1;
    WarpLayout A{};
    return warp_layout(*dags, window, occpow_len < 1 ? 1 : occpow_len, A, mat_dim) ? A.total : -1;
}

extern "C" int ss_replay_warp(const ss_dag_set* dags, const ss_replay_state* st, const double* occpow,
                              int32_t occpow_len, int32_t window, int32_t n_req, const ss_replay_out* out,
                              const double* mat, int32_t mat_dim, void* stream_h) {
    if (!dags || !st || !occpow || occpow_len < 1 || n_req < 1) return SS_BAD_INPUT;
    const ss_dag_set& D = *dags;
    if (D.n_dags <= 0) return SS_OK;
    if (!D.edge_val || !D.edge_off) return SS_BAD_INPUT;
    WarpLayout A{};
    if (!warp_layout(D, window, occpow_len, A, mat ? mat_dim : 0)) return SS_BAD_INPUT;
    int lpd = warp_pad_lpd(D, A.mat_dim > 0);
    if (lpd > 0) {
        WarpLayout Ap{};
        if (warp_layout(D, window, occpow_len, Ap, 0, warp_pad_width(lpd, D.max_hosts))) A = Ap;
        else lpd = 0;                                            // padded blocks do not fit: mw_route
    }
    WarpReplay R{};
    R.mat = mat;
    R.st = *st;
    if (out) R.out = *out;
    R.occpow = occpow;
    R.occpow_len = occpow_len;
    R.window = window;
    R.n_req = n_req;
    cudaStream_t s = ss_stream(stream_h);
    if (getenv("SS_WARP_PROF") && cudaMalloc(&R.prof, 4 * sizeof(unsigned long long)) == cudaSuccess)
        cudaMemsetAsync(R.prof, 0, 4 * sizeof(unsigned long long), s);
    // One CTA per scenario.  An earlier split of each column's SOURCES over warps (partials merged through
    // shared memory) measured slower at C2 (27e3 vs 33e3 sel/s); splitting the DESTINATIONS (mw_route) keeps
    // every merge inside a warp and only adds the boundary barrier.
    auto run = [&](auto kern, int threads) -> int {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, A.total) != cudaSuccess)
            return SS_CUDA_ERROR;
        kern<<<D.n_dags, threads, A.total, s>>>(D, A, R);
        return SS_OK;
    };
    int rc;
    const bool mm = A.mat_dim > 0;                               // matrix mode: separate instantiations
    if (lpd > 0) {
        const int P = A.pad;
        if (lpd == 1) {
            if (P == 12) rc = run(replay_warp_kernel<1, 12, false, 1>, 32);
            else if (P == 18) rc = run(replay_warp_kernel<1, 18, false, 1>, 32);
            else if (P == 24) rc = run(replay_warp_kernel<1, 24, false, 1>, 32);
            else rc = run(replay_warp_kernel<1, 32, false, 1>, 32);
        } else if (lpd == 2) {
            if (P == 12) rc = run(replay_warp_kernel<1, 6, false, 2>, 32);
            else if (P == 18) rc = run(replay_warp_kernel<2, 9, false, 2>, 64);
            else if (P == 24) rc = run(replay_warp_kernel<2, 12, false, 2>, 64);
            else rc = run(replay_warp_kernel<2, 16, false, 2>, 64);
        } else {
            if (P == 12) rc = run(replay_warp_kernel<2, 3, false, 4>, 64);
            else if (P == 20) rc = run(replay_warp_kernel<3, 5, false, 4>, 96);
            else if (P == 24) rc = run(replay_warp_kernel<3, 6, false, 4>, 96);
            else rc = run(replay_warp_kernel<4, 8, false, 4>, 128);
        }
    } else {
    // destinations per boundary over ceil(hosts / 8) warps (C2's 17 hosts -> 3 warps)
    switch ((D.max_hosts + 3) / 4) {                             // source slots per lane
        case 0: case 1: case 2: rc = mm ? run(replay_warp_kernel<1, 8, true>, 32) : run(replay_warp_kernel<1, 8>, 32); break;
        case 3: rc = mm ? run(replay_warp_kernel<2, 3, true>, 64) : run(replay_warp_kernel<2, 3>, 64); break;
        case 4: rc = mm ? run(replay_warp_kernel<2, 4, true>, 64) : run(replay_warp_kernel<2, 4>, 64); break;
        case 5: rc = mm ? run(replay_warp_kernel<3, 5, true>, 96) : run(replay_warp_kernel<3, 5>, 96); break;
        case 6: rc = mm ? run(replay_warp_kernel<3, 6, true>, 96) : run(replay_warp_kernel<3, 6>, 96); break;
        case 7: rc = mm ? run(replay_warp_kernel<4, 7, true>, 128) : run(replay_warp_kernel<4, 7>, 128); break;
        default: rc = mm ? run(replay_warp_kernel<4, 8, true>, 128) : run(replay_warp_kernel<4, 8>, 128); break;
    }
    }
    if (rc != SS_OK) return rc;
    SS_CHECK_LAUNCH();
    if (R.prof) {
        unsigned long long h[4];
        cudaMemcpyAsync(h, R.prof, sizeof(h), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        const double d = (double)D.n_dags * n_req;
        fprintf(stderr, "warp prof: cycles per request: release+tau %.0f  DP %.0f  argmin+update %.0f\n", h[0] / d,
                h[1] / d, h[2] / d);
        cudaFree(R.prof);
    }
    return SS_OK;
}

extern "C" int ss_admission_warp(const ss_dag_set* dags, const int32_t* gpu_ptr, const double* base_tau,
                                 const int64_t* token_cap, const double* occpow, int32_t occpow_len,
                                 const int64_t* seeds, int32_t tok_lo, int32_t tok_hi, int32_t steps, int32_t window,
                                 int32_t* adm_gpus, int32_t* step_out, double* cost_out, int16_t* gpus_out,
                                 int64_t* kv_out, int32_t* occ_out, int32_t* status, int32_t* aux,
                                 const double* mat, int32_t mat_dim, void* stream_h) {
    if (!dags || !gpu_ptr || !base_tau || !token_cap || !occpow || occpow_len < 1 || !seeds || !adm_gpus ||
        !step_out || !cost_out || !kv_out || !occ_out || !status || !aux)
        return SS_BAD_INPUT;
    if (steps < 1 || window < 1 || tok_lo < 0 || tok_hi < tok_lo) return SS_BAD_INPUT;
    const ss_dag_set& D = *dags;
    if (D.n_dags <= 0) return SS_OK;
    if (!D.edge_val || !D.edge_off) return SS_BAD_INPUT;
    WarpLayout A{};
    if (!warp_layout(D, 0, occpow_len, A, mat ? mat_dim : 0)) return SS_BAD_INPUT;
    AdmissionArgs Q{gpu_ptr, base_tau, token_cap, occpow, occpow_len, seeds, tok_lo, tok_hi, steps, window,
                    adm_gpus, step_out, cost_out, gpus_out, kv_out, occ_out, status, aux, mat};
    cudaStream_t s = ss_stream(stream_h);
    auto run = [&](auto kern, int threads) -> int {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, A.total) != cudaSuccess)
            return SS_CUDA_ERROR;
        kern<<<D.n_dags, threads, A.total, s>>>(D, A, Q);
        return SS_OK;
    };
    int rc;
    const bool mm = A.mat_dim > 0;                               // matrix mode: separate instantiations
    switch ((D.max_hosts + 3) / 4) {                             // source slots per lane
        case 0: case 1: case 2: rc = mm ? run(admission_warp_kernel<1, 8, true>, 32) : run(admission_warp_kernel<1, 8>, 32); break;
        case 3: rc = mm ? run(admission_warp_kernel<2, 3, true>, 64) : run(admission_warp_kernel<2, 3>, 64); break;
        case 4: rc = mm ? run(admission_warp_kernel<2, 4, true>, 64) : run(admission_warp_kernel<2, 4>, 64); break;
        case 5: rc = mm ? run(admission_warp_kernel<3, 5, true>, 96) : run(admission_warp_kernel<3, 5>, 96); break;
        case 6: rc = mm ? run(admission_warp_kernel<3, 6, true>, 96) : run(admission_warp_kernel<3, 6>, 96); break;
        case 7: rc = mm ? run(admission_warp_kernel<4, 7, true>, 128) : run(admission_warp_kernel<4, 7>, 128); break;
        default: rc = mm ? run(admission_warp_kernel<4, 8, true>, 128) : run(admission_warp_kernel<4, 8>, 128); break;
    }
    if (rc != SS_OK) return rc;
    SS_CHECK_LAUNCH();
    return SS_OK;
}
