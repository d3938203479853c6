// Batched Phase-2 chain DP for sm_100a.
//
// Reference arithmetic (router.py:163-185):
//   cost_1 = tau(col_1)
//   for l = 2..L:  cand[i,j] = cost[i] + E[i,j];  bp[j] = first argmin_i cand[i,j]
//                  cost[j]   = cand[bp[j], j] + tau(col_l[j])
//   final = first argmin cost; NoPath when not finite; backtrack bp.
// Every value is one IEEE fp64 add in the same association, and the argmin is
// reproduced as a lexicographic (value, source index) minimum, which is
// order-independent -- so sources can be split over independent chains and
// still yield numpy's first-occurrence index.
//
// Warp-specialised pipeline, one CTA per DAG / scenario (it owns the scenario
// for all of its requests, so the replay's sequential dependence stays on-SM):
//   * producer warp: streams the scenario's edge blocks (row-major, row =
//     source host) HBM -> shared memory with 1-D TMA bulk copies
//     (cp.async.bulk, SASS UBLKCP) into NBUF tiles, full/empty mbarriers;
//     edge blocks do not depend on costs, so it runs ahead across layer and
//     request boundaries;
//   * CW consumer warps: warp w owns destinations 32w..32w+31 of every block
//     and scans ALL source rows (conflict-free LDS.64 row segments, source
//     cost as an LDS.128 broadcast) into 4 independent min-chains for ILP;
//     no cross-warp combine, one named barrier per layer boundary;
//   * replay state (occupancy, tau(g), backpointers, chain picks) lives in
//     shared memory; the load update after each selection is a parallel
//     distinct-gpu pass (atomicExch stamps); release of chain i-W reads a
//     per-scenario ring of distinct gpus.
#include <float.h>

#include "ss_common.cuh"

namespace {

constexpr int IDX_NONE = 0x7fffffff;
constexpr int CONSUMER_BAR = 1;   // named barrier id for consumer warps

int g_smem_budget = 56 * 1024;    // per CTA: four CTAs per SM for CW = 3
int g_nbuf = 4;

struct ReplayArgs {
    ss_replay_state st;
    ss_replay_out out;
    const double* occpow;
    int32_t occpow_len;
    int32_t window;
    int32_t n_req;
};

struct SelectArgs {
    int32_t* pick_out;
    double* cost_out;
    int32_t* status_out;
};

struct Tiling {
    int nbuf, tile_bytes, rmaxp, lmax, gmax;
    int off_full, off_empty, off_cost, off_bp, off_picks, off_blk, off_boff, off_tau, off_occ, off_stamp,
        off_misc, off_red, off_part, total;
};

inline int align_up(int x, int a) { return (x + a - 1) / a * a; }

Tiling make_tiling(const ss_dag_set& D, bool replay, int cw, int sg = 1) {
    // A batch that cannot fill the GPU (one drop-in select_chain / route: a single DAG) gets one CTA per SM
    // anyway, so it takes most of the SM's shared memory as TMA ring: more edge bytes in flight per boundary.
    const bool small = D.n_dags <= 64;
    const int budget = small ? 200 * 1024 : g_smem_budget;
    Tiling t{};
    t.rmaxp = 32 * cw;
    t.lmax = D.max_layers;
    t.gmax = replay ? D.max_gpus : 0;
    const int fixed = 2 * 8 * 8 /*bars*/ + 2 * t.rmaxp * 8 + align_up(t.lmax * t.rmaxp, 16) +
                      align_up(t.lmax * 4, 16) + align_up(t.lmax * 16, 16) + align_up(t.lmax * 8, 16) +
                      t.gmax * 16 + 64 + cw * 16 + 256 + (sg > 1 ? sg * t.rmaxp * 12 + 16 : 0);
    const int nbuf = small ? 8 : g_nbuf;
    int tile = (budget - fixed) / nbuf / 128 * 128;
    const int max_block = align_up(t.rmaxp * t.rmaxp * 8 + 32, 128);
    if (tile > max_block) tile = max_block;
    const int min_tile = align_up(4 * t.rmaxp * 8 + 32, 128);     // at least 4 rows of the widest block
    if (tile < min_tile) tile = min_tile;
    t.nbuf = nbuf;
    t.tile_bytes = tile;
    int o = nbuf * tile;
    t.off_full = o;  o += 8 * 8;
    t.off_empty = o; o += 8 * 8;
    t.off_cost = o;  o += 2 * t.rmaxp * 8;
    t.off_boff = o;  o += align_up(t.lmax * 8, 16);
    t.off_blk = o;   o += align_up(t.lmax * 16, 16);
    t.off_bp = o;    o += align_up(t.lmax * t.rmaxp, 16);
    t.off_picks = o; o += align_up(t.lmax * 4, 16);
    t.off_tau = o;   o += t.gmax * 8;
    t.off_occ = o;   o += t.gmax * 4;
    t.off_stamp = o; o += t.gmax * 4;
    t.off_red = o;   o += align_up(cw * 16, 16);
    t.off_misc = o;  o += 64;
    t.off_part = o;  o += sg > 1 ? align_up(sg * t.rmaxp * 12, 16) : 0;
    t.total = o;
    return t;
}

// per-block geometry cached in shared memory: rs, rd, rows per tile, tiles
struct Blk {
    int rs, rd, rpt, ntile;
};

__device__ __forceinline__ void consumer_sync(int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"n"(CONSUMER_BAR), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void lex_min(double& v, int& i, double v2, int i2) {
    if (v2 < v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

// SG > 1 (batches too small to fill the GPU: one DAG per SM, e.g. a drop-in select_chain / route): every
// destination group is served by SG warps, each scanning every SG-th group of four source rows; their
// (value, row) partials meet in shared memory and merge lexicographically (order-free) behind the boundary
// barrier -- SG times less serial work per warp on the single-DAG latency path.
template <int CW, bool REPLAY, int SG = 1>
__global__ void __launch_bounds__((CW * SG + 1) * 32)
chain_dp_kernel(ss_dag_set D, Tiling T, ReplayArgs R, SelectArgs S) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int NC = CW * SG * 32;            // consumer threads
    const int dag = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int l0 = D.layer_ptr[dag];
    const int nl = D.layer_ptr[dag + 1] - l0;
    const int nblk = nl - 1;

    uint64_t* full = reinterpret_cast<uint64_t*>(smem + T.off_full);
    uint64_t* empty = reinterpret_cast<uint64_t*>(smem + T.off_empty);
    double* cost_a = reinterpret_cast<double*>(smem + T.off_cost);
    double* cost_b = cost_a + T.rmaxp;
    int64_t* boff = reinterpret_cast<int64_t*>(smem + T.off_boff);
    Blk* blk = reinterpret_cast<Blk*>(smem + T.off_blk);
    uint8_t* bp = smem + T.off_bp;
    int* picks = reinterpret_cast<int*>(smem + T.off_picks);
    double* tau_g = reinterpret_cast<double*>(smem + T.off_tau);
    int* occ_s = reinterpret_cast<int*>(smem + T.off_occ);
    int* stamp = reinterpret_cast<int*>(smem + T.off_stamp);
    double* red_v = reinterpret_cast<double*>(smem + T.off_red);
    int* red_i = reinterpret_cast<int*>(smem + T.off_red + CW * 8);
    volatile int* misc = reinterpret_cast<int*>(smem + T.off_misc);   // [0] status [1] aux [2] ring count [3] tiles/request

    // ---- setup: validation, block geometry, barriers (whole CTA) --------------
    if (tid == 0) {
        misc[0] = SS_OK;
        misc[1] = 0;
        if (REPLAY && R.st.status[dag] != SS_OK) misc[0] = -1;   // sticky failure: skip
        if (nl < 1 || nl > T.lmax) misc[0] = SS_BAD_INPUT;
        for (int b = 0; b < T.nbuf; ++b) {
            mbar_init(&full[b], 1);
            mbar_init(&empty[b], CW * SG);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (misc[0] == SS_OK) {
        for (int l = tid; l < nl; l += blockDim.x) {
            const int len = D.col_len[l0 + l];
            if (len == 0) atomicExch((int*)&misc[0], SS_UNCOVERED_LAYER);
            if (len > T.rmaxp) atomicExch((int*)&misc[0], SS_BAD_INPUT);
            if (l < nblk) {
                const int rd = D.col_len[l0 + l + 1];
                Blk bk;
                bk.rs = len;
                bk.rd = rd;
                int rpt = rd > 0 ? (T.tile_bytes - 32) / (rd * 8) : 1;
                rpt = rpt >= 4 ? (rpt & ~3) : (rpt < 1 ? 1 : rpt);
                bk.rpt = rpt;
                bk.ntile = (len + rpt - 1) / rpt;
                blk[l] = bk;
                boff[l] = D.edge_off[l0 + l];
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        if (misc[0] == SS_UNCOVERED_LAYER) {
            for (int l = 0; l < nl; ++l)
                if (D.col_len[l0 + l] == 0) { misc[1] = l + 1; break; }
        }
        int tiles = 0;
        if (misc[0] == SS_OK)
            for (int b = 0; b < nblk; ++b) tiles += blk[b].ntile;
        misc[3] = tiles;
    }
    __syncthreads();
    if (misc[0] != SS_OK) {
        if (tid == 0 && misc[0] != -1) {
            if (REPLAY) { R.st.status[dag] = misc[0]; R.st.aux[dag] = misc[1]; }
            else { S.status_out[dag] = misc[0]; S.cost_out[dag] = __longlong_as_double(0x7ff8000000000000ll); }
        }
        return;
    }
    const int n_req = REPLAY ? R.n_req : 1;

    // =========================================================================
    // producer warp
    // =========================================================================
    if (warp == CW * SG) {
        if (lane == 0 && nblk > 0) {
            int64_t n = 0;
            for (int r = 0; r < n_req; ++r) {
                for (int b = 0; b < nblk; ++b) {
                    const Blk bk = blk[b];
                    for (int t = 0; t < bk.ntile; ++t, ++n) {
                        const int buf = (int)(n % T.nbuf);
                        const int use = (int)(n / T.nbuf);
                        if (use > 0) mbar_wait(&empty[buf], (uint32_t)((use - 1) & 1));
                        const int row0 = t * bk.rpt;
                        const int nr = min(bk.rpt, bk.rs - row0);
                        const int64_t start = boff[b] + (int64_t)row0 * bk.rd;
                        const int64_t a0 = start & ~(int64_t)1;
                        const int64_t a1 = (start + (int64_t)nr * bk.rd + 1) & ~(int64_t)1;
                        const uint32_t bytes = (uint32_t)((a1 - a0) * 8);
                        fence_proxy_async_smem();
                        mbar_expect_tx(&full[buf], bytes);
                        bulk_g2s(smem + (size_t)buf * T.tile_bytes, D.edge_val + a0, bytes, &full[buf]);
                    }
                }
            }
        }
        return;
    }

    // =========================================================================
    // consumer warps
    // =========================================================================
    int gbase = 0, ng = 0, window = 0;
    int64_t req0 = 0;
    int* ring = nullptr;
    const int ring_stride = T.lmax + 1;
    if constexpr (REPLAY) {
        gbase = R.st.gpu_ptr[dag];
        ng = R.st.gpu_ptr[dag + 1] - gbase;
        window = R.window;
        req0 = R.st.next_req[dag];
        ring = R.st.ring + (int64_t)dag * (window > 0 ? window : 1) * ring_stride;
        for (int g = tid; g < ng; g += NC) {
            occ_s[g] = R.st.occ[gbase + g];
            stamp[g] = 0;
        }
    }
    const int dgrp = warp % CW, sgrp = warp / CW;
    const int j = dgrp * 32 + lane;          // destination owned by this lane
    double* part_v = reinterpret_cast<double*>(smem + T.off_part);          // [SG][rmaxp] source-group partials
    int* part_i = reinterpret_cast<int*>(part_v + SG * T.rmaxp);
    int64_t consumed = 0;
    // after a failure the producer still issues every tile: acknowledge them all so
    // no bulk copy is in flight into this CTA's shared memory when it exits
    auto drain = [&]() {
        const int64_t total = (int64_t)n_req * misc[3];
        for (; consumed < total; ++consumed) {
            const int buf = (int)(consumed % T.nbuf);
            mbar_wait(&full[buf], (uint32_t)((consumed / T.nbuf) & 1));
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[buf]);
        }
    };
    double* cur = cost_a;
    double* nxt = cost_b;
    int done = 0;
    consumer_sync(NC);

    for (int r = 0; r < n_req; ++r) {
        const int64_t req = req0 + r;
        // ---- release chain req-W, refresh tau(g) ---------------------------
        if constexpr (REPLAY) {
            if (window > 0 && req >= window) {
                const int* slot = ring + (int64_t)(req % window) * ring_stride;
                const int cnt = slot[0];
                for (int k = tid; k < cnt; k += NC) occ_s[slot[1 + k]] -= 1;   // distinct gpus
            }
            consumer_sync(NC);
            for (int g = tid; g < ng; g += NC) {
                const int o = occ_s[g];
                if (o < 0 || o >= R.occpow_len) {
                    atomicExch((int*)&misc[0], o < 0 ? SS_OCC_UNDERFLOW : SS_BAD_INPUT);
                    misc[1] = g;
                }
                tau_g[g] = R.st.base_tau[gbase + g] * R.occpow[o < 0 ? 0 : (o >= R.occpow_len ? R.occpow_len - 1 : o)];
            }
            if (tid == 0) misc[2] = 0;
            consumer_sync(NC);
            if (misc[0] != SS_OK) { drain(); break; }
        }
        // ---- layer 1 -----------------------------------------------------------
        {
            const int off = D.col_off[l0], len = D.col_len[l0];
            for (int q = tid; q < len; q += NC) {
                if constexpr (REPLAY) cur[q] = tau_g[D.node_gpu[off + q]];
                else cur[q] = D.node_tau[off + q];
            }
        }
        consumer_sync(NC);

        // ---- boundaries ----------------------------------------------------------
        for (int b = 0; b < nblk; ++b) {
            const Blk bk = blk[b];
            const bool active = j < bk.rd;
            // tau of this lane's destination: issue the gather early, use after the scan
            int g_dst = 0;
            double tau_dst = 0.0;
            if (active) {
                if constexpr (REPLAY) g_dst = D.node_gpu[D.col_off[l0 + b + 1] + j];
                else tau_dst = D.node_tau[D.col_off[l0 + b + 1] + j];
            }
            double v0 = __longlong_as_double(0x7ff0000000000000ll), v1 = v0, v2 = v0, v3 = v0;
            int i0 = IDX_NONE, i1 = IDX_NONE, i2 = IDX_NONE, i3 = IDX_NONE;
            const int64_t base_start = boff[b];
            for (int t = 0; t < bk.ntile; ++t, ++consumed) {
                const int buf = (int)(consumed % T.nbuf);
                mbar_wait(&full[buf], (uint32_t)((consumed / T.nbuf) & 1));
                const int row0 = t * bk.rpt;
                const int nr = min(bk.rpt, bk.rs - row0);
                const int shift = (int)((base_start + (int64_t)row0 * bk.rd) & 1);
                const double* tile = reinterpret_cast<const double*>(smem + (size_t)buf * T.tile_bytes) + shift + j;
                if (active) {
                    int q = 4 * sgrp;
                    // rows in groups of 4 -> four independent (value, index) chains; SG > 1: every SG-th group
                    for (; q + 4 <= nr; q += 4 * SG) {
                        const int i = row0 + q;                       // multiple of 4: 16-B aligned pairs
                        const double2 c01 = *reinterpret_cast<const double2*>(cur + i);
                        const double2 c23 = *reinterpret_cast<const double2*>(cur + i + 2);
                        const double c0 = c01.x, c1 = c01.y, c2 = c23.x, c3 = c23.y;
                        const double e0 = tile[(q + 0) * bk.rd], e1 = tile[(q + 1) * bk.rd];
                        const double e2 = tile[(q + 2) * bk.rd], e3 = tile[(q + 3) * bk.rd];
                        const double a0 = __dadd_rn(c0, e0), a1 = __dadd_rn(c1, e1);
                        const double a2 = __dadd_rn(c2, e2), a3 = __dadd_rn(c3, e3);
                        if (a0 < v0) { v0 = a0; i0 = i; }
                        if (a1 < v1) { v1 = a1; i1 = i + 1; }
                        if (a2 < v2) { v2 = a2; i2 = i + 2; }
                        if (a3 < v3) { v3 = a3; i3 = i + 3; }
                    }
                    if (q < nr)                              // the tail group (< 4 rows) belongs to its group's warp
                        for (; q < nr; ++q) {
                            const int i = row0 + q;
                            const double a = __dadd_rn(cur[i], tile[q * bk.rd]);
                            if (a < v0) { v0 = a; i0 = i; }
                        }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[buf]);
            }
            if (active) {
                // chains hold ascending rows each; merge lexicographically (first index on ties)
                lex_min(v0, i0, v1, i1);
                lex_min(v0, i0, v2, i2);
                lex_min(v0, i0, v3, i3);
            }
            if constexpr (SG > 1) {
                if (active) { part_v[sgrp * T.rmaxp + j] = v0; part_i[sgrp * T.rmaxp + j] = i0; }
                consumer_sync(NC);
                if (sgrp == 0 && active)
#pragma unroll
                    for (int g = 1; g < SG; ++g) lex_min(v0, i0, part_v[g * T.rmaxp + j], part_i[g * T.rmaxp + j]);
            }
            if (active && sgrp == 0) {
                if (i0 == IDX_NONE) i0 = 0;                 // all-inf column: numpy argmin -> 0
                if constexpr (REPLAY) tau_dst = tau_g[g_dst];
                nxt[j] = __dadd_rn(v0, tau_dst);
                bp[b * T.rmaxp + j] = (uint8_t)i0;
            }
            consumer_sync(NC);
            double* tmp = cur; cur = nxt; nxt = tmp;
        }

        // ---- final argmin (per warp, then across warps) + backtrack -------------
        {
            const int len = D.col_len[l0 + nl - 1];
            double v = __longlong_as_double(0x7ff0000000000000ll);
            int idx = IDX_NONE;
            if (j < len && sgrp == 0) { v = cur[j]; idx = j; }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
                const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
                lex_min(v, idx, v2, i2);
            }
            if (lane == 0 && sgrp == 0) { red_v[dgrp] = v; red_i[dgrp] = idx; }
        }
        consumer_sync(NC);
        if (tid == 0) {
            double v = red_v[0];
            int idx = red_i[0];
            for (int w = 1; w < CW; ++w) lex_min(v, idx, red_v[w], red_i[w]);
            if (!(v <= DBL_MAX)) {                          // inf: no finite chain
                misc[0] = SS_NO_PATH;
            } else {
                int p = idx;
                picks[nl - 1] = p;
                for (int b = nblk - 1; b >= 0; --b) {
                    p = bp[b * T.rmaxp + p];
                    picks[b] = p;
                }
            }
            if constexpr (REPLAY) {
                if (R.out.cost) R.out.cost[(int64_t)dag * n_req + r] = v;
            } else {
                S.cost_out[dag] = v;
            }
        }
        consumer_sync(NC);
        if (misc[0] != SS_OK) { drain(); break; }

        if constexpr (!REPLAY) {
            for (int l = tid; l < nl; l += NC) S.pick_out[l0 + l] = picks[l];
        } else {
            // ---- load update: +1 per distinct gpu, ring bookkeeping, outputs -----
            const int tag = (int)(req & 0x3fffffff) + 1;
            int* slot = window > 0 ? ring + (int64_t)(req % window) * ring_stride : nullptr;
            uint64_t h = 0;
            for (int l = tid; l < nl; l += NC) {
                const int g = D.node_gpu[D.col_off[l0 + l] + picks[l]];
                h += ss_splitmix64(((uint64_t)l << 32) | (uint64_t)g);
                if (R.out.gpus) R.out.gpus[((int64_t)dag * n_req + r) * T.lmax + l] = (int16_t)g;
                if (atomicExch(&stamp[g], tag) != tag && window != 0) {
                    occ_s[g] += 1;
                    if (slot) slot[1 + atomicAdd((int*)&misc[2], 1)] = g;
                }
            }
            if (R.out.chain_hash) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
                if (lane == 0)
                    atomicAdd(reinterpret_cast<unsigned long long*>(&R.out.chain_hash[(int64_t)dag * n_req + r]),
                              (unsigned long long)h);
            }
            consumer_sync(NC);
            if (tid == 0 && slot) slot[0] = misc[2];
            consumer_sync(NC);   // ring slot complete before a W=1 release reads it
        }
        ++done;
    }

    if constexpr (REPLAY) {
        for (int g = tid; g < ng; g += NC) R.st.occ[gbase + g] = occ_s[g];
        if (tid == 0) {
            R.st.next_req[dag] = req0 + done;
            if (misc[0] != SS_OK) { R.st.status[dag] = misc[0]; R.st.aux[dag] = misc[1]; }
        }
    } else {
        if (tid == 0) S.status_out[dag] = misc[0];
    }
}

template <bool REPLAY>
int launch(const ss_dag_set& D, const ReplayArgs& R, const SelectArgs& S, cudaStream_t stream) {
    if (D.n_dags <= 0) return SS_OK;
    if (D.max_hosts < 1 || D.max_hosts > SS_MAX_HOSTS || D.max_layers < 1 || D.max_layers > SS_MAX_LAYERS)
        return SS_BAD_INPUT;
    if (REPLAY && (D.max_gpus < 1 || D.max_gpus > SS_MAX_GPUS)) return SS_BAD_INPUT;
    const int cw = (D.max_hosts + 31) / 32;
    // fewer DAGs than SMs: each DAG's CTA is alone on its SM, so split the sources over 4 warp groups
    const int sg = D.n_dags <= 64 && cw <= 4 ? 4 : 1;
    Tiling T = make_tiling(D, REPLAY, cw, sg);
    if (T.total > 227 * 1024) return SS_BAD_INPUT;
    auto run = [&](auto kern, int threads) -> int {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, T.total) != cudaSuccess)
            return SS_CUDA_ERROR;
        kern<<<D.n_dags, threads, T.total, stream>>>(D, T, R, S);
        SS_CHECK_LAUNCH();
        return SS_OK;
    };
    if (sg == 4) {
        switch (cw) {
            case 1: return run(chain_dp_kernel<1, REPLAY, 4>, 5 * 32);
            case 2: return run(chain_dp_kernel<2, REPLAY, 4>, 9 * 32);
            case 3: return run(chain_dp_kernel<3, REPLAY, 4>, 13 * 32);
            default: return run(chain_dp_kernel<4, REPLAY, 4>, 17 * 32);
        }
    }
    switch (cw) {
        case 1: return run(chain_dp_kernel<1, REPLAY>, 64);
        case 2: return run(chain_dp_kernel<2, REPLAY>, 96);
        case 3: return run(chain_dp_kernel<3, REPLAY>, 128);
        case 4: return run(chain_dp_kernel<4, REPLAY>, 160);
        case 5: return run(chain_dp_kernel<5, REPLAY>, 192);
        case 6: return run(chain_dp_kernel<6, REPLAY>, 224);
        case 7: return run(chain_dp_kernel<7, REPLAY>, 256);
        default: return run(chain_dp_kernel<8, REPLAY>, 288);
    }
}

}  // namespace

extern "C" int ss_select(const ss_dag_set* dags, int32_t* pick_out, double* cost_out, int32_t* status_out,
                         void* stream) {
    if (!dags || !pick_out || !cost_out || !status_out) return SS_BAD_INPUT;
    ReplayArgs R{};
    R.n_req = 1;
    SelectArgs S{pick_out, cost_out, status_out};
    if (!dags->node_tau) return SS_BAD_INPUT;
    return launch<false>(*dags, R, S, ss_stream(stream));
}

extern "C" int ss_replay(const ss_dag_set* dags, const ss_replay_state* st, const double* occpow, int32_t occpow_len,
                         int32_t window, int32_t n_req, const ss_replay_out* out, void* stream) {
    if (!dags || !st || !occpow || occpow_len < 1 || n_req < 1) return SS_BAD_INPUT;
    ReplayArgs R{};
    R.st = *st;
    if (out) R.out = *out;
    R.occpow = occpow;
    R.occpow_len = occpow_len;
    R.window = window;
    R.n_req = n_req;
    SelectArgs S{};
    if (R.out.chain_hash)
        cudaMemsetAsync(R.out.chain_hash, 0, sizeof(uint64_t) * (size_t)dags->n_dags * n_req, ss_stream(stream));
    return launch<true>(*dags, R, S, ss_stream(stream));
}

extern "C" int ss_set_tiling(int32_t smem_budget_bytes, int32_t n_buffers, int32_t* old_budget_h, int32_t* old_buffers_h) {
    if (old_budget_h) *old_budget_h = g_smem_budget;
    if (old_buffers_h) *old_buffers_h = g_nbuf;
    if (smem_budget_bytes > 0) g_smem_budget = smem_budget_bytes;
    if (n_buffers > 0) g_nbuf = n_buffers > 8 ? 8 : n_buffers;
    return SS_OK;
}
