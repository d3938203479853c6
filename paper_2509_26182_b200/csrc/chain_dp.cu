// Batched Phase-2 chain DP for sm_100a.
//
// Reference arithmetic (router.py:163-185):
//   cost_1 = tau(col_1)
//   for l = 2..L:  cand[i,j] = cost[i] + E[i,j];  bp[j] = first argmin_i cand[i,j]
//                  cost[j]   = cand[bp[j], j] + tau(col_l[j])
//   final = first argmin cost; NoPath when not finite; backtrack bp.
// Every value is one IEEE fp64 add in the same association, and the argmin
// is reproduced as a lexicographic (value, source index) minimum, which is
// order-independent -- so the reduction can be split across warps freely and
// still return numpy's first-occurrence index.
//
// Layout / data movement (HBM-bound, no tensor cores: nothing here is a
// contraction):
//   * one CTA (8 warps) owns one DAG / scenario for all of its requests, so a
//     scenario's edge blocks stream through the same SM;
//   * edge blocks live in HBM row-major (row = source host), and are streamed
//     into shared memory with 1-D TMA bulk copies (cp.async.bulk, SASS
//     UBLKCP) completing on mbarriers, NBUF tiles in flight;
//   * inside a tile, lane j of every warp owns destinations j, j+32, ... so
//     each warp reads whole contiguous row segments (conflict-free LDS.64) and
//     the source cost is a shared-memory broadcast; warps split the source
//     rows, and a per-destination lexicographic combine across the 8 warps
//     finishes the column;
//   * replay keeps occupancy, tau(g) and the backpointers in shared memory;
//     the load update after each selection is a parallel distinct-gpu pass
//     (atomicExch stamps), the release of chain i-W reads a per-scenario ring.
#include <float.h>

#include "ss_common.cuh"

namespace {

constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int IDX_NONE = 0x7fffffff;

int g_smem_budget = 110 * 1024;  // per CTA: two CTAs per SM
int g_nbuf = 3;

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
    int nbuf;
    int tile_bytes;   // capacity of one buffer (multiple of 128)
    int rmaxp;        // padded max hosts (32 * D)
    int lmax;         // max layers
    int gmax;         // max gpus (replay)
    // byte offsets inside dynamic smem
    int off_bar, off_cost, off_pv, off_pi, off_bp, off_picks, off_tau, off_occ, off_stamp, off_misc, total;
};

__host__ __device__ inline int align_up(int x, int a) { return (x + a - 1) / a * a; }

Tiling make_tiling(const ss_dag_set& D, bool replay, int D_per_lane) {
    Tiling t{};
    t.rmaxp = 32 * D_per_lane;
    t.lmax = D.max_layers;
    t.gmax = replay ? D.max_gpus : 0;
    int fixed = 0;
    t.off_bar = 0;  // after tiles; filled below
    int bytes = 0;
    bytes += 8 * 8;                                   // up to 8 barriers
    const int cost = 2 * t.rmaxp * 8;
    const int pv = NW * t.rmaxp * 8;
    const int pi = NW * t.rmaxp * 4;
    const int bp = align_up(t.lmax * t.rmaxp, 16);
    const int picks = align_up(t.lmax * 4, 16);
    const int tau = t.gmax * 8, occ = t.gmax * 4, stamp = t.gmax * 4;
    fixed = bytes + cost + pv + pi + bp + picks + tau + occ + stamp + 64;
    int nbuf = g_nbuf;
    int budget = g_smem_budget;
    // largest edge block of the set bounds a useful tile
    const int max_block = t.rmaxp * t.rmaxp * 8 + 32;
    int tile = (budget - fixed) / nbuf;
    tile = tile / 128 * 128;
    if (tile > align_up(max_block, 128)) tile = align_up(max_block, 128);
    const int min_tile = align_up(2 * 256 * 8 + 64, 128);
    if (tile < min_tile) tile = min_tile;
    t.nbuf = nbuf;
    t.tile_bytes = tile;
    int o = nbuf * tile;
    t.off_bar = o;   o += 8 * 8;
    t.off_cost = o;  o += cost;
    t.off_pv = o;    o += pv;
    t.off_pi = o;    o += pi;
    t.off_bp = o;    o += bp;
    t.off_picks = o; o += picks;
    t.off_tau = o;   o += tau;
    t.off_occ = o;   o += occ;
    t.off_stamp = o; o += stamp;
    t.off_misc = o;  o += 64;
    t.total = o;
    return t;
}

// Tile geometry of block `blk` (layer blk -> blk+1) of one DAG.
struct TileGeom {
    const double* src;   // 16-B aligned global source
    uint32_t bytes;      // multiple of 16
    int row0, nrows, shift;
};

__device__ __forceinline__ int rows_per_tile(int rd, int tile_bytes) {
    int r = (tile_bytes - 32) / (rd * 8);
    return r < 1 ? 1 : r;
}

__device__ __forceinline__ int tiles_of_block(int rs, int rd, int tile_bytes) {
    const int rpt = rows_per_tile(rd, tile_bytes);
    return (rs + rpt - 1) / rpt;
}

__device__ __forceinline__ TileGeom tile_geom(const ss_dag_set& D, int fl, int tile, int tile_bytes) {
    const int rs = D.col_len[fl], rd = D.col_len[fl + 1];
    const int rpt = rows_per_tile(rd, tile_bytes);
    TileGeom g;
    g.row0 = tile * rpt;
    g.nrows = min(rpt, rs - g.row0);
    const int64_t start = D.edge_off[fl] + (int64_t)g.row0 * rd;      // in doubles
    const int64_t end = start + (int64_t)g.nrows * rd;
    const int64_t a0 = start & ~(int64_t)1;                            // 16-B aligned
    const int64_t a1 = (end + 1) & ~(int64_t)1;
    g.src = D.edge_val + a0;
    g.bytes = (uint32_t)((a1 - a0) * 8);
    g.shift = (int)(start - a0);
    return g;
}

// Producer cursor over (request, block, tile) -- owned by thread 0.
struct Cursor {
    int req, blk, tile;
};

__device__ __forceinline__ void cursor_next(Cursor& c, const ss_dag_set& D, int l0, int nl, int tile_bytes) {
    const int fl = l0 + c.blk;
    if (c.tile + 1 < tiles_of_block(D.col_len[fl], D.col_len[fl + 1], tile_bytes)) {
        c.tile++;
        return;
    }
    c.tile = 0;
    if (c.blk + 1 < nl - 1) {
        c.blk++;
        return;
    }
    c.blk = 0;
    c.req++;
}

template <int DPL, bool REPLAY>
__global__ void __launch_bounds__(NT, 2)
chain_dp_kernel(ss_dag_set D, Tiling T, ReplayArgs R, SelectArgs S) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int dag = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int l0 = D.layer_ptr[dag];
    const int nl = D.layer_ptr[dag + 1] - l0;

    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + T.off_bar);
    double* cost_a = reinterpret_cast<double*>(smem + T.off_cost);
    double* cost_b = cost_a + T.rmaxp;
    double* pv = reinterpret_cast<double*>(smem + T.off_pv);
    int* pi = reinterpret_cast<int*>(smem + T.off_pi);
    uint8_t* bp = smem + T.off_bp;
    int* picks = reinterpret_cast<int*>(smem + T.off_picks);
    double* tau_g = reinterpret_cast<double*>(smem + T.off_tau);
    int* occ_s = reinterpret_cast<int*>(smem + T.off_occ);
    int* stamp = reinterpret_cast<int*>(smem + T.off_stamp);
    int* misc = reinterpret_cast<int*>(smem + T.off_misc);   // [0] status [1] aux [2] ring count [3] final

    // ---- validate the DAG (all columns non-empty and within limits) --------
    if (tid == 0) {
        misc[0] = SS_OK;
        misc[1] = 0;
        if (REPLAY && R.st.status[dag] != SS_OK) misc[0] = -1;   // sticky failure: skip
        if (nl < 1 || nl > T.lmax) misc[0] = SS_BAD_INPUT;
    }
    __syncthreads();
    if (misc[0] == SS_OK) {
        for (int l = tid; l < nl; l += NT) {
            const int len = D.col_len[l0 + l];
            if (len == 0) atomicExch(&misc[0], SS_UNCOVERED_LAYER);
            if (len > T.rmaxp) atomicExch(&misc[0], SS_BAD_INPUT);
        }
    }
    __syncthreads();
    if (misc[0] == SS_UNCOVERED_LAYER && tid == 0) {
        int first = 0;
        for (int l = 0; l < nl; ++l)
            if (D.col_len[l0 + l] == 0) { first = l + 1; break; }
        misc[1] = first;
    }
    __syncthreads();
    if (misc[0] != SS_OK) {
        if (tid == 0 && misc[0] != -1) {
            if (REPLAY) { R.st.status[dag] = misc[0]; R.st.aux[dag] = misc[1]; }
            else { S.status_out[dag] = misc[0]; S.cost_out[dag] = __longlong_as_double(0x7ff8000000000000ll); }
        }
        return;
    }

    // ---- replay state in shared memory -------------------------------------
    int gbase = 0, ng = 0, window = 0, n_req = 1;
    int64_t req0 = 0;
    int* ring = nullptr;
    const int ring_stride = T.lmax + 1;
    if constexpr (REPLAY) {
        gbase = R.st.gpu_ptr[dag];
        ng = R.st.gpu_ptr[dag + 1] - gbase;
        window = R.window;
        n_req = R.n_req;
        req0 = R.st.next_req[dag];
        ring = R.st.ring + (int64_t)dag * (window > 0 ? window : 1) * ring_stride;
        for (int g = tid; g < ng; g += NT) {
            occ_s[g] = R.st.occ[gbase + g];
            stamp[g] = 0;
        }
    }

    // ---- TMA bulk-copy pipeline --------------------------------------------
    const int nblk = nl - 1;
    int tiles_per_req = 0;
    if (tid == 0) {
        for (int b = 0; b < nblk; ++b)
            tiles_per_req += tiles_of_block(D.col_len[l0 + b], D.col_len[l0 + b + 1], T.tile_bytes);
        for (int b = 0; b < T.nbuf; ++b) mbar_init(&bars[b], 1);
        fence_mbar_init();
    }
    __syncthreads();
    const int64_t total_tiles = (int64_t)tiles_per_req * n_req;   // valid in thread 0 only
    Cursor pc{0, 0, 0};
    int64_t issued = 0;
    auto issue = [&](int buf) {
        const TileGeom g = tile_geom(D, l0 + pc.blk, pc.tile, T.tile_bytes);
        unsigned char* dst = smem + (size_t)buf * T.tile_bytes;
        fence_proxy_async_smem();
        mbar_expect_tx(&bars[buf], g.bytes);
        bulk_g2s(dst, g.src, g.bytes, &bars[buf]);
        cursor_next(pc, D, l0, nl, T.tile_bytes);
        ++issued;
    };
    if (tid == 0 && nblk > 0) {
        for (int b = 0; b < T.nbuf && issued < total_tiles; ++b) issue(b);
    }
    int64_t consumed = 0;   // tiles consumed (identical in every thread)

    double* cur = cost_a;
    double* nxt = cost_b;
    int done = 0;   // requests fully routed in this launch

    for (int r = 0; r < n_req; ++r) {
        const int64_t req = req0 + r;
        // ---- release chain req-W, refresh tau(g) -------------------------
        if constexpr (REPLAY) {
            if (window > 0 && req >= window) {
                const int* slot = ring + (int64_t)(req % window) * ring_stride;
                const int cnt = slot[0];
                for (int k = tid; k < cnt; k += NT) {
                    const int g = slot[1 + k];
                    occ_s[g] -= 1;     // distinct gpus: no two threads share g
                }
            }
            __syncthreads();
            for (int g = tid; g < ng; g += NT) {
                const int o = occ_s[g];
                if (o < 0 || o >= R.occpow_len) { atomicExch(&misc[0], o < 0 ? SS_OCC_UNDERFLOW : SS_BAD_INPUT); misc[1] = g; }
                tau_g[g] = R.st.base_tau[gbase + g] * R.occpow[o < 0 ? 0 : (o >= R.occpow_len ? R.occpow_len - 1 : o)];
            }
            if (tid == 0) misc[2] = 0;
            __syncthreads();
            if (misc[0] != SS_OK) break;
        }
        // ---- layer 1 costs -------------------------------------------------
        {
            const int off = D.col_off[l0], len = D.col_len[l0];
            for (int j = tid; j < len; j += NT) {
                if constexpr (REPLAY) cur[j] = tau_g[D.node_gpu[off + j]];
                else cur[j] = D.node_tau[off + j];
            }
        }
        __syncthreads();

        // ---- relax boundary by boundary ------------------------------------
        for (int b = 0; b < nblk; ++b) {
            const int fl = l0 + b;
            const int rs = D.col_len[fl], rd = D.col_len[fl + 1];
            const int ntile = tiles_of_block(rs, rd, T.tile_bytes);
            double bv[DPL];
            int bi[DPL];
#pragma unroll
            for (int q = 0; q < DPL; ++q) { bv[q] = __longlong_as_double(0x7ff0000000000000ll); bi[q] = IDX_NONE; }

            for (int t = 0; t < ntile; ++t) {
                const int buf = (int)(consumed % T.nbuf);
                const uint32_t parity = (uint32_t)((consumed / T.nbuf) & 1);
                const TileGeom g = tile_geom(D, fl, t, T.tile_bytes);
                mbar_wait(&bars[buf], parity);
                const double* tile = reinterpret_cast<const double*>(smem + (size_t)buf * T.tile_bytes) + g.shift;
#pragma unroll 2
                for (int ii = warp; ii < g.nrows; ii += NW) {
                    const int i = g.row0 + ii;
                    const double c = cur[i];
                    const double* row = tile + ii * rd;
#pragma unroll
                    for (int q = 0; q < DPL; ++q) {
                        const int j = lane + 32 * q;
                        if (j < rd) {
                            const double v = __dadd_rn(c, row[j]);
                            if (v < bv[q]) { bv[q] = v; bi[q] = i; }
                        }
                    }
                }
                ++consumed;
                if (t + 1 < ntile) {
                    __syncthreads();                 // buffer free
                    if (tid == 0 && issued < total_tiles) issue(buf);
                }
            }
            // partials of this warp
#pragma unroll
            for (int q = 0; q < DPL; ++q) {
                const int j = lane + 32 * q;
                if (j < rd) { pv[warp * T.rmaxp + j] = bv[q]; pi[warp * T.rmaxp + j] = bi[q]; }
            }
            __syncthreads();                         // partials visible, last buffer free
            if (tid == 0 && issued < total_tiles) issue((int)((consumed - 1) % T.nbuf));
            const int noff = D.col_off[fl + 1];
            for (int j = tid; j < rd; j += NT) {
                double v = pv[j];
                int idx = pi[j];
#pragma unroll
                for (int w = 1; w < NW; ++w) {
                    const double v2 = pv[w * T.rmaxp + j];
                    const int i2 = pi[w * T.rmaxp + j];
                    if (v2 < v || (v2 == v && i2 < idx)) { v = v2; idx = i2; }
                }
                if (idx == IDX_NONE) idx = 0;          // all-inf column: numpy argmin -> 0
                double tau_j;
                if constexpr (REPLAY) tau_j = tau_g[D.node_gpu[noff + j]];
                else tau_j = D.node_tau[noff + j];
                nxt[j] = __dadd_rn(v, tau_j);
                bp[b * T.rmaxp + j] = (uint8_t)idx;
            }
            __syncthreads();
            double* tmp = cur; cur = nxt; nxt = tmp;
        }

        // ---- final argmin + backtrack ---------------------------------------
        if (warp == 0) {
            const int len = D.col_len[l0 + nl - 1];
            double v = __longlong_as_double(0x7ff0000000000000ll);
            int idx = IDX_NONE;
            for (int j = lane; j < len; j += 32) {
                const double c = cur[j];
                if (c < v) { v = c; idx = j; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
                const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
                if (v2 < v || (v2 == v && i2 < idx)) { v = v2; idx = i2; }
            }
            if (lane == 0) {
                if (!(v <= DBL_MAX)) {               // inf (or nan): no finite chain
                    misc[0] = SS_NO_PATH;
                    misc[3] = 0;
                } else {
                    int p = idx;
                    picks[nl - 1] = p;
                    for (int b = nblk - 1; b >= 0; --b) {
                        p = bp[b * T.rmaxp + p];
                        picks[b] = p;
                    }
                }
                if constexpr (REPLAY) {
                    const int64_t o = (int64_t)dag * n_req + r;
                    if (R.out.cost) R.out.cost[o] = v;
                } else {
                    S.cost_out[dag] = v;
                }
            }
        }
        __syncthreads();
        if (misc[0] != SS_OK) break;

        if constexpr (!REPLAY) {
            for (int l = tid; l < nl; l += NT) S.pick_out[l0 + l] = picks[l];
        } else {
            // ---- load update: +1 per distinct gpu, ring bookkeeping, outputs --
            const int tag = (int)(req & 0x3fffffff) + 1;
            int* slot = window > 0 ? ring + (int64_t)(req % window) * ring_stride : nullptr;
            uint64_t h = 0;
            for (int l = tid; l < nl; l += NT) {
                const int g = D.node_gpu[D.col_off[l0 + l] + picks[l]];
                h += ss_splitmix64(((uint64_t)l << 32) | (uint64_t)g);
                if (R.out.gpus) R.out.gpus[((int64_t)dag * n_req + r) * T.lmax + l] = (int16_t)g;
                if (atomicExch(&stamp[g], tag) != tag && window != 0) {
                    occ_s[g] += 1;
                    if (slot) slot[1 + atomicAdd(&misc[2], 1)] = g;
                }
            }
            if (R.out.chain_hash) {
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
                if (lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&R.out.chain_hash[(int64_t)dag * n_req + r]),
                                         (unsigned long long)h);
            }
            __syncthreads();
            if (tid == 0 && slot) slot[0] = misc[2];
            __syncthreads();   // ring slot complete before a W=1 release reads it
        }
        ++done;
    }

    // drain any tile still in flight (only when a failure broke the loop)
    if (tid == 0) {
        while (consumed < issued) {
            const int buf = (int)(consumed % T.nbuf);
            mbar_wait(&bars[buf], (uint32_t)((consumed / T.nbuf) & 1));
            ++consumed;
        }
    }
    __syncthreads();
    if constexpr (REPLAY) {
        for (int g = tid; g < ng; g += NT) R.st.occ[gbase + g] = occ_s[g];
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
    const int dpl = D.max_hosts <= 32 ? 1 : D.max_hosts <= 64 ? 2 : D.max_hosts <= 96 ? 3 : D.max_hosts <= 128 ? 4 : 8;
    Tiling T = make_tiling(D, REPLAY, dpl);
    if (T.total > 227 * 1024) return SS_BAD_INPUT;
    auto run = [&](auto kern) -> int {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, T.total) != cudaSuccess)
            return SS_CUDA_ERROR;
        kern<<<D.n_dags, NT, T.total, stream>>>(D, T, R, S);
        SS_CHECK_LAUNCH();
        return SS_OK;
    };
    switch (dpl) {
        case 1: return run(chain_dp_kernel<1, REPLAY>);
        case 2: return run(chain_dp_kernel<2, REPLAY>);
        case 3: return run(chain_dp_kernel<3, REPLAY>);
        case 4: return run(chain_dp_kernel<4, REPLAY>);
        default: return run(chain_dp_kernel<8, REPLAY>);
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
    if (R.out.chain_hash) cudaMemsetAsync(R.out.chain_hash, 0, sizeof(uint64_t) * (size_t)dags->n_dags * n_req, ss_stream(stream));
    return launch<true>(*dags, R, S, ss_stream(stream));
}

extern "C" int ss_set_tiling(int32_t smem_budget_bytes, int32_t n_buffers, int32_t* old_budget_h, int32_t* old_buffers_h) {
    if (old_budget_h) *old_budget_h = g_smem_budget;
    if (old_buffers_h) *old_buffers_h = g_nbuf;
    if (smem_budget_bytes > 0) g_smem_budget = smem_budget_bytes;
    if (n_buffers > 0) g_nbuf = n_buffers > 8 ? 8 : n_buffers;
    return SS_OK;
}
