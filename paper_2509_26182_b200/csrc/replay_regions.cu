// Region-tiled replay: Phase-2 replay for pools whose GPUs fall into regions with
// cheap links inside a region and expensive links between regions -- the reference bench pool
// (bench.py:114-138: intra-region links 1 ms, every other pair the 10 ms default_cross_region_rtt_s of
// topology.py:133-142) and the C5 pools (inter-region 5-80 ms).
//
// The DP of router.py:163-185 relaxes every (source, destination) pair of a boundary:
//     cand[i][j] = c_b[i] + E_b[i][j],  v_j = min_i cand[i][j] (first index),  c_{b+1}[j] = v_j + tau_j.
// Split the hosts of a boundary by region.  For a destination region D and a source region S != D:
//     every S candidate  >= fl(cmin_S + lb[S][D])           (lb: lower bound of the S x D entries)
//     every v_j (j in D) <= fl(cmin_D + ub[D])              (ub: upper bound of the D x D entries; the D source
//                                                           with cost cmin_D reaches every j in D)
// (fl is monotone, so the bounds survive rounding).  When fl(cmin_S + lb) > fl(cmin_D + ub), no S candidate
// reaches the minimum of any destination in D -- not even as a tie -- so skipping the S x D block leaves every
// v_j and every first-index argmin unchanged.  On C4 > 99% of the cross-region blocks are skipped this way, on
// C5 > 99.9% (measured with the oracle over 1,000-request steady states); the rest are relaxed exactly, with
// their entries recomputed from the pool matrix and the scenario jitter (the same IEEE product the other
// kernels stream).  Results are bit-identical to the dense DP for ANY input; only the work changes.
//
// Layout.  Each region ("tile") keeps a shared-memory RTT tile T_t[src slot][dst slot] over <= 32 slots,
// interval-partitioned per region exactly like replay_slots.cu (a GPU keeps one slot while it is in the frontier
// col_b U col_{b+1}; slots are reused one boundary late).  One consumer warp per tile, lane = destination slot:
// every lane owns complete destination minima (no cross-warp merge), and the relaxation is one LDS.64 + DADD +
// DSETP + 2 FSEL + SEL per (source, lane).  One producer warp streams the entering GPUs' row / column units
// with 1-D TMA bulk copies and writes them into the tiles while the consumers relax.  One named barrier per
// boundary publishes every tile's source costs and minimum (the bound test reads the other tiles' minima).
#include <float.h>
#include <stdio.h>
#include <stdlib.h>

#include "ss_common.cuh"

namespace {

#ifndef RG_UNROLL
#define RG_UNROLL 8                      // source pairs per unrolled step of the intra-tile relaxation
#endif
#ifndef RG_MINB_WIDE
#define RG_MINB_WIDE 3                   // CTAs per SM the register budget is sized for (5..8 tiles)
#endif
#ifndef RG_KB
#define RG_KB 4                          // kept cross-tile sources per round (<= 4 tiles)
#endif
#ifndef RG_KB_WIDE
#define RG_KB_WIDE 2                     // ... with 5-8 tiles (C5: +0.5-2% over 4; C4: 4 beats 2 and 8)
#endif

constexpr int RG_UNROLL_N = RG_UNROLL;

constexpr int RG_HDR = 16;
constexpr int RG_MAX_TILES = 8;
constexpr int RG_BAR_ALL = 3;          // consumers + producer
constexpr int RG_BAR_CONS = 4;         // consumers only
constexpr int RG_POS_NONE = 0xffff;

int g_rg_stage_bytes = 2 * 1024;
int g_rg_nbuf = 3;

// Per-scenario program (byte offsets):
//   hdr   : [0] RT (max local slots used by a tile) [1] Wp (unit length, even) [2] units [3] entries
//   blk   : per boundary {n_ins, ins_start, unit_start}
//   ins   : per entering GPU {tile * 32 + local slot, gpu}
//   pairs : per tile, per column, 32 entries {local slot | position << 8} of the tile's hosts in position
//           (sorted-id) order, 0xffff past the last -- read by the consumers straight from L1/L2
//   lbg   : per pool GPU g and tile t, a float rounded down <= every jittered g -> h entry with h in tile t, h != g
//           (the per-source bound of the cross-tile filter; staged in shared memory)
// The first three parts (up to off_pairs) are staged in shared memory by the replay kernel.
struct RgLayout {
    int n_blk, n_tiles, pos_cap, n_cap;
    __host__ __device__ int off_blk() const { return RG_HDR; }
    __host__ __device__ int off_ins() const { return RG_HDR + n_blk * 8; }
    __host__ __device__ int off_pairs() const { return (off_ins() + n_cap * 4 + 127) / 128 * 128; }
    __host__ __device__ int off_lbg() const { return (off_pairs() + n_tiles * (n_blk + 1) * 64 + 15) / 16 * 16; }
    __host__ __device__ int bytes() const { return (off_lbg() + n_cap * n_tiles * 4 + 127) / 128 * 128; }
};

constexpr uint16_t RG_PAIR_NONE = 0xffff;

struct RgBlk {
    int16_t n_ins, ins_start;
    int32_t unit_start;
};

// ---------------------------------------------------------------------------
// program generation: one CTA per scenario
// ---------------------------------------------------------------------------
__global__ void region_program_kernel(int32_t layers, int32_t n_gpus, const int32_t* lo, const int32_t* hi,
                                      int64_t slice_stride, const uint8_t* leave, const double* rtt,
                                      const int64_t* jitter_seed, const int32_t* tile_of, int32_t n_tiles,
                                      int32_t pos_cap, int64_t meta_stride, int64_t stream_stride, uint8_t* meta,
                                      double* stream, int32_t* rt_out, int32_t* status) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int s = blockIdx.x;
    const int n_blk = layers - 1;
    const int tslots = n_tiles * 32;
    const uint8_t* gone = leave ? leave + (int64_t)s * n_gpus : nullptr;
    lo += s * slice_stride;
    hi += s * slice_stride;
    RgLayout ml{n_blk, n_tiles, pos_cap, n_gpus};
    uint8_t* mt = meta + (int64_t)s * meta_stride;
    double* st = stream + (int64_t)s * stream_stride;
    int16_t* slot_of = reinterpret_cast<int16_t*>(sm);                                  // [n_gpus] tile*32+q
    int16_t* occ_tl = slot_of + ((n_gpus + 7) / 8) * 8;                                 // [n_blk][tslots]
    int* ins_head = reinterpret_cast<int*>(occ_tl + ((n_blk * tslots + 7) / 8) * 8);   // [n_blk + 2]
    int* free_head = ins_head + n_blk + 2;
    int* ins_next = free_head + n_blk + 2;                                              // [n_gpus]
    int* free_next = ins_next + n_gpus;
    __shared__ int bad, wp_s;
    const int tid = threadIdx.x;
    for (int i = tid; i < n_blk * tslots; i += blockDim.x) occ_tl[i] = -1;
    for (int g = tid; g < n_gpus; g += blockDim.x) slot_of[g] = -1;
    for (int b = tid; b < n_blk + 2; b += blockDim.x) { ins_head[b] = -1; free_head[b] = -1; }
    __syncthreads();
    if (tid == 0) {
        // GPU g is in the frontier col_b U col_{b+1} for boundaries [max(lo-2,0), hi-1]; its slot is held one
        // boundary longer (zombie) so the producer can write boundary b+1's units while b is relaxed
        for (int g = n_gpus - 1; g >= 0; --g) {
            if (hi[g] < lo[g] || hi[g] < 1 || (gone && gone[g])) continue;
            const int sb = lo[g] - 2 < 0 ? 0 : lo[g] - 2;
            if (sb >= n_blk) continue;
            ins_next[g] = ins_head[sb];
            ins_head[sb] = g;
            const int fb = hi[g] + 1;
            if (fb < n_blk) {
                free_next[g] = free_head[fb];
                free_head[fb] = g;
            }
        }
        bad = 0;
        int rt = 0;
        uint32_t freem[RG_MAX_TILES];
        for (int t = 0; t < RG_MAX_TILES; ++t) freem[t] = ~0u;
        RgBlk* bm = reinterpret_cast<RgBlk*>(mt + ml.off_blk());
        int16_t* ins = reinterpret_cast<int16_t*>(mt + ml.off_ins());
        int n_ins_total = 0, unit = 0;
        for (int b = 0; b < n_blk && !bad; ++b) {
            for (int g = free_head[b]; g >= 0; g = free_next[g]) {
                const int q = slot_of[g];
                if (q >= 0) freem[q >> 5] |= 1u << (q & 31);
            }
            const int start = n_ins_total;
            for (int g = ins_head[b]; g >= 0; g = ins_next[g]) {
                const int t = tile_of[g];
                if (t < 0 || t >= n_tiles || freem[t] == 0) { bad = 1; break; }
                const int q = __ffs(freem[t]) - 1;
                freem[t] &= ~(1u << q);
                slot_of[g] = (int16_t)(t * 32 + q);
                if (q + 1 > rt) rt = q + 1;
                ins[2 * n_ins_total] = (int16_t)(t * 32 + q);
                ins[2 * n_ins_total + 1] = (int16_t)g;
                ++n_ins_total;
            }
            RgBlk m;
            m.n_ins = (int16_t)(n_ins_total - start);
            m.ins_start = (int16_t)start;
            m.unit_start = unit;
            bm[b] = m;
            unit += (b == 0 ? 1 : 2) * (n_ins_total - start);
        }
        const int wp = (rt + 1) & ~1;
        wp_s = wp;
        int32_t* hdr = reinterpret_cast<int32_t*>(mt);
        hdr[0] = rt;
        hdr[1] = wp;
        hdr[2] = unit;
        hdr[3] = n_ins_total;
        if ((int64_t)unit * wp > stream_stride) bad = 2;
        status[s] = bad ? SS_BAD_INPUT : SS_OK;
        rt_out[s] = bad ? 0 : rt;
    }
    __syncthreads();
    if (bad) return;
    for (int g = tid; g < n_gpus; g += blockDim.x) {
        const int q = slot_of[g];
        if (q < 0) continue;
        const int sb = lo[g] - 2 < 0 ? 0 : lo[g] - 2;
        const int eb = hi[g] < n_blk - 1 ? hi[g] : n_blk - 1;
        for (int b = sb; b <= eb; ++b) occ_tl[b * tslots + q] = (int16_t)g;
    }
    __syncthreads();
    // per column: the hosts of every tile in position (sorted-id) order, with their global positions
    uint16_t* pairs = reinterpret_cast<uint16_t*>(mt + ml.off_pairs());
    for (int i = tid; i < n_tiles * (n_blk + 1) * 32; i += blockDim.x) pairs[i] = RG_PAIR_NONE;
    __syncthreads();
    const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    for (int c = warp; c <= n_blk; c += nw) {
        int tcount[RG_MAX_TILES];
        for (int t = 0; t < RG_MAX_TILES; ++t) tcount[t] = 0;
        int pos = 0;
        for (int g0 = 0; g0 < n_gpus; g0 += 32) {
            const int g = g0 + lane;
            const bool in_col = g < n_gpus && !(gone && gone[g]) && lo[g] <= c + 1 && hi[g] >= c + 1;
            const unsigned ms = __ballot_sync(0xffffffffu, in_col);
            const int t = in_col ? tile_of[g] : -1;
            for (int u = 0; u < n_tiles; ++u) {
                const unsigned mu = __ballot_sync(0xffffffffu, t == u);
                if (t == u) {
                    const int k = tcount[u] + __popc(mu & ((1u << lane) - 1u));
                    const int p = pos + __popc(ms & ((1u << lane) - 1u));
                    if (k < 32 && p < pos_cap)
                        pairs[(u * (n_blk + 1) + c) * 32 + k] = (uint16_t)((slot_of[g] & 31) | (p << 8));
                    else
                        atomicExch(&status[s], SS_BAD_INPUT);
                }
                tcount[u] += __popc(mu);
            }
            pos += __popc(ms);
        }
    }
    // stream units: rows (b == 0) or row / column pairs over the entering GPU's tile
    const RgBlk* bm = reinterpret_cast<const RgBlk*>(mt + ml.off_blk());
    const int16_t* ins = reinterpret_cast<const int16_t*>(mt + ml.off_ins());
    const bool jit = jitter_seed != nullptr;
    const uint64_t mix = jit ? ss_splitmix64((uint64_t)jitter_seed[s]) : 0;
    const int64_t dim = n_gpus;
    const int wp = wp_s;
    for (int b = 0; b < n_blk; ++b) {
        const RgBlk m = bm[b];
        const int units = (b == 0 ? 1 : 2) * m.n_ins;
        for (int e = tid; e < units * wp; e += blockDim.x) {
            const int u = e / wp, t = e - u * wp;
            const int k = b == 0 ? u : (u >> 1);
            const bool col = b != 0 && (u & 1);
            const int code = ins[2 * (m.ins_start + k)];
            const int g = ins[2 * (m.ins_start + k) + 1];
            const int o = t < 32 ? occ_tl[b * tslots + (code & ~31) + t] : -1;
            double v = __longlong_as_double(0x7ff0000000000000ll);
            if (o >= 0) {
                const int a = col ? o : g, c = col ? g : o;
                v = rtt[(int64_t)a * dim + c];
                if (jit) v = v * ss_jitter(mix, (uint32_t)a, (uint32_t)c);
            }
            st[(int64_t)(m.unit_start + u) * wp + t] = v;
        }
    }
    // per-source cross-tile bounds: min over the pool GPUs h of tile t of the jittered g -> h entry, rounded down
    float* lbg = reinterpret_cast<float*>(mt + ml.off_lbg());
    for (int e = tid; e < n_gpus * n_tiles; e += blockDim.x) {
        const int g = e / n_tiles, t = e - g * n_tiles;
        double lo_v = __longlong_as_double(0x7ff0000000000000ll);
        for (int h = 0; h < n_gpus; ++h) {
            if (h == g || tile_of[h] != t) continue;
            double v = rtt[(int64_t)g * dim + h];
            if (jit) v = v * ss_jitter(mix, (uint32_t)g, (uint32_t)h);
            lo_v = v < lo_v ? v : lo_v;
        }
        lbg[e] = __double2float_rd(lo_v);
    }
}

// ---------------------------------------------------------------------------
// replay kernel
// ---------------------------------------------------------------------------
struct RgArgs {
    const uint8_t* meta;
    int64_t meta_stride;
    const double* stream;
    int64_t stream_stride;
    const double* bounds;        // lb[n_tiles][n_tiles], ub[n_tiles], uni[n_tiles][n_tiles]
    const double* base_rtt;      // [n_gpus][n_gpus] pool matrix (cross-tile blocks that survive the bound test)
    const int64_t* jitter_seed;  // [n_dags] or NULL
    int pos_cap, rt, tp, nbuf, stage_bytes;
    int off_T, off_stage, off_bar, off_meta, meta_smem, off_cw, off_rw, off_cmin, off_bp, off_picks, off_tau,
        off_occ, off_stamp, off_slotgpu, off_cl, off_coff, off_red, off_misc, off_pow, pow_len, off_rel, off_seg,
        off_bnd, off_jq, off_lbg, total;
    int use_lbg;                 // 1: per-source cross-tile bounds staged in shared memory (off_lbg)
    unsigned long long* cross;   // diagnostics (env SS_REGION_STATS=1): [0] blocks tested [1] blocks relaxed
};

struct RgReplayArgs {
    ss_replay_state st;
    ss_replay_out out;
    const double* occpow;
    int32_t occpow_len;
    int32_t window;
    int32_t n_req;
};

__device__ __forceinline__ void rg_bar_all(int n) { asm volatile("bar.sync %0, %1;" ::"n"(RG_BAR_ALL), "r"(n) : "memory"); }
__device__ __forceinline__ void rg_bar_cons(int n) { asm volatile("bar.sync %0, %1;" ::"n"(RG_BAR_CONS), "r"(n) : "memory"); }

__device__ __forceinline__ void rg_lex_min(double& v, int& i, double v2, int i2) {
    if (v2 < v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

__device__ __forceinline__ void rg_cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void rg_cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ int rg_ld_pair(const uint16_t* p) {
    unsigned short v;
    asm volatile("ld.global.nc.u16 %0, [%1];" : "=h"(v) : "l"(p));
    return (int)v;
}

// blockDim = (NTL + 1) * 32: warp t < NTL relaxes tile t's destinations, warp NTL streams and applies the entering
// GPUs' units.  Per boundary b, ONE named barrier over all warps:
//   consumers, before it: finish column b of their tile (v + tau, backpointers of boundary b-1) and publish its
//              sources' costs, row offsets and minimum bounds;
//   producer, before it : apply the units of the GPUs entering at b (rows + columns of the tiles; slots are
//              reused one boundary late, so nothing relaxed at b-1 is overwritten);
//   consumers, after it : relax boundary b inside the tile, then the cross-tile blocks the bound test keeps.
template <int NTL>
__global__ void __launch_bounds__((NTL + 1) * 32, NTL <= 4 ? 4 : RG_MINB_WIDE)
replay_regions_kernel(ss_dag_set D, RgArgs A, RgReplayArgs R) {
    extern __shared__ __align__(128) unsigned char smem[];
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    constexpr int NC = NTL * 32;
    constexpr int NT = NC + 32;
    const int dag = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int PC = A.pos_cap;
    const int RT = A.rt;
    const int TP = A.tp;                                      // tile row pitch (doubles, even)
    const int l0 = D.layer_ptr[dag];
    const int nl = D.layer_ptr[dag + 1] - l0;
    const int nblk = nl - 1;
    RgLayout ml{nblk, NTL, PC, D.max_gpus};

    double* T = reinterpret_cast<double*>(smem + A.off_T);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + A.off_bar);          // [nbuf]
    uint64_t* rows_bar = full + 8;
    unsigned char* meta_s = smem + A.off_meta;
    double* cw_all = reinterpret_cast<double*>(smem + A.off_cw);             // [2][NTL][32]
    int* rw_all = reinterpret_cast<int*>(smem + A.off_rw);                   // [2][NTL][32]
    double* cmin_all = reinterpret_cast<double*>(smem + A.off_cmin);         // [2][NTL] lower bounds
    uint8_t* bp = smem + A.off_bp;                                            // [nblk][PC]
    int* picks = reinterpret_cast<int*>(smem + A.off_picks);
    double* tau_g = reinterpret_cast<double*>(smem + A.off_tau);
    int* occ_s = reinterpret_cast<int*>(smem + A.off_occ);
    int* stamp = reinterpret_cast<int*>(smem + A.off_stamp);
    int* slot_gpu = reinterpret_cast<int*>(smem + A.off_slotgpu);            // [NTL][32]
    int* coff = reinterpret_cast<int*>(smem + A.off_coff);
    double* red_v = reinterpret_cast<double*>(smem + A.off_red);
    int* red_i = reinterpret_cast<int*>(smem + A.off_red + RG_MAX_TILES * 8);
    volatile int* misc = reinterpret_cast<int*>(smem + A.off_misc);          // [0] status [1] aux [2] ring [3] chunks
    double* pow_s = reinterpret_cast<double*>(smem + A.off_pow);
    int* rel = reinterpret_cast<int*>(smem + A.off_rel);
    uint8_t* seg_end = smem + A.off_seg;                                      // [NTL][PC]
    int* seg_start = reinterpret_cast<int*>(smem + A.off_seg + ((NTL * PC + 15) & ~15));
    double* lb_s = reinterpret_cast<double*>(smem + A.off_bnd);              // [NTL][NTL]
    double* ub_s = lb_s + NTL * NTL;                                          // [NTL]
    const double* uni_s = ub_s + NTL;                                         // [NTL][NTL] uniform S->D entry or NaN
    float* jq_s = reinterpret_cast<float*>(smem + A.off_jq);                  // [1024] jitter quantiles
    float* lbg_s = reinterpret_cast<float*>(smem + A.off_lbg);                // [n_gpus][NTL] per-source bounds

    // ---- setup ---------------------------------------------------------------
    const uint8_t* meta_g = A.meta + (int64_t)dag * A.meta_stride;
    if (tid == 0) {
        misc[0] = SS_OK;
        misc[1] = 0;
        if (R.st.status[dag] != SS_OK) misc[0] = -1;
        for (int b = 0; b < A.nbuf; ++b) mbar_init(&full[b], 1);
        mbar_init(rows_bar, 1);
        fence_mbar_init();
    }
    const int gbase = R.st.gpu_ptr[dag];
    const int ng = R.st.gpu_ptr[dag + 1] - gbase;
    {
        const int4* srcv = reinterpret_cast<const int4*>(meta_g);
        int4* dstv = reinterpret_cast<int4*>(meta_s);
        for (int q = tid; q < A.meta_smem / 16; q += NT) dstv[q] = srcv[q];
        for (int l = tid; l < nl; l += NT) coff[l] = D.col_off[l0 + l];
        for (int o = tid; o < A.pow_len; o += NT) pow_s[o] = R.occpow[o];
        for (int q = tid; q < 2 * NTL * NTL + NTL; q += NT) lb_s[q] = A.bounds[q];
        for (int q = tid; q < NTL * 32; q += NT) slot_gpu[q] = 0;
        const float* lbg_g = reinterpret_cast<const float*>(meta_g + ml.off_lbg());
        if (A.use_lbg)
            for (int q = tid; q < D.max_gpus * NTL; q += NT) lbg_s[q] = lbg_g[q];
        if (A.jitter_seed)
            for (int q = tid; q < 1024; q += NT) jq_s[q] = ss_jitter_q[q];
    }
    __syncthreads();
    const int32_t* hdr = reinterpret_cast<const int32_t*>(meta_s);
    const RgBlk* bm = reinterpret_cast<const RgBlk*>(meta_s + ml.off_blk());
    const int16_t* ins = reinterpret_cast<const int16_t*>(meta_s + ml.off_ins());
    const uint16_t* pairs_g = reinterpret_cast<const uint16_t*>(meta_g + ml.off_pairs());
    const int Wp = hdr[1];
    const int upc = max(2, (A.stage_bytes / (Wp * 8)) & ~1);   // units per chunk: whole (row, column) pairs
    const int tw = min(Wp, RT);                                // unit entries that land in a tile
    if (tid == 0 && misc[0] == SS_OK) {
        if (hdr[0] > RT || nl < 2) misc[0] = SS_BAD_INPUT;
        int chunks = 0;
        for (int b = 1; b < nblk; ++b) chunks += (2 * bm[b].n_ins + upc - 1) / upc;
        misc[3] = chunks;
    }
    __syncthreads();
    if (misc[0] != SS_OK) {
        if (tid == 0 && misc[0] != -1) { R.st.status[dag] = misc[0]; R.st.aux[dag] = misc[1]; }
        return;
    }
    const int n_req = R.n_req;
    const double* stream_g = A.stream + (int64_t)dag * A.stream_stride;

    // ========================= producer: TMA ring + apply(1..nblk-1) ===============
    if (warp == NTL) {
        const int64_t total = (int64_t)n_req * misc[3];
        int64_t issued = 0;
        int ib = 1, iu0 = 0;
        auto issue_next = [&](int buf) {
            while (ib < nblk && iu0 >= 2 * bm[ib].n_ins) { ++ib; iu0 = 0; }
            if (ib >= nblk) { ib = 1; iu0 = 0; while (ib < nblk && 2 * bm[ib].n_ins == 0) ++ib; }
            const RgBlk m = bm[ib];
            const int nu = min(upc, 2 * m.n_ins - iu0);
            const uint32_t bytes = (uint32_t)nu * Wp * 8;
            fence_proxy_async_smem();
            mbar_expect_tx(&full[buf], bytes);
            bulk_g2s(smem + A.off_stage + (size_t)buf * A.stage_bytes, stream_g + (int64_t)(m.unit_start + iu0) * Wp,
                     bytes, &full[buf]);
            iu0 += nu;
            ++issued;
        };
        int rows_issued = 0;
        auto issue_rows = [&]() {                            // boundary 0: rows straight into the tiles
            const RgBlk m = bm[0];
            const uint32_t ub = (uint32_t)Wp * 8;
            if (lane == 0) mbar_expect_tx(rows_bar, ub * (uint32_t)m.n_ins);
            __syncwarp();
            fence_proxy_async_smem();
            const double* s0 = stream_g + (int64_t)m.unit_start * Wp;
            for (int u = lane; u < m.n_ins; u += 32) {
                const int code = ins[2 * (m.ins_start + u)];
                bulk_g2s(T + ((code >> 5) * RT + (code & 31)) * TP, s0 + (int64_t)u * Wp, ub, rows_bar);
            }
            ++rows_issued;
        };
        if (n_req > 0) issue_rows();
        if (lane == 0)
            for (int b = 0; b < A.nbuf && issued < total; ++b) issue_next(b);
        int cbuf = 0;
        uint32_t cphase = 0;
        int64_t consumed = 0;
        const bool live = lane < tw;
        for (int r = 0; r < n_req; ++r) {
            rg_bar_all(NT);                                  // request start: tau ready, initial rows landed
            if (misc[0] != SS_OK) break;
            for (int b = 0; b < nblk; ++b) {
                if (b >= 1) {
                    const RgBlk m = bm[b];
                    const int units = 2 * m.n_ins;
                    for (int u0 = 0; u0 < units; u0 += upc) {
                        const int nu = min(upc, units - u0);
                        mbar_wait(&full[cbuf], cphase);
                        const double* stg = reinterpret_cast<const double*>(smem + A.off_stage +
                                                                            (size_t)cbuf * A.stage_bytes) + lane;
                        // unit pairs (row, column) of one entering GPU: T_t[q][lane] and T_t[lane][q]
                        for (int ul = 0; ul < nu; ul += 2) {
                            const int code = ins[2 * (m.ins_start + ((u0 + ul) >> 1))];
                            double* Tt = T + (code >> 5) * RT * TP;
                            const int q = code & 31;
                            const double xr = stg[ul * Wp];
                            const double xc = stg[(ul + 1) * Wp];
                            if (live) {
                                Tt[q * TP + lane] = xr;
                                Tt[lane * TP + q] = xc;
                            }
                        }
                        __syncwarp();
                        if (lane == 0 && issued < total) issue_next(cbuf);
                        ++consumed;
                        if (++cbuf == A.nbuf) { cbuf = 0; cphase ^= 1u; }
                    }
                    for (int k = lane; k < m.n_ins; k += 32)
                        slot_gpu[ins[2 * (m.ins_start + k)]] = ins[2 * (m.ins_start + k) + 1];
                }
                rg_bar_all(NT);                              // boundary b
            }
            rg_bar_all(NT);                                  // the last relaxation is done: T is free
            if (r + 1 < n_req) issue_rows();
        }
        if (rows_issued > 0) mbar_wait(rows_bar, (uint32_t)((rows_issued - 1) & 1));
        while (consumed < issued) {
            mbar_wait(&full[cbuf], cphase);
            ++consumed;
            if (++cbuf == A.nbuf) { cbuf = 0; cphase ^= 1u; }
        }
        return;
    }

    // ========================= consumers: warp = tile ==========================
    const int w = warp;
    const int window = R.window;
    const int64_t req0 = R.st.next_req[dag];
    const int ring_stride = D.max_layers + 1;
    int* ring = R.st.ring + (int64_t)dag * (window > 0 ? window : 1) * ring_stride;
    const int G = D.max_gpus;
    const uint64_t mix = A.jitter_seed ? ss_splitmix64((uint64_t)A.jitter_seed[dag]) : 0;
    for (int g = tid; g < ng; g += NC) {
        occ_s[g] = R.st.occ[gbase + g];
        stamp[g] = 0;
    }
    auto prefetch_release = [&](int64_t req) {
        if (window > 0 && req >= window) {
            const int* slot = ring + (int64_t)(req % window) * ring_stride;
            for (int k = tid; k < ring_stride; k += NC) rg_cp_async4(rel + k, slot + k);
        }
    };
    if (n_req > 0) prefetch_release(req0);
    const double* Tw = T + w * RT * TP;
    int* sg_w = slot_gpu + w * 32;
    const double ub_w = ub_s[w];
    // lane S < NTL, S != w: the bound of source tile S against this tile (lane-parallel block test)
    const bool cross_lane = lane < NTL && lane != w;
    const double lb_lane = cross_lane ? lb_s[lane * NTL + w] : 0.0;
    const uint16_t* pw_g = pairs_g + (int64_t)w * (nblk + 1) * 32 + lane;   // column c: pw_g[c * 32]
    double* const cw0 = cw_all + w * 32;
    int* const rw0 = rw_all + w * 32;
    unsigned n_cross = 0, n_src = 0;
    const bool stats = A.cross != nullptr;
    int done = 0;
    rg_bar_cons(NC);

    for (int r = 0; r < n_req; ++r) {
        const int64_t req = req0 + r;
        if (misc[0] == SS_OK) {
            const RgBlk m = bm[0];
            for (int k = tid; k < m.n_ins; k += NC) slot_gpu[ins[2 * (m.ins_start + k)]] = ins[2 * (m.ins_start + k) + 1];
            rg_cp_async_wait_all();
            mbar_wait(rows_bar, (uint32_t)(r & 1));
            rg_bar_cons(NC);
            if (window > 0 && req >= window) {
                const int cntr = rel[0];
                for (int k = tid; k < cntr; k += NC) occ_s[rel[1 + k]] -= 1;
            }
            rg_bar_cons(NC);
            for (int g = tid; g < ng; g += NC) {
                const int o = occ_s[g];
                if (o < 0 || o >= R.occpow_len) {
                    atomicExch((int*)&misc[0], o < 0 ? SS_OCC_UNDERFLOW : SS_BAD_INPUT);
                    misc[1] = g;
                }
                const int oc = o < 0 ? 0 : (o >= R.occpow_len ? R.occpow_len - 1 : o);
                tau_g[g] = R.st.base_tau[gbase + g] * (oc < A.pow_len ? pow_s[oc] : R.occpow[oc]);
            }
            if (tid == 0) misc[2] = 0;
        }
        rg_bar_all(NT);                                         // request start (the producer joins)
        if (misc[0] != SS_OK) break;

        double cost_lane = INF;      // cost of the GPU in slot `lane` for the column being finished
        int bpos_lane = 0;           // its backpointer (position in the previous column)
        // (local slot | position << 8) of source `lane` of the next two columns (L1 / L2 reads in flight)
        int pr_n1 = rg_ld_pair(pw_g);
        int pr_n2 = rg_ld_pair(pw_g + 32);
        const uint16_t* pw_next = pw_g + 64;                 // pair list of column b + 2
        uint8_t* bp_prev = bp - PC;                          // backpointers of boundary b - 1
        for (int b = 0; b < nblk; ++b) {
            // ---- column b of this tile: costs (+ backpointers of boundary b-1), published for boundary b ------
            const int pr = pr_n1;
            pr_n1 = pr_n2;
            if (b + 2 <= nblk) pr_n2 = rg_ld_pair(pw_next);
            pw_next += 32;
            const bool src = pr != RG_PAIR_NONE;
            const int n = __popc(__ballot_sync(0xffffffffu, src));       // sources are lanes 0..n-1
            const int sl = pr & 31, pos = (pr >> 8) & 0xff;
            double c;
            if (b == 0) {
                c = tau_g[sg_w[sl]];
            } else {
                c = __shfl_sync(0xffffffffu, cost_lane, sl);
                const int bpk = __shfl_sync(0xffffffffu, bpos_lane, sl);
                if (src) bp_prev[pos] = (uint8_t)bpk;
            }
            bp_prev += PC;
            if (!src) c = INF;
            const int boff = (b & 1) * NTL;
            double* cw = cw0 + boff * 32;
            int* rw = rw0 + boff * 32;
            cw[lane] = c;                                        // lanes >= n: +inf, row 0 (pairs of sources)
            rw[lane] = sl * (TP * 8);
            // bounds on this column's minimum cost from the high words (costs are >= 0, so their bit patterns
            // order like the values): [hi:0] <= min <= [hi+1:0] -- one REDUX instead of a 5-step shuffle tree
            const unsigned hmin = __reduce_min_sync(0xffffffffu, (unsigned)__double2hiint(c));
            const double cmin_hi = hmin >= 0x7ff00000u ? INF : __hiloint2double((int)(hmin + 1u), 0);
            if (lane == 0) cmin_all[boff + w] = __hiloint2double((int)hmin, 0);
            rg_bar_all(NT);                                     // boundary b: all tiles published, units applied
            const double tau_d = tau_g[sg_w[lane]];             // destination `lane`'s tau (final after the barrier)
            // lane-parallel bound test of every source tile S against this tile
            const double ubd = __dadd_rn(cmin_hi, ub_w);                                // >= every v_j here
            const bool keep_S = cross_lane && !(__dadd_rn(cmin_all[boff + (lane < NTL ? lane : 0)], lb_lane) > ubd);
            unsigned tiles = __ballot_sync(0xffffffffu, keep_S);

            // ---- relax boundary b inside the tile: sources in position order, strict <, two chains (even / odd
            //      sources) merged lexicographically == numpy's first-index argmin ---------------------------------
            double v = INF, v1 = INF;
            int ix = 0x7fff, ix1 = 0x7fff;
            const char* Tb = reinterpret_cast<const char*>(Tw + lane);
#pragma unroll RG_UNROLL_N
            for (int k = 0; k < n; k += 2) {
                const double2 c01 = *reinterpret_cast<const double2*>(cw + k);
                const int2 r2 = *reinterpret_cast<const int2*>(rw + k);
                const double a0 = __dadd_rn(c01.x, *reinterpret_cast<const double*>(Tb + r2.x));
                const double a1 = __dadd_rn(c01.y, *reinterpret_cast<const double*>(Tb + r2.y));
                if (a0 < v) { v = a0; ix = k; }
                if (a1 < v1) { v1 = a1; ix1 = k + 1; }
            }
            rg_lex_min(v, ix, v1, ix1);
            const int pix = __shfl_sync(0xffffffffu, pos, ix & 31);      // position of source ix in column b
            int pv = ix < 32 ? pix : RG_POS_NONE;
            // ---- cross-tile blocks the bound test keeps (rare): only their sources whose candidates can still
            //      reach ubd, entries recomputed from the pool matrix eight at a time (one L2 round trip per batch)
            double vmax = ubd;
            if (tiles) {
                // destination slots of boundary b (the sources of column b + 1): only their minima bound the test
                const unsigned dmask = __reduce_or_sync(0xffffffffu, pr_n1 != RG_PAIR_NONE ? 1u << (pr_n1 & 31) : 0u);
                // the intra-region minima are known now: a source can only matter where fl(c + lb) <= some v_j,
                // so bound by the largest destination minimum ([hi+1:0] >= v for v >= 0) instead of ubd
                const unsigned hv = __reduce_max_sync(0xffffffffu, ((dmask >> lane) & 1u) ? (unsigned)__double2hiint(v) : 0u);
                const double vb = hv >= 0x7ff00000u ? INF : __hiloint2double((int)(hv + 1u), 0);
                vmax = vb < ubd ? vb : ubd;
                unsigned t2 = 0;
                for (unsigned tt = tiles; tt; tt &= tt - 1) {
                    const int S = __ffs(tt) - 1;
                    if (!(__dadd_rn(cmin_all[boff + S], lb_s[S * NTL + w]) > vmax)) t2 |= 1u << S;
                }
                tiles = t2;
            }
            while (tiles) {
                const int S = __ffs(tiles) - 1;
                tiles &= tiles - 1;
                const double lbS = lb_s[S * NTL + w];
                const double uS = uni_s[S * NTL + w];                     // every S->D pool entry, or NaN
                const bool uniform = uS == uS;
                const double* cwS = cw_all + (boff + S) * 32;
                // sources of S: lanes whose cost is finite (lanes >= the column length publish +inf)
                // lane k: source k's GPU and position (tile S's pair list of column b; its slots are held through b)
                const int prS = rg_ld_pair(pairs_g + ((int64_t)S * (nblk + 1) + b) * 32 + lane);
                const int gsl = prS != RG_PAIR_NONE ? slot_gpu[S * 32 + (prS & 31)] : 0;
                // source k can only reach a destination of this tile if c_k + (its own bound to the tile) <= vmax
                const double lbk = (A.use_lbg && cwS[lane] < INF) ? (double)lbg_s[gsl * NTL + w] : lbS;
                unsigned keep = __ballot_sync(0xffffffffu, cwS[lane] < INF && !(__dadd_rn(cwS[lane], lbk) > vmax));
                if (stats) { n_cross += keep != 0; n_src += __popc(keep); }
                const int psl = (prS >> 8) & 0xff;
                const int gd = sg_w[lane];
                // entries: the tile pair's uniform pool value (or the pool matrix) x the pair's jitter quantile
                // from the shared-memory table, four sources per round
                while (keep) {
                    constexpr int KB = NTL <= 4 ? RG_KB : RG_KB_WIDE;
                    int kk[KB], gs[KB];
                    double e[KB];
#pragma unroll
                    for (int q = 0; q < KB; ++q) {
                        kk[q] = keep ? __ffs(keep) - 1 : -1;
                        keep &= keep - 1;
                    }
#pragma unroll
                    for (int q = 0; q < KB; ++q) gs[q] = __shfl_sync(0xffffffffu, gsl, kk[q] & 31);
#pragma unroll
                    for (int q = 0; q < KB; ++q) {
                        double x = kk[q] < 0 ? INF : (uniform ? uS : A.base_rtt[(int64_t)gs[q] * G + gd]);
                        if (A.jitter_seed && kk[q] >= 0)
                            x = __dmul_rn(x, (double)jq_s[ss_jitter_index(mix, (uint32_t)gs[q], (uint32_t)gd)]);
                        e[q] = x;
                    }
#pragma unroll
                    for (int q = 0; q < KB; ++q) {
                        const int p = __shfl_sync(0xffffffffu, psl, kk[q] & 31);
                        if (kk[q] < 0) continue;
                        const double a = __dadd_rn(cwS[kk[q]], e[q]);
                        if (a < v || (a == v && p < pv)) { v = a; pv = p; }
                    }
                }
            }
            // ---- finish destination `lane` of column b+1 ---------------------------------------------------------
            bpos_lane = v < INF ? pv : 0;                        // np.argmin of an all-inf column is 0
            cost_lane = __dadd_rn(v, tau_d);
        }
        {
            // last column: backpointers of the last boundary, then this tile's (cost, position) minimum
            const int pr = pr_n1;
            const bool src = pr != RG_PAIR_NONE;
            const int sl = pr & 31, pos = (pr >> 8) & 0xff;
            double c = __shfl_sync(0xffffffffu, cost_lane, sl);
            const int bpk = __shfl_sync(0xffffffffu, bpos_lane, sl);
            if (src) bp[(nblk - 1) * PC + pos] = (uint8_t)bpk;
            else c = INF;
            int idx = src ? pos : 0x7fffffff;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double v2 = __shfl_xor_sync(0xffffffffu, c, o);
                const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
                rg_lex_min(c, idx, v2, i2);
            }
            if (lane == 0) { red_v[w] = c; red_i[w] = idx; }
        }
        rg_bar_all(NT);                                         // every tile's minimum; T is free again
        // backtrack, segment-parallel over the consumer warps (as replay_slots.cu)
        {
            const int blo = w * nblk / NTL, bhi = (w + 1) * nblk / NTL;
            for (int st = lane; st < PC; st += 32) {
                int p = st;
                for (int b = bhi - 1; b >= blo; --b) p = min((int)bp[b * PC + p], PC - 1);
                seg_end[w * PC + st] = (uint8_t)p;
            }
        }
        rg_bar_cons(NC);
        if (tid == 0) {
            double v = red_v[0];
            int idx = red_i[0];
            for (int t = 1; t < NTL; ++t) rg_lex_min(v, idx, red_v[t], red_i[t]);
            if (!(v <= DBL_MAX)) {
                misc[0] = SS_NO_PATH;
            } else {
                int p = idx;
                picks[nl - 1] = p;
                for (int t = NTL - 1; t >= 0; --t) {
                    seg_start[t] = p;
                    p = seg_end[t * PC + p];
                }
            }
            if (R.out.cost) R.out.cost[(int64_t)dag * n_req + r] = v;
        }
        rg_bar_cons(NC);
        if (lane == 0 && misc[0] == SS_OK) {
            const int blo = w * nblk / NTL, bhi = (w + 1) * nblk / NTL;
            int p = seg_start[w];
            for (int b = bhi - 1; b >= blo; --b) {
                p = bp[b * PC + p];
                picks[b] = p;
            }
        }
        rg_bar_cons(NC);
        if (misc[0] != SS_OK) continue;

        const int tag = (int)(req & 0x3fffffff) + 1;
        int* slot = window > 0 ? ring + (int64_t)(req % window) * ring_stride : nullptr;
        uint64_t h = 0;
        for (int l = tid; l < nl; l += NC) {
            const int g = D.node_gpu[coff[l] + picks[l]];
            h += ss_splitmix64(((uint64_t)l << 32) | (uint64_t)g);
            if (R.out.gpus) R.out.gpus[((int64_t)dag * n_req + r) * D.max_layers + l] = (int16_t)g;
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
        rg_bar_cons(NC);
        if (tid == 0 && slot) slot[0] = misc[2];
        rg_bar_cons(NC);
        if (r + 1 < n_req) prefetch_release(req + 1);
        ++done;
    }
    rg_cp_async_wait_all();
    if (stats && lane == 0) {
        atomicAdd(&A.cross[0], (unsigned long long)(NTL - 1) * (unsigned long long)nblk * (unsigned long long)done);
        atomicAdd(&A.cross[1], (unsigned long long)n_cross);
        atomicAdd(&A.cross[2], (unsigned long long)n_src);
    }
    for (int g = tid; g < ng; g += NC) R.st.occ[gbase + g] = occ_s[g];
    if (tid == 0) {
        R.st.next_req[dag] = req0 + done;
        if (misc[0] != SS_OK) { R.st.status[dag] = misc[0]; R.st.aux[dag] = misc[1]; }
    }
}

inline int rg_align(int x, int a) { return (x + a - 1) / a * a; }

}  // namespace

extern "C" int64_t ss_region_meta_bytes(int32_t layers, int32_t n_gpus, int32_t n_tiles, int32_t pos_cap) {
    RgLayout ml{layers - 1, n_tiles, pos_cap, n_gpus};
    return ml.bytes();
}

extern "C" int ss_region_program(int32_t n_scen, int32_t layers, int32_t n_gpus, const int32_t* slice_lo,
                                 const int32_t* slice_hi, int64_t slice_stride, const uint8_t* leave,
                                 const double* rtt, const int64_t* jitter_seed, const int32_t* tile_of,
                                 int32_t n_tiles, int32_t pos_cap, int64_t meta_stride, int64_t stream_stride,
                                 uint8_t* meta, double* stream, int32_t* rt_used, int32_t* status, void* stream_h) {
    if (n_scen <= 0) return SS_OK;
    if (layers < 2 || n_gpus < 1 || n_gpus > 32767 || n_tiles < 1 || n_tiles > RG_MAX_TILES || pos_cap < 1 ||
        pos_cap > 256 || !tile_of)
        return SS_BAD_INPUT;
    if (meta_stride < ss_region_meta_bytes(layers, n_gpus, n_tiles, pos_cap) || (meta_stride & 15))
        return SS_BAD_INPUT;
    const int n_blk = layers - 1;
    const int smem = ((n_gpus + 7) / 8) * 8 * 2 + ((n_blk * n_tiles * 32 + 7) / 8) * 8 * 2 + (n_blk + 2) * 8 +
                     n_gpus * 8 + 64;
    if (smem > 200 * 1024) return SS_BAD_INPUT;
    if (cudaFuncSetAttribute(region_program_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return SS_CUDA_ERROR;
    region_program_kernel<<<n_scen, 256, smem, ss_stream(stream_h)>>>(
        layers, n_gpus, slice_lo, slice_hi, slice_stride, leave, rtt, jitter_seed, tile_of, n_tiles, pos_cap,
        meta_stride, stream_stride, meta, stream, rt_used, status);
    SS_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_replay_regions(const ss_dag_set* dags, const uint8_t* meta, int64_t meta_stride,
                                 const double* stream, int64_t stream_stride, int32_t n_tiles, int32_t pos_cap,
                                 int32_t rt_rows, const double* bounds, const double* base_rtt,
                                 const int64_t* jitter_seed, const ss_replay_state* st, const double* occpow,
                                 int32_t occpow_len, int32_t window, int32_t n_req, const ss_replay_out* out,
                                 void* stream_h) {
    if (!dags || !st || !occpow || occpow_len < 1 || n_req < 1 || !meta || !stream || !bounds || !base_rtt)
        return SS_BAD_INPUT;
    const ss_dag_set& D = *dags;
    if (D.n_dags <= 0) return SS_OK;
    if (n_tiles < 1 || n_tiles > RG_MAX_TILES || rt_rows < 1 || rt_rows > 32 || pos_cap < 1 || pos_cap > 256 ||
        D.max_layers < 2 || D.max_hosts > pos_cap)
        return SS_BAD_INPUT;
    RgArgs A{};
    A.meta = meta;
    A.meta_stride = meta_stride;
    A.stream = stream;
    A.stream_stride = stream_stride;
    A.bounds = bounds;
    A.base_rtt = base_rtt;
    A.jitter_seed = jitter_seed;
    A.pos_cap = pos_cap;
    A.rt = rt_rows;
    RgLayout ml{D.max_layers - 1, n_tiles, pos_cap, D.max_gpus};
    if (meta_stride < ml.bytes()) return SS_BAD_INPUT;
    A.meta_smem = ml.off_pairs();
    const int unit_min = rg_align((rt_rows + 1) * 8 * 2, 128);          // one entering GPU: row + column
    A.stage_bytes = max(g_rg_stage_bytes, unit_min);
    A.nbuf = g_rg_nbuf;
    const int L = D.max_layers;
    int o = 0;
    // tile row pitch: >= the unit length (rt_rows + 1, even), even so bulk-copied rows stay 16-B aligned; lanes past
    // the pitch read the next row (their slots are not destinations), the last row's by the 32-double pad
    A.tp = (rt_rows + 2) & ~1;
    if (const char* e = getenv("SS_REGION_TP")) { const int tp = atoi(e); if (tp >= A.tp && tp % 2 == 0) A.tp = tp; }
    if (const char* e = getenv("SS_REGION_NBUF")) { const int nb = atoi(e); if (nb >= 1 && nb <= 8) A.nbuf = nb; }
    A.off_T = o;       o += rg_align((n_tiles * rt_rows * A.tp + 32) * 8, 128);
    A.off_stage = o;   o += A.nbuf * A.stage_bytes;
    A.off_bar = o;     o += 128;
    A.off_meta = o;    o += rg_align(A.meta_smem, 16);
    A.off_cw = o;      o += 2 * n_tiles * 32 * 8;
    A.off_rw = o;      o += 2 * n_tiles * 32 * 4;
    A.off_cmin = o;    o += rg_align(2 * n_tiles * 8, 16);
    A.off_bnd = o;     o += rg_align((2 * n_tiles * n_tiles + n_tiles) * 8, 16);
    A.off_bp = o;      o += rg_align((L - 1) * pos_cap, 16);
    A.off_picks = o;   o += rg_align(L * 4, 16);
    A.off_tau = o;     o += rg_align(D.max_gpus * 8, 16);
    A.off_occ = o;     o += rg_align(D.max_gpus * 4, 16);
    A.off_stamp = o;   o += rg_align(D.max_gpus * 4, 16);
    A.off_slotgpu = o; o += n_tiles * 32 * 4;
    A.off_coff = o;    o += rg_align(L * 4, 16);
    A.off_red = o;     o += RG_MAX_TILES * 12 + 16;
    A.off_misc = o;    o += 64;
    A.pow_len = occpow_len < 64 ? occpow_len : 64;
    A.off_pow = o;     o += rg_align(A.pow_len * 8, 16);
    A.off_rel = o;     o += rg_align((L + 1) * 4, 16);
    A.off_seg = o;     o += rg_align(n_tiles * pos_cap, 16) + rg_align(n_tiles * 4, 16);
    A.off_jq = o;      o += jitter_seed ? 1024 * 4 : 0;
    A.off_lbg = o;     o += rg_align(D.max_gpus * n_tiles * 4, 16);   // last: dropped when it costs occupancy
    A.use_lbg = 1;
    A.total = o;
    if (A.total > 227 * 1024) return SS_BAD_INPUT;
    RgReplayArgs R{};
    R.st = *st;
    if (out) R.out = *out;
    R.occpow = occpow;
    R.occpow_len = occpow_len;
    R.window = window;
    R.n_req = n_req;
    cudaStream_t s = ss_stream(stream_h);
    if (R.out.chain_hash) cudaMemsetAsync(R.out.chain_hash, 0, sizeof(uint64_t) * (size_t)D.n_dags * n_req, s);
    const bool stats = getenv("SS_REGION_STATS") != nullptr;
    if (stats && cudaMalloc(&A.cross, 3 * sizeof(unsigned long long)) == cudaSuccess)
        cudaMemsetAsync(A.cross, 0, 3 * sizeof(unsigned long long), s);
    auto run = [&](auto kern) -> int {
        const int threads = (n_tiles + 1) * 32;
        // the per-source bound table rides in shared memory only when it costs no CTA per SM
        const int with_lbg = A.total, without_lbg = A.off_lbg;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, with_lbg) != cudaSuccess)
            return SS_CUDA_ERROR;
        int b_with = 0, b_without = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b_with, kern, threads, with_lbg) == cudaSuccess &&
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b_without, kern, threads, without_lbg) == cudaSuccess &&
            b_with < b_without) {
            A.use_lbg = 0;
            A.total = without_lbg;
        }
        kern<<<D.n_dags, threads, A.total, s>>>(D, A, R);
        SS_CHECK_LAUNCH();
        return SS_OK;
    };
    int rc;
    switch (n_tiles) {
        case 1: rc = run(replay_regions_kernel<1>); break;
        case 2: rc = run(replay_regions_kernel<2>); break;
        case 3: rc = run(replay_regions_kernel<3>); break;
        case 4: rc = run(replay_regions_kernel<4>); break;
        case 5: rc = run(replay_regions_kernel<5>); break;
        case 6: rc = run(replay_regions_kernel<6>); break;
        case 7: rc = run(replay_regions_kernel<7>); break;
        default: rc = run(replay_regions_kernel<8>); break;
    }
    if (rc != SS_OK) return rc;
    if (A.cross) {
        unsigned long long h[3];
        cudaMemcpyAsync(h, A.cross, sizeof(h), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        fprintf(stderr, "region stats: smem=%d rt=%d tiles=%d | cross blocks tested %llu relaxed %llu (%.4f%%), "
                "%.2f sources per relaxed block\n", A.total, rt_rows, n_tiles, h[0], h[1],
                h[0] ? 100.0 * (double)h[1] / (double)h[0] : 0.0, h[1] ? (double)h[2] / (double)h[1] : 0.0);
        cudaFree(A.cross);
    }
    return SS_OK;
}

extern "C" int ss_set_region_staging(int32_t stage_bytes, int32_t n_buffers) {
    if (stage_bytes > 0) g_rg_stage_bytes = (stage_bytes + 127) / 128 * 128;
    if (n_buffers > 0) g_rg_nbuf = n_buffers > 8 ? 8 : n_buffers;
    return SS_OK;
}
