// Slot-tile replay: Phase-2 replay for interval-slice scenario sets with an
// SM-resident RTT tile (beyond the streaming roofline).
//
// Why it is exact.  The DP of router.py:163-185 only ever reads
// E_b[i][j] = M[col_b[i]][col_{b+1}[j]].  In a plan produced by allocate()
// (and in any churned version of it) every GPU hosts one contiguous layer slice,
// so GPU g belongs to the frontier held(b) = col_b U col_{b+1} for exactly one
// interval of boundaries [max(lo-2,0), hi-1].  Interval partitioning gives each
// GPU one fixed "slot" for its whole interval; the CTA keeps a shared-memory tile
// T[slot][slot] = M[gpu][gpu] over the slots and, when a GPU enters the frontier,
// writes its row and column (streamed from HBM).  The relaxation reads exactly
// the same fp64 values as the edge-block path -- only their transport changes:
// ~0.24 MB per C4 selection instead of 2.48 MB.
//
// Tie order.  Every layer column is cut into NW contiguous position ranges, one
// per consumer warp; a warp scans its sources in position order with a strict
// `<`, and the NW partials of a destination are merged lexicographically on
// (value, position) -- numpy's first-index argmin.  Lanes own destination SLOTS
// (row segments of T are contiguous -> conflict-free LDS.64).
//
// Slots are reused one boundary late (a freed slot stays a "zombie" for one
// boundary), so the rows / columns of the GPUs entering at b+1 can be written
// while boundary b is relaxed: one named barrier per boundary.
//
// Program (built on device by slot_program_kernel, identical for every request):
//   meta  : header, per-boundary (n_ins, ins_start, unit_start), insert list
//           (slot, gpu), src_slot_by_pos[layer][S_CAP]
//   stream: per boundary, the inserted GPUs' T rows (b == 0) or rows+columns
//           (b > 0), each a "unit" of Wp doubles (Wp even -> 16-B aligned units)
//
// Measured (B200, C4 = L64/N256/k73, 1184 scenarios x 32 requests): 2.8e6 sel/s
// vs 2.65-2.77e6 for the streamed-block kernel, at ~0.33 MB of L2/HBM traffic
// per selection instead of 2.48 MB.  It is issue-bound, not memory-bound:
// ~9.7 instructions per relaxation (LDS, DADD, DSETP, 2x FSEL, SEL + per-source
// broadcast and address) plus the per-boundary merge / apply work, at 2 CTAs
// (10 warps) per SM -- see DESIGN.md.
#include <float.h>
#include <stdio.h>
#include <stdlib.h>

#include "ss_common.cuh"

namespace {

constexpr int IDX_NONE = 0x7fffffff;
constexpr int CONSUMER_BAR = 1;
constexpr int META_HDR = 16;

int g_stage_bytes = 8 * 1024;
int g_nbuf = 4;

// meta layout for one scenario (byte offsets), shared by generator and kernel.
// src[c][pos] (c = 0..n_blk) = slot of the GPU at position pos of layer c+1's host column;
// 16 zero bytes follow (the relaxation never reads past a column, the pad keeps vector loads in bounds).
struct MetaLayout {
    int n_blk, s_cap, n_cap;
    __host__ __device__ int off_blk() const { return META_HDR; }
    __host__ __device__ int off_ins() const { return META_HDR + n_blk * 8; }
    __host__ __device__ int off_src() const { return (off_ins() + n_cap * 4 + 15) / 16 * 16; }
    __host__ __device__ int bytes() const { return (off_src() + (n_blk + 1) * s_cap + 16 + 15) / 16 * 16; }
};

struct BlkMeta {
    int16_t n_ins, ins_start;
    int32_t unit_start;
};

// ---------------------------------------------------------------------------
// program generation: one CTA per scenario
// ---------------------------------------------------------------------------
__global__ void slot_program_kernel(int32_t layers, int32_t n_gpus, const int32_t* lo, const int32_t* hi,
                                    int64_t slice_stride, const uint8_t* leave, const double* rtt, const int64_t* jitter_seed,
                                    int32_t s_cap, int64_t meta_stride, int64_t stream_stride, uint8_t* meta,
                                    double* stream, int32_t* s_used_out, int32_t* status) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int s = blockIdx.x;
    const int n_blk = layers - 1;
    const uint8_t* gone = leave ? leave + (int64_t)s * n_gpus : nullptr;
    lo += s * slice_stride;                               // per-scenario slices (joins) or the shared plan
    hi += s * slice_stride;
    MetaLayout ml{n_blk, s_cap, n_gpus};
    uint8_t* mt = meta + (int64_t)s * meta_stride;
    double* st = stream + (int64_t)s * stream_stride;
    // smem: slot_of[n_gpus] int16, occ_tl[n_blk][s_cap] int16, bucket lists (insert / free boundary)
    int16_t* slot_of = reinterpret_cast<int16_t*>(sm);
    int16_t* occ_tl = slot_of + ((n_gpus + 7) / 8) * 8;
    int* ins_head = reinterpret_cast<int*>(occ_tl + ((n_blk * s_cap + 7) / 8) * 8);   // [n_blk + 2]
    int* free_head = ins_head + n_blk + 2;                                             // [n_blk + 2]
    int* ins_next = free_head + n_blk + 2;                                             // [n_gpus]
    int* free_next = ins_next + n_gpus;                                                // [n_gpus]
    __shared__ int s_used, bad, wp_s;
    const int tid = threadIdx.x;
    for (int i = tid; i < n_blk * s_cap; i += blockDim.x) occ_tl[i] = -1;
    for (int g = tid; g < n_gpus; g += blockDim.x) slot_of[g] = -1;
    for (int b = tid; b < n_blk + 2; b += blockDim.x) { ins_head[b] = -1; free_head[b] = -1; }
    __syncthreads();
    if (tid == 0) {
        // bucket the GPUs by first frontier boundary max(lo-2, 0) and by the boundary hi+1 at which their slot
        // becomes reusable (interval [max(lo-2,0), hi-1] plus one zombie boundary); pushing front while
        // walking g downwards keeps every bucket in ascending GPU order
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
        int used = 0;
        uint64_t freem[4] = {~0ull, ~0ull, ~0ull, ~0ull};      // s_cap <= 256
        BlkMeta* bm = reinterpret_cast<BlkMeta*>(mt + ml.off_blk());
        int16_t* ins = reinterpret_cast<int16_t*>(mt + ml.off_ins());
        int n_ins_total = 0;
        int unit = 0;
        for (int b = 0; b < n_blk && !bad; ++b) {
            // slots are reused one boundary late, so the kernel can write boundary b+1's rows / columns while
            // boundary b is still being relaxed
            for (int g = free_head[b]; g >= 0; g = free_next[g]) {
                const int q = slot_of[g];
                if (q >= 0) freem[q >> 6] |= 1ull << (q & 63);
            }
            const int start = n_ins_total;
            for (int g = ins_head[b]; g >= 0; g = ins_next[g]) {
                int q = -1;
                for (int w = 0; w < 4 && q < 0; ++w)
                    if (freem[w]) q = w * 64 + __ffsll((long long)freem[w]) - 1;
                if (q < 0 || q >= s_cap) { bad = 1; break; }
                freem[q >> 6] &= ~(1ull << (q & 63));
                slot_of[g] = (int16_t)q;
                if (q + 1 > used) used = q + 1;
                ins[2 * n_ins_total] = (int16_t)q;
                ins[2 * n_ins_total + 1] = (int16_t)g;
                ++n_ins_total;
            }
            BlkMeta m;
            m.n_ins = (int16_t)(n_ins_total - start);
            m.ins_start = (int16_t)start;
            m.unit_start = unit;
            bm[b] = m;
            unit += (b == 0 ? 1 : 2) * (n_ins_total - start);
        }
        s_used = used;
        const int wp = (used + 1) & ~1;
        wp_s = wp;
        int32_t* hdr = reinterpret_cast<int32_t*>(mt);
        hdr[0] = used;
        hdr[1] = wp;
        hdr[2] = unit;
        hdr[3] = n_ins_total;
        if ((int64_t)unit * wp > stream_stride) bad = 2;
        status[s] = bad ? SS_BAD_INPUT : SS_OK;
        s_used_out[s] = bad ? 0 : used;
    }
    __syncthreads();
    // occupancy timeline: GPU g holds its slot for boundaries [max(lo-2,0), hi] (interval + zombie boundary)
    for (int g = tid; g < n_gpus; g += blockDim.x) {
        const int q = slot_of[g];
        if (q < 0) continue;
        const int sb = lo[g] - 2 < 0 ? 0 : lo[g] - 2;
        const int eb = hi[g] < n_blk - 1 ? hi[g] : n_blk - 1;
        for (int b = sb; b <= eb; ++b) occ_tl[b * s_cap + q] = (int16_t)g;
    }
    __syncthreads();
    if (bad) return;
    const int wp = wp_s;
    // per-layer position -> slot maps
    uint8_t* src = mt + ml.off_src();
    const int lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    if (tid < 16) src[(n_blk + 1) * s_cap + tid] = 0;
    for (int c = warp; c <= n_blk; c += nw) {
        for (int q = lane; q < s_cap; q += 32) src[c * s_cap + q] = 0;
        __syncwarp();
        int cs = 0;
        for (int g0 = 0; g0 < n_gpus; g0 += 32) {
            const int g = g0 + lane;
            const bool alive = g < n_gpus && !(gone && gone[g]);
            const bool in_col = alive && lo[g] <= c + 1 && hi[g] >= c + 1;   // hosts layer c+1 (1-based)
            const unsigned ms = __ballot_sync(0xffffffffu, in_col);
            if (in_col) src[c * s_cap + cs + __popc(ms & ((1u << lane) - 1u))] = (uint8_t)slot_of[g];
            cs += __popc(ms);
        }
    }
    // stream units: rows (b == 0) or row/column pairs
    const BlkMeta* bm = reinterpret_cast<const BlkMeta*>(mt + ml.off_blk());
    const int16_t* ins = reinterpret_cast<const int16_t*>(mt + ml.off_ins());
    const bool jit = jitter_seed != nullptr;
    const uint64_t mix = jit ? ss_splitmix64((uint64_t)jitter_seed[s]) : 0;
    const int64_t dim = n_gpus;
    for (int b = 0; b < n_blk; ++b) {
        const BlkMeta m = bm[b];
        const int units = (b == 0 ? 1 : 2) * m.n_ins;
        for (int e = tid; e < units * wp; e += blockDim.x) {
            const int u = e / wp, t = e - u * wp;
            const int k = b == 0 ? u : (u >> 1);
            const bool col = b != 0 && (u & 1);
            const int g = ins[2 * (m.ins_start + k) + 1];
            const int o = t < s_cap ? occ_tl[b * s_cap + t] : -1;
            double v = __longlong_as_double(0x7ff0000000000000ll);
            if (o >= 0) {
                const int a = col ? o : g, c = col ? g : o;
                v = rtt[(int64_t)a * dim + c];
                if (jit) v = v * ss_jitter(mix, (uint32_t)a, (uint32_t)c);
            }
            st[(int64_t)(m.unit_start + u) * wp + t] = v;
        }
    }
}

// ---------------------------------------------------------------------------
// replay kernel
// ---------------------------------------------------------------------------
struct SlotArgs {
    const uint8_t* meta;
    int64_t meta_stride;
    const double* stream;
    int64_t stream_stride;
    int s_rows, w, nbuf, stage_bytes;
    int off_T, off_stage, off_full, off_empty, off_meta, meta_bytes, off_part, off_bp, off_picks, off_tau, off_occ,
        off_stamp, off_slotgpu, off_cl, off_red, off_misc, off_base, off_pow, pow_len, off_rel, off_coff, off_costw, off_seg,
        total;
    unsigned long long* prof;   // diagnostics (env SS_SLOT_PROF=1): per-warp phase cycle totals, else NULL
};

struct ReplayArgs {
    ss_replay_state st;
    ss_replay_out out;
    const double* occpow;
    int32_t occpow_len;
    int32_t window;
    int32_t n_req;
};

constexpr int PART_NONE = 0x7fff;

__device__ __forceinline__ void consumer_sync(int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"n"(CONSUMER_BAR), "r"(nthreads) : "memory");
}

constexpr int ALL_BAR = 2;
// boundary / request-start barrier of the consumers AND the unit-producer warp
__device__ __forceinline__ void all_sync(int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"n"(ALL_BAR), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void lex_min(double& v, int& i, double v2, int i2) {
    if (v2 < v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

// LDGSTS: global -> shared without a register round trip; every copy of a phase is in flight at once
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// One source row against the DPL destination slots a lane owns (lane, lane+32, ...):
// one address, DPL conflict-free LDS.64, strict `<` (positions arrive ascending).
template <int DPL>
__device__ __forceinline__ void relax_row(const double* row, double c, int p, double (&v)[DPL], int (&ix)[DPL]) {
#pragma unroll
    for (int d = 0; d < DPL; ++d) {
        const double a = __dadd_rn(c, row[d * 32]);
        if (a < v[d]) { v[d] = a; ix[d] = p; }
    }
}

// Warp roles: NW consumer warps (the DP), warp NW owns the row/column units: it streams them with 1-D TMA
// bulk copies through a ring of staging buffers it alone consumes, and writes them into T ("apply").
//
// Every layer column is cut into NW contiguous position ranges (warp w owns
// [w*R/NW, (w+1)*R/NW)).  Per boundary b, ONE named barrier over all NW + 1 warps:
//   consumers: merge -- warp w finishes the costs of ITS positions of column b: the lexicographic
//              (value, position) min over the NW range partials of boundary b-1 (== numpy first-index
//              argmin), + tau; backpointers;
//              relax -- lanes own DPL destination slots and scan the warp's sources -> partial (value,
//              position) per slot;
//   producer : apply(b+1) -- rows / columns of the GPUs entering at b+1, concurrently with relax(b): slots are
//              reused one boundary late, so nothing relaxed at b is overwritten, and the copy is off the
//              consumers' critical path.
template <int DPL, int NW>
__global__ void __launch_bounds__((NW + 1) * 32, 2)
replay_slots_kernel(ss_dag_set D, SlotArgs A, ReplayArgs R) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int SC = DPL * 32;
    constexpr int NC = NW * 32;
    constexpr int NT = NC + 32;
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    const int dag = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int l0 = D.layer_ptr[dag];
    const int nl = D.layer_ptr[dag + 1] - l0;
    const int nblk = nl - 1;
    const int W = A.w;
    MetaLayout ml{nblk, SC, D.max_gpus};

    double* T = reinterpret_cast<double*>(smem + A.off_T);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + A.off_full);
    uint64_t* rows_bar = reinterpret_cast<uint64_t*>(smem + A.off_empty);   // the request's initial rows landed
    unsigned char* meta_s = smem + A.off_meta;
    double* part_v = reinterpret_cast<double*>(smem + A.off_part);          // [2][NW][SC]
    int16_t* part_i = reinterpret_cast<int16_t*>(part_v + 2 * NW * SC);     // [2][NW][SC]
    uint8_t* bp = smem + A.off_bp;
    int* picks = reinterpret_cast<int*>(smem + A.off_picks);
    double* tau_g = reinterpret_cast<double*>(smem + A.off_tau);
    int* occ_s = reinterpret_cast<int*>(smem + A.off_occ);
    int* stamp = reinterpret_cast<int*>(smem + A.off_stamp);
    int* slot_gpu = reinterpret_cast<int*>(smem + A.off_slotgpu);
    int* col_len = reinterpret_cast<int*>(smem + A.off_cl);
    double* red_v = reinterpret_cast<double*>(smem + A.off_red);
    int* red_i = reinterpret_cast<int*>(smem + A.off_red + NW * 8);
    volatile int* misc = reinterpret_cast<int*>(smem + A.off_misc);  // [0] status [1] aux [2] ring [3] chunks/req
    double* base_s = reinterpret_cast<double*>(smem + A.off_base);   // per-GPU base tau (static per launch)
    double* pow_s = reinterpret_cast<double*>(smem + A.off_pow);     // occpow[0 .. pow_len)
    int* rel = reinterpret_cast<int*>(smem + A.off_rel);             // prefetched ring slot of the next release
    int* coff = reinterpret_cast<int*>(smem + A.off_coff);           // this DAG's column offsets
    uint8_t* seg_end = smem + A.off_seg;                              // [NW][SC] backtrack segment ends
    int* seg_start = reinterpret_cast<int*>(smem + A.off_seg + NW * SC);   // [NW] true segment starts
    constexpr int CW_LEN = SC / NW + 8;                               // >= ceil(SC / NW) + 1, even
    double* cost_w = reinterpret_cast<double*>(smem + A.off_costw);  // [NW][CW_LEN] each warp's source costs
    int* row_w = reinterpret_cast<int*>(cost_w + NW * CW_LEN);        // [NW][CW_LEN] their T row byte offsets

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
    // static program metadata -> shared memory (once per launch, reused by every request)
    {
        const int4* srcv = reinterpret_cast<const int4*>(meta_g);
        int4* dstv = reinterpret_cast<int4*>(meta_s);
        for (int q = tid; q < A.meta_bytes / 16; q += blockDim.x) dstv[q] = srcv[q];
        for (int l = tid; l < nl; l += blockDim.x) {
            col_len[l] = D.col_len[l0 + l];
            coff[l] = D.col_off[l0 + l];
        }
        const int gb = R.st.gpu_ptr[dag], gn = R.st.gpu_ptr[dag + 1] - gb;
        for (int g = tid; g < gn; g += blockDim.x) base_s[g] = R.st.base_tau[gb + g];
        for (int o = tid; o < A.pow_len; o += blockDim.x) pow_s[o] = R.occpow[o];
    }
    __syncthreads();
    const int32_t* hdr = reinterpret_cast<const int32_t*>(meta_s);
    const BlkMeta* bm = reinterpret_cast<const BlkMeta*>(meta_s + ml.off_blk());
    const int16_t* ins = reinterpret_cast<const int16_t*>(meta_s + ml.off_ins());
    const uint8_t* src_map = meta_s + ml.off_src();
    const int Wp = hdr[1];
    const int upc = max(1, A.stage_bytes / (Wp * 8));          // units per chunk
    const int tw = min(Wp, A.s_rows);                          // unit entries that land in T (Wp may pad by one)
    if (tid == 0 && misc[0] == SS_OK) {
        if (hdr[0] > A.s_rows || nl < 2) misc[0] = SS_BAD_INPUT;
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
    unsigned long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // prologue relax apply barrier epilogue argmin+backtrack chain-update initial-rows

    // ========================= producer: TMA ring + apply(1..nblk-1) ===============
    if (warp == NW) {
        const int64_t total = (int64_t)n_req * misc[3];
        int64_t issued = 0;
        int ib = 1, iu0 = 0;                                 // next chunk to issue: boundary, first unit
        auto issue_next = [&](int buf) {                     // lane 0; buffer `buf` is free
            while (ib < nblk && iu0 >= 2 * bm[ib].n_ins) { ++ib; iu0 = 0; }
            if (ib >= nblk) { ib = 1; iu0 = 0; while (ib < nblk && 2 * bm[ib].n_ins == 0) ++ib; }
            const BlkMeta m = bm[ib];
            const int nu = min(upc, 2 * m.n_ins - iu0);
            const uint32_t bytes = (uint32_t)nu * Wp * 8;
            fence_proxy_async_smem();
            mbar_expect_tx(&full[buf], bytes);
            bulk_g2s(smem + A.off_stage + (size_t)buf * A.stage_bytes, stream_g + (int64_t)(m.unit_start + iu0) * Wp,
                     bytes, &full[buf]);
            iu0 += nu;
            ++issued;
        };
        // the initial frontier's rows (boundary 0, one unit per GPU of col_0 U col_1) go straight into their T rows:
        // 1-D bulk copies (T rows are 16-B aligned: even pitch), completing on rows_bar
        int rows_issued = 0;
        auto issue_rows = [&]() {
            const BlkMeta m = bm[0];
            const uint32_t ub = (uint32_t)Wp * 8;
            if (lane == 0) mbar_expect_tx(rows_bar, ub * (uint32_t)m.n_ins);
            __syncwarp();
            fence_proxy_async_smem();
            const double* s0 = stream_g + (int64_t)m.unit_start * Wp;
            for (int u = lane; u < m.n_ins; u += 32)
                bulk_g2s(T + ins[2 * (m.ins_start + u)] * W, s0 + (int64_t)u * Wp, ub, rows_bar);
            ++rows_issued;
        };
        if (n_req > 0) issue_rows();
        if (lane == 0)
            for (int b = 0; b < A.nbuf && issued < total; ++b) issue_next(b);
        int cbuf = 0;
        uint32_t cphase = 0;
        int64_t consumed = 0;
        for (int r = 0; r < n_req; ++r) {
            all_sync(NT);                                    // request start: tau ready, initial rows landed
            if (misc[0] != SS_OK) break;
            long long tp = A.prof ? clock64() : 0;
            for (int b = 0; b < nblk; ++b) {
                if (b + 1 < nblk) {
                    const BlkMeta m = bm[b + 1];
                    const int units = 2 * m.n_ins;
                    for (int u0 = 0; u0 < units; u0 += upc) {
                        const int nu = min(upc, units - u0);
                        mbar_wait(&full[cbuf], cphase);
                        const double* stg = reinterpret_cast<const double*>(smem + A.off_stage +
                                                                            (size_t)cbuf * A.stage_bytes);
                        for (int ul = 0; ul < nu; ++ul) {
                            const int u = u0 + ul;
                            const int slot = ins[2 * (m.ins_start + (u >> 1))];
                            const double* su = stg + ul * Wp;
                            // tw <= s_rows <= SC: all DPL loads in flight before the stores
                            double x[DPL];
#pragma unroll
                            for (int d = 0; d < DPL; ++d) x[d] = lane + 32 * d < tw ? su[lane + 32 * d] : 0.0;
                            const int step = (u & 1) ? 32 * W : 32;      // column: stride W; row: contiguous
                            double* dst = T + ((u & 1) ? lane * W + slot : slot * W + lane);
#pragma unroll
                            for (int d = 0; d < DPL; ++d)
                                if (lane + 32 * d < tw) dst[d * step] = x[d];
                        }
                        __syncwarp();                        // the buffer is read: refill it
                        if (lane == 0 && issued < total) issue_next(cbuf);
                        ++consumed;
                        if (++cbuf == A.nbuf) { cbuf = 0; cphase ^= 1u; }
                    }
                    for (int k = lane; k < m.n_ins; k += 32)
                        slot_gpu[ins[2 * (m.ins_start + k)]] = ins[2 * (m.ins_start + k) + 1];
                }
                if (A.prof) { const long long t = clock64(); pacc[2] += (unsigned long long)(t - tp); tp = t; }
                all_sync(NT);                                // boundary b
                if (A.prof) { const long long t = clock64(); pacc[3] += (unsigned long long)(t - tp); tp = t; }
            }
            if (r + 1 < n_req) issue_rows();                 // T is no longer read by this request
        }
        if (rows_issued > 0) mbar_wait(rows_bar, (uint32_t)((rows_issued - 1) & 1));   // earlier phases were awaited
        // an aborted launch leaves copies in flight: land them before the CTA exits
        while (consumed < issued) {
            mbar_wait(&full[cbuf], cphase);
            ++consumed;
            if (++cbuf == A.nbuf) { cbuf = 0; cphase ^= 1u; }
        }
        if (A.prof && lane == 0)
            for (int k = 0; k < 8; ++k) atomicAdd(&A.prof[warp * 8 + k], pacc[k]);
        return;
    }

    // ========================= consumers ======================================
    const int gbase = R.st.gpu_ptr[dag];
    const int ng = R.st.gpu_ptr[dag + 1] - gbase;
    const int window = R.window;
    const int64_t req0 = R.st.next_req[dag];
    const int ring_stride = D.max_layers + 1;
    int* ring = R.st.ring + (int64_t)dag * (window > 0 ? window : 1) * ring_stride;
    for (int g = tid; g < ng; g += NC) {
        occ_s[g] = R.st.occ[gbase + g];
        stamp[g] = 0;
    }
    // ring slot read by request req's release (chain req - W): prefetched one request ahead
    auto prefetch_release = [&](int64_t req) {
        if (window > 0 && req >= window) {
            const int* slot = ring + (int64_t)(req % window) * ring_stride;
            for (int k = tid; k < ring_stride; k += NC) cp_async4(rel + k, slot + k);
        }
    };
    if (n_req > 0) prefetch_release(req0);
    // Costs of this warp's positions [p0, p0+n) of column c into cw[], their T row byte offsets into rw[]
    // (padded with +inf / row 0 to an even count).  c == 0: tau of the first layer's hosts; c >= 1: the
    // lexicographic (value, position) min over the NW range partials of boundary c-1 (== numpy first-index
    // argmin) + tau, recording the backpointers of boundary c-1.
    auto stage_sources = [&](int c, int p0, int n, double* cw, int* rw) {
        const int n2 = (n + 1) & ~1;
        for (int q = lane; q < n2; q += 32) {
            double cst = INF;
            int sl = 0;
            if (q < n) {
                const int p = p0 + q;
                sl = src_map[c * SC + p];
                if (c == 0) {
                    cst = tau_g[slot_gpu[sl]];
                } else {
                    const double* pv = part_v + ((c - 1) & 1) * NW * SC;
                    const int16_t* pi = part_i + ((c - 1) & 1) * NW * SC;
                    double v = pv[sl];
                    int i = pi[sl];
#pragma unroll
                    for (int w = 1; w < NW; ++w) lex_min(v, i, pv[w * SC + sl], (int)pi[w * SC + sl]);
                    if (i == PART_NONE) i = 0;                  // np.argmin of an all-inf column
                    cst = __dadd_rn(v, tau_g[slot_gpu[sl]]);
                    bp[(c - 1) * SC + p] = (uint8_t)i;
                }
            }
            cw[q] = cst;
            rw[q] = sl * W * 8;
        }
        __syncwarp();
    };
    int done = 0;
    consumer_sync(NC);

    long long tp = clock64();
#define SS_PROF(k)                                                   \
    if (A.prof) {                                                    \
        const long long _t = clock64();                              \
        pacc[k] += (unsigned long long)(_t - tp);                    \
        tp = _t;                                                     \
    }
    for (int r = 0; r < n_req; ++r) {
        const int64_t req = req0 + r;
        SS_PROF(4)
        // apply(0): the initial frontier's rows, bulk-copied into T by the producer warp as soon as the previous
        // request's last boundary had released T, so they land during that request's epilogue.
        if (misc[0] == SS_OK) {
            const BlkMeta m = bm[0];
            for (int k = tid; k < m.n_ins; k += NC) slot_gpu[ins[2 * (m.ins_start + k)]] = ins[2 * (m.ins_start + k) + 1];
            cp_async_wait_all();                                // the prefetched release slot
            mbar_wait(rows_bar, (uint32_t)(r & 1));             // the initial rows
            consumer_sync(NC);
            if (window > 0 && req >= window) {
                const int cnt = rel[0];
                for (int k = tid; k < cnt; k += NC) occ_s[rel[1 + k]] -= 1;
            }
            consumer_sync(NC);
            for (int g = tid; g < ng; g += NC) {
                const int o = occ_s[g];
                if (o < 0 || o >= R.occpow_len) {
                    atomicExch((int*)&misc[0], o < 0 ? SS_OCC_UNDERFLOW : SS_BAD_INPUT);
                    misc[1] = g;
                }
                const int oc = o < 0 ? 0 : (o >= R.occpow_len ? R.occpow_len - 1 : o);
                tau_g[g] = base_s[g] * (oc < A.pow_len ? pow_s[oc] : R.occpow[oc]);
            }
            if (tid == 0) misc[2] = 0;
        }
        all_sync(NT);                                           // request start (the producer joins)
        if (misc[0] != SS_OK) break;

        SS_PROF(0)
        double* cw = cost_w + warp * CW_LEN;
        int* rw = row_w + warp * CW_LEN;
        for (int b = 0; b < nblk; ++b) {
            const int rs = col_len[b];
            const int p0 = warp * rs / NW, n = (warp + 1) * rs / NW - p0;
            stage_sources(b, p0, n, cw, rw);
            // ---- relax boundary b over this warp's sources (2 per step: LDS.128 costs, LDS.64 rows) ------
            double v[DPL];
            int ix[DPL];
#pragma unroll
            for (int d = 0; d < DPL; ++d) { v[d] = INF; ix[d] = PART_NONE; }
            const char* Tb = reinterpret_cast<const char*>(T + lane);
#pragma unroll 4
            for (int k = 0; k < n; k += 2) {
                const double2 c01 = *reinterpret_cast<const double2*>(cw + k);
                const int2 r2 = *reinterpret_cast<const int2*>(rw + k);
                relax_row<DPL>(reinterpret_cast<const double*>(Tb + r2.x), c01.x, p0 + k, v, ix);
                relax_row<DPL>(reinterpret_cast<const double*>(Tb + r2.y), c01.y, p0 + k + 1, v, ix);
            }
            {
                double* pv = part_v + (b & 1) * NW * SC + warp * SC;
                int16_t* pi = part_i + (b & 1) * NW * SC + warp * SC;
#pragma unroll
                for (int d = 0; d < DPL; ++d) {
                    pv[d * 32 + lane] = v[d];
                    pi[d * 32 + lane] = (int16_t)ix[d];
                }
            }
            SS_PROF(1)
            all_sync(NT);                                       // boundary b (the producer has applied b+1)
            SS_PROF(3)
        }

        SS_PROF(7)
        // ---- last column: costs, argmin (first index), backtrack ----------------
        {
            const int rs = col_len[nblk];
            const int p0 = warp * rs / NW, n = (warp + 1) * rs / NW - p0;
            stage_sources(nblk, p0, n, cw, rw);
            double v = INF;
            int idx = IDX_NONE;
            for (int q = lane; q < n; q += 32) lex_min(v, idx, cw[q], p0 + q);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
                const int i2 = __shfl_xor_sync(0xffffffffu, idx, o);
                lex_min(v, idx, v2, i2);
            }
            if (lane == 0) { red_v[warp] = v; red_i[warp] = idx; }
        }
        consumer_sync(NC);
        // backtrack, segment-parallel: warp w owns boundaries [w*nblk/NW, (w+1)*nblk/NW); its lanes walk the
        // backpointers down from EVERY position of the segment's top layer at once (seg_end[w][start]); then the
        // true segment starts chain from the final argmin through seg_end (NW lookups), and each warp re-walks
        // its segment from its true start writing the picks -- ~2 x (nblk / NW) dependent steps instead of nblk
        {
            const int blo = warp * nblk / NW, bhi = (warp + 1) * nblk / NW;
            for (int st = lane; st < SC; st += 32) {
                int p = st;
                for (int b = bhi - 1; b >= blo; --b) p = min((int)bp[b * SC + p], SC - 1);   // rows past a column
                seg_end[warp * SC + st] = (uint8_t)p;                                       // hold stale bytes
            }
        }
        consumer_sync(NC);
        if (tid == 0) {
            double v = red_v[0];
            int idx = red_i[0];
            for (int w = 1; w < NW; ++w) lex_min(v, idx, red_v[w], red_i[w]);
            if (!(v <= DBL_MAX)) {
                misc[0] = SS_NO_PATH;
            } else {
                int p = idx;
                picks[nl - 1] = p;
                for (int w = NW - 1; w >= 0; --w) {
                    seg_start[w] = p;
                    p = seg_end[w * SC + p];
                }
            }
            if (R.out.cost) R.out.cost[(int64_t)dag * n_req + r] = v;
        }
        consumer_sync(NC);
        if (lane == 0 && misc[0] == SS_OK) {
            const int blo = warp * nblk / NW, bhi = (warp + 1) * nblk / NW;
            int p = seg_start[warp];
            for (int b = bhi - 1; b >= blo; --b) {
                p = bp[b * SC + p];
                picks[b] = p;
            }
        }
        consumer_sync(NC);
        SS_PROF(5)
        if (misc[0] != SS_OK) continue;                        // the next request-start barrier ends the launch

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
        consumer_sync(NC);
        if (tid == 0 && slot) slot[0] = misc[2];
        consumer_sync(NC);
        if (r + 1 < n_req) prefetch_release(req + 1);
        SS_PROF(6)
        ++done;
    }
    cp_async_wait_all();
    SS_PROF(4)
#undef SS_PROF
    if (A.prof && lane == 0)
        for (int k = 0; k < 8; ++k) atomicAdd(&A.prof[warp * 8 + k], pacc[k]);
    for (int g = tid; g < ng; g += NC) R.st.occ[gbase + g] = occ_s[g];
    if (tid == 0) {
        R.st.next_req[dag] = req0 + done;
        if (misc[0] != SS_OK) { R.st.status[dag] = misc[0]; R.st.aux[dag] = misc[1]; }
    }
}

// ---------------------------------------------------------------------------
// Cluster slot replay: the slot tile split by DESTINATION slots over a thread-block cluster
// ---------------------------------------------------------------------------
// For frontiers too wide for two single-CTA tiles per SM (C5: 110-150 slots), the CL CTAs of a cluster share
// one scenario: CTA q keeps Tq[src slot][c] = T[src][q*SCQ + c] -- every source row, its own SCQ destination
// columns -- so each CTA relaxes every source of a column against its own destinations and owns complete
// destination minima (no cross-CTA merge of partials).  Per boundary b:
//   stage(b)  the owner CTA of each position of column b merges its NW range partials (lexicographic
//             (value, position) == numpy first-index argmin), adds tau, and broadcasts (cost, Tq row offset)
//             into EVERY CTA's source table through distributed shared memory (st.shared::cluster); the
//             backpointer goes to CTA 0, which holds the whole table for the backtrack;
//   barrier.cluster (release / acquire): the source table is complete everywhere;
//   relax(b)  as the single-CTA kernel, over the CTA's own destination columns;
//   CTA barrier: partials visible, the producer warp has applied boundary b+1's rows / own columns.
// The request epilogue (final argmin, backtrack, occupancy update, ring, outputs) runs on CTA 0, which sends
// the chain's distinct GPUs to the other CTAs (each keeps its own occupancy / tau copy).  The relaxation
// reads the same fp64 values in the same order as ss_replay / ss_replay_slots: bit-identical results.
struct ClusterArgs {
    const uint8_t* meta;
    int64_t meta_stride;
    const double* stream;
    int64_t stream_stride;
    int s_rows, w, nbuf, stage_bytes, cl, sc, s_cap;
    int off_T, off_stage, off_full, off_meta, meta_bytes, off_part, off_src, off_bp, off_picks, off_tau, off_occ,
        off_stamp, off_slotgpu, off_cl, off_coff, off_red, off_cred, off_clist, off_misc, off_base, off_pow, pow_len,
        off_rel, off_seg, total;
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t peer_addr(const void* p, uint32_t rank) {
    uint32_t a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
    return a;
}
__device__ __forceinline__ void st_cl_f64(uint32_t a, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void st_cl_u32(uint32_t a, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cl_u8(uint32_t a, uint32_t v) {
    asm volatile("st.shared::cluster.u8 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int DPLC, int NW>
__global__ void __launch_bounds__((NW + 1) * 32, 2)
replay_cluster_kernel(ss_dag_set D, ClusterArgs A, ReplayArgs R) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int SCQ = DPLC * 32;
    constexpr int NC = NW * 32;
    constexpr int NT = NC + 32;
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    const int CL = A.cl;
    const int q = (int)cluster_rank();
    const int dag = blockIdx.x / CL;
    const int qlo = q * SCQ;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int l0 = D.layer_ptr[dag];
    const int nl = D.layer_ptr[dag + 1] - l0;
    const int nblk = nl - 1;
    const int W = A.w;
    const int SC = A.sc;
    MetaLayout ml{nblk, A.s_cap, D.max_gpus};

    double* T = reinterpret_cast<double*>(smem + A.off_T);            // [s_rows][W]: own destination columns
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + A.off_full);
    unsigned char* meta_s = smem + A.off_meta;
    double* part_v = reinterpret_cast<double*>(smem + A.off_part);     // [2][NW][SCQ]
    int16_t* part_i = reinterpret_cast<int16_t*>(part_v + 2 * NW * SCQ);
    double* src_c = reinterpret_cast<double*>(smem + A.off_src);       // [2][SC] source costs by position
    int* src_r = reinterpret_cast<int*>(src_c + 2 * SC);                // [2][SC] their Tq row byte offsets
    uint8_t* bp = smem + A.off_bp;                                      // [L][SC] (CTA 0)
    int* picks = reinterpret_cast<int*>(smem + A.off_picks);
    double* tau_g = reinterpret_cast<double*>(smem + A.off_tau);
    int* occ_s = reinterpret_cast<int*>(smem + A.off_occ);
    int* stamp = reinterpret_cast<int*>(smem + A.off_stamp);
    int* slot_gpu = reinterpret_cast<int*>(smem + A.off_slotgpu);
    int* col_len = reinterpret_cast<int*>(smem + A.off_cl);
    int* coff = reinterpret_cast<int*>(smem + A.off_coff);
    double* red_v = reinterpret_cast<double*>(smem + A.off_red);       // [NW] CTA-local argmin partials
    int* red_i = reinterpret_cast<int*>(smem + A.off_red + NW * 8);
    double* cred_v = reinterpret_cast<double*>(smem + A.off_cred);     // [8] per-CTA argmin partials (CTA 0)
    int* cred_i = reinterpret_cast<int*>(smem + A.off_cred + 64);
    int* clist = reinterpret_cast<int*>(smem + A.off_clist);           // [1 + L]: the chain's distinct GPUs
    volatile int* misc = reinterpret_cast<int*>(smem + A.off_misc);    // [0] status [1] aux [3] chunks/req
    double* base_s = reinterpret_cast<double*>(smem + A.off_base);
    double* pow_s = reinterpret_cast<double*>(smem + A.off_pow);
    int* rel = reinterpret_cast<int*>(smem + A.off_rel);
    uint8_t* seg_end = smem + A.off_seg;                                // [NW][SC]
    int* seg_start = reinterpret_cast<int*>(smem + A.off_seg + NW * SC);

    // ---- setup (every CTA of the cluster reaches the same decisions from the same inputs) -------------
    const uint8_t* meta_g = A.meta + (int64_t)dag * A.meta_stride;
    if (tid == 0) {
        misc[0] = SS_OK;
        misc[1] = 0;
        if (R.st.status[dag] != SS_OK) misc[0] = -1;
        for (int b = 0; b < A.nbuf; ++b) mbar_init(&full[b], 1);
        fence_mbar_init();
    }
    {
        const int4* srcv = reinterpret_cast<const int4*>(meta_g);
        int4* dstv = reinterpret_cast<int4*>(meta_s);
        for (int x = tid; x < A.meta_bytes / 16; x += blockDim.x) dstv[x] = srcv[x];
        for (int l = tid; l < nl; l += blockDim.x) {
            col_len[l] = D.col_len[l0 + l];
            coff[l] = D.col_off[l0 + l];
        }
        const int gb = R.st.gpu_ptr[dag], gn = R.st.gpu_ptr[dag + 1] - gb;
        for (int g = tid; g < gn; g += blockDim.x) base_s[g] = R.st.base_tau[gb + g];
        for (int o = tid; o < A.pow_len; o += blockDim.x) pow_s[o] = R.occpow[o];
    }
    __syncthreads();
    const int32_t* hdr = reinterpret_cast<const int32_t*>(meta_s);
    const BlkMeta* bm = reinterpret_cast<const BlkMeta*>(meta_s + ml.off_blk());
    const int16_t* ins = reinterpret_cast<const int16_t*>(meta_s + ml.off_ins());
    const uint8_t* src_map = meta_s + ml.off_src();
    const int Wp = hdr[1];
    const int upc = max(1, A.stage_bytes / (Wp * 8));
    const int tw = min(Wp, A.s_rows);
    if (tid == 0 && misc[0] == SS_OK) {
        if (hdr[0] > A.s_rows || hdr[0] > SC || nl < 2) misc[0] = SS_BAD_INPUT;
        int chunks = 0;
        for (int b = 1; b < nblk; ++b) chunks += (2 * bm[b].n_ins + upc - 1) / upc;
        misc[3] = chunks;
    }
    __syncthreads();
    if (misc[0] != SS_OK) {
        if (q == 0 && tid == 0 && misc[0] != -1) { R.st.status[dag] = misc[0]; R.st.aux[dag] = misc[1]; }
        return;                                                  // uniform over the cluster
    }
    cluster_sync_all();                                          // every CTA started before any DSMEM write
    const int n_req = R.n_req;
    const double* stream_g = A.stream + (int64_t)dag * A.stream_stride;

    // ========================= producer: TMA ring + apply(1..nblk-1) of own columns ==========
    if (warp == NW) {
        const int64_t total = (int64_t)n_req * misc[3];
        int64_t issued = 0;
        int ib = 1, iu0 = 0;
        auto issue_next = [&](int buf) {
            while (ib < nblk && iu0 >= 2 * bm[ib].n_ins) { ++ib; iu0 = 0; }
            if (ib >= nblk) { ib = 1; iu0 = 0; while (ib < nblk && 2 * bm[ib].n_ins == 0) ++ib; }
            const BlkMeta m = bm[ib];
            const int nu = min(upc, 2 * m.n_ins - iu0);
            const uint32_t bytes = (uint32_t)nu * Wp * 8;
            fence_proxy_async_smem();
            mbar_expect_tx(&full[buf], bytes);
            bulk_g2s(smem + A.off_stage + (size_t)buf * A.stage_bytes, stream_g + (int64_t)(m.unit_start + iu0) * Wp,
                     bytes, &full[buf]);
            iu0 += nu;
            ++issued;
        };
        if (lane == 0)
            for (int b = 0; b < A.nbuf && issued < total; ++b) issue_next(b);
        int cbuf = 0;
        uint32_t cphase = 0;
        int64_t consumed = 0;
        for (int r = 0; r < n_req; ++r) {
            cluster_sync_all();                                  // request start
            if (misc[0] != SS_OK) break;
            for (int b = 0; b < nblk; ++b) {
                cluster_sync_all();                              // source table of boundary b complete
                if (b + 1 < nblk) {
                    const BlkMeta m = bm[b + 1];
                    const int units = 2 * m.n_ins;
                    for (int u0 = 0; u0 < units; u0 += upc) {
                        const int nu = min(upc, units - u0);
                        mbar_wait(&full[cbuf], cphase);
                        const double* stg = reinterpret_cast<const double*>(smem + A.off_stage +
                                                                            (size_t)cbuf * A.stage_bytes);
                        for (int ul = 0; ul < nu; ++ul) {
                            const int u = u0 + ul;
                            const int slot = ins[2 * (m.ins_start + (u >> 1))];
                            const double* su = stg + ul * Wp;
                            if (u & 1) {                         // column of the entering GPU: own slots only
                                const int c = slot - qlo;
                                if (c >= 0 && c < SCQ)
                                    for (int x = lane; x < tw; x += 32) T[x * W + c] = su[x];
                            } else {                             // row: this CTA's destination range
#pragma unroll
                                for (int d = 0; d < DPLC; ++d) {
                                    const int c = lane + 32 * d;
                                    if (qlo + c < tw) T[slot * W + c] = su[qlo + c];
                                }
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
                all_sync(NT);                                    // boundary b done locally
            }
            cluster_sync_all();                                  // epilogue: argmin partials at CTA 0
            cluster_sync_all();                                  // epilogue: chain broadcast
        }
        while (consumed < issued) {
            mbar_wait(&full[cbuf], cphase);
            ++consumed;
            if (++cbuf == A.nbuf) { cbuf = 0; cphase ^= 1u; }
        }
        __syncwarp();
        cluster_sync_all();                                      // matches the consumers' exit barrier
        return;
    }

    // ========================= consumers ======================================
    const int gbase = R.st.gpu_ptr[dag];
    const int ng = R.st.gpu_ptr[dag + 1] - gbase;
    const int window = R.window;
    const int64_t req0 = R.st.next_req[dag];
    const int ring_stride = D.max_layers + 1;
    int* ring = R.st.ring + (int64_t)dag * (window > 0 ? window : 1) * ring_stride;
    for (int g = tid; g < ng; g += NC) {
        occ_s[g] = R.st.occ[gbase + g];
        stamp[g] = 0;
    }
    auto issue_initial_rows = [&]() {
        const BlkMeta m = bm[0];
        const double* s0 = stream_g + (int64_t)m.unit_start * Wp;
        for (int u = warp; u < m.n_ins; u += NW) {
            const int slot = ins[2 * (m.ins_start + u)];
            const double* su = s0 + (int64_t)u * Wp;
            for (int c = lane; c < SCQ; c += 32)
                if (qlo + c < tw) cp_async8(T + slot * W + c, su + qlo + c);
        }
    };
    // the release list of the first request comes from the ring in global memory (written by an earlier
    // launch); later ones are sent by CTA 0 with each chain (the ring is CTA 0's)
    if (n_req > 0) {
        if (window > 0 && req0 >= window) {
            const int* slot = ring + (int64_t)(req0 % window) * ring_stride;
            for (int k = tid; k < ring_stride; k += NC) rel[k] = slot[k];
        } else if (tid == 0) {
            rel[0] = 0;
        }
        issue_initial_rows();
    }
    const uint32_t bp_0 = peer_addr(bp, 0);
    int done = 0;
    consumer_sync(NC);

    // stage(c) for c >= 1: the owner of each position merges its range partials of boundary c-1, adds tau and
    // broadcasts (cost, row) to every CTA (table c & 1); c == 0: every CTA fills the whole table locally
    auto stage = [&](int c) {
        const int rs = col_len[c];
        const int buf = c & 1;
        if (c == 0) {
            for (int p = tid; p < rs; p += NC) {
                const int sl = src_map[p];
                src_c[p] = tau_g[slot_gpu[sl]];
                src_r[p] = sl * W * 8;
            }
            return;
        }
        const double* pv = part_v + ((c - 1) & 1) * NW * SCQ;
        const int16_t* pi = part_i + ((c - 1) & 1) * NW * SCQ;
        for (int p = tid; p < rs; p += NC) {
            const int sl = src_map[c * A.s_cap + p];
            const int lc = sl - qlo;
            if (lc < 0 || lc >= SCQ) continue;                       // another CTA owns this destination
            double v = pv[lc];
            int i = pi[lc];
#pragma unroll
            for (int w = 1; w < NW; ++w) lex_min(v, i, pv[w * SCQ + lc], (int)pi[w * SCQ + lc]);
            if (i == PART_NONE) i = 0;
            const double cst = __dadd_rn(v, tau_g[slot_gpu[sl]]);
            st_cl_u8(bp_0 + (c - 1) * SC + p, (uint32_t)i);
            for (int k = 0; k < CL; ++k) {
                st_cl_f64(peer_addr(src_c + buf * SC + p, k), cst);
                st_cl_u32(peer_addr(src_r + buf * SC + p, k), (uint32_t)(sl * W * 8));
            }
        }
    };

    for (int r = 0; r < n_req; ++r) {
        const int64_t req = req0 + r;
        if (misc[0] == SS_OK) {
            const BlkMeta m = bm[0];
            for (int k = tid; k < m.n_ins; k += NC) slot_gpu[ins[2 * (m.ins_start + k)]] = ins[2 * (m.ins_start + k) + 1];
            cp_async_wait_all();                                     // initial rows
            consumer_sync(NC);
            if (window > 0 && req >= window) {
                const int cnt = rel[0];
                for (int k = tid; k < cnt; k += NC) occ_s[rel[1 + k]] -= 1;
            }
            consumer_sync(NC);
            for (int g = tid; g < ng; g += NC) {
                const int o = occ_s[g];
                if (o < 0 || o >= R.occpow_len) {
                    atomicExch((int*)&misc[0], o < 0 ? SS_OCC_UNDERFLOW : SS_BAD_INPUT);
                    misc[1] = g;
                }
                const int oc = o < 0 ? 0 : (o >= R.occpow_len ? R.occpow_len - 1 : o);
                tau_g[g] = base_s[g] * (oc < A.pow_len ? pow_s[oc] : R.occpow[oc]);
            }
        }
        cluster_sync_all();                                          // request start
        if (misc[0] != SS_OK) break;

        for (int b = 0; b < nblk; ++b) {
            stage(b);                                                // tau / slot_gpu / partials of b-1: visible
            cluster_sync_all();                                      // the source table of b is complete
            const int rs = col_len[b];
            const int p0 = warp * rs / NW, n = (warp + 1) * rs / NW - p0;
            const double* cw = src_c + (b & 1) * SC;
            const int* rw = src_r + (b & 1) * SC;
            double v[DPLC];
            int ix[DPLC];
#pragma unroll
            for (int d = 0; d < DPLC; ++d) { v[d] = INF; ix[d] = PART_NONE; }
            const char* Tb = reinterpret_cast<const char*>(T + lane);
            for (int k = 0; k < n; ++k) {
                const int p = p0 + k;
                relax_row<DPLC>(reinterpret_cast<const double*>(Tb + rw[p]), cw[p], p, v, ix);
            }
            double* pv = part_v + (b & 1) * NW * SCQ + warp * SCQ;
            int16_t* pi = part_i + (b & 1) * NW * SCQ + warp * SCQ;
#pragma unroll
            for (int d = 0; d < DPLC; ++d) {
                pv[d * 32 + lane] = v[d];
                pi[d * 32 + lane] = (int16_t)ix[d];
            }
            all_sync(NT);                                            // partials visible; the producer applied b+1
        }
        if (r + 1 < n_req) issue_initial_rows();                     // this CTA's tile is no longer read

        // ---- last column: owned costs, CTA argmin partial -> CTA 0 ----------------------------------
        {
            const int c = nblk;
            const int rs = col_len[c];
            const double* pv = part_v + ((c - 1) & 1) * NW * SCQ;
            const int16_t* pi = part_i + ((c - 1) & 1) * NW * SCQ;
            double bv = INF;
            int bi = IDX_NONE;
            for (int p = tid; p < rs; p += NC) {
                const int sl = src_map[c * A.s_cap + p];
                const int lc = sl - qlo;
                if (lc < 0 || lc >= SCQ) continue;
                double v = pv[lc];
                int i = pi[lc];
#pragma unroll
                for (int w = 1; w < NW; ++w) lex_min(v, i, pv[w * SCQ + lc], (int)pi[w * SCQ + lc]);
                if (i == PART_NONE) i = 0;
                const double cst = __dadd_rn(v, tau_g[slot_gpu[sl]]);
                st_cl_u8(bp_0 + (c - 1) * SC + p, (uint32_t)i);
                lex_min(bv, bi, cst, p);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double v2 = __shfl_xor_sync(0xffffffffu, bv, o);
                const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
                lex_min(bv, bi, v2, i2);
            }
            if (lane == 0) { red_v[warp] = bv; red_i[warp] = bi; }
            consumer_sync(NC);
            if (tid == 0) {
                for (int w = 1; w < NW; ++w) lex_min(bv, bi, red_v[w], red_i[w]);
                st_cl_f64(peer_addr(cred_v + q, 0), bv);
                st_cl_u32(peer_addr(cred_i + q, 0), (uint32_t)bi);
            }
        }
        cluster_sync_all();                                          // argmin partials + backpointers at CTA 0
        if (q == 0) {
            if (tid == 0) {
                double v = cred_v[0];
                int idx = cred_i[0];
                for (int k = 1; k < CL; ++k) lex_min(v, idx, cred_v[k], cred_i[k]);
                if (!(v <= DBL_MAX)) {
                    for (int k = 0; k < CL; ++k) st_cl_u32(peer_addr((const void*)&misc[0], k), (uint32_t)SS_NO_PATH);
                } else {
                    picks[nl - 1] = idx;
                    seg_start[NW] = idx;
                }
                if (R.out.cost) R.out.cost[(int64_t)dag * n_req + r] = v;
            }
            consumer_sync(NC);
            if (misc[0] == SS_OK) {
                {   // segment-parallel backtrack over the consumer warps
                    const int blo = warp * nblk / NW, bhi = (warp + 1) * nblk / NW;
                    for (int st = lane; st < SC; st += 32) {
                        int p = st;
                        for (int b = bhi - 1; b >= blo; --b) p = min((int)bp[b * SC + p], SC - 1);
                        seg_end[warp * SC + st] = (uint8_t)p;
                    }
                }
                consumer_sync(NC);
                if (tid == 0) {
                    int p = seg_start[NW];
                    for (int w = NW - 1; w >= 0; --w) {
                        seg_start[w] = p;
                        p = seg_end[w * SC + p];
                    }
                }
                consumer_sync(NC);
                if (lane == 0) {
                    const int blo = warp * nblk / NW, bhi = (warp + 1) * nblk / NW;
                    int p = seg_start[warp];
                    for (int b = bhi - 1; b >= blo; --b) {
                        p = bp[b * SC + p];
                        picks[b] = p;
                    }
                }
                consumer_sync(NC);
                // load update: +1 per distinct GPU (CTA 0's stamps), ring, outputs; the list goes to the peers
                const int tag = (int)(req & 0x3fffffff) + 1;
                int* slot = window > 0 ? ring + (int64_t)(req % window) * ring_stride : nullptr;
                if (tid == 0) clist[0] = 0;
                consumer_sync(NC);
                uint64_t h = 0;
                for (int l = tid; l < nl; l += NC) {
                    const int g = D.node_gpu[coff[l] + picks[l]];
                    h += ss_splitmix64(((uint64_t)l << 32) | (uint64_t)g);
                    if (R.out.gpus) R.out.gpus[((int64_t)dag * n_req + r) * D.max_layers + l] = (int16_t)g;
                    if (atomicExch(&stamp[g], tag) != tag && window != 0) {
                        occ_s[g] += 1;
                        const int at = atomicAdd(&clist[0], 1);
                        clist[1 + at] = g;
                        if (slot) slot[1 + at] = g;
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
                const int cnt = clist[0];
                if (tid == 0 && slot) slot[0] = cnt;
                for (int k = 1; k < CL; ++k)
                    for (int x = tid; x <= cnt; x += NC) st_cl_u32(peer_addr(clist + x, k), (uint32_t)clist[x]);
                // the next request's release list (chain req+1-W, already in CTA 0's ring) for every CTA
                if (r + 1 < n_req && window > 0 && req + 1 >= window) {
                    consumer_sync(NC);
                    const int* ns = ring + (int64_t)((req + 1) % window) * ring_stride;
                    const int ncnt = ns[0];
                    for (int k = 0; k < CL; ++k)
                        for (int x = tid; x <= ncnt; x += NC) st_cl_u32(peer_addr(rel + x, k), (uint32_t)ns[x]);
                }
            }
        }
        cluster_sync_all();                                          // the chain's distinct GPUs everywhere
        if (misc[0] != SS_OK) continue;                              // the next request-start barrier ends it
        if (q != 0) {
            const int cnt = clist[0];
            for (int k = tid; k < cnt; k += NC) occ_s[clist[1 + k]] += 1;
        }
        ++done;
    }
    cp_async_wait_all();
    if (q == 0) {
        for (int g = tid; g < ng; g += NC) R.st.occ[gbase + g] = occ_s[g];
        if (tid == 0) {
            R.st.next_req[dag] = req0 + done;
            if (misc[0] != SS_OK) { R.st.status[dag] = misc[0]; R.st.aux[dag] = misc[1]; }
        }
    }
    __syncwarp();
    cluster_sync_all();                                              // no CTA exits while peers may write to it
}

inline int align_up(int x, int a) { return (x + a - 1) / a * a; }

constexpr int kSmemPerSM = 228 * 1024;
constexpr int kSmemPerCtaReserved = 1024;

}  // namespace

extern "C" int64_t ss_slot_meta_bytes(int32_t layers, int32_t n_gpus, int32_t s_cap) {
    MetaLayout ml{layers - 1, s_cap, n_gpus};
    return ml.bytes();
}

extern "C" int ss_slot_program(int32_t n_scen, int32_t layers, int32_t n_gpus, const int32_t* slice_lo,
                               const int32_t* slice_hi, int64_t slice_stride, const uint8_t* leave, const double* rtt,
                               const int64_t* jitter_seed, int32_t s_cap, int64_t meta_stride, int64_t stream_stride,
                               uint8_t* meta, double* stream, int32_t* s_used, int32_t* status, void* stream_h) {
    if (n_scen <= 0) return SS_OK;
    if (layers < 2 || n_gpus < 1 || s_cap < 32 || s_cap > 256 || (s_cap & 31)) return SS_BAD_INPUT;
    if (meta_stride < ss_slot_meta_bytes(layers, n_gpus, s_cap) || (meta_stride & 15)) return SS_BAD_INPUT;
    const int smem = ((n_gpus + 7) / 8) * 8 * 2 + (((layers - 1) * s_cap + 7) / 8) * 8 * 2 + (layers + 1) * 8 +
                     n_gpus * 8 + 64;
    if (smem > 200 * 1024) return SS_BAD_INPUT;
    if (cudaFuncSetAttribute(slot_program_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return SS_CUDA_ERROR;
    slot_program_kernel<<<n_scen, 256, smem, ss_stream(stream_h)>>>(layers, n_gpus, slice_lo, slice_hi, slice_stride,
                                                                    leave, rtt,
                                                                    jitter_seed, s_cap, meta_stride, stream_stride,
                                                                    meta, stream, s_used, status);
    SS_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_replay_slots(const ss_dag_set* dags, const uint8_t* meta, int64_t meta_stride, const double* stream,
                               int64_t stream_stride, int32_t s_cap, int32_t s_rows, const ss_replay_state* st,
                               const double* occpow, int32_t occpow_len, int32_t window, int32_t n_req,
                               const ss_replay_out* out, void* stream_h) {
    if (!dags || !st || !occpow || occpow_len < 1 || n_req < 1 || !meta || !stream) return SS_BAD_INPUT;
    const ss_dag_set& D = *dags;
    if (D.n_dags <= 0) return SS_OK;
    if (s_cap < 32 || s_cap > 256 || (s_cap & 31) || s_rows < 1 || s_rows > s_cap || D.max_layers < 2) return SS_BAD_INPUT;
    const int dpl = s_cap / 32;
    // 4 source ranges: measured best on B200 (C4: 2.8e6 sel/s vs 2.65e6 with 8 -- the per-position merge of
    // NW partials and the per-warp fixed costs outgrow the shorter relax loops)
    // 4 source ranges: measured best on B200 with the in-warp apply (C4: 2.8e6 sel/s vs 2.65e6 with 8 -- the
    // per-position merge of NW partials and the per-warp fixed costs outgrow the shorter relax loops);
    // SS_SLOT_NW = 6 / 8 selects the wider split at DPL = 3 (experiments)
    int nw = 4;
    if (const char* e = getenv("SS_SLOT_NW")) {
        const int v = atoi(e);
        if ((v == 6 || v == 8) && dpl == 3) nw = v;
    }
    SlotArgs A{};
    A.meta = meta;
    A.meta_stride = meta_stride;
    A.stream = stream;
    A.stream_stride = stream_stride;
    A.s_rows = s_rows;
    // row pitch >= s_rows with W = 2 (mod 4): rows are 16-B aligned (bulk copies land the initial rows straight in
    // T) and the producer's column writes see at most 2-way bank conflicts
    A.w = s_rows;
    while (A.w % 4 != 2) ++A.w;
    MetaLayout ml{D.max_layers - 1, s_cap, D.max_gpus};
    A.meta_bytes = ml.bytes();
    auto layout = [&](int nbuf, int stage) {
        A.nbuf = nbuf;
        A.stage_bytes = stage;
        int o = 0;
        A.off_T = o;       o += align_up((s_rows * A.w + s_cap) * 8, 128);
        A.off_stage = o;   o += A.nbuf * A.stage_bytes;
        A.off_full = o;    o += 64;
        A.off_empty = o;   o += 64;
        A.off_meta = o;    o += align_up(A.meta_bytes, 16);
        A.off_part = o;    o += 2 * nw * s_cap * 10;
        A.off_bp = o;      o += align_up(D.max_layers * s_cap, 16);
        A.off_picks = o;   o += align_up(D.max_layers * 4, 16);
        A.off_tau = o;     o += align_up(D.max_gpus * 8, 16);
        A.off_occ = o;     o += align_up(D.max_gpus * 4, 16);
        A.off_stamp = o;   o += align_up(D.max_gpus * 4, 16);
        A.off_slotgpu = o; o += s_cap * 4;
        A.off_cl = o;      o += align_up(D.max_layers * 4, 16);
        A.off_red = o;     o += align_up(nw * 12, 16);
        A.off_misc = o;    o += 64;
        A.off_base = o;    o += align_up(D.max_gpus * 8, 16);
        A.pow_len = occpow_len < 256 ? occpow_len : 256;
        A.off_pow = o;     o += align_up(A.pow_len * 8, 16);
        A.off_rel = o;     o += align_up((D.max_layers + 1) * 4, 16);
        A.off_coff = o;    o += align_up(D.max_layers * 4, 16);
        A.off_costw = o;   o += nw * (s_cap / nw + 8) * 12;
        A.off_seg = o;     o += align_up(nw * s_cap + nw * 4, 16);
        A.total = o;
    };
    // two CTAs per SM when the staging ring can shrink to fit (>= 2 buffers of >= one unit);
    // otherwise one CTA with the configured ring
    const int unit_min = align_up((s_rows + 1) * 8, 128);
    const int stage_cfg = max(g_stage_bytes, unit_min);
    const int two_cta = kSmemPerSM / 2 - kSmemPerCtaReserved;
    layout(0, 0);
    const int rest = A.total;
    int nb = g_nbuf, st_b = stage_cfg;
    while (nb > 2 && rest + nb * st_b > two_cta) --nb;
    if (rest + nb * st_b > two_cta) st_b = ((two_cta - rest) / 2) / 128 * 128;
    if (st_b >= unit_min) layout(nb, st_b);
    else layout(g_nbuf, stage_cfg);
    if (A.total > 227 * 1024) return SS_BAD_INPUT;
    ReplayArgs R{};
    R.st = *st;
    if (out) R.out = *out;
    R.occpow = occpow;
    R.occpow_len = occpow_len;
    R.window = window;
    R.n_req = n_req;
    cudaStream_t s = ss_stream(stream_h);
    if (R.out.chain_hash) cudaMemsetAsync(R.out.chain_hash, 0, sizeof(uint64_t) * (size_t)D.n_dags * n_req, s);
    const bool prof = getenv("SS_SLOT_PROF") != nullptr;
    if (prof && cudaMalloc(&A.prof, 64 * 8 * sizeof(unsigned long long)) == cudaSuccess)
        cudaMemsetAsync(A.prof, 0, 64 * 8 * sizeof(unsigned long long), s);
    auto run = [&](auto kern, int threads) -> int {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, A.total) != cudaSuccess)
            return SS_CUDA_ERROR;
        kern<<<D.n_dags, threads, A.total, s>>>(D, A, R);
        SS_CHECK_LAUNCH();
        if (A.prof) {
            unsigned long long h[64 * 8];
            cudaMemcpyAsync(h, A.prof, sizeof(h), cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            fprintf(stderr, "slot prof: smem=%d nbuf=%d stage=%d s_rows=%d | per CTA-request cycles, by warp:\n",
                    A.total, A.nbuf, A.stage_bytes, A.s_rows);
            for (int w = 0; w <= nw; ++w) {
                const double d = (double)D.n_dags * n_req;
                fprintf(stderr, "  w%d prologue %.0f relax %.0f apply %.0f barrier %.0f | epilogue: initial-rows %.0f "
                        "argmin+backtrack %.0f chain-update %.0f rest %.0f\n",
                        w, h[w * 8 + 0] / d, h[w * 8 + 1] / d, h[w * 8 + 2] / d, h[w * 8 + 3] / d, h[w * 8 + 7] / d,
                        h[w * 8 + 5] / d, h[w * 8 + 6] / d, h[w * 8 + 4] / d);
            }
            cudaFree(A.prof);
        }
        return SS_OK;
    };
    switch (dpl) {
        case 1: return run(replay_slots_kernel<1, 4>, 5 * 32);
        case 2: return run(replay_slots_kernel<2, 4>, 5 * 32);
        case 3:
            if (nw == 6) return run(replay_slots_kernel<3, 6>, 7 * 32);
            if (nw == 8) return run(replay_slots_kernel<3, 8>, 9 * 32);
            return run(replay_slots_kernel<3, 4>, 5 * 32);
        case 4: return run(replay_slots_kernel<4, 4>, 5 * 32);
        case 5: return run(replay_slots_kernel<5, 4>, 5 * 32);
        case 6: return run(replay_slots_kernel<6, 4>, 5 * 32);
        case 7: return run(replay_slots_kernel<7, 4>, 5 * 32);
        default: return run(replay_slots_kernel<8, 4>, 5 * 32);
    }
}

extern "C" int ss_set_slot_staging(int32_t stage_bytes, int32_t n_buffers) {
    if (stage_bytes > 0) g_stage_bytes = (stage_bytes + 127) / 128 * 128;
    if (n_buffers > 0) g_nbuf = n_buffers > 8 ? 8 : n_buffers;
    return SS_OK;
}

// Cluster slot replay (replay_cluster_kernel): same program, state, outputs and op script as ss_replay_slots;
// the scenario's slot tile is split by destination slots over a cluster of ceil(s_rows / (32 * dplc)) CTAs
// (<= 8).  dplc = 1 or 2 destination slots per lane; 0 = default (1; env SS_CLUSTER_DPL overrides).
extern "C" int ss_replay_slots_cluster(const ss_dag_set* dags, const uint8_t* meta, int64_t meta_stride,
                                       const double* stream, int64_t stream_stride, int32_t s_cap, int32_t s_rows,
                                       const ss_replay_state* st, const double* occpow, int32_t occpow_len,
                                       int32_t window, int32_t n_req, const ss_replay_out* out, int32_t dplc,
                                       void* stream_h) {
    if (!dags || !st || !occpow || occpow_len < 1 || n_req < 1 || !meta || !stream) return SS_BAD_INPUT;
    const ss_dag_set& D = *dags;
    if (D.n_dags <= 0) return SS_OK;
    if (s_cap < 32 || s_cap > 256 || (s_cap & 31) || s_rows < 1 || s_rows > s_cap || D.max_layers < 2)
        return SS_BAD_INPUT;
    if (dplc <= 0) {
        const char* e = getenv("SS_CLUSTER_DPL");
        dplc = e ? atoi(e) : 1;
    }
    if (dplc != 1 && dplc != 2) return SS_BAD_INPUT;
    const int scq = 32 * dplc;
    const int cl = (s_rows + scq - 1) / scq;
    if (cl < 1 || cl > 8) return SS_BAD_INPUT;
    const int nw = 4;
    ClusterArgs A{};
    A.meta = meta;
    A.meta_stride = meta_stride;
    A.stream = stream;
    A.stream_stride = stream_stride;
    A.s_rows = s_rows;
    A.w = scq + 1;                                       // odd pitch: the producer's column writes are conflict-free
    A.cl = cl;
    A.sc = cl * scq;
    A.s_cap = s_cap;
    MetaLayout ml{D.max_layers - 1, s_cap, D.max_gpus};
    A.meta_bytes = ml.bytes();
    const int SC = A.sc;
    auto layout = [&](int nbuf, int stage) {
        A.nbuf = nbuf;
        A.stage_bytes = stage;
        int o = 0;
        A.off_T = o;       o += align_up(s_rows * A.w * 8, 128);
        A.off_stage = o;   o += A.nbuf * A.stage_bytes;
        A.off_full = o;    o += 64;
        A.off_meta = o;    o += align_up(A.meta_bytes, 16);
        A.off_part = o;    o += align_up(2 * nw * scq * 10, 16);
        A.off_src = o;     o += align_up(2 * SC * 12, 16);
        A.off_bp = o;      o += align_up(D.max_layers * SC, 16);
        A.off_picks = o;   o += align_up(D.max_layers * 4, 16);
        A.off_tau = o;     o += align_up(D.max_gpus * 8, 16);
        A.off_occ = o;     o += align_up(D.max_gpus * 4, 16);
        A.off_stamp = o;   o += align_up(D.max_gpus * 4, 16);
        A.off_slotgpu = o; o += align_up(SC * 4, 16);
        A.off_cl = o;      o += align_up(D.max_layers * 4, 16);
        A.off_coff = o;    o += align_up(D.max_layers * 4, 16);
        A.off_red = o;     o += align_up(nw * 12, 16);
        A.off_cred = o;    o += 128;
        A.off_clist = o;   o += align_up((D.max_layers + 1) * 4, 16);
        A.off_misc = o;    o += 64;
        A.off_base = o;    o += align_up(D.max_gpus * 8, 16);
        A.pow_len = occpow_len < 256 ? occpow_len : 256;
        A.off_pow = o;     o += align_up(A.pow_len * 8, 16);
        A.off_rel = o;     o += align_up((D.max_layers + 1) * 4, 16);
        A.off_seg = o;     o += align_up(nw * SC + (nw + 1) * 4, 16);
        A.total = o;
    };
    const int unit_min = align_up((s_rows + 1) * 8, 128);
    layout(2, max(g_stage_bytes, unit_min));
    if (A.total > 227 * 1024) return SS_BAD_INPUT;
    ReplayArgs R{};
    R.st = *st;
    if (out) R.out = *out;
    R.occpow = occpow;
    R.occpow_len = occpow_len;
    R.window = window;
    R.n_req = n_req;
    cudaStream_t s = ss_stream(stream_h);
    if (R.out.chain_hash) cudaMemsetAsync(R.out.chain_hash, 0, sizeof(uint64_t) * (size_t)D.n_dags * n_req, s);
    auto run = [&](auto kern) -> int {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, A.total) != cudaSuccess)
            return SS_CUDA_ERROR;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(D.n_dags * cl), 1, 1);
        cfg.blockDim = dim3((nw + 1) * 32, 1, 1);
        cfg.dynamicSmemBytes = A.total;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = cl;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, kern, D, A, R) != cudaSuccess) return SS_CUDA_ERROR;
        SS_CHECK_LAUNCH();
        return SS_OK;
    };
    return dplc == 1 ? run(replay_cluster_kernel<1, 4>) : run(replay_cluster_kernel<2, 4>);
}
