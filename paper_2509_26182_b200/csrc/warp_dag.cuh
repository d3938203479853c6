// Warp-resident DAG helpers shared by the warp replay, admission and simulator kernels.
//
// One CTA owns one scenario: its host columns, node ids and edge blocks (the ss_dag_edges layout, <= 32
// hosts per column) live in shared memory.  warp_route() runs one chain DP (router.py:163-197) on a single
// warp without a CTA barrier; mw_route() spreads the destinations over NWD warps (one barrier per boundary).
#pragma once

#include <float.h>

#include "ss_common.cuh"

namespace ssw {

constexpr int NONE = 0x7fffffff;
constexpr unsigned FULL = 0xffffffffu;

struct WarpLayout {
    int e_cap, ring_len, pow_len;
    int mat_dim;       // > 0: the scenario's whole RTT matrix (mat_dim^2 fp64) replaces the edge blocks in E
    int mat_pitch;     // its row pitch in E: odd (mat_dim | 1), so lanes gathering one column from different
                       // source rows (mw_route: 4 source lanes per destination) hit different banks
    int pad;           // > 0: padded edge blocks (pad_route): block b = E + b * pad^2, E_b[i * pad + j], +inf padded
    int off_E, off_node, off_cl, off_noff, off_eoff, off_bp, off_picks, off_tau, off_base, off_occ, off_stamp,
        off_ring, off_pow, off_cost, off_kv, off_tcap, off_dst, off_path, total;
};

__device__ __forceinline__ void lexmin(double& v, int& i, double v2, int i2) {
    if (v2 < v || (v2 == v && i2 < i)) { v = v2; i = i2; }
}

// Stages one DAG's host columns and edge blocks into shared memory (compact, row-major per boundary), or --
// matrix mode, A.mat_dim > 0 -- the scenario's RTT matrix `mat` (mat_dim x mat_dim, the values the edge blocks
// are gathered from: E_b[i][j] = M[node_i][node_j]), which is smaller whenever the pool has fewer GPUs than
// sqrt(sum of R_b R_{b+1}).  Returns false (warp-uniform) when a column exceeds 32 hosts or the edges exceed
// the layout.
__device__ inline bool stage_dag(const ss_dag_set& D, const WarpLayout& A, int l0, int nl, double* E, int* node, int* cl,
                          int* noff, int* eoff, int lane, const double* mat = nullptr) {
    const int nblk = nl - 1;
    for (int l = lane; l < nl; l += 32) cl[l] = D.col_len[l0 + l];
    __syncwarp();
    if (lane == 0) {
        int n = 0, e = 0, bad = 0;
        for (int l = 0; l < nl; ++l) {
            if (cl[l] > 32) bad = 1;
            noff[l] = n;
            n += cl[l];
            if (l < nblk) {
                eoff[l] = e;
                e += cl[l] * cl[l + 1];
            }
        }
        if (A.pad > 0) {
            if ((int64_t)nblk * A.pad * A.pad > A.e_cap) bad = 1;
            for (int l = 0; l < nl; ++l) if (cl[l] > A.pad) bad = 1;
        } else if (A.mat_dim == 0 && e > A.e_cap) {
            bad = 1;
        }
        cl[nl] = bad;                                            // scratch flag (cl has max_layers + 1 slots)
    }
    __syncwarp();
    if (cl[nl]) return false;
    for (int l = 0; l < nl; ++l) {
        const int len = cl[l];
        if (lane < len) node[noff[l] + lane] = D.node_gpu[D.col_off[l0 + l] + lane];
        if (l < nblk && A.pad > 0) {
            const double INF = __longlong_as_double(0x7ff0000000000000ll);
            const double* src = D.edge_val + D.edge_off[l0 + l];
            const int P = A.pad, rd = cl[l + 1];
            double* dst = E + (int64_t)l * P * P;
            for (int q = lane; q < P * P; q += 32) {
                const int i = q / P, j = q - i * P;
                dst[q] = (i < len && j < rd) ? src[i * rd + j] : INF;
            }
        } else if (l < nblk && A.mat_dim == 0) {
            const double* src = D.edge_val + D.edge_off[l0 + l];
            const int cnt = len * cl[l + 1];
            for (int q = lane; q < cnt; q += 32) E[eoff[l] + q] = src[q];
        }
    }
    if (A.mat_dim > 0) {
        const int n = A.mat_dim, P = A.mat_pitch;
        for (int q = lane; q < n * n; q += 32) {
            const int r = q / n;
            E[r * P + (q - r * n)] = mat[q];
        }
    }
    __syncwarp();
    return true;
}

// pad_route's destination table: dst[b * P + j] = the GPU of position j in column b + 1 (its tau index), or
// `sentinel` (a tau slot holding +inf) past the column and for the two spare rows b = nblk, nblk + 1 that the
// two-boundary-ahead prefetch reads.  Called by one warp after stage_dag.
__device__ inline void stage_pad_dst(const int* node, const int* cl, const int* noff, int nblk, int P, int sentinel,
                                     int* dst, int lane) {
    for (int q = lane; q < (nblk + 2) * P; q += 32) {
        const int b = q / P, j = q - b * P;
        dst[q] = (b < nblk && j < cl[b + 1]) ? node[noff[b + 1] + j] : sentinel;
    }
    __syncwarp();
}

// Chain DP of one request on a warp-resident DAG (router.py:163-197): lane j owns host j of the next column;
// candidates c_i + E_b[i][j] eight sources at a time (independent loads / DADDs) and a first-index tournament
// (left operand = lower positions, loses only to a strictly smaller right value), groups merged in ascending
// order with the same rule == numpy first-index argmin; cost = (c_i + r_ij) + tau_j.  Returns the chain cost
// (+inf: no path); when finite, picks[l] (shared memory) holds the chosen position of every layer.
template <bool MAT = false>
__device__ inline double warp_route(const double* E, const int* node, const int* cl, const int* noff, const int* eoff,
                             int nblk, const double* tau, double* costs, uint8_t* bp, int* picks, int lane,
                             int G = 0) {
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    double* cur = costs;                                     // 32 hosts + 8 pad for the group loop
    double* nxt = costs + 40;
    cur[lane] = lane < cl[0] ? tau[node[lane]] : INF;
    __syncwarp();
    double c = cur[lane];
    for (int b = 0; b < nblk; ++b) {
        const int rs = cl[b], rd = cl[b + 1];
        const bool act = lane < rd;
        const int dn = act ? node[noff[b + 1] + lane] : 0;
        const double tdst = act ? tau[dn] : 0.0;
        const double* ep = MAT ? E + dn : E + eoff[b] + lane;      // matrix mode: column dn, rows by source node
        const int* sn = node + noff[b];
        double best = INF;
        int bi = 0;                                          // +inf everywhere -> 0 == np.argmin
        for (int g0 = 0; g0 < rs; g0 += 8) {
            double a[8];
            int ix[8];
#pragma unroll
            for (int q = 0; q < 8; q += 2) {
                const double2 c2 = *reinterpret_cast<const double2*>(cur + g0 + q);
                const double e0 = (act && g0 + q < rs) ? (MAT ? ep[sn[g0 + q] * G] : ep[q * rd]) : INF;
                const double e1 = (act && g0 + q + 1 < rs) ? (MAT ? ep[sn[g0 + q + 1] * G] : ep[(q + 1) * rd]) : INF;
                a[q] = __dadd_rn(c2.x, e0);
                a[q + 1] = __dadd_rn(c2.y, e1);
                ix[q] = g0 + q;
                ix[q + 1] = g0 + q + 1;
            }
#pragma unroll
            for (int st = 1; st < 8; st *= 2) {
#pragma unroll
                for (int q = 0; q < 8; q += 2 * st) {
                    if (a[q + st] < a[q]) { a[q] = a[q + st]; ix[q] = ix[q + st]; }
                }
            }
            if (a[0] < best) { best = a[0]; bi = ix[0]; }
            if (!MAT) ep += 8 * rd;
        }
        if (act) bp[b * 32 + lane] = (uint8_t)bi;
        c = act ? __dadd_rn(best, tdst) : INF;
        nxt[lane] = c;
        __syncwarp();
        double* t = cur; cur = nxt; nxt = t;
    }
    double v = c;
    int idx = lane < cl[nblk] ? lane : NONE;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(FULL, v, o);
        const int i2 = __shfl_xor_sync(FULL, idx, o);
        lexmin(v, idx, v2, i2);
    }
    if (lane == 0 && v <= DBL_MAX) {
        int p = idx;
        picks[nblk] = p;
        for (int b = nblk - 1; b >= 0; --b) {
            p = bp[b * 32 + p];
            picks[b] = p;
        }
    }
    __syncwarp();
    return v;
}

// Chain DP of one request over padded edge blocks (A.pad = P = LPD * HS >= every column length): lane group j
// (LPD adjacent lanes, NWD = ceil(P * LPD / 32) warps) owns destination j; lane h of the group scans the HS
// sources [h * HS, (h + 1) * HS).  Block b is E + b * P^2 with E_b[i][j] at i * P + j and +inf past the column
// lengths, so every edge load has a compile-time offset from one per-boundary base and needs no predicate; the
// destination's tau comes from dst[] (stage_pad_dst; +inf sentinel past the column, so c = v + tau is +inf there
// without a branch), loaded two boundaries ahead.  Per lane: HS independent DADDs and a first-index tournament
// (left operands hold lower source indices, the right one wins only on a strict `<`); then log2(LPD) shuffle
// rounds in which the lane holding the lower index range takes its partner only on `<`, the other on `<=`, so
// every lane of the group ends with the same lexicographic (value, index) minimum == numpy's first-index argmin
// (all-+inf resolves to 0) and all of them store it (same value, same address: no predicate).  The costs of a
// column sit in shared memory with every lane group's segment 16-B aligned (slot(i) = (i / HS) * CS + i % HS,
// CS = HS rounded up to even) and are read as double2 broadcasts.  One warp: __syncwarp per boundary; more:
// one named barrier.  The backtrack is segment-parallel: every thread but the last chases one start position of
// a lower segment (recording its path), the last thread chases the chosen end through the top segment, and the
// segment ends are chained by one thread.  Same contract as warp_route.
template <int LPD, int HS, int NWD>
__device__ double pad_route(const double* E, const int* dst, const int* node, const int* cl, int nblk,
                            const double* tau, double* costs, uint8_t* bp, int* picks, uint8_t* path, int L,
                            double* vshare, int* ishare, int tid) {
    constexpr int P = LPD * HS;
    constexpr int CS = (HS + 1) & ~1;
    constexpr int NT = NWD * 32;
    static_assert(LPD == 1 || LPD == 2 || LPD == 4, "pad_route: 1, 2 or 4 lanes per destination");
    static_assert(LPD * CS <= 39 && P <= 32 && P * LPD <= NT, "pad_route: shape");
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    const int j0 = tid / LPD, h = tid % LPD;
    const bool own = j0 < P;                                   // idle lanes store into spare slots
    const int j = own ? j0 : 0;
    const int js = own ? (j / HS) * CS + j % HS : 39;          // cost slot written (39: spare)
    const int jb = own ? j : 31;                               // backpointer column written (31: spare when P < 32)
    auto sync = [] { if (NWD == 1) __syncwarp(); else asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); };
    for (int i = tid; i < P; i += NT) costs[(i / HS) * CS + i % HS] = i < cl[0] ? tau[node[i]] : INF;
    const double* ep = E + (h * HS) * P + j;
    double e[HS];
#pragma unroll
    for (int k = 0; k < HS; ++k) e[k] = nblk > 0 ? ep[k * P] : INF;
    double td = tau[dst[j]];                                   // boundary 0's destination tau
    int dn1 = dst[P + j];                                      // boundary 1's destination GPU
    sync();
    for (int b = 0; b < nblk; ++b) {
        const double* cs = costs + (b & 1) * 40 + h * CS;
        double* nx = costs + ((b & 1) ^ 1) * 40;
        // every cost load issued before the first add (one shared-memory round trip per boundary)
        double c[HS];
#pragma unroll
        for (int k = 0; k + 1 < HS; k += 2) {
            const double2 c2 = *reinterpret_cast<const double2*>(cs + k);
            c[k] = c2.x;
            c[k + 1] = c2.y;
        }
        if (HS & 1) c[HS - 1] = cs[HS - 1];
        double a[HS];
        int ix[HS];
#pragma unroll
        for (int k = 0; k < HS; ++k) {
            a[k] = __dadd_rn(c[k], e[k]);
            ix[k] = k;
        }
#pragma unroll
        for (int w = 1; w < HS; w <<= 1)
#pragma unroll
            for (int k = 0; k + w < HS; k += 2 * w)
                if (a[k + w] < a[k]) { a[k] = a[k + w]; ix[k] = ix[k + w]; }
        double best = a[0];
        int bi = h * HS + ix[0];
#pragma unroll
        for (int o = 1; o < LPD; o <<= 1) {
            const double v2 = __shfl_xor_sync(FULL, best, o);
            const int i2 = __shfl_xor_sync(FULL, bi, o);
            const bool take = (h & o) ? !(best < v2) : (v2 < best);   // partner holds lower indices iff h & o
            best = take ? v2 : best;
            bi = take ? i2 : bi;
        }
        nx[js] = __dadd_rn(best, td);
        bp[b * 32 + jb] = (uint8_t)bi;
        // next boundary's operands (independent of the costs): edges, tau of its destinations, GPUs of b + 2's
        ep += P * P;
        if (b + 1 < nblk) {
#pragma unroll
            for (int k = 0; k < HS; ++k) e[k] = ep[k * P];
        }
        td = tau[dn1];
        dn1 = dst[(b + 2) * P + j];
        sync();
    }
    const double* cl_last = costs + (nblk & 1) * 40;
    if (tid < 32) {
        const int ln = tid;
        double v = ln < cl[nblk] ? cl_last[(ln / HS) * CS + ln % HS] : INF;
        int idx = ln < cl[nblk] ? ln : NONE;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double v2 = __shfl_xor_sync(FULL, v, o);
            const int i2 = __shfl_xor_sync(FULL, idx, o);
            lexmin(v, idx, v2, i2);
        }
        if (ln == 0) {
            *vshare = v;
            ishare[0] = idx;
        }
    }
    if (NWD == 1) __syncwarp(); else __syncthreads();
    const double v = *vshare;
    if (!(v <= DBL_MAX)) return v;
    // segment-parallel backtrack: nlow lower segments x P start positions + one thread for the top segment
    constexpr int NLOW = (NT - 1) / P;
    constexpr int NSEG = NLOW + 1;
    const int top_lo = NLOW * nblk / NSEG;
    if (tid == NT - 1) {
        int p = ishare[0];
        picks[nblk] = p;
        for (int b = nblk - 1; b >= top_lo; --b) {
            p = bp[b * 32 + p];
            picks[b] = p;
        }
    } else if (tid < NLOW * P) {
        const int sg = tid / P;
        const int lo = sg * nblk / NSEG, hi = (sg + 1) * nblk / NSEG;
        int p = tid % P;
        uint8_t* pt = path + tid * L;
        for (int b = hi - 1; b >= lo; --b) {
            p = bp[b * 32 + min(p, 31)];
            pt[b - lo] = (uint8_t)p;
        }
    }
    if (NWD == 1) __syncwarp(); else __syncthreads();
    if (tid == 0) {
        int cur = picks[top_lo];                                 // position at the top segment's low column
        for (int sg = NLOW - 1; sg >= 0; --sg) {
            ishare[1 + sg] = cur;
            cur = path[(sg * P + cur) * L];                       // position at the segment's low column
        }
    }
    if (NWD == 1) __syncwarp(); else __syncthreads();
    for (int b = tid; b < top_lo; b += NT) {
        int sg = 0;
        while (sg + 1 < NLOW && b >= (sg + 1) * nblk / NSEG) ++sg;
        const int lo = sg * nblk / NSEG;
        picks[b] = path[(sg * P + ishare[1 + sg]) * L + (b - lo)];
    }
    if (NWD == 1) __syncwarp(); else __syncthreads();
    return v;
}

inline int align16(int x) { return (x + 15) / 16 * 16; }

// mat_dim > 0 offers matrix mode (the caller has per-scenario RTT matrices of that dimension).  It is taken
// when the matrix is smaller than the edge blocks AND there are more scenarios than SMs: then the smaller
// footprint puts more CTAs on each SM (C2-shaped batches: 2x replay throughput).  With one CTA per SM anyway
// the gather M[node_i][node_j] only adds latency (single-scenario C2: 46.8e3 vs 63.2e3 sel/s), so the edge
// blocks stay.
inline int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) !=
                cudaSuccess || n <= 0)
            n = 148;
    }
    return n;
}

inline bool warp_layout(const ss_dag_set& D, int32_t window, int32_t occpow_len, WarpLayout& A, int mat_dim = 0,
                        int pad = 0) {
    if (D.max_hosts > 32 || D.max_layers < 1 || pad < 0 || pad > 32 || (pad > 0 && pad < D.max_hosts)) return false;
    const int hw = pad > 0 ? pad : D.max_hosts;
    const int64_t e_cap = (int64_t)(D.max_layers > 1 ? D.max_layers - 1 : 0) * hw * hw;
    A.pad = pad;
    A.mat_dim = (pad == 0 && mat_dim > 0 && (int64_t)mat_dim * (mat_dim | 1) < e_cap && D.n_dags > sm_count())
                    ? mat_dim : 0;
    A.mat_pitch = A.mat_dim | 1;
    const int64_t ring_len = window > 0 ? (int64_t)window * (D.max_layers + 1) : 0;
    if (e_cap > (1 << 20) || ring_len > (1 << 20)) return false;
    A.e_cap = (int)e_cap;
    A.ring_len = (int)ring_len;
    A.pow_len = occpow_len < 256 ? occpow_len : 256;
    int o = 0;
    A.off_E = o;      o += align16((A.mat_dim ? A.mat_dim * A.mat_pitch : A.e_cap) * 8);
    A.off_node = o;   o += align16(D.max_layers * D.max_hosts * 4);
    A.off_cl = o;     o += align16((D.max_layers + 1) * 4);
    A.off_noff = o;   o += align16(D.max_layers * 4);
    A.off_eoff = o;   o += align16(D.max_layers * 4);
    A.off_bp = o;     o += align16(D.max_layers * 32);
    A.off_picks = o;  o += align16(D.max_layers * 4);
    A.off_tau = o;    o += align16((D.max_gpus + 1) * 8);          // + the +inf sentinel slot (pad_route)
    A.off_base = o;   o += align16(D.max_gpus * 8);
    A.off_occ = o;    o += align16(D.max_gpus * 4);
    A.off_stamp = o;  o += align16(D.max_gpus * 4);
    A.off_ring = o;   o += align16(A.ring_len * 4);
    A.off_pow = o;    o += align16(A.pow_len * 8);
    A.off_cost = o;   o += 2 * 40 * 8;
    A.off_kv = o;     o += align16(D.max_gpus * 8);
    A.off_tcap = o;   o += align16(D.max_gpus * 8);
    A.off_dst = o;    o += pad > 0 ? align16((D.max_layers + 1) * pad * 4) : 0;
    A.off_path = o;   o += pad > 0 ? align16(128 * D.max_layers) : 0;
    A.total = o;
    return A.total <= 227 * 1024;
}

// Chain DP spread over NWD warps (9..32 hosts per column): warp w owns destinations [8w, 8w+8); lane
// (d, q) = (lane & 7, lane >> 3) takes the sources q, q+4, ..., q+28 of destination 8w+d.  The argmin is a
// lexicographic (value, index) minimum -- identical to numpy's first-index argmin with a strict `<` scan
// (all-+inf resolves to index 0, as np.argmin does) -- formed as an in-lane tree plus two shuffle rounds, so
// every merge stays inside the warp and a boundary costs one CTA barrier.  The boundary's edge entries,
// column lengths and destination latencies do not depend on the running costs: they are fetched into
// registers one boundary ahead, leaving only cur[] loads -> DADD -> tree -> shuffles -> store on the
// critical path.  Same contract as warp_route (picks valid when the returned cost is finite).
struct MwBoundary {
    int rs, rd;
    double e[8];
    double td;
};

template <int SPL, bool MAT>
__device__ __forceinline__ void mw_fetch(MwBoundary& m, const double* E, const int* node, const int* cl,
                                         const int* noff, const int* eoff, const double* tau, int b, int j, int q,
                                         int G) {
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    m.rs = cl[b];
    m.rd = cl[b + 1];
    const bool act = j < m.rd;
    const int dn = act ? node[noff[b + 1] + j] : 0;
    const double* ep = MAT ? E + dn : E + eoff[b] + j;           // matrix mode: column dn, rows by source node
    const int* sn = node + noff[b];
#pragma unroll
    for (int k = 0; k < SPL; ++k) {
        const int i = q + 4 * k;
        m.e[k] = (act && i < m.rs) ? (MAT ? ep[sn[i] * G] : ep[i * m.rd]) : INF;
    }
    m.td = act ? tau[dn] : 0.0;
}

// SPL = ceil(widest column / 4): source slots per lane (the tree and the prefetch shrink with the column)
template <int NWD, int SPL, bool MAT = false>
__device__ double mw_route(const double* E, const int* node, const int* cl, const int* noff, const int* eoff,
                           int nblk, const double* tau, double* costs, uint8_t* bp, int* picks, double* vshare,
                           int tid, int G = 0) {
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    constexpr int NT = NWD * 32;
    const int warp = tid >> 5, lane = tid & 31, d = lane & 7, q = lane >> 3;
    const int j = warp * 8 + d;
    const uint32_t bp_s = (uint32_t)__cvta_generic_to_shared(bp);   // hoisted: no per-boundary window lookup
    double* cur = costs;                                     // [40]: 32 hosts + 8 pad (+inf)
    double* nxt = costs + 40;
    for (int p = tid; p < 32; p += NT) cur[p] = p < cl[0] ? tau[node[p]] : INF;
    MwBoundary m;
    if (nblk > 0) mw_fetch<SPL, MAT>(m, E, node, cl, noff, eoff, tau, 0, j, q, G);
    __syncthreads();
    for (int b = 0; b < nblk; ++b) {
        double a[SPL];
#pragma unroll
        for (int k = 0; k < SPL; ++k) a[k] = __dadd_rn(cur[q + 4 * k], m.e[k]);
        const int rd = m.rd;
        const double td = m.td;
        // in-lane tree: left operands always carry the smaller source index -> take the right one on `<`
        int ix[SPL];
#pragma unroll
        for (int k = 0; k < SPL; ++k) ix[k] = k;
#pragma unroll
        for (int w = 1; w < SPL; w <<= 1)
#pragma unroll
            for (int k = 0; k + w < SPL; k += 2 * w)
                if (a[k + w] < a[k]) { a[k] = a[k + w]; ix[k] = ix[k + w]; }
        double best = a[0];
        int bi = q + 4 * ix[0];
#pragma unroll
        for (int o = 8; o <= 16; o <<= 1) {
            const double v2 = __shfl_xor_sync(FULL, best, o);
            const int i2 = __shfl_xor_sync(FULL, bi, o);
            lexmin(best, bi, v2, i2);
        }
        if (q == 0 && j < rd) {
            asm volatile("st.shared.u8 [%0], %1;" ::"r"(bp_s + b * 32 + j), "r"(bi));
            nxt[j] = __dadd_rn(best, td);
        }
        // next boundary's operands: issued behind the shuffles (shared LSU queue), landing during the barrier
        if (b + 1 < nblk) mw_fetch<SPL, MAT>(m, E, node, cl, noff, eoff, tau, b + 1, j, q, G);
        __syncthreads();
        double* t = cur; cur = nxt; nxt = t;
    }
    if (warp == 0) {
        double v = lane < cl[nblk] ? cur[lane] : INF;
        int idx = lane < cl[nblk] ? lane : NONE;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double v2 = __shfl_xor_sync(FULL, v, o);
            const int i2 = __shfl_xor_sync(FULL, idx, o);
            lexmin(v, idx, v2, i2);
        }
        if (lane == 0) {
            *vshare = v;
            if (v <= DBL_MAX) {
                int p = idx;
                picks[nblk] = p;
                for (int b = nblk - 1; b >= 0; --b) {
                    p = bp[b * 32 + p];
                    picks[b] = p;
                }
            }
        }
    }
    __syncthreads();
    return *vshare;
}

}  // namespace ssw
