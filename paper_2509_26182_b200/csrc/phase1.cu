// Phase-1 on device: stage-count search, objective,
// score / best k, water-filling -- bit-exact restatements of the reference's
// branchy Python (allocator.py, waterfill.py) as integer / fp64 device code.
//
//  * constructive cover (allocator.py:267-470): ONE THREAD PER CANDIDATE
//    (pool, k).  Groups are intrusive linked lists so Python list semantics
//    (append, pop(pos), positional swap, remove-first, stable sort) carry over
//    exactly; the budgeted peel recursion (353-423) is an explicit frame stack
//    whose "remaining" lists are 128-bit masks (they are always ascending
//    subsets of range(m)) and whose subset-sum reach sets are 256-bit words.
//  * exact sweep (allocator.py:138-264): one thread per pool, level frontier in
//    a global workspace with packed 16-byte residual keys whose unsigned order
//    is Python's tuple order (shorter prefix first); "first producer wins" is a
//    stable (key, producer-order) sort + dedup.
//  * objective (allocator.py:516-538) and water-fill (waterfill.py:47-183)
//    reproduce CPython 3.12 sum() (Neumaier with int/float item typing) and
//    IEEE rounding of every operation (built with -fmad=false).
// Phase-1 is issue-bound integer work, not HBM-bound.
#include <float.h>
#include <math.h>

#include "ss_common.cuh"

namespace {

constexpr int NMAX = 256;      // usable gpus per pool (constructive path)
constexpr int KMAX = 256;
constexpr int LMAX_PEEL = 128; // 2L <= 256-bit reach words
constexpr int BWORDS = 4;
constexpr int EXACT_LIMIT = 16;
constexpr uint16_t NIL = 0xFFFF;

// ---------------------------------------------------------------------------
// water-fill (waterfill.py:47-183)
// ---------------------------------------------------------------------------
__device__ double fill_at(double level, const double* fl, const int* cap, int n) {
    PySum s;
    s.init();
    for (int i = 0; i < n; ++i) {
        const double x = __dmul_rn(level, fl[i]);
        if (x < (double)cap[i]) s.add_float(x);   // min(c, x) is the float only when x < c
        else s.add_int(cap[i]);
    }
    return s.value();
}

__device__ int water_level(const double* fl, const int* cap, int n, int L, double* targets, int* tflag,
                           double* level_out, int* aux) {
    if (n < 1 || L < 1) return SS_BAD_INPUT;
    long long total = 0;
    double minf = fl[0];
    for (int i = 0; i < n; ++i) {
        if (!(fl[i] > 0.0)) return SS_BAD_INPUT;
        total += cap[i];
        if (fl[i] < minf) minf = fl[i];
    }
    if (total < L) { *aux = (int)total; return SS_INFEASIBLE_CAPACITY; }
    const double Ld = (double)L;
    double lo = 0.0;
    double hi = __dadd_rn(__ddiv_rn(Ld, minf), 1.0);
    const double tol = __dmul_rn(1e-9, Ld);
    for (int it = 0; it < 200; ++it) {
        if (fabs(__dsub_rn(fill_at(hi, fl, cap, n), Ld)) <= tol) break;
        const double mid = __dmul_rn(0.5, __dadd_rn(lo, hi));
        if (fill_at(mid, fl, cap, n) >= Ld) hi = mid;
        else lo = mid;
    }
    if (fabs(__dsub_rn(fill_at(hi, fl, cap, n), Ld)) > __dmul_rn(2.0, tol)) return SS_ROUNDING_OVERFLOW;
    for (int i = 0; i < n; ++i) {
        const double x = __dmul_rn(hi, fl[i]);
        const bool f = x < (double)cap[i];
        if (targets) targets[i] = f ? x : (double)cap[i];
        if (tflag) tflag[i] = f ? 0 : 1;
    }
    if (level_out) *level_out = hi;
    return SS_OK;
}

// largest-remainder rounding; targets given as (value, is_int)
__device__ int hamilton(const double* t, const int* tint, const int* cap, int n, long long total, int* out) {
    long long fl_sum = 0;
    for (int i = 0; i < n; ++i) {
        long long f = tint[i] ? (long long)t[i] : (long long)floor(t[i]);
        if (f > cap[i]) f = cap[i];
        out[i] = (int)f;
        fl_sum += f;
    }
    long long left = total - fl_sum;
    if (left < 0) return SS_ROUNDING_OVERFLOW;
    // order by (-(t - floor), i): remainder descending, index ascending
    int order[NMAX];
    double rem[NMAX];
    for (int i = 0; i < n; ++i) {
        rem[i] = __dsub_rn(t[i], (double)out[i]);     // t - min(floor(t), c): positive for an int t above its cap
        int j = i;
        while (j > 0 && rem[order[j - 1]] < rem[i]) { order[j] = order[j - 1]; --j; }
        order[j] = i;
    }
    for (int q = 0; q < n && left > 0; ++q) {
        const int i = order[q];
        if (out[i] < cap[i]) { out[i] += 1; --left; }
    }
    for (int i = 0; i < n && left > 0; ++i)
        while (left > 0 && out[i] < cap[i]) { out[i] += 1; --left; }
    return left > 0 ? SS_ROUNDING_OVERFLOW : SS_OK;
}

__device__ int stage_lengths(const double* fl, const int* cap, int n, int L, int* out, int* aux) {
    if (n > NMAX) return SS_BAD_INPUT;
    for (int i = 0; i < n; ++i)
        if (cap[i] < 1) { *aux = i; return SS_ZERO_CAPACITY; }
    double t[NMAX];
    int ti[NMAX];
    double lvl;
    int st = water_level(fl, cap, n, L, t, ti, &lvl, aux);
    if (st != SS_OK) return st;
    st = hamilton(t, ti, cap, n, L, out);
    if (st != SS_OK) return st;
    for (;;) {
        int needy = -1;
        for (int i = 0; i < n; ++i) if (out[i] == 0) { needy = i; break; }
        if (needy < 0) break;
        int donor = 0;
        for (int i = 1; i < n; ++i) if (out[i] > out[donor]) donor = i;   // (count, -i): lowest index on ties
        if (out[donor] < 2) return SS_ROUNDING_OVERFLOW;
        out[donor] -= 1;
        out[needy] += 1;
    }
    return SS_OK;
}

// ---------------------------------------------------------------------------
// constructive cover: best-fit with repairs (allocator.py:267-350)
// ---------------------------------------------------------------------------
struct Lists {
    uint16_t head[KMAX], tail[KMAX], size[KMAX];
    uint16_t next[NMAX], item[NMAX];
    int tot[KMAX];

    __device__ void reset(int k) {
        for (int g = 0; g < k; ++g) { head[g] = tail[g] = NIL; size[g] = 0; tot[g] = 0; }
    }
    __device__ void append(int g, int node) {
        next[node] = NIL;
        if (head[g] == NIL) head[g] = (uint16_t)node;
        else next[tail[g]] = (uint16_t)node;
        tail[g] = (uint16_t)node;
        size[g]++;
    }
    __device__ int node_at(int g, int pos) const {
        int nd = head[g];
        for (int p = 0; p < pos; ++p) nd = next[nd];
        return nd;
    }
    __device__ void unlink(int g, int prev, int nd) {
        if (prev == NIL) head[g] = next[nd];
        else next[prev] = next[nd];
        if (tail[g] == nd) tail[g] = (uint16_t)prev;
        size[g]--;
    }
    __device__ int pop_at(int g, int pos) {
        int prev = NIL, nd = head[g];
        for (int p = 0; p < pos; ++p) { prev = nd; nd = next[nd]; }
        unlink(g, prev, nd);
        return nd;
    }
    __device__ void remove_item(int g, int it) {
        int prev = NIL, nd = head[g];
        while (nd != NIL && item[nd] != it) { prev = nd; nd = next[nd]; }
        if (nd != NIL) unlink(g, prev, nd);
    }
};

__device__ __forceinline__ int cval(const int* caps, int i, int L) { return caps[i] < L ? caps[i] : L; }

__device__ bool best_fit(const int* caps, int m, int k, int L, Lists& G, const volatile int32_t* cancel = nullptr) {
    G.reset(k);
    for (int g = 0; g < k; ++g) {
        G.item[g] = (uint16_t)g;
        G.append(g, g);
        G.tot[g] = cval(caps, g, L);
    }
    for (int i = k; i < m; ++i) {
        int best = -1;
        for (int g = 0; g < k; ++g)
            if (G.tot[g] < L && (best < 0 || G.tot[g] > G.tot[best])) best = g;
        if (best < 0) break;
        G.item[i] = (uint16_t)i;
        G.append(best, i);
        G.tot[best] += cval(caps, i, L);
    }
    uint16_t opened[KMAX];
    for (int round = 0; round < 4; ++round) {
        if (cancel && *cancel < m) return false;            // parallel-m search: a smaller m already succeeded
        int n_open = 0;
        for (int g = 0; g < k; ++g) if (G.tot[g] < L) opened[n_open++] = (uint16_t)g;
        if (n_open == 0) break;
        bool changed = false;
        for (int q = 0; q < n_open; ++q) {
            const int u = opened[q];
            if (G.tot[u] >= L) continue;
            // move: key (closes, closes ? -val : val), strict >, first (g, pos) wins
            int bg = -1, bpos = -1, bclose = 0, bval = 0;
            for (int g = 0; g < k; ++g) {
                if (g == u) continue;
                int pos = 0;
                for (int nd = G.head[g]; nd != NIL; nd = G.next[nd], ++pos) {
                    const int v = cval(caps, G.item[nd], L);
                    if (G.size[g] == 1 || G.tot[g] - v < L) continue;
                    const int closes = G.tot[u] + v >= L;
                    const int key = closes ? -v : v;
                    if (bg < 0 || closes > bclose || (closes == bclose && key > bval)) {
                        bg = g; bpos = pos; bclose = closes; bval = key;
                    }
                }
            }
            if (bg >= 0) {
                const int nd = G.pop_at(bg, bpos);
                const int v = cval(caps, G.item[nd], L);
                G.tot[bg] -= v;
                G.tot[u] += v;
                G.append(u, nd);
                changed = true;
                continue;
            }
            // swap: max strictly positive gain keeping the donor closed
            int sg = -1, sgp = -1, sup = -1, gain_best = 0;
            for (int g = 0; g < k; ++g) {
                if (g == u || G.tot[g] < L) continue;
                int gp = 0;
                for (int nb = G.head[g]; nb != NIL; nb = G.next[nb], ++gp) {
                    const int vb = cval(caps, G.item[nb], L);
                    int up = 0;
                    for (int na = G.head[u]; na != NIL; na = G.next[na], ++up) {
                        const int gain = vb - cval(caps, G.item[na], L);
                        if (gain <= gain_best) continue;
                        if (G.tot[g] - gain >= L) { gain_best = gain; sg = g; sgp = gp; sup = up; }
                    }
                }
            }
            if (sg >= 0) {
                const int nb = G.node_at(sg, sgp), na = G.node_at(u, sup);
                const uint16_t t = G.item[nb];
                G.item[nb] = G.item[na];
                G.item[na] = t;
                G.tot[sg] -= gain_best;
                G.tot[u] += gain_best;
                changed = true;
            }
        }
        if (!changed) break;
    }
    for (int g = 0; g < k; ++g) if (G.tot[g] < L) return false;
    // minimal witness: shed spare members in stable ascending-value order
    uint16_t order[NMAX];
    for (int g = 0; g < k; ++g) {
        int cnt = 0;
        for (int nd = G.head[g]; nd != NIL; nd = G.next[nd]) {
            const uint16_t it = G.item[nd];
            const int v = cval(caps, it, L);
            int j = cnt++;
            while (j > 0 && cval(caps, order[j - 1], L) > v) { order[j] = order[j - 1]; --j; }
            order[j] = it;
        }
        for (int q = 0; q < cnt; ++q) {
            const int it = order[q];
            const int v = cval(caps, it, L);
            if (G.size[g] > 1 && G.tot[g] - v >= L) {
                G.remove_item(g, it);
                G.tot[g] -= v;
            }
        }
    }
    return true;
}

// ---------------------------------------------------------------------------
// constructive cover: budgeted peel (allocator.py:353-423)
// ---------------------------------------------------------------------------
struct Mask {   // subset of range(m), m <= 256
    uint64_t w[4];
    __device__ void clear() { w[0] = w[1] = w[2] = w[3] = 0; }
    __device__ bool test(int i) const { return (w[i >> 6] >> (i & 63)) & 1ull; }
    __device__ void set(int i) { w[i >> 6] |= 1ull << (i & 63); }
    __device__ int count() const { return __popcll(w[0]) + __popcll(w[1]) + __popcll(w[2]) + __popcll(w[3]); }
};


struct Frame {          // one peel() activation
    Mask picked;
    Mask avail;         // its pool: range(m) minus the picks of the frames above it (set when the frame is entered)
    int total, need;
    short targets[4];
    signed char nt, ti;
};

__device__ void range_mask(int m, Mask& pool) {
#pragma unroll
    for (int w = 0; w < 4; ++w) {                            // range(m) word by word
        const int lo = w * 64;
        pool.w[w] = m >= lo + 64 ? ~0ull : (m > lo ? (1ull << (m - lo)) - 1ull : 0ull);
    }
}


// Subset-sum reach rows reach[p + 1] = reach[p] | ((reach[p] << v_p) & (2^(2L) - 1)), up to 256 bits.  The rows
// live in the thread's local memory and only their ceil(2L / 64) live words are stored and read back (2 of 4 at
// L = 64), which halves the peel's local-memory traffic there.  Checkpointing every 2nd-8th row and rebuilding the
// rest in registers during the walk cut DRAM traffic 5x but measured 5-9% slower at C3 (L = 80), so every row is
// kept.
struct Reach4 { uint64_t r0, r1, r2, r3; };

// NW = ceil(2L / 64) live words (templated: the dead words' shifts drop out)
template <int NW>
__device__ __forceinline__ void reach_step(Reach4& r, int s, const uint64_t* lim) {
    const int ws = s >> 6, bs = s & 63;
    const uint64_t w0 = ws == 0 ? r.r0 : 0ull;
    const uint64_t w1 = ws == 0 ? r.r1 : (ws == 1 ? r.r0 : 0ull);
    // (lo >> 1) >> (63 - bs) == lo >> (64 - bs) for bs >= 1 and 0 for bs == 0 (no 64-bit shift by 64)
    if constexpr (NW > 2) {
        const uint64_t w2 = ws == 0 ? r.r2 : (ws == 1 ? r.r1 : (ws == 2 ? r.r0 : 0ull));
        if constexpr (NW > 3) {
            const uint64_t w3 = ws == 0 ? r.r3 : (ws == 1 ? r.r2 : (ws == 2 ? r.r1 : (ws == 3 ? r.r0 : 0ull)));
            r.r3 |= ((w3 << bs) | ((w2 >> 1) >> (63 - bs))) & lim[3];
        }
        r.r2 |= ((w2 << bs) | ((w1 >> 1) >> (63 - bs))) & lim[2];
    }
    if constexpr (NW > 1) r.r1 |= ((w1 << bs) | ((w0 >> 1) >> (63 - bs))) & lim[1];
    r.r0 |= (w0 << bs) & lim[0];
}

__device__ __forceinline__ void reach_limits(int L, uint64_t* lim) {
    const int nbits = 2 * L;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int lo = q * 64;
        lim[q] = lo >= nbits ? 0ull : (nbits - lo >= 64 ? ~0ull : (1ull << (nbits - lo)) - 1ull);
    }
}

__device__ __forceinline__ bool reach_test(const Reach4& r, int i) {
    const int w = i >> 6;
    const uint64_t x = w == 0 ? r.r0 : (w == 1 ? r.r1 : (w == 2 ? r.r2 : r.r3));
    return (x >> (i & 63)) & 1ull;
}

template <int NW>
__device__ __forceinline__ void reach_store(Reach4& dst, const Reach4& r) {
    dst.r0 = r.r0;
    if constexpr (NW > 1) dst.r1 = r.r1;
    if constexpr (NW > 2) dst.r2 = r.r2;
    if constexpr (NW > 3) dst.r3 = r.r3;
}

__device__ __forceinline__ bool reach_load_test(const Reach4& src, int i) {
    const uint64_t x = (&src.r0)[i >> 6];                    // one load: the word holding bit i (< 2L, live)
    return (x >> (i & 63)) & 1ull;
}

// forward pass over the pool's items in ascending order (set bits of the mask): rows[p] = reach[p] for p <= n
// (live words only); returns reach[n] and the item count
template <int NW>
__device__ Reach4 compute_reach(const int* caps, int L, const Mask& pool, Reach4* rows, int& n_out) {
    static_assert(BWORDS == 4, "reach rows are 4 words");
    uint64_t lim[4];
    reach_limits(L, lim);
    Reach4 r{1ull, 0ull, 0ull, 0ull};
    reach_store<NW>(rows[0], r);
    int p = 0;
#pragma unroll
    for (int w = 0; w < 4; ++w)
        for (uint64_t x = pool.w[w]; x; x &= x - 1) {
            reach_step<NW>(r, cval(caps, w * 64 + __ffsll((long long)x) - 1, L), lim);
            reach_store<NW>(rows[++p], r);
        }
    n_out = p;
    return r;
}

// the try's backward walk (allocator.py:401-409): from the last item down (set bits in descending order), an item
// is picked unless the reach row before it already holds the remaining target.  (Loading four positions' rows
// ahead of their tests measured slower: 143 registers per thread.)
template <int NW>
__device__ void reach_walk(const int* caps, int L, const Mask& pool, int n, const Reach4* rows, int tgt,
                           Mask& picked) {
    int rem = tgt, pos = n - 1;
#pragma unroll
    for (int w = 3; w >= 0; --w)
        for (uint64_t x = pool.w[w]; x; --pos) {
            const int b = 63 - __clzll((long long)x);
            x &= ~(1ull << b);
            if (reach_load_test(rows[pos], rem)) continue;
            const int i = w * 64 + b;
            picked.set(i);
            rem -= cval(caps, i, L);
        }
}

// returns true on success; the k groups are then fr[0..k-1].picked, in peel order
// cancel (optional): the parallel-m search's best success so far; an attempt at a larger m gives up
template <int NW>
__device__ bool peel(const int* caps, int m, int k, int L, Frame* fr, Reach4* ck,
                     const volatile int32_t* cancel = nullptr) {
    int budget = m <= 24 ? 300 : 80;
    int d = 0;
    int total = 0;
    for (int i = 0; i < m; ++i) total += cval(caps, i, L);
    fr[0].total = total;
    fr[0].need = k;
    range_mask(m, fr[0].avail);
    enum { ENTER, TRY, RET } state = ENTER;
    bool ok = false;
    int reach_owner = -1, owner_n = 0;
    for (;;) {
        if (state == ENTER) {
            Frame& f = fr[d];
            if (f.need == 0) { ok = true; state = RET; continue; }
            if (budget <= 0) { ok = false; state = RET; continue; }
            --budget;
            if (cancel && *cancel < m) return false;        // a smaller m already succeeded
            const Mask pool = f.avail;
            if (f.total < f.need * L || pool.count() < f.need) { ok = false; state = RET; continue; }
            if (f.need == 1) {
                int short_ = L;
                f.picked.clear();
                ok = false;
                for (int i = 0; i < m; ++i) {
                    if (!pool.test(i)) continue;
                    f.picked.set(i);
                    short_ -= cval(caps, i, L);
                    if (short_ <= 0) { ok = true; break; }
                }
                state = RET;
                continue;
            }
            int n = 0;
            const Reach4 last = compute_reach<NW>(caps, L, pool, ck, n);
            reach_owner = d;
            owner_n = n;
            f.nt = 0;
            // the first (up to) four reachable totals in [L, 2L): set bits of reach[n] from bit L up
            {
                const uint64_t words[4] = {last.r0, last.r1, last.r2, last.r3};
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    const int lo = w * 64;
                    if (lo + 64 <= L || f.nt >= 4) continue;
                    uint64_t x = words[w];
                    if (L > lo) x &= ~0ull << (L - lo);          // bits >= L (the reach limits clear >= 2L)
                    for (; x && f.nt < 4; x &= x - 1) f.targets[f.nt++] = (short)(lo + __ffsll((long long)x) - 1);
                }
            }
            f.ti = 0;
            state = TRY;
            continue;
        }
        if (state == TRY) {
            Frame& f = fr[d];
            if (f.ti >= f.nt) { ok = false; state = RET; continue; }
            // the reach rows (and item count) still hold this frame's unless a deeper frame overwrote them
            int n = owner_n;
            if (reach_owner != d) {
                compute_reach<NW>(caps, L, f.avail, ck, n);
                reach_owner = d;
                owner_n = n;
            }
            const int tgt = f.targets[f.ti];
            f.picked.clear();
            reach_walk<NW>(caps, L, f.avail, n, ck, tgt, f.picked);
            Frame& c = fr[d + 1];
            c.total = f.total - tgt;
            c.need = f.need - 1;
#pragma unroll
            for (int w = 0; w < 4; ++w) c.avail.w[w] = f.avail.w[w] & ~f.picked.w[w];
            ++d;
            state = ENTER;
            continue;
        }
        // RET (on success fr[0..k-1].picked already hold the groups)
        if (d == 0) break;
        --d;
        if (ok) continue;             // keep unwinding, recording picks
        fr[d].ti++;
        state = TRY;
    }
    return ok;
}

// ---------------------------------------------------------------------------
// exact sweep (allocator.py:114-264): state records shared by the CTA sweep and the one-thread replay
// ---------------------------------------------------------------------------
struct SRec {            // one state: residual bytes (value+1, zero padded) as a 128-bit big-endian key
    uint64_t hi, lo;
    uint8_t done, m, action;   // action: slot, or 0xFF = start
    uint8_t pad;
    int32_t aux;               // children: producer order; kept states: parent index in previous level
};

__device__ __forceinline__ void unpack(const SRec& r, uint8_t* res) {
    for (int p = 0; p < r.m; ++p) {
        const uint64_t w = p < 8 ? r.hi : r.lo;
        res[p] = (uint8_t)((w >> (8 * (7 - (p & 7)))) & 0xFF) - 1;
    }
}

__device__ __forceinline__ void pack(SRec& r, const uint8_t* res, int m) {
    r.hi = r.lo = 0;
    for (int p = 0; p < m; ++p) {
        const uint64_t b = (uint64_t)(res[p] + 1) << (8 * (7 - (p & 7)));
        if (p < 8) r.hi |= b; else r.lo |= b;
    }
    r.m = (uint8_t)m;
}

__device__ __forceinline__ bool key_less(const SRec& a, const SRec& b) {
    if (a.hi != b.hi) return a.hi < b.hi;
    if (a.lo != b.lo) return a.lo < b.lo;
    return a.done < b.done;
}

__device__ __forceinline__ bool key_eq(const SRec& a, const SRec& b) {
    return a.hi == b.hi && a.lo == b.lo && a.done == b.done;
}

__device__ __forceinline__ void insert_sorted(uint8_t* res, int& m, uint8_t v) {
    int j = m++;
    while (j > 0 && res[j - 1] > v) { res[j] = res[j - 1]; --j; }
    res[j] = v;
}

// rebuild the k groups of the state ((), k) found at `level` (allocator.py:228-264)
__device__ void sweep_replay(const int* caps, int L, const SRec* states, const int* level_start, int k, int level,
                             int* members_out, int* gsize_out) {
    // locate ((), k)
    int s = -1;
    for (int q = level_start[level]; q < level_start[level + 1]; ++q)
        if (states[q].m == 0 && states[q].done == k) { s = q; break; }
    uint8_t acts[EXACT_LIMIT + 1];
    for (int lv = level; lv >= 1; --lv) {
        acts[lv - 1] = states[s].action;
        s = level_start[lv - 1] + states[s].aux;
    }
    int open_res[EXACT_LIMIT], open_cnt[EXACT_LIMIT];
    uint8_t open_mem[EXACT_LIMIT][EXACT_LIMIT];
    int n_open = 0, n_closed = 0, out_pos = 0;
    for (int gi = 0; gi < level; ++gi) {
        const int cap = caps[gi];
        int rem, cnt;
        uint8_t mem[EXACT_LIMIT];
        if (acts[gi] == 0xFF) {
            rem = L - cap;
            cnt = 1;
            mem[0] = (uint8_t)gi;
        } else {
            const int slot = acts[gi];
            rem = open_res[slot];
            cnt = open_cnt[slot];
            for (int p = 0; p < cnt; ++p) mem[p] = open_mem[slot][p];
            for (int q = slot; q + 1 < n_open; ++q) {
                open_res[q] = open_res[q + 1];
                open_cnt[q] = open_cnt[q + 1];
                for (int p = 0; p < open_cnt[q]; ++p) open_mem[q][p] = open_mem[q + 1][p];
            }
            --n_open;
            mem[cnt++] = (uint8_t)gi;
            rem -= cap;
        }
        if (rem <= 0) {
            for (int p = 0; p < cnt; ++p) members_out[out_pos++] = mem[p];
            gsize_out[n_closed++] = cnt;
        } else {
            int j = n_open;     // stable insert after equal residuals
            while (j > 0 && open_res[j - 1] > rem) {
                open_res[j] = open_res[j - 1];
                open_cnt[j] = open_cnt[j - 1];
                for (int p = 0; p < open_cnt[j]; ++p) open_mem[j][p] = open_mem[j - 1][p];
                --j;
            }
            open_res[j] = rem;
            open_cnt[j] = cnt;
            for (int p = 0; p < cnt; ++p) open_mem[j][p] = mem[p];
            ++n_open;
        }
    }
}

__device__ __forceinline__ int usable_count(const int* caps, int n) {
    int u = 0;
    while (u < n && caps[u] > 0) ++u;
    return u;
}

__device__ bool sorted_nonincreasing(const int* caps, int n) {
    for (int j = 0; j + 1 < n; ++j) if (caps[j] < caps[j + 1]) return false;
    return true;
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// exact sweep, one CTA per pool (the level loop of allocator.py:138-225 with every step data-parallel):
//   expand   thread per parent state (sorted key order) -> children in producer order (parent, then extend
//            slots ascending, then start), positions by a block scan of the per-parent counts;
//   sort     stable merge sort of the children by (residual key, done): each pass places every record by a
//            binary search in the partner run, so equal keys keep producer order -> "first producer wins";
//   filter   first of each key run that passes feasibility (open <= remaining, sum(res) <= suffix);
//   prune    x is dropped iff some other state of its (done, open) class is pointwise <= x.  Sorted
//            lexicographically a dominator precedes what it dominates and domination is transitive, so this
//            order-free test equals the reference's forward pass over kept tuples (_prune_dominated 114-135);
//   keep     survivors in key order become the next level (sorted(frontier.keys())).
// The per-(pool, k) replay (228-264) stays one thread.
// ---------------------------------------------------------------------------
constexpr int SWEEP_NT = 256;

__device__ __forceinline__ bool rec_key_less(const SRec& a, const SRec& b) { return key_less(a, b); }

// exclusive scan of v[0..n) in place (global memory), returns the total; all threads of the CTA call it
__device__ int block_scan_excl(int* v, int n, int* sh) {
    const int tid = threadIdx.x;
    const int per = (n + SWEEP_NT - 1) / SWEEP_NT;
    const int a = tid * per, b = min(a + per, n);
    int sum = 0;
    for (int q = a; q < b; ++q) sum += v[q];
    sh[tid] = sum;
    __syncthreads();
    for (int o = 1; o < SWEEP_NT; o <<= 1) {               // Hillis-Steele inclusive scan of the partials
        const int x = tid >= o ? sh[tid - o] : 0;
        __syncthreads();
        sh[tid] += x;
        __syncthreads();
    }
    int run = sh[tid] - sum;
    const int total = sh[SWEEP_NT - 1];
    for (int q = a; q < b; ++q) { const int x = v[q]; v[q] = run; run += x; }
    __syncthreads();
    return total;
}

// y <= x pointwise (same open count; residual bytes stored value+1, zero padded, big-endian in hi/lo)
__device__ __forceinline__ bool pointwise_le(const SRec& y, const SRec& x) {
    const unsigned long long yh = y.hi, yl = y.lo, xh = x.hi, xl = x.lo;
    return __vcmpgeu4((unsigned)xh, (unsigned)yh) == 0xFFFFFFFFu &&
           __vcmpgeu4((unsigned)(xh >> 32), (unsigned)(yh >> 32)) == 0xFFFFFFFFu &&
           __vcmpgeu4((unsigned)xl, (unsigned)yl) == 0xFFFFFFFFu &&
           __vcmpgeu4((unsigned)(xl >> 32), (unsigned)(yl >> 32)) == 0xFFFFFFFFu;
}

struct CtaSweepWs {
    SRec* states;     // kept states, level after level
    SRec* a;          // children / sort ping
    SRec* b;          // sort pong / filtered list
    int32_t* i0;      // counts, flags, scan
    int32_t* i1;      // class buckets
};

__global__ void __launch_bounds__(SWEEP_NT) exact_sweep_cta_kernel(ss_pool_set P, const int64_t* koff,
        int32_t* stages, int32_t* members, int32_t* gsize, int32_t* pool_status, int32_t* pool_aux,
        unsigned char* ws_base, int64_t ws_bytes_per, int fcap, int ccap, const int32_t* exact_list, int n_exact,
        int32_t* sweep_stats) {
    __shared__ int sh[SWEEP_NT];
    __shared__ int level_start[EXACT_LIMIT + 2];
    __shared__ int found[EXACT_LIMIT + 1];
    __shared__ int suffix[EXACT_LIMIT + 1];
    __shared__ int caps_s[EXACT_LIMIT];
    __shared__ int cls_cnt[(EXACT_LIMIT + 1) * (EXACT_LIMIT + 1)], cls_off[(EXACT_LIMIT + 1) * (EXACT_LIMIT + 1)];
    __shared__ int s_nfound, s_stop, s_status, s_need, s_stats[4];
    const int e = blockIdx.x, tid = threadIdx.x;
    if (e >= n_exact) return;
    const int p = exact_list[e];
    if (pool_status[p] != SS_OK) return;
    const int off = P.pool_ptr[p], n_all = P.pool_ptr[p + 1] - off;
    const int* caps = P.caps + off;
    const int L = P.layers[p], kmax = P.kmax[p];
    const int n = usable_count(caps, n_all);
    const int kcap = kmax < EXACT_LIMIT ? kmax : EXACT_LIMIT;
    unsigned char* w = ws_base + (int64_t)e * ws_bytes_per;
    CtaSweepWs ws;
    ws.states = reinterpret_cast<SRec*>(w);  w += (int64_t)fcap * sizeof(SRec);
    ws.a = reinterpret_cast<SRec*>(w);       w += (int64_t)ccap * sizeof(SRec);
    ws.b = reinterpret_cast<SRec*>(w);       w += (int64_t)ccap * sizeof(SRec);
    ws.i0 = reinterpret_cast<int32_t*>(w);   w += (int64_t)ccap * 4;
    ws.i1 = reinterpret_cast<int32_t*>(w);
    if (tid == 0) {
        suffix[n] = 0;
        for (int i = n - 1; i >= 0; --i) suffix[i] = suffix[i + 1] + caps[i];
        for (int i = 0; i < n; ++i) caps_s[i] = caps[i];
        for (int k = 0; k <= EXACT_LIMIT; ++k) found[k] = 0;
        SRec root;
        root.hi = root.lo = 0; root.done = 0; root.m = 0; root.action = 0; root.pad = 0; root.aux = -1;
        ws.states[0] = root;
        level_start[0] = 0;
        level_start[1] = 1;
        s_nfound = 0; s_stop = 0; s_status = SS_OK; s_need = 0;
        s_stats[0] = s_stats[1] = s_stats[2] = s_stats[3] = 0;
    }
    __syncthreads();
    for (int i = 0; i < n; ++i) {
        const int cap = caps_s[i];
        const int f0 = level_start[i], f1 = level_start[i + 1], np = f1 - f0;
        // ---- expand: counts, scan, children in producer order -> a[] ----------
        if (np > ccap) { if (tid == 0) { s_status = SS_WORKSPACE; s_need = np + 1; } break; }
        for (int q = tid; q < np; q += SWEEP_NT) {
            const SRec st = ws.states[f0 + q];
            uint8_t res[EXACT_LIMIT + 1];
            unpack(st, res);
            int cnt = 0;
            for (int slot = 0; slot < st.m; ++slot) cnt += !(slot > 0 && res[slot] == res[slot - 1]);
            cnt += st.done + st.m < kmax;
            ws.i0[q] = cnt;
        }
        __syncthreads();
        const int nk = block_scan_excl(ws.i0, np, sh);
        if (nk > ccap) { if (tid == 0) { s_status = SS_WORKSPACE; s_need = nk + 1; } break; }
        for (int q = tid; q < np; q += SWEEP_NT) {
            const SRec st = ws.states[f0 + q];
            uint8_t res[EXACT_LIMIT + 1], child[EXACT_LIMIT + 1];
            unpack(st, res);
            const int m = st.m;
            int o = ws.i0[q];
            for (int slot = 0; slot <= m; ++slot) {
                const bool start = slot == m;
                if (!start && slot > 0 && res[slot] == res[slot - 1]) continue;
                if (start && !(st.done + m < kmax)) continue;
                int cm = 0, left;
                if (start) {
                    for (int t = 0; t < m; ++t) child[cm++] = res[t];
                    left = L - cap;
                } else {
                    for (int t = 0; t < m; ++t) if (t != slot) child[cm++] = res[t];
                    left = (int)res[slot] - cap;
                }
                SRec c;
                c.done = st.done;
                if (left <= 0) c.done = st.done + 1;
                else insert_sorted(child, cm, (uint8_t)left);
                pack(c, child, cm);
                c.action = start ? 0xFF : (uint8_t)slot;
                c.pad = 0;
                c.aux = q;                                   // parent index within the level
                ws.a[o++] = c;
            }
        }
        __syncthreads();
        // ---- stable merge sort of a[0..nk) by (key, done) ------------------------
        SRec* src = ws.a;
        SRec* dst = ws.b;
        for (int wd = 1; wd < nk; wd <<= 1) {
            for (int q = tid; q < nk; q += SWEEP_NT) {
                const int lo = q / (2 * wd) * (2 * wd), mid = min(lo + wd, nk), hi = min(lo + 2 * wd, nk);
                const SRec x = src[q];
                int pos;
                if (q < mid) {                               // A element: count B elements strictly less
                    int l = mid, r = hi;
                    while (l < r) { const int mm = (l + r) >> 1; if (rec_key_less(src[mm], x)) l = mm + 1; else r = mm; }
                    pos = lo + (q - lo) + (l - mid);
                } else {                                     // B element: count A elements less or equal
                    int l = lo, r = mid;
                    while (l < r) { const int mm = (l + r) >> 1; if (!rec_key_less(x, src[mm])) l = mm + 1; else r = mm; }
                    pos = lo + (q - mid) + (l - lo);
                }
                dst[pos] = x;
            }
            __syncthreads();
            SRec* t = src; src = dst; dst = t;
        }
        // ---- first of each key run + feasibility -> flags, scan, compact into dst --
        const int remaining = n - (i + 1);
        for (int q = tid; q < nk; q += SWEEP_NT) {
            const SRec c = src[q];
            bool keep = q == 0 || !key_eq(src[q - 1], c);
            if (keep) {
                uint8_t r[EXACT_LIMIT + 1];
                unpack(c, r);
                int sum = 0;
                for (int t = 0; t < c.m; ++t) sum += r[t];
                keep = !(c.m > remaining || sum > suffix[i + 1]);
            }
            ws.i0[q] = keep;
        }
        __syncthreads();
        const int nf = block_scan_excl(ws.i0, nk, sh);
        for (int q = tid; q < nk; q += SWEEP_NT) {
            const int pos = ws.i0[q];
            const bool keep = (q + 1 < nk ? ws.i0[q + 1] : nf) != pos;
            if (keep) dst[pos] = src[q];
        }
        __syncthreads();
        SRec* cand = dst;                                    // nf feasible unique children in key order
        // ---- dominance inside (done, open) classes: bucket, then test each against its bucket --------
        const int ncls = (EXACT_LIMIT + 1) * (EXACT_LIMIT + 1);
        for (int q = tid; q < ncls; q += SWEEP_NT) cls_cnt[q] = 0;
        __syncthreads();
        for (int q = tid; q < nf; q += SWEEP_NT) atomicAdd(&cls_cnt[cand[q].done * (EXACT_LIMIT + 1) + cand[q].m], 1);
        __syncthreads();
        if (tid == 0) {
            int run = 0;
            for (int q = 0; q < ncls; ++q) { cls_off[q] = run; run += cls_cnt[q]; cls_cnt[q] = cls_off[q]; }
        }
        __syncthreads();
        for (int q = tid; q < nf; q += SWEEP_NT) {
            const int cl = cand[q].done * (EXACT_LIMIT + 1) + cand[q].m;
            ws.i1[atomicAdd(&cls_cnt[cl], 1)] = q;
        }
        __syncthreads();
        for (int q = tid; q < nf; q += SWEEP_NT) {
            const SRec x = cand[q];
            const int cl = x.done * (EXACT_LIMIT + 1) + x.m;
            const int b0 = cls_off[cl], b1 = cls_cnt[cl];    // after the scatter, cls_cnt = bucket end
            bool dominated = false;
            for (int t = b0; t < b1 && !dominated; ++t) {
                const int yq = ws.i1[t];
                if (yq == q) continue;
                dominated = pointwise_le(cand[yq], x);
            }
            ws.i0[q] = !dominated;
        }
        __syncthreads();
        const int nn = block_scan_excl(ws.i0, nf, sh);
        const int base = level_start[i + 1];
        if (base + nn > fcap) { if (tid == 0) { s_status = SS_WORKSPACE; s_need = base + nn + 1; } break; }
        for (int q = tid; q < nf; q += SWEEP_NT) {
            const int pos = ws.i0[q];
            const bool keep = (q + 1 < nf ? ws.i0[q + 1] : nn) != pos;
            if (keep) {
                const SRec c = cand[q];
                ws.states[base + pos] = c;
                if (c.m == 0 && c.done >= 1 && c.done <= kcap && atomicCAS(&found[c.done], 0, i + 1) == 0)
                    atomicAdd(&s_nfound, 1);
            }
        }
        __syncthreads();
        if (tid == 0) {
            level_start[i + 2] = base + nn;
            s_stats[0] = i + 1;
            s_stats[1] += np;
            if (nn > s_stats[2]) s_stats[2] = nn;
            s_stats[3] += nf - nn;
            s_stop = s_nfound == kmax || nn == 0;
        }
        __syncthreads();
        if (s_stop) break;
    }
    __syncthreads();
    if (tid != 0) return;
    if (sweep_stats) for (int q = 0; q < 4; ++q) sweep_stats[4 * e + q] = s_stats[q];
    if (s_status != SS_OK) { pool_status[p] = s_status; pool_aux[p] = s_need; return; }
    int ls[EXACT_LIMIT + 2];
    for (int q = 0; q < EXACT_LIMIT + 2; ++q) ls[q] = level_start[q];
    for (int k = 1; k <= kmax; ++k) {
        const int64_t ko = koff[p] + k - 1;
        if (k > EXACT_LIMIT || found[k] == 0) { stages[ko] = 0; continue; }
        stages[ko] = found[k];
        sweep_replay(caps, L, ws.states, ls, k, found[k], members + P.memb_off[p] + (int64_t)(k - 1) * n_all,
                     gsize + P.gsz_off[p] + (int64_t)(k - 1) * kmax);
    }
}

constexpr int COVER_UNSET = 0x7f7f7f7f;
int g_cover_parallel_limit = 2048;      // candidates up to which the group counts are searched in parallel

// Constructive path of one (pool, k) candidate (allocator.py:426-470): m runs from m0 upward and the first m
// whose best-fit or (failing that) peel succeeds gives the groups.  Split into setup / one attempt so the m
// loop can run serially (cover_kernel, large batches) or with every m in parallel (cover_try_kernel +
// cover_finish_kernel, small batches such as one allocate() call) -- the smallest successful m is the same.
struct CoverCand {
    const int* caps;
    int n, n_all, L, kmax, m0;
    int64_t ko;
};

// false: k is infeasible for the pool (the reference's `break` on prefix < k*L)
__device__ bool cover_setup(const ss_pool_set& P, const int64_t* koff, int p, int k, CoverCand& cc) {
    const int off = P.pool_ptr[p];
    cc.n_all = P.pool_ptr[p + 1] - off;
    cc.caps = P.caps + off;
    cc.L = P.layers[p];
    cc.kmax = P.kmax[p];
    cc.n = usable_count(cc.caps, cc.n_all);
    cc.ko = koff[p] + k - 1;
    long long prefix_n = 0;
    for (int i = 0; i < cc.n; ++i) prefix_n += cval(cc.caps, i, cc.L);
    const long long target = (long long)k * cc.L;
    if (prefix_n < target) return false;
    const int pgm = (cc.L + cval(cc.caps, 0, cc.L) - 1) / cval(cc.caps, 0, cc.L);
    int m_cap = 0;
    long long acc = 0;
    while (m_cap < cc.n && acc < target) acc += cval(cc.caps, m_cap++, cc.L);   // bisect_left(prefix, target)
    cc.m0 = k * pgm > m_cap ? k * pgm : m_cap;
    return true;
}

// One attempt at group count m: best-fit, then peel.  On success writes the groups when mout != nullptr.
__device__ bool cover_try(const CoverCand& cc, int k, int m, Lists& G, Frame* fr, Reach4* reach,
                          int* mout, int* gout, int32_t* stage_out, const volatile int32_t* cancel = nullptr) {
    if (best_fit(cc.caps, m, k, cc.L, G, cancel)) {
        if (mout) {
            int pos = 0, stg = 0;
            for (int g = 0; g < k; ++g) {
                for (int nd = G.head[g]; nd != NIL; nd = G.next[nd]) mout[pos++] = G.item[nd];
                gout[g] = G.size[g];
                stg += G.size[g];
            }
            *stage_out = stg;
        }
        return true;
    }
    const int nw = (2 * cc.L + 63) >> 6;                     // live reach words (L <= 128)
    const bool peeled = nw <= 1 ? peel<1>(cc.caps, m, k, cc.L, fr, reach, cancel)
                      : nw == 2 ? peel<2>(cc.caps, m, k, cc.L, fr, reach, cancel)
                      : nw == 3 ? peel<3>(cc.caps, m, k, cc.L, fr, reach, cancel)
                                : peel<4>(cc.caps, m, k, cc.L, fr, reach, cancel);
    if (peeled) {
        if (mout) {
            int pos = 0, stg = 0;
            for (int g = 0; g < k; ++g) {
                int cnt = 0;
                for (int i = 0; i < m; ++i) if (fr[g].picked.test(i)) { mout[pos++] = i; ++cnt; }
                gout[g] = cnt;
                stg += cnt;
            }
            *stage_out = stg;
        }
        return true;
    }
    return false;
}

#ifndef P1_NARROW_MAX_L
#define P1_NARROW_MAX_L 64               // batches with every L <= this run cover_kernel_narrow
#endif

// one thread per (pool, k) on the constructive path; stage 0 = absent / stalled
__device__ __forceinline__ void cover_candidate(const ss_pool_set& P, const int64_t* koff, int32_t* stages,
                                                int32_t* members, int32_t* gsize, const int32_t* pool_status,
                                                const int32_t* cand_pool, const int32_t* cand_k, int n_cand,
                                                int32_t* stall) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_cand) return;
    const int p = cand_pool[c], k = cand_k[c];
    if (pool_status[p] != SS_OK) return;
    CoverCand cc;
    const bool feasible = cover_setup(P, koff, p, k, cc);
    stages[cc.ko] = 0;
    stall[cc.ko] = 0;
    if (!feasible) { stall[cc.ko] = 2; return; }                // reference `break` (infeasible k)
    Lists G;
    Frame fr[KMAX + 2];
    Reach4 reach[NMAX + 1];
    int* mout = members + P.memb_off[p] + (int64_t)(k - 1) * cc.n_all;
    int* gout = gsize + P.gsz_off[p] + (int64_t)(k - 1) * cc.kmax;
    for (int m = cc.m0; m <= cc.n; ++m)
        if (cover_try(cc, k, m, G, fr, reach, mout, gout, stages + cc.ko)) return;
    stall[cc.ko] = 1;                                            // constructive grouping stalled
}

__global__ void cover_kernel(ss_pool_set P, const int64_t* koff, int32_t* stages, int32_t* members, int32_t* gsize,
                             const int32_t* pool_status, const int32_t* cand_pool, const int32_t* cand_k, int n_cand,
                             int32_t* stall) {
    cover_candidate(P, koff, stages, members, gsize, pool_status, cand_pool, cand_k, n_cand, stall);
}

// the same for batches whose pools all have L <= 64 (two live reach words): a register budget sized for 12 blocks of
// 64 per SM (79 registers) -- their long m loops are latency-bound and more resident warps hide it (+4% at L = 64
// in a same-box A/B, identical plans; the same bound costs ~3% at L = 80, which keeps cover_kernel's 84)
__global__ void __launch_bounds__(64, 12) cover_kernel_narrow(ss_pool_set P, const int64_t* koff, int32_t* stages,
                                                              int32_t* members, int32_t* gsize,
                                                              const int32_t* pool_status, const int32_t* cand_pool,
                                                              const int32_t* cand_k, int n_cand, int32_t* stall) {
    cover_candidate(P, koff, stages, members, gsize, pool_status, cand_pool, cand_k, n_cand, stall);
}

// small batches, one round: thread (c, j) attempts m = m0 + m_off + j of candidate c unless an earlier round (a
// smaller m) already succeeded; best_m[c] = the smallest m that succeeds
__global__ void cover_try_kernel(ss_pool_set P, const int64_t* koff, const int32_t* pool_status,
                                 const int32_t* cand_pool, const int32_t* cand_k, int n_cand, int m_off, int span,
                                 int32_t* best_m) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (int64_t)n_cand * span) return;
    const int c = (int)(t / span), j = (int)(t % span);
    if (best_m[c] != COVER_UNSET) return;                   // resolved by an earlier round (smaller m)
    const int p = cand_pool[c], k = cand_k[c];
    if (pool_status[p] != SS_OK) return;
    CoverCand cc;
    if (!cover_setup(P, koff, p, k, cc)) return;
    const int m = cc.m0 + m_off + j;
    if (m > cc.n) return;
    Lists G;
    Frame fr[KMAX + 2];
    Reach4 reach[NMAX + 1];
    if (cover_try(cc, k, m, G, fr, reach, nullptr, nullptr, nullptr, best_m + c)) atomicMin(&best_m[c], m);
}

// small batches: rebuild the groups at the smallest successful m (or record the stall)
__global__ void cover_finish_kernel(ss_pool_set P, const int64_t* koff, int32_t* stages, int32_t* members,
                                    int32_t* gsize, const int32_t* pool_status, const int32_t* cand_pool,
                                    const int32_t* cand_k, int n_cand, const int32_t* best_m, int32_t* stall) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_cand) return;
    const int p = cand_pool[c], k = cand_k[c];
    if (pool_status[p] != SS_OK) return;
    CoverCand cc;
    const bool feasible = cover_setup(P, koff, p, k, cc);
    stages[cc.ko] = 0;
    stall[cc.ko] = 0;
    if (!feasible) { stall[cc.ko] = 2; return; }
    const int m = best_m[c];
    if (m < cc.m0 || m > cc.n) { stall[cc.ko] = 1; return; }
    Lists G;
    Frame fr[KMAX + 2];
    Reach4 reach[NMAX + 1];
    int* mout = members + P.memb_off[p] + (int64_t)(k - 1) * cc.n_all;
    int* gout = gsize + P.gsz_off[p] + (int64_t)(k - 1) * cc.kmax;
    if (!cover_try(cc, k, m, G, fr, reach, mout, gout, stages + cc.ko)) stall[cc.ko] = 1;
}

// per pool: apply "first stalled / infeasible k drops every larger k"; validate order
__global__ void cover_fixup_kernel(ss_pool_set P, const int64_t* koff, int32_t* stages, const int32_t* stall,
                                   int32_t* pool_status) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P.n_pools) return;
    const int off = P.pool_ptr[p], n_all = P.pool_ptr[p + 1] - off;
    const int* caps = P.caps + off;
    if (usable_count(caps, n_all) <= EXACT_LIMIT) return;
    bool dead = false;
    for (int k = 1; k <= P.kmax[p]; ++k) {
        const int64_t ko = koff[p] + k - 1;
        if (dead) { stages[ko] = 0; continue; }
        if (stall[ko]) { dead = true; stages[ko] = 0; }
    }
}

__global__ void validate_pools_kernel(ss_pool_set P, const int64_t* koff, int32_t* stages, int32_t* pool_status,
                                      int32_t* pool_aux) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P.n_pools) return;
    const int off = P.pool_ptr[p], n_all = P.pool_ptr[p + 1] - off;
    const int* caps = P.caps + off;
    int st = SS_OK;
    const int L = P.layers[p];
    const int n = usable_count(caps, n_all);
    if (!sorted_nonincreasing(caps, n_all) || L < 1) st = SS_BAD_INPUT;
    else if (n > EXACT_LIMIT && (n > NMAX || L > LMAX_PEEL || P.kmax[p] > KMAX)) st = SS_BAD_INPUT;
    else if (n <= EXACT_LIMIT && L > 254) st = SS_BAD_INPUT;
    pool_status[p] = st;
    pool_aux[p] = 0;
    for (int k = 1; k <= P.kmax[p]; ++k) stages[koff[p] + k - 1] = 0;
}

__global__ void objective_kernel(int32_t n_items, const int32_t* item_ptr, const double* flops, const int64_t* rtt_off,
                                 const double* rtt, double fpl, const int32_t* layers, double tokens, double* out_t,
                                 double* out_r) {
    const int it = blockIdx.x * blockDim.x + threadIdx.x;
    if (it >= n_items) return;
    const int off = item_ptr[it], n = item_ptr[it + 1] - off;
    const double* f = flops + off;
    PySum inv;
    inv.init();
    for (int i = 0; i < n; ++i) inv.add_float(__ddiv_rn(1.0, f[i]));
    const double harmonic = __ddiv_rn((double)n, inv.value());
    const double t = __ddiv_rn(__dmul_rn(__dmul_rn(fpl, (double)layers[it]), tokens), harmonic);
    const double* m = rtt + rtt_off[it];
    PySum s;
    s.init();
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b)
            if (a != b) s.add_float(m[(int64_t)a * n + b]);
    const long long cnt = (long long)n * (n - 1);
    out_t[it] = t;
    out_r[it] = cnt ? __ddiv_rn(s.value(), (double)cnt) : 0.0;
}

// Same arithmetic as objective_kernel with the region gathered from a pool: flops[gpu[i]] in cluster order and
// rtt_s(a, b) = base_rtt[a][b] (x the scenario's pair jitter when a seed is given, scenarios.py), so churned pools
// of many scenarios need no per-scenario dense matrices.
__global__ void objective_pool_kernel(int32_t n_items, const int32_t* item_ptr, const int32_t* gpu,
                                      const double* pool_flops, const double* base_rtt, int32_t n_pool,
                                      const int64_t* seeds, double fpl, const int32_t* layers, double tokens,
                                      double* out_t, double* out_r) {
    const int it = blockIdx.x * blockDim.x + threadIdx.x;
    if (it >= n_items) return;
    const int off = item_ptr[it], n = item_ptr[it + 1] - off;
    const int32_t* g = gpu + off;
    PySum inv;
    inv.init();
    for (int i = 0; i < n; ++i) inv.add_float(__ddiv_rn(1.0, pool_flops[g[i]]));
    const double harmonic = __ddiv_rn((double)n, inv.value());
    const double t = __ddiv_rn(__dmul_rn(__dmul_rn(fpl, (double)layers[it]), tokens), harmonic);
    const uint64_t mix = seeds ? ss_splitmix64((uint64_t)seeds[it]) : 0;
    PySum s;
    s.init();
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
            if (a == b) continue;
            double v = base_rtt[(int64_t)g[a] * n_pool + g[b]];
            if (seeds) v = __dmul_rn(v, ss_jitter(mix, (uint32_t)g[a], (uint32_t)g[b]));
            s.add_float(v);
        }
    const long long cnt = (long long)n * (n - 1);
    out_t[it] = t;
    out_r[it] = cnt ? __ddiv_rn(s.value(), (double)cnt) : 0.0;
}

__device__ __forceinline__ int score_one(int k, int s, double kp, double t, double r, double* z) {
    if (k < 1 || s < k) return SS_BAD_INPUT;
    const double denom = __dadd_rn(t, __dmul_rn(__ddiv_rn((double)s, (double)k), r));
    if (!(denom > 0.0)) return SS_DEGENERATE_OBJECTIVE;
    *z = __ddiv_rn(kp, denom);
    return SS_OK;
}

// grid: one thread per (pool, k); scores, and water-fills the groups when asked
__global__ void score_fill_kernel(ss_pool_set P, const int64_t* koff, const int32_t* stages, const int32_t* members,
                                  const int32_t* gsize, const double* t_comp, const double* rtt, const double* kpow,
                                  int kpow_len, int fill_all, double* z, int32_t* counts, int32_t* kstatus,
                                  int32_t* fstatus, const int32_t* cand_pool, const int32_t* cand_k, int n_cand) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_cand) return;
    const int p = cand_pool[c], k = cand_k[c];
    const int64_t ko = koff[p] + k - 1;
    kstatus[ko] = SS_OK;
    if (fstatus) fstatus[ko] = SS_OK;
    const int s = stages[ko];
    if (s == 0) return;
    if (k >= kpow_len) { kstatus[ko] = SS_BAD_INPUT; return; }
    double zz = 0.0;
    const int st = score_one(k, s, kpow[k], t_comp[p], rtt[p], &zz);
    z[ko] = zz;
    if (st != SS_OK) { kstatus[ko] = st; return; }
    if (!fill_all) return;
    const int off = P.pool_ptr[p], n_all = P.pool_ptr[p + 1] - off;
    const int kmax = P.kmax[p];
    const int* mem = members + P.memb_off[p] + (int64_t)(k - 1) * n_all;
    const int* gs = gsize + P.gsz_off[p] + (int64_t)(k - 1) * kmax;
    int* cnt = counts + P.memb_off[p] + (int64_t)(k - 1) * n_all;
    int pos = 0;
    int capv[NMAX];
    double flv[NMAX];
    for (int g = 0; g < k; ++g) {
        const int sz = gs[g];
        for (int q = 0; q < sz; ++q) {
            capv[q] = P.caps[off + mem[pos + q]];
            flv[q] = P.flops[off + mem[pos + q]];
        }
        int aux = 0;
        const int wst = stage_lengths(flv, capv, sz, P.layers[p], cnt + pos, &aux);
        if (wst != SS_OK) { if (fstatus) fstatus[ko] = wst; return; }
        pos += sz;
    }
}

// per pool: best k by (z, k); water-fill the best k's groups unless already filled
// One CTA per pool: thread 0 picks the best k (ascending k, ties -> the larger k, the first failing score raises);
// without fill_all the chosen k's groups are water-filled in parallel, one thread per group, and the pool takes
// the status of the lowest failing group -- the group the reference's sequential loop raises on.
__global__ void best_k_kernel(ss_pool_set P, const int64_t* koff, const int32_t* stages, const int32_t* members,
                              const int32_t* gsize, const double* z, const int32_t* kstatus,
                              const int32_t* fstatus, int fill_all, int32_t* best_k, int32_t* counts,
                              int32_t* pool_status) {
    const int p = blockIdx.x;
    __shared__ int s_bk;
    __shared__ unsigned long long s_err;                     // (group << 32) | status of the lowest failing group
    if (threadIdx.x == 0) {
        s_bk = 0;
        s_err = ~0ull;
        best_k[p] = 0;
        if (pool_status[p] == SS_OK) {
            int bk = 0;
            double bz = 0.0;
            bool bad = false;
            for (int k = 1; k <= P.kmax[p] && !bad; ++k) {
                const int64_t ko = koff[p] + k - 1;
                if (stages[ko] == 0) continue;
                if (kstatus[ko] != SS_OK) { pool_status[p] = kstatus[ko]; bad = true; break; }
                if (bk == 0 || z[ko] >= bz) { bk = k; bz = z[ko]; }
            }
            if (!bad) {
                best_k[p] = bk;
                if (bk > 0 && fill_all && fstatus && fstatus[koff[p] + bk - 1] != SS_OK)
                    pool_status[p] = fstatus[koff[p] + bk - 1];
                if (!fill_all) s_bk = bk;
            }
        }
    }
    __syncthreads();
    const int bk = s_bk;
    if (bk == 0) return;
    const int off = P.pool_ptr[p], n_all = P.pool_ptr[p + 1] - off;
    const int kmax = P.kmax[p];
    const int* mem = members + P.memb_off[p] + (int64_t)(bk - 1) * n_all;
    const int* gs = gsize + P.gsz_off[p] + (int64_t)(bk - 1) * kmax;
    int* cnt = counts + P.memb_off[p] + (int64_t)(bk - 1) * n_all;
    for (int g = threadIdx.x; g < bk; g += blockDim.x) {
        int pos = 0;
        for (int q = 0; q < g; ++q) pos += gs[q];
        const int sz = gs[g];
        int capv[NMAX];
        double flv[NMAX];
        for (int q = 0; q < sz; ++q) {
            capv[q] = P.caps[off + mem[pos + q]];
            flv[q] = P.flops[off + mem[pos + q]];
        }
        int aux = 0;
        const int wst = stage_lengths(flv, capv, sz, P.layers[p], cnt + pos, &aux);
        if (wst != SS_OK) atomicMin(&s_err, ((unsigned long long)g << 32) | (unsigned)wst);
    }
    __syncthreads();
    if (threadIdx.x == 0 && s_err != ~0ull) pool_status[p] = (int32_t)(unsigned)(s_err & 0xffffffffull);
}

__global__ void variant_reduce_kernel(int32_t n_var, const int32_t* var_ptr, const int64_t* koff, const int32_t* best_k,
                                      const double* z, const int32_t* pool_status, double* total, int32_t* feasible) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n_var) return;
    double acc = 0.0;
    int state = 0;   // 0 no pipeline, 1 feasible, -status on a pool error
    for (int p = var_ptr[v]; p < var_ptr[v + 1]; ++p) {
        if (pool_status[p] != SS_OK) { state = -pool_status[p]; break; }
        if (best_k[p] > 0) { acc = __dadd_rn(acc, z[koff[p] + best_k[p] - 1]); state = 1; }
    }
    total[v] = acc;
    feasible[v] = state;
}

__global__ void variant_argmax_kernel(int32_t n_var, const double* total, const int32_t* feasible, int32_t* best,
                                      double* best_total) {
    // single warp: (total desc, v asc)
    const int lane = threadIdx.x;
    double bt = -DBL_MAX;
    int bv = -1;
    for (int v = lane; v < n_var; v += 32) {
        if (feasible[v] != 1) continue;
        if (bv < 0 || total[v] > bt) { bt = total[v]; bv = v; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double t2 = __shfl_xor_sync(0xffffffffu, bt, o);
        const int v2 = __shfl_xor_sync(0xffffffffu, bv, o);
        if (v2 >= 0 && (bv < 0 || t2 > bt || (t2 == bt && v2 < bv))) { bt = t2; bv = v2; }
    }
    if (lane == 0) { *best = bv; *best_total = bv >= 0 ? bt : 0.0; }
}

__global__ void waterfill_kernel(int32_t n_groups, const int32_t* grp_ptr, const double* flops, const int32_t* caps,
                                 const int32_t* layers, int mode, double* targets, int32_t* tflag, double* level,
                                 int32_t* counts, int32_t* status, int32_t* aux) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n_groups) return;
    const int off = grp_ptr[g], n = grp_ptr[g + 1] - off;
    int a = 0, st;
    if (n > NMAX) { status[g] = SS_BAD_INPUT; return; }
    if (mode == 2) {
        st = stage_lengths(flops + off, caps + off, n, layers[g], counts + off, &a);
    } else {
        double lv = 0.0;
        st = water_level(flops + off, caps + off, n, layers[g], targets + off, tflag + off, &lv, &a);
        if (level) level[g] = lv;
        if (st == SS_OK && mode == 1) st = hamilton(targets + off, tflag + off, caps + off, n, layers[g], counts + off);
    }
    status[g] = st;
    if (aux) aux[g] = a;
}

__global__ void hamilton_kernel(int32_t n_groups, const int32_t* grp_ptr, const double* targets, const int32_t* tflag,
                                const int32_t* caps, const int32_t* total, int32_t* counts, int32_t* status) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n_groups) return;
    const int off = grp_ptr[g], n = grp_ptr[g + 1] - off;
    if (n > NMAX) { status[g] = SS_BAD_INPUT; return; }
    long long tot = total[g];
    if (tot < 0) {     // round(sum(targets)) with CPython sum semantics, round-half-even
        PySum s;
        s.init();
        for (int i = 0; i < n; ++i) {
            if (tflag[off + i]) s.add_int((long long)targets[off + i]);
            else s.add_float(targets[off + i]);
        }
        tot = s.is_int ? s.iacc : (long long)rint(s.value());
    }
    status[g] = hamilton(targets + off, tflag + off, caps + off, n, tot, counts + off);
}

__global__ void score_kernel(int32_t n, const int32_t* k, const int32_t* s, const double* kpow, const double* t,
                             const double* r, double* z, int32_t* status) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double zz = 0.0;
    status[i] = score_one(k[i], s[i], kpow[i], t[i], r[i], &zz);
    z[i] = zz;
}

inline int grid_for(int n, int b) { return (n + b - 1) / b; }

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" int64_t ss_stage_counts_workspace(int32_t frontier_cap, int32_t children_cap, int32_t max_levels) {
    (void)max_levels;
    return (int64_t)frontier_cap * sizeof(SRec) + (int64_t)children_cap * (2 * sizeof(SRec) + 8) + 256;
}

extern "C" int ss_stage_counts_validate(const ss_pool_set* pools, const int64_t* koff, int32_t* stages,
                                        int32_t* pool_status, int32_t* pool_aux, void* stream) {
    if (!pools || pools->n_pools <= 0) return SS_OK;
    validate_pools_kernel<<<grid_for(pools->n_pools, 128), 128, 0, ss_stream(stream)>>>(*pools, koff, stages,
                                                                                        pool_status, pool_aux);
    SS_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_stage_counts_exact(const ss_pool_set* pools, const int64_t* koff, int32_t* stages, int32_t* members,
                                     int32_t* gsize, int32_t* pool_status, int32_t* pool_aux, const int32_t* exact_list,
                                     int32_t n_exact, void* workspace, int64_t ws_bytes_per, int32_t frontier_cap,
                                     int32_t children_cap, int32_t* sweep_stats, void* stream) {
    if (n_exact <= 0) return SS_OK;
    exact_sweep_cta_kernel<<<n_exact, SWEEP_NT, 0, ss_stream(stream)>>>(
        *pools, koff, stages, members, gsize, pool_status, pool_aux, static_cast<unsigned char*>(workspace),
        ws_bytes_per, frontier_cap, children_cap, exact_list, n_exact, sweep_stats);
    SS_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_stage_counts_cover(const ss_pool_set* pools, const int64_t* koff, int32_t* stages, int32_t* members,
                                     int32_t* gsize, int32_t* pool_status, const int32_t* cand_pool,
                                     const int32_t* cand_k, int32_t n_cand, int32_t* stall, int32_t max_layers,
                                     void* stream) {
    cudaStream_t s = ss_stream(stream);
    // The cover kernels keep their peel frames / reach bitsets on the thread stack (~28 KB).  Reserving that
    // stack size once stops the driver from resizing the device's local-memory pool between launches of
    // kernels with different stack needs (measured: sporadic 0.4-1.7 s stalls on a single allocate() call).
    static bool stack_reserved = false;
    if (!stack_reserved) {
        size_t cur = 0;
        cudaFuncAttributes fa{};
        size_t need = 0;
        if (cudaFuncGetAttributes(&fa, cover_kernel) == cudaSuccess) need = fa.localSizeBytes;
        if (cudaFuncGetAttributes(&fa, cover_kernel_narrow) == cudaSuccess && fa.localSizeBytes > need)
            need = fa.localSizeBytes;
        if (need && cudaDeviceGetLimit(&cur, cudaLimitStackSize) == cudaSuccess && cur < need)
            cudaDeviceSetLimit(cudaLimitStackSize, need);
        stack_reserved = true;
    }
    // A batch too small to fill the GPU (one allocate() call: ~4 regions x k_max candidates) tries every group
    // count m of every candidate in parallel; an attempt gives up as soon as a smaller m of its candidate has
    // succeeded (peel polls best_m), and the smallest success is the reference's first-success m.  A large sweep
    // keeps the work-efficient serial m loop of cover_kernel.
    int32_t* best_m = nullptr;
    if (n_cand > 0 && n_cand <= g_cover_parallel_limit &&
        cudaMallocAsync(&best_m, sizeof(int32_t) * n_cand, s) == cudaSuccess) {
        cudaMemsetAsync(best_m, 0x7f, sizeof(int32_t) * n_cand, s);          // COVER_UNSET
        int m_off = 0;
        for (int span : {NMAX}) {                                             // m0 .. m0 + NMAX - 1 >= n
            const int64_t nt = (int64_t)n_cand * span;
            cover_try_kernel<<<(unsigned)((nt + 63) / 64), 64, 0, s>>>(*pools, koff, pool_status, cand_pool, cand_k,
                                                                       n_cand, m_off, span, best_m);
            SS_CHECK_LAUNCH();
            m_off += span;
        }
        cover_finish_kernel<<<grid_for(n_cand, 64), 64, 0, s>>>(*pools, koff, stages, members, gsize, pool_status,
                                                                 cand_pool, cand_k, n_cand, best_m, stall);
        SS_CHECK_LAUNCH();
        cudaFreeAsync(best_m, s);
    } else if (n_cand > 0) {
        auto kern = max_layers > 0 && max_layers <= P1_NARROW_MAX_L ? cover_kernel_narrow : cover_kernel;
        kern<<<grid_for(n_cand, 64), 64, 0, s>>>(*pools, koff, stages, members, gsize, pool_status, cand_pool, cand_k,
                                                  n_cand, stall);
        SS_CHECK_LAUNCH();
    }
    cover_fixup_kernel<<<grid_for(pools->n_pools, 128), 128, 0, s>>>(*pools, koff, stages, stall, pool_status);
    SS_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_objective(int32_t n_items, const int32_t* item_ptr, const double* flops, const int64_t* rtt_off,
                            const double* rtt, double fpl, const int32_t* layers, double tokens, double* out_t,
                            double* out_r, void* stream) {
    if (n_items <= 0) return SS_OK;
    objective_kernel<<<grid_for(n_items, 64), 64, 0, ss_stream(stream)>>>(n_items, item_ptr, flops, rtt_off, rtt, fpl,
                                                                         layers, tokens, out_t, out_r);
    SS_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_objective_pool(int32_t n_items, const int32_t* item_ptr, const int32_t* gpu, const double* pool_flops,
                                 const double* base_rtt, int32_t n_pool, const int64_t* seeds, double fpl,
                                 const int32_t* layers, double tokens, double* out_t, double* out_r, void* stream) {
    if (n_items <= 0) return SS_OK;
    if (!item_ptr || !gpu || !pool_flops || !base_rtt || n_pool < 1 || !layers || !out_t || !out_r)
        return SS_BAD_INPUT;
    objective_pool_kernel<<<grid_for(n_items, 64), 64, 0, ss_stream(stream)>>>(
        n_items, item_ptr, gpu, pool_flops, base_rtt, n_pool, seeds, fpl, layers, tokens, out_t, out_r);
    SS_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_phase1_score(const ss_pool_set* pools, const int64_t* koff, const int32_t* stages,
                               const int32_t* members, const int32_t* gsize, const double* t_comp, const double* rtt,
                               const double* kpow, int32_t kpow_len, int32_t fill_all, double* z, int32_t* counts,
                               int32_t* kstatus, int32_t* fstatus, const int32_t* cand_pool, const int32_t* cand_k,
                               int32_t n_cand, void* stream) {
    if (n_cand <= 0) return SS_OK;
    score_fill_kernel<<<grid_for(n_cand, 64), 64, 0, ss_stream(stream)>>>(*pools, koff, stages, members, gsize, t_comp,
                                                                         rtt, kpow, kpow_len, fill_all, z, counts,
                                                                         kstatus, fstatus, cand_pool, cand_k, n_cand);
    SS_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_phase1_best(const ss_pool_set* pools, const int64_t* koff, const int32_t* stages,
                              const int32_t* members, const int32_t* gsize, const double* z, const int32_t* kstatus,
                              const int32_t* fstatus, int32_t fill_all, int32_t* best_k, int32_t* counts,
                              int32_t* pool_status, void* stream) {
    if (!pools || pools->n_pools <= 0) return SS_OK;
    best_k_kernel<<<pools->n_pools, fill_all ? 32 : 128, 0, ss_stream(stream)>>>(*pools, koff, stages, members, gsize,
                                                                                z, kstatus, fstatus, fill_all, best_k,
                                                                                counts, pool_status);
    SS_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_variant_reduce(int32_t n_var, const int32_t* var_ptr, const int64_t* koff, const int32_t* best_k,
                                 const double* z, const int32_t* pool_status, double* total, int32_t* feasible,
                                 int32_t* best_variant, double* best_total, void* stream) {
    if (n_var <= 0) return SS_OK;
    cudaStream_t s = ss_stream(stream);
    variant_reduce_kernel<<<grid_for(n_var, 128), 128, 0, s>>>(n_var, var_ptr, koff, best_k, z, pool_status, total,
                                                                feasible);
    SS_CHECK_LAUNCH();
    if (best_variant) {
        variant_argmax_kernel<<<1, 32, 0, s>>>(n_var, total, feasible, best_variant, best_total);
        SS_CHECK_LAUNCH();
    }
    return SS_OK;
}

extern "C" int ss_waterfill(int32_t n_groups, const int32_t* grp_ptr, const double* flops, const int32_t* caps,
                            const int32_t* layers, int32_t mode, double* targets, int32_t* tflag, double* level,
                            int32_t* counts, int32_t* status, int32_t* aux, void* stream) {
    if (n_groups <= 0) return SS_OK;
    waterfill_kernel<<<grid_for(n_groups, 64), 64, 0, ss_stream(stream)>>>(n_groups, grp_ptr, flops, caps, layers, mode,
                                                                          targets, tflag, level, counts, status, aux);
    SS_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_hamilton(int32_t n_groups, const int32_t* grp_ptr, const double* targets, const int32_t* tflag,
                           const int32_t* caps, const int32_t* total, int32_t* counts, int32_t* status, void* stream) {
    if (n_groups <= 0) return SS_OK;
    hamilton_kernel<<<grid_for(n_groups, 64), 64, 0, ss_stream(stream)>>>(n_groups, grp_ptr, targets, tflag, caps, total,
                                                                          counts, status);
    SS_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_score(int32_t n, const int32_t* k, const int32_t* s_star, const double* kpow, const double* t_comp,
                        const double* rtt, double* z, int32_t* status, void* stream) {
    if (n <= 0) return SS_OK;
    score_kernel<<<grid_for(n, 128), 128, 0, ss_stream(stream)>>>(n, k, s_star, kpow, t_comp, rtt, z, status);
    SS_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int32_t ss_set_cover_parallel_limit(int32_t max_candidates) {
    const int32_t old = g_cover_parallel_limit;
    if (max_candidates >= 0) g_cover_parallel_limit = max_candidates;
    return old;
}
