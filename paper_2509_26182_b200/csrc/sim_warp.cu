// Serving simulator on device (the admission path with occupancy-dependent step time).
//
// One warp (<= 8 hosts per layer) or a lockstep CTA of NWD warps (9..32 hosts, sim_mw_kernel) runs one scenario's
// discrete-event simulation of pkg/src/swarmsched/sim.py:_Simulation (no membership events), with the scenario's
// DAG resident in shared memory (warp_dag.cuh); ss_sim_cta covers wider pools with streamed edges:
//   * events are ordered by (time, seq) exactly like the reference heap: arrivals take seq 0..n-1 in trace
//     order, the first publish tick seq n, every later push the next number (sim.py:238-265);
//   * a publish tick re-arms while work remains (sim.py:432-436) and changes nothing the router reads, but it
//     advances the clock, so the run's duration is the last tick's time;
//   * arrival: joins the back of the queue, or is admitted at once when the queue is empty (sim.py:361-366);
//     admission routes with the KV-blocked GPUs excluded (+inf latency: the same chain as removing them),
//     reserves total_tokens and +1 occupancy on the chain's distinct GPUs and schedules the prefill at
//     now + compute * prompt + chain RTT, compute = CPython sum(base_s * hop.length) (sim.py:303-307,319-338);
//   * prefill / step: a step lasts sum over hops of (base_s * max(1, occ)^e) * hop.length (+ chain RTT unless
//     amortized), occupancy read when the step starts (sim.py:309-317, 375-392);
//   * completion: release, then the strict FIFO drain (sim.py:345-357, 394-399).
// Strict FIFO without aborts admits in arrival order, so the queue is the arrival range [admitted, arrived).
#include <float.h>

#include "warp_dag.cuh"

namespace {

using namespace ssw;

constexpr int HMAX = 32;              // hops per live chain kept in shared memory
constexpr int K_PREFILL = 1, K_STEP = 2;   // live-chain event kinds (arrivals and ticks are not stored)

struct SimLayout {
    int max_live, pow_len;            // pow_len: entries cached in shared memory (the tables may be longer)
    int off_time, off_seq, off_req, off_rem, off_kind, off_nh, off_crtt, off_tok, off_hops, off_xpw, total;
};

struct SimArgs {
    const int32_t* gpu_ptr;
    const double* base_tau;           // flops_per_layer_per_token / flops == LatencyModel.base_s (sim.py:179-180)
    const int64_t* token_cap;         // ram_token_capacity
    const double* rtt;                // [n_dags * max_gpus^2] declared one-way RTT (manager.rtt_s)
    const double* pub_pow;            // (1 + o) ** e   (published latency, sim.py:182-183)
    const double* exec_pow;           // max(1, o) ** e (executing latency, sim.py:185-186)
    int32_t pow_len;
    const int32_t* trace_ptr;         // [n_dags + 1] requests per scenario, arrival order
    const double* arrival;
    const int32_t* prompt;
    const int32_t* output;
    double publish_interval;
    int32_t amortize_rtt;
    double* done_time;                // per request: completion time (NaN = unserved)
    int32_t* done_rank;               // per request: completion order (-1 = unserved)
    double* duration;                 // per scenario
    int32_t* completed, *queue_peak;
    int64_t* n_events;
    int32_t* status, *aux;
};

template <bool MAT = false>
__global__ void __launch_bounds__(32) sim_warp_kernel(ss_dag_set D, WarpLayout A, SimLayout B, SimArgs P) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int dag = blockIdx.x;
    const int lane = threadIdx.x;
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
    double* ppw = reinterpret_cast<double*>(smem + A.off_pow);
    double* costs = reinterpret_cast<double*>(smem + A.off_cost);
    long long* kv = reinterpret_cast<long long*>(smem + A.off_kv);
    long long* tcap = reinterpret_cast<long long*>(smem + A.off_tcap);
    double* ev_time = reinterpret_cast<double*>(smem + B.off_time);
    int* ev_seq = reinterpret_cast<int*>(smem + B.off_seq);
    int* ev_req = reinterpret_cast<int*>(smem + B.off_req);
    int* ev_rem = reinterpret_cast<int*>(smem + B.off_rem);
    uint8_t* ev_kind = smem + B.off_kind;
    uint8_t* ev_nh = smem + B.off_nh;
    double* ev_crtt = reinterpret_cast<double*>(smem + B.off_crtt);
    long long* ev_tok = reinterpret_cast<long long*>(smem + B.off_tok);
    short2* ev_hops = reinterpret_cast<short2*>(smem + B.off_hops);     // [max_live][HMAX] (gpu, length)
    double* xpw = reinterpret_cast<double*>(smem + B.off_xpw);

    if (!stage_dag(D, A, l0, nl, E, node, cl, noff, eoff, lane,
                   A.mat_dim ? P.rtt + (int64_t)dag * A.mat_dim * A.mat_dim : nullptr)) {
        if (lane == 0) P.status[dag] = SS_BAD_INPUT;
        return;
    }
    const int gbase = P.gpu_ptr[dag];
    const int ng = P.gpu_ptr[dag + 1] - gbase;
    for (int g = lane; g < ng; g += 32) {
        occ[g] = 0;
        kv[g] = 0;
        stamp[g] = 0;
        base[g] = P.base_tau[gbase + g];
        tcap[g] = P.token_cap[gbase + g];
    }
    for (int o = lane; o < B.pow_len; o += 32) { ppw[o] = P.pub_pow[o]; xpw[o] = P.exec_pow[o]; }
    for (int e = lane; e < B.max_live; e += 32) ev_kind[e] = 0xFF;
    if (lane < 8) { costs[32 + lane] = INF; costs[72 + lane] = INF; }
    __syncwarp();
    const double* rtt = P.rtt + (int64_t)dag * D.max_gpus * D.max_gpus;
    const int r0 = P.trace_ptr[dag], n = P.trace_ptr[dag + 1] - r0;
    const double* arr = P.arrival + r0;
    const int32_t* prm = P.prompt + r0;
    const int32_t* outp = P.output + r0;

    int ap = 0, adm = 0, live_n = 0, live_hw = 0, next_seq = n + 1, completed = 0, peak = 0, status = SS_OK;
    bool tick = n > 0;                          // sim.py:264-265: first tick only if work remains
    double tick_t = P.publish_interval, now = 0.0;
    int tick_seq = n;
    long long events = 0;

    // route + reserve + schedule the prefill of request i at time t; false when no finite chain exists
    auto try_admit = [&](int i, double t) -> bool {
        const long long tok = (long long)prm[i] + outp[i];
        for (int g = lane; g < ng; g += 32) {
            const int o = occ[g];
            tau[g] = tcap[g] - kv[g] < tok ? INF : base[g] * (o < B.pow_len ? ppw[o] : P.pub_pow[o]);  // KV-blocked excluded
        }
        __syncwarp();
        const double v = warp_route<MAT>(E, node, cl, noff, eoff, nblk, tau, costs, bp, picks, lane, A.mat_pitch);
        if (!(v <= DBL_MAX)) return false;
        // a free live slot (warp-uniform search)
        int slot = -1;
        for (int e0 = 0; e0 < B.max_live && slot < 0; e0 += 32) {
            const unsigned m = __ballot_sync(FULL, e0 + lane < B.max_live && ev_kind[e0 + lane] == 0xFF);
            if (m) slot = e0 + __ffs(m) - 1;
        }
        if (slot < 0) { status = SS_BAD_INPUT; return false; }
        // distinct GPUs: +1 occupancy and the tokens (sim.py:330-331; perfmap.py:356-382)
        const int tag = i + 1;
        for (int c0 = 0; c0 < nl; c0 += 32) {
            const int l = c0 + lane;
            int g = 0;
            bool first = false;
            if (l < nl) {
                g = node[noff[l] + picks[l]];
                first = atomicExch(&stamp[g], tag) != tag;
            }
            if (first) { occ[g] += 1; kv[g] += tok; }
        }
        __syncwarp();
        if (lane == 0) {
            // merged hops, chain RTT, prefill = CPython sum(base_s * length) * prompt + chain RTT
            int nh = 0, prev = -1;
            short2* hp = ev_hops + slot * HMAX;
            for (int l = 0; l < nl; ++l) {
                const int g = node[noff[l] + picks[l]];
                if (g == prev) { hp[nh - 1].y += 1; continue; }
                if (nh == HMAX) { nh = HMAX + 1; break; }
                hp[nh].x = (short)g;
                hp[nh].y = 1;
                ++nh;
                prev = g;
            }
            if (nh > HMAX) {
                status = SS_BAD_INPUT;
            } else {
                double crtt = 0.0;
                for (int h = 0; h + 1 < nh; ++h) crtt = __dadd_rn(crtt, rtt[(int64_t)hp[h].x * D.max_gpus + hp[h + 1].x]);
                PySum compute;
                compute.init();
                for (int h = 0; h < nh; ++h) compute.add_float(__dmul_rn(base[hp[h].x], (double)hp[h].y));
                const double pre = __dadd_rn(__dmul_rn(compute.value(), (double)prm[i]), crtt);
                ev_time[slot] = __dadd_rn(t, pre);
                ev_seq[slot] = next_seq;
                ev_req[slot] = i;
                ev_rem[slot] = outp[i];
                ev_kind[slot] = K_PREFILL;
                ev_nh[slot] = (uint8_t)nh;
                ev_crtt[slot] = crtt;
                ev_tok[slot] = tok;
            }
        }
        status = __shfl_sync(FULL, status, 0);
        ++next_seq;
        ++live_n;
        if (slot + 1 > live_hw) live_hw = slot + 1;
        __syncwarp();
        return status == SS_OK;
    };

    int rank = 0;
    while (status == SS_OK) {
        // next event: lexicographic (time, seq) over live chains, the next arrival and the pending tick
        double bt = INF;
        int bs = 0x7fffffff, bk = -1;
        for (int e = lane; e < live_hw; e += 32) {
            if (ev_kind[e] == 0xFF) continue;
            const double t = ev_time[e];
            const int q = ev_seq[e];
            if (t < bt || (t == bt && q < bs)) { bt = t; bs = q; bk = e; }
        }
        if (lane == 0) {
            if (ap < n && (arr[ap] < bt || (arr[ap] == bt && ap < bs))) { bt = arr[ap]; bs = ap; bk = -2; }
            if (tick && (tick_t < bt || (tick_t == bt && tick_seq < bs))) { bt = tick_t; bs = tick_seq; bk = -3; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double t2 = __shfl_xor_sync(FULL, bt, o);
            const int s2 = __shfl_xor_sync(FULL, bs, o);
            const int k2 = __shfl_xor_sync(FULL, bk, o);
            if (t2 < bt || (t2 == bt && s2 < bs)) { bt = t2; bs = s2; bk = k2; }
        }
        if (bk == -1) break;                                     // heap empty
        now = bt;
        ++events;
        if (bk == -3) {                                          // publish tick (sim.py:432-436)
            if (live_n > 0 || ap < n) { tick_t = __dadd_rn(now, P.publish_interval); tick_seq = next_seq++; }
            else tick = false;
            continue;
        }
        if (bk == -2) {                                          // arrival (sim.py:361-366)
            const int i = ap++;
            if (adm < i || !try_admit(i, now)) {
                if (status != SS_OK) break;
                peak = max(peak, ap - adm);
            } else {
                ++adm;
            }
            continue;
        }
        // prefill / step of live chain bk (sim.py:375-392)
        const int e = bk;
        bool finish = false;
        if (lane == 0) {
            if (ev_kind[e] == K_STEP) ev_rem[e] -= 1;
            finish = ev_rem[e] == 0;
            if (!finish) {
                const short2* hp = ev_hops + e * HMAX;
                double total = 0.0;
                for (int h = 0; h < ev_nh[e]; ++h) {
                    const int g = hp[h].x;
                    const int o = occ[g];
                    const double xp = o < B.pow_len ? xpw[o] : P.exec_pow[o];
                    total = __dadd_rn(total, __dmul_rn(__dmul_rn(base[g], xp), (double)hp[h].y));
                }
                if (!P.amortize_rtt) total = __dadd_rn(total, ev_crtt[e]);
                ev_time[e] = __dadd_rn(now, total);
                ev_seq[e] = next_seq;
                ev_kind[e] = K_STEP;
            }
        }
        finish = __shfl_sync(FULL, (int)finish, 0) != 0;
        if (!finish) { ++next_seq; __syncwarp(); continue; }
        // completion: release (sim.py:353-357), record, strict FIFO drain (sim.py:345-351)
        {
            const int i = ev_req[e];
            const short2* hp = ev_hops + e * HMAX;
            const long long tok = ev_tok[e];
            const int tag = -(i + 1);
            for (int h = lane; h < ev_nh[e]; h += 32) {
                const int g = hp[h].x;
                if (atomicExch(&stamp[g], tag) != tag) { occ[g] -= 1; kv[g] -= tok; }
            }
            __syncwarp();
            if (lane == 0) {
                P.done_time[r0 + i] = now;
                P.done_rank[r0 + i] = rank;
                ev_kind[e] = 0xFF;
            }
            ++rank;
            --live_n;
            ++completed;
            __syncwarp();
            while (adm < ap) {
                if (!try_admit(adm, now)) break;
                ++adm;
            }
        }
    }
    // requests never completed keep the caller's NaN / -1 (done_time / done_rank are written on completion)
    if (lane == 0) {
        P.duration[dag] = now;
        P.completed[dag] = completed;
        P.queue_peak[dag] = peak;
        P.n_events[dag] = events;
        P.status[dag] = status;
        P.aux[dag] = 0;
    }
}

// ---------------------------------------------------------------------------
// Wide pools (columns of up to 256 hosts): one CTA of NT threads per scenario.  The event loop runs in lockstep
// on every thread (warp-level argmins are computed redundantly per warp, scalar updates by thread 0 behind a
// barrier); the chain DP spreads destinations over the CTA and streams the edge blocks (ss_dag_edges layout)
// from global memory -- L2-resident for the scenarios in flight.
// ---------------------------------------------------------------------------
struct CtaLayout {
    int off_cl, off_noff, off_node, off_bp, off_picks, off_cost, off_red, off_tau, off_base, off_occ, off_stamp,
        off_kv, off_tcap, off_ppw, off_xpw, off_time, off_seq, off_req, off_rem, off_kind, off_nh, off_crtt, off_tok,
        off_hops, off_misc, total;
    int max_live, pow_len, cw;         // cw: padded column width (>= max hosts, multiple of 4) + 4
};

template <int NT>
__device__ double cta_route(const ss_dag_set& D, int l0, int nl, const int* cl, const int* noff, const int* node,
                            const double* tau, double* cost_a, double* cost_b, uint8_t* bp, int cw, int* picks,
                            double* red_v, int* red_i, int tid) {
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    const int nblk = nl - 1;
    double* cur = cost_a;
    double* nxt = cost_b;
    for (int q = tid; q < cl[0]; q += NT) cur[q] = tau[node[q]];
    __syncthreads();
    for (int b = 0; b < nblk; ++b) {
        const int rs = cl[b], rd = cl[b + 1];
        const double* Eb = D.edge_val + D.edge_off[l0 + b];
        for (int j = tid; j < rd; j += NT) {
            double best = INF;
            int bi = 0;                                          // +inf everywhere -> 0 == np.argmin
#pragma unroll 8
            for (int i = 0; i < rs; ++i) {
                const double a = __dadd_rn(cur[i], __ldg(Eb + (int64_t)i * rd + j));
                if (a < best) { best = a; bi = i; }              // ascending sources, strict <: first index
            }
            nxt[j] = __dadd_rn(best, tau[node[noff[b + 1] + j]]);
            bp[b * cw + j] = (uint8_t)bi;
        }
        __syncthreads();
        double* t = cur; cur = nxt; nxt = t;
    }
    // final argmin, first index (router.py:178)
    const int lane = tid & 31, warp = tid >> 5;
    double v = INF;
    int idx = NONE;
    for (int j = tid; j < cl[nblk]; j += NT) lexmin(v, idx, cur[j], j);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(FULL, v, o);
        const int i2 = __shfl_xor_sync(FULL, idx, o);
        lexmin(v, idx, v2, i2);
    }
    if (lane == 0) { red_v[warp] = v; red_i[warp] = idx; }
    __syncthreads();
    v = red_v[0];
    idx = red_i[0];
    for (int w = 1; w < NT / 32; ++w) lexmin(v, idx, red_v[w], red_i[w]);
    if (tid == 0 && v <= DBL_MAX) {
        int p = idx;
        picks[nblk] = p;
        for (int b = nblk - 1; b >= 0; --b) {
            p = bp[b * cw + p];
            picks[b] = p;
        }
    }
    __syncthreads();
    return v;
}

template <int NT>
__global__ void __launch_bounds__(NT) sim_cta_kernel(ss_dag_set D, CtaLayout B, SimArgs P) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int dag = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31;
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    const int l0 = D.layer_ptr[dag];
    const int nl = D.layer_ptr[dag + 1] - l0;
    int* cl = reinterpret_cast<int*>(smem + B.off_cl);
    int* noff = reinterpret_cast<int*>(smem + B.off_noff);
    int* node = reinterpret_cast<int*>(smem + B.off_node);
    uint8_t* bp = smem + B.off_bp;
    int* picks = reinterpret_cast<int*>(smem + B.off_picks);
    double* cost_a = reinterpret_cast<double*>(smem + B.off_cost);
    double* cost_b = cost_a + B.cw;
    double* red_v = reinterpret_cast<double*>(smem + B.off_red);
    int* red_i = reinterpret_cast<int*>(red_v + NT / 32);
    double* tau = reinterpret_cast<double*>(smem + B.off_tau);
    double* base = reinterpret_cast<double*>(smem + B.off_base);
    int* occ = reinterpret_cast<int*>(smem + B.off_occ);
    int* stamp = reinterpret_cast<int*>(smem + B.off_stamp);
    long long* kv = reinterpret_cast<long long*>(smem + B.off_kv);
    long long* tcap = reinterpret_cast<long long*>(smem + B.off_tcap);
    double* ppw = reinterpret_cast<double*>(smem + B.off_ppw);
    double* xpw = reinterpret_cast<double*>(smem + B.off_xpw);
    double* ev_time = reinterpret_cast<double*>(smem + B.off_time);
    int* ev_seq = reinterpret_cast<int*>(smem + B.off_seq);
    int* ev_req = reinterpret_cast<int*>(smem + B.off_req);
    int* ev_rem = reinterpret_cast<int*>(smem + B.off_rem);
    uint8_t* ev_kind = smem + B.off_kind;
    uint8_t* ev_nh = smem + B.off_nh;
    double* ev_crtt = reinterpret_cast<double*>(smem + B.off_crtt);
    long long* ev_tok = reinterpret_cast<long long*>(smem + B.off_tok);
    short2* ev_hops = reinterpret_cast<short2*>(smem + B.off_hops);
    volatile int* misc = reinterpret_cast<volatile int*>(smem + B.off_misc);     // [0] status [1] finish

    // ---- staging: columns and node ids (edges stay in global memory) -------------------------------------
    for (int l = tid; l < nl; l += NT) cl[l] = D.col_len[l0 + l];
    __syncthreads();
    if (tid == 0) {
        int nn = 0, bad = 0;
        for (int l = 0; l < nl; ++l) {
            if (cl[l] > B.cw - 4) bad = 1;
            noff[l] = nn;
            nn += cl[l];
        }
        misc[0] = bad ? SS_BAD_INPUT : SS_OK;
    }
    __syncthreads();
    if (misc[0] != SS_OK) {
        if (tid == 0) P.status[dag] = SS_BAD_INPUT;
        return;
    }
    for (int l = 0; l < nl; ++l)
        for (int q = tid; q < cl[l]; q += NT) node[noff[l] + q] = D.node_gpu[D.col_off[l0 + l] + q];
    const int gbase = P.gpu_ptr[dag];
    const int ng = P.gpu_ptr[dag + 1] - gbase;
    for (int g = tid; g < ng; g += NT) {
        occ[g] = 0;
        kv[g] = 0;
        stamp[g] = 0;
        base[g] = P.base_tau[gbase + g];
        tcap[g] = P.token_cap[gbase + g];
    }
    for (int o = tid; o < B.pow_len; o += NT) { ppw[o] = P.pub_pow[o]; xpw[o] = P.exec_pow[o]; }
    for (int e = tid; e < B.max_live; e += NT) ev_kind[e] = 0xFF;
    __syncthreads();
    const double* rtt = P.rtt + (int64_t)dag * D.max_gpus * D.max_gpus;
    const int r0 = P.trace_ptr[dag], n = P.trace_ptr[dag + 1] - r0;
    const double* arr = P.arrival + r0;
    const int32_t* prm = P.prompt + r0;
    const int32_t* outp = P.output + r0;

    int ap = 0, adm = 0, live_n = 0, live_hw = 0, next_seq = n + 1, completed = 0, peak = 0, status = SS_OK;
    bool tick = n > 0;
    double tick_t = P.publish_interval, now = 0.0;
    int tick_seq = n;
    long long events = 0;

    auto try_admit = [&](int i, double t) -> bool {
        const long long tok = (long long)prm[i] + outp[i];
        for (int g = tid; g < ng; g += NT) {
            const int o = occ[g];
            tau[g] = tcap[g] - kv[g] < tok ? INF : base[g] * (o < B.pow_len ? ppw[o] : P.pub_pow[o]);  // KV-blocked excluded
        }
        __syncthreads();
        const double v = cta_route<NT>(D, l0, nl, cl, noff, node, tau, cost_a, cost_b, bp, B.cw, picks, red_v, red_i,
                                       tid);
        if (!(v <= DBL_MAX)) return false;
        int slot = -1;                                           // same result in every warp
        for (int e0 = 0; e0 < B.max_live && slot < 0; e0 += 32) {
            const unsigned m = __ballot_sync(FULL, e0 + lane < B.max_live && ev_kind[e0 + lane] == 0xFF);
            if (m) slot = e0 + __ffs(m) - 1;
        }
        if (slot < 0) { status = SS_BAD_INPUT; return false; }
        const int tag = i + 1;
        for (int l = tid; l < nl; l += NT) {
            const int g = node[noff[l] + picks[l]];
            if (atomicExch(&stamp[g], tag) != tag) { atomicAdd(&occ[g], 1); atomicAdd((unsigned long long*)&kv[g], (unsigned long long)tok); }
        }
        __syncthreads();
        if (tid == 0) {
            int nh = 0, prev = -1;
            short2* hp = ev_hops + slot * HMAX;
            for (int l = 0; l < nl; ++l) {
                const int g = node[noff[l] + picks[l]];
                if (g == prev) { hp[nh - 1].y += 1; continue; }
                if (nh == HMAX) { nh = HMAX + 1; break; }
                hp[nh].x = (short)g;
                hp[nh].y = 1;
                ++nh;
                prev = g;
            }
            if (nh > HMAX) {
                misc[0] = SS_BAD_INPUT;
            } else {
                double crtt = 0.0;
                for (int h = 0; h + 1 < nh; ++h) crtt = __dadd_rn(crtt, rtt[(int64_t)hp[h].x * D.max_gpus + hp[h + 1].x]);
                PySum compute;
                compute.init();
                for (int h = 0; h < nh; ++h) compute.add_float(__dmul_rn(base[hp[h].x], (double)hp[h].y));
                const double pre = __dadd_rn(__dmul_rn(compute.value(), (double)prm[i]), crtt);
                ev_time[slot] = __dadd_rn(t, pre);
                ev_seq[slot] = next_seq;
                ev_req[slot] = i;
                ev_rem[slot] = outp[i];
                ev_kind[slot] = K_PREFILL;
                ev_nh[slot] = (uint8_t)nh;
                ev_crtt[slot] = crtt;
                ev_tok[slot] = tok;
            }
        }
        __syncthreads();
        status = misc[0];
        ++next_seq;
        ++live_n;
        if (slot + 1 > live_hw) live_hw = slot + 1;
        return status == SS_OK;
    };

    int rank = 0;
    while (status == SS_OK) {
        double bt = INF;
        int bs = 0x7fffffff, bk = -1;
        for (int e = lane; e < live_hw; e += 32) {               // every warp reduces all entries
            if (ev_kind[e] == 0xFF) continue;
            const double t = ev_time[e];
            const int q = ev_seq[e];
            if (t < bt || (t == bt && q < bs)) { bt = t; bs = q; bk = e; }
        }
        if (lane == 0) {
            if (ap < n && (arr[ap] < bt || (arr[ap] == bt && ap < bs))) { bt = arr[ap]; bs = ap; bk = -2; }
            if (tick && (tick_t < bt || (tick_t == bt && tick_seq < bs))) { bt = tick_t; bs = tick_seq; bk = -3; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double t2 = __shfl_xor_sync(FULL, bt, o);
            const int s2 = __shfl_xor_sync(FULL, bs, o);
            const int k2 = __shfl_xor_sync(FULL, bk, o);
            if (t2 < bt || (t2 == bt && s2 < bs)) { bt = t2; bs = s2; bk = k2; }
        }
        if (bk == -1) break;
        now = bt;
        ++events;
        if (bk == -3) {
            if (live_n > 0 || ap < n) { tick_t = __dadd_rn(now, P.publish_interval); tick_seq = next_seq++; }
            else tick = false;
            continue;
        }
        if (bk == -2) {
            const int i = ap++;
            if (adm < i || !try_admit(i, now)) {
                if (status != SS_OK) break;
                peak = max(peak, ap - adm);
            } else {
                ++adm;
            }
            continue;
        }
        const int e = bk;
        if (tid == 0) {
            if (ev_kind[e] == K_STEP) ev_rem[e] -= 1;
            const bool finish = ev_rem[e] == 0;
            misc[1] = finish;
            if (!finish) {
                const short2* hp = ev_hops + e * HMAX;
                double total = 0.0;
                for (int h = 0; h < ev_nh[e]; ++h) {
                    const int g = hp[h].x;
                    const int o = occ[g];
                    const double xp = o < B.pow_len ? xpw[o] : P.exec_pow[o];
                    total = __dadd_rn(total, __dmul_rn(__dmul_rn(base[g], xp), (double)hp[h].y));
                }
                if (!P.amortize_rtt) total = __dadd_rn(total, ev_crtt[e]);
                ev_time[e] = __dadd_rn(now, total);
                ev_seq[e] = next_seq;
                ev_kind[e] = K_STEP;
            }
        }
        __syncthreads();
        if (!misc[1]) { ++next_seq; __syncthreads(); continue; }
        {
            const int i = ev_req[e];
            const short2* hp = ev_hops + e * HMAX;
            const long long tok = ev_tok[e];
            const int tag = -(i + 1);
            for (int h = tid; h < ev_nh[e]; h += NT) {
                const int g = hp[h].x;
                if (atomicExch(&stamp[g], tag) != tag) { atomicSub(&occ[g], 1); atomicAdd((unsigned long long*)&kv[g], (unsigned long long)(-tok)); }
            }
            __syncthreads();
            if (tid == 0) {
                P.done_time[r0 + i] = now;
                P.done_rank[r0 + i] = rank;
                ev_kind[e] = 0xFF;
            }
            ++rank;
            --live_n;
            ++completed;
            __syncthreads();
            while (adm < ap) {
                if (!try_admit(adm, now)) break;
                ++adm;
            }
        }
    }
    if (tid == 0) {
        P.duration[dag] = now;
        P.completed[dag] = completed;
        P.queue_peak[dag] = peak;
        P.n_events[dag] = events;
        P.status[dag] = status;
        P.aux[dag] = 0;
    }
}

// ---------------------------------------------------------------------------
// 9..32 hosts per layer: the warp-resident layout of sim_warp_kernel (edges staged in shared memory), the
// lockstep event loop of sim_cta_kernel over NWD warps, and the destination-split chain DP (mw_route) for
// every admission attempt -- the route is most of a request's cost at C2 shape.
// ---------------------------------------------------------------------------
template <int NWD, int SPL, bool MAT = false>
__global__ void __launch_bounds__(NWD * 32) sim_mw_kernel(ss_dag_set D, WarpLayout A, SimLayout B, SimArgs P) {
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int NT = NWD * 32;
    const int dag = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const double INF = __longlong_as_double(0x7ff0000000000000ll);
    const int l0 = D.layer_ptr[dag];
    const int nl = D.layer_ptr[dag + 1] - l0;
    const int nblk = nl - 1;
    __shared__ double vshare;
    __shared__ int misc[2];                                     // [0] status / staging flag, [1] finish
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
    double* ppw = reinterpret_cast<double*>(smem + A.off_pow);
    double* costs = reinterpret_cast<double*>(smem + A.off_cost);
    long long* kv = reinterpret_cast<long long*>(smem + A.off_kv);
    long long* tcap = reinterpret_cast<long long*>(smem + A.off_tcap);
    double* ev_time = reinterpret_cast<double*>(smem + B.off_time);
    int* ev_seq = reinterpret_cast<int*>(smem + B.off_seq);
    int* ev_req = reinterpret_cast<int*>(smem + B.off_req);
    int* ev_rem = reinterpret_cast<int*>(smem + B.off_rem);
    uint8_t* ev_kind = smem + B.off_kind;
    uint8_t* ev_nh = smem + B.off_nh;
    double* ev_crtt = reinterpret_cast<double*>(smem + B.off_crtt);
    long long* ev_tok = reinterpret_cast<long long*>(smem + B.off_tok);
    short2* ev_hops = reinterpret_cast<short2*>(smem + B.off_hops);
    double* xpw = reinterpret_cast<double*>(smem + B.off_xpw);

    if (warp == 0)
        misc[0] = stage_dag(D, A, l0, nl, E, node, cl, noff, eoff, lane,
                            A.mat_dim ? P.rtt + (int64_t)dag * A.mat_dim * A.mat_dim : nullptr) ? SS_OK : SS_BAD_INPUT;
    __syncthreads();
    if (misc[0] != SS_OK) {
        if (tid == 0) P.status[dag] = SS_BAD_INPUT;
        return;
    }
    const int gbase = P.gpu_ptr[dag];
    const int ng = P.gpu_ptr[dag + 1] - gbase;
    for (int g = tid; g < ng; g += NT) {
        occ[g] = 0;
        kv[g] = 0;
        stamp[g] = 0;
        base[g] = P.base_tau[gbase + g];
        tcap[g] = P.token_cap[gbase + g];
    }
    for (int o = tid; o < B.pow_len; o += NT) { ppw[o] = P.pub_pow[o]; xpw[o] = P.exec_pow[o]; }
    for (int e = tid; e < B.max_live; e += NT) ev_kind[e] = 0xFF;
    if (tid < 8) { costs[32 + tid] = INF; costs[72 + tid] = INF; }
    __syncthreads();
    const double* rtt = P.rtt + (int64_t)dag * D.max_gpus * D.max_gpus;
    const int r0 = P.trace_ptr[dag], n = P.trace_ptr[dag + 1] - r0;
    const double* arr = P.arrival + r0;
    const int32_t* prm = P.prompt + r0;
    const int32_t* outp = P.output + r0;

    int ap = 0, adm = 0, live_n = 0, live_hw = 0, next_seq = n + 1, completed = 0, peak = 0, status = SS_OK;
    bool tick = n > 0;                          // sim.py:264-265: first tick only if work remains
    double tick_t = P.publish_interval, now = 0.0;
    int tick_seq = n;
    long long events = 0;

    auto try_admit = [&](int i, double t) -> bool {
        const long long tok = (long long)prm[i] + outp[i];
        for (int g = tid; g < ng; g += NT) {
            const int o = occ[g];
            tau[g] = tcap[g] - kv[g] < tok ? INF : base[g] * (o < B.pow_len ? ppw[o] : P.pub_pow[o]);  // KV-blocked excluded
        }
        __syncthreads();
        const double v = mw_route<NWD, SPL, MAT>(E, node, cl, noff, eoff, nblk, tau, costs, bp, picks, &vshare,
                                                 tid, A.mat_pitch);
        if (!(v <= DBL_MAX)) return false;
        int slot = -1;                                           // same result in every warp
        for (int e0 = 0; e0 < B.max_live && slot < 0; e0 += 32) {
            const unsigned m = __ballot_sync(FULL, e0 + lane < B.max_live && ev_kind[e0 + lane] == 0xFF);
            if (m) slot = e0 + __ffs(m) - 1;
        }
        if (slot < 0) { status = SS_BAD_INPUT; return false; }
        const int tag = i + 1;
        for (int l = tid; l < nl; l += NT) {
            const int g = node[noff[l] + picks[l]];
            if (atomicExch(&stamp[g], tag) != tag) { atomicAdd(&occ[g], 1); atomicAdd((unsigned long long*)&kv[g], (unsigned long long)tok); }
        }
        __syncthreads();
        if (tid == 0) {
            // merged hops, chain RTT, prefill = CPython sum(base_s * length) * prompt + chain RTT
            int nh = 0, prev = -1;
            short2* hp = ev_hops + slot * HMAX;
            for (int l = 0; l < nl; ++l) {
                const int g = node[noff[l] + picks[l]];
                if (g == prev) { hp[nh - 1].y += 1; continue; }
                if (nh == HMAX) { nh = HMAX + 1; break; }
                hp[nh].x = (short)g;
                hp[nh].y = 1;
                ++nh;
                prev = g;
            }
            if (nh > HMAX) {
                misc[0] = SS_BAD_INPUT;
            } else {
                double crtt = 0.0;
                for (int h = 0; h + 1 < nh; ++h) crtt = __dadd_rn(crtt, rtt[(int64_t)hp[h].x * D.max_gpus + hp[h + 1].x]);
                PySum compute;
                compute.init();
                for (int h = 0; h < nh; ++h) compute.add_float(__dmul_rn(base[hp[h].x], (double)hp[h].y));
                const double pre = __dadd_rn(__dmul_rn(compute.value(), (double)prm[i]), crtt);
                ev_time[slot] = __dadd_rn(t, pre);
                ev_seq[slot] = next_seq;
                ev_req[slot] = i;
                ev_rem[slot] = outp[i];
                ev_kind[slot] = K_PREFILL;
                ev_nh[slot] = (uint8_t)nh;
                ev_crtt[slot] = crtt;
                ev_tok[slot] = tok;
            }
        }
        __syncthreads();
        status = misc[0];
        ++next_seq;
        ++live_n;
        if (slot + 1 > live_hw) live_hw = slot + 1;
        return status == SS_OK;
    };

    int rank = 0;
    while (status == SS_OK) {
        // next event: lexicographic (time, seq) over live chains, the next arrival and the pending tick
        double bt = INF;
        int bs = 0x7fffffff, bk = -1;
        for (int e = lane; e < live_hw; e += 32) {               // every warp reduces all entries
            if (ev_kind[e] == 0xFF) continue;
            const double t = ev_time[e];
            const int q = ev_seq[e];
            if (t < bt || (t == bt && q < bs)) { bt = t; bs = q; bk = e; }
        }
        if (lane == 0) {
            if (ap < n && (arr[ap] < bt || (arr[ap] == bt && ap < bs))) { bt = arr[ap]; bs = ap; bk = -2; }
            if (tick && (tick_t < bt || (tick_t == bt && tick_seq < bs))) { bt = tick_t; bs = tick_seq; bk = -3; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double t2 = __shfl_xor_sync(FULL, bt, o);
            const int s2 = __shfl_xor_sync(FULL, bs, o);
            const int k2 = __shfl_xor_sync(FULL, bk, o);
            if (t2 < bt || (t2 == bt && s2 < bs)) { bt = t2; bs = s2; bk = k2; }
        }
        if (bk == -1) break;                                     // heap empty
        now = bt;
        ++events;
        if (bk == -3) {                                          // publish tick (sim.py:432-436)
            if (live_n > 0 || ap < n) { tick_t = __dadd_rn(now, P.publish_interval); tick_seq = next_seq++; }
            else tick = false;
            continue;
        }
        if (bk == -2) {                                          // arrival (sim.py:361-366)
            const int i = ap++;
            if (adm < i || !try_admit(i, now)) {
                if (status != SS_OK) break;
                peak = max(peak, ap - adm);
            } else {
                ++adm;
            }
            continue;
        }
        // prefill / step of live chain bk (sim.py:375-392)
        const int e = bk;
        if (tid == 0) {
            if (ev_kind[e] == K_STEP) ev_rem[e] -= 1;
            const bool finish = ev_rem[e] == 0;
            misc[1] = finish;
            if (!finish) {
                const short2* hp = ev_hops + e * HMAX;
                double total = 0.0;
                for (int h = 0; h < ev_nh[e]; ++h) {
                    const int g = hp[h].x;
                    const int o = occ[g];
                    const double xp = o < B.pow_len ? xpw[o] : P.exec_pow[o];
                    total = __dadd_rn(total, __dmul_rn(__dmul_rn(base[g], xp), (double)hp[h].y));
                }
                if (!P.amortize_rtt) total = __dadd_rn(total, ev_crtt[e]);
                ev_time[e] = __dadd_rn(now, total);
                ev_seq[e] = next_seq;
                ev_kind[e] = K_STEP;
            }
        }
        __syncthreads();
        const bool finish = misc[1] != 0;
        __syncthreads();                                         // misc[1] is rewritten by the next step event
        if (!finish) { ++next_seq; continue; }
        // completion: release (sim.py:353-357), record, strict FIFO drain (sim.py:345-351)
        {
            const int i = ev_req[e];
            const short2* hp = ev_hops + e * HMAX;
            const long long tok = ev_tok[e];
            const int tag = -(i + 1);
            for (int h = tid; h < ev_nh[e]; h += NT) {
                const int g = hp[h].x;
                if (atomicExch(&stamp[g], tag) != tag) { atomicSub(&occ[g], 1); atomicAdd((unsigned long long*)&kv[g], (unsigned long long)(-tok)); }
            }
            __syncthreads();
            if (tid == 0) {
                P.done_time[r0 + i] = now;
                P.done_rank[r0 + i] = rank;
                ev_kind[e] = 0xFF;
            }
            ++rank;
            --live_n;
            ++completed;
            __syncthreads();
            while (adm < ap) {
                if (!try_admit(adm, now)) break;
                ++adm;
            }
        }
    }
    // requests never completed keep the caller's NaN / -1 (done_time / done_rank are written on completion)
    if (tid == 0) {
        P.duration[dag] = now;
        P.completed[dag] = completed;
        P.queue_peak[dag] = peak;
        P.n_events[dag] = events;
        P.status[dag] = status;
        P.aux[dag] = 0;
    }
}

inline int align16s(int x) { return (x + 15) / 16 * 16; }

}  // namespace

extern "C" int ss_sim_warp(const ss_dag_set* dags, const int32_t* gpu_ptr, const double* base_tau,
                           const int64_t* token_cap, const double* rtt, const double* pub_pow, const double* exec_pow,
                           int32_t pow_len, const int32_t* trace_ptr, const double* arrival, const int32_t* prompt,
                           const int32_t* output, double publish_interval, int32_t amortize_rtt, int32_t max_live,
                           double* done_time, int32_t* done_rank, double* duration, int32_t* completed,
                           int32_t* queue_peak, int64_t* n_events, int32_t* status, int32_t* aux, void* stream) {
    if (!dags || !gpu_ptr || !base_tau || !token_cap || !rtt || !pub_pow || !exec_pow || pow_len < 2 || !trace_ptr ||
        !arrival || !prompt || !output || !done_time || !done_rank || !duration || !completed || !queue_peak ||
        !n_events || !status || !aux)
        return SS_BAD_INPUT;
    if (!(publish_interval > 0.0) || max_live < 1 || pow_len < max_live + 2) return SS_BAD_INPUT;
    const ss_dag_set& D = *dags;
    if (D.n_dags <= 0) return SS_OK;
    if (!D.edge_val || !D.edge_off) return SS_BAD_INPUT;
    WarpLayout A{};
    if (!warp_layout(D, 0, pow_len, A, D.max_gpus)) return SS_BAD_INPUT;   // rtt doubles as matrix-mode input
    SimLayout B{};
    B.pow_len = A.pow_len;                                   // cached prefix (<= 256); longer tables stay global
    // as many live-chain entries as shared memory holds (a scenario that needs more reports SS_BAD_INPUT)
    const int per_live = 8 + 4 + 4 + 4 + 1 + 1 + 8 + 8 + HMAX * 4;
    const int room = 227 * 1024 - A.total - align16s(B.pow_len * 8) - 10 * 16;
    if (room < per_live * 32) return SS_BAD_INPUT;
    B.max_live = max_live < room / per_live ? max_live : room / per_live;
    max_live = B.max_live;
    int o = A.total;
    B.off_time = o;  o += align16s(max_live * 8);
    B.off_seq = o;   o += align16s(max_live * 4);
    B.off_req = o;   o += align16s(max_live * 4);
    B.off_rem = o;   o += align16s(max_live * 4);
    B.off_kind = o;  o += align16s(max_live);
    B.off_nh = o;    o += align16s(max_live);
    B.off_crtt = o;  o += align16s(max_live * 8);
    B.off_tok = o;   o += align16s(max_live * 8);
    B.off_hops = o;  o += align16s(max_live * HMAX * 4);
    B.off_xpw = o;   o += align16s(B.pow_len * 8);
    B.total = o;
    if (B.total > 227 * 1024) return SS_BAD_INPUT;
    SimArgs P{gpu_ptr, base_tau, token_cap, rtt, pub_pow, exec_pow, pow_len, trace_ptr, arrival, prompt, output,
              publish_interval, amortize_rtt, done_time, done_rank, duration, completed, queue_peak, n_events,
              status, aux};
    cudaStream_t st = ss_stream(stream);
    auto run = [&](auto kern, int threads) -> int {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, B.total) != cudaSuccess)
            return SS_CUDA_ERROR;
        kern<<<D.n_dags, threads, B.total, st>>>(D, A, B, P);
        return SS_OK;
    };
    int rc;
    const bool mm = A.mat_dim > 0;
    switch ((D.max_hosts + 3) / 4) {                         // as ss_replay_warp: warps x source slots per lane
        case 0: case 1: case 2: rc = mm ? run(sim_warp_kernel<true>, 32) : run(sim_warp_kernel<false>, 32); break;
        case 3: rc = mm ? run(sim_mw_kernel<2, 3, true>, 64) : run(sim_mw_kernel<2, 3>, 64); break;
        case 4: rc = mm ? run(sim_mw_kernel<2, 4, true>, 64) : run(sim_mw_kernel<2, 4>, 64); break;
        case 5: rc = mm ? run(sim_mw_kernel<3, 5, true>, 96) : run(sim_mw_kernel<3, 5>, 96); break;
        case 6: rc = mm ? run(sim_mw_kernel<3, 6, true>, 96) : run(sim_mw_kernel<3, 6>, 96); break;
        case 7: rc = mm ? run(sim_mw_kernel<4, 7, true>, 128) : run(sim_mw_kernel<4, 7>, 128); break;
        default: rc = mm ? run(sim_mw_kernel<4, 8, true>, 128) : run(sim_mw_kernel<4, 8>, 128); break;
    }
    if (rc != SS_OK) return rc;
    SS_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_sim_cta(const ss_dag_set* dags, const int32_t* gpu_ptr, const double* base_tau,
                          const int64_t* token_cap, const double* rtt, const double* pub_pow, const double* exec_pow,
                          int32_t pow_len, const int32_t* trace_ptr, const double* arrival, const int32_t* prompt,
                          const int32_t* output, double publish_interval, int32_t amortize_rtt, int32_t max_live,
                          double* done_time, int32_t* done_rank, double* duration, int32_t* completed,
                          int32_t* queue_peak, int64_t* n_events, int32_t* status, int32_t* aux, void* stream) {
    if (!dags || !gpu_ptr || !base_tau || !token_cap || !rtt || !pub_pow || !exec_pow || pow_len < 2 || !trace_ptr ||
        !arrival || !prompt || !output || !done_time || !done_rank || !duration || !completed || !queue_peak ||
        !n_events || !status || !aux)
        return SS_BAD_INPUT;
    if (!(publish_interval > 0.0) || max_live < 1 || pow_len < max_live + 2) return SS_BAD_INPUT;
    const ss_dag_set& D = *dags;
    if (D.n_dags <= 0) return SS_OK;
    if (!D.edge_val || !D.edge_off || D.max_hosts > 256 || D.max_layers < 1) return SS_BAD_INPUT;
    constexpr int NT = 128;
    CtaLayout B{};
    B.pow_len = pow_len < 256 ? pow_len : 256;               // cached prefix; longer tables stay global
    B.cw = (D.max_hosts + 3) / 4 * 4 + 4;
    const int L = D.max_layers, G = D.max_gpus;
    B.max_live = max_live;
    for (;;) {                                               // as many live entries as shared memory holds
        const int fixed = align16s((L + 1) * 4) + align16s(L * 4) + align16s(L * D.max_hosts * 4) +
                          align16s(L * B.cw) + align16s(L * 4) + align16s(2 * B.cw * 8) + align16s(NT / 32 * 12) +
                          2 * align16s(G * 8) + 2 * align16s(G * 4) + 2 * align16s(G * 8) +
                          2 * align16s(B.pow_len * 8) + 16;
        const int per_live = 8 + 4 + 4 + 4 + 1 + 1 + 8 + 8 + HMAX * 4;
        const int room = 227 * 1024 - fixed - 9 * 16;
        if (room < per_live * 32) return SS_BAD_INPUT;
        if (B.max_live > room / per_live) B.max_live = room / per_live;
        break;
    }
    max_live = B.max_live;
    int o = 0;
    B.off_cl = o;    o += align16s((L + 1) * 4);
    B.off_noff = o;  o += align16s(L * 4);
    B.off_node = o;  o += align16s(L * D.max_hosts * 4);
    B.off_bp = o;    o += align16s(L * B.cw);
    B.off_picks = o; o += align16s(L * 4);
    B.off_cost = o;  o += align16s(2 * B.cw * 8);
    B.off_red = o;   o += align16s(NT / 32 * 12);
    B.off_tau = o;   o += align16s(G * 8);
    B.off_base = o;  o += align16s(G * 8);
    B.off_occ = o;   o += align16s(G * 4);
    B.off_stamp = o; o += align16s(G * 4);
    B.off_kv = o;    o += align16s(G * 8);
    B.off_tcap = o;  o += align16s(G * 8);
    B.off_ppw = o;   o += align16s(B.pow_len * 8);
    B.off_xpw = o;   o += align16s(B.pow_len * 8);
    B.off_time = o;  o += align16s(max_live * 8);
    B.off_seq = o;   o += align16s(max_live * 4);
    B.off_req = o;   o += align16s(max_live * 4);
    B.off_rem = o;   o += align16s(max_live * 4);
    B.off_kind = o;  o += align16s(max_live);
    B.off_nh = o;    o += align16s(max_live);
    B.off_crtt = o;  o += align16s(max_live * 8);
    B.off_tok = o;   o += align16s(max_live * 8);
    B.off_hops = o;  o += align16s(max_live * HMAX * 4);
    B.off_misc = o;  o += 16;
    B.total = o;
    if (B.total > 227 * 1024) return SS_BAD_INPUT;
    SimArgs P{gpu_ptr, base_tau, token_cap, rtt, pub_pow, exec_pow, pow_len, trace_ptr, arrival, prompt, output,
              publish_interval, amortize_rtt, done_time, done_rank, duration, completed, queue_peak, n_events,
              status, aux};
    if (cudaFuncSetAttribute(sim_cta_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, B.total) != cudaSuccess)
        return SS_CUDA_ERROR;
    sim_cta_kernel<NT><<<D.n_dags, NT, B.total, ss_stream(stream)>>>(D, B, P);
    SS_CHECK_LAUNCH();
    return SS_OK;
}
