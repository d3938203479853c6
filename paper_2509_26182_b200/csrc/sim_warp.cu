// Serving simulator on device (the admission path with occupancy-dependent step time).
//
// One warp runs one scenario's discrete-event simulation of pkg/src/swarmsched/sim.py:_Simulation (no
// membership events), with the scenario's DAG warp-resident (<= 32 hosts per layer, warp_dag.cuh):
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
    int max_live, pow_len;
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

    if (!stage_dag(D, A, l0, nl, E, node, cl, noff, eoff, lane)) {
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
            const int o = occ[g] < B.pow_len ? occ[g] : B.pow_len - 1;
            tau[g] = tcap[g] - kv[g] < tok ? INF : base[g] * ppw[o];    // KV-blocked GPUs excluded
        }
        __syncwarp();
        const double v = warp_route(E, node, cl, noff, eoff, nblk, tau, costs, bp, picks, lane);
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
                    const int o = occ[g] < B.pow_len ? occ[g] : B.pow_len - 1;
                    total = __dadd_rn(total, __dmul_rn(__dmul_rn(base[g], xpw[o]), (double)hp[h].y));
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
    if (!(publish_interval > 0.0) || max_live < 1) return SS_BAD_INPUT;
    const ss_dag_set& D = *dags;
    if (D.n_dags <= 0) return SS_OK;
    if (!D.edge_val || !D.edge_off) return SS_BAD_INPUT;
    WarpLayout A{};
    if (!warp_layout(D, 0, pow_len, A)) return SS_BAD_INPUT;
    SimLayout B{};
    B.max_live = max_live;
    B.pow_len = pow_len;
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
    B.off_xpw = o;   o += align16s(pow_len * 8);
    B.total = o;
    // the published-power table shares A's pow slot: make sure it holds pow_len entries
    if (A.pow_len < pow_len) return SS_BAD_INPUT;
    if (B.total > 227 * 1024) return SS_BAD_INPUT;
    SimArgs P{gpu_ptr, base_tau, token_cap, rtt, pub_pow, exec_pow, pow_len, trace_ptr, arrival, prompt, output,
              publish_interval, amortize_rtt, done_time, done_rank, duration, completed, queue_peak, n_events,
              status, aux};
    if (cudaFuncSetAttribute(sim_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, B.total) != cudaSuccess)
        return SS_CUDA_ERROR;
    sim_warp_kernel<<<D.n_dags, 32, B.total, ss_stream(stream)>>>(D, A, B, P);
    SS_CHECK_LAUNCH();
    return SS_OK;
}
