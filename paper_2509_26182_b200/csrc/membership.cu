// Membership churn and rebalance triggers on device.
//
//   ss_scenario_membership  membership.py:303-357  on_leave / on_join (bottleneck_layer) per scenario
//   ss_membership_triggers  membership.py:359-396  layer_loads / evaluate_triggers, perfmap.py:86-114
//
// One CTA per scenario.  The event generator is integer work: a bitonic sort of
// 64-bit splitmix keys in shared memory, then a warp-serial accept loop (each
// candidate's coverage test is one warp vote over its slice).  The trigger
// kernel replays CPython's float evaluation order exactly (PySum for sum(),
// plain folds for +=, -fmad=false), so decisions near the threshold agree
// with the reference bit for bit.
#include <float.h>

#include "ss_common.cuh"

namespace {

constexpr uint64_t LEAVE_SALT = 0xC4ull << 40;
constexpr uint64_t JOIN_SALT = 0x4Aull << 40;
constexpr unsigned FULL = 0xffffffffu;

// ascending (key, idx) bitonic sort of n2 (power of two) entries, all threads of the CTA
__device__ void bitonic_sort(uint64_t* key, int* idx, int n2) {
    for (int k = 2; k <= n2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                const int p = i ^ j;
                if (p > i) {
                    const bool up = (i & k) == 0;
                    const bool gt = key[i] > key[p] || (key[i] == key[p] && idx[i] > idx[p]);
                    if (gt == up) {
                        const uint64_t tk = key[i]; key[i] = key[p]; key[p] = tk;
                        const int ti = idx[i]; idx[i] = idx[p]; idx[p] = ti;
                    }
                }
            }
            __syncthreads();
        }
    }
}

__global__ void membership_kernel(int32_t layers, int32_t n_gpus, int32_t n2, const int32_t* lo, const int32_t* hi,
                                  const uint8_t* present0, const int64_t* token_cap, const int32_t* layer_cap,
                                  const int64_t* seeds, int32_t want_leave, int32_t n_join, uint8_t* absent,
                                  int32_t* lo_s, int32_t* hi_s, int32_t* joined, int32_t* status, int32_t* aux) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int s = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint64_t* key = reinterpret_cast<uint64_t*>(sm);
    int* idx = reinterpret_cast<int*>(key + n2);
    long long* tot = reinterpret_cast<long long*>(idx + n2 + (n2 & 1));   // [layers + 2]
    int* cover = reinterpret_cast<int*>(tot + layers + 2);                 // [layers + 2]
    int* slo = cover + layers + 2;                                         // working slices [n_gpus]
    int* shi = slo + n_gpus;
    uint8_t* gone = reinterpret_cast<uint8_t*>(shi + n_gpus);              // [n_gpus]
    __shared__ int n_cand, first_hole;

    const uint64_t mix = ss_splitmix64((uint64_t)seeds[s]);
    for (int l = tid; l < layers + 2; l += blockDim.x) { tot[l] = 0; cover[l] = 0; }
    if (tid == 0) first_hole = 0x7fffffff;
    __syncthreads();
    for (int g = tid; g < n_gpus; g += blockDim.x) {
        const bool here = present0[g] != 0;
        const bool has = here && lo[g] <= hi[g];
        slo[g] = has ? lo[g] : 0;
        shi[g] = has ? hi[g] : -1;
        gone[g] = here ? 0 : 1;
        if (has)
            for (int l = lo[g]; l <= hi[g]; ++l) {
                atomicAdd(&cover[l], 1);
                atomicAdd(reinterpret_cast<unsigned long long*>(&tot[l]), (unsigned long long)token_cap[g]);
            }
    }
    __syncthreads();

    // ---- 1. departures: seeded order over the plan GPUs present now ---------------------------------
    if (want_leave > 0) {
        for (int i = tid; i < n2; i += blockDim.x) {
            const bool cand = i < n_gpus && !gone[i] && slo[i] <= shi[i];
            key[i] = cand ? ss_splitmix64(mix ^ LEAVE_SALT ^ (uint64_t)i) : ~0ull;
            idx[i] = cand ? i : 0x7fffffff;
        }
        __syncthreads();
        bitonic_sort(key, idx, n2);
        if (warp == 0) {
            int taken = 0;
            for (int i = 0; i < n2 && taken < want_leave; ++i) {
                const int g = idx[i];
                if (g == 0x7fffffff) break;
                const int a = slo[g], b = shi[g];
                bool ok = true;
                for (int l = a + lane; l <= b; l += 32) ok &= cover[l] >= 2;
                if (__all_sync(FULL, ok)) {
                    for (int l = a + lane; l <= b; l += 32) {
                        cover[l] -= 1;
                        tot[l] -= token_cap[g];
                    }
                    if (lane == 0) {
                        gone[g] = 1;
                        slo[g] = 0;
                        shi[g] = -1;
                    }
                    ++taken;
                }
                __syncwarp();
            }
        }
        __syncthreads();
    }

    // ---- 2. joins: seeded order over the absent pool, each at the current bottleneck layer -----------
    if (n_join > 0) {
        if (tid == 0) n_cand = 0;
        __syncthreads();
        for (int i = tid; i < n2; i += blockDim.x) {
            const bool cand = i < n_gpus && present0[i] == 0;
            key[i] = cand ? ss_splitmix64(mix ^ JOIN_SALT ^ (uint64_t)i) : ~0ull;
            idx[i] = cand ? i : 0x7fffffff;
            if (cand) atomicAdd(&n_cand, 1);
        }
        __syncthreads();
        bitonic_sort(key, idx, n2);
        if (warp == 0) {
            for (int j = 0; j < n_join; ++j) {
                const int g = j < n_cand ? idx[j] : -1;
                if (lane == 0) joined[(int64_t)s * n_join + j] = g;
                if (g < 0) continue;
                // bottleneck_layer: first layer with the least summed token capacity (membership.py:303-315)
                long long best = LLONG_MAX;
                int bl = 0x7fffffff;
                for (int l = 1 + lane; l <= layers; l += 32)
                    if (tot[l] < best) { best = tot[l]; bl = l; }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const long long b2 = __shfl_xor_sync(FULL, best, o);
                    const int l2 = __shfl_xor_sync(FULL, bl, o);
                    if (b2 < best || (b2 == best && l2 < bl)) { best = b2; bl = l2; }
                }
                const int cap = layer_cap[g];
                if (cap >= 1) {
                    const int end = min(bl + cap - 1, layers);
                    for (int l = bl + lane; l <= end; l += 32) {
                        cover[l] += 1;
                        tot[l] += token_cap[g];
                    }
                    if (lane == 0) { slo[g] = bl; shi[g] = end; }
                }
                if (lane == 0) gone[g] = 0;
                __syncwarp();
            }
        }
        __syncthreads();
    }

    // ---- outputs ------------------------------------------------------------------------------------
    for (int g = tid; g < n_gpus; g += blockDim.x) {
        absent[(int64_t)s * n_gpus + g] = gone[g];
        lo_s[(int64_t)s * n_gpus + g] = slo[g];
        hi_s[(int64_t)s * n_gpus + g] = shi[g];
    }
    for (int l = 1 + tid; l <= layers; l += blockDim.x)
        if (cover[l] == 0) atomicMin(&first_hole, l);
    __syncthreads();
    if (tid == 0) {
        const bool bad = first_hole != 0x7fffffff;
        status[s] = bad ? SS_UNCOVERED_LAYER : SS_OK;
        aux[s] = bad ? first_hole : 0;
    }
}

__global__ void triggers_kernel(int32_t layers, int32_t n_gpus, const uint8_t* absent, const int32_t* lo_s,
                                const int32_t* hi_s, int64_t slice_stride, const int32_t* gpu_order, int32_t n_order,
                                const int32_t* slice_order, int32_t n_slice_order, int64_t order_stride,
                                const int32_t* joined,
                                int32_t n_join, const double* vram, const double* reserve, const double* flops,
                                const int64_t* token_cap, const int64_t* kv_reserved, const int32_t* occ,
                                int64_t state_stride, double mix_alpha, double cov_threshold, double* loads_out,
                                double* cov_out, int32_t* decision, int32_t* first_uncovered) {
    extern __shared__ __align__(16) unsigned char sm[];
    const int s = blockIdx.x;
    const int tid = threadIdx.x;
    double* loads = reinterpret_cast<double*>(sm);                       // [layers]
    __shared__ double tmem, tflops;
    __shared__ int first_hole;
    const uint8_t* gone = absent + (int64_t)s * n_gpus;
    const int32_t* lo = lo_s + s * slice_stride;
    const int32_t* hi = hi_s + s * slice_stride;
    const int32_t* jn = joined ? joined + (int64_t)s * n_join : nullptr;
    const int64_t* kv = kv_reserved ? kv_reserved + s * state_stride : nullptr;
    const int32_t* oc = occ ? occ + s * state_stride : nullptr;

    // total_memory / total_flops: CPython sum() over _gpus in insertion order (membership.py:366-369)
    if (tid == 0) {
        PySum m, f;
        m.init();
        f.init();
        for (int i = 0; i < n_order; ++i) {
            const int g = gpu_order[i];
            if (gone[g]) continue;
            m.add_float(__dmul_rn(vram[g], reserve[g]));
            f.add_float(flops[g]);
        }
        for (int j = 0; j < n_join && jn; ++j) {
            const int g = jn[j];
            if (g < 0 || gone[g]) continue;
            m.add_float(__dmul_rn(vram[g], reserve[g]));
            f.add_float(flops[g]);
        }
        tmem = m.value();
        tflops = f.value();
        first_hole = 0x7fffffff;
    }
    __syncthreads();
    // per layer: plain += folds in slices order (plan.gpu_slices() order, then joins)
    for (int l = 1 + tid; l <= layers; l += blockDim.x) {
        double kvb = 0.0, comp = 0.0;
        bool covered = false;
        auto visit = [&](int g) {
            if (g < 0 || gone[g] || lo[g] > l || hi[g] < l) return;
            covered = true;
            const long long cap = token_cap[g];
            if (cap > 0) {
                const double uf = __ddiv_rn((double)(kv ? kv[g] : 0), (double)cap);
                kvb = __dadd_rn(kvb, __dmul_rn(__dmul_rn(uf, vram[g]), reserve[g]));
            }
            const int o = oc ? oc[g] : 0;
            comp = __dadd_rn(comp, __dmul_rn(flops[g], (double)(o < 1 ? o : 1)));
        };
        // slices order: the plan's, then joins (on_join appends); after a rebalance each scenario has its own
        // plan order (order_stride > 0) that already contains every serving GPU
        const int32_t* so = slice_order + s * order_stride;
        for (int i = 0; i < n_slice_order; ++i) visit(so[i]);
        if (order_stride == 0)
            for (int j = 0; j < n_join && jn; ++j) visit(jn[j]);
        const double kvf = tmem > 0.0 ? __ddiv_rn(kvb, tmem) : 0.0;
        const double cf = tflops > 0.0 ? __ddiv_rn(comp, tflops) : 0.0;
        loads[l - 1] = __dadd_rn(__dmul_rn(mix_alpha, kvf), __dmul_rn(__dsub_rn(1.0, mix_alpha), cf));
        if (!covered) atomicMin(&first_hole, l);
    }
    __syncthreads();
    if (tid == 0) {
        // layer_load_cov: population CoV with sum()-based mean and variance (perfmap.py:105-114)
        double cov = 0.0;
        if (layers > 0) {
            PySum a;
            a.init();
            for (int l = 0; l < layers; ++l) a.add_float(loads[l]);
            const double mean = __ddiv_rn(a.value(), (double)layers);
            if (mean != 0.0) {
                PySum v;
                v.init();
                for (int l = 0; l < layers; ++l) {
                    const double d = __dsub_rn(loads[l], mean);
                    v.add_float(__dmul_rn(d, d));
                }
                cov = __ddiv_rn(__dsqrt_rn(__ddiv_rn(v.value(), (double)layers)), mean);
            }
        }
        const bool hole = first_hole != 0x7fffffff;
        cov_out[s] = cov;
        first_uncovered[s] = hole ? first_hole : 0;
        decision[s] = hole ? 1 : (cov > cov_threshold ? 2 : 0);
    }
    if (loads_out)
        for (int l = tid; l < layers; l += blockDim.x) loads_out[(int64_t)s * layers + l] = loads[l];
}

}  // namespace

extern "C" int ss_scenario_membership(int32_t n_scen, int32_t layers, int32_t n_gpus, const int32_t* slice_lo,
                                      const int32_t* slice_hi, const uint8_t* present0, const int64_t* token_cap,
                                      const int32_t* layer_cap, const int64_t* seeds, int32_t want_leave,
                                      int32_t n_join, uint8_t* absent, int32_t* lo_s, int32_t* hi_s, int32_t* joined,
                                      int32_t* status, int32_t* aux, void* stream) {
    if (n_scen <= 0) return SS_OK;
    if (layers < 1 || n_gpus < 1 || n_gpus > SS_MAX_GPUS || want_leave < 0 || n_join < 0) return SS_BAD_INPUT;
    if (n_join > 0 && !joined) return SS_BAD_INPUT;
    int n2 = 1;
    while (n2 < n_gpus) n2 <<= 1;
    const size_t smem = (size_t)n2 * 8 + (size_t)(n2 + (n2 & 1)) * 4 + (size_t)(layers + 2) * 12 +
                        (size_t)n_gpus * 9 + 16;
    if (smem > 227 * 1024) return SS_BAD_INPUT;
    if (cudaFuncSetAttribute(membership_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return SS_CUDA_ERROR;
    membership_kernel<<<n_scen, 256, smem, ss_stream(stream)>>>(layers, n_gpus, n2, slice_lo, slice_hi, present0,
                                                                token_cap, layer_cap, seeds, want_leave, n_join,
                                                                absent, lo_s, hi_s, joined, status, aux);
    SS_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_membership_triggers(int32_t n_scen, int32_t layers, int32_t n_gpus, const uint8_t* absent,
                                      const int32_t* lo_s, const int32_t* hi_s, int64_t slice_stride,
                                      const int32_t* gpu_order, int32_t n_order, const int32_t* slice_order,
                                      int32_t n_slice_order, int64_t order_stride, const int32_t* joined, int32_t n_join,
                                      const double* vram,
                                      const double* reserve, const double* flops, const int64_t* token_cap,
                                      const int64_t* kv_reserved, const int32_t* occ, int64_t state_stride,
                                      double mix_alpha, double cov_threshold, double* loads, double* cov,
                                      int32_t* decision, int32_t* first_uncovered, void* stream) {
    if (n_scen <= 0) return SS_OK;
    if (layers < 1 || n_gpus < 1 || !absent || !lo_s || !hi_s || !cov || !decision || !first_uncovered)
        return SS_BAD_INPUT;
    if (!(mix_alpha >= 0.0 && mix_alpha <= 1.0)) return SS_BAD_INPUT;    // perfmap.py:98-99 ValueError
    const size_t smem = (size_t)layers * 8;
    if (smem > 227 * 1024) return SS_BAD_INPUT;
    if (cudaFuncSetAttribute(triggers_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return SS_CUDA_ERROR;
    triggers_kernel<<<n_scen, 128, smem, ss_stream(stream)>>>(layers, n_gpus, absent, lo_s, hi_s, slice_stride,
                                                              gpu_order, n_order, slice_order, n_slice_order,
                                                              order_stride, joined,
                                                              n_join, vram, reserve, flops, token_cap, kv_reserved,
                                                              occ, state_stride, mix_alpha, cov_threshold, loads, cov,
                                                              decision, first_uncovered);
    SS_CHECK_LAUNCH();
    return SS_OK;
}

// ---------------------------------------------------------------------------
// abort of live chains (sim.py:401-411 _abort_chains_on): every chain still in the release window that
// touches a marked GPU is released now (occupancy -1 on each of its distinct GPUs) and its ring slot
// emptied, so the later release(i - W) is a no-op.  One warp per scenario.
// ---------------------------------------------------------------------------
namespace {
__global__ void ring_abort_kernel(int32_t n_gpus, int32_t max_layers, int32_t window, const uint8_t* mark,
                                  int32_t* occ, int32_t* ring, const int64_t* next_req, int32_t* n_aborted,
                                  uint8_t* aborted) {
    const int s = blockIdx.x, lane = threadIdx.x;
    const int stride = max_layers + 1;
    const uint8_t* mk = mark + (int64_t)s * n_gpus;
    int32_t* oc = occ + (int64_t)s * n_gpus;
    int32_t* rg = ring + (int64_t)s * window * stride;
    const int64_t nr = next_req[s];
    const int64_t first = nr - window < 0 ? 0 : nr - window;
    int count = 0;
    for (int64_t i = first; i < nr; ++i) {                    // request-id order, as sim.py sorts victims
        int32_t* slot = rg + (int)(i % window) * stride;
        const int cnt = slot[0];
        bool hit = false;
        for (int k = lane; k < cnt; k += 32) hit |= mk[slot[1 + k]] != 0;
        hit = __any_sync(0xffffffffu, hit);
        if (hit) {
            for (int k = lane; k < cnt; k += 32) oc[slot[1 + k]] -= 1;
            __syncwarp();
            if (lane == 0) slot[0] = 0;
            ++count;
        }
        if (aborted && lane == 0) aborted[(int64_t)s * window + (int)(i % window)] = hit ? 1 : 0;
        __syncwarp();
    }
    if (lane == 0 && n_aborted) n_aborted[s] = count;
}
}  // namespace

extern "C" int ss_ring_abort(int32_t n_scen, int32_t n_gpus, int32_t max_layers, int32_t window, const uint8_t* mark,
                             int32_t* occ, int32_t* ring, const int64_t* next_req, int32_t* n_aborted,
                             uint8_t* aborted, void* stream) {
    if (n_scen <= 0 || window == 0) return SS_OK;            // W = 0 keeps no live chain
    if (window < 0 || n_gpus < 1 || max_layers < 1 || !mark || !occ || !ring || !next_req) return SS_BAD_INPUT;
    ring_abort_kernel<<<n_scen, 32, 0, ss_stream(stream)>>>(n_gpus, max_layers, window, mark, occ, ring, next_req,
                                                            n_aborted, aborted);
    SS_CHECK_LAUNCH();
    return SS_OK;
}
