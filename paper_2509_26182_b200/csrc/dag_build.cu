// On-device DAG construction.
//
//   ss_rtt_fill         router.py:118-143 rtt_matrix / topology.py:133-142 rtt_s
//   ss_dag_columns      router.py:87-115  build_dag (sorted host columns, UncoveredLayer)
//   ss_scenario_columns membership.py:193-206 hosts_of_layer after on_leave (C4/C5 states)
//   ss_dag_edges        router.py:169     E_l = M[col_l, col_{l+1}] gather, row-major
//
// These are byte/index-movement kernels: coalesced stores, warp-ballot stream
// compaction that preserves sorted-id order, no floating-point arithmetic
// except the scenario generator's jitter multiply (one IEEE product by a LogNormal(0, 0.2) quantile).
#include "ss_common.cuh"

namespace {

__global__ void rtt_fill_default(const int64_t* mat_off, const int32_t* mat_dim, double* out, double dflt) {
    const int item = blockIdx.y;
    const int64_t n = mat_dim[item];
    double* m = out + mat_off[item];
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = e / n, b = e - a * n;
        m[e] = (a == b) ? 0.0 : dflt;
    }
}

// pass 0 writes the mirror (b,a) of every link, pass 1 the direct (a,b): a
// directly published direction therefore always wins over a mirrored one.
__global__ void rtt_scatter(int32_t n_links, const int64_t* mat_off, const int32_t* mat_dim, double* out,
                            const int32_t* link_item, const int32_t* link_a, const int32_t* link_b,
                            const double* link_v, int pass) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_links) return;
    const int item = link_item ? link_item[t] : 0;
    const int a = link_a[t], b = link_b[t];
    if (a == b || a < 0 || b < 0) return;
    const int64_t n = mat_dim[item];
    double* m = out + mat_off[item];
    if (pass == 0)
        m[(int64_t)b * n + a] = link_v[t];
    else
        m[(int64_t)a * n + b] = link_v[t];
}

// One CTA per DAG, one warp per layer: ordered compaction with ballot/popc.
__global__ void dag_columns_kernel(const int32_t* layer_ptr, const int32_t* gpu_ptr, const int64_t* tau_off,
                                   const double* tau_table, const uint8_t* exclude, const int32_t* col_off,
                                   int32_t* col_len, int32_t* node_gpu, double* node_tau, int32_t* status,
                                   int32_t* aux) {
    const int d = blockIdx.x;
    const int l0 = layer_ptr[d], nl = layer_ptr[d + 1] - l0;
    const int g0 = gpu_ptr[d], ng = gpu_ptr[d + 1] - g0;
    const double* tau = tau_table + tau_off[d];
    __shared__ int first_empty;
    if (threadIdx.x == 0) first_empty = 0x7fffffff;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int l = warp; l < nl; l += nw) {
        const int base = col_off[l0 + l];
        int count = 0;
        for (int g = lane; g - lane < ng; g += 32) {
            double v = 0.0;
            bool present = false;
            if (g < ng) {
                v = tau[(int64_t)l * ng + g];
                present = !isnan(v) && !(exclude && exclude[g0 + g]);
            }
            const unsigned mask = __ballot_sync(0xffffffffu, present);
            if (present) {
                const int pos = count + __popc(mask & ((1u << lane) - 1u));
                node_gpu[base + pos] = g;
                if (node_tau) node_tau[base + pos] = v;
            }
            count += __popc(mask);
        }
        if (lane == 0) {
            col_len[l0 + l] = count;
            if (count == 0) atomicMin(&first_empty, l + 1);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const bool bad = first_empty != 0x7fffffff;
        status[d] = bad ? SS_UNCOVERED_LAYER : SS_OK;
        aux[d] = bad ? first_empty : 0;
    }
}

__global__ void scenario_columns_kernel(int32_t layers, int32_t n_gpus, const int32_t* lo, const int32_t* hi,
                                        int64_t slice_stride, const uint8_t* leave, const int32_t* col_off,
                                        int32_t* col_len, int32_t* node_gpu, int32_t* status, int32_t* aux) {
    const int s = blockIdx.x;
    lo += s * slice_stride;                               // per-scenario slices (joins) or the shared plan
    hi += s * slice_stride;
    const uint8_t* gone = leave ? leave + (int64_t)s * n_gpus : nullptr;
    __shared__ int first_empty;
    if (threadIdx.x == 0) first_empty = 0x7fffffff;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int l = warp; l < layers; l += nw) {
        const int fl = s * layers + l;
        const int base = col_off[fl];
        const int layer = l + 1;
        int count = 0;
        for (int g = lane; g - lane < n_gpus; g += 32) {
            const bool present = g < n_gpus && lo[g] <= layer && hi[g] >= layer && !(gone && gone[g]);
            const unsigned mask = __ballot_sync(0xffffffffu, present);
            if (present) node_gpu[base + count + __popc(mask & ((1u << lane) - 1u))] = g;
            count += __popc(mask);
        }
        if (lane == 0) {
            col_len[fl] = count;
            if (count == 0) atomicMin(&first_empty, layer);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const bool bad = first_empty != 0x7fffffff;
        status[s] = bad ? SS_UNCOVERED_LAYER : SS_OK;
        aux[s] = bad ? first_empty : 0;
    }
}

// grid (max_layers-1, n_dags): one CTA per boundary.
__global__ void dag_edges_kernel(ss_dag_set D, const int64_t* rtt_off, const int32_t* rtt_dim, const double* rtt,
                                 const int64_t* jitter_seed, int32_t n_pool, double* edge_val) {
    const int d = blockIdx.y, l = blockIdx.x;
    const int l0 = D.layer_ptr[d], nl = D.layer_ptr[d + 1] - l0;
    if (l >= nl - 1) return;
    const int fl = l0 + l;
    const int rs = D.col_len[fl], rd = D.col_len[fl + 1];
    const int* src = D.node_gpu + D.col_off[fl];
    const int* dst = D.node_gpu + D.col_off[fl + 1];
    double* out = edge_val + D.edge_off[fl];
    const bool jit = jitter_seed != nullptr;
    const int64_t dim = jit ? n_pool : rtt_dim[d];
    const double* m = jit ? rtt : rtt + rtt_off[d];
    const uint64_t mix = jit ? ss_splitmix64((uint64_t)jitter_seed[d]) : 0;
    const int total = rs * rd;
    // odd-sized blocks carry one pad double (16-B aligned starts); make it +inf
    if (threadIdx.x == 0 && (total & 1)) out[total] = __longlong_as_double(0x7ff0000000000000ll);
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
        const int i = e / rd, j = e - i * rd;
        const int a = src[i], b = dst[j];
        double v = m[(int64_t)a * dim + b];
        if (jit) v = v * ss_jitter(mix, (uint32_t)a, (uint32_t)b);
        out[e] = v;
    }
}

// out[s][a][b] = base[a][b] * jitter(seed_s, a, b) (scenarios.py:ScenarioSet.scenario_rtt: the pool matrix times the
// scenario's pair jitter: one IEEE product by the pair's LogNormal(0, 0.2) quantile, diagonal untouched)
__global__ void scenario_rtt_kernel(int32_t n_gpus, const double* base, const int64_t* seeds, double* out) {
    const int s = blockIdx.y;
    const uint64_t mix = ss_splitmix64((uint64_t)seeds[s]);
    const int64_t nn = (int64_t)n_gpus * n_gpus;
    double* o = out + (int64_t)s * nn;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nn; e += (int64_t)gridDim.x * blockDim.x) {
        const int a = (int)(e / n_gpus), b = (int)(e - (int64_t)a * n_gpus);
        const double v = base[e];
        o[e] = a == b ? v : v * ss_jitter(mix, (uint32_t)a, (uint32_t)b);
    }
}

}  // namespace

extern "C" int ss_rtt_fill(int32_t n_items, const int64_t* mat_off, const int32_t* mat_dim, double* out,
                           double default_value, int32_t n_links, const int32_t* link_item, const int32_t* link_a,
                           const int32_t* link_b, const double* link_v, void* stream) {
    if (n_items <= 0) return SS_OK;
    if (n_items > 65535 || !mat_off || !mat_dim || !out) return SS_BAD_INPUT;
    cudaStream_t s = ss_stream(stream);
    rtt_fill_default<<<dim3(64, n_items), 256, 0, s>>>(mat_off, mat_dim, out, default_value);
    SS_CHECK_LAUNCH();
    if (n_links > 0) {
        const int blocks = (n_links + 255) / 256;
        rtt_scatter<<<blocks, 256, 0, s>>>(n_links, mat_off, mat_dim, out, link_item, link_a, link_b, link_v, 0);
        SS_CHECK_LAUNCH();
        rtt_scatter<<<blocks, 256, 0, s>>>(n_links, mat_off, mat_dim, out, link_item, link_a, link_b, link_v, 1);
        SS_CHECK_LAUNCH();
    }
    return SS_OK;
}

extern "C" int ss_dag_columns(int32_t n_dags, const int32_t* layer_ptr, const int32_t* gpu_ptr,
                              const int64_t* tau_off, const double* tau_table, const uint8_t* exclude,
                              const int32_t* col_off, int32_t* col_len, int32_t* node_gpu, double* node_tau,
                              int32_t* status, int32_t* aux, void* stream) {
    if (n_dags <= 0) return SS_OK;
    dag_columns_kernel<<<n_dags, 256, 0, ss_stream(stream)>>>(layer_ptr, gpu_ptr, tau_off, tau_table, exclude,
                                                              col_off, col_len, node_gpu, node_tau, status, aux);
    SS_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_scenario_columns(int32_t n_scen, int32_t layers, int32_t n_gpus, const int32_t* slice_lo,
                                   const int32_t* slice_hi, int64_t slice_stride, const uint8_t* leave,
                                   const int32_t* col_off, int32_t* col_len, int32_t* node_gpu, int32_t* status,
                                   int32_t* aux, void* stream) {
    if (n_scen <= 0) return SS_OK;
    if (layers < 1 || n_gpus < 1 || slice_stride < 0) return SS_BAD_INPUT;
    scenario_columns_kernel<<<n_scen, 256, 0, ss_stream(stream)>>>(layers, n_gpus, slice_lo, slice_hi, slice_stride,
                                                                   leave, col_off, col_len, node_gpu, status, aux);
    SS_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_dag_edges(const ss_dag_set* dags, const int64_t* rtt_off, const int32_t* rtt_dim,
                            const double* rtt, const int64_t* jitter_seed, int32_t n_pool_gpus, double* edge_val,
                            void* stream) {
    if (!dags || dags->n_dags <= 0 || dags->max_layers < 2) return SS_OK;
    if (dags->n_dags > 65535) return SS_BAD_INPUT;
    dim3 grid(dags->max_layers - 1, dags->n_dags);
    dag_edges_kernel<<<grid, 256, 0, ss_stream(stream)>>>(*dags, rtt_off, rtt_dim, rtt, jitter_seed, n_pool_gpus,
                                                          edge_val);
    SS_CHECK_LAUNCH();
    return SS_OK;
}

extern "C" int ss_scenario_rtt(int32_t n_scen, int32_t n_gpus, const double* base_rtt, const int64_t* seeds,
                               double* out, void* stream) {
    if (n_scen <= 0) return SS_OK;
    if (n_gpus < 1 || !base_rtt || !seeds || !out || n_scen > 65535) return SS_BAD_INPUT;
    const int64_t nn = (int64_t)n_gpus * n_gpus;
    dim3 grid((unsigned)((nn + 255) / 256 < 64 ? (nn + 255) / 256 : 64), n_scen);
    scenario_rtt_kernel<<<grid, 256, 0, ss_stream(stream)>>>(n_gpus, base_rtt, seeds, out);
    SS_CHECK_LAUNCH();
    return SS_OK;
}
