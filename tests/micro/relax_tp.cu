// Throughput microbenchmark of the slot-tile relaxation (replay_slots.cu) in isolation: per boundary every
// warp scans its source range against its destination slots (value + first index), stores its partials and
// the CTA meets at one barrier.  Varies the warp split (source ranges x destination groups), destinations per
// lane and the index tracking, at 2 CTAs per SM -- which mapping keeps the issue slots busy?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tests/micro/relax_tp tests/micro/relax_tp.cu
#include <cstdio>
#include <cstdint>

constexpr int S = 96;        // slots
constexpr int R = 73;        // sources per boundary (C4 k)

template <int DPL, int NSR, int NDG, bool IDX, int MODE = 0, int W = 97, bool BC = false>
__global__ void __launch_bounds__(NSR * NDG * 32, 2) relax(int nbnd, double* out, long long* cyc) {
    extern __shared__ __align__(16) double sm[];
    double* T = sm;                                  // [S][W]
    double* cost = T + S * W;                        // [NSR][40] per source range, 16-B aligned
    int* rowoff = reinterpret_cast<int*>(cost + NSR * 40);   // [NSR][40]
    double* part_v = reinterpret_cast<double*>(rowoff + NSR * 40);   // [NSR][S]
    int* part_i = reinterpret_cast<int*>(part_v + NSR * S);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nt = blockDim.x;
    for (int i = tid; i < S * W; i += nt) T[i] = (double)((i * 2654435761u) & 1023) * 1e-3;
    for (int i = tid; i < NSR * 40; i += nt) { cost[i] = (double)(i & 7) * 1e-3; rowoff[i] = ((i * 37) % S) * W * 8; }
    __syncthreads();
    const int sr = warp / NDG, dg = warp % NDG;
    const int p0 = sr * R / NSR, n = (sr + 1) * R / NSR - p0;
    const char* Tb = reinterpret_cast<const char*>(T + dg * DPL * 32 + (BC ? 0 : lane));
    long long t0 = clock64();
    double acc = 0.0;
    for (int b = 0; b < nbnd; ++b) {
        double v[DPL];
        int ix[DPL];
#pragma unroll
        for (int d = 0; d < DPL; ++d) { v[d] = 1e300; ix[d] = 0x7fff; }
#pragma unroll 2
        for (int k = 0; k < n; k += 2) {
            const double2 c = *reinterpret_cast<const double2*>(cost + sr * 40 + k);
            const int2 r2 = *reinterpret_cast<const int2*>(rowoff + sr * 40 + k);
#pragma unroll
            for (int d = 0; d < DPL; ++d) {
                const double t1 = reinterpret_cast<const double*>(Tb + r2.x)[d * 32];
                const double t2 = reinterpret_cast<const double*>(Tb + r2.y)[d * 32];
                if (MODE == 0) {
                    const double a = __dadd_rn(c.x, t1);
                    if (IDX) { if (a < v[d]) { v[d] = a; ix[d] = p0 + k; } }
                    else v[d] = fmin(v[d], a);
                    const double a2 = __dadd_rn(c.y, t2);
                    if (IDX) { if (a2 < v[d]) { v[d] = a2; ix[d] = p0 + k + 1; } }
                    else v[d] = fmin(v[d], a2);
                } else {
                    // MODE 1: DADD + 64-bit integer compare (non-negative doubles order like their bit patterns)
                    // MODE 2: integer add + integer compare (no FP64 at all -- pipe probe, not exact)
                    long long vi = __double_as_longlong(v[d]);
                    const long long a = MODE == 1 ? __double_as_longlong(__dadd_rn(c.x, t1))
                                                  : __double_as_longlong(c.x) + __double_as_longlong(t1);
                    if (a < vi) { vi = a; ix[d] = p0 + k; }
                    const long long a2 = MODE == 1 ? __double_as_longlong(__dadd_rn(c.y, t2))
                                                   : __double_as_longlong(c.y) + __double_as_longlong(t2);
                    if (a2 < vi) { vi = a2; ix[d] = p0 + k + 1; }
                    v[d] = __longlong_as_double(vi);
                }
            }
        }
#pragma unroll
        for (int d = 0; d < DPL; ++d) {
            part_v[sr * S + dg * DPL * 32 + d * 32 + lane] = v[d];
            part_i[sr * S + dg * DPL * 32 + d * 32 + lane] = ix[d];
        }
        __syncthreads();
        // merge stand-in: one lane per slot reads the NSR partials (what the next boundary's stage does)
        if (tid < S) {
            double m = part_v[tid];
            int mi = part_i[tid];
            for (int w = 1; w < NSR; ++w) {
                const double x = part_v[w * S + tid];
                const int xi = part_i[w * S + tid];
                if (x < m || (x == m && xi < mi)) { m = x; mi = xi; }
            }
            acc += m + mi;
            if (tid < R) cost[(tid % NSR) * 40 + tid / NSR] += m * 1e-9;
        }
        __syncthreads();
    }
    long long t1 = clock64();
    out[blockIdx.x * nt + tid] = acc;
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int DPL, int NSR, int NDG, bool IDX, int MODE = 0, int W = 97, bool BC = false>
void run(const char* name, double* o, long long* c, int sms, int per_sm = 2) {
    const int threads = NSR * NDG * 32;
    const int smem = (S * W + NSR * 40) * 8 + NSR * 40 * 4 + NSR * S * 12 + 64;
    cudaFuncSetAttribute(relax<DPL, NSR, NDG, IDX, MODE, W, BC>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int nb = 2000, grid = per_sm * sms;
    relax<DPL, NSR, NDG, IDX, MODE, W, BC><<<grid, threads, smem>>>(10, o, c);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    relax<DPL, NSR, NDG, IDX, MODE, W, BC><<<grid, threads, smem>>>(nb, o, c);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h;
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    const double relax_per_s = (double)grid * nb * R * 73 / (ms * 1e-3);
    printf("%-34s threads %3d smem %6d | %7.1f cycles/boundary/CTA | %.3e useful relax/s (C4 sel/s eq %.2e) %s\n",
           name, threads, smem, (double)h / nb, relax_per_s, relax_per_s / (63.0 * 73 * 73),
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* o;
    long long* c;
    cudaMalloc(&o, 2 * sms * 1024 * 8);
    cudaMalloc(&c, 2 * sms * 8);
    run<3, 4, 1, true>("DPL3 x 4 source ranges (today)", o, c, sms);
    run<3, 4, 1, false>("DPL3 x 4 ranges, value only", o, c, sms);
    run<3, 8, 1, true>("DPL3 x 8 ranges", o, c, sms);
    run<1, 4, 3, true>("DPL1 x 3 dest groups x 4 ranges", o, c, sms);
    run<1, 3, 3, true>("DPL1 x 3 dest groups x 3 ranges", o, c, sms);
    run<1, 5, 3, true>("DPL1 x 3 dest groups x 5 ranges", o, c, sms);
    run<3, 6, 1, true>("DPL3 x 6 ranges", o, c, sms);
    run<1, 4, 3, false>("DPL1 x 3 x 4, value only", o, c, sms);
    run<3, 4, 1, true, 0, 96>("DPL3 x 4, pitch 96 (aligned rows)", o, c, sms);
    run<3, 4, 1, true, 0, 97, true>("DPL3 x 4, broadcast T reads", o, c, sms);
    run<3, 4, 1, true>("DPL3 x 4, 1 CTA per SM", o, c, sms, 1);
    run<3, 4, 1, true, 0, 96>("DPL3 x 4, pitch 96, 1 CTA per SM", o, c, sms, 1);
    run<3, 4, 1, true, 1>("DPL3 x 4, DADD + int64 compare", o, c, sms);
    run<3, 4, 1, true, 2>("DPL3 x 4, int add + int compare", o, c, sms);
    run<1, 4, 3, true, 1>("DPL1 x 3 x 4, DADD + int64 cmp", o, c, sms);
    run<1, 4, 3, true, 2>("DPL1 x 3 x 4, int add + int cmp", o, c, sms);
    return 0;
}
