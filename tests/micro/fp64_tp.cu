// FP64 / select / shuffle / barrier latency and single-warp throughput on B200 (sm_100a): which primitive bounds a
// one-scenario chain DP?  Dependent chains give latency; 8 independent chains per lane give single-warp issue rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tests/micro/fp64_tp tests/micro/fp64_tp.cu
#include <cstdio>
#include <cstdint>

template <int MODE>
__global__ void k(double* out, long long* cyc, double x0, int n) {
    __shared__ double sm[64];
    const int lane = threadIdx.x & 31;
    if (threadIdx.x < 64) sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    double a[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = x0 + q + lane;
    long long idx = lane;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        if (MODE == 0) a[0] = __dadd_rn(a[0], 1.0);                                   // DADD latency
        if (MODE == 1) {                                                                // DADD throughput (8 indep)
#pragma unroll
            for (int q = 0; q < 8; ++q) a[q] = __dadd_rn(a[q], 1.0);
        }
        if (MODE == 2) { a[0] = a[1] < a[0] ? a[1] : a[0]; a[1] = __longlong_as_double(__double_as_longlong(a[0]) ^ 1); }  // min step lat
        if (MODE == 3) {                                                                // DSETP+FSEL throughput
#pragma unroll
            for (int q = 0; q < 4; ++q) { a[q] = a[q + 4] < a[q] ? a[q + 4] : a[q]; a[q + 4] = __longlong_as_double(__double_as_longlong(a[q + 4]) + 1); }
        }
        if (MODE == 4) a[0] = __shfl_xor_sync(0xffffffffu, a[0], 1) + 0.0;              // SHFL.64 + DADD
        if (MODE == 5) { idx = (long long)sm[(int)(idx & 63)]; }                          // LDS.64 + F2I chain
        if (MODE == 6) { __syncthreads(); a[0] += 1.0; }                                  // bar.sync (blockDim)
        if (MODE == 7) { sm[lane] = a[0]; __syncwarp(); a[0] = sm[(lane + 1) & 31] + 1.0; __syncwarp(); }  // STS->LDS
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) s += a[q];
    out[threadIdx.x] = s + (double)idx;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int MODE>
double run(int threads, int n) {
    double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 64);
    k<MODE><<<1, threads>>>(o, c, 1.0, n); cudaDeviceSynchronize();
    k<MODE><<<1, threads>>>(o, c, 1.0, n);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    cudaFree(o); cudaFree(c);
    return h / (double)n;
}

int main() {
    const int n = 4096;
    printf("cycles per iteration\n");
    printf("DADD dependent            %.1f\n", run<0>(32, n));
    printf("DADD x8 independent, 1 warp  %.1f   (4 warps/CTA: %.1f, 16 warps: %.1f)\n", run<1>(32, n), run<1>(128, n), run<1>(512, n));
    printf("min step (DSETP+FSEL) + LOP dependent %.1f\n", run<2>(32, n));
    printf("4x min step independent, 1 warp %.1f   (4 warps: %.1f)\n", run<3>(32, n), run<3>(128, n));
    printf("SHFL.64 + DADD dependent %.1f\n", run<4>(32, n));
    printf("LDS.64 + F2I dependent   %.1f\n", run<5>(32, n));
    printf("bar.sync 1 warp %.1f  2 warps %.1f  3 warps %.1f  4 warps %.1f  8 warps %.1f\n", run<6>(32, n), run<6>(64, n),
           run<6>(96, n), run<6>(128, n), run<6>(256, n));
    printf("STS + syncwarp + LDS + DADD %.1f\n", run<7>(32, n));
}
