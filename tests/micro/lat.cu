// Latency microbenchmark (dependent chains, one warp): DADD, DSETP+FSEL min, int64 compare+select, LDS.64.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o tests/micro/lat tests/micro/lat.cu
#include <cstdio>
#include <cstdint>
__global__ void k(double* out, long long* cyc, double x0, int n) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += 32) sm[i] = (double)((i * 7) & 1023);
    __syncwarp();
    double a = x0, v = 1e300;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) a = __dadd_rn(a, 1.0);            // dependent DADD
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) { double b = a + i; v = b < v ? b : v; a = v + 0.5; }  // DSETP/FSEL + DADD
    long long t2 = clock64();
    long long ka = __double_as_longlong(a), kv = 0x7fefffffffffffffll;
    for (int i = 0; i < n; ++i) { long long b = ka + i; kv = b < kv ? b : kv; ka = kv ^ 1; }  // int64 compare/select
    long long t3 = clock64();
    int idx = (int)a & 1023;
    for (int i = 0; i < n; ++i) idx = ((int)sm[idx] + 1) & 1023;  // LDS.64 chain (+cvt)
    long long t4 = clock64();
    out[threadIdx.x] = a + v + (double)kv + idx;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
    const int n = 4096;
    k<<<1, 32>>>(o, c, 1.0, n); cudaDeviceSynchronize();
    k<<<1, 32>>>(o, c, 1.0, n); long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("cycles/iter: DADD chain %.1f | DADD+DSETP/FSEL-min chain %.1f | int64 add+cmp/sel chain %.1f | LDS.64+CVT chain %.1f\n",
           h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n);
}
