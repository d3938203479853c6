// Shared device helpers for the sm_100a scheduling kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/swarmsched_b200.h"

#define SS_MAX_HOSTS 256
#define SS_MAX_LAYERS 1024
#define SS_MAX_GPUS 4096

#define SS_CHECK_LAUNCH()                                   \
    do {                                                    \
        cudaError_t _e = cudaGetLastError();                \
        if (_e != cudaSuccess) return SS_CUDA_ERROR;        \
    } while (0)

static inline cudaStream_t ss_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

__host__ __device__ __forceinline__ uint64_t ss_splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

// Pair jitter of scenarios.py:jitter_factor -- one LogNormal(0, 0.2) factor per unordered GPU pair (SURVEY.md
// 8(d) C4), drawn by inverse-CDF sampling on the 1024 float32 quantiles of jitter_lognormal.inc (the file
// scenarios.py parses too, so host and device scenario matrices are the same IEEE products rtt * (double)Q[i]).
// Global memory, not __constant__: the lanes of a warp index different entries.
static __device__ const float ss_jitter_q[1024] = {
#include "jitter_lognormal.inc"
};

// quantile index of the unordered pair (i, j) under seed_mix = splitmix64(scenario seed): the pair folded into 32 bits
// with two odd multipliers and the seed, then the lowbias32 finaliser (xorshift-multiply); top 10 bits.  Cheap
// enough to run per entry in the region replay's kept cross-region blocks.
__device__ __forceinline__ uint32_t ss_jitter_index(uint64_t seed_mix, uint32_t i, uint32_t j) {
    if (i > j) { uint32_t t = i; i = j; j = t; }
    uint32_t x = i * 0x9E3779B1u + j * 0x85EBCA77u + ((uint32_t)seed_mix ^ (uint32_t)(seed_mix >> 32));
    x ^= x >> 16;
    x *= 0x7FEB352Du;
    x ^= x >> 15;
    x *= 0x846CA68Bu;
    x ^= x >> 16;
    return x >> 22;
}

__device__ __forceinline__ double ss_jitter(uint64_t seed_mix, uint32_t i, uint32_t j) {
    return (double)__ldg(&ss_jitter_q[ss_jitter_index(seed_mix, i, j)]);
}

// ---------------------------------------------------------------------------
// mbarrier + bulk async copy (TMA 1-D, SASS UBLKCP) helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// producer-side wait: back off so a spinning lane does not steal issue slots from the consumers
// Producer-side wait with exponential backoff (128 ns .. max_ns): a ring refill is due about once per
// boundary, so a polling producer would only steal issue slots from the consumer warps of its SM sub-partition
// (a fixed 64 ns sleep measured 25% of the slot kernel's instructions in this loop).
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity, unsigned max_ns = 1024) {
    unsigned ns = 128;
    while (!mbar_try_wait(bar, parity)) {
        __nanosleep(ns);
        ns = ns < max_ns ? 2 * ns : max_ns;
    }
}

// ---------------------------------------------------------------------------
// CPython 3.12 sum() over int / float items, start = 0
// ---------------------------------------------------------------------------
struct PySum {   // SURVEY.md hazard H2; modelled by oracle/waterfill_ref.py:cpython_sum_model
    bool is_int;
    long long iacc;
    double f, c;
    __device__ void init() { is_int = true; iacc = 0; f = 0.0; c = 0.0; }
    __device__ void add_int(long long v) {
        if (is_int) iacc += v;
        else f = __dadd_rn(f, (double)v);
    }
    __device__ void add_float(double x) {
        if (is_int) {           // int accumulator meets its first float: plain add, compensation starts
            f = __dadd_rn((double)iacc, x);
            c = 0.0;
            is_int = false;
            return;
        }
        const double t = __dadd_rn(f, x);
        if (fabs(f) >= fabs(x)) c = __dadd_rn(c, __dadd_rn(__dsub_rn(f, t), x));
        else c = __dadd_rn(c, __dadd_rn(__dsub_rn(x, t), f));
        f = t;
    }
    __device__ double value() const {
        if (is_int) return (double)iacc;
        double r = f;
        if (c != 0.0 && isfinite(c)) r = __dadd_rn(r, c);
        return r;
    }
};


