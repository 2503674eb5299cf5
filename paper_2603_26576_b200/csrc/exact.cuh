// exact.cuh -- exact arithmetic shared by the analysis (engine.cu) and the
// region kernels (regions.cu): Python's correctly rounded int / int for u128
// operands and the two metric trees (metrics.py:66-122).
#pragma once
#include <cstdint>

#include "engine.cuh"
#include "ptx.cuh"

// The engine's namespace: `hb`, or another name for a second compilation of the
// analysis kernel with a different tile geometry (engine_cols.cu).
#ifndef HB_ENGINE_NS
#define HB_ENGINE_NS hb
#endif
namespace HB_ENGINE_NS {

// =========================================================================
// exact u128 / u128 -> nearest double, ties to even (Python int / int)
// =========================================================================
static __device__ __forceinline__ int bitlen128(u128 x)
{
    const u64 hi = (u64)(x >> 64), lo = (u64)x;
    return hi ? 128 - __clzll((long long)hi) : (lo ? 64 - __clzll((long long)lo) : 0);
}

static __device__ __noinline__ double div_exact(u128 a, u128 b)
{
    if (a == 0) return 0.0;
    if ((a >> 53) == 0 && (b >> 53) == 0) return (double)(u64)a / (double)(u64)b;  // IEEE: correctly rounded
    const int la = bitlen128(a), lb = bitlen128(b);
    u128 r = a, M = 0;
    int e2 = 0;
    for (int i = la - lb; i >= 0; --i) {              // integer quotient bits
        const u128 d = b << i;
        M <<= 1;
        if (r >= d) { r -= d; M |= 1; }
    }
    while (bitlen128(M) < 55) {                        // fractional bits
        r <<= 1;
        M <<= 1;
        if (r >= b) { r -= b; M |= 1; }
        --e2;
    }
    bool sticky = r != 0;
    const int lm = bitlen128(M);
    if (lm > 55) {
        const int sh = lm - 55;
        if (M & ((((u128)1) << sh) - 1)) sticky = true;
        M >>= sh;
        e2 += sh;
    }
    const unsigned low2 = (unsigned)(M & 3);
    u64 mant = (u64)(M >> 2);
    e2 += 2;
    const bool guard = (low2 >> 1) & 1, rest = (low2 & 1) || sticky;
    if (guard && (rest || (mant & 1))) ++mant;
    if (mant == (1ull << 53)) { mant >>= 1; ++e2; }
    return ldexp((double)mant, e2);
}

// block reductions of u128 for the finalize: warp shuffles, then warp 0
static __device__ __forceinline__ u128 shfl_xor128(u128 v, int d)
{
    const u64 lo = __shfl_xor_sync(0xffffffffu, (u64)v, d), hi = __shfl_xor_sync(0xffffffffu, (u64)(v >> 64), d);
    return ((u128)hi << 64) | lo;
}

template <bool MAX>
__device__ u128 block_reduce128(u128 v, u128 *scratch, int tid, int nt)
{
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const u128 o = shfl_xor128(v, d);
        v = MAX ? (o > v ? o : v) : v + o;
    }
    const int w = tid >> 5, nw = nt >> 5;
    if ((tid & 31) == 0) scratch[w] = v;
    __syncthreads();
    if (w == 0) {
        v = (tid < nw) ? scratch[tid] : (u128)0;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const u128 o = shfl_xor128(v, d);
            v = MAX ? (o > v ? o : v) : v + o;
        }
        if (tid == 0) scratch[32] = v;
    }
    __syncthreads();
    const u128 t = scratch[32];
    __syncthreads();
    return t;
}

// metric trees (metrics.py:66-122); threads 0..4 / 32..35 each do one division
template <typename Out>
__device__ void metric_trees(Out *res, bool host_side, bool dev_side, u64 E, int32_t n, int32_t m,
                             u128 sum_u, u128 sum_uw, u128 max_uw, u128 sum_k, u128 max_k, u128 max_km, int tid)
{
    if (host_side && tid < 5) {
        if (sum_uw == 0) {
            if (tid == 0) { res->host_metrics[0] = 0.0; res->host_mask = 1u; }
        } else {
            const u128 En = (u128)E * (u128)(uint32_t)n;
            double v = 0.0;
            switch (tid) {
            case 0: v = div_exact(sum_u, En); break;
            case 1: v = div_exact(sum_uw, En); break;
            case 2: v = div_exact(max_uw, (u128)E); break;
            case 3: v = div_exact(sum_uw, (u128)(uint32_t)n * max_uw); break;
            default: v = div_exact(sum_u, sum_uw); break;
            }
            res->host_metrics[tid] = v;
            if (tid == 0) res->host_mask = 0x1fu;
        }
    }
    if (dev_side && tid >= 32 && tid < 36) {
        const int i = tid - 32;
        const u128 Em = (u128)E * (u128)(uint32_t)m;
        if (max_k == 0) {
            if (i == 0) res->device_metrics[0] = div_exact(sum_k, Em);
            if (i == 3) res->device_metrics[3] = max_km > 0 ? div_exact(max_km, (u128)E) : 0.0;
            if (i == 0) res->device_mask = 0x9u;
        } else {
            double v = 0.0;
            switch (i) {
            case 0: v = div_exact(sum_k, Em); break;
            case 1: v = div_exact(sum_k, (u128)(uint32_t)m * max_k); break;
            case 2: v = div_exact(max_k, max_km); break;
            default: v = div_exact(max_km, (u128)E); break;
            }
            res->device_metrics[i] = v;
            if (i == 0) res->device_mask = 0xfu;
        }
    }
}

}  // namespace HB_ENGINE_NS
