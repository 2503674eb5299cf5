// gen.cu -- K0: deterministic config-shaped synthetic traces written directly
// into HBM.  Counter-based RNG keyed by (seed, global resource id, record
// index), so any rank shard regenerates identically on any GPU count, and
// oracle/gen.py (numpy) reproduces every array bit for bit.
//
// Per resource: record j draws gap ~ U[0, gap_max], dur ~ U[1, dur_max]
// (x dur_scale0 for global resource 0) and a state / kind.  Starts are a
// prefix sum: serialized chains (host ranks, serialized streams)
//   start_j = sum_{i<j}(gap_i + dur_i) + gap_j
// or an arrival process (overlapping device streams)
//   start_j = sum_{i<=j} gap_i.
// One CTA per resource scans its records in 1024-record chunks.
#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/heteff_b200.h"

namespace hb {

typedef unsigned long long u64;

__device__ __forceinline__ u64 mix64(u64 z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ u64 uni(u64 x32, u64 n) { return (x32 * n) >> 32; }

constexpr int kGenThreads = 1024;

__global__ void __launch_bounds__(kGenThreads) gen_kernel(heteff_gen_side g, u64 *S, u64 *E, int32_t *R,
                                                          uint8_t *K)
{
    __shared__ u64 warp_tot[kGenThreads / 32];
    const int local = blockIdx.x;
    const long long gid = (long long)g.res_base + local;
    const long long extra = g.extra_below;
    const long long count = g.per_res + (gid < extra ? 1 : 0);
    const long long lo_x = g.res_base < extra ? g.res_base : extra;
    const long long hi_x = gid < extra ? gid : extra;
    const long long offset = (long long)local * g.per_res + (hi_x > lo_x ? hi_x - lo_x : 0);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const u64 scale = (gid == 0 && g.dur_scale0 > 1) ? g.dur_scale0 : 1;
    u64 carry = 0;
    for (long long c0 = 0; c0 < count; c0 += kGenThreads) {
        const long long j = c0 + tid;
        const bool valid = j < count;
        const u64 u1 = mix64(g.seed ^ ((u64)gid << 40) ^ (u64)j);
        const u64 u2 = mix64(u1 ^ 0xD1B54A32D192ED03ull);
        const u64 gap = uni(u1 & 0xffffffffull, (u64)g.gap_max + 1);
        const u64 dur = (1 + uni(u1 >> 32, g.dur_max)) * scale;
        const u64 inc = valid ? (g.serialized ? gap + dur : gap) : 0;
        // block inclusive scan of inc
        u64 v = inc;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u64 o = __shfl_up_sync(0xffffffffu, v, d);
            if (lane >= d) v += o;
        }
        if (lane == 31) warp_tot[warp] = v;
        __syncthreads();
        if (warp == 0) {
            u64 w = warp_tot[lane];
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const u64 o = __shfl_up_sync(0xffffffffu, w, d);
                if (lane >= d) w += o;
            }
            warp_tot[lane] = w;
        }
        __syncthreads();
        const u64 incl = v + (warp > 0 ? warp_tot[warp - 1] : 0) + carry;
        const u64 total = warp_tot[31];
        if (valid) {
            const u64 start = g.serialized ? incl - dur : incl;
            const long long o = offset + j;
            S[o] = start;
            E[o] = start + dur;
            R[o] = local;
            K[o] = g.is_host ? (uint8_t)uni(u2 & 0xffffffffull, 3)
                             : (uint8_t)(uni(u2 & 0xffffffffull, 100) < g.kernel_pct ? 0 : 1);
        }
        carry += total;
        __syncthreads();
    }
}

cudaError_t launch_generate(const heteff_gen_side &g, u64 *S, u64 *E, int32_t *R, uint8_t *K, cudaStream_t s)
{
    if (g.n_res <= 0) return cudaSuccess;
    gen_kernel<<<g.n_res, kGenThreads, 0, s>>>(g, S, E, R, K);
    return cudaGetLastError();
}

}  // namespace hb
