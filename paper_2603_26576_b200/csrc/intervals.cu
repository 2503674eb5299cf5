// intervals.cu -- the reference's interval algebra (intervals.py:40-105) on the
// GPU, as stand-alone operations over device arrays of [start, end) pairs:
//
//   flatten     validate (first malformed index), drop zero-length, sort by
//               start (K3 radix sort), merge overlapping AND adjacent
//               intervals: a record opens a new run iff start > running max
//               of earlier ends (strict: `start <= last.end` merges,
//               intervals.py:55-60); run ends are the running max at the
//               next run start.  Device-wide scans in three kernels.
//   subtract    a - b of two flat sets.  Every output piece starts either at
//               some a.start not covered by b, or at some b.end inside some
//               a; one thread per a interval and per b interval decides (two
//               binary searches each), and output positions come from prefix
//               counts of both kinds (a merge by rank) -- O((|a|+|b|) log),
//               balanced however the two sets interleave.
//   intersect   clip to [lo, hi) and compact (intervals.py:98-105).
//   total       exact sum of durations as u128 (intervals.py:93-95).
//
// complement(a, bounds) is subtract([bounds], a), exactly as the reference
// defines it (intervals.py:84-90); the Python layer composes it.
#include <cuda_runtime.h>
#include <climits>
#include <cstdint>

#include "engine.cuh"
#include "ptx.cuh"

namespace hb {
namespace iv {

constexpr int kT = 256, kI = 4, kB = kT * kI;   // 1024 elements per block

__host__ __device__ __forceinline__ int64_t nblocks(int64_t n) { return (n + kB - 1) / kB; }

// block-wide exclusive scan of one u32 per thread (sum); returns the block total via `tot`
__device__ __forceinline__ uint32_t block_excl_sum(uint32_t x, uint32_t *ws, uint32_t &tot)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
    }
    if (lane == 31) ws[warp] = inc;
    __syncthreads();
    if (tid == 0) {
        uint32_t run = 0;
        for (int w = 0; w < kT / 32; ++w) { const uint32_t v = ws[w]; ws[w] = run; run += v; }
        ws[kT / 32] = run;
    }
    __syncthreads();
    const uint32_t r = ws[warp] + inc - x;
    tot = ws[kT / 32];
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------------------
// flatten
// ---------------------------------------------------------------------------
__global__ void fl_malformed(const u64 *__restrict__ s, const u64 *__restrict__ e, int64_t n,
                             unsigned long long *first_bad)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (s[i] > e[i]) atomicMin(first_bad, (unsigned long long)i);
}

// per block (of sorted records): max end over positive-length records + presence flag
__global__ void __launch_bounds__(kT) fl_blockmax(const u64 *__restrict__ s, const u64 *__restrict__ e, int64_t n,
                                                  u64 *__restrict__ bmax, uint32_t *__restrict__ bany)
{
    const int64_t b0 = (int64_t)blockIdx.x * kB;
    u64 mx = 0;
    bool any = false;
    for (int q = 0; q < kI; ++q) {
        const int64_t i = b0 + q * kT + threadIdx.x;
        if (i < n && e[i] > s[i]) { mx = umax(mx, e[i]); any = true; }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) mx = umax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
    any = __syncthreads_or(any);
    __shared__ u64 wm[kT / 32];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < kT / 32; ++w) mx = umax(mx, wm[w]);
        bmax[blockIdx.x] = mx;
        bany[blockIdx.x] = any ? 1u : 0u;
    }
}

// one block: exclusive max-carry over blocks (in place: bmax -> carry, bany -> "some earlier block had one")
__global__ void __launch_bounds__(1024) fl_carry(u64 *bmax, uint32_t *bany, int64_t nb, u64 *gmax, uint32_t *gany)
{
    if (threadIdx.x != 0) return;
    u64 run = 0;
    uint32_t have = 0;
    for (int64_t b = 0; b < nb; ++b) {
        const u64 m = bmax[b];
        const uint32_t a = bany[b];
        bmax[b] = run;
        bany[b] = have;
        if (a) { run = umax(run, m); have = 1; }
    }
    *gmax = run;
    *gany = have;
}

// run-start flags of one block, from the block carry and an in-block exclusive max scan
__device__ __forceinline__ void fl_block_flags(const u64 *s, const u64 *e, int64_t n, u64 carry, bool have,
                                               bool (&flag)[kI], u64 (&R)[kI], u64 *wmax, uint32_t *whave)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t b0 = (int64_t)blockIdx.x * kB + (int64_t)tid * kI;   // blocked: kI consecutive per thread
    u64 v[kI];
    bool pos[kI];
    u64 tm = 0;
    bool th = false;
#pragma unroll
    for (int q = 0; q < kI; ++q) {
        const int64_t i = b0 + q;
        pos[q] = i < n && e[i] > s[i];
        v[q] = pos[q] ? e[i] : 0;
        if (pos[q]) { tm = umax(tm, v[q]); th = true; }
    }
    // exclusive (max, have) over threads
    u64 im = tm;
    bool ih = th;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const u64 om = __shfl_up_sync(0xffffffffu, im, d);
        const bool oh = __shfl_up_sync(0xffffffffu, ih, d);
        if (lane >= d) { im = umax(im, om); ih = ih || oh; }
    }
    if (lane == 31) { wmax[warp] = im; whave[warp] = ih; }
    __syncthreads();
    u64 em = __shfl_up_sync(0xffffffffu, im, 1);
    bool eh = __shfl_up_sync(0xffffffffu, ih, 1);
    if (lane == 0) { em = 0; eh = false; }
    for (int w = 0; w < warp; ++w) { em = umax(em, wmax[w]); eh = eh || whave[w]; }
    if (have) { em = umax(em, carry); eh = true; }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kI; ++q) {
        const int64_t i = b0 + q;
        flag[q] = pos[q] && (!eh || s[i] > em);
        R[q] = em;
        if (pos[q]) { em = umax(em, v[q]); eh = true; }
    }
}

__global__ void __launch_bounds__(kT) fl_count(const u64 *__restrict__ s, const u64 *__restrict__ e, int64_t n,
                                               const u64 *__restrict__ carry, const uint32_t *__restrict__ have,
                                               uint32_t *__restrict__ bcount)
{
    __shared__ u64 wmax[kT / 32];
    __shared__ uint32_t whave[kT / 32], ws[kT / 32 + 1];
    bool flag[kI];
    u64 R[kI];
    fl_block_flags(s, e, n, carry[blockIdx.x], have[blockIdx.x] != 0, flag, R, wmax, whave);
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < kI; ++q) c += flag[q];
    uint32_t tot;
    block_excl_sum(c, ws, tot);
    if (threadIdx.x == 0) bcount[blockIdx.x] = tot;
}

// exclusive scan of per-block u32 counts into int64 offsets (one block)
__global__ void __launch_bounds__(1024) scan_counts(const uint32_t *__restrict__ c, int64_t nb,
                                                    int64_t *__restrict__ off, int64_t *total)
{
    if (threadIdx.x != 0) return;
    int64_t run = 0;
    for (int64_t b = 0; b < nb; ++b) { off[b] = run; run += c[b]; }
    *total = run;
}

__global__ void __launch_bounds__(kT) fl_write(const u64 *__restrict__ s, const u64 *__restrict__ e, int64_t n,
                                               const u64 *__restrict__ carry, const uint32_t *__restrict__ have,
                                               const int64_t *__restrict__ boff, const u64 *gmax,
                                               const int64_t *total, u64 *__restrict__ os, u64 *__restrict__ oe)
{
    __shared__ u64 wmax[kT / 32];
    __shared__ uint32_t whave[kT / 32], ws[kT / 32 + 1];
    bool flag[kI];
    u64 R[kI];
    fl_block_flags(s, e, n, carry[blockIdx.x], have[blockIdx.x] != 0, flag, R, wmax, whave);
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < kI; ++q) c += flag[q];
    uint32_t tot;
    int64_t k = boff[blockIdx.x] + block_excl_sum(c, ws, tot);
    const int64_t b0 = (int64_t)blockIdx.x * kB + (int64_t)threadIdx.x * kI;
#pragma unroll
    for (int q = 0; q < kI; ++q) {
        if (flag[q]) {
            os[k] = s[b0 + q];
            if (k > 0) oe[k - 1] = R[q];   // the previous run ends at the running max before this start
            ++k;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && *total > 0) oe[*total - 1] = *gmax;
}

// ---------------------------------------------------------------------------
// subtract(a, b) for flat sets (sorted, disjoint, non-adjacent, no empties)
// ---------------------------------------------------------------------------
// first index in [0, n) with v[i] > x (v non-decreasing)
__device__ __forceinline__ int64_t upper(const u64 *v, int64_t n, u64 x)
{
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (v[mid] <= x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// first index in [0, n) with v[i] >= x
__device__ __forceinline__ int64_t lower(const u64 *v, int64_t n, u64 x)
{
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (v[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// does a.start open a piece (not covered by b)?  does b.end open one (inside some a)?
__device__ __forceinline__ bool a_opens(const u64 *bs, const u64 *be, int64_t nb, u64 x)
{
    const int64_t k = upper(bs, nb, x) - 1;   // last b with start <= x
    return k < 0 || be[k] <= x;
}

__device__ __forceinline__ bool b_opens(const u64 *as, const u64 *ae, int64_t na, u64 y)
{
    const int64_t i = upper(as, na, y) - 1;   // last a with start <= y
    return i >= 0 && ae[i] > y && as[i] < y;  // strictly inside: at a.start the a thread emits the piece
}

__global__ void sub_flags(const u64 *__restrict__ as, const u64 *__restrict__ ae, int64_t na,
                          const u64 *__restrict__ bs, const u64 *__restrict__ be, int64_t nb,
                          uint32_t *__restrict__ fa, uint32_t *__restrict__ fb)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < na + nb;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i < na) fa[i] = a_opens(bs, be, nb, as[i]) ? 1u : 0u;
        else fb[i - na] = b_opens(as, ae, na, be[i - na]) ? 1u : 0u;
    }
}

// multi-block exclusive prefix of u32 flags into int64 positions (out[n] = total):
// per-block sums, a scan of the block sums (scan_counts), per-block apply
__global__ void __launch_bounds__(kT) flag_sums(const uint32_t *__restrict__ f, int64_t n, uint32_t *__restrict__ bsum)
{
    __shared__ uint32_t ws[kT / 32 + 1];
    const int64_t b0 = (int64_t)blockIdx.x * kB + (int64_t)threadIdx.x * kI;
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < kI; ++q) c += b0 + q < n ? f[b0 + q] : 0u;
    uint32_t tot;
    block_excl_sum(c, ws, tot);
    if (threadIdx.x == 0) bsum[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kT) flag_apply(const uint32_t *__restrict__ f, int64_t n,
                                                 const int64_t *__restrict__ boff, const int64_t *total,
                                                 int64_t *__restrict__ out)
{
    __shared__ uint32_t ws[kT / 32 + 1];
    const int64_t b0 = (int64_t)blockIdx.x * kB + (int64_t)threadIdx.x * kI;
    uint32_t v[kI], c = 0;
#pragma unroll
    for (int q = 0; q < kI; ++q) { v[q] = b0 + q < n ? f[b0 + q] : 0u; c += v[q]; }
    uint32_t tot;
    int64_t run = boff[blockIdx.x] + block_excl_sum(c, ws, tot);
#pragma unroll
    for (int q = 0; q < kI; ++q) {
        if (b0 + q < n) out[b0 + q] = run;
        run += v[q];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = *total;
}

__global__ void sub_write(const u64 *__restrict__ as, const u64 *__restrict__ ae, int64_t na,
                          const u64 *__restrict__ bs, const u64 *__restrict__ be, int64_t nb,
                          const uint32_t *__restrict__ fa, const uint32_t *__restrict__ fb,
                          const int64_t *__restrict__ pa, const int64_t *__restrict__ pb,
                          u64 *__restrict__ os, u64 *__restrict__ oe)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < na + nb;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i < na) {
            if (!fa[i]) continue;
            const u64 x = as[i];
            // pieces starting before x: a-pieces of earlier a's + b-pieces with b.end < x
            const int64_t kb = lower(be, nb, x);                 // b with end < x
            const int64_t pos = pa[i] + pb[kb];
            const int64_t nx = lower(bs, nb, x);                 // next b starting at or after x
            const u64 stop = nx < nb ? umin(ae[i], bs[nx]) : ae[i];
            os[pos] = x;
            oe[pos] = stop;
        } else {
            const int64_t k = i - na;
            if (!fb[k]) continue;
            const u64 y = be[k];
            const int64_t ia = upper(as, na, y) - 1;             // the a containing y
            const int64_t ka = lower(as, na, y);                 // a with start < y
            const int64_t pos = pb[k] + pa[ka];
            const u64 stop = k + 1 < nb ? umin(ae[ia], bs[k + 1]) : ae[ia];
            os[pos] = y;
            oe[pos] = stop;
        }
    }
}

// ---------------------------------------------------------------------------
// intersect with [lo, hi) + compaction; total duration (u128)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kT) ix_count(const u64 *__restrict__ s, const u64 *__restrict__ e, int64_t n, u64 lo,
                                               u64 hi, uint32_t *__restrict__ bcount)
{
    __shared__ uint32_t ws[kT / 32 + 1];
    const int64_t b0 = (int64_t)blockIdx.x * kB + (int64_t)threadIdx.x * kI;
    uint32_t c = 0;
    for (int q = 0; q < kI; ++q) {
        const int64_t i = b0 + q;
        if (i < n && umax(s[i], lo) < umin(e[i], hi)) ++c;
    }
    uint32_t tot;
    block_excl_sum(c, ws, tot);
    if (threadIdx.x == 0) bcount[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kT) ix_write(const u64 *__restrict__ s, const u64 *__restrict__ e, int64_t n, u64 lo,
                                               u64 hi, const int64_t *__restrict__ boff, u64 *__restrict__ os,
                                               u64 *__restrict__ oe)
{
    __shared__ uint32_t ws[kT / 32 + 1];
    const int64_t b0 = (int64_t)blockIdx.x * kB + (int64_t)threadIdx.x * kI;
    uint32_t c = 0;
    for (int q = 0; q < kI; ++q) {
        const int64_t i = b0 + q;
        if (i < n && umax(s[i], lo) < umin(e[i], hi)) ++c;
    }
    uint32_t tot;
    int64_t k = boff[blockIdx.x] + block_excl_sum(c, ws, tot);
    for (int q = 0; q < kI; ++q) {
        const int64_t i = b0 + q;
        if (i < n) {
            const u64 cs = umax(s[i], lo), ce = umin(e[i], hi);
            if (cs < ce) { os[k] = cs; oe[k] = ce; ++k; }
        }
    }
}

__global__ void __launch_bounds__(256) total_kernel(const u64 *__restrict__ s, const u64 *__restrict__ e, int64_t n,
                                                    u64 *out /* [2]: lo, hi words of the u128 sum */)
{
    u128 t = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        t += (u128)(e[i] - s[i]);
    u64 lo = (u64)t, hi = (u64)(t >> 64);
    // (lo, hi) add with carry: reduce lo in 2 x 32-bit limbs to keep it exact
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const u64 olo = __shfl_xor_sync(0xffffffffu, lo, d), ohi = __shfl_xor_sync(0xffffffffu, hi, d);
        const u64 nlo = lo + olo;
        hi += ohi + (nlo < lo ? 1 : 0);
        lo = nlo;
    }
    if ((threadIdx.x & 31) == 0) {
        // 128-bit atomic add via two 64-bit atomics with carry
        const u64 old = atomicAdd(out, lo);
        const u64 carry = (old + lo < old) ? 1ull : 0ull;
        if (hi + carry) atomicAdd(out + 1, hi + carry);
    }
}

}  // namespace iv

// ---------------------------------------------------------------------------
// host orchestration (workspace from the caller)
// ---------------------------------------------------------------------------
static size_t up256(size_t x) { return (x + 255) & ~(size_t)255; }

size_t iv_flatten_ws(int64_t n)
{
    const int64_t nb = iv::nblocks(n) + 1;
    return up256((size_t)nb * 8) * 2 + up256((size_t)nb * 4) * 2 + 256 + sort_workspace_bytes(n) +
           2 * up256((size_t)n * 8) + up256((size_t)n * 4) + up256((size_t)n);
}

static int grid_of(int64_t n, int bs)
{
    int64_t g = (n + bs - 1) / bs;
    if (g > 148 * 16) g = 148 * 16;
    return g < 1 ? 1 : (int)g;
}

// flatten: returns cudaErrorInvalidValue with *bad = first malformed index when one exists
cudaError_t iv_flatten(const u64 *s, const u64 *e, int64_t n, u64 *os, u64 *oe, int64_t *out_n, int64_t *bad,
                       void *ws, size_t ws_bytes, cudaStream_t st)
{
    *out_n = 0;
    *bad = -1;
    if (n <= 0) return cudaSuccess;
    if (ws_bytes < iv_flatten_ws(n)) return cudaErrorInvalidValue;
    const int64_t nb = iv::nblocks(n);
    uint8_t *w = static_cast<uint8_t *>(ws);
    size_t o = 0;
    auto take = [&](size_t b) { void *p = w + o; o += up256(b); return p; };
    u64 *bmax = static_cast<u64 *>(take((size_t)(nb + 1) * 8));
    int64_t *boff = static_cast<int64_t *>(take((size_t)(nb + 1) * 8));
    uint32_t *bany = static_cast<uint32_t *>(take((size_t)(nb + 1) * 4));
    uint32_t *bcnt = static_cast<uint32_t *>(take((size_t)(nb + 1) * 4));
    u64 *misc = static_cast<u64 *>(take(64));   // [0] first bad, [1] gmax, [2] gany, [3] total
    void *sws = take(sort_workspace_bytes(n));
    u64 *ss = static_cast<u64 *>(take((size_t)n * 8));
    u64 *se = static_cast<u64 *>(take((size_t)n * 8));
    int32_t *zr = static_cast<int32_t *>(take((size_t)n * 4));
    uint8_t *zk = static_cast<uint8_t *>(take((size_t)n));
    cudaError_t err;
    if ((err = cudaMemsetAsync(misc, 0xff, 8, st)) != cudaSuccess) return err;
    iv::fl_malformed<<<grid_of(n, 256), 256, 0, st>>>(s, e, n, reinterpret_cast<unsigned long long *>(misc));
    unsigned long long first = 0;
    if ((err = cudaMemcpyAsync(&first, misc, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return err;
    if ((err = cudaStreamSynchronize(st)) != cudaSuccess) return err;
    if (first != ~0ull) { *bad = (int64_t)first; return cudaErrorInvalidValue; }
    // sort by start (records of one "resource")
    if ((err = cudaMemsetAsync(zr, 0, (size_t)n * 4, st)) != cudaSuccess) return err;
    if ((err = cudaMemsetAsync(zk, 0, (size_t)n, st)) != cudaSuccess) return err;
    if ((err = sort_records(s, e, zr, zk, n, ss, se, zr, zk, nullptr, sws, sort_workspace_bytes(n), st, nullptr)) !=
        cudaSuccess)
        return err;
    iv::fl_blockmax<<<(unsigned)nb, iv::kT, 0, st>>>(ss, se, n, bmax, bany);
    iv::fl_carry<<<1, 1024, 0, st>>>(bmax, bany, nb, misc + 1, reinterpret_cast<uint32_t *>(misc + 2));
    iv::fl_count<<<(unsigned)nb, iv::kT, 0, st>>>(ss, se, n, bmax, bany, bcnt);
    iv::scan_counts<<<1, 1024, 0, st>>>(bcnt, nb, boff, reinterpret_cast<int64_t *>(misc + 3));
    iv::fl_write<<<(unsigned)nb, iv::kT, 0, st>>>(ss, se, n, bmax, bany, boff, misc + 1,
                                                  reinterpret_cast<int64_t *>(misc + 3), os, oe);
    if ((err = cudaMemcpyAsync(out_n, misc + 3, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return err;
    return cudaStreamSynchronize(st);
}

size_t iv_subtract_ws(int64_t na, int64_t nb)
{
    const int64_t ba = iv::nblocks(na) + 1, bb = iv::nblocks(nb) + 1;
    return up256((size_t)(na + 1) * 4) + up256((size_t)(nb + 1) * 4) + up256((size_t)(na + 1) * 8) +
           up256((size_t)(nb + 1) * 8) + 2 * up256((size_t)(ba + bb) * 12) + 256;
}

// exclusive positions of n flags (out[n] = total) with the multi-block scan
static void flag_prefix(const uint32_t *f, int64_t n, int64_t *out, uint32_t *bsum, int64_t *boff, int64_t *total,
                        cudaStream_t st)
{
    const int64_t nb = iv::nblocks(n > 0 ? n : 1);
    iv::flag_sums<<<(unsigned)nb, iv::kT, 0, st>>>(f, n, bsum);
    iv::scan_counts<<<1, 1024, 0, st>>>(bsum, nb, boff, total);
    iv::flag_apply<<<(unsigned)nb, iv::kT, 0, st>>>(f, n, boff, total, out);
}

cudaError_t iv_subtract(const u64 *as, const u64 *ae, int64_t na, const u64 *bs, const u64 *be, int64_t nb, u64 *os,
                        u64 *oe, int64_t *out_n, void *ws, size_t ws_bytes, cudaStream_t st)
{
    *out_n = 0;
    if (na <= 0) return cudaSuccess;
    if (ws_bytes < iv_subtract_ws(na, nb)) return cudaErrorInvalidValue;
    uint8_t *w = static_cast<uint8_t *>(ws);
    size_t o = 0;
    auto take = [&](size_t b) { void *p = w + o; o += up256(b); return p; };
    uint32_t *fa = static_cast<uint32_t *>(take((size_t)(na + 1) * 4));
    uint32_t *fb = static_cast<uint32_t *>(take((size_t)(nb + 1) * 4));
    int64_t *pa = static_cast<int64_t *>(take((size_t)(na + 1) * 8));
    int64_t *pb = static_cast<int64_t *>(take((size_t)(nb + 1) * 8));
    iv::sub_flags<<<grid_of(na + nb, 256), 256, 0, st>>>(as, ae, na, bs, be, nb, fa, fb);
    const int64_t ba = iv::nblocks(na) + 1, bb = iv::nblocks(nb) + 1;
    uint32_t *bsa = static_cast<uint32_t *>(take((size_t)ba * 4));
    int64_t *boa = static_cast<int64_t *>(take((size_t)ba * 8));
    uint32_t *bsb = static_cast<uint32_t *>(take((size_t)bb * 4));
    int64_t *bob = static_cast<int64_t *>(take((size_t)bb * 8));
    int64_t *tots = static_cast<int64_t *>(take(16));
    flag_prefix(fa, na, pa, bsa, boa, tots, st);
    flag_prefix(fb, nb, pb, bsb, bob, tots + 1, st);
    iv::sub_write<<<grid_of(na + nb, 256), 256, 0, st>>>(as, ae, na, bs, be, nb, fa, fb, pa, pb, os, oe);
    int64_t ca = 0, cb = 0;
    cudaError_t err;
    if ((err = cudaMemcpyAsync(&ca, pa + na, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return err;
    if (nb > 0 && (err = cudaMemcpyAsync(&cb, pb + nb, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return err;
    if ((err = cudaStreamSynchronize(st)) != cudaSuccess) return err;
    *out_n = ca + cb;
    return cudaSuccess;
}

size_t iv_intersect_ws(int64_t n) { return up256((size_t)(iv::nblocks(n) + 1) * 12) + 256; }

cudaError_t iv_intersect(const u64 *s, const u64 *e, int64_t n, u64 lo, u64 hi, u64 *os, u64 *oe, int64_t *out_n,
                         void *ws, size_t ws_bytes, cudaStream_t st)
{
    *out_n = 0;
    if (n <= 0) return cudaSuccess;
    if (ws_bytes < iv_intersect_ws(n)) return cudaErrorInvalidValue;
    const int64_t nb = iv::nblocks(n);
    uint8_t *w = static_cast<uint8_t *>(ws);
    uint32_t *bcnt = reinterpret_cast<uint32_t *>(w);
    int64_t *boff = reinterpret_cast<int64_t *>(w + up256((size_t)(nb + 1) * 4));
    int64_t *tot = boff + nb + 1;
    iv::ix_count<<<(unsigned)nb, iv::kT, 0, st>>>(s, e, n, lo, hi, bcnt);
    iv::scan_counts<<<1, 1024, 0, st>>>(bcnt, nb, boff, tot);
    iv::ix_write<<<(unsigned)nb, iv::kT, 0, st>>>(s, e, n, lo, hi, boff, os, oe);
    cudaError_t err;
    if ((err = cudaMemcpyAsync(out_n, tot, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return err;
    return cudaStreamSynchronize(st);
}

cudaError_t iv_total(const u64 *s, const u64 *e, int64_t n, u64 *out2_dev, cudaStream_t st)
{
    cudaError_t err;
    if ((err = cudaMemsetAsync(out2_dev, 0, 16, st)) != cudaSuccess) return err;
    if (n > 0) iv::total_kernel<<<grid_of(n, 256), 256, 0, st>>>(s, e, n, out2_dev);
    return cudaGetLastError();
}

}  // namespace hb
