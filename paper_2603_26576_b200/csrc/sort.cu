// sort.cu -- K3: stable LSD radix sort of one record set into the canonical
// order the analysis kernel expects: grouped by resource id, start-sorted
// within a resource (reference: Trace.__post_init__'s canonical sort,
// model.py:74-80,99-107, and flatten's items.sort(), intervals.py:53).
//
// Keys are compressed before sorting: with s' = start - min(start) and
// r' = flip(res) - min(flip(res)) (flip = sign-bit flip so negative ids order
// first), a record's key is (r' << bt) | s' where bt = bits(max s').  When
// bits(r') + bt <= 64 (the normal case) one u64 key carries both, and the
// sorted key alone reconstructs start and res -- only end and kind are
// gathered through the permutation at the end.  Otherwise the sort runs in two
// stable stages (by s', then by r').
//
// The first pass's digit counts come from the key-building kernel, and the last pass of
// a narrow sort writes the output columns itself (start, res, end and kind from the key
// and the index), so no pass re-reads the keys only to count or to unpack them.
//
// Each digit pass is reduce-then-scan: an upsweep kernel counts the digits of
// every tile (digit-major count matrix), a three-kernel scan turns the matrix
// into the global position of every (digit, tile) run, and the downsweep
// kernel ranks its tile's keys stably with warp-level match/popc (warp-striped
// items, warps in order), reorders the tile in shared memory and writes digit
// runs back coalesced.  No inter-CTA chain: every tile is independent, so the
// passes stay bandwidth-bound (a decoupled look-back variant measured 2-4x
// slower here -- its per-tile chain, not HBM, was the limit).
//
// Ties (equal res and start) keep their input order.  Summaries and metrics
// do not depend on tie order (the union and the sums are order-free;
// SURVEY.md appendix A.5).
#include <cuda_runtime.h>
#include <cstdint>

#include "engine.cuh"
#include "ptx.cuh"

namespace hb {
namespace rsort {

#ifndef HB_SORT_T
#define HB_SORT_T 512
#endif
#ifndef HB_SORT_I
#define HB_SORT_I 11
#endif
#ifndef HB_SORT_VEARLY
#define HB_SORT_VEARLY 1
#endif
#ifndef HB_SORT_MINB
#define HB_SORT_MINB (HB_SORT_T <= 512 ? 1024 / HB_SORT_T : 1)   // resident CTAs per SM (64 registers)
#endif
constexpr int kT = HB_SORT_T;           // threads per CTA (512: 2 CTAs / SM)
constexpr int kW = kT / 32;
constexpr int kI = HB_SORT_I;           // keys per thread
constexpr int kTileKeys = kT * kI;      // 7680 keys per tile
constexpr int kDMax = 8;                 // max bits per digit (9-bit digits / 4 passes measured slower:
constexpr int kBins = 1 << kDMax;        // shorter digit runs scatter the writes)

struct Range {
    u64 smin, smax;
    unsigned int rmin, rmax;            // flipped domain
    unsigned int start_desc;            // some start is below its predecessor's
    unsigned int kind_wide;             // some kind code > 3: not packable into the index
    u64 dmax;                           // max end - start
    unsigned int neg;                   // some end < start (malformed)
    unsigned int pad;
};

__device__ __forceinline__ unsigned int flip(int32_t r) { return (unsigned int)r ^ 0x80000000u; }
__device__ __forceinline__ int32_t unflip(unsigned int r) { return (int32_t)(r ^ 0x80000000u); }

// ---------------------------------------------------------------------------
// range of start / res
// ---------------------------------------------------------------------------
__global__ void range_init(Range *g)
{
    g->smin = ~0ull;
    g->smax = 0;
    g->rmin = 0xffffffffu;
    g->rmax = 0;
    g->start_desc = 0;
    g->kind_wide = 0;
    g->dmax = 0;
    g->neg = 0;
    g->pad = 0;   // every byte the D2H reads is defined (compute-sanitizer initcheck)
}

// VEC: each thread takes record pairs (16-byte start / end loads, 8-byte res loads); a
// pair's predecessor start comes from the neighbouring lane
template <bool VEC>
__global__ void __launch_bounds__(512) range_kernel(const u64 *__restrict__ S, const u64 *__restrict__ E,
                                                    const int32_t *__restrict__ R, int64_t n, Range *g)
{
    u64 smin = ~0ull, smax = 0, dmax = 0;
    unsigned int rmin = 0xffffffffu, rmax = 0;
    bool desc = false, neg = false;
    auto one = [&](u64 s, u64 e, int32_t rr) {
        const unsigned int r = flip(rr);
        smin = umin(smin, s);
        smax = umax(smax, s);
        rmin = min(rmin, r);
        rmax = max(rmax, r);
        neg = neg || e < s;
        dmax = umax(dmax, e - s);
    };
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (VEC) {
        const int64_t pairs = n >> 1;
        const int lane = threadIdx.x & 31;
        // every lane of a warp runs the same trip count (the shuffle needs them all)
        const int64_t trips = (pairs + stride - 1) / stride;
        for (int64_t t = 0; t < trips; ++t) {
            const int64_t p = t0 + t * stride;
            const bool in = p < pairs;
            ulonglong2 s2 = make_ulonglong2(0, 0), e2 = make_ulonglong2(0, 0);
            int2 r2 = make_int2(0, 0);
            if (in) {
                s2 = __ldcs(reinterpret_cast<const ulonglong2 *>(S) + p);
                e2 = __ldcs(reinterpret_cast<const ulonglong2 *>(E) + p);
                r2 = __ldcs(reinterpret_cast<const int2 *>(R) + p);
            }
            u64 prev = __shfl_up_sync(0xffffffffu, s2.y, 1);
            if (lane == 0 && in && p > 0) prev = __ldg(S + 2 * p - 1);
            if (in) {
                desc = desc || (p > 0 && prev > s2.x) || s2.x > s2.y;
                one(s2.x, e2.x, r2.x);
                one(s2.y, e2.y, r2.y);
            }
        }
        if (t0 == 0 && (n & 1)) {   // the odd last record
            const int64_t i = n - 1;
            const u64 si = __ldg(S + i);
            desc = desc || (i > 0 && __ldg(S + i - 1) > si);
            one(si, __ldg(E + i), __ldg(R + i));
        }
    } else {
        for (int64_t i = t0; i < n; i += stride) {
            const u64 si = __ldg(S + i);
            desc = desc || (i > 0 && __ldg(S + i - 1) > si);
            one(si, __ldcs(E + i), __ldcs(R + i));
        }
    }
    // 64-bit warp reductions by shuffles (the kernel is bandwidth-bound)
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        smin = umin(smin, __shfl_xor_sync(0xffffffffu, smin, d));
        smax = umax(smax, __shfl_xor_sync(0xffffffffu, smax, d));
        dmax = umax(dmax, __shfl_xor_sync(0xffffffffu, dmax, d));
    }
    neg = __any_sync(0xffffffffu, neg);
    rmin = __reduce_min_sync(0xffffffffu, rmin);
    rmax = __reduce_max_sync(0xffffffffu, rmax);
    desc = __any_sync(0xffffffffu, desc);
    if ((threadIdx.x & 31) == 0) {
        if (desc) atomicOr(&g->start_desc, 1u);
        if (neg) atomicOr(&g->neg, 1u);
        atomicMax(&g->dmax, dmax);
        atomicMin(&g->smin, smin);
        atomicMax(&g->smax, smax);
        atomicMin(&g->rmin, rmin);
        atomicMax(&g->rmax, rmax);
    }
}

// ---------------------------------------------------------------------------
// key building + every pass's global digit histogram
// ---------------------------------------------------------------------------
struct KeyPlan {
    u64 smin;
    unsigned int rmin;
    int bt;            // bits of the start offset
    int wide;          // 1: stage 1 keys are s' only (res sorted in stage 2)
    int res_only;      // 1: input already start-sorted: one stable sort by r' suffices
    int passes;        // digit passes of this stage
    int dbits;         // bits per digit
    int packk;         // narrow keys, n <= 2^30: the kind rides in the index's top two bits
    int dshift;        // > 0: end - start stashed in key bits [dshift, 64), above every digit pass
    int br;            // bits of the resource offset
};

__device__ __forceinline__ u64 make_key(const KeyPlan &kp, u64 s, int32_t r)
{
    const u64 so = s - kp.smin;
    if (kp.res_only) return (u64)(flip(r) - kp.rmin);
    if (kp.wide || kp.bt >= 64) return so;
    return ((u64)(flip(r) - kp.rmin) << kp.bt) | so;
}

// durations stashed above the digit passes ride through every pass for free: the
// finish rebuilds end = start + duration and no random gather is left

// packk: V = index | kind << 30, so the final gather fetches the end column alone
// (one random 32-byte sector per record instead of two); kinds > 3 raise kind_wide
// and the finish gathers them instead
constexpr uint32_t kIdxMask = 0x3fffffffu;

// one CTA per sort tile: the keys and indices of the tile, and the tile's digit counts of
// the first pass (the upsweep the first pass would otherwise run over the keys again)
constexpr int kBT = 256;
__global__ void __launch_bounds__(kBT) build_keys(const u64 *__restrict__ S, const u64 *__restrict__ E,
                                                  const int32_t *__restrict__ R,
                                                  const uint8_t *__restrict__ KD, int64_t n, KeyPlan kp,
                                                  u64 *__restrict__ K, uint32_t *__restrict__ V,
                                                  unsigned int *__restrict__ kind_wide,
                                                  uint32_t *__restrict__ counts, int64_t tiles)
{
    __shared__ uint32_t h[kBT / 32][kBins];
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t bins = 1u << kp.dbits;
    const u64 mask = bins - 1;
    for (int i = tid; i < (kBT / 32) * kBins; i += kBT) (&h[0][0])[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kTileKeys;
    const int64_t end = n - base < kTileKeys ? n : base + kTileKeys;
    bool wide = false;
    auto one = [&](int64_t i, u64 si, int32_t ri, u64 ei, uint32_t ki) {
        u64 key = make_key(kp, si, ri);
        if (kp.dshift) key |= (ei - si) << kp.dshift;
        K[i] = key;
        atomicAdd(&h[warp][(uint32_t)(key & mask)], 1u);
        uint32_t v = (uint32_t)i;
        if (kp.packk) {
            wide = wide || ki > 3u;
            v |= (ki & 3u) << 30;
        }
        V[i] = v;
    };
    constexpr int kU = 11;   // records in flight per thread (loads issued before the keys are built)
    int64_t i = base + tid;
    for (; i + (kU - 1) * kBT < end; i += kU * kBT) {
        u64 s[kU], e[kU];
        int32_t r[kU];
        uint32_t k[kU];
#pragma unroll
        for (int q = 0; q < kU; ++q) {
            const int64_t j = i + q * kBT;
            s[q] = __ldcs(S + j);
            r[q] = __ldcs(R + j);
            e[q] = kp.dshift ? __ldcs(E + j) : 0ull;
            k[q] = kp.packk ? __ldcs(KD + j) : 0u;
        }
#pragma unroll
        for (int q = 0; q < kU; ++q) one(i + q * kBT, s[q], r[q], e[q], k[q]);
    }
    for (; i < end; i += kBT)
        one(i, __ldcs(S + i), __ldcs(R + i), kp.dshift ? __ldcs(E + i) : 0ull, kp.packk ? __ldcs(KD + i) : 0u);
    if (__syncthreads_or(wide) && tid == 0) atomicOr(kind_wide, 1u);
    for (int d = tid; d < (int)bins; d += kBT) {
        uint32_t c = 0;
#pragma unroll
        for (int w = 0; w < kBT / 32; ++w) c += h[w][d];
        counts[(int64_t)d * tiles + blockIdx.x] = c;
    }
}

// wide keys, stage 2: r' of each record in stage-1 order
__global__ void __launch_bounds__(512) build_res_keys(const int32_t *__restrict__ R, const uint32_t *__restrict__ V,
                                                      int64_t n, KeyPlan kp, u64 *__restrict__ K)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        K[i] = (u64)(flip(__ldg(R + V[i])) - kp.rmin);
}

// ---------------------------------------------------------------------------
// one digit pass
// ---------------------------------------------------------------------------
struct PassSmem {
    u64 k[kTileKeys];
    uint32_t v[kTileKeys];
    uint16_t src[kTileKeys];     // payload passes: in-tile source position of each sorted key
    uint32_t whist[kW][kBins];   // per-warp digit counts -> warp-exclusive offsets
    uint32_t bexcl[kBins];       // tile-local exclusive digit offsets
    uint32_t gbase[kBins];       // destination of the tile's first key of each digit
    uint32_t wsum[kW];
};

// exclusive scan of one value per thread t < kBins (all threads must call)
__device__ __forceinline__ uint32_t block_excl_scan_bins(uint32_t x, uint32_t *wsum, int tid)
{
    const int lane = tid & 31, warp = tid >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
    }
    __syncthreads();
    if (tid < kBins && lane == 31) wsum[warp] = inc;
    __syncthreads();
    uint32_t off = 0;
    if (tid < kBins)
        for (int w = 0; w < warp; ++w) off += wsum[w];
    return off + inc - x;
}

// per-tile digit counts of one pass, digit-major: counts[d * tiles + t].
// Warp-private shared counters (atomics conflict only inside a warp); a
// 256-thread CTA per tile keeps more tiles' loads in flight per SM.
constexpr int kUT = 256, kUW = kUT / 32, kUI = kTileKeys / kUT;
static_assert(kTileKeys % kUT == 0, "the upsweep covers a tile in whole 256-thread strides (HB_SORT_T x HB_SORT_I)");
__global__ void __launch_bounds__(kUT) upsweep(const u64 *__restrict__ kin, int64_t n, int shift, int dbits,
                                               uint32_t *__restrict__ counts, int64_t tiles)
{
    __shared__ uint32_t h[kUW][kBins];
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t bins = 1u << dbits;
    const u64 mask = bins - 1;
    for (int i = tid; i < kUW * kBins; i += kUT) (&h[0][0])[i] = 0;
    __syncthreads();
    const int64_t tile = blockIdx.x;
    const int64_t base = tile * kTileKeys;
    const int cnt = (int)((n - base) < kTileKeys ? (n - base) : kTileKeys);
    const u64 *kt = kin + base;
    if (cnt == kTileKeys) {
        u64 k[kUI];
#pragma unroll
        for (int j = 0; j < kUI; ++j) k[j] = __ldcs(kt + j * kUT + tid);
#pragma unroll
        for (int j = 0; j < kUI; ++j) atomicAdd(&h[warp][(uint32_t)((k[j] >> shift) & mask)], 1u);
    } else {
        for (int i = tid; i < cnt; i += kUT) atomicAdd(&h[warp][(uint32_t)((__ldcs(kt + i) >> shift) & mask)], 1u);
    }
    __syncthreads();
    for (int d = tid; d < (int)bins; d += kUT) {
        uint32_t c = 0;
#pragma unroll
        for (int w = 0; w < kUW; ++w) c += h[w][d];
        counts[(int64_t)d * tiles + tile] = c;
    }
}

// exclusive scan of the digit-major count matrix (global positions of every
// (digit, tile) run): block sums, a one-block scan of those, then the blocks
constexpr int kScanT = 1024, kScanI = 4, kScanBlock = kScanT * kScanI;

__device__ __forceinline__ uint32_t block_scan_excl_1024(uint32_t x, uint32_t *ws, uint32_t &total)
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
    if (warp == 0) {
        uint32_t v = ws[lane], vi = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, vi, d);
            if (lane >= d) vi += o;
        }
        ws[lane] = vi - v;
        if (lane == 31) ws[32] = vi;
    }
    __syncthreads();
    const uint32_t r = ws[warp] + inc - x;
    total = ws[32];
    __syncthreads();
    return r;
}

__global__ void __launch_bounds__(kScanT) scan_sums(const uint32_t *__restrict__ c, int64_t m, uint32_t *__restrict__ bsum)
{
    __shared__ uint32_t ws[33];
    const int64_t b0 = (int64_t)blockIdx.x * kScanBlock;
    uint32_t acc = 0;
#pragma unroll
    for (int q = 0; q < kScanI; ++q) {
        const int64_t i = b0 + (int64_t)q * kScanT + threadIdx.x;
        acc += i < m ? c[i] : 0u;
    }
    uint32_t total;
    block_scan_excl_1024(acc, ws, total);
    if (threadIdx.x == 0) bsum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(kScanT) scan_top(uint32_t *bsum, int64_t nb)
{
    __shared__ uint32_t ws[33];
    uint32_t carry = 0;
    for (int64_t b0 = 0; b0 < nb; b0 += kScanT) {
        const int64_t i = b0 + threadIdx.x;
        const uint32_t x = i < nb ? bsum[i] : 0u;
        uint32_t total;
        const uint32_t ex = block_scan_excl_1024(x, ws, total);
        if (i < nb) bsum[i] = carry + ex;
        carry += total;
    }
}

__global__ void __launch_bounds__(kScanT) scan_blocks(uint32_t *c, int64_t m, const uint32_t *__restrict__ bsum)
{
    __shared__ uint32_t ws[33];
    const int64_t b0 = (int64_t)blockIdx.x * kScanBlock + (int64_t)threadIdx.x * kScanI;   // blocked
    uint32_t v[kScanI], acc = 0;
#pragma unroll
    for (int q = 0; q < kScanI; ++q) {
        v[q] = b0 + q < m ? c[b0 + q] : 0u;
        acc += v[q];
    }
    uint32_t total;
    uint32_t run = bsum[blockIdx.x] + block_scan_excl_1024(acc, ws, total);
#pragma unroll
    for (int q = 0; q < kScanI; ++q) {
        if (b0 + q < m) c[b0 + q] = run;
        run += v[q];
    }
}

// lanes holding the same digit as this lane, from dbits ballots (faster than
// match.any on this part, measured: the upsweep went 348 -> 61 us without it)
template <int DB>
__device__ __forceinline__ uint32_t peers_of(uint32_t d, uint32_t valid_mask)
{
    uint32_t m = valid_mask;
#pragma unroll
    for (int b = 0; b < DB; ++b) {
        const uint32_t bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        m &= ((d >> b) & 1u) ? bb : ~bb;
    }
    return m;
}

// one digit pass: stable rank of the tile's keys, reorder in shared memory,
// coalesced digit runs to their scanned global positions
// payload columns moved with the keys (start-ordered input: start, end, kind ride
// along, so the sorted columns need no random gather at the end)
struct Payload {
    const u64 *s_in, *e_in;
    const uint8_t *k_in;
    u64 *s_out, *e_out;
    uint8_t *k_out;
};

// the last pass of a narrow sort writes the output columns itself (what finish_narrow
// does after the passes otherwise): start and res from the key, end from the stashed
// duration or a gather, kind from the index's top bits or a gather
struct Finish {
    KeyPlan kp;
    const unsigned int *kind_wide;
    const u64 *E;
    const uint8_t *KD;
    u64 *os, *oe;
    int32_t *orr;
    uint8_t *ok;
    int64_t *perm;
};

enum { kPlain = 0, kCarry = 1, kFinish = 2 };

// DB (bits per digit) is a template argument: the ballot ranking unrolls exactly DB bits
template <int MODE, int DB>
__global__ void __launch_bounds__(kT, HB_SORT_MINB) downsweep(const u64 *__restrict__ kin, const uint32_t *__restrict__ vin,
                                                   u64 *__restrict__ kout, uint32_t *__restrict__ vout, int64_t n,
                                                   int shift, const uint32_t *__restrict__ offs,
                                                   int64_t tiles, Payload pl, Finish fin)
{
    constexpr bool PL = MODE == kCarry;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    PassSmem &sm = *reinterpret_cast<PassSmem *>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr uint32_t bins = 1u << DB;
    constexpr u64 mask = bins - 1;
    const int64_t tile = blockIdx.x;
    for (int i = tid; i < kW * kBins; i += kT) (&sm.whist[0][0])[i] = 0;
    for (int d = tid; d < (int)bins; d += kT) sm.gbase[d] = offs[(int64_t)d * tiles + tile];
    __syncthreads();
    const int64_t base = tile * kTileKeys;
    const int64_t wbase = base + (int64_t)warp * 32 * kI;
    const int64_t wrem64 = n - wbase;   // records of this warp's slice still in range
    const int wrem = wrem64 <= 0 ? 0 : (wrem64 > 32 * kI ? 32 * kI : (int)wrem64);
    const u64 *kw = kin + wbase;

    u64 k[kI];
    uint32_t rk[(kI + 1) / 2];   // warp ranks (< 2^9), two per register
#pragma unroll
    for (int j = 0; j < kI; ++j) {
        const int o = j * 32 + lane;
        k[j] = o < wrem ? __ldcs(kw + o) : 0ull;
    }
    // stable warp-level ranking (items j, then lanes, are in input order);
    // invalid lanes carry a digit no valid lane has, so the match never diverges
    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < (kI + 1) / 2; ++j) rk[j] = 0;
#pragma unroll
    for (int j = 0; j < kI; ++j) {
        const bool valid = j * 32 + lane < wrem;
        const uint32_t dj = (uint32_t)((k[j] >> shift) & mask);
        const uint32_t pm = peers_of<DB>(dj, __ballot_sync(0xffffffffu, valid));
        const int leader = __ffs(pm) - 1;
        const uint32_t b = valid ? sm.whist[warp][dj] : 0u;
        __syncwarp();
        if (valid && lane == leader) sm.whist[warp][dj] = b + __popc(pm);
        __syncwarp();
        rk[j >> 1] |= (b + __popc(pm & lt)) << (16 * (j & 1));
    }
#if HB_SORT_VEARLY
    // the index column's loads overlap the digit scan below
    uint32_t vv[kI];
#pragma unroll
    for (int j = 0; j < kI; ++j) vv[j] = j * 32 + lane < wrem ? __ldcs(vin + wbase + j * 32 + lane) : 0u;
#endif
    __syncthreads();
    // per digit: warp-exclusive offsets and the tile total
    uint32_t total = 0;
    if (tid < (int)bins) {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kW; ++w) {
            const uint32_t c = sm.whist[w][tid];
            sm.whist[w][tid] = run;
            run += c;
        }
        total = run;
    }
    {
        const uint32_t ex = block_excl_scan_bins(total, sm.wsum, tid);
        if (tid < kBins) sm.bexcl[tid] = ex;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kI; ++j) {
        const int o = j * 32 + lane;
        if (o < wrem) {
            const uint32_t dj = (uint32_t)((k[j] >> shift) & mask);
            const uint32_t pos = sm.bexcl[dj] + sm.whist[warp][dj] + ((rk[j >> 1] >> (16 * (j & 1))) & 0xffffu);
            sm.k[pos] = k[j];
#if HB_SORT_VEARLY
            sm.v[pos] = vv[j];
#else
            sm.v[pos] = __ldcs(vin + wbase + o);
#endif
            if (PL) sm.src[pos] = (uint16_t)(warp * 32 * kI + o);
        }
    }
    __syncthreads();
    const int cnt = (int)((n - base) < kTileKeys ? (n - base) : kTileKeys);
    if constexpr (MODE == kFinish) {
        const KeyPlan &kp = fin.kp;
        const u64 tmask = kp.bt >= 64 ? ~0ull : ((1ull << kp.bt) - 1);
        const bool gather_k = !kp.packk || *fin.kind_wide;
        for (int i = tid; i < cnt; i += kT) {
            const u64 key = sm.k[i];
            const uint32_t pv = sm.v[i];
            const uint32_t dd = (uint32_t)((key >> shift) & mask);
            const u64 dst = (u64)sm.gbase[dd] + (u64)(i - (int)sm.bexcl[dd]);
            const uint32_t v = kp.packk ? pv & kIdxMask : pv;
            const u64 st = (key & tmask) + kp.smin;
            fin.os[dst] = st;
            const u64 rbits = kp.bt >= 64 ? 0ull : (key >> kp.bt) & ((1ull << kp.br) - 1);
            fin.orr[dst] = unflip((unsigned int)rbits + kp.rmin);
            fin.oe[dst] = kp.dshift ? st + (key >> kp.dshift) : __ldg(fin.E + v);
            fin.ok[dst] = gather_k ? __ldg(fin.KD + v) : (uint8_t)(pv >> 30);
            if (fin.perm) fin.perm[dst] = v;
        }
    } else {
        for (int i = tid; i < cnt; i += kT) {
            const u64 key = sm.k[i];
            const uint32_t dd = (uint32_t)((key >> shift) & mask);
            const u64 dst = (u64)sm.gbase[dd] + (u64)(i - (int)sm.bexcl[dd]);
            kout[dst] = key;
            vout[dst] = sm.v[i];
            if (PL) {   // tile-local gather (L2-resident), coalesced digit-run writes
                const int64_t src = base + sm.src[i];
                pl.s_out[dst] = __ldg(pl.s_in + src);
                pl.e_out[dst] = __ldg(pl.e_in + src);
                pl.k_out[dst] = __ldg(pl.k_in + src);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// output columns
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512) finish_narrow(const u64 *__restrict__ K, const uint32_t *__restrict__ V,
                                                     int64_t n, KeyPlan kp, const unsigned int *__restrict__ kind_wide,
                                                     const u64 *__restrict__ E,
                                                     const uint8_t *__restrict__ KD, u64 *__restrict__ os,
                                                     u64 *__restrict__ oe, int32_t *__restrict__ orr,
                                                     uint8_t *__restrict__ ok, int64_t *__restrict__ perm)
{
    const u64 tmask = kp.bt >= 64 ? ~0ull : ((1ull << kp.bt) - 1);
    const bool gather_k = !kp.packk || *kind_wide;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const u64 key = __ldcs(K + i);
        const uint32_t pv = __ldcs(V + i);
        const uint32_t v = kp.packk ? pv & kIdxMask : pv;
        const u64 st = (key & tmask) + kp.smin;
        os[i] = st;
        const u64 rbits = kp.bt >= 64 ? 0ull : (key >> kp.bt) & ((1ull << kp.br) - 1);
        orr[i] = unflip((unsigned int)rbits + kp.rmin);
        oe[i] = kp.dshift ? st + (key >> kp.dshift) : __ldg(E + v);
        ok[i] = gather_k ? __ldg(KD + v) : (uint8_t)(pv >> 30);
        if (perm) perm[i] = v;
    }
}

__global__ void __launch_bounds__(512) finish_payload(const u64 *__restrict__ K, const uint32_t *__restrict__ V,
                                                      int64_t n, KeyPlan kp, int32_t *__restrict__ orr,
                                                      int64_t *__restrict__ perm)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        orr[i] = unflip((unsigned int)__ldcs(K + i) + kp.rmin);
        if (perm) perm[i] = __ldcs(V + i);
    }
}

__global__ void __launch_bounds__(512) finish_gather(const uint32_t *__restrict__ V, int64_t n,
                                                     const u64 *__restrict__ S, const u64 *__restrict__ E,
                                                     const int32_t *__restrict__ R, const uint8_t *__restrict__ KD,
                                                     u64 *__restrict__ os, u64 *__restrict__ oe,
                                                     int32_t *__restrict__ orr, uint8_t *__restrict__ ok,
                                                     int64_t *__restrict__ perm)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = __ldcs(V + i);
        os[i] = __ldg(S + v);
        oe[i] = __ldg(E + v);
        orr[i] = __ldg(R + v);
        ok[i] = __ldg(KD + v);
        if (perm) perm[i] = v;
    }
}

__global__ void remap_kernel(int64_t *list, int64_t k, const int64_t *__restrict__ perm)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x)
        list[i] = perm[list[i]];
}

// canonical-order check of one record set: (res, start) non-decreasing
__global__ void __launch_bounds__(512) order_check(const int32_t *__restrict__ R, const u64 *__restrict__ S, int64_t n,
                                                   unsigned int *bad)
{
    bool b = false;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x + 1; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = __ldcs(R + i), rp = __ldg(R + i - 1);
        b = b || r < rp || (r == rp && __ldcs(S + i) < __ldg(S + i - 1));
    }
    if (__any_sync(0xffffffffu, b) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

}  // namespace rsort

cudaError_t launch_order_check(const int32_t *R, const u64 *S, int64_t n, unsigned int *bad, cudaStream_t s)
{
    if (n < 2) return cudaSuccess;
    int64_t g = (n + 511) / 512;
    if (g > 148 * 8) g = 148 * 8;
    rsort::order_check<<<(unsigned)g, 512, 0, s>>>(R, S, n, bad);
    return cudaGetLastError();
}

cudaError_t launch_remap(int64_t *list, int64_t k, const int64_t *perm, cudaStream_t s)
{
    const int64_t g = (k + 255) / 256;
    rsort::remap_kernel<<<(unsigned)(g > 4096 ? 4096 : g), 256, 0, s>>>(list, k, perm);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------
static size_t up256(size_t x) { return (x + 255) & ~(size_t)255; }

static int64_t tiles_of(int64_t n) { return (n + rsort::kTileKeys - 1) / rsort::kTileKeys; }

size_t sort_workspace_bytes(int64_t n)
{
    const int64_t m = tiles_of(n) * rsort::kBins;
    return 2 * up256((size_t)n * 8) + 2 * up256((size_t)n * 4) + up256((size_t)m * 4) +
           up256((size_t)(m / rsort::kScanBlock + 1) * 4) + up256(sizeof(rsort::Range)) +
           2 * up256((size_t)n * 8) + up256((size_t)n);   // payload ping-pong (start-ordered input)
}

static int bits_of(u64 x) { return x ? 64 - __builtin_clzll(x) : 0; }

using DownFn = void (*)(const u64 *, const uint32_t *, u64 *, uint32_t *, int64_t, int, const uint32_t *, int64_t,
                        rsort::Payload, rsort::Finish);
// downsweep instantiations by [mode][bits per digit]
static DownFn down_table(int mode, int dbits)
{
    using namespace rsort;
#define HB_DS_ROW(M) {nullptr, downsweep<M, 1>, downsweep<M, 2>, downsweep<M, 3>, downsweep<M, 4>, \
                      downsweep<M, 5>, downsweep<M, 6>, downsweep<M, 7>, downsweep<M, 8>}
    static const DownFn tbl[3][kDMax + 1] = {HB_DS_ROW(kPlain), HB_DS_ROW(kCarry), HB_DS_ROW(kFinish)};
#undef HB_DS_ROW
    return tbl[mode][dbits];
}

static int grid_for(int64_t n, int sms)
{
    int64_t g = (n + 511) / 512;
    const int64_t cap = (int64_t)sms * 8;
    if (g > cap) g = cap;
    return g < 1 ? 1 : (int)g;
}

cudaError_t sort_records(const u64 *S, const u64 *E, const int32_t *R, const uint8_t *KD, int64_t n, u64 *os, u64 *oe,
                         int32_t *orr, uint8_t *ok, int64_t *perm, void *ws, size_t ws_bytes, cudaStream_t s,
                         SortStats *stats)
{
    using namespace rsort;
    if (n <= 0) return cudaSuccess;
    if (n >= (int64_t)0xffffffffll) return cudaErrorInvalidValue;          // 32-bit permutation indices
    if (ws_bytes < sort_workspace_bytes(n)) return cudaErrorInvalidValue;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    static bool attr_done = false;
    if (!attr_done) {
        for (int mode = 0; mode < 3; ++mode)
            for (int db = 1; db <= kDMax; ++db) {
                const cudaError_t e = cudaFuncSetAttribute(down_table(mode, db),
                                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                           (int)sizeof(PassSmem));
                if (e != cudaSuccess) return e;
            }
        attr_done = true;
    }
    const int64_t tiles = tiles_of(n);
    const int64_t m = tiles * kBins;
    const int64_t nb = (m + kScanBlock - 1) / kScanBlock;
    uint8_t *b = static_cast<uint8_t *>(ws);
    size_t o = 0;
    auto take = [&](size_t bytes) { void *p = b + o; o += up256(bytes); return p; };
    u64 *K0 = static_cast<u64 *>(take((size_t)n * 8));
    u64 *K1 = static_cast<u64 *>(take((size_t)n * 8));
    uint32_t *V0 = static_cast<uint32_t *>(take((size_t)n * 4));
    uint32_t *V1 = static_cast<uint32_t *>(take((size_t)n * 4));
    uint32_t *counts = static_cast<uint32_t *>(take((size_t)m * 4));
    uint32_t *bsum = static_cast<uint32_t *>(take((size_t)(m / kScanBlock + 1) * 4));
    Range *range = static_cast<Range *>(take(sizeof(Range)));
    u64 *PS = static_cast<u64 *>(take((size_t)n * 8));
    u64 *PE = static_cast<u64 *>(take((size_t)n * 8));
    uint8_t *PK = static_cast<uint8_t *>(take((size_t)n));
    cudaError_t e;

    // 1. key range (one D2H of 32 bytes decides the key layout)
    range_init<<<1, 1, 0, s>>>(range);
    // one resident wave (4 CTAs of 512 per SM); 16-byte loads when the columns allow them
    {
        const bool vec = ((reinterpret_cast<uintptr_t>(S) | reinterpret_cast<uintptr_t>(E)) & 15) == 0 &&
                         (reinterpret_cast<uintptr_t>(R) & 7) == 0;
        int64_t g = ((n + 1) / 2 + 511) / 512;
        g = g < 1 ? 1 : (g > (int64_t)sms * 4 ? (int64_t)sms * 4 : g);
        if (vec) range_kernel<true><<<(unsigned)g, 512, 0, s>>>(S, E, R, n, range);
        else range_kernel<false><<<grid_for(n, sms), 512, 0, s>>>(S, E, R, n, range);
    }
    Range rg;
    if ((e = cudaMemcpyAsync(&rg, range, sizeof(Range), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    const int bt = bits_of(rg.smax - rg.smin);
    const int br = bits_of((u64)(rg.rmax - rg.rmin));
    KeyPlan kp;
    kp.smin = rg.smin;
    kp.rmin = rg.rmin;
    kp.bt = bt;
    kp.br = br;
    kp.dshift = 0;
    // input already ordered by start (e.g. a globally time-ordered event log):
    // a stable sort by resource alone yields the canonical order
    kp.res_only = rg.start_desc ? 0 : 1;
    kp.wide = (!kp.res_only && bt + br > 64) ? 1 : 0;
    kp.packk = (!kp.wide && !kp.res_only && n <= (int64_t)kIdxMask + 1) ? 1 : 0;
    const int stage_bits[2] = {kp.res_only ? br : (kp.wide ? bt : bt + br), kp.wide ? br : 0};

    u64 *kin = K0, *kout = K1;
    uint32_t *vin = V0, *vout = V1;
    int total_passes = 0;
    // start-ordered input: start / end / kind ride along with the keys (no final gather);
    // the last pass writes them straight into the output columns
    const bool carry = kp.res_only && stage_bits[0] > 0;
    Payload pl{S, E, KD, nullptr, nullptr, nullptr};
    // narrow keys: the last pass writes the output columns (no finish kernel)
    const bool narrow = !kp.wide && !kp.res_only;
    Finish fin{};
    for (int stage = 0; stage < 2; ++stage) {
        const int bits = stage_bits[stage];
        if (stage == 1 && !kp.wide) break;
        const int passes = bits == 0 ? 0 : (bits + kDMax - 1) / kDMax;
        kp.passes = passes;
        kp.dbits = passes ? (bits + passes - 1) / passes : 1;
        if (stage == 0) {
            // narrow keys: stash end - start above the bits the passes examine when it fits
            kp.dshift = 0;
            const int cover = passes * kp.dbits;
            if (!kp.wide && !kp.res_only && !rg.neg && cover < 64 && bits_of(rg.dmax) <= 64 - cover) kp.dshift = cover;
            build_keys<<<(unsigned)tiles, kBT, 0, s>>>(S, E, R, KD, n, kp, kin, vin, &range->kind_wide, counts, tiles);
        }
        else build_res_keys<<<grid_for(n, sms), 512, 0, s>>>(R, vin, n, kp, kin);
        for (int p = 0; p < passes; ++p) {
            const int shift = p * kp.dbits;
            const int64_t mm = ((int64_t)1 << kp.dbits) * tiles;   // this pass's matrix (digit-major)
            const int64_t nbb = (mm + kScanBlock - 1) / kScanBlock;
            if (stage == 1 || p > 0)   // the first pass's counts come from build_keys
                upsweep<<<(unsigned)tiles, kUT, 0, s>>>(kin, n, shift, kp.dbits, counts, tiles);
            scan_sums<<<(unsigned)nbb, kScanT, 0, s>>>(counts, mm, bsum);
            scan_top<<<1, kScanT, 0, s>>>(bsum, nbb);
            scan_blocks<<<(unsigned)nbb, kScanT, 0, s>>>(counts, mm, bsum);
            int mode = kPlain;
            if (carry) {
                const bool to_out = ((passes - 1 - p) & 1) == 0;
                pl.s_out = to_out ? os : PS;
                pl.e_out = to_out ? oe : PE;
                pl.k_out = to_out ? ok : PK;
                mode = kCarry;
            } else if (narrow && p == passes - 1) {
                fin = Finish{kp, &range->kind_wide, E, KD, os, oe, orr, ok, perm};
                mode = kFinish;
            }
            down_table(mode, kp.dbits)<<<(unsigned)tiles, kT, sizeof(PassSmem), s>>>(kin, vin, kout, vout, n, shift,
                                                                                   counts, tiles, pl, fin);
            if (carry) {
                pl.s_in = pl.s_out;
                pl.e_in = pl.e_out;
                pl.k_in = pl.k_out;
            }
            u64 *tk = kin; kin = kout; kout = tk;
            uint32_t *tv = vin; vin = vout; vout = tv;
            ++total_passes;
        }
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    (void)nb;
    if (narrow && total_passes > 0) {
        // written by the last pass
    } else if (narrow) {
        finish_narrow<<<grid_for(n, sms), 512, 0, s>>>(kin, vin, n, kp, &range->kind_wide, E, KD, os, oe, orr, ok,
                                                       perm);
    } else if (carry) {
        finish_payload<<<grid_for(n, sms), 512, 0, s>>>(kin, vin, n, kp, orr, perm);
    } else {
        finish_gather<<<grid_for(n, sms), 512, 0, s>>>(vin, n, S, E, R, KD, os, oe, orr, ok, perm);
    }
    if (stats) {
        stats->key_bits = kp.res_only ? br : bt + br;
        stats->passes = total_passes;
        stats->wide = kp.wide;
        stats->start_sorted = kp.res_only;
    }
    return cudaGetLastError();
}

}  // namespace hb
