// regions.cu -- K5/K6, EXTENSIONS beyond the reference (SURVEY.md section 8,
// rows a22/a23).
//
// K5 monitoring regions.  Region j is a window [a_j, b_j).  Its trace is the
// full trace with every record intersected with the window (intervals.py:
// 98-105 semantics) and shifted by -a_j; a zero-length record survives iff
// a_j <= s < b_j.  The region's report is the reference's compute_report
// (metrics.py:125-154) of that trace.  All windows of a pass are computed in
// ONE read of the trace, without materializing any clipped trace:
//   host   per (window, rank): offload / mpi = sums of clipped durations,
//          span = max clipped end - a_j; E_j = max span over ranks
//          (summarize.py:57-92), or the max clipped device end when n == 0;
//   device per (window, device): the running-max identity of the main kernel
//          with the clamp window [a_j, a_j + E_j):
//            e' = clamp(e), s' = clamp(s), c = max(run, e') - max(run, s')
//          where run is the running max of the RAW ends of earlier records of
//          the device -- records outside the window move run only outside
//          [a_j, a_j + E_j), so the same run serves every window.
//
// K6 offload-wait / device-busy overlap.  With runKM the running max over
// kernel|memory records, [max(run, s), max(run, e)) are disjoint pieces whose
// union is the device's busy set.  Each piece is intersected with the owner
// rank's offload records (walked forward through the rank's host records, a
// merge of two sorted sequences) and every overlap segment is clipped to each
// window: busy_j(g) = |offload(owner(g)) ∩ busy(g) ∩ [a_j, a_j + E_j)|.
//
// Kernels (one pass over each record set, plus tiny scans):
//   reg_hseg     host CSR offsets (binary search per rank id)
//   reg_host<R>  host sums/maxima per (window, rank), warp-striped, coalesced
//   reg_dev_agg  per device tile: segment flag + last-segment max ends
//                (+ device-only traces: max clipped end per window)
//   reg_dev_carry  one block: segmented max scan over tiles -> carries
//   reg_E        E_j per window
//   reg_dev<R>   tile in shared memory, blocked records per thread, in-tile
//                segmented scan, per-window union contributions, clamps and
//                the overlap walk; per-(window, device) totals leave as L2 REDs
//   reg_final    summaries in declaration order, both metric trees with exact
//                division (exact.cuh), the busy fraction
#include <cuda_runtime.h>
#include <climits>
#include <cstdint>

#include "engine.cuh"
#include "exact.cuh"
#include "ptx.cuh"

namespace hb {
namespace reg {

constexpr int kHT = 256;            // host kernel threads
constexpr int kHI = 16;             // host records per thread (warp-striped)
constexpr int kDT = 128;            // device kernel threads
constexpr int kDI = 9;              // device records per thread (odd: conflict-free smem)
constexpr int kDTile = kDT * kDI;   // 1152 records per tile

__device__ __forceinline__ bool is_declared(const int32_t *decl, int32_t ids, int32_t n, int32_t r)
{
    if (r < 0 || r >= ids) return false;
    return decl ? (decl[r] >= 0) : (r < n);
}

__device__ __forceinline__ int32_t decl_pos(const int32_t *decl, int32_t r) { return decl ? decl[r] : r; }

// ---------------------------------------------------------------------------
// host CSR: hseg[id] = first record of dense id `id` (records grouped by id)
// ---------------------------------------------------------------------------
__global__ void reg_hseg(const int32_t *__restrict__ hr, int64_t hn, int32_t ids, int64_t *__restrict__ hseg)
{
    const int32_t id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id > ids) return;
    int64_t lo = 0, hi = hn;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (hr[mid] < id) lo = mid + 1;
        else hi = mid;
    }
    hseg[id] = lo;
}

// ---------------------------------------------------------------------------
// host side: per (window, rank) offload / mpi sums and span
// ---------------------------------------------------------------------------
template <int R>
__device__ __forceinline__ void host_flush(const RegParams &p, int32_t r, const u64 (&off)[R], const u64 (&mpi)[R],
                                           const u64 (&span)[R], const bool (&any)[R])
{
    if (r < 0 || r >= p.host_ids) return;
#pragma unroll
    for (int j = 0; j < R; ++j) {
        u64 *a = p.h_acc + ((size_t)j * p.host_ids + r) * 3;
        if (off[j]) red_add(a + 0, off[j]);
        if (mpi[j]) red_add(a + 1, mpi[j]);
        if (any[j] && span[j]) red_max(a + 2, span[j]);
    }
}

template <int R>
__global__ void __launch_bounds__(kHT) reg_host(const __grid_constant__ RegParams p)
{
    const u64 *lo = p.wlo, *hi = p.whi;    // kernel-parameter (constant bank) operands
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (kHT / 32);
    const int64_t chunk = 32 * kHI;
    for (int64_t w = (blockIdx.x * (int64_t)kHT + threadIdx.x) >> 5; w * chunk < p.hn; w += warps) {
        u64 off[R], mpi[R], span[R];
        bool any[R];
#pragma unroll
        for (int j = 0; j < R; ++j) { off[j] = mpi[j] = span[j] = 0; any[j] = false; }
        int32_t cur = INT_MIN;
#pragma unroll 4
        for (int q = 0; q < kHI; ++q) {
            const int64_t i = w * chunk + q * 32 + lane;
            if (i >= p.hn) break;
            const int32_t r = __ldcs(p.hr + i);
            const u64 s = __ldcs(p.hs + i), e = __ldcs(p.he + i);
            const uint8_t k = __ldcs(p.hk + i);
            if (r != cur) {
                if (cur != INT_MIN) host_flush<R>(p, cur, off, mpi, span, any);
#pragma unroll
                for (int j = 0; j < R; ++j) { off[j] = mpi[j] = span[j] = 0; any[j] = false; }
                cur = r;
            }
#pragma unroll
            for (int j = 0; j < R; ++j) {
                if (s < e) {
                    const u64 cs = umax(s, lo[j]), ce = umin(e, hi[j]);
                    if (cs < ce) {
                        const u64 d = ce - cs;
                        off[j] += k == 1 ? d : 0ull;
                        mpi[j] += k == 2 ? d : 0ull;
                        span[j] = umax(span[j], ce - lo[j]);
                        any[j] = true;
                    }
                } else if (s == e && s >= lo[j] && s < hi[j]) {
                    span[j] = umax(span[j], s - lo[j]);
                    any[j] = true;
                }
            }
        }
        if (cur != INT_MIN) host_flush<R>(p, cur, off, mpi, span, any);
    }
}

// ---------------------------------------------------------------------------
// device tiles: segment flag + last-segment max ends (kernel-only, all)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) reg_dev_agg(const __grid_constant__ RegParams p)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * 8;
    for (int64_t t = (blockIdx.x * 256ll + threadIdx.x) >> 5; t < p.tiles; t += warps) {
        const int64_t b = t * kDTile, e = umin((u64)(b + kDTile), (u64)p.dn);
        // last segment start inside the tile (-1: none, the tile continues its predecessor's segment)
        int64_t last = -1;
        for (int64_t i = b + lane; i < e; i += 32)
            if (i == 0 || p.dr[i] != p.dr[i - 1]) last = i;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const int64_t o = __shfl_xor_sync(0xffffffffu, last, d);
            last = o > last ? o : last;
        }
        const int64_t from = last < 0 ? b : last;
        u64 mk = 0, mkm = 0;
        for (int64_t i = from + lane; i < e; i += 32) {
            const u64 en = p.de[i];
            mkm = umax(mkm, en);
            if (p.dk[i] == 0) mk = umax(mk, en);
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            mk = umax(mk, __shfl_xor_sync(0xffffffffu, mk, d));
            mkm = umax(mkm, __shfl_xor_sync(0xffffffffu, mkm, d));
        }
        if (lane == 0) {
            p.tagg[3 * t + 0] = last >= 0 ? 1ull : 0ull;
            p.tagg[3 * t + 1] = mk;
            p.tagg[3 * t + 2] = mkm;
        }
        if (p.n == 0) {   // device-only trace: E_j = max clipped end of the region's records
            for (int j = 0; j < p.R; ++j) {
                const u64 a = p.wlo[j], w = p.whi[j];
                u64 mx = 0;
                bool any = false;
                for (int64_t i = b + lane; i < e; i += 32) {
                    const u64 s = p.ds[i], en = p.de[i];
                    if (s < en) {
                        const u64 cs = umax(s, a), ce = umin(en, w);
                        if (cs < ce) { mx = umax(mx, ce - a); any = true; }
                    } else if (s == en && s >= a && s < w) {
                        mx = umax(mx, s - a);
                        any = true;
                    }
                }
                any = __any_sync(0xffffffffu, any);
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) mx = umax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
                if (lane == 0 && any && mx) red_max(p.dmax + j, mx);
            }
        }
    }
}

// carries into every tile: sequential over per-thread chunks of tiles
__global__ void __launch_bounds__(1024) reg_dev_carry(const __grid_constant__ RegParams p)
{
    __shared__ u64 sf[1024], sk[1024], skm[1024];
    const int tid = threadIdx.x;
    const int64_t per = (p.tiles + 1023) / 1024;
    const int64_t t0 = tid * per, t1 = umin((u64)(t0 + per), (u64)p.tiles);
    u64 f = 0, k = 0, km = 0;
    for (int64_t t = t0; t < t1; ++t) {
        if (p.tagg[3 * t]) { f = 1; k = p.tagg[3 * t + 1]; km = p.tagg[3 * t + 2]; }
        else { k = umax(k, p.tagg[3 * t + 1]); km = umax(km, p.tagg[3 * t + 2]); }
    }
    sf[tid] = f; sk[tid] = k; skm[tid] = km;
    __syncthreads();
    if (tid == 0) {   // exclusive segmented max over the 1024 chunk aggregates
        u64 ck = 0, ckm = 0;
        for (int c = 0; c < 1024; ++c) {
            const u64 fc = sf[c], kc = sk[c], kmc = skm[c];
            sk[c] = ck; skm[c] = ckm;
            if (fc) { ck = kc; ckm = kmc; }
            else { ck = umax(ck, kc); ckm = umax(ckm, kmc); }
        }
    }
    __syncthreads();
    k = sk[tid];
    km = skm[tid];
    for (int64_t t = t0; t < t1; ++t) {
        p.tcarry[2 * t] = k;
        p.tcarry[2 * t + 1] = km;
        if (p.tagg[3 * t]) { k = p.tagg[3 * t + 1]; km = p.tagg[3 * t + 2]; }
        else { k = umax(k, p.tagg[3 * t + 1]); km = umax(km, p.tagg[3 * t + 2]); }
    }
}

// E_j: max span over declared ranks, or the device-only maximum
__global__ void __launch_bounds__(256) reg_E(const __grid_constant__ RegParams p)
{
    const int j = blockIdx.x;
    u64 mx = 0;
    if (p.n >= 1) {
        for (int32_t id = threadIdx.x; id < p.host_ids; id += 256)
            if (is_declared(p.host_decl, p.host_ids, p.n, id)) {
                mx = umax(mx, p.h_acc[((size_t)j * p.host_ids + id) * 3 + 2]);
            }
    } else if (threadIdx.x == 0) {
        mx = p.dmax[j];
    }
    __shared__ u64 sm[8];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) mx = umax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) mx = umax(mx, sm[w]);
        p.E[j] = mx;
    }
}

// ---------------------------------------------------------------------------
// device side: per (window, device) union contributions, clamps, overlap
// ---------------------------------------------------------------------------
struct DevTile {
    u64 s[kDTile];
    u64 e[kDTile];
    int32_t r[kDTile];
    uint8_t k[kDTile];
};

template <int R>
struct DevAcc {
    u64 K[R], KM[R], busy[R];
    uint32_t clamp[R];
    __device__ __forceinline__ void zero()
    {
#pragma unroll
        for (int j = 0; j < R; ++j) { K[j] = KM[j] = busy[j] = 0; clamp[j] = 0; }
    }
    __device__ __forceinline__ void flush(const RegParams &p, int32_t d)
    {
        if (d < 0 || d >= p.dev_ids) return;
#pragma unroll
        for (int j = 0; j < R; ++j) {
            u64 *a = p.d_acc + ((size_t)j * p.dev_ids + d) * 4;
            if (K[j]) red_add(a + 0, K[j]);
            if (KM[j]) red_add(a + 1, KM[j]);
            if (clamp[j]) red_add(a + 2, (u64)clamp[j]);
            if (busy[j]) red_add(a + 3, busy[j]);
        }
    }
};

// overlap walk state: the owner rank's host records [q, qe)
struct Walk {
    int64_t q, qe;
    bool init;
};

template <int R>
__device__ __forceinline__ void overlap_piece(const RegParams &p, Walk &w, int32_t owner, u64 x, u64 y, DevAcc<R> &A)
{
    if (owner < 0 || owner >= p.host_ids) return;
    if (!w.init) {   // last host record of the owner starting at or before x (binary search)
        int64_t a = p.hseg[owner], b = p.hseg[owner + 1];
        w.qe = b;
        while (a < b) {
            const int64_t mid = (a + b) >> 1;
            if (__ldg(p.hs + mid) <= x) a = mid + 1;
            else b = mid;
        }
        w.q = a > p.hseg[owner] ? a - 1 : a;
        w.init = true;
    }
    while (w.q < w.qe) {
        const u64 hs = __ldg(p.hs + w.q);
        if (hs >= y) break;
        const u64 he = __ldg(p.he + w.q);
        if (__ldg(p.hk + w.q) == 1 && hs < he) {
            const u64 u = umax(hs, x), v = umin(he, y);
            if (u < v) {
#pragma unroll
                for (int j = 0; j < R; ++j) {
                    const u64 cu = umax(u, p.wlo[j]), cv = umin(v, p.wtop[j]);
                    A.busy[j] += cv > cu ? cv - cu : 0ull;
                }
            }
        }
        if (he > y) break;          // this record continues into the next piece
        ++w.q;
    }
}

template <int R>
__global__ void __launch_bounds__(kDT) reg_dev(const __grid_constant__ RegParams p)
{
    __shared__ DevTile T;
    __shared__ u64 w_f[kDT / 32], w_k[kDT / 32], w_km[kDT / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // windows and clamp tops [a, a + E) are kernel parameters (constant-bank operands)
    const u64 *lo = p.wlo, *hi = p.whi, *top = p.wtop;

    for (int64_t t = blockIdx.x; t < p.tiles; t += gridDim.x) {
        const int64_t base = t * kDTile;
        const int cnt = (int)umin((u64)kDTile, (u64)(p.dn - base));
        __syncthreads();
        for (int i = tid; i < cnt; i += kDT) {
            T.s[i] = __ldcs(p.ds + base + i);
            T.e[i] = __ldcs(p.de + base + i);
            T.r[i] = __ldcs(p.dr + base + i);
            T.k[i] = __ldcs(p.dk + base + i);
        }
        const int32_t prev_r = base > 0 ? __ldg(p.dr + base - 1) : INT_MIN;
        __syncthreads();
        // thread aggregate over its blocked records: segment flag, last-segment max ends
        const int b = tid * kDI;
        const int nv = cnt - b < 0 ? 0 : (cnt - b < kDI ? cnt - b : kDI);
        bool f = false;
        u64 ak = 0, akm = 0;
        for (int q = 0; q < nv; ++q) {
            const int i = b + q;
            const int32_t pr = i > 0 ? T.r[i - 1] : prev_r;
            if (T.r[i] != pr) { f = true; ak = 0; akm = 0; }
            akm = umax(akm, T.e[i]);
            if (T.k[i] == 0) ak = umax(ak, T.e[i]);
        }
        // block exclusive segmented max scan over threads
        bool xf = f;
        u64 xk = ak, xkm = akm;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const bool of = __shfl_up_sync(0xffffffffu, xf, d);
            const u64 ok = __shfl_up_sync(0xffffffffu, xk, d), okm = __shfl_up_sync(0xffffffffu, xkm, d);
            if (lane >= d) {
                if (!xf) { xk = umax(xk, ok); xkm = umax(xkm, okm); }
                xf = xf || of;
            }
        }
        if (lane == 31) { w_f[warp] = xf; w_k[warp] = xk; w_km[warp] = xkm; }
        __syncthreads();
        // exclusive value for this thread: lane-1's inclusive, then earlier warps, then the tile carry
        bool ef = __shfl_up_sync(0xffffffffu, xf, 1);
        u64 ek = __shfl_up_sync(0xffffffffu, xk, 1), ekm = __shfl_up_sync(0xffffffffu, xkm, 1);
        if (lane == 0) { ef = false; ek = 0; ekm = 0; }
        for (int w = warp - 1; w >= 0 && !ef; --w) {
            ek = umax(ek, w_k[w]);
            ekm = umax(ekm, w_km[w]);
            ef = w_f[w] != 0;
        }
        if (!ef) { ek = umax(ek, p.tcarry[2 * t]); ekm = umax(ekm, p.tcarry[2 * t + 1]); }
        // per record work
        DevAcc<R> A;
        A.zero();
        u64 runK = ek, runKM = ekm;
        int32_t cur = nv > 0 ? T.r[b] : INT_MIN;
        int32_t owner = (p.owner && cur >= 0 && cur < p.dev_ids) ? p.owner[cur] : -1;
        Walk wk;
        wk.init = false;
        for (int q = 0; q < nv; ++q) {
            const int i = b + q;
            const int32_t pr = i > 0 ? T.r[i - 1] : prev_r;
            const int32_t r = T.r[i];
            if (r != pr) {
                if (q > 0) A.flush(p, cur);
                A.zero();
                runK = runKM = 0;
                cur = r;
                owner = (p.owner && r >= 0 && r < p.dev_ids) ? p.owner[r] : -1;
                wk.init = false;
            }
            const u64 s = T.s[i], e = T.e[i];
            const bool kern = T.k[i] == 0;
#pragma unroll
            for (int j = 0; j < R; ++j) {
                const u64 ec = umin(umax(e, lo[j]), top[j]), sc = umin(umax(s, lo[j]), ec);
                const u64 ckm = umax(runKM, ec) - umax(runKM, sc);
                const u64 ck = kern ? umax(runK, ec) - umax(runK, sc) : 0ull;
                A.KM[j] += ckm;
                A.K[j] += ck;
                // clamped: kept in the region and its clipped end passes a + E
                const bool kept = s < e ? (umax(s, lo[j]) < umin(e, hi[j])) : (s >= lo[j] && s < hi[j]);
                A.clamp[j] += (kept && umin(e, hi[j]) > top[j]) ? 1u : 0u;
            }
            // K6: the new busy piece [max(run, s), max(run, e)) against the owner's offload records
            const u64 x = umax(runKM, s), y = umax(runKM, e);
            if (x < y) overlap_piece<R>(p, wk, owner, x, y, A);
            runKM = umax(runKM, e);
            if (kern) runK = umax(runK, e);
        }
        if (nv > 0) A.flush(p, cur);
    }
}

// ---------------------------------------------------------------------------
// per window: summaries in declaration order, metric trees, busy fraction
// ---------------------------------------------------------------------------
constexpr int kFT = 256;

__global__ void __launch_bounds__(kFT) reg_final(const __grid_constant__ RegParams p)
{
    __shared__ u128 scratch[33];
    const int j = blockIdx.x, tid = threadIdx.x;
    const u64 E = p.E[j];
    RegionResultDev *res = p.res + j;
    if (tid == 0) {
        res->status = E == 0 ? 2 : 0;   // HETEFF_ANALYSIS_ERROR: the region records no activity
        res->elapsed = E;
        res->host_mask = res->device_mask = res->busy_mask = 0;
    }
    u128 su = 0, suw = 0, muw = 0, sk = 0, mk = 0, mkm = 0, num = 0, den = 0;
    for (int32_t id = tid; id < p.host_ids; id += kFT) {
        if (!is_declared(p.host_decl, p.host_ids, p.n, id)) continue;
        const u64 *a = p.h_acc + ((size_t)j * p.host_ids + id) * 3;
        const u64 off = a[0], mpi = a[1], span = a[2];
        const u64 useful = span - off - mpi;
        const int32_t pos = decl_pos(p.host_decl, id);
        if (p.host_out) {
            u64 *o = p.host_out + ((size_t)j * p.n + pos) * 4;
            o[0] = useful; o[1] = off; o[2] = mpi; o[3] = span;
        }
        su += useful;
        const u128 uw = (u128)useful + off;
        suw += uw;
        if (uw > muw) muw = uw;
    }
    for (int32_t id = tid; id < p.dev_ids; id += kFT) {
        if (!is_declared(p.dev_decl, p.dev_ids, p.m, id)) continue;
        const u64 *a = p.d_acc + ((size_t)j * p.dev_ids + id) * 4;
        const u64 kk = a[0], km = a[1];
        const int32_t pos = decl_pos(p.dev_decl, id);
        if (p.dev_out) {
            u64 *o = p.dev_out + ((size_t)j * p.m + pos) * 4;
            o[0] = kk; o[1] = km - kk; o[2] = E - km; o[3] = a[2];
        }
        if (p.busy_out) p.busy_out[(size_t)j * p.m + pos] = a[3];
        sk += kk;
        if (kk > mk) mk = kk;
        if (km > mkm) mkm = km;
        const int32_t ow = p.owner ? p.owner[id] : -1;
        if (ow >= 0 && ow < p.host_ids && is_declared(p.host_decl, p.host_ids, p.n, ow)) {
            num += a[3];
            den += p.h_acc[((size_t)j * p.host_ids + ow) * 3 + 0];
        }
    }
    su = block_reduce128<false>(su, scratch, tid, kFT);
    suw = block_reduce128<false>(suw, scratch, tid, kFT);
    muw = block_reduce128<true>(muw, scratch, tid, kFT);
    sk = block_reduce128<false>(sk, scratch, tid, kFT);
    mk = block_reduce128<true>(mk, scratch, tid, kFT);
    mkm = block_reduce128<true>(mkm, scratch, tid, kFT);
    num = block_reduce128<false>(num, scratch, tid, kFT);
    den = block_reduce128<false>(den, scratch, tid, kFT);
    if (E == 0) return;
    metric_trees(res, p.n >= 1, p.m >= 1, E, p.n, p.m, su, suw, muw, sk, mk, mkm, tid);
    if (tid == 64 && den > 0) {
        res->busy_fraction = div_exact(num, den);
        res->busy_mask = 1u;
    }
}

}  // namespace reg

size_t region_tiles(int64_t dn) { return (size_t)((dn + reg::kDTile - 1) / reg::kDTile); }

static int grid_cap(int64_t g, int sms)
{
    if (g > (int64_t)sms * 8) g = (int64_t)sms * 8;
    return g < 1 ? 1 : (int)g;
}

template <int R>
static void phase1_r(const RegParams &p, int sms, cudaStream_t s)
{
    using namespace reg;
    const int64_t hw = (p.hn + 32 * kHI - 1) / (32 * kHI);
    reg_host<R><<<grid_cap((hw + kHT / 32 - 1) / (kHT / 32), sms), kHT, 0, s>>>(p);
    if (p.tiles > 0) {
        reg_dev_agg<<<grid_cap((p.tiles + 7) / 8, sms), 256, 0, s>>>(p);
        reg_dev_carry<<<1, 1024, 0, s>>>(p);
    }
    reg_E<<<p.R, 256, 0, s>>>(p);
}

template <int R>
static void phase2_r(const RegParams &p, int sms, cudaStream_t s)
{
    using namespace reg;
    if (p.tiles > 0) reg_dev<R><<<grid_cap(p.tiles, sms), kDT, 0, s>>>(p);
    reg_final<<<p.R, kFT, 0, s>>>(p);
}

static int sm_count()
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// phase 1: host CSR, host sums, device tile carries, E per window (p.E)
cudaError_t launch_regions_phase1(const RegParams &p, cudaStream_t s)
{
    const int sms = sm_count();
    reg::reg_hseg<<<(p.host_ids + 1 + 255) / 256, 256, 0, s>>>(p.hr, p.hn, p.host_ids, p.hseg);
    if (p.R <= 1) phase1_r<1>(p, sms, s);
    else if (p.R <= 4) phase1_r<4>(p, sms, s);
    else if (p.R <= 8) phase1_r<8>(p, sms, s);
    else phase1_r<16>(p, sms, s);
    return cudaGetLastError();
}

// phase 2 (p.wtop = window start + E filled in by the caller): device pass, finalize
cudaError_t launch_regions_phase2(const RegParams &p, cudaStream_t s)
{
    const int sms = sm_count();
    if (p.R <= 1) phase2_r<1>(p, sms, s);
    else if (p.R <= 4) phase2_r<4>(p, sms, s);
    else if (p.R <= 8) phase2_r<8>(p, sms, s);
    else phase2_r<16>(p, sms, s);
    return cudaGetLastError();
}

}  // namespace hb
