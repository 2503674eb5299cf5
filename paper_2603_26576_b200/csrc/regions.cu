// regions.cu -- K5/K6, EXTENSIONS beyond the reference (SURVEY.md section 8,
// rows a22/a23).
//
// K5 monitoring regions.  Region j is a window [a_j, b_j).  Its trace is the
// full trace with every record intersected with the window (intervals.py:
// 98-105 semantics) and shifted by -a_j; a zero-length record survives iff
// a_j <= s < b_j.  The region's report is the reference's compute_report
// (metrics.py:125-154) of that trace.
//
// K6 offload-wait / device-busy overlap per device g with owner rank p:
//   busy_j(g) = |offload(p) ∩ (kernel ∪ memory)(g) ∩ [a_j, a_j + E_j)|.
//
// Design: everything window-dependent is a POINT QUERY on window-independent
// prefix functions, so the trace is streamed a fixed number of times however
// many windows there are, and each window costs O(chunk) work per resource.
// For a resource with records sorted by start and a time t, let i*(t) be the
// number of its records starting before t and M(t) the max end over them.
//   host   F_k(t) = |∪ kind-k records ∩ [0,t)| = P_k(i*) - max(0, M_k(i*) - t)
//          (usable host records are disjoint, so only one can cross t), hence
//          offload_j = F_off(b) - F_off(a), mpi_j likewise, and
//          span_j = max(0, min(M(b), b) - a);
//   device with the running-max pieces [max(run,s), max(run,e)) of the main
//          kernel (disjoint, increasing, union = busy set), c_i their lengths:
//          G(t) = |busy ∩ [0,t)| = Σ_{i<i*} c_i - max(0, M(i*) - t)
//          (every record before i* starts before t, so busy ∩ [t,∞) = [t,M));
//          kernel_j = G_K(a+E) - G_K(a), kernel|memory_j = G_KM(a+E) - G_KM(a);
//          H(t) = |offload ∩ busy ∩ [0,t)| = Σ_{i<i*} o_i - |offload ∩ [t, M)|
//          with o_i = |offload ∩ piece_i| (a forward merge with the owner's
//          host records) and |offload ∩ [u,v)| = F_off(v) - F_off(u);
//          clamped_j = #{s < b, e > a+E} = #{s < b} - #{s <= a+E} +
//          #{s <= a+E < e} (the last term by a backward scan bounded by the
//          prefix max end).
// Prefix values are checkpointed at every chunk start (segmented scans over
// chunk aggregates), so a query is two binary searches plus a scan of at most
// one chunk.
//
// Kernels: reg_seg (CSR), rh_agg + scan (host checkpoints), rd_runagg + scan
// (device running-max carries, device-only E), rd_sums + scan (device U_K,
// U_KM, busy checkpoints), rh_query (per window x rank), reg_E, rd_query
// (per window x device), reg_final (summaries, metric trees, fractions).
#include <cuda_runtime.h>
#include <climits>
#include <cstdint>

#include "engine.cuh"
#include "exact.cuh"
#include "ptx.cuh"

namespace hb {
namespace reg {

constexpr int kHC = 256;             // host records per checkpoint chunk
#ifndef HB_REG_DT
#define HB_REG_DT 128
#endif
#ifndef HB_REG_STAGE
// staged offload intervals per tile.  Measured on C4 (region call 17.5 -> 16.0 ms; 640,
// 704, 832, 896 and 1024 all ~17.5 ms): likely because five ~39 KB CTAs fit the 196 KB
// shared-memory carveout, leaving ~60 KB of L1 for the staging loop's second read of the
// owner's host records
#define HB_REG_STAGE 768
#endif
constexpr int kDT = HB_REG_DT;       // device tile threads
#ifndef HB_REG_DI
#define HB_REG_DI 9   // C4 region call (ms): 7 -> 17.4, 9 -> 15.3, 11 -> 16.8, 13 -> 20.7
#endif
constexpr int kDI = HB_REG_DI;       // device records per thread (odd: conflict-free smem)
constexpr int kDTile = kDT * kDI;    // 1152 device records per tile (= checkpoint chunk)
constexpr int kST = 1024;            // scan block
constexpr int kSub = 16;             // device sub-checkpoint every kSub threads (kSub * kDI records)
constexpr int kSubs = kDT / kSub;    // sub-checkpoints per tile

__device__ __forceinline__ bool is_declared(const int32_t *decl, int32_t ids, int32_t n, int32_t r)
{
    if (r < 0 || r >= ids) return false;
    return decl ? (decl[r] >= 0) : (r < n);
}

__device__ __forceinline__ int32_t decl_pos(const int32_t *decl, int32_t r) { return decl ? decl[r] : r; }

__device__ __forceinline__ u64 sub0(u64 a, u64 b) { return a > b ? a - b : 0ull; }

// window of region j for host rank `id`: its own (per-rank regions) or the global one
__device__ __forceinline__ void host_window(const RegParams &p, int j, int32_t id, u64 &a, u64 &b)
{
    if (p.hwin) {
        const u64 *w = p.hwin + ((size_t)j * p.host_ids + id) * 2;
        a = w[0];
        b = umax(w[1], a);
    } else {
        a = p.wlo[j];
        b = p.whi[j];
    }
}

// window of region j for device `id`: its owner rank's (per-rank regions; none without
// an owner) or the global one
__device__ __forceinline__ void dev_window(const RegParams &p, int j, int32_t id, u64 &a, u64 &b)
{
    if (p.hwin) {
        const int32_t o = p.owner ? p.owner[id] : -1;
        if (o < 0 || o >= p.host_ids) { a = b = 0; return; }
        host_window(p, j, o, a, b);
    } else {
        a = p.wlo[j];
        b = p.whi[j];
    }
}

// first index in [lo, hi) with v[i] >= x  (lower) / > x (upper); v non-decreasing there
__device__ __forceinline__ int64_t lower_idx(const u64 *v, int64_t lo, int64_t hi, u64 x)
{
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(v + mid) < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ int64_t upper_idx(const u64 *v, int64_t lo, int64_t hi, u64 x)
{
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (__ldg(v + mid) <= x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// CSR: seg[id] = first record of dense id `id` (records grouped by ascending id)
__global__ void reg_seg(const int32_t *__restrict__ r, int64_t n, int32_t ids, int64_t *__restrict__ seg)
{
    const int32_t id = blockIdx.x * blockDim.x + threadIdx.x;
    if (id > ids) return;
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (r[mid] < id) lo = mid + 1;
        else hi = mid;
    }
    seg[id] = lo;
}

// ---------------------------------------------------------------------------
// segmented scan of chunk aggregates: agg[c] = {flag, NS sums, NM maxes} over
// the chunk's LAST segment; carry[c] = the same values over the part of chunk
// c's first segment that lies in earlier chunks (carry[C] = after the last)
// ---------------------------------------------------------------------------
template <int NS, int NM>
struct SAgg {
    bool f;
    u64 v[NS + NM];
};

template <int NS, int NM>
__device__ __forceinline__ SAgg<NS, NM> combine(const SAgg<NS, NM> &a, const SAgg<NS, NM> &b)   // a earlier
{
    if (b.f) return b;
    SAgg<NS, NM> r;
    r.f = a.f;
#pragma unroll
    for (int k = 0; k < NS; ++k) r.v[k] = a.v[k] + b.v[k];
#pragma unroll
    for (int k = NS; k < NS + NM; ++k) r.v[k] = umax(a.v[k], b.v[k]);
    return r;
}

template <int NS, int NM>
__device__ __forceinline__ SAgg<NS, NM> ident()
{
    SAgg<NS, NM> r;
    r.f = false;
#pragma unroll
    for (int k = 0; k < NS + NM; ++k) r.v[k] = 0;
    return r;
}

template <int NS, int NM>
__device__ __forceinline__ SAgg<NS, NM> shfl_up_agg(const SAgg<NS, NM> &x, int d)
{
    SAgg<NS, NM> r;
    r.f = __shfl_up_sync(0xffffffffu, x.f, d);
#pragma unroll
    for (int k = 0; k < NS + NM; ++k) r.v[k] = __shfl_up_sync(0xffffffffu, x.v[k], d);
    return r;
}

// block-wide exclusive segmented scan (blockDim.x threads, multiple of 32); `ws` >= 33 entries
template <int NS, int NM>
__device__ SAgg<NS, NM> block_seg_scan(const SAgg<NS, NM> &x, SAgg<NS, NM> *ws, SAgg<NS, NM> &total)
{
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    SAgg<NS, NM> inc = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const SAgg<NS, NM> o = shfl_up_agg(inc, d);
        if (lane >= d) inc = combine(o, inc);
    }
    if (lane == 31) ws[warp] = inc;
    __syncthreads();
    if (tid == 0) {
        SAgg<NS, NM> run = ident<NS, NM>();
        for (int w = 0; w < nw; ++w) {
            const SAgg<NS, NM> t = ws[w];
            ws[w] = run;
            run = combine(run, t);
        }
        ws[32] = run;
    }
    __syncthreads();
    SAgg<NS, NM> ex = shfl_up_agg(inc, 1);
    if (lane == 0) ex = ident<NS, NM>();
    const SAgg<NS, NM> r = combine(ws[warp], ex);
    total = ws[32];
    __syncthreads();
    return r;
}

template <int NS, int NM>
__device__ __forceinline__ SAgg<NS, NM> load_agg(const u64 *agg, int64_t c, int64_t C)
{
    constexpr int W = 1 + NS + NM;
    SAgg<NS, NM> a = ident<NS, NM>();
    if (c < C) {
        a.f = agg[c * W] != 0;
#pragma unroll
        for (int k = 0; k < NS + NM; ++k) a.v[k] = agg[c * W + 1 + k];
    }
    return a;
}

template <int NS, int NM>
__global__ void __launch_bounds__(kST) scan_a(const u64 *__restrict__ agg, int64_t C, u64 *__restrict__ tmp)
{
    __shared__ SAgg<NS, NM> ws[33];
    const int64_t c = (int64_t)blockIdx.x * kST + threadIdx.x;
    SAgg<NS, NM> total;
    block_seg_scan<NS, NM>(load_agg<NS, NM>(agg, c, C), ws, total);
    if (threadIdx.x == 0) {
        u64 *t = tmp + (size_t)blockIdx.x * 8;
        t[0] = total.f;
#pragma unroll
        for (int k = 0; k < NS + NM; ++k) t[1 + k] = total.v[k];
    }
}

template <int NS, int NM>
__global__ void __launch_bounds__(kST) scan_b(u64 *tmp, int64_t nb)
{
    __shared__ SAgg<NS, NM> ws[33];
    SAgg<NS, NM> carry = ident<NS, NM>();
    for (int64_t b0 = 0; b0 < nb; b0 += kST) {
        const int64_t b = b0 + threadIdx.x;
        SAgg<NS, NM> x = ident<NS, NM>();
        if (b < nb) {
            x.f = tmp[b * 8] != 0;
#pragma unroll
            for (int k = 0; k < NS + NM; ++k) x.v[k] = tmp[b * 8 + 1 + k];
        }
        SAgg<NS, NM> total;
        const SAgg<NS, NM> ex = combine(carry, block_seg_scan<NS, NM>(x, ws, total));
        if (b < nb) {
            tmp[b * 8] = ex.f;
#pragma unroll
            for (int k = 0; k < NS + NM; ++k) tmp[b * 8 + 1 + k] = ex.v[k];
        }
        carry = combine(carry, total);
    }
}

template <int NS, int NM>
__global__ void __launch_bounds__(kST) scan_c(const u64 *__restrict__ agg, int64_t C, const u64 *__restrict__ tmp,
                                              u64 *__restrict__ carry)
{
    __shared__ SAgg<NS, NM> ws[33];
    constexpr int V = NS + NM;
    const int64_t c = (int64_t)blockIdx.x * kST + threadIdx.x;
    const SAgg<NS, NM> x = load_agg<NS, NM>(agg, c, C);
    SAgg<NS, NM> total;
    SAgg<NS, NM> bc;
    bc.f = tmp[(size_t)blockIdx.x * 8] != 0;
#pragma unroll
    for (int k = 0; k < V; ++k) bc.v[k] = tmp[(size_t)blockIdx.x * 8 + 1 + k];
    const SAgg<NS, NM> ex = combine(bc, block_seg_scan<NS, NM>(x, ws, total));
    if (c < C) {
#pragma unroll
        for (int k = 0; k < V; ++k) carry[c * V + k] = ex.v[k];
    }
    if (c == C - 1) {
        const SAgg<NS, NM> fin = combine(ex, x);
#pragma unroll
        for (int k = 0; k < V; ++k) carry[(c + 1) * V + k] = fin.v[k];
    }
}

template <int NS, int NM>
static void seg_scan(const u64 *agg, int64_t C, u64 *tmp, u64 *carry, cudaStream_t s)
{
    if (C <= 0) return;
    const int64_t nb = (C + kST - 1) / kST;
    scan_a<NS, NM><<<(unsigned)nb, kST, 0, s>>>(agg, C, tmp);
    scan_b<NS, NM><<<1, kST, 0, s>>>(tmp, nb);
    scan_c<NS, NM><<<(unsigned)nb, kST, 0, s>>>(agg, C, tmp, carry);
}

// ---------------------------------------------------------------------------
// host: chunk aggregates over the last segment: offload / mpi durations and
// max ends (all records, offload, mpi)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) rh_agg(const __grid_constant__ RegParams p)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * 8;
    for (int64_t c = (blockIdx.x * 256ll + threadIdx.x) >> 5; c < p.hchunks; c += warps) {
        const int64_t b = c * kHC, e = umin((u64)(b + kHC), (u64)p.hn);
        int64_t last = -1;
        for (int64_t i = b + lane; i < e; i += 32)
            if (i == 0 || __ldg(p.hr + i) != __ldg(p.hr + i - 1)) last = i;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const int64_t o = __shfl_xor_sync(0xffffffffu, last, d);
            last = o > last ? o : last;
        }
        u64 so = 0, sm = 0, ma = 0, mo = 0, mm = 0;
        for (int64_t i = (last < 0 ? b : last) + lane; i < e; i += 32) {
            const u64 s = __ldg(p.hs + i), en = __ldg(p.he + i);
            const uint8_t k = __ldg(p.hk + i);
            const u64 d = en > s ? en - s : 0;
            ma = umax(ma, en);
            if (k == 1) { so += d; mo = umax(mo, en); }
            if (k == 2) { sm += d; mm = umax(mm, en); }
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            so += __shfl_xor_sync(0xffffffffu, so, d);
            sm += __shfl_xor_sync(0xffffffffu, sm, d);
            ma = umax(ma, __shfl_xor_sync(0xffffffffu, ma, d));
            mo = umax(mo, __shfl_xor_sync(0xffffffffu, mo, d));
            mm = umax(mm, __shfl_xor_sync(0xffffffffu, mm, d));
        }
        if (lane == 0) {
            u64 *a = p.hagg + c * 6;
            a[0] = last >= 0; a[1] = so; a[2] = sm; a[3] = ma; a[4] = mo; a[5] = mm;
        }
    }
}

// prefix values of host rank `id` over its records starting before t
struct HostQ {
    u64 so, sm, ma, mo, mm;
};

__device__ HostQ host_query(const RegParams &p, int32_t id, u64 t)
{
    const int64_t b0 = p.hseg[id], b1 = p.hseg[id + 1];
    const int64_t is = lower_idx(p.hs, b0, b1, t);
    const int64_t c = is / kHC;
    int64_t cs = c * kHC;
    HostQ q{0, 0, 0, 0, 0};
    if (cs > b0) {
        const u64 *k = p.hck + c * 5;
        q.so = k[0]; q.sm = k[1]; q.ma = k[2]; q.mo = k[3]; q.mm = k[4];
    } else {
        cs = b0;
    }
    for (int64_t i = cs; i < is; ++i) {
        const u64 s = __ldg(p.hs + i), e = __ldg(p.he + i);
        const uint8_t k = __ldg(p.hk + i);
        const u64 d = e > s ? e - s : 0;
        q.ma = umax(q.ma, e);
        if (k == 1) { q.so += d; q.mo = umax(q.mo, e); }
        if (k == 2) { q.sm += d; q.mm = umax(q.mm, e); }
    }
    return q;
}

// |offload(rank id) ∩ [0, t)|
__device__ __forceinline__ u64 offload_before(const RegParams &p, int32_t id, u64 t)
{
    const HostQ q = host_query(p, id, t);
    return q.so - sub0(q.mo, t);
}

// per (window, rank): offload, mpi, span of the region trace
__global__ void __launch_bounds__(128) rh_query(const __grid_constant__ RegParams p)
{
    const int64_t x = blockIdx.x * 128ll + threadIdx.x;
    if (x >= (int64_t)p.R * p.host_ids) return;
    const int j = (int)(x / p.host_ids);
    const int32_t id = (int32_t)(x % p.host_ids);
    u64 a, b;
    host_window(p, j, id, a, b);
    u64 off = 0, mpi = 0, span = 0;
    if (a < b) {
        const HostQ qa = host_query(p, id, a), qb = host_query(p, id, b);
        off = (qb.so - sub0(qb.mo, b)) - (qa.so - sub0(qa.mo, a));
        mpi = (qb.sm - sub0(qb.mm, b)) - (qa.sm - sub0(qa.mm, a));
        span = sub0(umin(qb.ma, b), a);
    }
    u64 *o = p.h_acc + ((size_t)j * p.host_ids + id) * 3;
    o[0] = off;
    o[1] = mpi;
    o[2] = span;
}

// ---------------------------------------------------------------------------
// device: running-max aggregates per tile (+ device-only E candidates)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) rd_runagg(const __grid_constant__ RegParams p)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * 8;
    for (int64_t t = (blockIdx.x * 256ll + threadIdx.x) >> 5; t < p.tiles; t += warps) {
        const int64_t b = t * kDTile, e = umin((u64)(b + kDTile), (u64)p.dn);
        // one pass, fixed trip (loads in flight): per lane the max ends over the tile, over
        // the tile's first device, and the tile's last segment start
        const int32_t r0 = __ldg(p.dr + b);
        int64_t last = -1;
        u64 mk = 0, mkm = 0, e0 = 0;
#pragma unroll 9
        for (int q = 0; q < kDTile / 32; ++q) {
            const int64_t i = b + q * 32 + lane;
            if (i < e) {
                const int32_t r = __ldg(p.dr + i);
                const u64 en = __ldg(p.de + i);
                const bool kern = __ldg(p.dk + i) == 0;
                if (i == 0 || r != __ldg(p.dr + i - 1)) last = i;
                mkm = umax(mkm, en);
                if (kern) mk = umax(mk, en);
                if (r == r0) e0 = umax(e0, en);
            }
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            const int64_t o = __shfl_xor_sync(0xffffffffu, last, d);
            last = o > last ? o : last;
        }
        if (last >= 0) {
            // a device starts in the tile (rare): the aggregate covers its last segment only
            mk = 0; mkm = 0;
            for (int64_t i = last + lane; i < e; i += 32) {
                const u64 en = __ldg(p.de + i);
                mkm = umax(mkm, en);
                if (__ldg(p.dk + i) == 0) mk = umax(mk, en);
            }
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            mk = umax(mk, __shfl_xor_sync(0xffffffffu, mk, d));
            mkm = umax(mkm, __shfl_xor_sync(0xffffffffu, mkm, d));
            e0 = umax(e0, __shfl_xor_sync(0xffffffffu, e0, d));
        }
        if (lane == 0) {
            u64 *a = p.dagg + t * 3;
            a[0] = last >= 0; a[1] = mk; a[2] = mkm;
            // host index range of the owner's records overlapping [first start, e0)
            int64_t q0 = 0, q1 = 0;
            const int32_t ow = (p.owner && r0 >= 0 && r0 < p.dev_ids) ? p.owner[r0] : -1;
            if (ow >= 0 && ow < p.host_ids) {
                const int64_t h0 = p.hseg[ow], h1 = p.hseg[ow + 1];
                q0 = upper_idx(p.hs, h0, h1, __ldg(p.ds + b)) - 1;
                while (q0 > h0 && __ldg(p.hs + q0) == __ldg(p.he + q0)) --q0;
                if (q0 < h0) q0 = h0;
                q1 = lower_idx(p.hs, q0, h1, e0);
            }
            p.tstage[2 * t] = q0;
            p.tstage[2 * t + 1] = q1;
        }
    }
}

// device-only traces: E_j = max clipped end of the region's records
__global__ void __launch_bounds__(256) rd_dmax(const __grid_constant__ RegParams p)
{
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * 8;
    for (int64_t t = (blockIdx.x * 256ll + threadIdx.x) >> 5; t < p.tiles; t += warps) {
        const int64_t b = t * kDTile, e = umin((u64)(b + kDTile), (u64)p.dn);
        for (int j = 0; j < p.R; ++j) {
            const u64 a = p.wlo[j], w = p.whi[j];
            u64 mx = 0;
            for (int64_t i = b + lane; i < e; i += 32) {
                const u64 s = __ldg(p.ds + i), en = __ldg(p.de + i);
                if (s < en) {
                    const u64 cs = umax(s, a), ce = umin(en, w);
                    if (cs < ce) mx = umax(mx, ce - a);
                } else if (s == en && s >= a && s < w) {
                    mx = umax(mx, s - a);
                }
            }
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) mx = umax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
            if (lane == 0 && mx) red_max(p.dmax + j, mx);
        }
    }
}

// ---------------------------------------------------------------------------
// overlap walk: |offload(owner) ∩ [x, y)| for pieces of one device in
// increasing order, merged forward through the owner's host records
// ---------------------------------------------------------------------------
struct Walk {
    int64_t q, h0, h1;
    bool init;
};

// last record of the owner starting at or before x, stepped back over
// zero-length records (a usable record containing x is the last USABLE one);
// gallops forward from `lo`, a known lower bound
__device__ __forceinline__ int64_t walk_locate(const RegParams &p, int64_t lo, int64_t h0, int64_t h1, u64 x)
{
    int64_t step = 1, a = lo;
    while (a + step < h1 && __ldg(p.hs + a + step) <= x) { a += step; step <<= 1; }
    const int64_t b = a + step < h1 ? a + step : h1;
    int64_t q = upper_idx(p.hs, a, b, x) - 1;
    while (q > h0 && __ldg(p.hs + q) == __ldg(p.he + q)) --q;
    return q < h0 ? h0 : q;
}

__device__ __forceinline__ u64 walk_overlap(const RegParams &p, Walk &w, u64 x, u64 y)
{
    u64 ov = 0;
    while (w.q < w.h1) {
        const u64 hs = __ldg(p.hs + w.q);
        if (hs >= y) break;
        const u64 he = __ldg(p.he + w.q);
        if (__ldg(p.hk + w.q) == 1 && hs < he) {
            const u64 u = umax(hs, x), v = umin(he, y);
            if (u < v) ov += v - u;
        }
        if (he > y) break;                 // continues into the next piece
        ++w.q;
    }
    return ov;
}

// ---------------------------------------------------------------------------
// device: per tile U_K, U_KM and busy sums over the last segment
// ---------------------------------------------------------------------------
struct DevTile {
    u64 s[kDTile];
    u64 e[kDTile];
    int32_t r[kDTile];
    uint8_t k[kDTile];
};

// the owner's OFFLOAD intervals overlapping a tile's time range, staged in
// shared memory (sorted, disjoint: ends increase too) so the per-thread merges
// run out of smem instead of chains of dependent global loads
constexpr int kStage = HB_REG_STAGE;

struct OffStage {
    u64 s[kStage];
    u64 e[kStage];
    int32_t count;       // -1: not staged (range too large / no owner)
    int32_t dev;         // the device whose owner was staged
};

// |A ∩ [x, y)| over staged disjoint intervals, cursor `q` moving forward
__device__ __forceinline__ u64 stage_overlap(const OffStage &S, int &q, u64 x, u64 y)
{
    u64 ov = 0;
    while (q < S.count && S.e[q] <= x) ++q;
    int k = q;
    while (k < S.count && S.s[k] < y) {
        const u64 u = umax(S.s[k], x), v = umin(S.e[k], y);
        if (u < v) ov += v - u;
        if (S.e[k] > y) break;
        ++k;
    }
    q = k;
    return ov;
}

__device__ __forceinline__ int stage_locate(const OffStage &S, u64 x)   // first staged interval with end > x
{
    int lo = 0, hi = S.count;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (S.e[mid] <= x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(kDT) rd_sums(const __grid_constant__ RegParams p)
{
    __shared__ DevTile T;
    __shared__ OffStage S;
    __shared__ SAgg<0, 2> ws2[33];
    __shared__ SAgg<3, 0> ws3[33];
    __shared__ int64_t s_q0, s_q1;
    __shared__ u64 s_wmax[kDT / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int64_t t = blockIdx.x; t < p.tiles; t += gridDim.x) {
        const int64_t base = t * kDTile;
        const int cnt = (int)umin((u64)kDTile, (u64)(p.dn - base));
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kDI; ++k) {   // every load of the tile in flight at once
            const int i = tid + k * kDT;
            if (i < cnt) {
                T.s[i] = __ldcs(p.ds + base + i);
                T.e[i] = __ldcs(p.de + base + i);
                T.r[i] = __ldcs(p.dr + base + i);
                T.k[i] = __ldcs(p.dk + base + i);
            }
        }
        const int32_t prev_r = base > 0 ? __ldg(p.dr + base - 1) : INT_MIN;
        __syncthreads();
        // thread aggregate: segment flag + last-segment max ends; max end of the tile's first device
        const int b = tid * kDI;
        const int nv = cnt - b < 0 ? 0 : (cnt - b < kDI ? cnt - b : kDI);
        const int32_t r0 = T.r[0];
        SAgg<0, 2> ta = ident<0, 2>();
        for (int q = 0; q < nv; ++q) {
            const int i = b + q;
            const int32_t pr = i > 0 ? T.r[i - 1] : prev_r;
            if (T.r[i] != pr) { ta.f = true; ta.v[0] = 0; ta.v[1] = 0; }
            ta.v[1] = umax(ta.v[1], T.e[i]);
            if (T.k[i] == 0) ta.v[0] = umax(ta.v[0], T.e[i]);
        }
        SAgg<0, 2> tot2;
        SAgg<0, 2> ex = block_seg_scan<0, 2>(ta, ws2, tot2);
        const SAgg<0, 2> ex_in = ex;       // in-tile part (sub-checkpoint)
        if (!ex.f) { ex.v[0] = umax(ex.v[0], p.drun[2 * t]); ex.v[1] = umax(ex.v[1], p.drun[2 * t + 1]); }
        // stage the first device's owner offload intervals over [first start, its max end)
        if (tid == 0) {
            S.count = -1;
            S.dev = r0;
            const int64_t q0 = p.tstage[2 * t], q1 = p.tstage[2 * t + 1];
            s_q0 = q0;
            s_q1 = q1;
            if (q1 > q0 && q1 - q0 <= 3 * kStage) S.count = 0;
        }
        __syncthreads();
        if (S.count == 0) {   // order-preserving compaction of the offload records: one block scan
            const int64_t q0 = s_q0, n = s_q1 - s_q0;
            const int64_t per = (n + kDT - 1) / kDT;
            const int64_t a0 = q0 + umin((u64)(tid * per), (u64)n), a1 = q0 + umin((u64)((tid + 1) * per), (u64)n);
            uint32_t c = 0;
            // every offload record is staged (zero-length ones contribute nothing and keep the
            // staged ends non-decreasing), so the count reads one byte per record
            for (int64_t i = a0; i < a1; ++i) c += __ldg(p.hk + i) == 1;
            uint32_t inc = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += o;
            }
            if (lane == 31) s_wmax[warp] = inc;
            __syncthreads();
            uint32_t pos = inc - c, all = 0;
            for (int w = 0; w < kDT / 32; ++w) {
                const uint32_t cw = (uint32_t)s_wmax[w];
                if (w < warp) pos += cw;
                all += cw;
            }
            if (all <= (uint32_t)kStage) {
                for (int64_t i = a0; i < a1; ++i) {
                    const u64 hs = __ldg(p.hs + i), he = __ldg(p.he + i);
                    if (__ldg(p.hk + i) == 1) { S.s[pos] = hs; S.e[pos] = he; ++pos; }
                }
            }
            __syncthreads();
            if (tid == 0) S.count = all <= (uint32_t)kStage ? (int32_t)all : -1;
        }
        __syncthreads();
        // per record: piece lengths and busy overlap; sums over the thread's last segment
        u64 runK = ex.v[0], runKM = ex.v[1];
        SAgg<3, 0> sa = ident<3, 0>();
        int32_t cur = nv > 0 ? T.r[b] : INT_MIN;
        int32_t owner = (p.owner && cur >= 0 && cur < p.dev_ids) ? p.owner[cur] : -1;
        Walk wk;
        wk.init = false;
        // cursor into the staged intervals, located ONCE per thread before the record loop
        // (every lane together): the thread's first start is <= every piece start x of
        // the first device, and stage_overlap moves the cursor forward from there
        int sq = (S.count > 0 && nv > 0 && cur == S.dev) ? stage_locate(S, T.s[b]) : 0;
        // contiguous pieces (a piece starting where the previous one ended: every record
        // under overlapping streams) merge into one range before the staged walk -- the
        // thread's sum of |offload ∩ piece| is |offload ∩ union|
        u64 px = 0, py = 0;
        bool pend = false;
        for (int q = 0; q < nv; ++q) {
            const int i = b + q;
            const int32_t pr = i > 0 ? T.r[i - 1] : prev_r;
            const int32_t r = T.r[i];
            if (r != pr) {
                if (pend) { sa.v[2] += stage_overlap(S, sq, px, py); pend = false; }
                sa = ident<3, 0>();
                sa.f = true;
                runK = runKM = 0;
                cur = r;
                owner = (p.owner && r >= 0 && r < p.dev_ids) ? p.owner[r] : -1;
                wk.init = false;
            }
            const u64 s = T.s[i], e = T.e[i];
            const u64 x = umax(runKM, s), y = umax(runKM, e);
            sa.v[1] += y - x;
            if (T.k[i] == 0) sa.v[0] += umax(runK, e) - umax(runK, s);
            if (x < y && owner >= 0 && owner < p.host_ids) {
                if (S.count >= 0 && cur == S.dev) {
                    if (pend && x == py) {
                        py = y;
                    } else {
                        if (pend) sa.v[2] += stage_overlap(S, sq, px, py);
                        px = x;
                        py = y;
                        pend = true;
                    }
                } else {
                    if (!wk.init) {
                        wk.h0 = p.hseg[owner];
                        wk.h1 = p.hseg[owner + 1];
                        wk.q = wk.h1 > wk.h0 ? walk_locate(p, wk.h0, wk.h0, wk.h1, x) : wk.h0;
                        wk.init = true;
                    }
                    sa.v[2] += walk_overlap(p, wk, x, y);
                }
            }
            runKM = umax(runKM, e);
            if (T.k[i] == 0) runK = umax(runK, e);
        }
        if (pend) sa.v[2] += stage_overlap(S, sq, px, py);
        SAgg<3, 0> tot3;
        const SAgg<3, 0> ex3 = block_seg_scan<3, 0>(sa, ws3, tot3);
        if (tid % kSub == 0) {   // in-tile prefix at this thread's first record: f, U_K, U_KM, busy, f, max K, max KM
            u64 *c = p.dsub + (t * kSubs + tid / kSub) * 8;
            c[0] = ex3.f; c[1] = ex3.v[0]; c[2] = ex3.v[1]; c[3] = ex3.v[2];
            c[4] = ex_in.f; c[5] = ex_in.v[0]; c[6] = ex_in.v[1];
        }
        if (tid == 0) {
            u64 *a = p.dsum + t * 4;
            a[0] = p.dagg[3 * t];    // the tile's segment flag
            a[1] = tot3.v[0]; a[2] = tot3.v[1]; a[3] = tot3.v[2];
        }
    }
}

// E_j: max span over declared ranks, or the device-only maximum
__global__ void __launch_bounds__(256) reg_E(const __grid_constant__ RegParams p)
{
    const int j = blockIdx.x;
    u64 mx = 0;
    if (p.n >= 1) {
        for (int32_t id = threadIdx.x; id < p.host_ids; id += 256)
            if (is_declared(p.host_decl, p.host_ids, p.n, id))
                mx = umax(mx, p.h_acc[((size_t)j * p.host_ids + id) * 3 + 2]);
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
// device queries: G_K, G_KM and H at t, per (window, device)
// ---------------------------------------------------------------------------
struct DevQ {
    u64 pk, pkm, hp, mk, mkm;
};

__device__ DevQ dev_query(const RegParams &p, int64_t d0, int64_t d1, int32_t owner, u64 t)
{
    const int64_t is = lower_idx(p.ds, d0, d1, t);
    const int64_t c = is / kDTile;
    const int64_t sub = (is - c * kDTile) / (kSub * kDI);
    int64_t cs = c * kDTile + sub * (kSub * kDI);
    DevQ q{0, 0, 0, 0, 0};
    if (cs > d0 && c < p.tiles) {
        const u64 *x = p.dsub + (c * kSubs + sub) * 8;
        if (x[0]) { q.pk = x[1]; q.pkm = x[2]; q.hp = x[3]; }
        else { q.pk = p.dck[3 * c] + x[1]; q.pkm = p.dck[3 * c + 1] + x[2]; q.hp = p.dck[3 * c + 2] + x[3]; }
        if (x[4]) { q.mk = x[5]; q.mkm = x[6]; }
        else { q.mk = umax(p.drun[2 * c], x[5]); q.mkm = umax(p.drun[2 * c + 1], x[6]); }
    } else if (cs > d0) {   // past the last tile: the final carries
        q.pk = p.dck[3 * c]; q.pkm = p.dck[3 * c + 1]; q.hp = p.dck[3 * c + 2];
        q.mk = p.drun[2 * c]; q.mkm = p.drun[2 * c + 1];
    } else {
        cs = d0;
    }
    Walk wk;
    wk.init = false;
    const bool own = owner >= 0 && owner < p.host_ids;
    for (int64_t i = cs; i < is; ++i) {
        const u64 s = __ldg(p.ds + i), e = __ldg(p.de + i);
        const bool kern = __ldg(p.dk + i) == 0;
        const u64 x = umax(q.mkm, s), y = umax(q.mkm, e);
        q.pkm += y - x;
        if (kern) q.pk += umax(q.mk, e) - umax(q.mk, s);
        if (x < y && own) {
            if (!wk.init) {
                wk.h0 = p.hseg[owner];
                wk.h1 = p.hseg[owner + 1];
                wk.q = wk.h1 > wk.h0 ? walk_locate(p, wk.h0, wk.h0, wk.h1, x) : wk.h0;
                wk.init = true;
            }
            q.hp += walk_overlap(p, wk, x, y);
        }
        q.mkm = umax(q.mkm, e);
        if (kern) q.mk = umax(q.mk, e);
    }
    return q;
}

__global__ void __launch_bounds__(128) rd_query(const __grid_constant__ RegParams p)
{
    const int64_t x = blockIdx.x * 128ll + threadIdx.x;
    if (x >= (int64_t)p.R * p.dev_ids) return;
    const int j = (int)(x / p.dev_ids);
    const int32_t id = (int32_t)(x % p.dev_ids);
    u64 lo, b;
    dev_window(p, j, id, lo, b);
    // the region's clamp end in trace time: window start + E_j (E_j <= b - lo for global
    // windows; a per-rank window may be shorter than the longest rank's region)
    const u64 E = p.E[j];
    const u64 top = E > b - lo ? b : lo + E;
    u64 K = 0, KM = 0, clamp = 0, busy = 0;
    if (top > lo) {
        const int64_t d0 = p.dseg[id], d1 = p.dseg[id + 1];
        const int32_t owner = p.owner ? p.owner[id] : -1;
        const bool own = owner >= 0 && owner < p.host_ids;
        const DevQ qa = dev_query(p, d0, d1, owner, lo), qt = dev_query(p, d0, d1, owner, top);
        K = (qt.pk - sub0(qt.mk, top)) - (qa.pk - sub0(qa.mk, lo));
        KM = (qt.pkm - sub0(qt.mkm, top)) - (qa.pkm - sub0(qa.mkm, lo));
        if (own) {   // H(t) = hp - |offload ∩ [t, M)|
            const u64 ht =
                qt.hp - (qt.mkm > top ? offload_before(p, owner, qt.mkm) - offload_before(p, owner, top) : 0);
            const u64 ha = qa.hp - (qa.mkm > lo ? offload_before(p, owner, qa.mkm) - offload_before(p, owner, lo) : 0);
            busy = ht - ha;
        }
        if (top < b) {   // clamped = #{s < b} - #{s <= top} + #{s <= top < e}
            const int64_t nb = lower_idx(p.ds, d0, d1, b) - d0;
            const int64_t ub = upper_idx(p.ds, d0, d1, top);
            int64_t strad = 0;
            int64_t idx = ub - 1;
            while (idx >= d0) {
                const int64_t c = idx / kDTile;
                const int64_t ts = c * kDTile > d0 ? c * kDTile : d0;
                for (int64_t i = ts; i <= idx; ++i) strad += __ldg(p.de + i) > top;
                if (ts == d0 || p.drun[2 * c + 1] <= top) break;   // nothing earlier ends past top
                idx = ts - 1;
            }
            clamp = (u64)(nb - (ub - d0) + strad);
        }
    }
    u64 *o = p.d_acc + ((size_t)j * p.dev_ids + id) * 4;
    o[0] = K;
    o[1] = KM;
    o[2] = clamp;
    o[3] = busy;
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
size_t region_subs() { return (size_t)reg::kSubs; }
size_t region_hchunks(int64_t hn) { return (size_t)((hn + reg::kHC - 1) / reg::kHC); }

static int grid_cap(int64_t g, int sms, int per_sm)
{
    if (g > (int64_t)sms * per_sm) g = (int64_t)sms * per_sm;
    return g < 1 ? 1 : (int)g;
}

static int sm_count()
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

// window-independent checkpoints (once per call, whatever the window count)
cudaError_t launch_regions_prepare(const RegParams &p, cudaStream_t s)
{
    using namespace reg;
    const int sms = sm_count();
    reg_seg<<<(p.host_ids + 1 + 255) / 256, 256, 0, s>>>(p.hr, p.hn, p.host_ids, p.hseg);
    reg_seg<<<(p.dev_ids + 1 + 255) / 256, 256, 0, s>>>(p.dr, p.dn, p.dev_ids, p.dseg);
    if (p.hchunks > 0) {
        rh_agg<<<grid_cap((p.hchunks + 7) / 8, sms, 8), 256, 0, s>>>(p);
        seg_scan<2, 3>(p.hagg, p.hchunks, p.scan_tmp, p.hck, s);
    }
    if (p.tiles > 0) {
        rd_runagg<<<grid_cap((p.tiles + 7) / 8, sms, 8), 256, 0, s>>>(p);
        seg_scan<0, 2>(p.dagg, p.tiles, p.scan_tmp, p.drun, s);
        rd_sums<<<grid_cap(p.tiles, sms, kDT <= 128 ? 5 : 3), kDT, 0, s>>>(p);
        seg_scan<3, 0>(p.dsum, p.tiles, p.scan_tmp, p.dck, s);
    }
    return cudaGetLastError();
}

// phase 1 (per pass of <= kMaxWindows windows): host queries, E per window
cudaError_t launch_regions_phase1(const RegParams &p, cudaStream_t s)
{
    using namespace reg;
    const int sms = sm_count();
    // device-only traces: E from the devices (per-rank regions: no rank owns a device -> E = 0)
    if (p.n == 0 && p.tiles > 0 && !p.hwin) rd_dmax<<<grid_cap((p.tiles + 7) / 8, sms, 8), 256, 0, s>>>(p);
    const int64_t hq = (int64_t)p.R * p.host_ids;
    if (hq > 0) rh_query<<<(unsigned)((hq + 127) / 128), 128, 0, s>>>(p);
    reg_E<<<p.R, 256, 0, s>>>(p);
    return cudaGetLastError();
}

// phase 2 (after phase 1 in stream order: E per window in p.E): device queries, finalize
cudaError_t launch_regions_phase2(const RegParams &p, cudaStream_t s)
{
    using namespace reg;
    const int64_t dq = (int64_t)p.R * p.dev_ids;
    if (dq > 0) rd_query<<<(unsigned)((dq + 127) / 128), 128, 0, s>>>(p);
    reg_final<<<p.R, kFT, 0, s>>>(p);
    return cudaGetLastError();
}

}  // namespace hb
