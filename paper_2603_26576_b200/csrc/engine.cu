// engine.cu -- the B200 analysis kernel for heteff's hot path.
//
// One persistent kernel turns the packed host + device record SoA into every
// per-rank / per-device summary, all validation findings and both metric
// trees (reference: compute_report, metrics.py:125-154).  Structure:
//
//  * Tiles of kTile=4352 records (17 per compute thread), host tiles first,
//    then device tiles, claimed in order through one global counter.
//  * A producer warp streams each tile HBM -> shared memory with 1-D TMA bulk
//    copies (cp.async.bulk, evict-first) into a 2-stage ring completed on
//    mbarriers; 8 compute warps pull their 17 records (blocked, odd stride =
//    bank-conflict free) into registers.  Every record byte is read once.
//  * The reference's device pipeline flatten/intersect/subtract/complement
//    (intervals.py:40-105, summarize.py:119-132) reduces to a segmented
//    running-max scan over start-sorted records:
//        c_i = max(0, min(e_i,E) - max(s_i, run_i)),  run_i = max earlier end
//    once over kernel records (U_K) and once over all records (U_KM):
//        d_kernel = U_K, d_memory = U_KM - U_K, d_idle = E - U_KM.
//    The host overlap check (model.py:203-215) is the same scan over ends.
//  * The scan carry across tiles is a decoupled look-back (32-wide window,
//    epoch-tagged flags, release/acquire).  Contributions are computed first
//    with the tile-local carry; after the look-back only the prefix of the
//    tile's head segment with max(s, run) < carry is corrected, so the
//    look-back latency overlaps the per-record work.
//  * Per-resource totals leave through warp-level segmented reductions and
//    one L2 reduction (red.add / red.max) per (segment, warp).
//  * Device tiles need E (= max host end, summarize.py:88-89): the producer
//    warp of the first device tile waits for the host tiles (all claimed
//    earlier, so no deadlock) -- no second launch.
//  * The last CTA to finish runs the finalize: summaries in declaration
//    order, the two metric trees with exactly rounded u128/u128 -> f64
//    divisions (Python int/int semantics), status, and resets the workspace.
#include <cuda_runtime.h>
#include <cstdint>
#include <climits>

#include "engine.cuh"
#include "ptx.cuh"

namespace hb {

struct StageSmem {
    u64 s[kTile];
    u64 e[kTile];
    int32_t r[kTile];
    uint8_t k[kTile];
};

struct Ctrl {
    uint64_t full[kStages];
    int64_t tile[kStages];
    int32_t cnt[kStages];
    int32_t has_prev[kStages];
    int32_t prev_res[kStages];
    int32_t pad0;
    u64 prev_start[kStages];
    // per-tile exchange
    int32_t w_flag[kComputeWarps];
    u64 w_v0[kComputeWarps];
    u64 w_v1[kComputeWarps];
    u64 w_max[kComputeWarps];
    u64 carry0[kStages], carry1[kStages];
    u64 E[kStages];
    int32_t head_cont[kStages];
    int32_t is_last;
};

size_t analyze_smem_bytes() { return sizeof(StageSmem) * kStages + sizeof(Ctrl) + 128; }

// -------------------------------------------------------------------------
// small helpers
// -------------------------------------------------------------------------
__device__ __forceinline__ bool declared(const int32_t *decl, int32_t ids, int32_t n, int32_t r)
{
    if (r < 0 || r >= ids) return false;
    return decl ? (__ldg(decl + r) >= 0) : (r < n);
}

__device__ __forceinline__ void push(const Params &p, int cls, int64_t gi)
{
    u64 idx = atomicAdd(&p.g->counts[cls], 1ull);
    if ((int64_t)idx < p.cap) p.lists[cls][idx] = gi;
}

__device__ __forceinline__ void contract(const Params &p, unsigned flag, int64_t gi)
{
    atomicOr(&p.g->contract_flags, flag);
    atomicMin(&p.g->contract_index, (long long)gi);
}

// B2: all kThreads threads, reached from the producer and the compute branch
__device__ __forceinline__ void bar_b2() { asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory"); }

__device__ __forceinline__ u64 warp_max(u64 v)
{
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = umax(v, __shfl_xor_sync(0xffffffffu, v, d));
    return v;
}

// -------------------------------------------------------------------------
// producer: claim a tile and stream it into a stage
// -------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ uint32_t bulk_bytes(int cnt, bool tma)
{
    return tma ? (((uint32_t)cnt * (uint32_t)sizeof(T)) & ~15u) : 0u;
}

// elements not covered by the 16-byte bulk copy (all of them without TMA)
template <typename T>
__device__ __forceinline__ void copy_tail(T *dst, const T *src, int cnt, bool tma, int lane)
{
    const int first = (int)(bulk_bytes<T>(cnt, tma) / sizeof(T));
    for (int i = first + lane; i < cnt; i += 32) dst[i] = src[i];
}

template <typename T>
__device__ __forceinline__ void issue_bulk(T *dst, const T *src, int cnt, bool tma, uint64_t *bar, uint64_t pol)
{
    const uint32_t b = bulk_bytes<T>(cnt, tma);
    if (b) tma_load_1d(dst, src, b, bar, pol);
}

__device__ void produce(const Params &p, StageSmem *stages, Ctrl *c, int st, int lane, uint64_t pol)
{
    int64_t t = 0;
    if (lane == 0) t = (int64_t)atomicAdd(&p.g->tile_counter, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    const int64_t total = p.host_tiles + p.dev_tiles;
    if (t >= total) {
        if (lane == 0) {
            c->tile[st] = -1;
            mbar_arrive(&c->full[st]);
        }
        return;
    }
    const bool dev = t >= p.host_tiles;
    const int64_t lt = dev ? t - p.host_tiles : t;
    const int64_t base = lt * kTile;
    const int64_t n = dev ? p.dn : p.hn;
    const int cnt = (int)((n - base) < kTile ? (n - base) : kTile);
    const u64 *S = (dev ? p.ds : p.hs) + base;
    const u64 *E = (dev ? p.de : p.he) + base;
    const int32_t *R = (dev ? p.dr : p.hr) + base;
    const uint8_t *K = (dev ? p.dk : p.hk) + base;
    StageSmem &sm = stages[st];
    const bool tma = p.use_tma != 0;
    if (lane == 0) {
        c->tile[st] = t;
        c->cnt[st] = cnt;
        c->has_prev[st] = base > 0;
        c->prev_res[st] = base > 0 ? R[-1] : 0;
        c->prev_start[st] = base > 0 ? S[-1] : 0;
    }
    copy_tail(sm.s, S, cnt, tma, lane);
    copy_tail(sm.e, E, cnt, tma, lane);
    copy_tail(sm.r, R, cnt, tma, lane);
    copy_tail(sm.k, K, cnt, tma, lane);
    __syncwarp();
    if (lane == 0) {
        const uint32_t tx = bulk_bytes<u64>(cnt, tma) * 2 + bulk_bytes<int32_t>(cnt, tma) + bulk_bytes<uint8_t>(cnt, tma);
        if (tx) {
            fence_proxy_async_smem();   // generic accesses of this stage -> async-proxy writes
            mbar_arrive_expect_tx(&c->full[st], tx);
            issue_bulk(sm.s, S, cnt, tma, &c->full[st], pol);
            issue_bulk(sm.e, E, cnt, tma, &c->full[st], pol);
            issue_bulk(sm.r, R, cnt, tma, &c->full[st], pol);
            issue_bulk(sm.k, K, cnt, tma, &c->full[st], pol);
        } else {
            mbar_arrive(&c->full[st]);
        }
    }
}

// -------------------------------------------------------------------------
// decoupled look-back over a 32-tile window (producer warp)
// -------------------------------------------------------------------------
template <int NV>
__device__ void look_back(const uint32_t *flags, const u64 *valA0, const u64 *valA1, const u64 *valP0,
                          const u64 *valP1, int64_t t, uint32_t epoch, int lane, u64 &c0, u64 &c1)
{
    u64 acc0 = 0, acc1 = 0;
    int64_t pos = t - 1;
    while (pos >= 0) {
        const int64_t i = pos - lane;
        uint32_t stt = 2;                      // before tile 0: identity, acts as prefix
        if (i >= 0) {
            const uint32_t f = ld_acquire(flags + i);
            stt = ((f >> 2) == epoch) ? (f & 3u) : 0u;
        }
        const unsigned pm = __ballot_sync(0xffffffffu, stt == 2);
        const unsigned xm = __ballot_sync(0xffffffffu, stt == 0);
        const int firstP = pm ? (__ffs(pm) - 1) : 32;
        const unsigned need = firstP >= 31 ? 0xffffffffu : ((2u << firstP) - 1u);
        if (xm & need) {
            __nanosleep(20);
            continue;
        }
        u64 v0 = 0, v1 = 0;
        if (i >= 0 && lane <= firstP) {
            if (lane == firstP) {
                v0 = ld_relaxed(valP0 + i);
                if (NV == 2) v1 = ld_relaxed(valP1 + i);
            } else {
                v0 = ld_relaxed(valA0 + i);
                if (NV == 2) v1 = ld_relaxed(valA1 + i);
            }
        }
        acc0 = umax(acc0, warp_max(v0));
        if (NV == 2) acc1 = umax(acc1, warp_max(v1));
        if (firstP < 32) break;
        pos -= 32;
    }
    c0 = acc0;
    c1 = acc1;
}

// -------------------------------------------------------------------------
// per-tile processing, shared skeleton
// -------------------------------------------------------------------------
struct TileCtx {
    int64_t lt;        // tile index within its side
    int64_t gbase;     // global record index of item 0 of this tile
    int cnt;
    int st;            // stage holding this tile
    int refill;        // stage the producer refills at B1 (-1: none)
};

// Phase A scan state of one compute thread over its kItems records.
struct Scan {
    uint32_t sfm;      // bit j: record j starts a new resource segment
    int nv;            // valid records of this thread
    bool t_flag;       // thread contains a segment start
    u64 t_v0, t_v1;    // max end over the thread's LAST segment (v0: kernel-only for devices)
    u64 t_max;         // max end over all records of the thread
};

// Phase A: stream the thread's records from shared memory once, derive the
// segment-start mask, check the canonical-order contract and the kind codes,
// and reduce the scan aggregate.
template <bool PARTIAL, bool DEV>
__device__ __forceinline__ Scan phase_a(const Params &p, const StageSmem &sm, const Ctrl *c, const TileCtx &tc,
                                        int ctid, int64_t gi0)
{
    Scan sc;
    const int b = ctid * kItems;
    sc.nv = PARTIAL ? max(0, min(kItems, tc.cnt - b)) : kItems;
    sc.sfm = 0;
    sc.t_flag = false;
    sc.t_v0 = sc.t_v1 = sc.t_max = 0;
    if (sc.nv == 0) return sc;
    bool hp;
    int32_t pr;
    u64 ps;
    if (ctid == 0) {
        hp = c->has_prev[tc.st] != 0;
        pr = c->prev_res[tc.st];
        ps = c->prev_start[tc.st];
    } else {
        hp = true;
        pr = sm.r[b - 1];
        ps = sm.s[b - 1];
    }
    int bad = -1;
    bool badkind = false;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        if (PARTIAL && j >= sc.nv) break;
        const int32_t r = sm.r[b + j];
        const u64 s = sm.s[b + j], e = sm.e[b + j];
        const uint8_t k = sm.k[b + j];
        const bool h = j > 0 || hp;
        if (!h || r != pr) {
            sc.sfm |= 1u << j;
            sc.t_flag = true;
            sc.t_v0 = 0;
            sc.t_v1 = 0;
        }
        if (bad < 0 && h && (r < pr || (r == pr && s < ps))) bad = j;
        if (DEV) {
            badkind |= k > 1;
            sc.t_v1 = umax(sc.t_v1, e);
            if (k == 0) sc.t_v0 = umax(sc.t_v0, e);
        } else {
            badkind |= k > 2;
            sc.t_v0 = umax(sc.t_v0, e);
        }
        sc.t_max = umax(sc.t_max, e);
        pr = r;
        ps = s;
    }
    if (bad >= 0) contract(p, DEV ? 2u : 1u, gi0 + bad);
    if (badkind) contract(p, DEV ? 8u : 4u, gi0);
    return sc;
}

// warp inclusive segmented max scan of (flag, v0, v1)
__device__ __forceinline__ void warp_seg_max(bool &f, u64 &v0, u64 &v1, int lane)
{
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const bool of = __shfl_up_sync(0xffffffffu, f, d);
        const u64 o0 = shfl_up64(v0, d), o1 = shfl_up64(v1, d);
        if (lane >= d) {
            if (!f) { v0 = umax(v0, o0); v1 = umax(v1, o1); }
            f |= of;
        }
    }
}

// thread-exclusive prefix inside the tile from the warp aggregates (smem)
// and the lane-inclusive scan values
__device__ __forceinline__ void tile_exclusive(const Ctrl *c, int warp, int lane, bool in_f, u64 in0, u64 in1,
                                               bool &xf, u64 &x0, u64 &x1)
{
    xf = false;
    x0 = x1 = 0;
#pragma unroll
    for (int w = 0; w < kComputeWarps; ++w) {
        if (w < warp) {
            if (c->w_flag[w]) { xf = true; x0 = c->w_v0[w]; x1 = c->w_v1[w]; }
            else { x0 = umax(x0, c->w_v0[w]); x1 = umax(x1, c->w_v1[w]); }
        }
    }
    const bool lf = __shfl_up_sync(0xffffffffu, in_f, 1);
    const u64 l0 = shfl_up64(in0, 1), l1 = shfl_up64(in1, 1);
    if (lane > 0) {
        if (lf) { xf = true; x0 = l0; x1 = l1; }
        else { x0 = umax(x0, l0); x1 = umax(x1, l1); }
    }
}

// Emit per-resource totals: warp-level segmented reduction of per-thread
// pieces, then one L2 reduction per (segment, warp).  A thread's record run
// splits into a head piece (records before its first segment start, which
// continue the left neighbour's segment), complete middle segments (already
// emitted) and a tail piece.  NA = number of add fields, field NA is a max.
template <int NA>
__device__ __forceinline__ void emit_segments(u64 (&head)[NA + 1], u64 (&tail)[NA + 1], uint32_t sfm, int nv,
                                              int32_t first_r, int32_t tail_r, int32_t ids, u64 *const (&dst)[NA + 1],
                                              int lane)
{
    const bool any = nv > 0;
    const bool f = sfm != 0;
    u64 v[NA + 1];
#pragma unroll
    for (int i = 0; i <= NA; ++i) v[i] = tail[i];
    int32_t sr = any ? tail_r : INT_MIN;
    bool sfl = f;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const bool of = __shfl_up_sync(0xffffffffu, sfl, d);
        const int32_t orr = __shfl_up_sync(0xffffffffu, sr, d);
        u64 o[NA + 1];
#pragma unroll
        for (int i = 0; i <= NA; ++i) o[i] = shfl_up64(v[i], d);
        if (lane >= d && !sfl) {
#pragma unroll
            for (int i = 0; i < NA; ++i) v[i] += o[i];
            v[NA] = umax(v[NA], o[NA]);
            if (!any) sr = orr;
        }
        if (lane >= d) sfl |= of;
    }
    u64 l[NA + 1];
#pragma unroll
    for (int i = 0; i <= NA; ++i) l[i] = shfl_up64(v[i], 1);
    const int32_t lr = __shfl_up_sync(0xffffffffu, sr, 1);
    if (any && f) {
        // the segment that ends right before this thread's first segment start
        const bool sf0 = sfm & 1u;
        bool have = !sf0;
        int32_t r = first_r;
        u64 w[NA + 1];
#pragma unroll
        for (int i = 0; i <= NA; ++i) w[i] = head[i];
        if (lane > 0 && lr != INT_MIN) {
#pragma unroll
            for (int i = 0; i < NA; ++i) w[i] += l[i];
            w[NA] = umax(w[NA], l[NA]);
            if (sf0) r = lr;
            have = true;
        }
        if (have && r >= 0 && r < ids) {
#pragma unroll
            for (int i = 0; i < NA; ++i)
                if (w[i]) red_add(dst[i] + r, w[i]);
            if (w[NA]) red_max(dst[NA] + r, w[NA]);
        }
    }
    if (lane == 31 && sr != INT_MIN && sr >= 0 && sr < ids) {
#pragma unroll
        for (int i = 0; i < NA; ++i)
            if (v[i]) red_add(dst[i] + sr, v[i]);
        if (v[NA]) red_max(dst[NA] + sr, v[NA]);
    }
}

// =========================================================================
// HOST tiles: per-rank sums + span, overlap validation (summarize.py:57-92,
// model.py:192-215)
// =========================================================================
template <bool PARTIAL>
__device__ __forceinline__ void host_tile(const Params &p, StageSmem *stages, Ctrl *c, const TileCtx &tc, int tid,
                                          uint64_t pol)
{
    const int warp = tid >> 5, lane = tid & 31;
    const bool producer = warp == kComputeWarps;
    const StageSmem &sm = stages[tc.st];
    const int b = tid * kItems;
    const int64_t gi0 = tc.gbase + (int64_t)b;

    Scan sc;
    bool in_f = false;
    u64 in0 = 0, in1 = 0;
    if (!producer) {
        sc = phase_a<PARTIAL, false>(p, sm, c, tc, tid, gi0);
        in_f = sc.t_flag; in0 = sc.t_v0;
        warp_seg_max(in_f, in0, in1, lane);
        const u64 wm = warp_max(sc.t_max);
        if (lane == 31) { c->w_flag[warp] = in_f; c->w_v0[warp] = in0; c->w_v1[warp] = 0; c->w_max[warp] = wm; }
    } else if (lane == 0) {
        c->head_cont[tc.st] = c->has_prev[tc.st] && sm.r[0] == c->prev_res[tc.st];
    }
    __syncthreads();  // B1 ------------------------------------------------

    if (producer) {
        bool f = false;
        u64 v = 0, mx = 0;
#pragma unroll
        for (int w = 0; w < kComputeWarps; ++w) {
            if (c->w_flag[w]) { f = true; v = c->w_v0[w]; }
            else v = umax(v, c->w_v0[w]);
            mx = umax(mx, c->w_max[w]);
        }
        if (lane == 0) {
            st_relaxed(f ? p.h_valP + tc.lt : p.h_valA + tc.lt, v);
            st_release(p.h_flag + tc.lt, (p.epoch << 2) | (f ? 2u : 1u));
            red_max(&p.g->host_max_end, mx);
            asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(&p.g->host_done) : "memory");
        }
        if (tc.refill >= 0) produce(p, stages, c, tc.refill, lane, pol);
        u64 carry = 0, dummy = 0;
        if (c->head_cont[tc.st]) {
            look_back<1>(p.h_flag, p.h_valA, nullptr, p.h_valP, nullptr, tc.lt, p.epoch, lane, carry, dummy);
            if (!f && lane == 0) {
                st_relaxed(p.h_valP + tc.lt, umax(carry, v));
                st_release(p.h_flag + tc.lt, (p.epoch << 2) | 2u);
            }
        }
        if (lane == 0) c->carry0[tc.st] = carry;
        bar_b2();  // B2 (producer side)
        return;
    }

    bool xf;
    u64 xv, xdummy;
    tile_exclusive(c, warp, lane, in_f, in0, in1, xf, xv, xdummy);
    // pieces: [0]=offload, [1]=mpi (adds), [2]=span (max)
    u64 head[3] = {0, 0, 0}, cur[3] = {0, 0, 0};
    bool head_open = !(sc.sfm & 1u);
    int32_t cur_r = sc.nv ? sm.r[b] : 0;
    const int32_t first_r = cur_r;
    bool cur_decl = sc.nv ? declared(p.host_decl, p.host_ids, p.n, cur_r) : false;
    u64 run = xv;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        if (PARTIAL && j >= sc.nv) break;
        if ((sc.sfm >> j) & 1u) {
            if (j > 0) {
                if (head_open) {
                    head[0] = cur[0]; head[1] = cur[1]; head[2] = cur[2];
                } else if (cur_r >= 0 && cur_r < p.host_ids) {   // complete segment inside the thread
                    if (cur[0]) red_add(p.h_off + cur_r, cur[0]);
                    if (cur[1]) red_add(p.h_mpi + cur_r, cur[1]);
                    if (cur[2]) red_max(p.h_span + cur_r, cur[2]);
                }
                head_open = false;
                cur_r = sm.r[b + j];
                cur_decl = declared(p.host_decl, p.host_ids, p.n, cur_r);
            }
            cur[0] = cur[1] = cur[2] = 0;
            run = 0;
        }
        const u64 s = sm.s[b + j], e = sm.e[b + j];
        const uint8_t k = sm.k[b + j];
        const int64_t gi = gi0 + j;
        if (s > e) push(p, 0, gi);
        else if (s == e) push(p, 1, gi);
        if (!cur_decl) push(p, 2, gi);
        if (cur_decl && s < e && s < run) push(p, 3, gi);
        run = umax(run, e);
        if (s <= e) {
            if (k == 1) cur[0] += e - s;
            else if (k == 2) cur[1] += e - s;
        }
        cur[2] = umax(cur[2], e);
    }
    bar_b2();  // B2 ------------------------------------------------

    // overlap fix-up: prefix of the tile head segment with start < carry
    if (c->head_cont[tc.st] && !xf && sc.nv > 0 && !(sc.sfm & 1u) && declared(p.host_decl, p.host_ids, p.n, first_r)) {
        const u64 carry = c->carry0[tc.st];
        u64 r2 = xv;
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            if ((PARTIAL && j >= sc.nv) || ((sc.sfm >> j) & 1u)) break;
            const u64 s = sm.s[b + j], e = sm.e[b + j];
            if (s >= carry) break;
            if (s < e && s >= r2) push(p, 3, gi0 + j);   // overlap only visible with the carry
            r2 = umax(r2, e);
        }
    }
    if (head_open) { head[0] = head[1] = head[2] = 0; }
    u64 *const dst[3] = {p.h_off, p.h_mpi, p.h_span};
    emit_segments<2>(head, cur, sc.sfm, sc.nv, first_r, cur_r, p.host_ids, dst, lane);
}

// =========================================================================
// DEVICE tiles: dual running-max union scan (summarize.py:95-138)
// =========================================================================
template <bool PARTIAL>
__device__ __forceinline__ void dev_tile(const Params &p, StageSmem *stages, Ctrl *c, const TileCtx &tc, int tid,
                                         uint64_t pol, u64 &E_cache, bool &E_known)
{
    const int warp = tid >> 5, lane = tid & 31;
    const bool producer = warp == kComputeWarps;
    const StageSmem &sm = stages[tc.st];
    const int b = tid * kItems;
    const int64_t gi0 = tc.gbase + (int64_t)b;

    Scan sc;
    bool in_f = false;
    u64 in0 = 0, in1 = 0;
    if (!producer) {
        sc = phase_a<PARTIAL, true>(p, sm, c, tc, tid, gi0);
        in_f = sc.t_flag; in0 = sc.t_v0; in1 = sc.t_v1;
        warp_seg_max(in_f, in0, in1, lane);
        if (lane == 31) { c->w_flag[warp] = in_f; c->w_v0[warp] = in0; c->w_v1[warp] = in1; }
    } else if (lane == 0) {
        c->head_cont[tc.st] = c->has_prev[tc.st] && sm.r[0] == c->prev_res[tc.st];
        if (!E_known) {
            u64 E;
            if (p.mode == kSummarizeDevice) E = p.elapsed_arg;
            else if ((p.mode == kReport || p.mode == kValidate) && p.n >= 1) {
                // E = max host end (summarize.py:88-89): wait for every host tile
                while (ld_acquire64(&p.g->host_done) < (u64)p.host_tiles) __nanosleep(64);
                E = umax(ld_relaxed(&p.g->host_max_end), p.host_elapsed_floor);
            } else {
                E = ~0ull;   // device-only trace: E = max device end, nothing is clamped
            }
            E_cache = E;
            E_known = true;
        }
        c->E[tc.st] = E_cache;
    }
    __syncthreads();  // B1 ------------------------------------------------

    if (producer) {
        bool f = false;
        u64 vk = 0, vkm = 0;
#pragma unroll
        for (int w = 0; w < kComputeWarps; ++w) {
            if (c->w_flag[w]) { f = true; vk = c->w_v0[w]; vkm = c->w_v1[w]; }
            else { vk = umax(vk, c->w_v0[w]); vkm = umax(vkm, c->w_v1[w]); }
        }
        if (lane == 0) {
            if (f) { st_relaxed(p.d_valP0 + tc.lt, vk); st_relaxed(p.d_valP1 + tc.lt, vkm); }
            else { st_relaxed(p.d_valA0 + tc.lt, vk); st_relaxed(p.d_valA1 + tc.lt, vkm); }
            st_release(p.d_flag + tc.lt, (p.epoch << 2) | (f ? 2u : 1u));
        }
        if (tc.refill >= 0) produce(p, stages, c, tc.refill, lane, pol);
        u64 ck = 0, ckm = 0;
        if (c->head_cont[tc.st]) {
            look_back<2>(p.d_flag, p.d_valA0, p.d_valA1, p.d_valP0, p.d_valP1, tc.lt, p.epoch, lane, ck, ckm);
            if (!f && lane == 0) {
                st_relaxed(p.d_valP0 + tc.lt, umax(ck, vk));
                st_relaxed(p.d_valP1 + tc.lt, umax(ckm, vkm));
                st_release(p.d_flag + tc.lt, (p.epoch << 2) | 2u);
            }
        }
        if (lane == 0) { c->carry0[tc.st] = ck; c->carry1[tc.st] = ckm; }
        bar_b2();  // B2 (producer side)
        return;
    }

    const u64 E = c->E[tc.st];
    const bool late_check = (p.mode == kReport || p.mode == kValidate) && p.n >= 1;
    bool xf;
    u64 xk, xkm;
    tile_exclusive(c, warp, lane, in_f, in0, in1, xf, xk, xkm);
    // pieces: [0]=U_K, [1]=U_KM, [2]=clamped (adds), [3]=max end (max)
    u64 head[4] = {0, 0, 0, 0}, cur[4] = {0, 0, 0, 0};
    bool head_open = !(sc.sfm & 1u);
    int32_t cur_r = sc.nv ? sm.r[b] : 0;
    const int32_t first_r = cur_r;
    bool cur_decl = sc.nv ? declared(p.dev_decl, p.dev_ids, p.m, cur_r) : false;
    u64 runK = xk, runKM = xkm;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        if (PARTIAL && j >= sc.nv) break;
        if ((sc.sfm >> j) & 1u) {
            if (j > 0) {
                if (head_open) {
                    head[0] = cur[0]; head[1] = cur[1]; head[2] = cur[2]; head[3] = cur[3];
                } else if (cur_r >= 0 && cur_r < p.dev_ids) {
                    if (cur[0]) red_add(p.d_k + cur_r, cur[0]);
                    if (cur[1]) red_add(p.d_km + cur_r, cur[1]);
                    if (cur[2]) red_add(p.d_clamp + cur_r, cur[2]);
                    if (cur[3]) red_max(p.d_maxend + cur_r, cur[3]);
                }
                head_open = false;
                cur_r = sm.r[b + j];
                cur_decl = declared(p.dev_decl, p.dev_ids, p.m, cur_r);
            }
            cur[0] = cur[1] = cur[2] = cur[3] = 0;
            runK = runKM = 0;
        }
        const u64 s = sm.s[b + j], e = sm.e[b + j];
        const uint8_t k = sm.k[b + j];
        const int64_t gi = gi0 + j;
        if (s > e) push(p, 4, gi);
        else if (s == e) push(p, 5, gi);
        if (!cur_decl) push(p, 6, gi);
        if (late_check && e > E) push(p, 7, gi);
        cur[2] += e > E ? 1 : 0;
        const u64 ee = umin(e, E);
        const u64 loKM = umax(s, runKM);
        cur[1] += ee > loKM ? ee - loKM : 0;
        runKM = umax(runKM, e);
        if (k == 0) {
            const u64 loK = umax(s, runK);
            cur[0] += ee > loK ? ee - loK : 0;
            runK = umax(runK, e);
        }
        cur[3] = umax(cur[3], e);
    }
    bar_b2();  // B2 ------------------------------------------------

    // carry fix-up: only the prefix of the tile head segment with max(s, run) < carry
    if (c->head_cont[tc.st] && !xf && sc.nv > 0 && !(sc.sfm & 1u)) {
        const u64 ck = c->carry0[tc.st], ckm = c->carry1[tc.st];
        u64 rK = xk, rKM = xkm, dk = 0, dkm = 0;
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            if ((PARTIAL && j >= sc.nv) || ((sc.sfm >> j) & 1u)) break;
            const u64 s = sm.s[b + j], e = sm.e[b + j];
            const uint8_t k = sm.k[b + j];
            const u64 loKM = umax(s, rKM), loK = umax(s, rK);
            if (loKM >= ckm && loK >= ck) break;
            const u64 ee = umin(e, E);
            const u64 nKM = umax(loKM, ckm);
            dkm += (ee > loKM ? ee - loKM : 0) - (ee > nKM ? ee - nKM : 0);
            rKM = umax(rKM, e);
            if (k == 0) {
                const u64 nK = umax(loK, ck);
                dk += (ee > loK ? ee - loK : 0) - (ee > nK ? ee - nK : 0);
                rK = umax(rK, e);
            }
        }
        if (head_open) { cur[0] -= dk; cur[1] -= dkm; }
        else { head[0] -= dk; head[1] -= dkm; }
    }
    if (head_open) { head[0] = head[1] = head[2] = head[3] = 0; }
    u64 *const dst[4] = {p.d_k, p.d_km, p.d_clamp, p.d_maxend};
    emit_segments<3>(head, cur, sc.sfm, sc.nv, first_r, cur_r, p.dev_ids, dst, lane);
}

// =========================================================================
// exact u128 / u128 -> nearest double, ties to even (Python int / int)
// =========================================================================
__device__ __forceinline__ int bitlen128(u128 x)
{
    const u64 hi = (u64)(x >> 64), lo = (u64)x;
    return hi ? 128 - __clzll((long long)hi) : (lo ? 64 - __clzll((long long)lo) : 0);
}

__device__ double div_exact(u128 a, u128 b)
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

// block reduction helpers for the finalize (NT threads)
__device__ u128 block_sum128(u128 v, u128 *scratch, int tid, int nt)
{
    scratch[tid] = v;
    __syncthreads();
    if (tid == 0) {
        u128 t = 0;
        for (int i = 0; i < nt; ++i) t += scratch[i];
        scratch[nt] = t;
    }
    __syncthreads();
    const u128 t = scratch[nt];
    __syncthreads();
    return t;
}

__device__ u128 block_max128(u128 v, u128 *scratch, int tid, int nt)
{
    scratch[tid] = v;
    __syncthreads();
    if (tid == 0) {
        u128 t = 0;
        for (int i = 0; i < nt; ++i) t = scratch[i] > t ? scratch[i] : t;
        scratch[nt] = t;
    }
    __syncthreads();
    const u128 t = scratch[nt];
    __syncthreads();
    return t;
}

// metric trees (metrics.py:66-122); threads 0..8 each do one division
__device__ void metric_trees(ResultDev *res, bool host_side, bool dev_side, u64 E, int32_t n, int32_t m,
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

// =========================================================================
// finalize (last CTA)
// =========================================================================
__device__ void finalize(const Params &p, u128 *scratch, int tid)
{
    Globals *g = p.g;
    ResultDev *res = p.res;
    const int nt = kThreads;
    __shared__ u64 s_E;
    __shared__ int s_status;
    // device-side max end over every device record (all ids)
    u64 dmx = 0;
    for (int32_t id = tid; id < p.dev_ids; id += nt) dmx = umax(dmx, ld_relaxed(p.d_maxend + id));
    const u64 dev_max_end = (u64)block_max128(dmx, scratch, tid, nt);
    const u64 host_elapsed = umax(ld_relaxed(&g->host_max_end), p.host_elapsed_floor);
    if (tid == 0) {
        u64 E;
        if (p.mode == kSummarizeDevice) E = p.elapsed_arg;
        else E = p.n >= 1 ? host_elapsed : dev_max_end;
        s_E = E;
        u64 cnt[8];
        for (int i = 0; i < 8; ++i) cnt[i] = ld_relaxed(&g->counts[i]);
        const bool invalid = (p.n == 0 && p.m == 0) || cnt[0] || cnt[2] || cnt[3] || cnt[4] || cnt[6];
        const unsigned cf = *(volatile unsigned *)&g->contract_flags;
        int st = 0;
        if (cf) st = 4;
        else if (p.mode == kSummarizeDevice && E == 0) st = 3;
        else if (invalid) st = 1;
        else if (p.mode == kReport && E == 0) st = 2;
        s_status = st;
        res->status = st;
        res->contract_flags = (int32_t)cf;
        res->contract_index = cf ? (int64_t)(*(volatile long long *)&g->contract_index) : -1;
        res->host_elapsed = host_elapsed;
        res->elapsed = E;
        res->dev_max_end = dev_max_end;
        res->host_present = p.n >= 1;
        res->device_present = p.m >= 1;
        res->host_mask = 0;
        res->device_mask = 0;
        for (int i = 0; i < 5; ++i) res->host_metrics[i] = 0.0;
        for (int i = 0; i < 4; ++i) res->device_metrics[i] = 0.0;
        for (int i = 0; i < 8; ++i) res->counts[i] = (int64_t)cnt[i];
    }
    __syncthreads();
    const u64 E = s_E;
    const bool ok = s_status == 0;

    // host summaries in declaration order; zero the accumulators
    u128 sum_u = 0, sum_uw = 0, max_uw = 0;
    for (int32_t id = tid; id < p.host_ids; id += nt) {
        const u64 off = ld_relaxed(p.h_off + id), mpi = ld_relaxed(p.h_mpi + id), span = ld_relaxed(p.h_span + id);
        p.h_off[id] = 0; p.h_mpi[id] = 0; p.h_span[id] = 0;
        const int32_t pos = p.host_decl ? p.host_decl[id] : (id < p.n ? id : -1);
        if (pos < 0 || pos >= p.n) continue;
        const u64 useful = span - off - mpi;
        u64 *o = p.host_out + 4 * (size_t)pos;
        o[0] = useful; o[1] = off; o[2] = mpi; o[3] = span;
        sum_u += useful;
        sum_uw += (u128)useful + off;
        const u128 uw = (u128)useful + off;
        if (uw > max_uw) max_uw = uw;
    }
    // device summaries
    u128 sum_k = 0, max_k = 0, max_km = 0;
    for (int32_t id = tid; id < p.dev_ids; id += nt) {
        const u64 k = ld_relaxed(p.d_k + id), km = ld_relaxed(p.d_km + id), cl = ld_relaxed(p.d_clamp + id);
        p.d_k[id] = 0; p.d_km[id] = 0; p.d_clamp[id] = 0; p.d_maxend[id] = 0;
        const int32_t pos = p.dev_decl ? p.dev_decl[id] : (id < p.m ? id : -1);
        if (pos < 0 || pos >= p.m) continue;
        u64 *o = p.dev_out + 4 * (size_t)pos;
        o[0] = k; o[1] = km - k; o[2] = E - km; o[3] = cl;
        sum_k += k;
        if (k > max_k) max_k = k;
        if (km > max_km) max_km = km;
    }
    sum_u = block_sum128(sum_u, scratch, tid, nt);
    sum_uw = block_sum128(sum_uw, scratch, tid, nt);
    max_uw = block_max128(max_uw, scratch, tid, nt);
    sum_k = block_sum128(sum_k, scratch, tid, nt);
    max_k = block_max128(max_k, scratch, tid, nt);
    max_km = block_max128(max_km, scratch, tid, nt);
    if (ok && p.mode == kReport) metric_trees(res, p.n >= 1, p.m >= 1, E, p.n, p.m, sum_u, sum_uw, max_uw, sum_k,
                                             max_k, max_km, tid);
    __syncthreads();
    if (tid == 0) {
        g->tile_counter = 0;
        g->host_done = 0;
        g->contract_flags = 0;
        g->host_max_end = 0;
        g->contract_index = LLONG_MAX;
        for (int i = 0; i < 8; ++i) g->counts[i] = 0;
        __threadfence();
        g->ctas_done = 0;
    }
}

// =========================================================================
// the kernel
// =========================================================================
__global__ void __launch_bounds__(kThreads, 1) analyze_kernel(const __grid_constant__ Params p)
{
    extern __shared__ __align__(128) uint8_t smem_raw[];
    StageSmem *stages = reinterpret_cast<StageSmem *>(smem_raw);
    Ctrl *c = reinterpret_cast<Ctrl *>(smem_raw + sizeof(StageSmem) * kStages);
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const uint64_t pol = l2_policy_evict_first();

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&c->full[s], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (warp == kComputeWarps)
        for (int s = 0; s < kStages - 1; ++s) produce(p, stages, c, s, lane, pol);
    u64 E_cache = 0;
    bool E_known = false;
    for (int it = 0;; ++it) {
        const int st = it % kStages;
        mbar_wait(&c->full[st], (uint32_t)((it / kStages) & 1));
        const int64_t t = c->tile[st];
        if (t < 0) break;
        TileCtx tc;
        tc.st = st;
        tc.refill = (it + kStages - 1) % kStages;   // stage of tile it-1: free once everyone passed B1
        tc.cnt = c->cnt[st];
        const bool dev = t >= p.host_tiles;
        tc.lt = dev ? t - p.host_tiles : t;
        tc.gbase = tc.lt * kTile;
        if (!dev) {
            if (tc.cnt == kTile) host_tile<false>(p, stages, c, tc, tid, pol);
            else host_tile<true>(p, stages, c, tc, tid, pol);
        } else {
            if (tc.cnt == kTile) dev_tile<false>(p, stages, c, tc, tid, pol, E_cache, E_known);
            else dev_tile<true>(p, stages, c, tc, tid, pol, E_cache, E_known);
        }
    }
    // CTA done: the last one finalizes
    __threadfence();
    __syncthreads();
    if (tid == 0) {
        const unsigned prev = atomicAdd(&p.g->ctas_done, 1u);
        c->is_last = prev == gridDim.x - 1;
    }
    __syncthreads();
    if (c->is_last) {
        __threadfence();
        finalize(p, reinterpret_cast<u128 *>(smem_raw), tid);
    }
}

// =========================================================================
// stand-alone metric trees (host_metrics / device_metrics stage functions)
// =========================================================================
__global__ void metrics_kernel(const u64 *sums, int32_t k, u64 E, int host_side, ResultDev *res)
{
    __shared__ u128 scratch[kThreads + 1];
    const int tid = threadIdx.x;
    u128 a = 0, b = 0, c = 0;   // host: sum_u, sum_uw, max_uw ; device: sum_k, max_k, max_km
    for (int32_t i = tid; i < k; i += kThreads) {
        const u64 *s = sums + 4 * (size_t)i;
        if (host_side) {
            const u128 uw = (u128)s[0] + s[1];
            a += s[0]; b += uw; if (uw > c) c = uw;
        } else {
            a += s[0]; if (s[0] > b) b = s[0];
            const u128 km = (u128)s[0] + s[1];
            if (km > c) c = km;
        }
    }
    a = block_sum128(a, scratch, tid, kThreads);
    if (host_side) { b = block_sum128(b, scratch, tid, kThreads); }
    else { b = block_max128(b, scratch, tid, kThreads); }
    c = block_max128(c, scratch, tid, kThreads);
    if (tid == 0) { res->host_mask = 0; res->device_mask = 0; res->status = 0; }
    __syncthreads();
    if (host_side) metric_trees(res, true, false, E, k, 0, a, b, c, 0, 0, 0, tid);
    else metric_trees(res, false, true, E, 0, k, 0, 0, 0, a, b, c, tid);
}

// =========================================================================
// error path: cover index of overlap errors (model.py:208-215) -- one
// thread per reported error walks back through its rank (first max end,
// ties keep the earlier record because of the strict '>' at model.py:214)
// =========================================================================
__global__ void covers_kernel(Params p, const int64_t *err, int64_t count, int64_t *cover)
{
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= count) return;
    const int64_t i = err[q];
    const int32_t r = p.hr[i];
    u64 best = 0;
    int64_t arg = -1;
    int64_t j = i - 1;
    while (j >= 0 && p.hr[j] == r) --j;
    for (int64_t x = j + 1; x < i; ++x) {
        const u64 s = p.hs[x], e = p.he[x];
        if (!(s < e)) continue;
        if (arg < 0 || e > best) { best = e; arg = x; }
    }
    cover[q] = arg;
}

int analyze_grid(int device)
{
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    cudaFuncSetAttribute(analyze_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)analyze_smem_bytes());
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, analyze_kernel, kThreads, analyze_smem_bytes());
    if (per < 1) per = 1;
    return sms * per;
}

cudaError_t launch_analyze(const Params &p, int grid, cudaStream_t s)
{
    analyze_kernel<<<grid, kThreads, analyze_smem_bytes(), s>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_metrics(const u64 *summaries, int32_t k, u64 elapsed, int host_side, ResultDev *res,
                           cudaStream_t s)
{
    metrics_kernel<<<1, kThreads, 0, s>>>(summaries, k, elapsed, host_side, res);
    return cudaGetLastError();
}

cudaError_t launch_covers(const Params &p, const int64_t *err_idx, int64_t count, int64_t *cover, cudaStream_t s)
{
    if (count <= 0) return cudaSuccess;
    const int bs = 128;
    covers_kernel<<<(unsigned)((count + bs - 1) / bs), bs, 0, s>>>(p, err_idx, count, cover);
    return cudaGetLastError();
}

}  // namespace hb
