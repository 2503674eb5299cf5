// engine.cu -- the B200 analysis kernel for heteff's hot path.
//
// One persistent kernel turns the packed host + device record SoA into every
// per-rank / per-device summary, all validation findings and both metric
// trees (reference: compute_report, metrics.py:125-154).
//
// Tiles of kTile records (kItems per compute thread), host tiles first, then
// device tiles, claimed in order through one global counter.  Each CTA is
// warp-specialized:
//
//  * a PRODUCER warp streams tiles HBM -> shared memory with 1-D TMA bulk
//    copies (cp.async.bulk, L2 evict-first) into a kStages ring (mbarriers
//    full[] / empty[]); after refilling a stage it runs the decoupled
//    look-back for the scan carry of the tile that just left it and applies
//    the carry correction to that tile's head segment (a few records, read
//    from global memory) -- off the critical path;
//  * kComputeWarps COMPUTE warps pull their records from shared memory
//    (blocked, odd stride = bank-conflict free), publish the tile's scan
//    aggregate, compute all per-record work with carry 0 and emit
//    per-resource totals.  They never wait for a look-back.
//
// The reference's device pipeline flatten/intersect/subtract/complement
// (intervals.py:40-105, summarize.py:119-132) reduces to a segmented
// running-max scan over start-sorted records: with e' = min(e,E),
// s' = min(s,e'), run = running max of earlier e',
//     c = max(run, e') - max(run, s')           (exact, empty if malformed)
// once over kernel records (U_K) and once over all records (U_KM):
//     d_kernel = U_K, d_memory = U_KM - U_K, d_idle = E - U_KM.
// The host overlap check (model.py:203-215) is the same scan over ends.
// When a tile's time range fits in 32 bits (the common case) the per-record
// arithmetic runs tile-relative in 32 bits; otherwise in 64 bits.
//
// E (= max host end, summarize.py:88-89) is needed by device tiles; host
// tiles come first and publish their max end, so the first device tile of a
// warp waits for the host phase once -- no second launch.  The last CTA to
// finish runs the finalize: summaries in declaration order, both metric
// trees with exactly rounded u128/u128 -> f64 divisions (Python int/int
// semantics), status, and the workspace reset.
#include <cuda_runtime.h>
#include <cstdint>
#include <climits>

#include "engine.cuh"
#include "ptx.cuh"
#include "exact.cuh"

#ifndef HB_DEV_SCHED
#define HB_DEV_SCHED 2   // single-segment device tiles: 0 two passes, 1 one pass + correction, 2 per-warp adaptive
#endif
#ifndef HB_UNROLL_G
#define HB_UNROLL_G 1   // general paths (~10% of tiles): compact code -- the hot set outgrows the 32 KB I-cache
#endif
#ifndef HB_UNROLL_A
#define HB_UNROLL_A HB_ITEMS
#endif
#ifndef HB_UNROLL_B
#define HB_UNROLL_B HB_ITEMS
#endif

namespace HB_ENGINE_NS {

#ifdef HB_PROF
// per-CTA clock64 phase counters (tools/prof build only): read back with heteff_prof_read
constexpr int kProfSlots = 32;
__device__ unsigned long long hb_prof_buf[1024 * kProfSlots];
#define PROF_DECL(x) long long x = 0
#define PROF_NOW() clock64()
#define PROF_ADD(acc, t0) (acc += clock64() - (t0))
#else
#define PROF_DECL(x)
#define PROF_NOW() 0
#define PROF_ADD(acc, t0)
#endif

struct Phases {
#ifdef HB_PROF
    long long a = 0, bar = 0, b = 0, emit = 0, t = 0;
    long long hb = 0, hemit = 0, hn = 0, dn = 0, hn2 = 0, mg = 0, nd = 0;
    __device__ __forceinline__ void mark() { t = clock64(); }
    __device__ __forceinline__ void add(long long &acc) { const long long n = clock64(); acc += n - t; t = n; }
#else
    __device__ __forceinline__ void mark() {}
    template <typename X>
    __device__ __forceinline__ void add(X &) {}
    int a, bar, b, emit, hb, hemit, hn, dn, hn2, mg, nd;
#endif
};

constexpr int kUnrollA = HB_UNROLL_A;
constexpr int kUnrollB = HB_UNROLL_B;
constexpr int kUnrollG = HB_UNROLL_G;   // general (multi-segment / multi-rank) paths: off the hot loop

struct StageSmem {
    u64 s[kTile];
    u64 e[kTile];
    int32_t r[kTile];
    uint8_t k[kTile];
};

constexpr int kRing = 8;       // device-tile epilogue descriptors in flight

// CSR offset-table sample per side (see csr_start)
#ifndef HB_SAMPLES
#define HB_SAMPLES 256
#endif
constexpr int kSamples = HB_SAMPLES;

struct CsrSample {
    int64_t v[kSamples];
    int32_t stride, count;
};

struct ClaimStage {      // shared memory of the CSR claim in flight
    int64_t v[96];       // seg[lo + i] (stride <= 64), past the table: LLONG_MAX
    u64 prev[2];         // start, end of the record before the tile
};

struct TileInfo {
    int64_t t;                 // global tile index, -1 = end
    int32_t cnt, head, tf;
    int32_t hcnt;              // CSR: records of the first resource in the tile (-1: res column)
    int32_t r0, pad;           // CSR: the first resource
    u64 t0, t1;
};

// Per-tile header and compute scratch live in kHdr slots indexed by the tile's
// sequence number in the CTA, not by its data stage, so the header of tile i+2
// never overwrites tile i's while any warp still reads it, whenever the warps
// release the stage.  (Releasing a stage early -- as soon as a warp holds its
// records in registers -- was measured: 0.4-2.6 % slower on C2 / C3 / C5, so
// warps release at the end of the tile.)  Warps drift at most two tiles apart
// (tile i+3 needs every warp's release of tile i+1): 4 slots never alias.
constexpr int kHdr = 4;

struct Ctrl {
    uint64_t full[kStages];    // TMA warp -> compute: tile data landed
    uint64_t empty[kStages];   // compute -> TMA warp: stage consumed
    uint64_t info_full[kRing];  // compute -> epilogue warp: device tile published
    uint64_t info_empty[kRing]; // epilogue warp -> compute: descriptor slot free
    TileInfo info[kRing];
    int64_t tile[kStages];     // read right after the full wait (before any release)
    int32_t cnt[kStages];
    int32_t has_prev[kHdr];
    int32_t prev_res[kHdr];
    int32_t is_last;
    int32_t r0[kHdr];          // CSR: first resource of the tile, leading records of it
    int32_t r0cnt[kHdr];
    int32_t uni[kHdr];         // CSR tile of ONE resource: its id (the stage's res column is not written), else -1
    u64 prev_start[kHdr];
    u64 prev_end[kHdr];
    // host tiles: per-tile max end and finished-warp count (smem atomics)
    u64 h_max[kHdr];
    unsigned int h_cnt[kHdr];
    // single-segment device tiles: per-warp 32-bit aggregates relative to the tile base
    uint32_t f_k[kHdr][kComputeWarps];
    uint32_t f_km[kHdr][kComputeWarps];
    int32_t f_fit[kHdr][kComputeWarps];
    // per-tile warp aggregates (written by compute warps)
    int32_t w_flag[kHdr][kComputeWarps];
    u64 w_v0[kHdr][kComputeWarps];
    u64 w_v1[kHdr][kComputeWarps];
    u64 w_mn[kHdr][kComputeWarps];
    u64 w_mx[kHdr][kComputeWarps];
    CsrSample csr[2];          // host, device (producer warp only)
    ClaimStage claim;          // the CSR claim in flight (producer warp only)
};

constexpr size_t kSmemBytes = sizeof(StageSmem) * kStages + sizeof(Ctrl) + 128;
static_assert(kSmemBytes <= 227 * 1024, "stages + control exceed the 227 KB of shared memory per CTA");
size_t analyze_smem_bytes() { return kSmemBytes; }

// -------------------------------------------------------------------------
// small helpers
// -------------------------------------------------------------------------
// dense id of stage record i: the uniform id of a one-resource CSR tile, else the stage column
__device__ __forceinline__ int32_t rid(const StageSmem &sm, int32_t uni, int i) { return uni >= 0 ? uni : sm.r[i]; }

__device__ __forceinline__ bool declared(const int32_t *decl, int32_t ids, int32_t n, int32_t r)
{
    if (r < 0 || r >= ids) return false;
    return decl ? (__ldg(decl + r) >= 0) : (r < n);
}

__device__ __noinline__ void push(const Params &p, int cls, int64_t gi)
{
    u64 idx = atomicAdd(&p.g->counts[cls], 1ull);
    if ((int64_t)idx < p.cap) p.lists[cls][idx] = gi;
}

__device__ __noinline__ void contract(const Params &p, unsigned flag, int64_t gi)
{
    // unsorted input flags (nearly) every thread: skip the atomics once an earlier index holds
    if ((*(volatile unsigned *)&p.g->contract_flags & flag) && *(volatile long long *)&p.g->contract_index <= gi)
        return;
    atomicOr(&p.g->contract_flags, flag);
    atomicMin(&p.g->contract_index, (long long)gi);
}

// named barrier over the compute warps only.  Non-.aligned (`bar.sync` is
// barrier.sync.aligned): the per-warp schedule choice (dev_single<true/false>) and
// lane-predicated stores mean the compiler cannot prove a warp converged here, and
// compute-sanitizer synccheck flagged the aligned form ("divergent thread(s)").
__device__ __forceinline__ void bar_compute()
{
    asm volatile("barrier.sync 1, %0;" ::"n"(kComputeThreads) : "memory");
}

__device__ __forceinline__ u64 warp_max(u64 v)
{
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = umax(v, __shfl_xor_sync(0xffffffffu, v, d));
    return v;
}

__device__ __forceinline__ u64 warp_min(u64 v)
{
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = umin(v, __shfl_xor_sync(0xffffffffu, v, d));
    return v;
}

// 64-bit warp reductions on the REDUX unit (32-bit ops): max/min via the
// high word first, sums via three 21-bit limbs (exact mod 2^64)
__device__ __forceinline__ u64 warp_max_rx(u64 v)
{
    const unsigned hi = (unsigned)(v >> 32), lo = (unsigned)v;
    const unsigned mh = __reduce_max_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_max_sync(0xffffffffu, hi == mh ? lo : 0u);
    return ((u64)mh << 32) | ml;
}

__device__ __forceinline__ u64 warp_min_rx(u64 v)
{
    const unsigned hi = (unsigned)(v >> 32), lo = (unsigned)v;
    const unsigned mh = __reduce_min_sync(0xffffffffu, hi);
    const unsigned ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
    return ((u64)mh << 32) | ml;
}

__device__ __forceinline__ u64 warp_sum_rx(u64 v)
{
    const unsigned l0 = (unsigned)v & 0x1fffffu, l1 = (unsigned)(v >> 21) & 0x1fffffu, l2 = (unsigned)(v >> 42);
    return (u64)__reduce_add_sync(0xffffffffu, l0) + ((u64)__reduce_add_sync(0xffffffffu, l1) << 21) +
           ((u64)__reduce_add_sync(0xffffffffu, l2) << 42);
}

__device__ __forceinline__ u64 warp_sum(u64 v)
{
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

// E for device tiles: the explicit window, the max host end (once every host
// tile is finished), or "no clamp" for device-only traces.  Progress does not
// depend on co-residency: tiles are claimed in order by running CTAs and host
// tiles never wait, so every claimed host tile completes whether or not the
// whole grid is resident (MPS limits, green contexts, co-running kernels, a
// grid larger than one wave).  A CTA releases the count of host tiles it
// finished once, when its compute warps move on to device tiles (after the
// CTA barrier of its first device tile) or end; E is known once the count
// reaches host_tiles.
__device__ __forceinline__ void host_tiles_done(const Params &p, int count)
{
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(&p.g->host_done), "l"((u64)count) : "memory");
}

__device__ u64 device_window(const Params &p)
{
    if (p.mode == kSummarizeDevice) return p.elapsed_ptr ? ld_relaxed(p.elapsed_ptr) : p.elapsed_arg;
    if ((p.mode == kReport || p.mode == kValidate) && p.n >= 1) {
        while (ld_acquire64(&p.g->host_done) < (u64)p.host_tiles) __nanosleep(64);
        return umax(ld_relaxed(&p.g->host_max_end), p.host_elapsed_floor);
    }
    return ~0ull;
}

// -------------------------------------------------------------------------
// producer: stream a claimed tile into a stage
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

// ---- CSR resource offsets ("SoA arrays plus CSR offsets") ----
// Records [seg[r], seg[r+1]) belong to dense id r.  Instead of streaming a
// 4-byte res column (21 -> 17 B per record), the producer locates each tile's
// first resource with a 128-ary search over seg (4 probes per lane, one L2
// round trip per level: 2 levels up to 16384 ids) and writes the tile's res
// values into shared memory itself -- the compute warps see the same stage as
// with a res column.
__device__ __forceinline__ int32_t csr_find(const int64_t *seg, int32_t lo, int32_t hi, int64_t i, int lane)
{
    // seg[lo] <= i (seg[0] = 0 <= i); the answer lies in [lo, hi]
    while (lo < hi) {
        const int64_t step = ((int64_t)hi - lo + 128) / 128;   // ceil(span / 128)
        int64_t v[4];
        bool in[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {   // probe k = 4 lane + q at lo + k step (k = 0: lo itself)
            const int k = 4 * lane + q;
            const int64_t pos = lo + (int64_t)k * step;
            in[q] = k > 0 && pos <= hi;
            v[q] = in[q] ? __ldg(seg + pos) : 0;
        }
        int K = 0;   // seg is non-decreasing: the probes with seg <= i are k = 1..K
#pragma unroll
        for (int q = 0; q < 4; ++q) K += __popc(__ballot_sync(0xffffffffu, in[q] && v[q] <= i));
        const int64_t nlo = lo + (int64_t)K * step;
        const int64_t nhi = nlo + step - 1;
        lo = (int32_t)nlo;
        hi = nhi < hi ? (int32_t)nhi : hi;
    }
    return lo;
}

// window of 32 offsets seg[rc + lane] (past the table: "never")
__device__ __forceinline__ int64_t csr_window(const int64_t *seg, int32_t ids, int32_t rc, int lane)
{
    return (int64_t)rc + lane <= (int64_t)ids ? __ldg(seg + rc + lane) : LLONG_MAX;
}

// Per-CTA sample of each offset table (shared memory, filled once by the
// producer warp): samp[j] = seg[j * stride], stride = ceil(ids / kSamples).
// It narrows a tile's first resource to one stride, so up to kSamples * 64 ids
// a single L2 round trip (3 offsets per lane) yields both the resource and the
// 32-offset window after it.

__device__ void csr_sample_fill(const int64_t *seg, int32_t ids, CsrSample &cs, int lane)
{
    if (!seg) return;
    const int32_t stride = ids <= kSamples ? 1 : (int32_t)(((int64_t)ids + kSamples - 1) / kSamples);
    const int32_t count = (int32_t)(((int64_t)ids + stride - 1) / stride);
    for (int j = lane; j < count; j += 32) cs.v[j] = __ldg(seg + (int64_t)j * stride);
    if (lane == 0) { cs.stride = stride; cs.count = count; }
    __syncwarp();
}

// the tile's first resource r0 (last r with seg[r] <= base) and w = seg[r0 + lane]
// A claimed tile in flight (CSR): its offset-window and previous-record loads are
// issued as cp.async copies into shared memory when the claim resolves and read one
// refill later, so the L2 round trip overlaps the producer's wait for the next free
// stage and no register stays live across it.
struct PendClaim {
    int64_t t;
    int32_t lo, hi;      // the tile's first resource lies in [lo, hi]
};

__device__ __forceinline__ void cp_async8(void *dst, const void *src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// stage 1: narrow with the CTA's sample (shared memory), issue the offset copies
__device__ __forceinline__ void csr_start(const int64_t *seg, int32_t ids, const CsrSample &cs, int64_t base,
                                          int lane, PendClaim &pc, ClaimStage &st)
{
    // samples <= base form a prefix (the table never decreases): count them in two
    // rounds, every 8th sample first, then the 8 after the last one that passed
    static_assert(kSamples == 256, "two-round sample scan");
    const int j1 = 8 * lane;
    const int K1 = __popc(__ballot_sync(0xffffffffu, j1 < cs.count && cs.v[j1] <= base));
    const int g = K1 > 0 ? K1 - 1 : 0;
    const int j2 = 8 * g + (lane & 7);
    const int K2 = __popc(__ballot_sync(0xffffffffu, lane < 8 && j2 < cs.count && cs.v[j2] <= base));
    const int K = 8 * g + K2;   // K1 = 0 only if sample 0 > base (a broken table): then K2 = 0 too
    pc.lo = (K > 0 ? K - 1 : 0) * cs.stride;
    pc.hi = min(ids - 1, pc.lo + cs.stride - 1);
    if (cs.stride <= 64) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {   // seg[lo .. lo + 95]: r0 <= lo + 63, its window <= lo + 94
            const int64_t pos = (int64_t)pc.lo + lane + 32 * q;
            if (pos <= ids) cp_async8(&st.v[lane + 32 * q], seg + pos);
            else st.v[lane + 32 * q] = LLONG_MAX;
        }
    }
}

// stage 2: the first resource r0 (last r with seg[r] <= base) and w = seg[r0 + lane]
__device__ __forceinline__ void csr_finish(const int64_t *seg, int32_t ids, const CsrSample &cs, int64_t base,
                                           int lane, const PendClaim &pc, const ClaimStage &st, int32_t &r0,
                                           int64_t &w)
{
    if (cs.stride <= 64) {
        int k = 0;
#pragma unroll
        for (int q = 0; q < 3; ++q)
            k += __popc(__ballot_sync(0xffffffffu, pc.lo + lane + 32 * q <= pc.hi && st.v[lane + 32 * q] <= base));
        r0 = pc.lo + (k > 0 ? k - 1 : 0);
        w = st.v[r0 - pc.lo + lane];   // seg[r0 + lane]: r0 - lo <= 63
    } else {   // > kSamples * 64 ids: a 128-ary search inside the stride
        r0 = csr_find(seg, pc.lo, pc.hi, base, lane);
        w = csr_window(seg, ids, r0, lane);
    }
}

// the record before a tile (for segment / order checks), loaded one
// iteration ahead of the refill so its latency is hidden; CSR: the tile's
// first resource and the offset window after it
struct Claim {
    int64_t t;
    int32_t prev_r;
    int32_t r0;        // CSR: resource of the tile's first record
    u64 prev_s, prev_e;
    int64_t w;         // CSR: seg[r0 + lane]
};

__device__ __forceinline__ int64_t claim_issue(const Params &p, int lane)
{
    int64_t t = 0;
    if (lane == 0) t = (int64_t)atomicAdd(&p.g->tile_counter, 1ull);
    return t;
}

// the claimed index (issued earlier by lane 0) and the record before the tile
__device__ __forceinline__ Claim claim_finish(const Params &p, int64_t issued)
{
    Claim cl;
    cl.t = __shfl_sync(0xffffffffu, issued, 0);
    cl.prev_r = 0;
    cl.r0 = 0;
    cl.prev_s = 0;
    cl.prev_e = 0;
    cl.w = LLONG_MAX;
    if (cl.t < p.host_tiles + p.dev_tiles) {
        const bool dev = cl.t >= p.host_tiles;
        const int64_t base = (dev ? cl.t - p.host_tiles : cl.t) * kTile;
        if (base > 0) {
            cl.prev_r = __ldcg((dev ? p.dr : p.hr) + base - 1);
            cl.prev_s = __ldcg((dev ? p.ds : p.hs) + base - 1);
            cl.prev_e = __ldcg((dev ? p.de : p.he) + base - 1);
        }
    }
    return cl;
}

// CSR claims, two stages: start (index resolved, copies issued) -> done (one refill later)
__device__ __forceinline__ PendClaim claim_start(const Params &p, const CsrSample *cs, ClaimStage &st,
                                                 int64_t issued, int lane)
{
    PendClaim pc;
    pc.t = __shfl_sync(0xffffffffu, issued, 0);
    pc.lo = pc.hi = 0;
    if (pc.t < p.host_tiles + p.dev_tiles) {
        const bool dev = pc.t >= p.host_tiles;
        const int64_t base = (dev ? pc.t - p.host_tiles : pc.t) * kTile;
        if (base > 0 && lane < 2) cp_async8(&st.prev[lane], (lane ? (dev ? p.de : p.he) : (dev ? p.ds : p.hs)) + base - 1);
        const int64_t *seg = dev ? p.dseg : p.hseg;
        if (seg) csr_start(seg, dev ? p.dev_ids : p.host_ids, cs[dev ? 1 : 0], base, lane, pc, st);
        else if (base > 0) pc.lo = __ldcg((dev ? p.dr : p.hr) + base - 1);   // a side with a res column
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    return pc;
}

__device__ __forceinline__ Claim claim_done(const Params &p, const CsrSample *cs, const PendClaim &pc,
                                            const ClaimStage &st, int lane)
{
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncwarp();
    Claim cl;
    cl.t = pc.t;
    cl.prev_r = 0;
    cl.r0 = 0;
    cl.prev_s = 0;
    cl.prev_e = 0;
    cl.w = LLONG_MAX;
    if (pc.t < p.host_tiles + p.dev_tiles) {
        const bool dev = pc.t >= p.host_tiles;
        const int64_t base = (dev ? pc.t - p.host_tiles : pc.t) * kTile;
        if (base > 0) {
            cl.prev_s = st.prev[0];
            cl.prev_e = st.prev[1];
        }
        const int64_t *seg = dev ? p.dseg : p.hseg;
        if (seg) {
            csr_finish(seg, dev ? p.dev_ids : p.host_ids, cs[dev ? 1 : 0], base, lane, pc, st, cl.r0, cl.w);
            // the record before the tile belongs to r0 unless r0 starts at the tile
            // (then to an earlier id: only inequality / order against r0 is ever used)
            const int64_t s0 = __shfl_sync(0xffffffffu, cl.w, 0);
            cl.prev_r = s0 < base ? cl.r0 : cl.r0 - 1;
        } else {
            cl.prev_r = pc.lo;
        }
    }
    __syncwarp();   // every lane has read the stage before the next claim's copies land
    return cl;
}

// r[a, z) = v, 32 lanes, 16-byte stores in the middle (r is 16-byte aligned)
__device__ __forceinline__ void fill_range(int32_t *r, int a, int z, int32_t v, int lane)
{
    const int a4 = min(z, (a + 3) & ~3);
    if (lane < a4 - a) r[a + lane] = v;
    const int z4 = max(a4, z & ~3);
    const int4 vv = make_int4(v, v, v, v);
    for (int i = a4 + 4 * lane; i < z4; i += 128) *reinterpret_cast<int4 *>(r + i) = vv;
    if (lane < z - z4) r[z4 + lane] = v;
}

// CSR: write the tile's res values into the stage; returns the number of leading
// records of the first resource.  Resource rc + l covers [w_l, w_{l+1}) (l < 31).
// Offsets that decrease, do not start at 0 or do not end at the record count
// (where a tile sees them) set `bad` (HETEFF_CONTRACT, never an out-of-range access).
__device__ __noinline__ int csr_fill(const int64_t *seg, int32_t ids, int64_t base, int cnt, int64_t n,
                                        const Claim &cl, int32_t *r, int lane, bool &bad)
{
    int32_t rc = cl.r0;
    int64_t w = cl.w;
    int first = -1;
    bool b = lane == 0 && (w > base || (base == 0 && w != 0));
    for (;;) {
        const int64_t wn = __shfl_down_sync(0xffffffffu, w, 1);
        b = b || (lane < 31 && wn < w);
        if ((int64_t)rc + lane == (int64_t)ids) b = b || w < base + cnt || (base + cnt == n && w != n);
        const int lo = (int)(w <= base ? 0 : (w - base < cnt ? w - base : cnt));
        const int hi = (int)(wn <= base ? 0 : (wn - base < cnt ? wn - base : cnt));
        if (first < 0) first = __shfl_sync(0xffffffffu, hi, 0);
        unsigned live = __ballot_sync(0xffffffffu, lane < 31 && hi > lo);
        while (live) {
            const int l = __ffs(live) - 1;
            live &= live - 1;
            fill_range(r, __shfl_sync(0xffffffffu, lo, l), __shfl_sync(0xffffffffu, hi, l), rc + l, lane);
        }
        if (__shfl_sync(0xffffffffu, hi, 30) >= cnt) break;
        rc += 31;   // 31 resources started inside the tile: the next window
        w = csr_window(seg, ids, rc, lane);
    }
    bad = __any_sync(0xffffffffu, b);
    return first;
}

template <bool CSR>
__device__ void produce(const Params &p, StageSmem *stages, Ctrl *c, int st, int hs, const Claim &cl, int lane,
                        uint64_t pol)
{
    const int64_t t = cl.t;
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
    const uint8_t *K = (dev ? p.dk : p.hk) + base;
    StageSmem &sm = stages[st];
    const bool tma = p.use_tma != 0;
    if constexpr (!CSR) {
        const int32_t *R = (dev ? p.dr : p.hr) + base;
        copy_tail(sm.s, S, cnt, tma, lane);
        copy_tail(sm.e, E, cnt, tma, lane);
        copy_tail(sm.r, R, cnt, tma, lane);
        copy_tail(sm.k, K, cnt, tma, lane);
        if (lane == 0) {
            c->tile[st] = t;
            c->cnt[st] = cnt;
            c->has_prev[hs] = base > 0;
            c->prev_res[hs] = cl.prev_r;
            c->prev_start[hs] = cl.prev_s;
            c->prev_end[hs] = cl.prev_e;
            c->r0cnt[hs] = -1;
            c->r0[hs] = 0;
            c->uni[hs] = -1;
        }
        __syncwarp();
        if (lane == 0) {
            const uint32_t tx =
                bulk_bytes<u64>(cnt, tma) * 2 + bulk_bytes<int32_t>(cnt, tma) + bulk_bytes<uint8_t>(cnt, tma);
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
    } else {
        const int64_t *seg = dev ? p.dseg : p.hseg;
        const int32_t *R = seg ? nullptr : (dev ? p.dr : p.hr) + base;
        // the bulk copies go out first (tx count only); the full barrier's single
        // arrival comes after the tails / CSR ids are in shared memory
        if (lane == 0) {
            const uint32_t tx = bulk_bytes<u64>(cnt, tma) * 2 + (R ? bulk_bytes<int32_t>(cnt, tma) : 0u) +
                                bulk_bytes<uint8_t>(cnt, tma);
            if (tx) {
                fence_proxy_async_smem();
                mbar_expect_tx(&c->full[st], tx);
                issue_bulk(sm.s, S, cnt, tma, &c->full[st], pol);
                issue_bulk(sm.e, E, cnt, tma, &c->full[st], pol);
                if (R) issue_bulk(sm.r, R, cnt, tma, &c->full[st], pol);
                issue_bulk(sm.k, K, cnt, tma, &c->full[st], pol);
            }
        }
        copy_tail(sm.s, S, cnt, tma, lane);
        copy_tail(sm.e, E, cnt, tma, lane);
        copy_tail(sm.k, K, cnt, tma, lane);
        int r0cnt = -1;
        int32_t uni = -1;
        if (R) {
            copy_tail(sm.r, R, cnt, tma, lane);
        } else {
            const int32_t ids = dev ? p.dev_ids : p.host_ids;
            bool bad = false;
            if (__shfl_sync(0xffffffffu, cl.w, 1) >= base + cnt) {
                // one resource: the compute warps take its id from uni, the column stays unwritten;
                // the offset checks of csr_fill on this window
                const int64_t wn = __shfl_down_sync(0xffffffffu, cl.w, 1);
                bool b = (lane == 0 && (cl.w > base || (base == 0 && cl.w != 0))) || (lane < 31 && wn < cl.w);
                if ((int64_t)cl.r0 + lane == (int64_t)ids) b = b || cl.w < base + cnt || (base + cnt == n && cl.w != n);
                bad = __any_sync(0xffffffffu, b);
                uni = cl.r0;
                r0cnt = cnt;
            } else {
                r0cnt = csr_fill(seg, ids, base, cnt, n, cl, sm.r, lane, bad);
            }
            if (bad && lane == 0) contract(p, dev ? 2u : 1u, base);
        }
        if (lane == 0) {
            c->tile[st] = t;
            c->cnt[st] = cnt;
            c->has_prev[hs] = base > 0;
            c->prev_res[hs] = cl.prev_r;
            c->prev_start[hs] = cl.prev_s;
            c->prev_end[hs] = cl.prev_e;
            c->r0cnt[hs] = r0cnt;
            c->r0[hs] = cl.r0;
            c->uni[hs] = uni;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&c->full[st]);
    }
}

// -------------------------------------------------------------------------
// decoupled look-back (producer warp), 32-tile window, one round trip:
// every slot word is (epoch << 32 | 32-bit half of the value), so a slot is
// valid iff all its words carry the current epoch -- no flag / value
// ordering needed.  Separate A (aggregate) and P (inclusive prefix) slots.
// -------------------------------------------------------------------------
template <int NV>
__device__ __forceinline__ void publish(u64 *slot, uint32_t epoch, u64 v0, u64 v1)
{
    const u64 tag = (u64)epoch << 32;
    st_relaxed(slot + 0, tag | (v0 >> 32));
    st_relaxed(slot + 1, tag | (v0 & 0xffffffffull));
    if (NV == 2) {
        st_relaxed(slot + 2, tag | (v1 >> 32));
        st_relaxed(slot + 3, tag | (v1 & 0xffffffffull));
    }
}

// 16-byte L2 loads (each 8-byte word is single-copy atomic; validity is per word)
template <int NV>
__device__ __forceinline__ bool read_slot(const u64 *slot, uint32_t epoch, u64 &v0, u64 &v1)
{
    const ulonglong2 ab = __ldcg(reinterpret_cast<const ulonglong2 *>(slot));
    bool ok = (ab.x >> 32) == epoch && (ab.y >> 32) == epoch;
    v0 = (ab.x << 32) | (ab.y & 0xffffffffull);
    v1 = 0;
    if (NV == 2) {
        const ulonglong2 cd = __ldcg(reinterpret_cast<const ulonglong2 *>(slot + 2));
        ok = ok && (cd.x >> 32) == epoch && (cd.y >> 32) == epoch;
        v1 = (cd.x << 32) | (cd.y & 0xffffffffull);
    }
    return ok;
}

template <int NV>
__device__ void look_back(const u64 *slotA, const u64 *slotP, int64_t t, uint32_t epoch, int lane, u64 &c0, u64 &c1)
{
    constexpr int W = 2 * NV;   // words per slot
    constexpr int Q = 4;        // tiles per lane: 128-tile window per round trip
    u64 acc0 = 0, acc1 = 0;
    int64_t pos = t - 1;
    while (pos >= 0) {
        uint32_t stt[Q];
        u64 v0[Q], v1[Q];
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int64_t i = pos - lane - 32 * q;
            stt[q] = 2;                        // before tile 0: identity, acts as prefix
            v0[q] = v1[q] = 0;
            if (i >= 0) {
                u64 p0, p1, a0, a1;
                const bool pv = read_slot<NV>(slotP + i * W, epoch, p0, p1);
                const bool av = read_slot<NV>(slotA + i * W, epoch, a0, a1);
                stt[q] = pv ? 2u : (av ? 1u : 0u);
                v0[q] = pv ? p0 : a0;
                v1[q] = pv ? p1 : a1;
            }
        }
        bool ready = true, done = false;
        u64 r0 = 0, r1 = 0;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            if (!done) {
                const unsigned pm = __ballot_sync(0xffffffffu, stt[q] == 2);
                const unsigned xm = __ballot_sync(0xffffffffu, stt[q] == 0);
                const int firstP = pm ? (__ffs(pm) - 1) : 32;
                const unsigned need = firstP >= 31 ? 0xffffffffu : ((2u << firstP) - 1u);
                if (xm & need) {
                    ready = false;
                    done = true;
                } else {
                    r0 = umax(r0, warp_max(lane <= firstP ? v0[q] : 0));
                    if (NV == 2) r1 = umax(r1, warp_max(lane <= firstP ? v1[q] : 0));
                    if (firstP < 32) done = true;
                }
            }
        }
        if (!ready) {
            __nanosleep(32);
            continue;
        }
        acc0 = umax(acc0, r0);
        acc1 = umax(acc1, r1);
        if (done) break;
        pos -= 32 * Q;
    }
    c0 = acc0;
    c1 = acc1;
}

struct TileCtx {
    int64_t lt;        // tile index within its side
    int64_t gbase;     // global record index of item 0 of this tile
    int cnt;
    int st;            // header / scratch slot of this tile (kHdr ring; the data stage is separate)
    uint64_t *empty;   // the data stage's empty barrier
    bool released;     // this warp has released the data stage
};

// The warp no longer reads the tile's stage: the producer may refill it.
// Warp-uniform; once per tile.
__device__ __forceinline__ void release(TileCtx &tc, int lane)
{
    if (tc.released) return;
    __syncwarp();
    if (lane == 0) mbar_arrive(tc.empty);
    tc.released = true;
}

// combine two segmented-max scan elements, a earlier than b
__device__ __forceinline__ void seg_combine(bool af, u64 a0, u64 a1, bool &bf, u64 &b0, u64 &b1)
{
    if (!bf) { b0 = umax(a0, b0); b1 = umax(a1, b1); }
    bf = bf || af;
}

// warp inclusive segmented max scan of (flag, v0, v1)
__device__ __forceinline__ void warp_seg_max(bool &f, u64 &v0, u64 &v1, int lane)
{
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const bool of = __shfl_up_sync(0xffffffffu, f, d);
        const u64 o0 = shfl_up64(v0, d), o1 = shfl_up64(v1, d);
        if (lane >= d) seg_combine(of, o0, o1, f, v0, v1);
    }
}

// warp inclusive max scan of two 32-bit values
__device__ __forceinline__ void warp_max_scan2(uint32_t &a, uint32_t &b, int lane)
{
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t oa = __shfl_up_sync(0xffffffffu, a, d), ob = __shfl_up_sync(0xffffffffu, b, d);
        if (lane >= d) { a = max(a, oa); b = max(b, ob); }
    }
}

// exact warp sum of 32-bit values (two 16-bit limbs on the REDUX unit)
__device__ __forceinline__ u64 warp_sum32(uint32_t v)
{
    return (u64)__reduce_add_sync(0xffffffffu, v & 0xffffu) + ((u64)__reduce_add_sync(0xffffffffu, v >> 16) << 16);
}

// Per-tile values every compute thread derives (cooperatively per warp)
// from the warp aggregates.
struct TileView {
    bool xf;           // a segment starts before this thread inside the tile
    u64 x0, x1;        // exclusive segmented max (v0 / v1) for this thread
    u64 base, top;     // min start / max end over the tile's records
    bool fits32;       // top - base < 2^32: tile-relative 32-bit arithmetic is exact
    bool tf;           // tile aggregate: a segment starts in the tile,
    u64 t0, t1;        //   max ends over the tile's last segment
};

__device__ __forceinline__ TileView tile_view(const Ctrl *c, int st, int warp, int lane, bool in_f, u64 in0, u64 in1)
{
    TileView v;
    bool f = false;
    u64 a0 = 0, a1 = 0, mn = ~0ull, mx = 0;
    if (lane < kComputeWarps) {
        f = c->w_flag[st][lane] != 0;
        a0 = c->w_v0[st][lane];
        a1 = c->w_v1[st][lane];
        mn = c->w_mn[st][lane];
        mx = c->w_mx[st][lane];
    }
    v.base = warp_min_rx(mn);
    v.top = warp_max_rx(mx);
    v.fits32 = v.top >= v.base && (v.top - v.base) < (1ull << 32);
    warp_seg_max(f, a0, a1, lane);                 // inclusive over warps 0..lane
    v.tf = __shfl_sync(0xffffffffu, f, kComputeWarps - 1);
    v.t0 = __shfl_sync(0xffffffffu, a0, kComputeWarps - 1);
    v.t1 = __shfl_sync(0xffffffffu, a1, kComputeWarps - 1);
    const int src = warp > 0 ? warp - 1 : 0;
    const bool wf = __shfl_sync(0xffffffffu, f, src);
    const u64 w0 = __shfl_sync(0xffffffffu, a0, src), w1 = __shfl_sync(0xffffffffu, a1, src);
    v.xf = warp > 0 && wf;
    v.x0 = warp > 0 ? w0 : 0;
    v.x1 = warp > 0 ? w1 : 0;
    const bool lf = __shfl_up_sync(0xffffffffu, in_f, 1);
    const u64 l0 = shfl_up64(in0, 1), l1 = shfl_up64(in1, 1);
    if (lane > 0) {
        bool bf = lf;
        u64 b0 = l0, b1 = l1;
        seg_combine(v.xf, v.x0, v.x1, bf, b0, b1);
        v.xf = bf; v.x0 = b0; v.x1 = b1;
    }
    return v;
}

// Right after the tile view: publish the tile aggregate (P if a segment
// starts in the tile -- its tail prefix is then local -- else A), the host
// max end for E, and hand the producer what its epilogue needs.
// hand a device tile's epilogue to the epilogue warp (descriptor ring)
__device__ __forceinline__ void post_info(Ctrl *c, int &k, int64_t t, int cnt, bool head, bool tf, u64 t0, u64 t1,
                                          int st = -1)
{
    const int slot = k % kRing;
    if (k >= kRing) mbar_wait(&c->info_empty[slot], (uint32_t)(((k / kRing) - 1) & 1));
    TileInfo &x = c->info[slot];
    x.t = t;
    x.cnt = cnt;
    x.head = head;
    x.tf = tf;
    x.hcnt = st >= 0 ? c->r0cnt[st] : -1;
    x.r0 = st >= 0 ? c->r0[st] : 0;
    x.t0 = t0;
    x.t1 = t1;
    mbar_arrive(&c->info_full[slot]);
    ++k;
}

template <bool DEV>
__device__ __forceinline__ void publish_tile(const Params &p, const StageSmem &sm, Ctrl *c, const TileCtx &tc,
                                             const TileView &tv, int &k)
{
    const int32_t uni = c->uni[tc.st];   // CSR tile of one resource: its id (sm.r not filled)
    const bool head = tc.cnt > 0 && c->has_prev[tc.st] && rid(sm, uni, 0) == c->prev_res[tc.st];
    if (DEV) publish<2>(tv.tf ? p.d_slotP + 4 * tc.lt : p.d_slotA + 4 * tc.lt, p.epoch, tv.t0, tv.t1);
    else publish<1>(tv.tf ? p.h_slotP + 2 * tc.lt : p.h_slotA + 2 * tc.lt, p.epoch, tv.t0, 0);
    if (head) post_info(c, k, tc.lt, tc.cnt, head, tv.tf, tv.t0, tv.t1, tc.st);
}

// Emit per-resource totals.  A thread's records split into a head piece
// (records before its first segment start -- they continue the left
// neighbour's segment), complete middle segments (emitted in the record
// loop) and a tail piece.  Warps without any segment start reduce with a
// butterfly; otherwise a warp-level segmented scan.  One L2 reduction per
// (segment, warp).  Fields [0, NA) are sums, field NA is a max.
template <int NA>
__device__ __forceinline__ void emit_segments(const u64 (&head)[NA + 1], const u64 (&tail)[NA + 1], uint32_t sfm,
                                              int nv, int32_t first_r, int32_t tail_r, int32_t ids,
                                              u64 *const (&dst)[NA + 1], int lane)
{
    const bool any = nv > 0;
    const bool f = sfm != 0;
    if (__ballot_sync(0xffffffffu, f) == 0) {
        u64 v[NA + 1];
#pragma unroll
        for (int i = 0; i < NA; ++i) v[i] = warp_sum_rx(tail[i]);
        v[NA] = warp_max_rx(tail[NA]);
        const int32_t r = __shfl_sync(0xffffffffu, first_r, 0);
        const bool a0 = __shfl_sync(0xffffffffu, any, 0);
        if (lane == 0 && a0 && r >= 0 && r < ids) {
#pragma unroll
            for (int i = 0; i < NA; ++i)
                if (v[i]) red_add(dst[i] + r, v[i]);
            if (v[NA]) red_max(dst[NA] + r, v[NA]);
        }
        return;
    }
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

// Phase A: segment-start mask, the scan aggregate (max end over the thread's
// LAST segment; devices: v0 kernel-only, v1 all) and the thread's min start /
// max end, from res + end (+ kind) in shared memory.
template <bool DEV>
__device__ __forceinline__ void phase_a(const StageSmem &sm, const Ctrl *c, int st, int b, int nv, uint32_t &sfm,
                                        u64 &v0, u64 &v1, u64 &mn, u64 &mx)
{
    const int32_t uni = c->uni[st];   // CSR tile of one resource: its id (sm.r not filled)
    sfm = 0;
    v0 = v1 = 0;
    mn = ~0ull;
    mx = 0;
    if (nv == 0) return;
    bool hp;
    int32_t pr;
    if (b == 0) {
        hp = c->has_prev[st] != 0;
        pr = c->prev_res[st];
    } else {
        hp = true;
        pr = rid(sm, uni, b - 1);
    }
    mn = sm.s[b];
    u64 ms = 0;   // max START: a (malformed) start above every end must still leave the 2^32 window
#pragma unroll kUnrollG
    for (int j = 0; j < kItems; ++j) {
        if (j < nv) {
            const int32_t r = rid(sm, uni, b + j);
            const u64 e = sm.e[b + j];
            ms = umax(ms, sm.s[b + j]);
            if ((j == 0 && !hp) || r != pr) {
                sfm |= 1u << j;
                mx = umax(mx, DEV ? v1 : v0);
                v0 = 0;
                v1 = 0;
                mn = umin(mn, sm.s[b + j]);
            }
            if (DEV) {
                if (sm.k[b + j] == 0) v0 = umax(v0, e);
                v1 = umax(v1, e);
            } else {
                v0 = umax(v0, e);
            }
            pr = r;
        }
    }
    mx = umax(umax(mx, DEV ? v1 : v0), ms);
}

// record values in the arithmetic domain of phase B: 32-bit tile-relative
// (exact when the tile's time range fits in 32 bits) or absolute 64-bit
template <typename T>
struct Dom;
template <>
struct Dom<uint32_t> {
    u64 base, top;
    uint32_t bl;
    __device__ __forceinline__ Dom(u64 b, u64 t) : base(b), top(t), bl((uint32_t)b) {}
    __device__ __forceinline__ uint32_t ld(const u64 *a, int i) const
    {
        return reinterpret_cast<const uint32_t *>(a)[2 * i] - bl;
    }
    // saturating map of an absolute value into [0, top - base]
    __device__ __forceinline__ uint32_t rel(u64 v) const
    {
        return v <= base ? 0u : (v >= top ? (uint32_t)(top - base) : (uint32_t)(v - base));
    }
    __device__ __forceinline__ u64 abs(uint32_t v) const { return base + v; }
};
template <>
struct Dom<u64> {
    __device__ __forceinline__ Dom(u64, u64) {}
    __device__ __forceinline__ u64 ld(const u64 *a, int i) const { return a[i]; }
    __device__ __forceinline__ u64 rel(u64 v) const { return v; }
    __device__ __forceinline__ u64 abs(u64 v) const { return v; }
};

template <typename T>
__device__ __forceinline__ T tmax(T a, T b) { return a > b ? a : b; }
template <typename T>
__device__ __forceinline__ T tmin(T a, T b) { return a < b ? a : b; }

struct Pieces3 {
    u64 head[3], cur[3];
    bool head_open;
    int32_t cur_r, first_r;
    bool cur_decl;
};

// close the running piece at a segment start: the first piece becomes the
// head piece, later ones are complete segments inside the thread
__device__ __forceinline__ void close_piece(Pieces3 &P, int32_t ids, u64 *d0, u64 *d1, u64 *d2)
{
    if (P.head_open) {
        P.head[0] = P.cur[0]; P.head[1] = P.cur[1]; P.head[2] = P.cur[2];
    } else if (P.cur_r >= 0 && P.cur_r < ids) {
        if (P.cur[0]) red_add(d0 + P.cur_r, P.cur[0]);
        if (P.cur[1]) red_add(d1 + P.cur_r, P.cur[1]);
        if (P.cur[2]) red_max(d2 + P.cur_r, P.cur[2]);
    }
    P.head_open = false;
}

// =========================================================================
// per-thread 64-bit rescan for threads whose fast pass flagged anything
// rare: findings lists (model.py:192-228), clamp counts (summarize.py:113),
// canonical-order contract.  Exact for any input, including records whose
// ends wrap the 32-bit tile-relative domain (malformed).
// =========================================================================
template <bool DEV>
__device__ __noinline__ void rescan(const Params &p, const StageSmem &sm, const Ctrl *c, int st, int b, int nv,
                                    u64 x0, u64 E, bool late_check, int64_t gi0)
{
    const int32_t uni = c->uni[st];   // CSR tile of one resource: its id (sm.r not filled)
    bool hp = true;
    int32_t pr = 0;
    u64 ps = 0;
    if (b == 0) {
        hp = c->has_prev[st] != 0;
        pr = c->prev_res[st];
        ps = c->prev_start[st];
    } else {
        pr = rid(sm, uni, b - 1);
        ps = sm.s[b - 1];
    }
    int32_t r = rid(sm, uni, b);
    bool decl = DEV ? declared(p.dev_decl, p.dev_ids, p.m, r) : declared(p.host_decl, p.host_ids, p.n, r);
    u64 run = x0;
    int bad = -1;
    for (int j = 0; j < nv; ++j) {
        const int32_t rj = rid(sm, uni, b + j);
        const u64 s = sm.s[b + j], e = sm.e[b + j];
        const bool h = j > 0 || hp;
        if (!h || rj != pr) {
            if (bad < 0 && h && rj < pr) bad = j;
            r = rj;
            decl = DEV ? declared(p.dev_decl, p.dev_ids, p.m, r) : declared(p.host_decl, p.host_ids, p.n, r);
            run = 0;
        } else if (bad < 0 && s < ps) {
            bad = j;
        }
        const int64_t gi = gi0 + j;
        if (DEV) {
            if (s > e) push(p, 4, gi);
            else if (s == e) push(p, 5, gi);
            if (!decl) push(p, 6, gi);
            if (e > E) {
                if (late_check) push(p, 7, gi);
                if (r >= 0 && r < p.dev_ids) red_add(p.d_clamp + r, 1ull);
            }
        } else {
            if (s > e) push(p, 0, gi);
            else if (s == e) push(p, 1, gi);
            if (!decl) push(p, 2, gi);
            else if (s < e && s < run) push(p, 3, gi);
            run = umax(run, e);
        }
        pr = rj;
        ps = s;
    }
    if (bad >= 0) contract(p, DEV ? 2u : 1u, gi0 + bad);
}

// =========================================================================
// HOST records: per-rank sums + span (summarize.py:57-92) -- no scan.
//
// Only usable records (positive length) take part in the overlap check
// (model.py:197-215).  With start-sorted records: if every usable record
// starts at or after the end of the previous usable record, usable ends are
// non-decreasing, so that end IS the running max and no usable record
// overlaps any earlier one -- the check is exact by induction.  The first
// violation is a real overlap: it raises ovl_suspect and the exact findings
// come from the error-path kernels (overlap_pass) before the finalize.
// span_end is the last usable end unless a thread holds zero-length /
// malformed records; those threads re-emit exact maxima in host_rare.
// =========================================================================
__device__ __noinline__ u64 host_rare(const Params &p, const StageSmem &sm, const Ctrl *c, int st, int b, int nv,
                                      int64_t gi0)
{
    const int32_t uni = c->uni[st];   // CSR tile of one resource: its id (sm.r not filled)
    bool hp = true;
    int32_t pr = 0;
    u64 ps = 0;
    if (b == 0) {
        hp = c->has_prev[st] != 0;
        pr = c->prev_res[st];
        ps = c->prev_start[st];
    } else {
        pr = rid(sm, uni, b - 1);
        ps = sm.s[b - 1];
    }
    bool decl = false, ovl = false;
    int32_t cur = 0;
    u64 mx = 0, seg = 0, pe = 0;
    int bad = -1;
    // end of the last usable record before this thread, when at hand (else: conservative)
    bool pe_known = true;
    {
        int q = b - 1;
        while (q >= 0 && rid(sm, uni, q) == rid(sm, uni, b) && sm.s[q] >= sm.e[q]) --q;
        if (q >= 0 && rid(sm, uni, q) == rid(sm, uni, b)) pe = sm.e[q];
        else if (q < 0 && hp && pr == rid(sm, uni, b)) {
            if (b == 0 && c->prev_start[st] < c->prev_end[st]) pe = c->prev_end[st];
            else pe_known = false;
        }
    }
    for (int j = 0; j < nv; ++j) {
        const int32_t r = rid(sm, uni, b + j);
        const u64 s = sm.s[b + j], e = sm.e[b + j];
        const bool h = j > 0 || hp;
        const bool start = !h || r != pr;
        if (start) {
            if (bad < 0 && h && r < pr) bad = j;
        } else if (bad < 0 && s < ps) {
            bad = j;
        }
        if (j == 0 || start) {
            if (j > 0 && seg && cur >= 0 && cur < p.host_ids) red_max(p.h_span + cur, seg);
            if (start) { pe = 0; pe_known = true; }
            cur = r;
            seg = 0;
            decl = declared(p.host_decl, p.host_ids, p.n, r);
        }
        if (s < e) {   // usable: adjacent overlap check against the last usable end
            if (s < pe || !pe_known) ovl = true;
            pe = e;
            pe_known = true;
        }
        const int64_t gi = gi0 + j;
        if (s > e) push(p, 0, gi);
        else if (s == e) push(p, 1, gi);
        if (!decl) push(p, 2, gi);
        mx = umax(mx, e);
        seg = umax(seg, e);
        pr = r;
        ps = s;
    }
    if (nv > 0 && seg && cur >= 0 && cur < p.host_ids) red_max(p.h_span + cur, seg);   // exact span maxima
    if (bad >= 0) contract(p, 1u, gi0 + bad);
    if (ovl && !*(volatile unsigned *)&p.g->ovl_suspect) atomicOr(&p.g->ovl_suspect, 1u);
    return mx;
}

// Fast path for a thread whose records all belong to one rank and lie in one
// aligned 2^32 ns window: every check and sum in 32 bits relative to the
// window.  Returns false (results unused) if a record leaves the window.
template <bool FULL>
__device__ __forceinline__ bool host_fast32(const StageSmem &sm, int b, int nv, bool cont, u64 ps64, u64 pe64,
                                            bool &rare, bool &ovl, u64 &off, u64 &mpi, u64 &last)
{
    if (FULL) nv = kItems;   // full tiles: the guard below folds away
    // the ALIGNED 2^32 window holding the thread's first start: relative values are the
    // low words and the window test is one compare of the high word per value
    const u64 first = sm.s[b];
    const u64 base = first & 0xffffffff00000000ull;
    const uint32_t bh = (uint32_t)(base >> 32), bl = (uint32_t)base;   // bl == 0
    // the previous record of the same rank (cont): order (64-bit), usable end clamped into the window
    uint32_t ps = 0, pe = 0;
    if (cont) {
        rare = rare || ps64 > first;                                    // order
        pe = pe64 <= base ? 0u : (pe64 - base > 0xffffffffull ? 0xffffffffu : (uint32_t)(pe64 - base));
    }
    bool out = false;
    uint32_t o = 0, m = 0, l = 0;
#pragma unroll kUnrollB
    for (int j = 0; j < kItems; ++j) {
        if (j < nv) {
            const int i = b + j;
            const u64 s64 = sm.s[i], e64 = sm.e[i];   // conflict-free LDS.64 at the odd record stride
            const uint32_t sl = (uint32_t)s64, sh = (uint32_t)(s64 >> 32), el = (uint32_t)e64, eh = (uint32_t)(e64 >> 32);
            const uint8_t k = sm.k[i];
            out = out || sh != bh || eh != bh;   // outside [base, base + 2^32)
            const uint32_t s = sl - bl, e = el - bl;
            rare = rare || (j > 0 && s < ps) || s >= e;   // order / zero-length / malformed
            const bool usable = s < e;
            ovl = ovl || (usable && s < pe);
            pe = usable ? e : pe;
            l = usable ? e : l;
            const uint32_t d = e - s;
            o += k == 1 ? d : 0u;
            m += k == 2 ? d : 0u;
            ps = s;
        }
    }
    off = o;
    mpi = m;
    last = base + l;
    return !out;
}

// Single-rank host tile (the common case: ~9 tiles per rank at C2): no segment
// flags or head pieces, every thread's records continue one rank, the per-thread
// 32-bit sums leave through REDUX (two 16-bit limbs) and one RED per field per warp.
// Per warp: returns false (nothing emitted) if some lane leaves its 2^32 window --
// that warp then runs the general path (host tiles need no CTA barrier).
__device__ __forceinline__ bool host_single(const Params &p, const StageSmem &sm, Ctrl *c, TileCtx &tc,
                                            int tid, Phases &ph)
{
    const int32_t uni = c->uni[tc.st];   // CSR tile of one resource: its id (sm.r not filled)
    ph.mark();
    const int lane = tid & 31;
    const int b = tid * kItems;
    constexpr int nv = kItems;   // full tiles only (host_compute)
    const int64_t gi0 = tc.gbase + (int64_t)b;
    const int32_t r0 = rid(sm, uni, 0);
    const bool has_prev = c->has_prev[tc.st] != 0;
    const int32_t prev_res = c->prev_res[tc.st];
    bool cont = true, ovl = false, rare = false;
    u64 ps = 0, pe = 0;   // previous start; end of the previous USABLE record of the rank
    if (nv > 0) {
        if (b == 0) {
            cont = has_prev && prev_res == r0;
            ps = c->prev_start[tc.st];
            pe = c->prev_end[tc.st];
            ovl = cont && ps >= pe;                     // previous record not usable: conservative
            rare = has_prev && !cont && r0 < prev_res;  // rank order across the tile boundary
        } else {
            ps = sm.s[b - 1];
            int q = b - 1;
            while (q >= 0 && sm.s[q] >= sm.e[q]) --q;   // rare: skip non-usable records
            if (q >= 0) pe = sm.e[q];
            else ovl = has_prev && prev_res == r0;
        }
        rare = rare || !declared(p.host_decl, p.host_ids, p.n, r0);
    }
    u64 off = 0, mpi = 0, last = 0;
    const bool ok = host_fast32<true>(sm, b, nv, cont, ps, pe, rare, ovl, off, mpi, last);
    if (!__all_sync(0xffffffffu, ok)) return false;
    u64 tmax = last;
    if (ovl && !*(volatile unsigned *)&p.g->ovl_suspect) atomicOr(&p.g->ovl_suspect, 1u);
    if (rare || ovl) tmax = host_rare(p, sm, c, tc.st, b, nv, gi0);
    ph.add(ph.hb);
    // 32-bit thread sums (disjoint durations inside one 2^32 window)
    const u64 so = warp_sum32((uint32_t)off), sp = warp_sum32((uint32_t)mpi);
    const u64 sl = warp_max_rx(last), wm = warp_max_rx(tmax);
    if (lane == 0) {
        if (r0 >= 0 && r0 < p.host_ids) {
            if (so) red_add(p.h_off + r0, so);
            if (sp) red_add(p.h_mpi + r0, sp);
            if (sl) red_max(p.h_span + r0, sl);
        }
        // tile max end for E (summarize.py:88-89): warp max -> CTA (smem) -> one RED per tile
        atomicMax(&c->h_max[tc.st], wm);
        __threadfence_block();
        if (atomicAdd(&c->h_cnt[tc.st], 1u) == kComputeWarps - 1) {
            const u64 m = atomicExch(&c->h_max[tc.st], 0ull);
            c->h_cnt[tc.st] = 0;
            red_max(&p.g->host_max_end, m);
        }
    }
    ph.add(ph.hemit);
    return true;
}

__device__ __forceinline__ void host_compute(const Params &p, const StageSmem &sm, Ctrl *c, TileCtx &tc,
                                             int tid, Phases &ph)
{
    const int32_t uni = c->uni[tc.st];   // CSR tile of one resource: its id (sm.r not filled)
#ifndef HB_NO_HOST_SINGLE
    // full single-rank tiles (every tile but the last of the side): the unguarded fast path
    if (tc.cnt == kTile && rid(sm, uni, 0) == rid(sm, uni, tc.cnt - 1) && host_single(p, sm, c, tc, tid, ph)) return;
#endif
    ph.mark();
    const int warp = tid >> 5, lane = tid & 31;
    const int b = tid * kItems;
    const int nv = max(0, min(kItems, tc.cnt - b));
    const int64_t gi0 = tc.gbase + (int64_t)b;
    bool hp = true, ovl = false;
    int32_t pr = 0;
    u64 ps = 0, pe = 0;   // previous start; end of the previous USABLE record of the segment
    if (nv > 0) {
        if (b == 0) {
            hp = c->has_prev[tc.st] != 0;
            pr = c->prev_res[tc.st];
            ps = c->prev_start[tc.st];
            pe = c->prev_end[tc.st];
            // previous record not usable: its predecessors are not at hand -> conservative
            ovl = hp && ps >= pe && rid(sm, uni, 0) == pr;
        } else {
            pr = rid(sm, uni, b - 1);
            ps = sm.s[b - 1];
            int q = b - 1;
            while (q >= 0 && rid(sm, uni, q) == pr && sm.s[q] >= sm.e[q]) --q;   // rare: skip non-usable records
            if (q >= 0 && rid(sm, uni, q) == pr) pe = sm.e[q];
            else ovl = c->has_prev[tc.st] && rid(sm, uni, 0) == c->prev_res[tc.st] && rid(sm, uni, 0) == pr;
        }
    }
    Pieces3 P;
    P.head[0] = P.head[1] = P.head[2] = 0;
    P.cur[0] = P.cur[1] = P.cur[2] = 0;
    P.head_open = true;
    P.cur_r = P.first_r = nv ? rid(sm, uni, b) : 0;
    P.cur_decl = nv ? declared(p.host_decl, p.host_ids, p.n, P.cur_r) : false;
    uint32_t sfm = 0;
    bool rare = nv > 0 && !P.cur_decl;
    u64 off = 0, mpi = 0, last = 0, tmax = 0;
    // one rank inside the thread (and in one 2^32 window): the 32-bit fast path
    bool done = false;
    if (nv > 0 && rid(sm, uni, b) == rid(sm, uni, b + nv - 1)) {
        const bool cont = hp && pr == rid(sm, uni, b);
        bool r2 = rare, o2 = ovl;
        u64 of2, mp2, la2;
        if (host_fast32<false>(sm, b, nv, cont, ps, pe, r2, o2, of2, mp2, la2)) {
            if (!cont) {
                sfm = 1u;
                P.head_open = false;
                r2 = r2 || (hp && rid(sm, uni, b) < pr);   // rank order across the segment start
            }
            rare = r2;
            ovl = o2;
            off = of2;
            mpi = mp2;
            last = la2;
            done = true;
        }
    }
#pragma unroll kUnrollG
    for (int j = 0; j < kItems; ++j) {
        if (!done && j < nv) {
            const int32_t r = rid(sm, uni, b + j);
            const u64 s = sm.s[b + j], e = sm.e[b + j];
            const uint8_t k = sm.k[b + j];
            if ((j == 0 && !hp) || r != pr) {
                sfm |= 1u << j;
                rare = rare || ((j > 0 || hp) && r < pr);
                if (j > 0) {
                    P.cur[0] = off; P.cur[1] = mpi; P.cur[2] = last;
                    close_piece(P, p.host_ids, p.h_off, p.h_mpi, p.h_span);
                    tmax = umax(tmax, last);
                    P.cur_r = r;
                    P.cur_decl = declared(p.host_decl, p.host_ids, p.n, r);
                    rare = rare || !P.cur_decl;
                }
                P.head_open = P.head_open && j > 0;
                off = mpi = last = 0;
                pe = 0;
            } else {
                rare = rare || s < ps;          // canonical order
            }
            const bool usable = s < e;
            ovl = ovl || (usable && s < pe);   // usable record before the last usable end
            rare = rare || !usable;             // zero-length / malformed
            pe = usable ? e : pe;
            last = usable ? e : last;
            const u64 d = e - s;
            if (k == 1) off += d;
            if (k == 2) mpi += d;
            pr = r;
            ps = s;
        }
    }
    P.cur[0] = off; P.cur[1] = mpi; P.cur[2] = last;
    tmax = umax(tmax, last);
    if (ovl && !*(volatile unsigned *)&p.g->ovl_suspect) atomicOr(&p.g->ovl_suspect, 1u);
    if (rare || ovl) tmax = host_rare(p, sm, c, tc.st, b, nv, gi0);
    ph.add(ph.hb);
    if (P.head_open) { P.head[0] = P.head[1] = P.head[2] = 0; }
    u64 *const dst[3] = {p.h_off, p.h_mpi, p.h_span};
    emit_segments<2>(P.head, P.cur, sfm, nv, P.first_r, P.cur_r, p.host_ids, dst, lane);
    // tile max end for E (summarize.py:88-89): warp max -> CTA (smem) -> one RED per tile
    const u64 wm = warp_max_rx(tmax);
    if (lane == 0) {
        atomicMax(&c->h_max[tc.st], wm);
        __threadfence_block();
        if (atomicAdd(&c->h_cnt[tc.st], 1u) == kComputeWarps - 1) {
            const u64 m = atomicExch(&c->h_max[tc.st], 0ull);
            c->h_cnt[tc.st] = 0;
            red_max(&p.g->host_max_end, m);
        }
    }
    ph.add(ph.hemit);
    (void)warp;
}

// =========================================================================
// DEVICE records: dual running-max union scan (summarize.py:95-138)
// =========================================================================
// fast pass; returns true if the thread needs the 64-bit rescan
template <typename T>
__device__ __forceinline__ bool dev_phase_b(const Params &p, const StageSmem &sm, const Ctrl *c, int st, int b, int nv,
                                            uint32_t sfm, const TileView &tv, Pieces3 &P, u64 E)
{
    const int32_t uni = c->uni[st];   // CSR tile of one resource: its id (sm.r not filled)
    const Dom<T> D(tv.base, tv.top);
    const T Er = D.rel(E);                  // <= top - base: also catches ends that wrap below the base
    bool rare = E < tv.base;                // every record of the tile ends after E
    T runK = tmin(D.rel(tv.x0), Er), runKM = tmin(D.rel(tv.x1), Er), cK = 0, cKM = 0, ps = 0;
    bool hp = true;
    int32_t pr = 0;
    if (b == 0) {
        hp = c->has_prev[st] != 0;
        pr = c->prev_res[st];
        rare = rare || (hp && nv > 0 && !(sfm & 1u) && sm.s[0] < c->prev_start[st]);
    } else {
        pr = rid(sm, uni, b - 1);
        ps = D.ld(sm.s, b - 1);
    }
#pragma unroll kUnrollG
    for (int j = 0; j < kItems; ++j) {
        if (j < nv) {
            const T s0 = D.ld(sm.s, b + j), e0 = D.ld(sm.e, b + j);
            const uint8_t k = sm.k[b + j];
            if ((sfm >> j) & 1u) {
                const int32_t r = rid(sm, uni, b + j);
                rare = rare || ((j > 0 || hp) && r < pr);
                if (j > 0) {
                    P.cur[0] = cK; P.cur[1] = cKM; P.cur[2] = D.abs(runKM);
                    close_piece(P, p.dev_ids, p.d_k, p.d_km, p.d_maxend);
                }
                P.cur_r = r;
                pr = r;
                P.cur_decl = declared(p.dev_decl, p.dev_ids, p.m, r);
                rare = rare || !P.cur_decl;
                cK = cKM = 0;
                runK = runKM = 0;
            } else if (j > 0 || b > 0) {
                rare = rare || s0 < ps;
            }
            rare = rare || s0 >= e0 || e0 > Er;     // zero-length / malformed / clamped
            const T e = tmin(e0, Er), s = tmin(s0, e);
            const T loKM = tmax(runKM, s);
            runKM = tmax(runKM, e);
            cKM += runKM - loKM;
            if (k == 0) {
                const T loK = tmax(runK, s);
                runK = tmax(runK, e);
                cK += runK - loK;
            }
            ps = s0;
        }
    }
    P.cur[0] = cK; P.cur[1] = cKM; P.cur[2] = D.abs(runKM);
    return rare;
}

// E once per warp, after the CTA barrier
__device__ __forceinline__ u64 device_E(const Params &p, int tid, int lane, u64 &E_cache, bool &E_known,
                                        int &hpend)
{
    if (!E_known) {
        if (tid == 0 && hpend > 0) host_tiles_done(p, hpend);   // every warp of this CTA is past its host tiles
        hpend = 0;
        u64 E = 0;
        if (lane == 0) E = device_window(p);
        E_cache = __shfl_sync(0xffffffffu, E, 0);
        E_known = true;
    }
    return E_cache;
}

// -------------------------------------------------------------------------
// Single-segment device tile (every record of one device -- the common case):
// no segment flags, the tile base is its first start (records are
// start-sorted), every running max is a plain 32-bit max relative to it.
// Each thread needs its tile-exclusive carry X (the running max of the ends
// before its records), known only after the CTA barrier.  Two schedules, chosen
// per warp from its previous device tile:
//  * ONE pass (serialized streams): before the barrier, the union pieces
//    c = max(run, e) - max(run, min(s, e)) with carry 0 and unclamped ends,
//    plus the thread's max ends (the scan aggregate).  X only changes the
//    records j with max(run_j, s_j) < X -- none when the thread's first start
//    is >= X; otherwise an early-exit correction over that prefix.  A thread
//    with an end beyond E redoes its pass clamped (records after the last
//    host end: rare).  A warp that needed a correction switches to
//  * TWO passes (overlapping streams): max ends (kept in registers) before the
//    barrier, the union pass with the carry after it -- and back to one pass
//    once no lane starts below its carry.
// Starts / ends outside the base's 2^32 window: ends -> the general path
// (tile-wide, decided after the barrier), starts -> findings (rescan).
// Returns false (nothing done) if some end leaves the window.
// -------------------------------------------------------------------------
template <bool MERGED>
__device__ __forceinline__ bool dev_single(const Params &p, const StageSmem &sm, Ctrl *c, TileCtx &tc, int tid,
                                           u64 &E_cache, bool &E_known, int &hpend, int &kq, bool &one_pass,
                                           Phases &ph)
{
    const int32_t uni = c->uni[tc.st];   // CSR tile of one resource: its id (sm.r not filled)
    ph.mark();
    const int warp = tid >> 5, lane = tid & 31;
    const int b = tid * kItems;
    constexpr int nv = kItems;   // full tiles only (dev_compute): the per-record guards fold away
    const int64_t gi0 = tc.gbase + (int64_t)b;
    // the ALIGNED 2^32 ns window holding the tile's first start: relative values are the
    // low words, one high-word compare per value tests the window
    const u64 base = sm.s[0] & 0xffffffff00000000ull;
    const uint32_t bl = (uint32_t)base, bh = (uint32_t)(base >> 32);   // bl == 0
    constexpr bool merged = MERGED;
    uint32_t runK = 0, runKM = 0, cK = 0, cKM = 0, ps = 0;
    uint32_t er[MERGED ? 1 : kItems], sr[MERGED ? 1 : kItems];
    uint32_t kmask = 0;             // bit j: record j is a kernel
    bool out = false, bad = false;  // bad: start outside the window / order / zero-length / malformed
    if (b > 0) {   // the predecessor's start (order of the first record): exact only inside the window
        const u64 p64 = sm.s[b - 1];
        ps = (uint32_t)p64 - bl;
        bad = (uint32_t)(p64 >> 32) != bh;
    }
    if constexpr (merged) {
        er[0] = 0;
#pragma unroll kUnrollB
        for (int j = 0; j < kItems; ++j) {
            if (j < nv) {
                const u64 s64 = sm.s[b + j], e64 = sm.e[b + j];   // conflict-free LDS.64 at the odd record stride
                const uint32_t sl = (uint32_t)s64, el = (uint32_t)e64;
                out = out || (uint32_t)(e64 >> 32) != bh;
                const uint32_t s0 = sl - bl, e = el - bl;
                bad = bad || (uint32_t)(s64 >> 32) != bh || ((j > 0 || b > 0) && s0 < ps) || s0 >= e;
                const uint32_t s = min(s0, e);
                const uint32_t loKM = max(runKM, s);
                runKM = max(runKM, e);
                cKM += runKM - loKM;
                if (sm.k[b + j] == 0) {
                    const uint32_t loK = max(runK, s);
                    runK = max(runK, e);
                    cK += runK - loK;
                }
                ps = s0;
            }
        }
    } else {
        // starts are loaded (and window-checked) here too, so the pass after the
        // barrier -- where every warp resumes at once -- runs on registers alone
#pragma unroll kUnrollA
        for (int j = 0; j < kItems; ++j) {
            er[j] = 0;
            sr[j] = 0;
            if (j < nv) {
                const u64 e64 = sm.e[b + j], s64 = sm.s[b + j];
                const uint32_t e = (uint32_t)e64 - bl, sl = (uint32_t)s64, s0 = sl - bl;
                out = out || (uint32_t)(e64 >> 32) != bh;
                bad = bad || (uint32_t)(s64 >> 32) != bh || ((j > 0 || b > 0) && s0 < ps) || s0 >= e;
                ps = s0;
                er[MERGED ? 0 : j] = e;
                sr[MERGED ? 0 : j] = s0;
                runKM = max(runKM, e);
                if (sm.k[b + j] == 0) { runK = max(runK, e); kmask |= 1u << j; }
            }
        }
    }
    const bool fit_w = __all_sync(0xffffffffu, !out);
    uint32_t vK = runK, vKM = runKM;   // the thread's max (unclamped) ends: scan aggregate
    warp_max_scan2(vK, vKM, lane);
    if (lane == 31) { c->f_k[tc.st][warp] = vK; c->f_km[tc.st][warp] = vKM; c->f_fit[tc.st][warp] = fit_w; }
    ph.add(ph.a);
    bar_compute();
    ph.add(ph.hn2);
    const u64 E = device_E(p, tid, lane, E_cache, E_known, hpend);
    // tile-wide: all warps in the window?  cross-warp exclusive prefix
    uint32_t wK = 0, wKM = 0;
    bool fit = true;
    if (lane < kComputeWarps) { wK = c->f_k[tc.st][lane]; wKM = c->f_km[tc.st][lane]; fit = c->f_fit[tc.st][lane] != 0; }
    if (!__all_sync(0xffffffffu, fit)) return false;
    // the max over earlier warps: one predicated REDUX each, no shuffle scan
    const uint32_t xwK = __reduce_max_sync(0xffffffffu, lane < warp ? wK : 0u);
    const uint32_t xwKM = __reduce_max_sync(0xffffffffu, lane < warp ? wKM : 0u);
    uint32_t xK = __shfl_up_sync(0xffffffffu, vK, 1), xKM = __shfl_up_sync(0xffffffffu, vKM, 1);
    if (lane == 0) { xK = 0; xKM = 0; }
    xK = max(xK, xwK);
    xKM = max(xKM, xwKM);
    const bool head = c->has_prev[tc.st] && rid(sm, uni, 0) == c->prev_res[tc.st];
    ph.add(ph.bar);
    if (warp == 0) {
        // tile aggregate (warp 0 only): the max over every warp
        const uint32_t tK = __reduce_max_sync(0xffffffffu, wK), tKM = __reduce_max_sync(0xffffffffu, wKM);
        if (lane == 0) {
            // a segment starts here iff the tile does not continue one
            publish<2>(!head ? p.d_slotP + 4 * tc.lt : p.d_slotA + 4 * tc.lt, p.epoch, base + tK, base + tKM);
            if (head) post_info(c, kq, tc.lt, tc.cnt, true, false, base + tK, base + tKM, tc.st);
        }
    }
    ph.add(ph.hb);
    const uint32_t Er = E <= base ? 0u : (E - base > 0xffffffffull ? 0xffffffffu : (uint32_t)(E - base));
    const int32_t r0 = rid(sm, uni, 0);
    const bool decl = declared(p.dev_decl, p.dev_ids, p.m, r0);
    const bool clamp = nv > 0 && (E < base || runKM > Er);   // some end beyond E
    bool rare = clamp || !decl;
    if (b == 0) rare = rare || (head && nv > 0 && sm.s[0] < c->prev_start[tc.st]);
    const uint32_t XK = min(xK, Er), XKM = min(xKM, Er);
    const uint32_t s_first = nv > 0 ? (uint32_t)sm.s[b] - bl : 0xffffffffu;
    const bool need = !clamp && s_first < XKM;   // the carry reaches into this thread's records
    one_pass = !__any_sync(0xffffffffu, need);
#ifdef HB_PROF
    ph.mg += merged;
    ph.nd += !one_pass;
#endif
    if constexpr (!merged) {
        // the union pass with the tile-exclusive carry and clamped ends
        runK = XK; runKM = XKM;
#pragma unroll kUnrollB
        for (int j = 0; j < kItems; ++j) {
            if (j < nv) {
                const uint32_t s0 = sr[MERGED ? 0 : j], e0 = er[MERGED ? 0 : j];
                const uint32_t e = min(e0, Er), s = min(s0, e);
                const uint32_t loKM = max(runKM, s);
                runKM = max(runKM, e);
                cKM += runKM - loKM;
                if ((kmask >> j) & 1u) {
                    const uint32_t loK = max(runK, s);
                    runK = max(runK, e);
                    cK += runK - loK;
                }
            }
        }
    } else if (clamp) {
        // the exact pass with the carry and clamped ends
        runK = XK; runKM = XKM; cK = cKM = 0;
        for (int j = 0; j < nv; ++j) {
            const uint32_t s0 = (uint32_t)sm.s[b + j] - bl;
            const uint32_t e = min((uint32_t)sm.e[b + j] - bl, Er), s = min(s0, e);
            const uint32_t loKM = max(runKM, s);
            runKM = max(runKM, e);
            cKM += runKM - loKM;
            if (sm.k[b + j] == 0) {
                const uint32_t loK = max(runK, s);
                runK = max(runK, e);
                cK += runK - loK;
            }
        }
    } else if (need) {
        // carry correction over the prefix the carry reaches (no end exceeds E here)
        uint32_t rK = 0, rKM = 0;
        for (int j = 0; j < nv && (rKM < XKM || rK < XK); ++j) {
            const uint32_t s0 = (uint32_t)sm.s[b + j] - bl, e = (uint32_t)sm.e[b + j] - bl, s = min(s0, e);
            if (rKM < XKM) {
                const uint32_t lo = max(rKM, s);
                cKM -= (max(rKM, e) - lo) - (max(XKM, e) - max(XKM, s));
            }
            rKM = max(rKM, e);
            if (sm.k[b + j] == 0) {
                if (rK < XK) {
                    const uint32_t lo = max(rK, s);
                    cK -= (max(rK, e) - lo) - (max(XK, e) - max(XK, s));
                }
                rK = max(rK, e);
            }
        }
    }
    rare = rare || bad;
    if (rare) rescan<true>(p, sm, c, tc.st, b, nv, 0, E, (p.mode == kReport || p.mode == kValidate) && p.n >= 1, gi0);
    ph.add(ph.b);
    // one piece for the whole tile: warp reductions, one RED per field per warp
    const u64 sK = warp_sum32(cK), sKM = warp_sum32(cKM);
    const uint32_t mx = __reduce_max_sync(0xffffffffu, nv > 0 ? min(runKM, Er) : 0u);
    if (lane == 0 && r0 >= 0 && r0 < p.dev_ids) {
        if (sK) red_add(p.d_k + r0, sK);
        if (sKM) red_add(p.d_km + r0, sKM);
        red_max(p.d_maxend + r0, base + mx);
    }
    ph.add(ph.emit);
    return true;
}

__device__ __forceinline__ void dev_general(const Params &p, const StageSmem &sm, Ctrl *c, const TileCtx &tc, int tid,
                                  u64 &E_cache, bool &E_known, int &hpend, int &k, Phases &ph);

__device__ __forceinline__ void dev_compute(const Params &p, const StageSmem &sm, Ctrl *c, TileCtx &tc, int tid,
                                            u64 &E_cache, bool &E_known, int &hpend, int &k, bool &one_pass,
                                            Phases &ph)
{
    const int32_t uni = c->uni[tc.st];   // CSR tile of one resource: its id (sm.r not filled)
    // full single-device tiles (every tile but the last of the side): the unguarded fast path
    if (tc.cnt == kTile && rid(sm, uni, 0) == rid(sm, uni, tc.cnt - 1)) {
#if HB_DEV_SCHED == 0
        const bool done = dev_single<false>(p, sm, c, tc, tid, E_cache, E_known, hpend, k, one_pass, ph);
#elif HB_DEV_SCHED == 1
        const bool done = dev_single<true>(p, sm, c, tc, tid, E_cache, E_known, hpend, k, one_pass, ph);
#else
        const bool done = one_pass ? dev_single<true>(p, sm, c, tc, tid, E_cache, E_known, hpend, k, one_pass, ph)
                                   : dev_single<false>(p, sm, c, tc, tid, E_cache, E_known, hpend, k, one_pass, ph);
#endif
        if (done) return;
    }
    dev_general(p, sm, c, tc, tid, E_cache, E_known, hpend, k, ph);
}

// tiles holding several devices (or leaving the 2^32 window): segmented scans, 64-bit fallback
__device__ __forceinline__ void dev_general(const Params &p, const StageSmem &sm, Ctrl *c, const TileCtx &tc, int tid,
                                  u64 &E_cache, bool &E_known, int &hpend, int &k, Phases &ph)
{
    const int32_t uni = c->uni[tc.st];   // CSR tile of one resource: its id (sm.r not filled)
    ph.mark();
    const int warp = tid >> 5, lane = tid & 31;
    const int b = tid * kItems;
    const int nv = max(0, min(kItems, tc.cnt - b));
    const int64_t gi0 = tc.gbase + (int64_t)b;
    uint32_t sfm;
    u64 in0, in1, mn, mx;
    phase_a<true>(sm, c, tc.st, b, nv, sfm, in0, in1, mn, mx);
    bool in_f = sfm != 0;
    warp_seg_max(in_f, in0, in1, lane);
    mn = warp_min_rx(mn);
    mx = warp_max_rx(mx);
    if (lane == 31) { c->w_flag[tc.st][warp] = in_f; c->w_v0[tc.st][warp] = in0; c->w_v1[tc.st][warp] = in1; }
    if (lane == 0) { c->w_mn[tc.st][warp] = mn; c->w_mx[tc.st][warp] = mx; }
    ph.add(ph.a);
    bar_compute();
    device_E(p, tid, lane, E_cache, E_known, hpend);
    const u64 E = E_cache;
    const bool late_check = (p.mode == kReport || p.mode == kValidate) && p.n >= 1;
    const TileView tv = tile_view(c, tc.st, warp, lane, in_f, in0, in1);
    if (tid == 0) publish_tile<true>(p, sm, c, tc, tv, k);
    ph.add(ph.bar);
    Pieces3 P;
    P.head[0] = P.head[1] = P.head[2] = 0;
    P.cur[0] = P.cur[1] = P.cur[2] = 0;
    P.head_open = !(sfm & 1u);
    P.cur_r = P.first_r = nv ? rid(sm, uni, b) : 0;
    P.cur_decl = nv ? declared(p.dev_decl, p.dev_ids, p.m, P.cur_r) : false;
    const bool rare = tv.fits32 ? dev_phase_b<uint32_t>(p, sm, c, tc.st, b, nv, sfm, tv, P, E)
                                : dev_phase_b<u64>(p, sm, c, tc.st, b, nv, sfm, tv, P, E);
    if (rare) rescan<true>(p, sm, c, tc.st, b, nv, 0, E, late_check, gi0);
    ph.add(ph.b);
    if (P.head_open) { P.head[0] = P.head[1] = P.head[2] = 0; }
    u64 *const dst[3] = {p.d_k, p.d_km, p.d_maxend};
    emit_segments<2>(P.head, P.cur, sfm, nv, P.first_r, P.cur_r, p.dev_ids, dst, lane);
    ph.add(ph.emit);
}

// =========================================================================
// producer-side tile epilogue, run after the stage was refilled: look back
// for the carry, publish P, and correct the tile's head segment (the compute
// warps used carry 0) reading the few affected records from global memory
// =========================================================================

__device__ void dev_epilogue(const Params &p, const TileInfo &x, int lane, u64 &E_cache, bool &E_known)
{
    // the first 32 records are loaded before the look-back (overlapped round trips)
    const int64_t g0 = x.t * kTile;
    const u64 *S = p.ds + g0, *En = p.de + g0;
    const bool csr = x.hcnt >= 0;   // CSR: the head segment is the tile's first hcnt records
    const int32_t *R = csr ? nullptr : p.dr + g0;
    const uint8_t *K = p.dk + g0;
    int32_t rj = -1;
    u64 sj = 0, ej = 0;
    uint8_t kj = 1;
    if (lane < x.cnt) {
        rj = csr ? (lane < x.hcnt ? x.r0 : -1) : __ldcg(R + lane);
        sj = __ldcg(S + lane); ej = __ldcg(En + lane); kj = __ldcg(K + lane);
    }
    u64 ck, ckm;
    look_back<2>(p.d_slotA, p.d_slotP, x.t, p.epoch, lane, ck, ckm);
    if (!x.tf && lane == 0) publish<2>(p.d_slotP + 4 * x.t, p.epoch, umax(ck, x.t0), umax(ckm, x.t1));
    if (!E_known) {
        u64 Ew = 0;
        if (lane == 0) Ew = device_window(p);
        E_cache = __shfl_sync(0xffffffffu, Ew, 0);
        E_known = true;
    }
    const u64 E = E_cache;
    ck = umin(ck, E);
    ckm = umin(ckm, E);
    // head-segment records whose contribution changes with the carried run:
    // the prefix with max(run_local, s') < carry (monotone along the segment)
    const int32_t r0 = __shfl_sync(0xffffffffu, rj, 0);
    u64 runK = 0, runKM = 0, dk = 0, dkm = 0;
    for (int base = 0; base < x.cnt; base += 32) {
        const int j = base + lane;
        bool in = j < x.cnt;
        u64 e = 0, s = 0;
        bool kern = false;
        if (in) {
            if (base > 0) {
                rj = csr ? (j < x.hcnt ? x.r0 : -1) : __ldcg(R + j);
                sj = __ldcg(S + j); ej = __ldcg(En + j); kj = __ldcg(K + j);
            }
            in = rj == r0;
            const u64 e0 = ej, s0 = sj;
            kern = kj == 0;
            if (in) {
                e = umin(e0, E);
                s = umin(s0, e);
            } else {
                kern = false;
            }
        }
        u64 xkm = e, xk = kern ? e : 0;   // inclusive running maxima (clamped)
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const u64 okm = shfl_up64(xkm, d), ok = shfl_up64(xk, d);
            if (lane >= d) { xkm = umax(xkm, okm); xk = umax(xk, ok); }
        }
        u64 ekm = shfl_up64(xkm, 1), ek = shfl_up64(xk, 1);
        if (lane == 0) { ekm = 0; ek = 0; }
        ekm = umax(ekm, runKM);
        ek = umax(ek, runK);
        bool live = false;
        if (in) {
            const u64 loKM = umax(ekm, s), nKM = umax(ekm, ckm);
            if (loKM < ckm) dkm += (umax(ekm, e) - loKM) - (umax(nKM, e) - umax(nKM, s));
            if (kern) {
                const u64 loK = umax(ek, s), nK = umax(ek, ck);
                if (loK < ck) dk += (umax(ek, e) - loK) - (umax(nK, e) - umax(nK, s));
            }
            live = umax(ekm, s) < ckm || umax(ek, s) < ck;
        }
        runKM = umax(runKM, __shfl_sync(0xffffffffu, xkm, 31));
        runK = umax(runK, __shfl_sync(0xffffffffu, xk, 31));
        if (!(__ballot_sync(0xffffffffu, live) >> 31)) break;
    }
    dk = warp_sum(dk);
    dkm = warp_sum(dkm);
    if (lane == 0 && r0 >= 0 && r0 < p.dev_ids) {
        if (dk) red_add(p.d_k + r0, (u64)0 - dk);      // two's complement: subtract
        if (dkm) red_add(p.d_km + r0, (u64)0 - dkm);
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
    u64 dmx = 0;
    for (int32_t id = tid; id < p.dev_ids; id += nt) dmx = umax(dmx, ld_relaxed(p.d_maxend + id));
    const u64 dev_max_end = (u64)block_reduce128<true>(dmx, scratch, tid, nt);
    const u64 host_elapsed = umax(ld_relaxed(&g->host_max_end), p.host_elapsed_floor);
    if (tid == 0) {
        u64 E;
        if (p.mode == kSummarizeDevice) E = p.elapsed_ptr ? ld_relaxed(p.elapsed_ptr) : p.elapsed_arg;
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
        // the device-only E (summarize.py:91); with ranks declared the per-device maxima are
        // kept clamped at E by the union passes, so there is no trace-wide value to report
        res->dev_max_end = p.n >= 1 ? 0ull : dev_max_end;
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
        const u128 uw = (u128)useful + off;
        sum_u += useful;
        sum_uw += uw;
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
    sum_u = block_reduce128<false>(sum_u, scratch, tid, nt);
    sum_uw = block_reduce128<false>(sum_uw, scratch, tid, nt);
    max_uw = block_reduce128<true>(max_uw, scratch, tid, nt);
    sum_k = block_reduce128<false>(sum_k, scratch, tid, nt);
    max_k = block_reduce128<true>(max_k, scratch, tid, nt);
    max_km = block_reduce128<true>(max_km, scratch, tid, nt);
    if (ok && p.mode == kReport)
        metric_trees(res, p.n >= 1, p.m >= 1, E, p.n, p.m, sum_u, sum_uw, max_uw, sum_k, max_k, max_km, tid);
    __syncthreads();
    if (tid == 0) {
        g->tile_counter = 0;
        g->host_done = 0;
        g->contract_flags = 0;
        g->host_max_end = 0;
        g->contract_index = LLONG_MAX;
        g->ovl_suspect = 0;
        for (int i = 0; i < 8; ++i) g->counts[i] = 0;
        __threadfence();
        g->ctas_done = 0;
    }
}

// =========================================================================
// the kernel
// =========================================================================
#ifndef HB_MINB
#define HB_MINB 1   // resident CTAs per SM the register budget is sized for
#endif
template <bool CSR>
__global__ void __launch_bounds__(kThreads, HB_MINB) analyze_kernel(const __grid_constant__ Params p)
{
    extern __shared__ __align__(128) uint8_t smem_raw[];
    StageSmem *stages = reinterpret_cast<StageSmem *>(smem_raw);
    Ctrl *c = reinterpret_cast<Ctrl *>(smem_raw + sizeof(StageSmem) * kStages);
    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;

    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&c->full[s], 1);
            mbar_init(&c->empty[s], kComputeWarps);
        }
        for (int s = 0; s < kHdr; ++s) {
            c->h_max[s] = 0;
            c->h_cnt[s] = 0;
        }
        for (int s = 0; s < kRing; ++s) {
            mbar_init(&c->info_full[s], 1);
            mbar_init(&c->info_empty[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    u64 E_cache = 0;
    bool E_known = false;
    if (warp == kComputeWarps && !CSR) {
        // ---------------- TMA warp: keep every stage in flight ----------------
        const uint64_t pol = l2_policy_evict_first();
        for (int s = 0; s < kStages; ++s)
            produce<false>(p, stages, c, s, s % kHdr, claim_finish(p, claim_issue(p, lane)), lane, pol);
        // claims run ahead of use: the atomic is issued one refill before its index is
        // needed and the previous-record loads one refill before the TMA issue
        Claim next = claim_finish(p, claim_issue(p, lane));
        int64_t pend = claim_issue(p, lane);
        PROF_DECL(pa); PROF_DECL(pb); PROF_DECL(pn);
        for (int it = 0;; ++it) {
            const int st = it % kStages;
            const uint32_t ph = (uint32_t)((it / kStages) & 1);
            if (c->tile[st] < 0) break;
            long long t0 = PROF_NOW();
            mbar_wait(&c->empty[st], ph);
            PROF_ADD(pa, t0);
            t0 = PROF_NOW();
            produce<false>(p, stages, c, st, (it + kStages) % kHdr, next, lane, pol);
            next = claim_finish(p, pend);
            pend = claim_issue(p, lane);
            PROF_ADD(pb, t0);
#ifdef HB_PROF
            ++pn;
#endif
            (void)t0;
        }
#ifdef HB_PROF
        if (lane == 0) {
            unsigned long long *o = hb_prof_buf + blockIdx.x * kProfSlots;
            o[8] = pa; o[9] = pb; o[12] = pn;
        }
#endif
    } else if (warp == kComputeWarps) {
        // ---------------- TMA warp (CSR offsets): claims run two refills ahead -- the
        // atomic, then the offset-window copies (resolved one refill later) -- so the
        // resource lookup never delays a refill
        const uint64_t pol = l2_policy_evict_first();
        csr_sample_fill(p.hseg, p.host_ids, c->csr[0], lane);
        csr_sample_fill(p.dseg, p.dev_ids, c->csr[1], lane);
        for (int s = 0; s < kStages; ++s) {
            const PendClaim pc = claim_start(p, c->csr, c->claim, claim_issue(p, lane), lane);
            produce<true>(p, stages, c, s, s % kHdr, claim_done(p, c->csr, pc, c->claim, lane), lane, pol);
        }
        Claim next;
        {
            const PendClaim pc = claim_start(p, c->csr, c->claim, claim_issue(p, lane), lane);
            next = claim_done(p, c->csr, pc, c->claim, lane);
        }
        PendClaim mid = claim_start(p, c->csr, c->claim, claim_issue(p, lane), lane);
        int64_t pend = claim_issue(p, lane);
        PROF_DECL(pa); PROF_DECL(pb); PROF_DECL(pn);
        for (int it = 0;; ++it) {
            const int st = it % kStages;
            const uint32_t ph = (uint32_t)((it / kStages) & 1);
            if (c->tile[st] < 0) break;
            long long t0 = PROF_NOW();
            mbar_wait(&c->empty[st], ph);
            PROF_ADD(pa, t0);
            t0 = PROF_NOW();
            produce<true>(p, stages, c, st, (it + kStages) % kHdr, next, lane, pol);
            next = claim_done(p, c->csr, mid, c->claim, lane);
            mid = claim_start(p, c->csr, c->claim, pend, lane);
            pend = claim_issue(p, lane);
            PROF_ADD(pb, t0);
#ifdef HB_PROF
            ++pn;
#endif
            (void)t0;
        }
#ifdef HB_PROF
        if (lane == 0) {
            unsigned long long *o = hb_prof_buf + blockIdx.x * kProfSlots;
            o[8] = pa; o[9] = pb; o[12] = pn;
        }
#endif
    } else if (warp > kComputeWarps) {
        // ---------------- epilogue warps: look-back + carry fix-up of device tiles ----------------
        // descriptor k goes to epilogue warp k % kEpiWarps
        PROF_DECL(pc); PROF_DECL(pw);
        for (int k = warp - kComputeWarps - 1;; k += kEpiWarps) {
            const int slot = k % kRing;
            long long t0 = PROF_NOW();
            mbar_wait(&c->info_full[slot], (uint32_t)((k / kRing) & 1));
            PROF_ADD(pw, t0);
            const TileInfo x = c->info[slot];
            __syncwarp();
            if (lane == 0) mbar_arrive(&c->info_empty[slot]);
            if (x.t < 0) break;
            t0 = PROF_NOW();
            dev_epilogue(p, x, lane, E_cache, E_known);
            PROF_ADD(pc, t0);
            (void)t0;
        }
#ifdef HB_PROF
        if (lane == 0 && warp == kComputeWarps + 1) {
            unsigned long long *o = hb_prof_buf + blockIdx.x * kProfSlots;
            o[10] = pc; o[11] = pw;
        }
#endif
    } else {
        // ---------------- compute warps ----------------
        PROF_DECL(ca); PROF_DECL(cb); PROF_DECL(cn);
        Phases phs;
        bool one_pass = true;
        int hpend = 0;   // host tiles finished by this CTA, not yet released
        int k = 0;
        for (int it = 0;; ++it) {
            const int st = it % kStages;
            long long t0 = PROF_NOW();
            mbar_wait(&c->full[st], (uint32_t)((it / kStages) & 1));
            PROF_ADD(ca, t0);
            const int64_t t = c->tile[st];
            if (t < 0) break;
            TileCtx tc;
            tc.st = it % kHdr;
            tc.cnt = c->cnt[st];
            tc.empty = &c->empty[st];
            tc.released = false;
            const bool dev = t >= p.host_tiles;
            tc.lt = dev ? t - p.host_tiles : t;
            tc.gbase = tc.lt * kTile;
            t0 = PROF_NOW();
            if (!dev) {
                host_compute(p, stages[st], c, tc, tid, phs);
                ++hpend;
            }
            else dev_compute(p, stages[st], c, tc, tid, E_cache, E_known, hpend, k, one_pass, phs);
#ifdef HB_PROF
            if (dev) ++phs.dn; else ++phs.hn;
#endif
            release(tc, lane);
            PROF_ADD(cb, t0);
#ifdef HB_PROF
            ++cn;
#endif
            (void)t0;
        }
        bar_compute();   // every compute warp is done with its last tile (incl. host max-end REDs)
        if (tid == 0) {
            for (int e = 0; e < kEpiWarps; ++e) post_info(c, k, -1, 0, false, false, 0, 0);   // end of stream
            if (hpend > 0) host_tiles_done(p, hpend);       // CTAs that saw no device tile
        }
#ifdef HB_PROF
        if (tid == 0) {
            unsigned long long *o = hb_prof_buf + blockIdx.x * kProfSlots;
            o[0] = ca; o[1] = cb; o[2] = cn;
            o[3] = phs.a; o[4] = phs.bar; o[5] = phs.b; o[6] = phs.emit;
            o[16] = phs.hb; o[17] = phs.hemit; o[18] = phs.hn; o[19] = phs.dn; o[20] = phs.hn2; o[21] = phs.mg; o[22] = phs.nd;
        }
#endif
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
        if (*(volatile unsigned *)&p.g->ovl_suspect) {
            // host records overlap somewhere: the exact findings come from the
            // error-path kernels (launch_overlap_pass), which then finalize -- or, in block
            // mode, from the caller's fallback: finalize now (the context's accumulators and
            // globals reset for the next call) and keep the status "pending"
            if (p.settle) {
                finalize(p, reinterpret_cast<u128 *>(smem_raw), tid);
                __syncthreads();
            }
            if (tid == 0) p.res->status = -1;
        } else {
            finalize(p, reinterpret_cast<u128 *>(smem_raw), tid);
        }
    }
}

// =========================================================================
// error path: exact host-overlap findings (model.py:203-215) for traces
// where some host record starts before its predecessor's end.  Three simple
// passes over the tiles (per-tile aggregate, carry scan, detection), then
// the finalize.  Only runs for invalid traces.
// =========================================================================
constexpr int kOvlThreads = 256;

// per-thread contiguous chunk of the tile: (segment start inside?, max end of its last segment)
__device__ void ovl_chunk(const Params &p, int64_t base, int cnt, int tid, int &lo, int &hi, bool &f, u64 &v)
{
    const int per = (cnt + kOvlThreads - 1) / kOvlThreads;
    lo = min(cnt, tid * per);
    hi = min(cnt, lo + per);
    f = false;
    v = 0;
    for (int j = lo; j < hi; ++j) {
        const int64_t g = base + j;
        if (g == 0 || p.hr[g] != p.hr[g - 1]) { f = true; v = 0; }
        v = umax(v, p.he[g]);
    }
}

__global__ void __launch_bounds__(kOvlThreads) ovl_agg_kernel(const __grid_constant__ Params p, u64 *agg)
{
    __shared__ int sf[kOvlThreads];
    __shared__ u64 sv[kOvlThreads];
    const int64_t t = blockIdx.x;
    const int64_t base = t * kTile;
    const int cnt = (int)min((int64_t)kTile, p.hn - base);
    int lo, hi;
    bool f;
    u64 v;
    ovl_chunk(p, base, cnt, threadIdx.x, lo, hi, f, v);
    sf[threadIdx.x] = f;
    sv[threadIdx.x] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        bool tf = false;
        u64 tv = 0;
        for (int i = 0; i < kOvlThreads; ++i) {
            if (sf[i]) { tf = true; tv = sv[i]; }
            else tv = umax(tv, sv[i]);
        }
        agg[2 * t] = tf;
        agg[2 * t + 1] = tv;
    }
}

// one thread: exclusive carry for every tile (max end of earlier records of
// the segment that continues into the tile)
__global__ void ovl_carry_kernel(int64_t tiles, const u64 *agg, u64 *carry)
{
    u64 run = 0;
    for (int64_t t = 0; t < tiles; ++t) {
        carry[t] = run;
        run = agg[2 * t] ? agg[2 * t + 1] : umax(run, agg[2 * t + 1]);
    }
}

__global__ void __launch_bounds__(kOvlThreads) ovl_detect_kernel(const __grid_constant__ Params p, const u64 *carry)
{
    __shared__ int sf[kOvlThreads];
    __shared__ u64 sv[kOvlThreads];
    const int64_t t = blockIdx.x;
    const int64_t base = t * kTile;
    const int cnt = (int)min((int64_t)kTile, p.hn - base);
    int lo, hi;
    bool f;
    u64 v;
    ovl_chunk(p, base, cnt, threadIdx.x, lo, hi, f, v);
    sf[threadIdx.x] = f;
    sv[threadIdx.x] = v;
    __syncthreads();
    // exclusive prefix for this thread: tile carry, then earlier chunks
    u64 run = carry[t];
    for (int i = 0; i < (int)threadIdx.x; ++i) run = sf[i] ? sv[i] : umax(run, sv[i]);
    bool decl = false;
    for (int j = lo; j < hi; ++j) {
        const int64_t g = base + j;
        const int32_t r = p.hr[g];
        if (g == 0 || r != p.hr[g - 1]) run = 0;
        if (j == lo || g == 0 || r != p.hr[g - 1]) decl = declared(p.host_decl, p.host_ids, p.n, r);
        const u64 s = p.hs[g], e = p.he[g];
        if (decl && s < e && s < run) push(p, 3, g);
        run = umax(run, e);
    }
}

// CSR offsets -> per-record dense ids (the res column of a CSR input): each block
// takes a chunk of records, finds the groups it touches once, then every record
// binary-searches only those (usually one) -- coalesced writes, no per-record
// search over the whole offset table.  Record i belongs to the last group r with
// seg[r] <= i (empty groups share an offset with the next one).
constexpr int kExpandChunk = 8192;
__device__ __forceinline__ int32_t last_le(const int64_t *seg, int32_t lo, int32_t hi, int64_t i)
{
    while (lo < hi) {   // last r in [lo, hi] with seg[r] <= i (seg[lo] <= i holds)
        const int32_t mid = lo + ((hi - lo + 1) >> 1);
        if (__ldg(seg + mid) <= i) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

__global__ void __launch_bounds__(256) expand_res_kernel(const int64_t *seg, int32_t ids, int64_t n, int32_t *res)
{
    __shared__ int32_t s_lo, s_hi;
    const int64_t c0 = (int64_t)blockIdx.x * kExpandChunk;
    const int64_t c1 = c0 + kExpandChunk < n ? c0 + kExpandChunk : n;
    if (threadIdx.x == 0) {
        s_lo = last_le(seg, 0, ids - 1, c0);
        s_hi = last_le(seg, s_lo, ids - 1, c1 - 1);
    }
    __syncthreads();
    const int32_t lo = s_lo, hi = s_hi;
    for (int64_t i = c0 + threadIdx.x; i < c1; i += 256) res[i] = lo == hi ? lo : last_le(seg, lo, hi, i);
}

cudaError_t launch_expand_res(const int64_t *seg, int32_t ids, int64_t n, int32_t *res, cudaStream_t s)
{
    if (n <= 0 || ids <= 0) return cudaSuccess;
    expand_res_kernel<<<(unsigned)((n + kExpandChunk - 1) / kExpandChunk), 256, 0, s>>>(seg, ids, n, res);
    return cudaGetLastError();
}

__global__ void __launch_bounds__(kThreads) finalize_kernel(const __grid_constant__ Params p)
{
    __shared__ u128 scratch[40];
    finalize(p, scratch, threadIdx.x);
}

cudaError_t launch_overlap_pass(const Params &p, u64 *scratch, cudaStream_t s)
{
    const int64_t tiles = p.host_tiles;
    if (tiles > 0) {
        ovl_agg_kernel<<<(unsigned)tiles, kOvlThreads, 0, s>>>(p, scratch);
        ovl_carry_kernel<<<1, 1, 0, s>>>(tiles, scratch, scratch + 2 * tiles);
        ovl_detect_kernel<<<(unsigned)tiles, kOvlThreads, 0, s>>>(p, scratch + 2 * tiles);
    }
    finalize_kernel<<<1, kThreads, 0, s>>>(p);
    return cudaGetLastError();
}

// =========================================================================
// stand-alone metric trees (host_metrics / device_metrics stage functions)
// =========================================================================
__global__ void __launch_bounds__(kThreads) metrics_kernel(const u64 *sums, int32_t k, u64 E, int host_side,
                                                           ResultDev *res)
{
    __shared__ u128 scratch[33];
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
    a = block_reduce128<false>(a, scratch, tid, kThreads);
    if (host_side) b = block_reduce128<false>(b, scratch, tid, kThreads);
    else b = block_reduce128<true>(b, scratch, tid, kThreads);
    c = block_reduce128<true>(c, scratch, tid, kThreads);
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

int prof_read(unsigned long long *out, int n)
{
#ifdef HB_PROF
    const int k = n < 1024 * kProfSlots ? n : 1024 * kProfSlots;
    cudaMemcpyFromSymbol(out, hb_prof_buf, sizeof(unsigned long long) * k);
    return k;
#else
    (void)out; (void)n;
    return 0;
#endif
}

// persistent grid: every SM x resident CTAs; 0 when the tile geometry does not fit
int analyze_grid(int device)
{
    int sms = 0, per = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (cudaFuncSetAttribute(analyze_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)analyze_smem_bytes()) != cudaSuccess ||
        cudaFuncSetAttribute(analyze_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)analyze_smem_bytes()) != cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, analyze_kernel<true>, kThreads, analyze_smem_bytes()) !=
            cudaSuccess) {
        cudaGetLastError();   // not sticky: clear it so later launches report their own status
        return 0;
    }
    return sms * (per < 1 ? 1 : per);
}

cudaError_t launch_analyze(const Params &p, int grid, cudaStream_t s)
{
    // CSR offsets on either side: the instantiation that reads them
    if (p.hseg || p.dseg) analyze_kernel<true><<<grid, kThreads, analyze_smem_bytes(), s>>>(p);
    else analyze_kernel<false><<<grid, kThreads, analyze_smem_bytes(), s>>>(p);
    return cudaGetLastError();
}

// entries for another compilation of this file (engine_cols.cu): the same Params layout,
// reached through its address; its tile size sets the tile counts of a call
cudaError_t launch_analyze_v(const void *p, int grid, cudaStream_t s)
{
    return launch_analyze(*static_cast<const Params *>(p), grid, s);
}

cudaError_t launch_overlap_pass_v(const void *p, u64 *scratch, cudaStream_t s)
{
    return launch_overlap_pass(*static_cast<const Params *>(p), scratch, s);
}

int tile_records() { return kTile; }

// =========================================================================
// multi-GPU merge of gathered per-rank result blocks.  Every rank
// ran two launches into its block [host header 256 B | device header 256 B |
// host rows [n_max][4] | device rows [m_max][4]]: its host records
// (SUMMARIZE_HOST) and, after the all-reduce of E, its device records
// clamped at the GLOBAL E (SUMMARIZE_DEVICE, window read from device memory).
// The merge concatenates the rows in rank order (every CTA a strided share,
// with partial sums / maxima) and the last CTA to finish reduces the partials
// and evaluates both metric trees; a non-OK shard makes it defer (status -2)
// to the host path.
// =========================================================================
constexpr int kMergeT = 256;
struct MergeScratch {
    unsigned int done;   // CTAs finished (zeroed before every launch)
    unsigned int pad[3];
    u128 part[kMergeCTAs][7];   // per CTA: sum u, sum u+w, max u+w, sum k, max k, max k+m, sum clamp
};

__device__ __forceinline__ u128 ldcg128(const u128 *p)
{
    const u64 *q = reinterpret_cast<const u64 *>(p);
    return ((u128)__ldcg(q + 1) << 64) | __ldcg(q);
}

__global__ void __launch_bounds__(kMergeT) merge_kernel(const uint8_t *blocks, int32_t world, size_t block_bytes,
                                                        int32_t n_max, int32_t m_max, const int32_t *n_of,
                                                        const int32_t *m_of, uint8_t *out, const u64 *E_global,
                                                        MergeScratch *ms)
{
    __shared__ u128 scratch[33];
    __shared__ int s_defer, s_last;
    const int tid = threadIdx.x, nt = blockDim.x;
    ResultDev *res = reinterpret_cast<ResultDev *>(out);
    const u64 E = ld_relaxed(E_global);
    if (tid == 0) {
        int defer = 0;
        for (int r = 0; r < world; ++r) {
            const uint8_t *blk = blocks + (size_t)r * block_bytes;
            const ResultDev *h = reinterpret_cast<const ResultDev *>(blk);
            const ResultDev *d = reinterpret_cast<const ResultDev *>(blk + 256);
            if (h->status != 0 || d->status != 0) defer = 1;
        }
        s_defer = defer;
        if (blockIdx.x == 0) {
            res->status = defer ? -2 : (E == 0 ? 2 : 0);
            res->elapsed = E;
            res->host_elapsed = E;
            res->host_mask = res->device_mask = 0;
        }
    }
    __syncthreads();
    if (s_defer) return;
    int64_t ntot = 0, mtot = 0;
    for (int r = 0; r < world; ++r) { ntot += n_of[r]; mtot += m_of[r]; }
    u64 *hout = reinterpret_cast<u64 *>(out + 256);
    u64 *dout = hout + 4 * (size_t)ntot;
    u128 su = 0, suw = 0, muw = 0, sk = 0, mk = 0, mkm = 0, scl = 0;
    for (int64_t g = (int64_t)blockIdx.x * nt + tid; g < ntot + mtot; g += (int64_t)gridDim.x * nt) {
        const bool host = g < ntot;
        int64_t i = host ? g : g - ntot;
        int r = 0;
        for (; r < world - 1; ++r) {   // the rank holding row i (rank order)
            const int32_t k = host ? n_of[r] : m_of[r];
            if (i < k) break;
            i -= k;
        }
        const u64 *hr = reinterpret_cast<const u64 *>(blocks + (size_t)r * block_bytes + 512);
        const u64 *x = (host ? hr : hr + 4 * (size_t)n_max) + 4 * (size_t)i;
        const ulonglong2 x01 = *reinterpret_cast<const ulonglong2 *>(x);
        const ulonglong2 x23 = *reinterpret_cast<const ulonglong2 *>(x + 2);
        u64 *o = (host ? hout : dout) + 4 * (size_t)(host ? g : g - ntot);
        *reinterpret_cast<ulonglong2 *>(o) = x01;
        *reinterpret_cast<ulonglong2 *>(o + 2) = x23;
        if (host) {
            const u128 uw = (u128)x01.x + x01.y;
            su += x01.x;
            suw += uw;
            if (uw > muw) muw = uw;
        } else {
            sk += x01.x;
            if ((u128)x01.x > mk) mk = x01.x;
            const u128 km = (u128)x01.x + x01.y;
            if (km > mkm) mkm = km;
            scl += x23.y;   // records clamped at E
        }
    }
    u128 v[7] = {su, suw, muw, sk, mk, mkm, scl};
    constexpr bool kMax[7] = {false, false, true, false, true, true, false};
#pragma unroll
    for (int k = 0; k < 7; ++k)
        v[k] = kMax[k] ? block_reduce128<true>(v[k], scratch, tid, nt) : block_reduce128<false>(v[k], scratch, tid, nt);
    if (tid == 0) {
#pragma unroll
        for (int k = 0; k < 7; ++k) ms->part[blockIdx.x][k] = v[k];
        __threadfence();
        s_last = atomicAdd(&ms->done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // the last CTA: every CTA's partials
    u128 a[7] = {0, 0, 0, 0, 0, 0, 0};
    for (int b = tid; b < (int)gridDim.x; b += nt) {
#pragma unroll
        for (int k = 0; k < 7; ++k) {
            const u128 x = ldcg128(&ms->part[b][k]);
            a[k] = kMax[k] ? (x > a[k] ? x : a[k]) : a[k] + x;
        }
    }
#pragma unroll
    for (int k = 0; k < 7; ++k)
        a[k] = kMax[k] ? block_reduce128<true>(a[k], scratch, tid, nt) : block_reduce128<false>(a[k], scratch, tid, nt);
    if (tid == 0) res->counts[7] = (int64_t)(u64)a[6];   // late device records (clamped at the global E)
    if (E == 0) return;
    metric_trees(res, ntot >= 1, mtot >= 1, E, (int32_t)ntot, (int32_t)mtot, a[0], a[1], a[2], a[3], a[4], a[5], tid);
}

size_t merge_scratch_bytes() { return sizeof(MergeScratch); }

cudaError_t launch_merge(const void *blocks, int32_t world, size_t block_bytes, int32_t n_max, int32_t m_max,
                         const int32_t *n_of, const int32_t *m_of, void *out, const u64 *E_global, void *scratch,
                         int64_t rows, cudaStream_t s)
{
    MergeScratch *ms = static_cast<MergeScratch *>(scratch);
    cudaError_t e = cudaMemsetAsync(&ms->done, 0, sizeof(unsigned int), s);
    if (e != cudaSuccess) return e;
    int64_t g = (rows + kMergeT - 1) / kMergeT;
    g = g < 1 ? 1 : (g > kMergeCTAs ? kMergeCTAs : g);
    merge_kernel<<<(unsigned)g, kMergeT, 0, s>>>(static_cast<const uint8_t *>(blocks), world, block_bytes, n_max, m_max,
                                                 n_of, m_of, static_cast<uint8_t *>(out), E_global, ms);
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

}  // namespace HB_ENGINE_NS
