// engine.cuh -- parameters shared by the analysis kernel (engine.cu) and the
// C ABI (capi.cu).  See DESIGN.md for the data layout and the algorithm.
#pragma once
#include <cstdint>

// The engine's namespace: `hb`, or another name for a second compilation of the
// analysis kernel with a different tile geometry (engine_cols.cu).
#ifndef HB_ENGINE_NS
#define HB_ENGINE_NS hb
#endif
namespace HB_ENGINE_NS {

typedef unsigned long long u64;

// tile geometry (compile-time knobs, see tools/build_variants.sh)
#ifndef HB_WARPS
#define HB_WARPS 15
#endif
#ifndef HB_EPI
#define HB_EPI 2
#endif
#ifndef HB_ITEMS
#define HB_ITEMS 11
#endif
#ifndef HB_STAGES
#define HB_STAGES 2
#endif
constexpr int kComputeWarps = HB_WARPS;
constexpr int kComputeThreads = kComputeWarps * 32;
constexpr int kEpiWarps = HB_EPI;                      // look-back / carry fix-up warps
constexpr int kThreads = kComputeThreads + 32 * (1 + kEpiWarps);   // + TMA warp + epilogue warps
constexpr int kItems = HB_ITEMS;                       // odd: conflict-free blocked smem reads
constexpr int kTile = kComputeThreads * kItems;        // records per tile (multiple of 16)
constexpr int kStages = HB_STAGES;
static_assert(kTile % 16 == 0, "tile must keep every column 16-byte aligned for TMA");
static_assert(kItems <= 32, "per-thread bit masks");

enum Mode { kReport = 0, kSummarizeDevice = 1, kValidate = 2, kSummarizeHost = 3 };

// grid-wide counters; the last CTA resets them (self-cleaning workspace)
struct Globals {
    u64 tile_counter;
    u64 host_done;
    unsigned int ctas_done;
    unsigned int contract_flags;
    u64 host_max_end;
    long long contract_index;
    u64 counts[8];
    unsigned int ovl_suspect;     // a host record starts before its predecessor's end
    unsigned int pad;
};

struct ResultDev {
    int32_t status;
    int32_t contract_flags;
    int64_t contract_index;
    u64 host_elapsed;
    u64 elapsed;
    u64 dev_max_end;
    int32_t host_present;
    int32_t device_present;
    double host_metrics[5];
    uint32_t host_mask;
    uint32_t device_mask;
    double device_metrics[4];
    int64_t counts[8];
    double kernel_ms;
};

struct Params {
    // record columns (device memory)
    const u64 *hs, *he;
    const int32_t *hr;
    const uint8_t *hk;
    int64_t hn;
    const u64 *ds, *de;
    const int32_t *dr;
    const uint8_t *dk;
    int64_t dn;
    // CSR offsets [ids + 1] instead of the res columns (hr / dr then unused; null = columns)
    const int64_t *hseg, *dseg;
    int32_t host_ids, dev_ids;
    const int32_t *host_decl, *dev_decl;
    int32_t n, m;
    u64 host_elapsed_floor;
    int32_t mode;
    int32_t use_tma;
    // 1: block mode (heteff_analyze_into): a trace with suspected host overlaps is
    // finalized right away (context state reset) and reported as status -1, so the
    // caller's fallback path re-runs it; 0: the error-path kernels finalize it
    int32_t settle;
    u64 elapsed_arg;
    const u64 *elapsed_ptr;   // SUMMARIZE_DEVICE: the window read from device memory (multi-GPU: all-reduced E)
    int64_t cap;
    int64_t host_tiles, dev_tiles;
    uint32_t epoch;
    // workspace: per dense id accumulators (zero between calls)
    u64 *h_off, *h_mpi, *h_span;
    u64 *d_k, *d_km, *d_clamp, *d_maxend;
    // decoupled look-back slots, self-validating (epoch-tagged 32-bit halves,
    // never cleared): host [tiles][2] words per slot, device [tiles][4]
    u64 *h_slotA, *h_slotP;
    u64 *d_slotA, *d_slotP;
    Globals *g;
    int64_t *lists[8];
    // outputs (device memory, copied to the caller by the C ABI)
    u64 *host_out;   // [n][4]
    u64 *dev_out;    // [m][4]
    ResultDev *res;
};

size_t analyze_smem_bytes();
int prof_read(unsigned long long *out, int n);
int analyze_grid(int device);
cudaError_t launch_analyze(const Params &p, int grid, cudaStream_t s);
cudaError_t launch_metrics(const u64 *summaries, int32_t k, u64 elapsed, int host_side, ResultDev *res,
                           cudaStream_t s);
// CSR offsets [ids + 1] -> res[n] (dense id of every record)
cudaError_t launch_expand_res(const int64_t *seg, int32_t ids, int64_t n, int32_t *res, cudaStream_t s);
// the merge runs on up to kMergeCTAs CTAs; the last one to finish reduces their partial
// aggregates (scratch: merge_scratch_bytes() of device memory)
constexpr int kMergeCTAs = 148;
size_t merge_scratch_bytes();
cudaError_t launch_merge(const void *blocks, int32_t world, size_t block_bytes, int32_t n_max, int32_t m_max,
                         const int32_t *n_of, const int32_t *m_of, void *out, const u64 *E_global, void *scratch,
                         int64_t rows, cudaStream_t s);
// error path: exact host-overlap findings (only when ovl_suspect), then finalize
cudaError_t launch_overlap_pass(const Params &p, u64 *scratch, cudaStream_t s);
cudaError_t launch_covers(const Params &p, const int64_t *err_idx, int64_t count, int64_t *cover, cudaStream_t s);

// K5/K6 (regions.cu, EXTENSIONS): monitoring regions + offload / busy overlap
constexpr int kMaxWindows = 16;      // windows per region pass

struct RegionResultDev {
    int32_t status;
    int32_t reserved;
    u64 elapsed;
    double host_metrics[5];
    uint32_t host_mask;
    uint32_t device_mask;
    double device_metrics[4];
    double busy_fraction;
    uint32_t busy_mask;
    uint32_t reserved2;
};

struct RegParams {
    const u64 *hs, *he;
    const int32_t *hr;
    const uint8_t *hk;
    int64_t hn;
    const u64 *ds, *de;
    const int32_t *dr;
    const uint8_t *dk;
    int64_t dn;
    int32_t host_ids, dev_ids;
    const int32_t *host_decl, *dev_decl;   // null = identity
    int32_t n, m;
    int32_t R;                              // windows of this pass (<= kMaxWindows)
    u64 wlo[kMaxWindows], whi[kMaxWindows]; // window bounds, padded with empty [0, 0)
    // per-rank regions: [R][host_ids][2] window of every rank for this pass (device
    // memory), devices take their owner's window, unowned devices an empty one;
    // null = the global windows wlo / whi
    const u64 *hwin;
    const int32_t *owner;                   // [dev_ids] dense host id or -1 (null = none)
    int64_t *hseg, *dseg;                   // [ids + 1] CSR offsets per dense id
    // window-independent checkpoints (prefix of the resource's segment at each chunk start)
    int64_t hchunks, tiles;
    u64 *hagg, *hck;                        // host chunks: [c][6] f,off,mpi,max end,max off end,max mpi end / [c+1][5]
    u64 *dagg, *drun;                       // device tiles: [t][3] f,max K end,max end / [t+1][2]
    u64 *dsum, *dck;                        // device tiles: [t][4] f,U_K,U_KM,busy / [t+1][3]
    int64_t *tstage;                        // device tiles: [t][2] owner host index range to stage
    u64 *dsub;                              // device tiles: [t][8 sub-checkpoints][8] in-tile prefixes
    u64 *scan_tmp;                          // [blocks][8] scan scratch
    u64 *h_acc;                             // [R][host_ids][3] offload, mpi, span
    u64 *d_acc;                             // [R][dev_ids][4] kernel, kernel|memory, clamped, busy
    u64 *E;                                 // [R]
    u64 *dmax;                              // [R] max clipped device end (device-only traces)
    u64 *host_out;                          // [R][n][4]
    u64 *dev_out;                           // [R][m][4]
    u64 *busy_out;                          // [R][m]
    RegionResultDev *res;                   // [R]
};

size_t region_hchunks(int64_t hn);
size_t region_subs();
size_t region_tiles(int64_t dn);
cudaError_t launch_regions_prepare(const RegParams &p, cudaStream_t s);
cudaError_t launch_regions_phase1(const RegParams &p, cudaStream_t s);
cudaError_t launch_regions_phase2(const RegParams &p, cudaStream_t s);

// interval algebra (intervals.cu): the reference's intervals.py:40-105
size_t iv_flatten_ws(int64_t n);
cudaError_t iv_flatten(const u64 *s, const u64 *e, int64_t n, u64 *os, u64 *oe, int64_t *out_n, int64_t *bad,
                       void *ws, size_t ws_bytes, cudaStream_t st);
size_t iv_subtract_ws(int64_t na, int64_t nb);
cudaError_t iv_subtract(const u64 *as, const u64 *ae, int64_t na, const u64 *bs, const u64 *be, int64_t nb, u64 *os,
                        u64 *oe, int64_t *out_n, void *ws, size_t ws_bytes, cudaStream_t st);
size_t iv_intersect_ws(int64_t n);
cudaError_t iv_intersect(const u64 *s, const u64 *e, int64_t n, u64 lo, u64 hi, u64 *os, u64 *oe, int64_t *out_n,
                         void *ws, size_t ws_bytes, cudaStream_t st);
cudaError_t iv_total(const u64 *s, const u64 *e, int64_t n, u64 *out2_dev, cudaStream_t st);

// K3 (sort.cu): stable radix sort of one record set by (res, start)
struct SortStats {
    int key_bits, passes, wide, start_sorted;
};
size_t sort_workspace_bytes(int64_t n);
cudaError_t sort_records(const u64 *S, const u64 *E, const int32_t *R, const uint8_t *KD, int64_t n, u64 *os, u64 *oe,
                         int32_t *orr, uint8_t *ok, int64_t *perm, void *ws, size_t ws_bytes, cudaStream_t s,
                         SortStats *stats);
cudaError_t launch_remap(int64_t *list, int64_t k, const int64_t *perm, cudaStream_t s);
cudaError_t launch_order_check(const int32_t *R, const u64 *S, int64_t n, unsigned int *bad, cudaStream_t s);

}  // namespace HB_ENGINE_NS
