// engine.cuh -- parameters shared by the analysis kernel (engine.cu) and the
// C ABI (capi.cu).  See DESIGN.md for the data layout and the algorithm.
#pragma once
#include <cstdint>

namespace hb {

typedef unsigned long long u64;

constexpr int kComputeWarps = 7;
constexpr int kComputeThreads = kComputeWarps * 32;    // 224
constexpr int kThreads = kComputeThreads + 32;         // + producer / look-back warp
constexpr int kItems = 13;                             // odd: conflict-free blocked smem reads
constexpr int kTile = kComputeThreads * kItems;        // 2912 records per tile
constexpr int kStages = 3;

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
    int32_t host_ids, dev_ids;
    const int32_t *host_decl, *dev_decl;
    int32_t n, m;
    u64 host_elapsed_floor;
    int32_t mode;
    int32_t use_tma;
    u64 elapsed_arg;
    int64_t cap;
    int64_t host_tiles, dev_tiles;
    uint32_t epoch;
    // workspace: per dense id accumulators (zero between calls)
    u64 *h_off, *h_mpi, *h_span;
    u64 *d_k, *d_km, *d_clamp, *d_maxend;
    // tile status for the decoupled look-back (epoch-tagged, never cleared)
    uint32_t *h_flag;
    u64 *h_valA, *h_valP;
    uint32_t *d_flag;
    u64 *d_valA0, *d_valA1, *d_valP0, *d_valP1;
    Globals *g;
    int64_t *lists[8];
    // outputs (device memory, copied to the caller by the C ABI)
    u64 *host_out;   // [n][4]
    u64 *dev_out;    // [m][4]
    ResultDev *res;
};

size_t analyze_smem_bytes();
int analyze_grid(int device);
cudaError_t launch_analyze(const Params &p, int grid, cudaStream_t s);
cudaError_t launch_metrics(const u64 *summaries, int32_t k, u64 elapsed, int host_side, ResultDev *res,
                           cudaStream_t s);
cudaError_t launch_covers(const Params &p, const int64_t *err_idx, int64_t count, int64_t *cover, cudaStream_t s);

}  // namespace hb
