// capi.cu -- the extern "C" boundary (include/heteff_b200.h): context,
// self-cleaning device workspace, host staging, result copy-back.
#include <cuda_runtime.h>
#include <climits>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>
#include <cstdlib>
#include <string>

#include "../../include/heteff_b200.h"
#include "engine.cuh"
#include "transfer.cuh"

// The analysis kernel is compiled once per tile geometry (engine.cu in namespaces hb,
// hb_cols -- engine_cols.cu -- and hb_long -- engine_long.cu); each exports the same entries.
#define HB_COMPILATION_ENTRIES                                                                   \
    cudaError_t launch_analyze_v(const void *p, int grid, cudaStream_t s);                       \
    cudaError_t launch_overlap_pass_v(const void *p, unsigned long long *scratch, cudaStream_t s); \
    int analyze_grid(int device);                                                               \
    int tile_records();
namespace hb { HB_COMPILATION_ENTRIES }
namespace hb_cols { HB_COMPILATION_ENTRIES }
namespace hb_long { HB_COMPILATION_ENTRIES }

struct Compilation {
    const char *name;
    cudaError_t (*launch)(const void *p, int grid, cudaStream_t s);
    cudaError_t (*overlap)(const void *p, unsigned long long *scratch, cudaStream_t s);
    int (*grid)(int device);
    int (*tile)();
};
// measured per input: CSR offsets -> 15 x 11; res columns -> 11 x 15,
// or 8 x 19 when devices hold long record runs
static const Compilation kCompilations[3] = {
    {"15x11", hb::launch_analyze_v, hb::launch_overlap_pass_v, hb::analyze_grid, hb::tile_records},
    {"11x15", hb_cols::launch_analyze_v, hb_cols::launch_overlap_pass_v, hb_cols::analyze_grid, hb_cols::tile_records},
    {"8x19", hb_long::launch_analyze_v, hb_long::launch_overlap_pass_v, hb_long::analyze_grid, hb_long::tile_records},
};
constexpr int64_t kLongRun = 200000;   // records per device (res-column inputs) for the 8 x 19 compilation

namespace hb {
cudaError_t launch_generate(const heteff_gen_side &g, u64 *S, u64 *E, int32_t *R, uint8_t *K, cudaStream_t s);
}

using hb::u64;

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
};

struct heteff_ctx {
    int device = 0;
    int grid[3] = {0, 0, 0};   // CTAs of the analysis launch, per kernel compilation
    std::string kernel;        // the compilation(s) of the last analysis
    std::string err;
    uint32_t epoch = 0;
    // per dense id accumulators (zero between calls)
    DevBuf host_acc, dev_acc;      // 3 / 4 arrays of u64
    int64_t host_ids_cap = 0, dev_ids_cap = 0;
    // look-back tile status
    DevBuf host_tiles, dev_tiles;
    int64_t host_tiles_cap = 0, dev_tiles_cap = 0;
    // outputs
    DevBuf host_out, dev_out, lists;
    int64_t lists_cap = 0;
    hb::Globals *g = nullptr;
    hb::ResultDev *res_d = nullptr;
    hb::ResultDev *res_h = nullptr;   // pinned
    // staging for heteff_analyze_host / metrics; scratch of the overlap error path
    DevBuf stage, aux;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t ev_split0 = nullptr, ev_split1 = nullptr;   // run_split's span (the merge uses ev0 / ev1)
    // K3 sort: workspace, sorted columns + permutations
    DevBuf sort_ws, sorted;
    // K5/K6 regions: accumulators, carries, outputs
    DevBuf reg_ws, reg_out;
    // interval algebra scratch
    DevBuf iv_ws;
    // one contiguous result block per analysis: [ResultDev | host summaries | device summaries],
    // mirrored into pinned host memory by a single D2H copy
    DevBuf out_blk;
    void *out_pin = nullptr;
    size_t out_pin_bytes = 0;
    // small host-buffer calls: every input column gathered into one pinned block, one H2D
    void *in_pin = nullptr;
    size_t in_pin_bytes = 0;
    // CSR inputs on the paths that need res columns (error path, K3 sort, regions)
    DevBuf csr_res;
    // large host-buffer calls: block-compressed column transfer (transfer.cu)
    hb::TransferCtx xfer;
    // split analysis (run_split): the shared result block + E, and its pinned mirror
    DevBuf split;
    void *split_pin = nullptr;
    size_t split_pin_bytes = 0;
};

static int fail(heteff_ctx *ctx, int code, const std::string &msg)
{
    if (ctx) ctx->err = msg;
    return code;
}

static int cuda_fail(heteff_ctx *ctx, cudaError_t e, const char *what)
{
    return fail(ctx, HETEFF_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CK(call, what)                                   \
    do {                                                 \
        cudaError_t e_ = (call);                         \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, what); \
    } while (0)

// grow a zero-initialized device buffer (contents are not preserved)
static cudaError_t ensure(DevBuf &b, size_t bytes, bool zero)
{
    if (bytes <= b.bytes && b.p) return cudaSuccess;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.bytes = 0;
    size_t want = bytes < 256 ? 256 : bytes + bytes / 4;
    cudaError_t e = cudaMalloc(&b.p, want);
    if (e != cudaSuccess) return e;
    b.bytes = want;
    if (zero) e = cudaMemset(b.p, 0, want);
    return e;
}

// which compilation analyses a trace: CSR inputs the 15 x 11 one; res-column inputs by the
// average device record run (the host side when there are no devices)
static int pick_compilation(const heteff_trace *t)
{
    if (t->host_seg || t->dev_seg) return 0;
    const int64_t run = t->dev_ids > 0 ? t->dev.count / t->dev_ids
                                       : (t->host_ids > 0 ? t->host.count / t->host_ids : 0);
    if (const char *e = getenv("HETEFF_COMPILATION")) {   // tuning / test override of the choice below
        const int c = atoi(e);
        if (c == 1 || c == 2) return c;
    }
    return run >= kLongRun ? 2 : 1;
}
static cudaError_t reset_globals(heteff_ctx *ctx)
{
    hb::Globals g0;
    memset(&g0, 0, sizeof(g0));
    g0.contract_index = LLONG_MAX;
    return cudaMemcpy(ctx->g, &g0, sizeof(g0), cudaMemcpyHostToDevice);
}

static_assert(sizeof(hb::ResultDev) <= 256, "result header slot of the output block");

extern "C" {

int heteff_abi_version(void) { return HETEFF_ABI_VERSION; }

heteff_ctx *heteff_create(int device)
{
    heteff_ctx *ctx = new heteff_ctx();
    ctx->device = device;
    if (cudaSetDevice(device) != cudaSuccess) { delete ctx; return nullptr; }
    if (cudaMalloc(&ctx->g, sizeof(hb::Globals)) != cudaSuccess) { delete ctx; return nullptr; }
    if (cudaMalloc(&ctx->res_d, sizeof(hb::ResultDev)) != cudaSuccess) { delete ctx; return nullptr; }
    if (cudaMallocHost(&ctx->res_h, sizeof(hb::ResultDev)) != cudaSuccess) { delete ctx; return nullptr; }
    if (reset_globals(ctx) != cudaSuccess) { delete ctx; return nullptr; }
    cudaEventCreate(&ctx->ev0);
    cudaEventCreate(&ctx->ev1);
    cudaEventCreate(&ctx->ev_split0);
    cudaEventCreate(&ctx->ev_split1);
    for (int c = 0; c < 3; ++c) {
        ctx->grid[c] = kCompilations[c].grid(device);
        if (ctx->grid[c] <= 0) { heteff_destroy(ctx); return nullptr; }   // a tile geometry does not fit this GPU
    }
    if (const char *g = getenv("HETEFF_GRID")) {
        const int v = atoi(g);
        if (v > 0) ctx->grid[0] = ctx->grid[1] = ctx->grid[2] = v;
    }
    return ctx;
}

const char *heteff_kernel_name(const heteff_ctx *ctx) { return ctx ? ctx->kernel.c_str() : ""; }

int heteff_set_grid(heteff_ctx *ctx, int grid)
{
    if (!ctx || grid < 0) return fail(ctx, HETEFF_BAD_ARG, "bad grid");
    for (int c = 0; c < 3; ++c) ctx->grid[c] = grid > 0 ? grid : kCompilations[c].grid(ctx->device);
    return HETEFF_OK;
}

void heteff_destroy(heteff_ctx *ctx)
{
    if (!ctx) return;
    DevBuf *bufs[] = {&ctx->host_acc, &ctx->dev_acc, &ctx->host_tiles, &ctx->dev_tiles, &ctx->host_out,
                      &ctx->dev_out, &ctx->lists, &ctx->stage, &ctx->aux, &ctx->sort_ws, &ctx->sorted, &ctx->reg_ws, &ctx->reg_out, &ctx->iv_ws, &ctx->out_blk, &ctx->csr_res, &ctx->split};
    for (DevBuf *b : bufs)
        if (b->p) cudaFree(b->p);
    if (ctx->g) cudaFree(ctx->g);
    if (ctx->res_d) cudaFree(ctx->res_d);
    if (ctx->res_h) cudaFreeHost(ctx->res_h);
    if (ctx->out_pin) cudaFreeHost(ctx->out_pin);
    if (ctx->in_pin) cudaFreeHost(ctx->in_pin);
    if (ctx->split_pin) cudaFreeHost(ctx->split_pin);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->ev_split0) cudaEventDestroy(ctx->ev_split0);
    if (ctx->ev_split1) cudaEventDestroy(ctx->ev_split1);
    hb::transfer_free(ctx->xfer);
    delete ctx;
}

const char *heteff_last_error(const heteff_ctx *ctx) { return ctx ? ctx->err.c_str() : "no context"; }

static bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

struct IntoBlock {   // heteff_analyze_into: results go to a caller-owned device block, no sync
    void *p;
    int32_t n_max, m_max;
};

static int run_once(heteff_ctx *ctx, const heteff_trace *t, const heteff_options *opt, heteff_result *result,
                    const heteff_outputs *out, cudaStream_t s, const int64_t *const perms[2] = nullptr,
                    const IntoBlock *into = nullptr)
{
    if (!ctx || !t || !opt || !result) return fail(ctx, HETEFF_BAD_ARG, "null argument");
    if (t->host.count < 0 || t->dev.count < 0 || t->host_ids < 0 || t->dev_ids < 0 || t->n < 0 || t->m < 0 ||
        opt->list_capacity < 0)
        return fail(ctx, HETEFF_BAD_ARG, "negative size");
    if (opt->mode < 0 || opt->mode > 3) return fail(ctx, HETEFF_BAD_ARG, "bad mode");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    const int comp = pick_compilation(t);
    const Compilation &K = kCompilations[comp];
    ctx->kernel = K.name;
    const int64_t tile = K.tile();
    const int64_t ht = (t->host.count + tile - 1) / tile;
    const int64_t dt = (t->dev.count + tile - 1) / tile;
    const int64_t hid = t->host_ids > 0 ? t->host_ids : 1, did = t->dev_ids > 0 ? t->dev_ids : 1;

    // workspace (grow on demand; accumulators and tile flags start zeroed)
    if (hid > ctx->host_ids_cap) {
        CK(ensure(ctx->host_acc, (size_t)hid * 3 * sizeof(u64), true), "alloc host accumulators");
        ctx->host_ids_cap = (int64_t)(ctx->host_acc.bytes / (3 * sizeof(u64)));
    }
    if (did > ctx->dev_ids_cap) {
        CK(ensure(ctx->dev_acc, (size_t)did * 4 * sizeof(u64), true), "alloc device accumulators");
        ctx->dev_ids_cap = (int64_t)(ctx->dev_acc.bytes / (4 * sizeof(u64)));
    }
    // look-back slots: host 2 x 2 words, device 2 x 4 words per tile
    if (ht + 1 > ctx->host_tiles_cap) {
        CK(ensure(ctx->host_tiles, (size_t)(ht + 1) * 32, true), "alloc host tile status");
        ctx->host_tiles_cap = (int64_t)(ctx->host_tiles.bytes / 32);
    }
    if (dt + 1 > ctx->dev_tiles_cap) {
        CK(ensure(ctx->dev_tiles, (size_t)(dt + 1) * 64, true), "alloc device tile status");
        ctx->dev_tiles_cap = (int64_t)(ctx->dev_tiles.bytes / 64);
    }
    const size_t ob_res = 256, ob_h = (size_t)(t->n > 0 ? t->n : 0) * 32, ob_d = (size_t)(t->m > 0 ? t->m : 0) * 32;
    const size_t ob_total = ob_res + ob_h + ob_d;
    CK(ensure(ctx->out_blk, ob_total, true), "alloc result block");   // zeroed once: every byte the D2H reads is defined
    if (ctx->out_pin_bytes < ob_total) {
        if (ctx->out_pin) cudaFreeHost(ctx->out_pin);
        ctx->out_pin = nullptr;
        ctx->out_pin_bytes = 0;
        CK(cudaMallocHost(&ctx->out_pin, ob_total + ob_total / 4), "alloc pinned results");
        ctx->out_pin_bytes = ob_total + ob_total / 4;
    }
    if (opt->list_capacity > ctx->lists_cap) {
        CK(ensure(ctx->lists, (size_t)opt->list_capacity * 8 * sizeof(int64_t), false), "alloc lists");
        ctx->lists_cap = opt->list_capacity;
    }
    if (++ctx->epoch >= (1u << 30)) {   // epoch wrap: clear tile status once
        CK(cudaMemset(ctx->host_tiles.p, 0, ctx->host_tiles.bytes), "memset");
        CK(cudaMemset(ctx->dev_tiles.p, 0, ctx->dev_tiles.bytes), "memset");
        ctx->epoch = 1;
    }

    hb::Params p;
    memset(&p, 0, sizeof(p));
    p.hs = (const u64 *)t->host.start; p.he = (const u64 *)t->host.end; p.hr = t->host.res; p.hk = t->host.kind; p.hn = t->host.count;
    p.ds = (const u64 *)t->dev.start; p.de = (const u64 *)t->dev.end; p.dr = t->dev.res; p.dk = t->dev.kind; p.dn = t->dev.count;
    p.hseg = t->host_seg; p.dseg = t->dev_seg;
    if (p.hseg) p.hr = nullptr;
    if (p.dseg) p.dr = nullptr;
    p.host_ids = t->host_ids; p.dev_ids = t->dev_ids;
    p.host_decl = t->host_decl; p.dev_decl = t->dev_decl;
    p.n = t->n; p.m = t->m;
    p.host_elapsed_floor = t->host_elapsed_floor;
    p.mode = opt->mode;
    p.elapsed_arg = opt->elapsed;
    p.cap = opt->list_capacity;
    p.host_tiles = ht; p.dev_tiles = dt;
    p.epoch = ctx->epoch;
    if ((t->host.count > 0 && ((!p.hr && !p.hseg) || (p.hseg && t->host_ids < 1))) ||
        (t->dev.count > 0 && ((!p.dr && !p.dseg) || (p.dseg && t->dev_ids < 1))))
        return fail(ctx, HETEFF_BAD_ARG, "records need a res column or CSR offsets");
    const void *cols[8] = {p.hs, p.he, p.hr, p.hk, p.ds, p.de, p.dr, p.dk};
    bool al = true;
    for (const void *c : cols) al = al && (!c || aligned16(c));
    p.use_tma = al ? 1 : 0;
    u64 *ha = static_cast<u64 *>(ctx->host_acc.p);
    const size_t hc = (size_t)ctx->host_ids_cap;
    p.h_off = ha; p.h_mpi = ha + hc; p.h_span = ha + 2 * hc;
    u64 *da = static_cast<u64 *>(ctx->dev_acc.p);
    const size_t dc = (size_t)ctx->dev_ids_cap;
    p.d_k = da; p.d_km = da + dc; p.d_clamp = da + 2 * dc; p.d_maxend = da + 3 * dc;
    {
        u64 *b = static_cast<u64 *>(ctx->host_tiles.p);
        p.h_slotA = b;
        p.h_slotP = b + 2 * (size_t)ctx->host_tiles_cap;
    }
    {
        u64 *b = static_cast<u64 *>(ctx->dev_tiles.p);
        p.d_slotA = b;
        p.d_slotP = b + 4 * (size_t)ctx->dev_tiles_cap;
    }
    p.g = ctx->g;
    int64_t *lb = static_cast<int64_t *>(ctx->lists.p);
    for (int i = 0; i < 8; ++i) p.lists[i] = lb ? lb + (size_t)i * (size_t)ctx->lists_cap : nullptr;
    uint8_t *blk = static_cast<uint8_t *>(ctx->out_blk.p);
    p.res = reinterpret_cast<hb::ResultDev *>(blk);
    p.host_out = reinterpret_cast<u64 *>(blk + ob_res);
    p.dev_out = reinterpret_cast<u64 *>(blk + ob_res + ob_h);
    if (opt->flags & HETEFF_FLAG_ELAPSED_DEVICE_PTR) p.elapsed_ptr = reinterpret_cast<const u64 *>(opt->elapsed);
    if (into) {   // [host header | device header | host rows [n_max] | device rows [m_max]]
        uint8_t *b = static_cast<uint8_t *>(into->p);
        p.res = reinterpret_cast<hb::ResultDev *>(b + (opt->mode == HETEFF_MODE_SUMMARIZE_DEVICE ? 256 : 0));
        p.host_out = reinterpret_cast<u64 *>(b + 512);
        p.dev_out = reinterpret_cast<u64 *>(b + 512 + (size_t)into->n_max * 32);
        p.settle = 1;   // no error-path kernels follow in block mode (status -1 defers)
        CK(K.launch(&p, ctx->grid[comp], s), "launch analyze");
        return HETEFF_OK;
    }
    const bool want_sums = out && (out->host_summaries || out->device_summaries);
    const size_t ob_copy = want_sums ? ob_total : sizeof(hb::ResultDev);

    CK(cudaEventRecord(ctx->ev0, s), "event");
    CK(K.launch(&p, ctx->grid[comp], s), "launch analyze");
    CK(cudaEventRecord(ctx->ev1, s), "event");
    CK(cudaMemcpyAsync(ctx->out_pin, blk, ob_copy, cudaMemcpyDeviceToHost, s), "d2h results");
    CK(cudaStreamSynchronize(s), "analysis");
    if (reinterpret_cast<const hb::ResultDev *>(ctx->out_pin)->status == -1) {
        // some host records overlap: exact overlap findings, then the finalize
        if (p.hseg) {   // the error-path kernels walk a res column: expand the offsets once
            CK(ensure(ctx->csr_res, (size_t)t->host.count * 4 + 256, false), "alloc res column");
            CK(hb::launch_expand_res(p.hseg, t->host_ids, t->host.count, static_cast<int32_t *>(ctx->csr_res.p), s),
               "expand host res");
            p.hr = static_cast<const int32_t *>(ctx->csr_res.p);
        }
        CK(ensure(ctx->aux, (size_t)(ht + 1) * 3 * sizeof(u64), false), "alloc overlap scratch");
        CK(K.overlap(&p, static_cast<u64 *>(ctx->aux.p), s), "launch overlap pass");   // same compilation
        CK(cudaMemcpyAsync(ctx->out_pin, blk, ob_copy, cudaMemcpyDeviceToHost, s), "d2h results");
        CK(cudaStreamSynchronize(s), "overlap pass");
    }
    *ctx->res_h = *reinterpret_cast<const hb::ResultDev *>(ctx->out_pin);
    if (out && out->host_summaries && t->n > 0)
        memcpy(out->host_summaries, static_cast<uint8_t *>(ctx->out_pin) + ob_res, ob_h);
    if (out && out->device_summaries && t->m > 0)
        memcpy(out->device_summaries, static_cast<uint8_t *>(ctx->out_pin) + ob_res + ob_h, ob_d);
    const hb::ResultDev &r = *ctx->res_h;
    if (perms && opt->list_capacity > 0) {   // sorted re-run: list entries back to input positions
        for (int i = 0; i < 8; ++i) {
            const int64_t k = r.counts[i] < opt->list_capacity ? r.counts[i] : opt->list_capacity;
            const int64_t *pm = perms[i < 4 ? 0 : 1];
            if (k > 0 && pm) CK(hb::launch_remap(p.lists[i], k, pm, s), "launch remap");
        }
    }
    if (out && opt->list_capacity > 0) {
        for (int i = 0; i < 8; ++i) {
            int64_t k = r.counts[i] < opt->list_capacity ? r.counts[i] : opt->list_capacity;
            if (k > 0 && out->lists[i])
                CK(cudaMemcpyAsync(out->lists[i], p.lists[i], (size_t)k * sizeof(int64_t), cudaMemcpyDeviceToHost, s),
                   "d2h lists");
        }
        CK(cudaStreamSynchronize(s), "lists");
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    result->status = r.status;
    result->contract_flags = r.contract_flags;
    result->contract_index = r.contract_index;
    result->host_elapsed = r.host_elapsed;
    result->elapsed = r.elapsed;
    result->dev_max_end = r.dev_max_end;
    result->host_present = r.host_present;
    result->device_present = r.device_present;
    for (int i = 0; i < 5; ++i) result->host_metrics[i] = r.host_metrics[i];
    for (int i = 0; i < 4; ++i) result->device_metrics[i] = r.device_metrics[i];
    result->host_mask = r.host_mask;
    result->device_mask = r.device_mask;
    for (int i = 0; i < 8; ++i) result->counts[i] = r.counts[i];
    result->kernel_ms = ms;
    ctx->err.clear();
    return r.status;
}

// sort one record set into ctx-owned columns (K3)
static int sort_side(heteff_ctx *ctx, const heteff_records &in, heteff_columns &out, int64_t *perm,
                     heteff_sort_info *info, cudaStream_t s)
{
    const int64_t n = in.count;
    if (n <= 0) return HETEFF_OK;
    const size_t need = hb::sort_workspace_bytes(n);
    CK(ensure(ctx->sort_ws, need, false), "alloc sort workspace");
    hb::SortStats st{};
    CK(cudaEventRecord(ctx->ev0, s), "event");
    CK(hb::sort_records((const u64 *)in.start, (const u64 *)in.end, in.res, in.kind, n, (u64 *)out.start,
                        (u64 *)out.end, out.res, out.kind, perm,
                        ctx->sort_ws.p, ctx->sort_ws.bytes, s, &st),
       "sort records");
    CK(cudaEventRecord(ctx->ev1, s), "event");
    if (info) {
        CK(cudaEventSynchronize(ctx->ev1), "sort");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        info->key_bits = st.key_bits;
        info->passes = st.passes;
        info->wide = st.wide;
        info->start_sorted = st.start_sorted;
        info->ms = ms;
    }
    return HETEFF_OK;
}

// CSR offsets -> res columns in ctx->csr_res (for the paths that walk res: K3, regions)
static int materialize_res(heteff_ctx *ctx, const heteff_trace *t, heteff_trace *o, cudaStream_t s)
{
    *o = *t;
    if (!t->host_seg && !t->dev_seg) return HETEFF_OK;
    const int64_t hn = t->host_seg ? t->host.count : 0, dn = t->dev_seg ? t->dev.count : 0;
    const size_t hb = ((size_t)hn * 4 + 255) & ~(size_t)255;
    CK(ensure(ctx->csr_res, hb + (size_t)dn * 4 + 256, false), "alloc res columns");
    int32_t *b = static_cast<int32_t *>(ctx->csr_res.p);
    if (t->host_seg) {
        CK(hb::launch_expand_res(t->host_seg, t->host_ids, hn, b, s), "expand host res");
        o->host.res = b;
        o->host_seg = nullptr;
    }
    if (t->dev_seg) {
        int32_t *d = reinterpret_cast<int32_t *>(reinterpret_cast<uint8_t *>(b) + hb);
        CK(hb::launch_expand_res(t->dev_seg, t->dev_ids, dn, d, s), "expand dev res");
        o->dev.res = d;
        o->dev_seg = nullptr;
    }
    return HETEFF_OK;
}

// Split analysis: the host records and the device records as two launches, each with the
// tile geometry best for its own record runs, E handed over in device memory, then the merge
// kernel -- the multi-GPU protocol at world size 1 (include/heteff_b200.h "multi-GPU").
// Taken for large REPORT calls without finding lists whose two sides prefer different
// compilations (C5: host runs of 2.4e5 -> 8 x 19, device runs of 6.1e4 -> 11 x 15): C5
// 7.05 -> 6.75 ms (tools/split_probe.py); identical results, the counts of the findings
// included (the late-record count is the clamp count: E is the host elapsed).  Returns
// HETEFF_PARSE_FALLBACK when the single launch must decide (a shard is not OK).
static bool split_wanted(const heteff_trace *t, const heteff_options *opt)
{
    if (opt->mode != HETEFF_MODE_REPORT || opt->flags != 0 || opt->list_capacity != 0) return false;
    if (t->n < 1 || t->m < 1 || getenv("HETEFF_NO_SPLIT")) return false;
    if (getenv("HETEFF_FORCE_SPLIT")) return true;   // tests / stress: every eligible call
    const int64_t min = getenv("HETEFF_SPLIT_MIN") ? atoll(getenv("HETEFF_SPLIT_MIN")) : ((int64_t)1 << 26);
    if (t->host.count < min || t->dev.count < min || 4 * t->host.count < t->host.count + t->dev.count) return false;
    heteff_trace h = *t, d = *t;
    h.dev.count = 0; h.dev_ids = 0; h.dev_seg = nullptr;
    d.host.count = 0; d.host_ids = 0; d.host_seg = nullptr;
    return pick_compilation(&h) != pick_compilation(&d);
}

static int run_split(heteff_ctx *ctx, const heteff_trace *t, heteff_result *result, const heteff_outputs *out,
                     cudaStream_t s)
{
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    const int32_t n = t->n, m = t->m;
    const size_t bytes = 512 + 32 * ((size_t)n + (size_t)m);
    CK(ensure(ctx->split, bytes + 256, true), "alloc split block");
    uint8_t *blk = static_cast<uint8_t *>(ctx->split.p);
    // the device pass and the merge read E where the host pass's finalize writes it: the
    // host header's host_elapsed (the device pass's header goes to blk + 256)
    u64 *e_dev = reinterpret_cast<u64 *>(blk + offsetof(hb::ResultDev, host_elapsed));
    heteff_trace th = *t, td = *t;   // host records only / device records only
    th.dev.count = 0; th.dev.start = th.dev.end = nullptr; th.dev.res = nullptr; th.dev.kind = nullptr;
    th.dev_ids = 0; th.m = 0; th.dev_decl = nullptr; th.dev_seg = nullptr;
    td.host.count = 0; td.host.start = td.host.end = nullptr; td.host.res = nullptr; td.host.kind = nullptr;
    td.host_ids = 0; td.n = 0; td.host_decl = nullptr; td.host_seg = nullptr; td.host_elapsed_floor = 0;
    heteff_options oh{}, od{};
    oh.mode = HETEFF_MODE_SUMMARIZE_HOST;
    od.mode = HETEFF_MODE_SUMMARIZE_DEVICE;
    od.flags = HETEFF_FLAG_ELAPSED_DEVICE_PTR;
    od.elapsed = (uint64_t)(uintptr_t)e_dev;
    IntoBlock into{blk, n, m};
    heteff_result r{};
    CK(cudaEventRecord(ctx->ev_split0, s), "event");
    int rc = run_once(ctx, &th, &oh, &r, nullptr, s, nullptr, &into);
    if (rc != HETEFF_OK) return rc;
    rc = run_once(ctx, &td, &od, &r, nullptr, s, nullptr, &into);
    if (rc != HETEFF_OK) return rc;
    // both passes' headers (finding counts) come back with the merged result: enqueued before
    // the merge, whose sync covers them; the merge sums the device rows' clamp counts
    constexpr size_t kHeads = 512;
    if (ctx->split_pin_bytes < kHeads) {
        if (ctx->split_pin) cudaFreeHost(ctx->split_pin);
        ctx->split_pin = nullptr;
        ctx->split_pin_bytes = 0;
        CK(cudaMallocHost(&ctx->split_pin, kHeads), "alloc pinned split headers");
        ctx->split_pin_bytes = kHeads;
    }
    CK(cudaMemcpyAsync(ctx->split_pin, blk, kHeads, cudaMemcpyDeviceToHost, s), "d2h split headers");
    const int32_t n_of = n, m_of = m;
    rc = heteff_merge_shards(ctx, blk, 1, bytes, n, m, &n_of, &m_of, reinterpret_cast<const uint64_t *>(e_dev), result,
                             out, s);
    if (rc != HETEFF_OK || result->status != HETEFF_OK) return HETEFF_PARSE_FALLBACK;
    CK(cudaEventRecord(ctx->ev_split1, s), "event");
    CK(cudaEventSynchronize(ctx->ev_split1), "split");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev_split0, ctx->ev_split1);   // both launches, the hand-over, the merge
    const uint8_t *hb_ = static_cast<const uint8_t *>(ctx->split_pin);
    const hb::ResultDev *hdr = reinterpret_cast<const hb::ResultDev *>(hb_);   // [0] host pass, at 256 the device pass
    const hb::ResultDev &hdev = *reinterpret_cast<const hb::ResultDev *>(hb_ + 256);
    // the late-device count is the clamp count (E = host elapsed), summed by the merge
    const hb::ResultDev &merged = *static_cast<const hb::ResultDev *>(ctx->out_pin);
    for (int i = 0; i < 8; ++i) result->counts[i] = hdr[0].counts[i] + hdev.counts[i];
    result->counts[7] = merged.counts[7];
    result->host_elapsed = result->elapsed;
    result->dev_max_end = 0;
    result->contract_flags = 0;
    result->contract_index = -1;
    result->kernel_ms = ms;
    ctx->kernel = std::string("split: host ") + kCompilations[pick_compilation(&th)].name + ", device " +
                  kCompilations[pick_compilation(&td)].name;
    ctx->err.clear();
    return HETEFF_OK;
}

static int run_analysis(heteff_ctx *ctx, const heteff_trace *t0, const heteff_options *opt, heteff_result *result,
                        const heteff_outputs *out, cudaStream_t s)
{
    if (split_wanted(t0, opt)) {
        const int rc = run_split(ctx, t0, result, out, s);
        if (rc != HETEFF_PARSE_FALLBACK) return rc;
    }
    if (!(opt->flags & HETEFF_FLAG_SORT_IF_NEEDED)) return run_once(ctx, t0, opt, result, out, s);
    heteff_trace tcol;   // the order check and K3 walk res columns
    {
        CK(cudaSetDevice(ctx->device), "cudaSetDevice");
        const int rc = materialize_res(ctx, t0, &tcol, s);
        if (rc != HETEFF_OK) return rc;
    }
    const heteff_trace *t = &tcol;
    // canonical-order check of both sides (12 B/record), then sort only what needs it
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    CK(ensure(ctx->aux, 256, false), "alloc order flags");
    unsigned int *bad = static_cast<unsigned int *>(ctx->aux.p);
    CK(cudaMemsetAsync(bad, 0, 8, s), "memset");
    CK(hb::launch_order_check(t->host.res, (const u64 *)t->host.start, t->host.count, bad, s), "order check");
    CK(hb::launch_order_check(t->dev.res, (const u64 *)t->dev.start, t->dev.count, bad + 1, s), "order check");
    unsigned int flags_h[2] = {0, 0};
    CK(cudaMemcpyAsync(flags_h, bad, 8, cudaMemcpyDeviceToHost, s), "d2h");
    CK(cudaStreamSynchronize(s), "order check");
    if (!flags_h[0] && !flags_h[1]) return run_once(ctx, t, opt, result, out, s);
    int rc;
    // K3: sort the offending side(s) into ctx-owned columns and analyze
    const bool sh = flags_h[0] != 0;
    const bool sd = flags_h[1] != 0;
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const int64_t hn = sh ? t->host.count : 0, dn = sd ? t->dev.count : 0;
    const size_t bytes = up((size_t)hn * 29) + up((size_t)hn * 8) + up((size_t)dn * 29) + up((size_t)dn * 8) + 2048;
    CK(ensure(ctx->sorted, bytes, false), "alloc sorted columns");
    uint8_t *b = static_cast<uint8_t *>(ctx->sorted.p);
    size_t o = 0;
    auto take = [&](size_t x) { void *q = b + o; o += up(x); return q; };
    heteff_trace ts = *t;
    int64_t *perm[2] = {nullptr, nullptr};
    const int64_t *perms[2] = {nullptr, nullptr};
    const heteff_records *src[2] = {&t->host, &t->dev};
    heteff_records *dst[2] = {&ts.host, &ts.dev};
    const bool doit[2] = {sh, sd};
    for (int side = 0; side < 2; ++side) {
        if (!doit[side]) continue;
        const int64_t n = src[side]->count;
        heteff_columns c;
        c.start = static_cast<uint64_t *>(take((size_t)n * 8));
        c.end = static_cast<uint64_t *>(take((size_t)n * 8));
        c.res = static_cast<int32_t *>(take((size_t)n * 4));
        c.kind = static_cast<uint8_t *>(take((size_t)n));
        perm[side] = static_cast<int64_t *>(take((size_t)n * 8));
        perms[side] = perm[side];
        if ((rc = sort_side(ctx, *src[side], c, perm[side], nullptr, s)) != HETEFF_OK) return rc;
        dst[side]->start = c.start;
        dst[side]->end = c.end;
        dst[side]->res = c.res;
        dst[side]->kind = c.kind;
    }
    rc = run_once(ctx, &ts, opt, result, out, s, perms);
    if (result->contract_index >= 0 && result->contract_index < LLONG_MAX) {
        const int side = (result->contract_flags & (HETEFF_CONTRACT_HOST_ORDER | HETEFF_CONTRACT_HOST_KIND)) ? 0 : 1;
        if (perm[side]) {
            int64_t orig = 0;
            CK(cudaMemcpyAsync(&orig, perm[side] + result->contract_index, 8, cudaMemcpyDeviceToHost, s), "d2h");
            CK(cudaStreamSynchronize(s), "sync");
            result->contract_index = orig;
        }
    }
    return rc;
}

int heteff_analyze_regions(heteff_ctx *ctx, const heteff_trace *t, const heteff_regions *rg,
                           heteff_region_outputs *out, void *stream)
{
    if (!ctx || !t || !rg || !out || rg->count < 0) return fail(ctx, HETEFF_BAD_ARG, "bad argument");
    if (rg->flags & ~HETEFF_REGIONS_PER_RANK) return fail(ctx, HETEFF_BAD_ARG, "unknown region flags");
    const bool per_rank = (rg->flags & HETEFF_REGIONS_PER_RANK) != 0;
    const bool no_table = per_rank && t->host_ids == 0;   // per-rank regions without ranks: empty tables
    if (rg->count > 0 && (!out->results || (!no_table && (!rg->start || !rg->end))))
        return fail(ctx, HETEFF_BAD_ARG, "null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    // the whole trace first: validity and canonical order are preconditions
    heteff_options o0{};
    o0.mode = HETEFF_MODE_REPORT;
    heteff_result r0{};
    int rc = run_analysis(ctx, t, &o0, &r0, nullptr, s);
    heteff_trace tcol;   // the region kernels walk res columns
    if (rc == HETEFF_OK || rc == HETEFF_ANALYSIS_ERROR) {
        const int mr = materialize_res(ctx, t, &tcol, s);
        if (mr != HETEFF_OK) return mr;
        t = &tcol;
    }
    if (rc != HETEFF_OK && rc != HETEFF_ANALYSIS_ERROR) return rc;
    out->kernel_ms = 0.0;
    if (rg->count == 0) return HETEFF_OK;

    const int W = hb::kMaxWindows;
    const int64_t hid = t->host_ids > 0 ? t->host_ids : 1, did = t->dev_ids > 0 ? t->dev_ids : 1;
    const int64_t tiles = (int64_t)hb::region_tiles(t->dev.count);
    const int64_t hch = (int64_t)hb::region_hchunks(t->host.count);
    const int64_t nn = t->n > 0 ? t->n : 1, mm = t->m > 0 ? t->m : 1;
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const int64_t scan_blocks = ((hch > tiles ? hch : tiles) + 1023) / 1024 + 1;   // per seg_scan
    const size_t b_hseg = up((size_t)(hid + 1) * 8), b_dseg = up((size_t)(did + 1) * 8);
    const size_t b_hagg = up((size_t)(hch + 1) * 48), b_hck = up((size_t)(hch + 1) * 40);
    const size_t b_dagg = up((size_t)(tiles + 1) * 24), b_drun = up((size_t)(tiles + 1) * 16);
    const size_t b_dsum = up((size_t)(tiles + 1) * 32), b_dck = up((size_t)(tiles + 1) * 24);
    const size_t b_scan = up((size_t)scan_blocks * 64), b_tst = up((size_t)(tiles + 1) * 16);
    const size_t b_dsub = up((size_t)(tiles + 1) * hb::region_subs() * 64);
    const size_t b_hacc = up((size_t)W * hid * 24), b_dacc = up((size_t)W * did * 32);
    const size_t b_E = up(W * 8), b_dmax = up(W * 8), b_own = up((size_t)did * 4);
    const size_t b_hwin = per_rank ? up((size_t)W * hid * 16) : 0;
    CK(ensure(ctx->reg_ws, b_hseg + b_dseg + b_hagg + b_hck + b_dagg + b_drun + b_dsum + b_dck + b_scan + b_tst + b_dsub + b_hacc +
                               b_dacc + b_E + b_dmax + b_own + b_hwin, false),
       "alloc regions");
    const size_t b_ho = up((size_t)W * nn * 32), b_do = up((size_t)W * mm * 32), b_bo = up((size_t)W * mm * 8);
    const size_t b_res = up(W * sizeof(hb::RegionResultDev));
    CK(ensure(ctx->reg_out, b_ho + b_do + b_bo + b_res, true), "alloc region outputs");   // zeroed once (initcheck)
    uint8_t *w = static_cast<uint8_t *>(ctx->reg_ws.p);
    hb::RegParams p;
    memset(&p, 0, sizeof(p));
    p.hs = (const u64 *)t->host.start; p.he = (const u64 *)t->host.end; p.hr = t->host.res; p.hk = t->host.kind;
    p.hn = t->host.count;
    p.ds = (const u64 *)t->dev.start; p.de = (const u64 *)t->dev.end; p.dr = t->dev.res; p.dk = t->dev.kind;
    p.dn = t->dev.count;
    p.host_ids = t->host_ids; p.dev_ids = t->dev_ids;
    p.host_decl = t->host_decl; p.dev_decl = t->dev_decl;
    p.n = t->n; p.m = t->m;
    size_t o = 0;
    auto take = [&](size_t b) { void *q = w + o; o += b; return q; };
    p.hseg = static_cast<int64_t *>(take(b_hseg));
    p.dseg = static_cast<int64_t *>(take(b_dseg));
    p.hagg = static_cast<u64 *>(take(b_hagg));
    p.hck = static_cast<u64 *>(take(b_hck));
    p.dagg = static_cast<u64 *>(take(b_dagg));
    p.drun = static_cast<u64 *>(take(b_drun));
    p.dsum = static_cast<u64 *>(take(b_dsum));
    p.dck = static_cast<u64 *>(take(b_dck));
    p.scan_tmp = static_cast<u64 *>(take(b_scan));
    p.tstage = static_cast<int64_t *>(take(b_tst));
    p.dsub = static_cast<u64 *>(take(b_dsub));
    p.h_acc = static_cast<u64 *>(take(b_hacc));
    p.d_acc = static_cast<u64 *>(take(b_dacc));
    p.E = static_cast<u64 *>(take(b_E));
    p.dmax = static_cast<u64 *>(take(b_dmax));
    int32_t *own = static_cast<int32_t *>(take(b_own));
    u64 *hwin = per_rank ? static_cast<u64 *>(take(b_hwin)) : nullptr;
    std::vector<u64> hwin_h(per_rank ? (size_t)W * hid * 2 : 0);
    p.tiles = tiles;
    p.hchunks = hch;
    if (rg->dev_owner && t->dev_ids > 0) {
        CK(cudaMemcpyAsync(own, rg->dev_owner, (size_t)t->dev_ids * 4, cudaMemcpyHostToDevice, s), "h2d owners");
        p.owner = own;
    }
    uint8_t *ob = static_cast<uint8_t *>(ctx->reg_out.p);
    p.host_out = reinterpret_cast<u64 *>(ob);
    p.dev_out = reinterpret_cast<u64 *>(ob + b_ho);
    p.busy_out = reinterpret_cast<u64 *>(ob + b_ho + b_do);
    p.res = reinterpret_cast<hb::RegionResultDev *>(ob + b_ho + b_do + b_bo);
    hb::RegionResultDev rh[hb::kMaxWindows];
    float total_ms = 0.f;
    // window-independent checkpoints, once
    CK(cudaEventRecord(ctx->ev0, s), "event");
    CK(hb::launch_regions_prepare(p, s), "launch regions prepare");
    CK(cudaEventRecord(ctx->ev1, s), "event");
    CK(cudaEventSynchronize(ctx->ev1), "regions prepare");
    {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        total_ms += ms;
    }
    for (int32_t j0 = 0; j0 < rg->count; j0 += W) {
        const int R = rg->count - j0 < W ? rg->count - j0 : W;
        p.R = R;
        if (per_rank) {   // [R][host_ids][2] of this pass, one H2D (start / end are [count][host_ids])
            for (int j = 0; j < R; ++j)
                for (int64_t id = 0; id < t->host_ids; ++id) {
                    const size_t src = (size_t)(j0 + j) * (size_t)t->host_ids + (size_t)id;
                    hwin_h[((size_t)j * t->host_ids + id) * 2] = rg->start[src];
                    hwin_h[((size_t)j * t->host_ids + id) * 2 + 1] = rg->end[src];
                }
            if (t->host_ids > 0)
                CK(cudaMemcpyAsync(hwin, hwin_h.data(), (size_t)R * t->host_ids * 16, cudaMemcpyHostToDevice, s),
                   "h2d windows");
            p.hwin = hwin;
        }
        for (int j = 0; j < W; ++j) {
            const bool live = j < R && !per_rank;
            const uint64_t a = live ? rg->start[j0 + j] : 0, b = live ? rg->end[j0 + j] : 0;
            p.wlo[j] = a;
            p.whi[j] = b > a ? b : a;
        }
        CK(cudaMemsetAsync(p.E, 0, b_E + b_dmax, s), "memset");
        CK(cudaEventRecord(ctx->ev0, s), "event");
        CK(hb::launch_regions_phase1(p, s), "launch regions phase 1");
        CK(hb::launch_regions_phase2(p, s), "launch regions phase 2");   // reads E_j from device memory
        CK(cudaEventRecord(ctx->ev1, s), "event");
        CK(cudaMemcpyAsync(rh, p.res, sizeof(hb::RegionResultDev) * R, cudaMemcpyDeviceToHost, s), "d2h results");
        if (out->host_summaries && t->n > 0)
            CK(cudaMemcpyAsync(out->host_summaries + (size_t)j0 * t->n * 4, p.host_out, (size_t)R * t->n * 32,
                               cudaMemcpyDeviceToHost, s), "d2h host summaries");
        if (out->device_summaries && t->m > 0)
            CK(cudaMemcpyAsync(out->device_summaries + (size_t)j0 * t->m * 4, p.dev_out, (size_t)R * t->m * 32,
                               cudaMemcpyDeviceToHost, s), "d2h device summaries");
        if (out->offload_busy && t->m > 0)
            CK(cudaMemcpyAsync(out->offload_busy + (size_t)j0 * t->m, p.busy_out, (size_t)R * t->m * 8,
                               cudaMemcpyDeviceToHost, s), "d2h busy");
        CK(cudaStreamSynchronize(s), "regions");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        total_ms += ms;
        for (int j = 0; j < R; ++j) {
            heteff_region_result &x = out->results[j0 + j];
            const hb::RegionResultDev &y = rh[j];
            x.status = y.status;
            x.reserved = 0;
            x.elapsed = y.elapsed;
            for (int i = 0; i < 5; ++i) x.host_metrics[i] = y.host_metrics[i];
            for (int i = 0; i < 4; ++i) x.device_metrics[i] = y.device_metrics[i];
            x.host_mask = y.host_mask;
            x.device_mask = y.device_mask;
            x.offload_busy_fraction = y.busy_fraction;
            x.offload_busy_defined = y.busy_mask;
            x.reserved2 = 0;
        }
    }
    out->kernel_ms = total_ms;
    ctx->err.clear();
    return HETEFF_OK;
}

int heteff_flatten(heteff_ctx *ctx, const uint64_t *start, const uint64_t *end, int64_t n, uint64_t *out_start,
                   uint64_t *out_end, int64_t *out_n, int64_t *malformed_index, void *stream)
{
    if (!ctx || n < 0 || !out_n || !malformed_index || (n > 0 && (!start || !end || !out_start || !out_end)))
        return fail(ctx, HETEFF_BAD_ARG, "bad argument");
    if (n >= (int64_t)0xffffffffll) return fail(ctx, HETEFF_BAD_ARG, "too many intervals for one call");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    CK(ensure(ctx->iv_ws, hb::iv_flatten_ws(n), false), "alloc interval scratch");
    const cudaError_t e = hb::iv_flatten((const u64 *)start, (const u64 *)end, n, (u64 *)out_start, (u64 *)out_end,
                                         out_n, malformed_index, ctx->iv_ws.p, ctx->iv_ws.bytes,
                                         static_cast<cudaStream_t>(stream));
    if (*malformed_index >= 0) return fail(ctx, HETEFF_VALUE_ERROR, "malformed interval");
    if (e != cudaSuccess) return cuda_fail(ctx, e, "flatten");
    ctx->err.clear();
    return HETEFF_OK;
}

int heteff_subtract(heteff_ctx *ctx, const uint64_t *a_start, const uint64_t *a_end, int64_t na,
                    const uint64_t *b_start, const uint64_t *b_end, int64_t nb, uint64_t *out_start,
                    uint64_t *out_end, int64_t *out_n, void *stream)
{
    if (!ctx || na < 0 || nb < 0 || !out_n) return fail(ctx, HETEFF_BAD_ARG, "bad argument");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    CK(ensure(ctx->iv_ws, hb::iv_subtract_ws(na, nb), false), "alloc interval scratch");
    CK(hb::iv_subtract((const u64 *)a_start, (const u64 *)a_end, na, (const u64 *)b_start, (const u64 *)b_end, nb,
                       (u64 *)out_start, (u64 *)out_end, out_n, ctx->iv_ws.p, ctx->iv_ws.bytes,
                       static_cast<cudaStream_t>(stream)),
       "subtract");
    ctx->err.clear();
    return HETEFF_OK;
}

int heteff_intersect(heteff_ctx *ctx, const uint64_t *start, const uint64_t *end, int64_t n, uint64_t lo,
                     uint64_t hi, uint64_t *out_start, uint64_t *out_end, int64_t *out_n, void *stream)
{
    if (!ctx || n < 0 || !out_n) return fail(ctx, HETEFF_BAD_ARG, "bad argument");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    CK(ensure(ctx->iv_ws, hb::iv_intersect_ws(n), false), "alloc interval scratch");
    CK(hb::iv_intersect((const u64 *)start, (const u64 *)end, n, lo, hi, (u64 *)out_start, (u64 *)out_end, out_n,
                        ctx->iv_ws.p, ctx->iv_ws.bytes, static_cast<cudaStream_t>(stream)),
       "intersect");
    ctx->err.clear();
    return HETEFF_OK;
}

int heteff_total_duration(heteff_ctx *ctx, const uint64_t *start, const uint64_t *end, int64_t n, uint64_t out[2],
                          void *stream)
{
    if (!ctx || n < 0 || !out) return fail(ctx, HETEFF_BAD_ARG, "bad argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    CK(ensure(ctx->iv_ws, 256, false), "alloc interval scratch");
    CK(hb::iv_total((const u64 *)start, (const u64 *)end, n, static_cast<u64 *>(ctx->iv_ws.p), s), "total");
    CK(cudaMemcpyAsync(out, ctx->iv_ws.p, 16, cudaMemcpyDeviceToHost, s), "d2h");
    CK(cudaStreamSynchronize(s), "total");
    ctx->err.clear();
    return HETEFF_OK;
}

int heteff_analyze_into(heteff_ctx *ctx, const heteff_trace *trace, const heteff_options *opt, void *dev_block,
                        size_t block_bytes, int32_t n_max, int32_t m_max, void *stream)
{
    if (!ctx || !trace || !opt || !dev_block || n_max < 0 || m_max < 0) return fail(ctx, HETEFF_BAD_ARG, "bad argument");
    if (trace->n > n_max || trace->m > m_max || block_bytes < 512 + 32 * ((size_t)n_max + (size_t)m_max))
        return fail(ctx, HETEFF_BAD_ARG, "result block too small");
    if (opt->flags & HETEFF_FLAG_SORT_IF_NEEDED) return fail(ctx, HETEFF_BAD_ARG, "sort_if_needed needs the sync path");
    heteff_result r{};
    IntoBlock into{dev_block, n_max, m_max};
    return run_once(ctx, trace, opt, &r, nullptr, static_cast<cudaStream_t>(stream), nullptr, &into);
}

int heteff_merge_shards(heteff_ctx *ctx, const void *gathered, int32_t world, size_t block_bytes, int32_t n_max,
                        int32_t m_max, const int32_t *n_of, const int32_t *m_of, const uint64_t *elapsed_dev,
                        heteff_result *result, const heteff_outputs *out, void *stream)
{
    if (!ctx || !gathered || world < 1 || !n_of || !m_of || !elapsed_dev || !result)
        return fail(ctx, HETEFF_BAD_ARG, "bad argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    int64_t ntot = 0, mtot = 0;
    for (int r = 0; r < world; ++r) { ntot += n_of[r]; mtot += m_of[r]; }
    const size_t need = 256 + 32 * (size_t)(ntot + mtot) + 8 * (size_t)world;
    const size_t sizes_at = (256 + 32 * (size_t)(ntot + mtot) + 255) & ~(size_t)255;
    const size_t scratch_at = (sizes_at + 8 * (size_t)world + 255) & ~(size_t)255;
    CK(ensure(ctx->aux, scratch_at + hb::merge_scratch_bytes() + 256, false), "alloc merge output");
    uint8_t *dout = static_cast<uint8_t *>(ctx->aux.p);
    int32_t *sizes_d = reinterpret_cast<int32_t *>(dout + sizes_at);
    if (ctx->out_pin_bytes < need) {
        if (ctx->out_pin) cudaFreeHost(ctx->out_pin);
        ctx->out_pin = nullptr;
        ctx->out_pin_bytes = 0;
        CK(cudaMallocHost(&ctx->out_pin, need + need / 4), "alloc pinned results");
        ctx->out_pin_bytes = need + need / 4;
    }
    int32_t *sizes_h = static_cast<int32_t *>(ctx->out_pin);   // staged through pinned memory
    for (int r = 0; r < world; ++r) { sizes_h[r] = n_of[r]; sizes_h[world + r] = m_of[r]; }
    CK(cudaMemcpyAsync(sizes_d, sizes_h, 8 * (size_t)world, cudaMemcpyHostToDevice, s), "h2d sizes");
    CK(cudaEventRecord(ctx->ev0, s), "event");
    CK(hb::launch_merge(gathered, world, block_bytes, n_max, m_max, sizes_d, sizes_d + world, dout,
                        (const u64 *)elapsed_dev, dout + scratch_at, ntot + mtot, s),
       "launch merge");
    CK(cudaEventRecord(ctx->ev1, s), "event");
    const bool sums = out && (out->host_summaries || out->device_summaries);
    const size_t copy = sums ? 256 + 32 * (size_t)(ntot + mtot) : sizeof(hb::ResultDev);
    CK(cudaMemcpyAsync(ctx->out_pin, dout, copy, cudaMemcpyDeviceToHost, s), "d2h merged");
    CK(cudaStreamSynchronize(s), "merge");
    const hb::ResultDev &r = *static_cast<const hb::ResultDev *>(ctx->out_pin);
    memset(result, 0, sizeof(*result));
    result->status = r.status;
    result->elapsed = r.elapsed;
    result->host_elapsed = r.host_elapsed;
    for (int i = 0; i < 5; ++i) result->host_metrics[i] = r.host_metrics[i];
    for (int i = 0; i < 4; ++i) result->device_metrics[i] = r.device_metrics[i];
    result->host_mask = r.host_mask;
    result->device_mask = r.device_mask;
    result->host_present = ntot >= 1;
    result->device_present = mtot >= 1;
    if (r.status == 0 && sums) {
        const uint8_t *b = static_cast<const uint8_t *>(ctx->out_pin) + 256;
        if (out->host_summaries) memcpy(out->host_summaries, b, 32 * (size_t)ntot);
        if (out->device_summaries) memcpy(out->device_summaries, b + 32 * (size_t)ntot, 32 * (size_t)mtot);
    }
    ctx->err.clear();
    return r.status == -2 ? HETEFF_PARSE_FALLBACK : HETEFF_OK;
}

int heteff_sort_records(heteff_ctx *ctx, const heteff_records *in, const heteff_columns *out, int64_t *perm,
                        heteff_sort_info *info, void *stream)
{
    if (!ctx || !in || !out || in->count < 0) return fail(ctx, HETEFF_BAD_ARG, "bad argument");
    if (in->count > 0 && (!in->start || !in->end || !in->res || !in->kind || !out->start || !out->end ||
                          !out->res || !out->kind))
        return fail(ctx, HETEFF_BAD_ARG, "null column");
    if (in->count >= (int64_t)0xffffffffll) return fail(ctx, HETEFF_BAD_ARG, "record set too large for one sort");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    heteff_columns c = *out;
    heteff_sort_info local{};
    const int rc = sort_side(ctx, *in, c, perm, info ? info : &local, s);
    if (rc != HETEFF_OK) return rc;
    CK(cudaStreamSynchronize(s), "sort");
    ctx->err.clear();
    return HETEFF_OK;
}

int heteff_analyze(heteff_ctx *ctx, const heteff_trace *trace, const heteff_options *opt, heteff_result *result,
                   const heteff_outputs *out, void *stream)
{
    return run_analysis(ctx, trace, opt, result, out, static_cast<cudaStream_t>(stream));
}

// stage host columns into the context's device buffer, then analyze
// CSR offsets of one record set: seg[0] = 0, non-decreasing, seg[ids] = count
static bool seg_ok(const int64_t *seg, int32_t ids, int64_t count)
{
    if (!seg || ids < 0 || seg[0] != 0 || seg[ids] != count) return false;
    for (int32_t r = 0; r < ids; ++r)
        if (seg[r + 1] < seg[r]) return false;
    return true;
}

// host buffers -> staging (H2D on the stream) -> run_analysis.  With CSR offsets
// (hseg / dseg non-null) the res columns are not copied but expanded on the device.
static int analyze_host_impl(heteff_ctx *ctx, const heteff_trace *trace, const int64_t *hseg, const int64_t *dseg,
                             const heteff_options *opt, heteff_result *result, const heteff_outputs *out, void *stream)
{
    if (!ctx || !trace) return fail(ctx, HETEFF_BAD_ARG, "null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    const int64_t hn = trace->host.count, dn = trace->dev.count;
    auto up = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t hb8 = up((size_t)hn * 8), hb4 = up((size_t)hn * 4), hb1 = up((size_t)hn);
    const size_t db8 = up((size_t)dn * 8), db4 = up((size_t)dn * 4), db1 = up((size_t)dn);
    const size_t hd = up((size_t)(trace->host_decl ? trace->host_ids : 0) * 4);
    const size_t dd = up((size_t)(trace->dev_decl ? trace->dev_ids : 0) * 4);
    const size_t hs8 = hseg ? up(((size_t)trace->host_ids + 1) * 8) : 0;
    const size_t ds8 = dseg ? up(((size_t)trace->dev_ids + 1) * 8) : 0;
    const size_t total = 2 * hb8 + (hseg ? 0 : hb4) + hb1 + 2 * db8 + (dseg ? 0 : db4) + db1 + hd + dd + hs8 + ds8;
    CK(ensure(ctx->stage, total, false), "alloc staging");
    uint8_t *b = static_cast<uint8_t *>(ctx->stage.p);
    // small inputs in pageable memory (the drop-in API on ordinary traces): gather every
    // column into one pinned block and issue ONE copy instead of one driver-staged copy per
    // column; large or pinned inputs are copied column by column at PCIe rate
    bool gather = total <= ((size_t)8 << 20);
    if (gather) {   // pinned caller memory already copies at full rate: gather pageable memory only
        const void *probe = hn ? (const void *)trace->host.start : (const void *)trace->dev.start;
        cudaPointerAttributes pa;
        if (probe && cudaPointerGetAttributes(&pa, probe) == cudaSuccess && pa.type != cudaMemoryTypeUnregistered)
            gather = false;
        cudaGetLastError();
    }
    if (gather && ctx->in_pin_bytes < total) {
        if (ctx->in_pin) cudaFreeHost(ctx->in_pin);
        ctx->in_pin = nullptr;
        ctx->in_pin_bytes = 0;
        CK(cudaMallocHost(&ctx->in_pin, total), "alloc pinned inputs");
        ctx->in_pin_bytes = total;
    }
    uint8_t *hpin = gather ? static_cast<uint8_t *>(ctx->in_pin) : nullptr;
    // large calls: start / end / kind cross PCIe block-compressed (transfer.cu), encoded by
    // host threads while earlier chunks copy and decode; HETEFF_RAW_TRANSFER=1 copies raw
    const int64_t codec_min = getenv("HETEFF_CODEC_MIN") ? atoll(getenv("HETEFF_CODEC_MIN")) : ((int64_t)1 << 22);
    const bool codec = !gather && !(getenv("HETEFF_RAW_TRANSFER") && atoi(getenv("HETEFF_RAW_TRANSFER")))
                       && hn + dn >= codec_min && (hn == 0 || (trace->host.start && trace->host.end && trace->host.kind))
                       && (dn == 0 || (trace->dev.start && trace->dev.end && trace->dev.kind));
    heteff_trace d = *trace;
    size_t o = 0;
    auto put = [&](const void *src, size_t bytes, size_t room) -> void * {
        void *dst = b + o;
        if (bytes && src) {
            if (gather) memcpy(hpin + o, src, bytes);
            else cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
        }
        o += room;
        return dst;
    };
    auto col = [&](const void *src, size_t bytes, size_t room) -> void * {   // the codec fills it
        return codec ? put(nullptr, bytes, room) : put(src, bytes, room);
    };
    d.host.start = static_cast<const uint64_t *>(col(trace->host.start, (size_t)hn * 8, hb8));
    d.host.end = static_cast<const uint64_t *>(col(trace->host.end, (size_t)hn * 8, hb8));
    d.host.res = static_cast<const int32_t *>(put(hseg ? nullptr : trace->host.res, (size_t)hn * 4, hseg ? 0 : hb4));
    d.host.kind = static_cast<const uint8_t *>(col(trace->host.kind, (size_t)hn, hb1));
    d.dev.start = static_cast<const uint64_t *>(col(trace->dev.start, (size_t)dn * 8, db8));
    d.dev.end = static_cast<const uint64_t *>(col(trace->dev.end, (size_t)dn * 8, db8));
    d.dev.res = static_cast<const int32_t *>(put(dseg ? nullptr : trace->dev.res, (size_t)dn * 4, dseg ? 0 : db4));
    d.dev.kind = static_cast<const uint8_t *>(col(trace->dev.kind, (size_t)dn, db1));
    if (codec) {
        hb::TransferSide sides[2] = {
            {trace->host.start, trace->host.end, trace->host.kind, hn, (uint64_t *)d.host.start, (uint64_t *)d.host.end,
             (uint8_t *)d.host.kind},
            {trace->dev.start, trace->dev.end, trace->dev.kind, dn, (uint64_t *)d.dev.start, (uint64_t *)d.dev.end,
             (uint8_t *)d.dev.kind}};
        // default: the host's hardware threads, shared by the ranks of this node when launched
        // one process per GPU (torchrun sets LOCAL_WORLD_SIZE), one left for the dispatcher
        int share = getenv("LOCAL_WORLD_SIZE") ? atoi(getenv("LOCAL_WORLD_SIZE")) : 1;
        share = share < 1 ? 1 : share;
        int nt = getenv("HETEFF_CODEC_THREADS") ? atoi(getenv("HETEFF_CODEC_THREADS"))
                                                 : (int)std::thread::hardware_concurrency() / share - 1;
        nt = nt < 1 ? 1 : (nt > 63 ? 63 : nt);
        std::string why;
        if (hb::transfer_columns(ctx->xfer, sides, 2, nt, s, why) != 0) return fail(ctx, HETEFF_CUDA_ERROR, "transfer: " + why);
    }
    d.host_decl = trace->host_decl
                      ? static_cast<const int32_t *>(put(trace->host_decl, (size_t)trace->host_ids * 4, hd))
                      : nullptr;
    d.dev_decl = trace->dev_decl
                     ? static_cast<const int32_t *>(put(trace->dev_decl, (size_t)trace->dev_ids * 4, dd))
                     : nullptr;
    const int64_t *hg = hseg ? static_cast<const int64_t *>(put(hseg, ((size_t)trace->host_ids + 1) * 8, hs8)) : nullptr;
    const int64_t *dg = dseg ? static_cast<const int64_t *>(put(dseg, ((size_t)trace->dev_ids + 1) * 8, ds8)) : nullptr;
    if (gather && o) CK(cudaMemcpyAsync(b, hpin, o, cudaMemcpyHostToDevice, s), "h2d");
    d.host_seg = hg;   // the kernel reads the offsets directly (no res column)
    d.dev_seg = dg;
    if (hg) d.host.res = nullptr;
    if (dg) d.dev.res = nullptr;
    CK(cudaGetLastError(), "h2d");
    return run_analysis(ctx, &d, opt, result, out, s);
}

int heteff_analyze_host(heteff_ctx *ctx, const heteff_trace *trace, const heteff_options *opt, heteff_result *result,
                        const heteff_outputs *out, void *stream)
{
    if (!trace) return fail(ctx, HETEFF_BAD_ARG, "null argument");
    if ((trace->host_seg && !seg_ok(trace->host_seg, trace->host_ids, trace->host.count)) ||
        (trace->dev_seg && !seg_ok(trace->dev_seg, trace->dev_ids, trace->dev.count)))
        return fail(ctx, HETEFF_BAD_ARG, "CSR offsets must start at 0, never decrease and end at the record count");
    return analyze_host_impl(ctx, trace, trace->host_seg, trace->dev_seg, opt, result, out, stream);
}

int heteff_analyze_host_csr(heteff_ctx *ctx, const heteff_trace *trace, const int64_t *host_seg,
                            const int64_t *dev_seg, const heteff_options *opt, heteff_result *result,
                            const heteff_outputs *out, void *stream)
{
    if (!trace) return fail(ctx, HETEFF_BAD_ARG, "null argument");
    if (!seg_ok(host_seg, trace->host_ids, trace->host.count) || !seg_ok(dev_seg, trace->dev_ids, trace->dev.count))
        return fail(ctx, HETEFF_BAD_ARG, "CSR offsets must start at 0, never decrease and end at the record count");
    return analyze_host_impl(ctx, trace, host_seg, dev_seg, opt, result, out, stream);
}

int heteff_overlap_covers(heteff_ctx *ctx, const heteff_trace *trace, int host_columns_on_host,
                          const int64_t *error_idx, int64_t count, int64_t *cover_idx, void *stream)
{
    if (!ctx || !trace || count < 0) return fail(ctx, HETEFF_BAD_ARG, "bad argument");
    if (count == 0) return HETEFF_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    const int64_t hn = trace->host.count;
    const size_t cols = host_columns_on_host ? (size_t)hn * 20 : 0;
    CK(ensure(ctx->stage, cols + (size_t)count * 16 + 1024, false), "alloc staging");
    uint8_t *b = static_cast<uint8_t *>(ctx->stage.p);
    hb::Params p;
    memset(&p, 0, sizeof(p));
    p.hn = hn;
    if (host_columns_on_host) {
        CK(cudaMemcpyAsync(b, trace->host.start, (size_t)hn * 8, cudaMemcpyHostToDevice, s), "h2d");
        CK(cudaMemcpyAsync(b + (size_t)hn * 8, trace->host.end, (size_t)hn * 8, cudaMemcpyHostToDevice, s), "h2d");
        CK(cudaMemcpyAsync(b + (size_t)hn * 16, trace->host.res, (size_t)hn * 4, cudaMemcpyHostToDevice, s), "h2d");
        p.hs = reinterpret_cast<const u64 *>(b);
        p.he = reinterpret_cast<const u64 *>(b + (size_t)hn * 8);
        p.hr = reinterpret_cast<const int32_t *>(b + (size_t)hn * 16);
    } else {
        p.hs = (const u64 *)trace->host.start; p.he = (const u64 *)trace->host.end; p.hr = trace->host.res;
    }
    size_t off = (cols + 255) & ~(size_t)255;
    int64_t *err_d = reinterpret_cast<int64_t *>(b + off);
    int64_t *cov_d = err_d + count;
    CK(cudaMemcpyAsync(err_d, error_idx, (size_t)count * 8, cudaMemcpyHostToDevice, s), "h2d");
    CK(hb::launch_covers(p, err_d, count, cov_d, s), "launch covers");
    CK(cudaMemcpyAsync(cover_idx, cov_d, (size_t)count * 8, cudaMemcpyDeviceToHost, s), "d2h");
    CK(cudaStreamSynchronize(s), "covers");
    return HETEFF_OK;
}

static int metrics_common(heteff_ctx *ctx, const uint64_t *summaries, int32_t k, uint64_t elapsed, int host_side,
                          double *metrics, uint32_t *mask, void *stream)
{
    if (!ctx || !metrics || !mask || (k > 0 && !summaries)) return fail(ctx, HETEFF_BAD_ARG, "null argument");
    if (k < 1) return fail(ctx, HETEFF_VALUE_ERROR,
                           host_side ? "host_metrics requires at least one rank"
                                     : "device_metrics requires at least one device");
    if (elapsed == 0) return fail(ctx, HETEFF_VALUE_ERROR, "elapsed must be positive, got 0");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    CK(ensure(ctx->stage, (size_t)k * 32, false), "alloc staging");
    CK(cudaMemcpyAsync(ctx->stage.p, summaries, (size_t)k * 32, cudaMemcpyHostToDevice, s), "h2d");
    CK(hb::launch_metrics(static_cast<const u64 *>(ctx->stage.p), k, elapsed, host_side, ctx->res_d, s),
       "launch metrics");
    CK(cudaMemcpyAsync(ctx->res_h, ctx->res_d, sizeof(hb::ResultDev), cudaMemcpyDeviceToHost, s), "d2h");
    CK(cudaStreamSynchronize(s), "metrics");
    if (host_side) {
        for (int i = 0; i < 5; ++i) metrics[i] = ctx->res_h->host_metrics[i];
        *mask = ctx->res_h->host_mask;
    } else {
        for (int i = 0; i < 4; ++i) metrics[i] = ctx->res_h->device_metrics[i];
        *mask = ctx->res_h->device_mask;
    }
    return HETEFF_OK;
}

int heteff_host_metrics(heteff_ctx *ctx, const uint64_t *summaries, int32_t n, uint64_t elapsed, double metrics[5],
                        uint32_t *mask, void *stream)
{
    return metrics_common(ctx, summaries, n, elapsed, 1, metrics, mask, stream);
}

int heteff_device_metrics(heteff_ctx *ctx, const uint64_t *summaries, int32_t m, uint64_t elapsed,
                          double metrics[4], uint32_t *mask, void *stream)
{
    return metrics_common(ctx, summaries, m, elapsed, 0, metrics, mask, stream);
}

// developer instrumentation (builds with -DHB_PROF): per-CTA clock64 phase counters
int heteff_prof_read(unsigned long long *out, int n) { return hb::prof_read(out, n); }

int heteff_generate(heteff_ctx *ctx, const heteff_gen_side *side, uint64_t *start, uint64_t *end, int32_t *res,
                    uint8_t *kind, void *stream)
{
    if (!ctx || !side) return fail(ctx, HETEFF_BAD_ARG, "null argument");
    if (side->n_res < 0 || side->per_res < 0 || side->dur_max < 1)
        return fail(ctx, HETEFF_BAD_ARG, "bad generator parameters");
    // the record count implied by per_res / extra_below must match
    long long lo = side->res_base, hi = (long long)side->res_base + side->n_res, ex = side->extra_below;
    long long extras = (hi < ex ? hi : ex) - (lo < ex ? lo : ex);
    if (extras < 0) extras = 0;
    if ((long long)side->per_res * side->n_res + extras != side->count)
        return fail(ctx, HETEFF_BAD_ARG, "count does not match per_res/extra_below");
    CK(cudaSetDevice(ctx->device), "cudaSetDevice");
    CK(hb::launch_generate(*side, (u64 *)start, (u64 *)end, res, kind, static_cast<cudaStream_t>(stream)), "launch generate");
    return HETEFF_OK;
}

}  // extern "C"
