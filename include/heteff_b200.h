/*
 * heteff_b200.h -- C ABI of the B200 engine for the heteff hot path
 *                  (state-interval trace -> host + device POP/TALP metric tree).
 *
 * The reference (`heteff`, pure Python) has no native FFI; its drop-in
 * surface is the Python API of pkg/src/heteff/__init__.py:3-51.  Each entry
 * point below is what a ctypes/cffi binding of that API binds, one per
 * reference stage function:
 *
 *   heteff_analyze(mode=REPORT)            <- compute_report   metrics.py:125-154
 *   heteff_analyze(mode=VALIDATE)          <- validate         model.py:160-230
 *   heteff_analyze(mode=SUMMARIZE_HOST)    <- summarize_host   summarize.py:57-92
 *   heteff_analyze(mode=SUMMARIZE_DEVICE)  <- summarize_device summarize.py:95-138
 *   heteff_host_metrics                    <- host_metrics     metrics.py:66-93
 *   heteff_device_metrics                  <- device_metrics   metrics.py:96-122
 *   heteff_analyze_host                    <- same, from HOST buffers (copies inside)
 *   heteff_generate                        <- (no reference counterpart) synthetic
 *                                             config-shaped traces written in HBM
 *
 * Conventions: plain pointers and sizes only, no torch types.  Record
 * columns are device pointers for heteff_analyze / heteff_generate and host
 * pointers for heteff_analyze_host.  All outputs (heteff_result and
 * heteff_outputs) are HOST memory; every call is stream-ordered on the
 * given stream and returns after the results are on the host.  A context
 * is not thread-safe; use one per thread / stream.  Status codes map 1:1
 * onto the reference's exceptions (see heteff_status).
 *
 * Packed SoA record layout (one set for host records, one for device):
 *   start u64[count], end u64[count]      half-open [start, end) ns (model.py:39-48)
 *   res   i32[count]                      dense resource id in [0, ids)
 *   kind  u8 [count]                      host: 0 useful 1 offload 2 mpi
 *                                         dev : 0 kernel 1 memory   (model.py:24-36)
 * (or, instead of res, CSR offsets per dense id: heteff_trace.host_seg /
 * dev_seg, 17 bytes per record).
 * Records must be grouped by res in ascending order and start-sorted
 * within a group -- the reference's canonical order (model.py:74-80,
 * 99-107) once dense ids follow the reference id order.  Violations are
 * detected per record and reported as HETEFF_CONTRACT (never silently
 * mis-summarized).  The stream column of the reference is never read
 * (summaries are stream-oblivious) and is not part of the ABI.
 */
#ifndef HETEFF_B200_H
#define HETEFF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HETEFF_ABI_VERSION 2

typedef enum {
    HETEFF_OK = 0,
    HETEFF_INVALID_TRACE = 1,   /* -> InvalidTraceError   (model.py:130-137)  */
    HETEFF_ANALYSIS_ERROR = 2,  /* -> AnalysisError       (metrics.py:136-137) */
    HETEFF_VALUE_ERROR = 3,     /* -> ValueError          (summarize.py:103-104, metrics.py:75-78) */
    HETEFF_CONTRACT = 4,        /* input not in canonical order / bad kind code */
    HETEFF_CUDA_ERROR = 5,
    HETEFF_NOMEM = 6,
    HETEFF_BAD_ARG = 7,
    HETEFF_PARSE_FALLBACK = 8   /* heteff_parse_trace: not decided by the fast path (see below) */
} heteff_status;

typedef enum {
    HETEFF_MODE_REPORT = 0,
    HETEFF_MODE_SUMMARIZE_DEVICE = 1,
    HETEFF_MODE_VALIDATE = 2,
    HETEFF_MODE_SUMMARIZE_HOST = 3
} heteff_mode;

/* index-list classes of heteff_result.counts / heteff_outputs.lists */
enum {
    HETEFF_HOST_MALFORMED = 0,  /* start > end                 model.py:152-153 */
    HETEFF_HOST_ZERO = 1,       /* zero-length (warning)       model.py:155-156 */
    HETEFF_HOST_UNDECLARED = 2, /* rank not declared           model.py:195-196 */
    HETEFF_HOST_OVERLAP = 3,    /* overlap with earlier record model.py:203-215 */
    HETEFF_DEV_MALFORMED = 4,
    HETEFF_DEV_ZERO = 5,
    HETEFF_DEV_UNDECLARED = 6,  /* device not declared         model.py:222-223 */
    HETEFF_DEV_LATE = 7,        /* ends after host elapsed     model.py:224-228 */
    HETEFF_NUM_LISTS = 8
};

/* contract_flags bits */
enum {
    HETEFF_CONTRACT_HOST_ORDER = 1,
    HETEFF_CONTRACT_DEV_ORDER = 2,
    HETEFF_CONTRACT_HOST_KIND = 4,
    HETEFF_CONTRACT_DEV_KIND = 8
};

typedef struct {
    const uint64_t *start;
    const uint64_t *end;
    const int32_t *res;
    const uint8_t *kind;
    int64_t count;
} heteff_records;

typedef struct {
    heteff_records host;
    heteff_records dev;
    int32_t host_ids;           /* size of the dense host id space */
    int32_t dev_ids;
    const int32_t *host_decl;   /* [host_ids] declaration position or -1; NULL = identity */
    const int32_t *dev_decl;    /* (same memory space as the record columns)             */
    int32_t n;                  /* number of distinct declared ranks   */
    int32_t m;                  /* number of distinct declared devices */
    uint64_t host_elapsed_floor;/* max end of host records kept out of the SoA (0 if none) */
    /* CSR alternative to the res columns (same memory space as the record columns):
       records [seg[r], seg[r+1]) have dense id r; seg[0] = 0, non-decreasing,
       seg[ids] = count (host_seg: host_ids + 1 entries, dev_seg: dev_ids + 1).
       When non-NULL the side's res column is not read (17 instead of 21 bytes per
       record stream through the analysis: start, end, kind). */
    const int64_t *host_seg;
    const int64_t *dev_seg;
} heteff_trace;

/* heteff_options.flags bits */
enum {
    /* records not in canonical order are sorted on the GPU (K3, heteff_sort_records)
       and the analysis re-run, instead of returning HETEFF_CONTRACT; list indices
       still refer to the caller's input positions */
    HETEFF_FLAG_SORT_IF_NEEDED = 1,
    /* SUMMARIZE_DEVICE: heteff_options.elapsed holds the DEVICE address of the u64
       window (read by the kernel; e.g. an all-reduced E that never visits the host) */
    HETEFF_FLAG_ELAPSED_DEVICE_PTR = 2
};

typedef struct {
    int32_t mode;               /* heteff_mode */
    int32_t flags;              /* HETEFF_FLAG_* */
    uint64_t elapsed;           /* SUMMARIZE_DEVICE: the explicit elapsed window */
    int64_t list_capacity;      /* capacity of each heteff_outputs list (0 = counts only) */
} heteff_options;

typedef struct {
    int32_t status;             /* heteff_status */
    int32_t contract_flags;
    int64_t contract_index;     /* first offending record (min over violations) */
    uint64_t host_elapsed;      /* max end over all host records (model.py:217) */
    uint64_t elapsed;           /* E (summarize.py:88-91) or the explicit window */
    uint64_t dev_max_end;       /* device-only traces (n == 0): max end over all device records (= E); else 0 */
    int32_t host_present;       /* n >= 1 */
    int32_t device_present;     /* m >= 1 */
    double host_metrics[5];     /* PE, MPI PE, MPI CE, MPI LB, device offload eff. */
    uint32_t host_mask;         /* bit i set: host_metrics[i] defined (else None) */
    uint32_t device_mask;
    double device_metrics[4];   /* PE, LB, CE, orchestration eff. */
    int64_t counts[HETEFF_NUM_LISTS];
    double kernel_ms;           /* device time of the analysis kernel (CUDA events) */
} heteff_result;

typedef struct {
    uint64_t *host_summaries;   /* [n][4] useful, offload, mpi, span_end (declaration order) */
    uint64_t *device_summaries; /* [m][4] kernel, memory, idle, clamped  (declaration order) */
    int64_t *lists[HETEFF_NUM_LISTS]; /* record indices, unordered, list_capacity each */
} heteff_outputs;

typedef struct heteff_ctx heteff_ctx;

int heteff_abi_version(void);
heteff_ctx *heteff_create(int device);
void heteff_destroy(heteff_ctx *ctx);
const char *heteff_last_error(const heteff_ctx *ctx);

/* Tuning / test knob: CTAs of the persistent analysis launch (0 = one per SM x
   resident CTAs, the default).  Any positive value is correct -- the kernel makes
   progress without co-residency; a grid larger than one wave only runs slower.
   The environment variable HETEFF_GRID sets the same at heteff_create. */
int heteff_set_grid(heteff_ctx *ctx, int grid);

/* The tile geometry of the analysis kernel compilation the context's last analysis used
   ("15x11" for CSR inputs; "11x15" or "8x19" for res columns, by device run length;
   "split: host <g>, device <g>" when a large REPORT call ran its two sides as two launches --
   DESIGN.md section 5), or "" before the first one.  Valid until the next call.
   Environment: HETEFF_NO_SPLIT=1 never splits; HETEFF_FORCE_SPLIT=1 splits every eligible
   REPORT call (tests). */
const char *heteff_kernel_name(const heteff_ctx *ctx);

/* trace columns in device memory */
int heteff_analyze(heteff_ctx *ctx, const heteff_trace *trace, const heteff_options *opt,
                   heteff_result *result, const heteff_outputs *out, void *stream);

/* trace columns in host memory (pinned for full PCIe rate); H2D inside.  Calls of
   >= 4 Mi records send start / end / kind block-compressed (csrc/transfer.cu: per block of
   4096 records the starts as gaps (sorted blocks) or offsets from the block's min start,
   and the durations, in 1, 2 or 4 bytes, raw 8-byte values where they do not fit), encoded
   by host threads while earlier chunks copy and decode on the GPU -- bit-exact columns in
   HBM, ~4x fewer PCIe bytes on dense traces.  Environment: HETEFF_RAW_TRANSFER=1 copies raw, HETEFF_CODEC_THREADS sets
   the encoder threads (default: hardware threads / LOCAL_WORLD_SIZE - 1), HETEFF_CODEC_MIN
   the size threshold. */
int heteff_analyze_host(heteff_ctx *ctx, const heteff_trace *trace, const heteff_options *opt,
                        heteff_result *result, const heteff_outputs *out, void *stream);

/* heteff_analyze_host with the res columns given as CSR offsets (HOST memory) instead:
   records [seg[r], seg[r+1]) have dense id r (seg[0] = 0, non-decreasing, seg[ids] =
   count; host_seg has host_ids + 1 entries, dev_seg dev_ids + 1).  trace->host.res /
   trace->dev.res are ignored; the offsets travel with the columns and the kernel reads
   them directly, so 4 bytes per record less cross PCIe and stream through HBM
   ("SoA arrays plus CSR offsets").
   Replaces the same reference entry points as heteff_analyze (compute_report,
   metrics.py:125-154, and the stage functions). */
int heteff_analyze_host_csr(heteff_ctx *ctx, const heteff_trace *trace, const int64_t *host_seg,
                            const int64_t *dev_seg, const heteff_options *opt, heteff_result *result,
                            const heteff_outputs *out, void *stream);

/* K3: stable GPU radix sort of one record set (device memory) into the canonical
 * order the analysis expects -- grouped by res ascending, start ascending within
 * a resource, ties kept in input order.  Replaces the canonical sort of
 * Trace.__post_init__ (model.py:74-80, 99-107) for columns that arrive unsorted
 * (e.g. per-stream device activity concatenated).  `out` columns must not alias
 * `in`; perm (optional, device memory, int64[count]) receives the input position
 * of every output record. */
typedef struct {
    uint64_t *start;
    uint64_t *end;
    int32_t *res;
    uint8_t *kind;
} heteff_columns;

typedef struct {
    int32_t key_bits;           /* bits of the compressed (res, start) key */
    int32_t passes;             /* onesweep digit passes */
    int32_t wide;               /* 1: key did not fit 64 bits (two stable stages) */
    int32_t start_sorted;       /* 1: input was start-ordered: sorted by res alone */
    double ms;                  /* device time of the sort (CUDA events) */
} heteff_sort_info;

int heteff_sort_records(heteff_ctx *ctx, const heteff_records *in, const heteff_columns *out, int64_t *perm,
                        heteff_sort_info *info, void *stream);

/* ---- interval algebra (intervals.py:40-105) over device arrays of [start, end) ----
 * flatten   <- flatten (intervals.py:40-61): HETEFF_VALUE_ERROR with *malformed_index
 *              = first input index with start > end ("malformed interval at index i");
 *              out capacity n.
 * subtract  <- subtract (intervals.py:64-81): a, b flat sets (sorted, disjoint,
 *              non-adjacent, no empties); out capacity na + nb.
 * intersect <- intersect (intervals.py:98-105): clip to [lo, hi); out capacity n.
 * total     <- total_duration (intervals.py:93-95): exact u128 sum, out[0] low
 *              word, out[1] high word (host memory).
 * complement (intervals.py:84-90) is subtract([bounds], a), as in the reference. */
int heteff_flatten(heteff_ctx *ctx, const uint64_t *start, const uint64_t *end, int64_t n, uint64_t *out_start,
                   uint64_t *out_end, int64_t *out_n, int64_t *malformed_index, void *stream);
int heteff_subtract(heteff_ctx *ctx, const uint64_t *a_start, const uint64_t *a_end, int64_t na,
                    const uint64_t *b_start, const uint64_t *b_end, int64_t nb, uint64_t *out_start,
                    uint64_t *out_end, int64_t *out_n, void *stream);
int heteff_intersect(heteff_ctx *ctx, const uint64_t *start, const uint64_t *end, int64_t n, uint64_t lo,
                     uint64_t hi, uint64_t *out_start, uint64_t *out_end, int64_t *out_n, void *stream);
int heteff_total_duration(heteff_ctx *ctx, const uint64_t *start, const uint64_t *end, int64_t n, uint64_t out[2],
                          void *stream);

/* ---- native trace documents (docs/formats.md:9-85) -> record columns ----
 * heteff_parse_trace <- read_trace (trace_io.py:96-158).  Host memory only; a
 * string-aware skip scan finds every hosts[] / devices[] entry, then the
 * entries are parsed in parallel (nthreads, 0 = all cores).  Records come out in
 * FILE order with the document's own rank / device ids.  Documents the fast path
 * cannot decide exactly (schema errors, integers beyond u64, duplicate keys,
 * non-integer numbers, escaped keys) return HETEFF_PARSE_FALLBACK with the byte
 * offset; the caller re-parses them with a strict reader for the reference's
 * exact TraceFormatError text. */
typedef struct heteff_parsed heteff_parsed;

typedef struct {
    int64_t n_hosts, n_devices, n_host_records, n_dev_records;
    const uint64_t *host_rank;  /* [n_hosts] */
    const int64_t *host_off;    /* [n_hosts + 1] record offsets per host entry */
    const uint64_t *dev_id;     /* [n_devices] */
    const int64_t *dev_owner;   /* [n_devices] owner_rank, -1 when absent / null */
    const int64_t *dev_off;     /* [n_devices + 1] */
    const uint8_t *h_kind;      /* 0 useful 1 offload 2 mpi */
    const uint64_t *h_start, *h_end;
    const uint8_t *d_kind;      /* 0 kernel 1 memory */
    const int64_t *d_stream;    /* -1 when absent / null */
    const uint64_t *d_start, *d_end;
} heteff_parsed_view;

int heteff_parse_trace(const char *data, size_t len, int nthreads, heteff_parsed **out, int64_t *fail_offset);
void heteff_parsed_info(const heteff_parsed *parsed, heteff_parsed_view *view);
void heteff_parsed_free(heteff_parsed *parsed);

/* ---- Chrome-trace-event documents + mapping rules -> records ----
 * heteff_import_events <- import_mapped (trace_io.py:263-342, docs/formats.md:87-132).
 * Only complete-span ("ph": "X") events count; microseconds become nanoseconds
 * exactly (x 1000; integer-valued floats accepted, fractional ones are the
 * reference's error); the first matching rule wins.  Matched events come out in
 * event order; unmapped "X" events are listed (index + name bytes) for the
 * caller's warnings / MappingError.  Anything the fast path cannot decide
 * exactly (an error the reference would raise, escaped strings, duplicate
 * keys) returns HETEFF_PARSE_FALLBACK. */
typedef struct {
    int32_t field;              /* 0 name, 1 category */
    int32_t mode;               /* 0 contains, 1 equals */
    const char *pattern;        /* UTF-8 bytes */
    int64_t pattern_len;
    int32_t target;             /* 0 useful 1 offload 2 mpi 3 kernel 4 memory */
    int32_t reserved;
    int64_t resource;           /* >= 0 fixed id, -1 "pid", -2 "tid" */
} heteff_rule;

typedef struct heteff_imported heteff_imported;

typedef struct {
    int64_t n_records, n_unmapped;
    const uint8_t *is_dev;      /* 1: device record */
    const uint8_t *kind;        /* host: 0 useful 1 offload 2 mpi; device: 0 kernel 1 memory */
    const uint64_t *res, *start, *end;
    const int64_t *unmapped;    /* event indices */
    const int64_t *name_off;    /* byte offset / length of each unmapped event's name */
    const int64_t *name_len;
} heteff_imported_view;

int heteff_import_events(const char *data, size_t len, const heteff_rule *rules, int nrules, int nthreads,
                         heteff_imported **out, int64_t *fail_offset);
void heteff_imported_info(const heteff_imported *imported, heteff_imported_view *view);
void heteff_imported_free(heteff_imported *imported);

/* ---- EXTENSIONS (not in the reference) ----
 * Monitoring regions (K5) and offload-wait / device-busy overlap (K6).
 * Region j is a window [start_j, end_j).  Its report is compute_report
 * (metrics.py:125-154) of the trace whose records are intersected with the
 * window (intervals.py:98-105 semantics) and shifted by -start_j, zero-length
 * records kept iff start_j <= s < end_j.  offload_busy[j][g] is
 * |offload(owner(g)) ∩ busy(g) ∩ [start_j, start_j + E_j)| where busy(g) is
 * the union of the device's kernel and memory records; the fraction is
 * sum_g offload_busy / sum_g d_offload(owner(g)).  The trace must be valid and
 * canonical: the call runs the full analysis first and returns its status
 * (INVALID_TRACE / CONTRACT) without computing regions otherwise.  All
 * windows are evaluated in one pass over the records per 16 windows. */
#define HETEFF_REGIONS_PER_RANK 1   /* heteff_regions.flags */

/* Per-rank regions (HETEFF_REGIONS_PER_RANK; TALP annotates regions per process,
 * PAPER.md:113): region j has one window per rank, start / end are [count][host_ids]
 * (window of dense host id h in region j at [j * host_ids + h]).  A rank's records are
 * clipped to its own window and shifted by its own start; a device's records to its
 * owner rank's window (dev_owner), a device without an owner records nothing in the
 * region.  E_j = the longest rank's region (max span, summarize.py:88-89), and every
 * device clamps at its owner's start + E_j. */
typedef struct {
    const uint64_t *start;      /* [count] window starts (host memory); per-rank: [count][host_ids] */
    const uint64_t *end;        /* [count] window ends (exclusive; end <= start = empty window); per-rank: [count][host_ids] */
    int32_t count;
    int32_t flags;              /* 0 (one window per region) or HETEFF_REGIONS_PER_RANK */
    const int32_t *dev_owner;   /* [dev_ids] dense host id owning each device, -1 none (host memory; NULL = none) */
} heteff_regions;

typedef struct {
    int32_t status;             /* HETEFF_OK, or HETEFF_ANALYSIS_ERROR: the region records no activity */
    int32_t reserved;
    uint64_t elapsed;           /* E of the region trace */
    double host_metrics[5];
    uint32_t host_mask;
    uint32_t device_mask;
    double device_metrics[4];
    double offload_busy_fraction;
    uint32_t offload_busy_defined;
    uint32_t reserved2;
} heteff_region_result;

typedef struct {
    heteff_region_result *results;  /* [count] (host memory) */
    uint64_t *host_summaries;       /* [count][n][4] useful, offload, mpi, span_end, or NULL */
    uint64_t *device_summaries;     /* [count][m][4] kernel, memory, idle, clamped, or NULL */
    uint64_t *offload_busy;         /* [count][m], or NULL */
    double kernel_ms;               /* device time of the region passes (out) */
} heteff_region_outputs;

/* trace columns in device memory */
int heteff_analyze_regions(heteff_ctx *ctx, const heteff_trace *trace, const heteff_regions *regions,
                           heteff_region_outputs *out, void *stream);

/* ---- multi-GPU (one process per GPU, rank-sharded trace) ----
 * Per step every rank runs, all stream-ordered and without host syncs:
 *   1. heteff_analyze_into(SUMMARIZE_HOST) on its host records -> block host header
 *      (local E = host_elapsed at byte 16) + host rows;
 *   2. all-reduce MAX of the local E over NVLink (8 bytes);
 *   3. heteff_analyze_into(SUMMARIZE_DEVICE, HETEFF_FLAG_ELAPSED_DEVICE_PTR -> the
 *      all-reduced E) on its device records -> block device header + device rows,
 *      clamped at the GLOBAL E (summarize.py:88-89, :113);
 *   4. all-gather of the fixed-size blocks; 5. heteff_merge_shards: one kernel launch
 *      (up to 148 CTAs; the last to finish reduces) -- concatenated summaries + both
 *      metric trees, one small D2H.
 * Block: [host header 256 B | device header 256 B | host rows [n_max][4] |
 * device rows [m_max][4]], block_bytes >= 512 + 32 (n_max + m_max).  Every record
 * is read once, as in the single-GPU launch.  heteff_merge_shards returns
 * HETEFF_PARSE_FALLBACK ("defer") when a shard's status is not OK (the caller then
 * takes the synchronous path for the exact error). */
int heteff_analyze_into(heteff_ctx *ctx, const heteff_trace *trace, const heteff_options *opt, void *dev_block,
                        size_t block_bytes, int32_t n_max, int32_t m_max, void *stream);
int heteff_merge_shards(heteff_ctx *ctx, const void *gathered, int32_t world, size_t block_bytes, int32_t n_max,
                        int32_t m_max, const int32_t *n_of, const int32_t *m_of, const uint64_t *elapsed_dev,
                        heteff_result *result, const heteff_outputs *out, void *stream);

/* overlap errors: cover index of each listed record (model.py:208-215), host memory */
int heteff_overlap_covers(heteff_ctx *ctx, const heteff_trace *trace, int host_columns_on_host,
                          const int64_t *error_idx, int64_t count, int64_t *cover_idx, void *stream);

/* metric trees from summaries (host memory [k][4] as laid out in heteff_outputs) */
int heteff_host_metrics(heteff_ctx *ctx, const uint64_t *summaries, int32_t n, uint64_t elapsed,
                        double metrics[5], uint32_t *mask, void *stream);
int heteff_device_metrics(heteff_ctx *ctx, const uint64_t *summaries, int32_t m, uint64_t elapsed,
                          double metrics[4], uint32_t *mask, void *stream);

/* ---- synthetic config-shaped traces (counter-based RNG, bit-identical to oracle/gen.py) ---- */
typedef struct {
    uint64_t seed;
    int32_t n_res;              /* resources generated by this call (local ids 0..n_res-1) */
    int32_t res_base;           /* global id of local resource 0 (rank sharding); RNG keys use global ids */
    int64_t per_res;            /* records per resource ...                                   */
    int32_t extra_below;        /* ... plus one for global ids < extra_below                  */
    int32_t serialized;         /* 1: start_j = sum(gap+dur) like a host chain, 0: arrival process */
    int64_t count;              /* total records of this call (must match per_res/extra_below) */
    uint32_t gap_max;           /* gap / inter-arrival ~ U[0, gap_max] */
    uint32_t dur_max;           /* duration ~ U[1, dur_max] */
    uint32_t dur_scale0;        /* duration multiplier for resource 0 (imbalance), >= 1 */
    uint32_t kernel_pct;        /* device side: P(kind == kernel) in percent */
    int32_t is_host;            /* 1: kind = state U{0,1,2}; 0: kind per kernel_pct */
    int32_t reserved;
} heteff_gen_side;

/* developer instrumentation: per-CTA clock64 phase counters of the last analysis
 * (only in builds with -DHB_PROF; returns the number of counters copied, 0 otherwise) */
int heteff_prof_read(unsigned long long *out, int n);

int heteff_generate(heteff_ctx *ctx, const heteff_gen_side *side, uint64_t *start, uint64_t *end,
                    int32_t *res, uint8_t *kind, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HETEFF_B200_H */
