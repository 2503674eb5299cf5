/*
 * talp_oracle.c -- CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference `heteff` hot path
 *   compute_report  (pkg/src/heteff/metrics.py:125-154)
 * over the same packed SoA the B200 engine consumes.  It exists so that
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg can check and time the CUDA engine.  The product package
 * (paper_2603_26576_b200/) never links, imports or executes this file.
 *
 * It follows the reference ALGORITHM literally -- canonical sort, then
 * flatten (sort + merge) / intersect / subtract / complement per device --
 * and deliberately does NOT use the running-max scan identity the GPU uses,
 * so agreement between the two is evidence, not tautology.
 *
 * Parity is pinned against the reference itself: the fixtures in tests/golden are
 * produced by importing /root/reference/pkg/src/heteff here
 * (tests/golden/make_golden.py) and tests/test_oracle_golden.py checks this
 * file against every vector.  Parallelism: a small pthread pool over
 * resources (no OpenMP runtime in this image).
 *
 * Record layout (shared with the engine, see include/heteff_b200.h):
 *   start u64[], end u64[], res i32[] (dense resource id), kind u8[]
 *   host kind: 0 useful, 1 offload, 2 mpi   (model.py:24-29)
 *   dev  kind: 0 kernel, 1 memory           (model.py:32-36)
 * Dense resource ids are assigned in ascending order of the reference's
 * rank/device id, so sorting by dense id == sorting by the reference id.
 * decl[id] = declaration position of that id, or -1 when undeclared.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>

typedef unsigned __int128 u128;

/* ------------------------------------------------------------------ */
/* minimal dynamic parallel-for over [0, n) with nthreads pthreads      */
/* ------------------------------------------------------------------ */
typedef void (*par_body)(void *arg, int64_t i, int tid);
typedef struct { par_body body; void *arg; int64_t n; atomic_llong next; int tid; } par_job;
typedef struct { par_job *job; int tid; } par_worker;

static void *par_run(void *p)
{
    par_worker *w = (par_worker *)p;
    for (;;) {
        int64_t i = atomic_fetch_add(&w->job->next, 1);
        if (i >= w->job->n) break;
        w->job->body(w->job->arg, i, w->tid);
    }
    return NULL;
}

static void par_for(int64_t n, int nthreads, par_body body, void *arg)
{
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if ((int64_t)nthreads > n) nthreads = n > 0 ? (int)n : 1;
    par_job job; job.body = body; job.arg = arg; job.n = n; atomic_init(&job.next, 0); job.tid = 0;
    pthread_t th[256]; par_worker w[256];
    for (int t = 0; t < nthreads; ++t) { w[t].job = &job; w[t].tid = t; }
    for (int t = 1; t < nthreads; ++t) pthread_create(&th[t], NULL, par_run, &w[t]);
    par_run(&w[0]);
    for (int t = 1; t < nthreads; ++t) pthread_join(th[t], NULL);
}

enum {
    ORC_OK = 0,
    ORC_INVALID = 1,      /* InvalidTraceError (validation errors present) */
    ORC_ANALYSIS = 2,     /* AnalysisError: elapsed == 0 (metrics.py:136-137) */
    ORC_VALUE = 3,        /* ValueError: elapsed <= 0 (summarize.py:103-104) */
    ORC_NOMEM = 6
};

enum { MODE_REPORT = 0, MODE_SUMMARIZE_DEVICE = 1, MODE_VALIDATE = 2, MODE_SUMMARIZE_HOST = 3 };

typedef struct {
    const uint64_t *h_start, *h_end; const int32_t *h_res; const uint8_t *h_kind; int64_t h_count;
    const uint64_t *d_start, *d_end; const int32_t *d_res; const uint8_t *d_kind; int64_t d_count;
    int32_t h_ids; const int32_t *h_decl; int32_t n;
    int32_t d_ids; const int32_t *d_decl; int32_t m;
    int32_t mode;
    uint64_t elapsed_arg;
    int32_t nthreads;
    int64_t cap;                 /* capacity of each index list below (0 = counts only) */
    uint64_t host_elapsed_floor; /* max end of host records the packer kept out of the SoA */
} orc_in;

typedef struct {
    int32_t status;
    int32_t host_defined, dev_defined;   /* host/device tree present (n>=1 / m>=1) */
    uint64_t host_elapsed;               /* max end over all host records (model.py:217) */
    uint64_t elapsed;                    /* E (summarize.py:88-91) */
    /* summaries in declaration order (caller-allocated, may be NULL) */
    uint64_t *host_sum;                  /* [n][4]: useful, offload, mpi, span_end */
    uint64_t *dev_sum;                   /* [m][4]: kernel, memory, idle, clamped */
    /* metrics (metrics.py:66-122); mask bit i => value i defined */
    double host_m[5]; uint32_t host_mask;
    double dev_m[4];  uint32_t dev_mask;
    /* validation counts */
    int64_t n_host_malformed, n_host_zero, n_host_undecl, n_overlap;
    int64_t n_dev_malformed, n_dev_zero, n_dev_undecl, n_dev_late;
    /* index lists in reference message order (caller-allocated, capacity cap) */
    int64_t *host_malformed, *host_zero, *host_undecl, *overlap /* [2*cap]: cover,i */;
    int64_t *dev_malformed, *dev_zero, *dev_undecl, *dev_late;
} orc_out;

/* ------------------------------------------------------------------ */
/* exact u128/u128 -> nearest double, ties to even (Python int/int)   */
/* ------------------------------------------------------------------ */
static int bitlen128(u128 x) { int n = 0; while (x) { x >>= 1; ++n; } return n; }

double orc_div_exact(u128 a, u128 b)
{
    if (a == 0) return 0.0;
    u128 q = a / b, r = a % b;
    int e2 = 0, sticky = 0;
    u128 M = q;
    int lq = bitlen128(q);
    if (lq > 55) {
        int s = lq - 55;
        u128 mask = (((u128)1) << s) - 1;
        if ((q & mask) != 0) sticky = 1;
        M = q >> s; e2 = s;
        if (r != 0) sticky = 1;
    } else {
        while (bitlen128(M) < 55) {
            r <<= 1;
            M <<= 1;
            if (r >= b) { M |= 1; r -= b; }
            e2 -= 1;
        }
        if (r != 0) sticky = 1;
    }
    /* M has exactly 55 significant bits: keep 53, guard bit, one more bit */
    unsigned low2 = (unsigned)(M & 3);
    uint64_t mant = (uint64_t)(M >> 2);
    e2 += 2;
    int guard = (low2 >> 1) & 1, rest = (low2 & 1) | sticky;
    if (guard && (rest || (mant & 1))) mant += 1;
    if (mant == (1ULL << 53)) { mant >>= 1; e2 += 1; }
    return ldexp((double)mant, e2);
}

/* ------------------------------------------------------------------ */
/* interval algebra restated from intervals.py:40-105                 */
/* ------------------------------------------------------------------ */
typedef struct { uint64_t s, e; } iv_t;

static int iv_cmp(const void *a, const void *b)
{
    const iv_t *x = (const iv_t *)a, *y = (const iv_t *)b;
    if (x->s != y->s) return x->s < y->s ? -1 : 1;
    if (x->e != y->e) return x->e < y->e ? -1 : 1;
    return 0;
}

/* flatten: drop zero-length (intervals.py:52), sort (:53), merge overlap
 * and adjacency `start <= last.end` (:55-60).  In place; returns length. */
static int64_t iv_flatten(iv_t *v, int64_t k)
{
    int64_t w = 0;
    for (int64_t i = 0; i < k; ++i) if (v[i].e > v[i].s) v[w++] = v[i];
    k = w;
    int sorted = 1;
    for (int64_t i = 1; i < k && sorted; ++i) if (iv_cmp(&v[i - 1], &v[i]) > 0) sorted = 0;
    if (!sorted) qsort(v, (size_t)k, sizeof(iv_t), iv_cmp);
    int64_t out = 0;
    for (int64_t i = 0; i < k; ++i) {
        if (out > 0 && v[i].s <= v[out - 1].e) {
            if (v[i].e > v[out - 1].e) v[out - 1].e = v[i].e;
        } else {
            v[out++] = v[i];
        }
    }
    return out;
}

/* intersect with [lo,hi) (intervals.py:98-105); in place */
static int64_t iv_intersect(iv_t *v, int64_t k, uint64_t lo, uint64_t hi)
{
    int64_t out = 0;
    for (int64_t i = 0; i < k; ++i) {
        uint64_t s = v[i].s > lo ? v[i].s : lo, e = v[i].e < hi ? v[i].e : hi;
        if (s < e) { v[out].s = s; v[out].e = e; ++out; }
    }
    return out;
}

/* subtract(a, b) -> out (intervals.py:64-81); out may not alias b */
static int64_t iv_subtract(const iv_t *a, int64_t ka, const iv_t *b, int64_t kb, iv_t *out)
{
    int64_t w = 0, j = 0;
    for (int64_t i = 0; i < ka; ++i) {
        uint64_t cursor = a[i].s;
        while (j < kb && b[j].e <= cursor) ++j;
        int64_t k = j;
        while (k < kb && b[k].s < a[i].e) {
            if (b[k].s > cursor) { out[w].s = cursor; out[w].e = b[k].s; ++w; }
            if (b[k].e > cursor) cursor = b[k].e;
            ++k;
        }
        if (cursor < a[i].e) { out[w].s = cursor; out[w].e = a[i].e; ++w; }
    }
    return w;
}

static u128 iv_total(const iv_t *v, int64_t k)
{
    u128 t = 0;
    for (int64_t i = 0; i < k; ++i) t += v[i].e - v[i].s;
    return t;
}

/* ------------------------------------------------------------------ */
/* canonical order (model.py:74-80, 99-107)                           */
/* ------------------------------------------------------------------ */
typedef struct { uint64_t s, e; int32_t r; uint8_t k; } rec_t;

static const uint8_t HOST_KIND_RANK[3] = {2, 1, 0}; /* "mpi" < "offload" < "useful" */

static int host_key_cmp(const rec_t *x, const rec_t *y)
{
    if (x->r != y->r) return x->r < y->r ? -1 : 1;
    if (x->s != y->s) return x->s < y->s ? -1 : 1;
    if (x->e != y->e) return x->e < y->e ? -1 : 1;
    uint8_t a = x->k < 3 ? HOST_KIND_RANK[x->k] : x->k, b = y->k < 3 ? HOST_KIND_RANK[y->k] : y->k;
    return a < b ? -1 : (a > b);
}
static int host_qcmp(const void *a, const void *b) { return host_key_cmp((const rec_t *)a, (const rec_t *)b); }

static int dev_key_cmp(const rec_t *x, const rec_t *y)
{
    if (x->r != y->r) return x->r < y->r ? -1 : 1;
    if (x->s != y->s) return x->s < y->s ? -1 : 1;
    if (x->e != y->e) return x->e < y->e ? -1 : 1;
    return x->k < y->k ? -1 : (x->k > y->k);   /* "kernel" < "memory" */
}
static int dev_qcmp(const void *a, const void *b) { return dev_key_cmp((const rec_t *)a, (const rec_t *)b); }

typedef struct {
    const uint64_t *s, *e; const int32_t *r; const uint8_t *k; int64_t n;
    rec_t *own;   /* non-NULL when we had to sort a copy */
} view_t;

static inline rec_t view_get(const view_t *v, int64_t i)
{
    if (v->own) return v->own[i];
    rec_t x = { v->s[i], v->e[i], v->r[i], v->k[i] };
    return x;
}

static int make_view(view_t *v, const uint64_t *s, const uint64_t *e, const int32_t *r, const uint8_t *k,
                     int64_t n, int is_host)
{
    v->s = s; v->e = e; v->r = r; v->k = k; v->n = n; v->own = NULL;
    int sorted = 1;
    for (int64_t i = 1; i < n && sorted; ++i) {
        rec_t a = { s[i - 1], e[i - 1], r[i - 1], k[i - 1] }, b = { s[i], e[i], r[i], k[i] };
        int c = is_host ? host_key_cmp(&a, &b) : dev_key_cmp(&a, &b);
        if (c > 0) sorted = 0;
    }
    if (sorted) return 0;
    v->own = (rec_t *)malloc(sizeof(rec_t) * (size_t)n);
    if (!v->own) return -1;
    for (int64_t i = 0; i < n; ++i) { v->own[i].s = s[i]; v->own[i].e = e[i]; v->own[i].r = r[i]; v->own[i].k = k[i]; }
    qsort(v->own, (size_t)n, sizeof(rec_t), is_host ? host_qcmp : dev_qcmp);
    return 0;
}

/* segment offsets per dense id: off[id]..off[id+1] (records sorted by id) */
static int64_t *segment_offsets(const view_t *v, int32_t ids)
{
    int64_t *off = (int64_t *)calloc((size_t)ids + 1, sizeof(int64_t));
    if (!off) return NULL;
    for (int64_t i = 0; i < v->n; ++i) {
        int32_t r = v->own ? v->own[i].r : v->r[i];
        if (r >= 0 && r < ids) off[r + 1]++;
    }
    for (int32_t i = 0; i < ids; ++i) off[i + 1] += off[i];
    /* records with out-of-range ids sort before/after; shift by the count
       of negative ids so offsets index the sorted view */
    int64_t neg = 0;
    for (int64_t i = 0; i < v->n; ++i) { int32_t r = v->own ? v->own[i].r : v->r[i]; if (r < 0) neg++; }
    for (int32_t i = 0; i <= ids; ++i) off[i] += neg;
    return off;
}

static inline int declared(const int32_t *decl, int32_t ids, int32_t r)
{
    if (r < 0 || r >= ids) return 0;
    return decl ? decl[r] >= 0 : 1;
}

/* summarize_host body for one declared rank (summarize.py:74-86) */
typedef struct { const view_t *hv; const int64_t *hoff; const int32_t *id_of; uint64_t *out; uint64_t *span; } host_job;

static void host_body(void *arg, int64_t p, int tid)
{
    host_job *j = (host_job *)arg;
    int32_t id = j->id_of[p];
    uint64_t off_ = 0, mpi = 0, span = 0;
    if (id >= 0) {
        for (int64_t i = j->hoff[id]; i < j->hoff[id + 1]; ++i) {
            rec_t x = view_get(j->hv, i);
            if (x.k == 1) off_ += x.e - x.s;
            else if (x.k == 2) mpi += x.e - x.s;
            if (x.e > span) span = x.e;
        }
    }
    if (j->out) { uint64_t *h = j->out + 4 * p; h[0] = span - off_ - mpi; h[1] = off_; h[2] = mpi; h[3] = span; }
    j->span[p] = span;
}

/* summarize_device body for one declared device (summarize.py:107-132) */
typedef struct { const view_t *dv; const int64_t *doff; const int32_t *id_of; uint64_t *out; uint64_t E; atomic_int fail; } dev_job;

static void dev_body(void *arg, int64_t q, int tid)
{
    dev_job *j = (dev_job *)arg;
    const uint64_t E = j->E;
    int32_t id = j->id_of[q];
    int64_t lo = id >= 0 ? j->doff[id] : 0, hi = id >= 0 ? j->doff[id + 1] : 0, k = hi - lo;
    iv_t *K = (iv_t *)malloc(sizeof(iv_t) * (size_t)(k + 1));
    iv_t *M = (iv_t *)malloc(sizeof(iv_t) * (size_t)(k + 1));
    iv_t *T = (iv_t *)malloc(sizeof(iv_t) * (size_t)(2 * k + 2));
    iv_t *A = (iv_t *)malloc(sizeof(iv_t) * (size_t)(2 * k + 2));
    iv_t *I = (iv_t *)malloc(sizeof(iv_t) * (size_t)(2 * k + 3));
    if (!K || !M || !T || !A || !I) { atomic_store(&j->fail, 1); goto out; }
    int64_t nk = 0, nm = 0; uint64_t clamped = 0;
    for (int64_t i = lo; i < hi; ++i) {
        rec_t x = view_get(j->dv, i);
        if (x.e > E) clamped++;                                   /* :113-114 */
        if (x.k == 0) { K[nk].s = x.s; K[nk].e = x.e; nk++; }
        else { M[nm].s = x.s; M[nm].e = x.e; nm++; }
    }
    nk = iv_intersect(K, iv_flatten(K, nk), 0, E);               /* :121 */
    nm = iv_intersect(M, iv_flatten(M, nm), 0, E);
    int64_t nmem = iv_subtract(M, nm, K, nk, T);                  /* :122 */
    u128 dk = iv_total(K, nk), dm = iv_total(T, nmem);
    /* active = flatten(kernel ++ memory); idle = complement (:123-124) */
    memcpy(A, K, sizeof(iv_t) * (size_t)nk);
    memcpy(A + nk, T, sizeof(iv_t) * (size_t)nmem);
    int64_t na = iv_flatten(A, nk + nmem);
    iv_t bounds = { 0, E };
    int64_t ni = iv_subtract(&bounds, 1, A, na, I);
    u128 di = iv_total(I, ni);
    if (j->out) { uint64_t *d = j->out + 4 * q; d[0] = (uint64_t)dk; d[1] = (uint64_t)dm; d[2] = (uint64_t)di; d[3] = clamped; }
out:
    free(K); free(M); free(T); free(A); free(I);
}

#define PUSH(list, cnt, val) do { if (o->list && (cnt) < in->cap) o->list[(cnt)] = (val); (cnt)++; } while (0)

int orc_analyze(const orc_in *in, orc_out *o)
{
    int rc = ORC_OK;
    int32_t n = in->n, m = in->m;
    view_t hv, dv;
    if (make_view(&hv, in->h_start, in->h_end, in->h_res, in->h_kind, in->h_count, 1)) return ORC_NOMEM;
    if (make_view(&dv, in->d_start, in->d_end, in->d_res, in->d_kind, in->d_count, 0)) { free(hv.own); return ORC_NOMEM; }

    /* declaration position -> dense id */
    int32_t *h_id_of = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    int32_t *d_id_of = (int32_t *)malloc(sizeof(int32_t) * (size_t)(m > 0 ? m : 1));
    for (int32_t i = 0; i < n; ++i) h_id_of[i] = -1;
    for (int32_t i = 0; i < m; ++i) d_id_of[i] = -1;
    for (int32_t id = 0; id < in->h_ids; ++id) {
        int32_t p = in->h_decl ? in->h_decl[id] : id;
        if (p >= 0 && p < n) h_id_of[p] = id;
    }
    for (int32_t id = 0; id < in->d_ids; ++id) {
        int32_t p = in->d_decl ? in->d_decl[id] : id;
        if (p >= 0 && p < m) d_id_of[p] = id;
    }

    /* ---------------- validate (model.py:160-230) ---------------- */
    int64_t c_hmal = 0, c_hzero = 0, c_hund = 0, c_ovl = 0;
    int64_t c_dmal = 0, c_dzero = 0, c_dund = 0, c_dlate = 0;
    uint64_t host_elapsed = in->host_elapsed_floor;  /* model.py:217 */
    for (int64_t i = 0; i < hv.n; ++i) {             /* model.py:192-198 */
        rec_t x = view_get(&hv, i);
        if (x.s > x.e) PUSH(host_malformed, c_hmal, i);
        else if (x.s == x.e) PUSH(host_zero, c_hzero, i);
        if (!declared(in->h_decl, in->h_ids, x.r)) PUSH(host_undecl, c_hund, i);
        if (x.e > host_elapsed) host_elapsed = x.e;
    }
    int64_t *hoff = segment_offsets(&hv, in->h_ids);
    int64_t *doff = segment_offsets(&dv, in->d_ids);
    if (!hoff || !doff) { rc = ORC_NOMEM; goto done; }
    for (int32_t p = 0; p < n; ++p) {                /* model.py:203-215 */
        int32_t id = h_id_of[p];
        if (id < 0) continue;
        int have = 0; uint64_t cover_end = 0; int64_t cover_idx = -1;
        for (int64_t i = hoff[id]; i < hoff[id + 1]; ++i) {
            rec_t x = view_get(&hv, i);
            if (!(x.e > x.s)) continue;              /* usable: ok and duration > 0 */
            if (have && x.s < cover_end) {
                if (o->overlap && c_ovl < in->cap) { o->overlap[2 * c_ovl] = cover_idx; o->overlap[2 * c_ovl + 1] = i; }
                c_ovl++;
            }
            if (!have || x.e > cover_end) { cover_end = x.e; cover_idx = i; have = 1; }
        }
    }
    for (int64_t i = 0; i < dv.n; ++i) {             /* model.py:219-228 */
        rec_t x = view_get(&dv, i);
        if (x.s > x.e) PUSH(dev_malformed, c_dmal, i);
        else if (x.s == x.e) PUSH(dev_zero, c_dzero, i);
        if (!declared(in->d_decl, in->d_ids, x.r)) PUSH(dev_undecl, c_dund, i);
        if (n >= 1 && x.e > host_elapsed) PUSH(dev_late, c_dlate, i);
    }
    o->n_host_malformed = c_hmal; o->n_host_zero = c_hzero; o->n_host_undecl = c_hund; o->n_overlap = c_ovl;
    o->n_dev_malformed = c_dmal; o->n_dev_zero = c_dzero; o->n_dev_undecl = c_dund; o->n_dev_late = c_dlate;
    o->host_elapsed = host_elapsed;
    o->host_defined = n >= 1; o->dev_defined = m >= 1;
    o->host_mask = o->dev_mask = 0;
    o->elapsed = 0;
    int invalid = (n == 0 && m == 0) || c_hmal || c_hund || c_ovl || c_dmal || c_dund;
    if (in->mode == MODE_VALIDATE) { rc = invalid ? ORC_INVALID : ORC_OK; goto done; }
    if (in->mode == MODE_SUMMARIZE_DEVICE && in->elapsed_arg == 0) { rc = ORC_VALUE; goto done; }
    if (invalid) { rc = ORC_INVALID; goto done; }

    /* ---------------- summarize_host (summarize.py:57-92) -------- */
    uint64_t E = 0;
    {
        host_job hj = { &hv, hoff, h_id_of, o->host_sum, NULL };
        hj.span = (uint64_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(uint64_t));
        if (!hj.span) { rc = ORC_NOMEM; goto done; }
        par_for(n, in->nthreads, host_body, &hj);
        uint64_t emax = 0;
        for (int32_t p = 0; p < n; ++p) if (hj.span[p] > emax) emax = hj.span[p];
        free(hj.span);
        if (n >= 1) E = emax;
        else {
            for (int64_t i = 0; i < dv.n; ++i) { rec_t x = view_get(&dv, i); if (x.e > E) E = x.e; }
        }
    }
    if (in->mode == MODE_SUMMARIZE_HOST) { o->elapsed = E; rc = ORC_OK; goto done; }
    if (in->mode == MODE_SUMMARIZE_DEVICE) E = in->elapsed_arg;
    o->elapsed = E;
    if (E == 0) { rc = ORC_ANALYSIS; goto done; }

    /* ---------------- summarize_device (summarize.py:95-138) ----- */
    {
        dev_job dj = { &dv, doff, d_id_of, o->dev_sum, E, 0 };
        par_for(m, in->nthreads, dev_body, &dj);
        if (atomic_load(&dj.fail)) { rc = ORC_NOMEM; goto done; }
    }
    if (in->mode == MODE_SUMMARIZE_DEVICE) { rc = ORC_OK; goto done; }

    /* ---------------- host_metrics (metrics.py:66-93) ------------- */
    if (n >= 1 && o->host_sum) {
        u128 sum_u = 0, sum_uw = 0, max_uw = 0;
        for (int32_t p = 0; p < n; ++p) {
            u128 u = o->host_sum[4 * p], w = o->host_sum[4 * p + 1];
            sum_u += u; sum_uw += u + w; if (u + w > max_uw) max_uw = u + w;
        }
        u128 En = (u128)E * (u128)(uint32_t)n;
        if (sum_uw == 0) { o->host_m[0] = 0.0; o->host_mask = 1; }
        else {
            o->host_m[0] = orc_div_exact(sum_u, En);
            o->host_m[1] = orc_div_exact(sum_uw, En);
            o->host_m[2] = orc_div_exact(max_uw, E);
            o->host_m[3] = orc_div_exact(sum_uw, (u128)(uint32_t)n * max_uw);
            o->host_m[4] = orc_div_exact(sum_u, sum_uw);
            o->host_mask = 0x1f;
        }
    }
    /* ---------------- device_metrics (metrics.py:96-122) ---------- */
    if (m >= 1 && o->dev_sum) {
        u128 sum_k = 0, max_k = 0, max_km = 0;
        for (int32_t q = 0; q < m; ++q) {
            u128 kk = o->dev_sum[4 * q], mm = o->dev_sum[4 * q + 1];
            sum_k += kk; if (kk > max_k) max_k = kk; if (kk + mm > max_km) max_km = kk + mm;
        }
        o->dev_m[0] = orc_div_exact(sum_k, (u128)E * (u128)(uint32_t)m);
        if (max_k == 0) {
            o->dev_m[3] = max_km > 0 ? orc_div_exact(max_km, E) : 0.0;
            o->dev_mask = 0x9;
        } else {
            o->dev_m[1] = orc_div_exact(sum_k, (u128)(uint32_t)m * max_k);
            o->dev_m[2] = orc_div_exact(max_k, max_km);
            o->dev_m[3] = orc_div_exact(max_km, E);
            o->dev_mask = 0xf;
        }
    }

done:
    o->status = rc;
    free(hoff); free(doff); free(h_id_of); free(d_id_of); free(hv.own); free(dv.own);
    return rc;
}

/* exposed for tests: exact division on (hi,lo) 64-bit halves */
double orc_div_exact_u64x2(uint64_t a_hi, uint64_t a_lo, uint64_t b_hi, uint64_t b_lo)
{
    u128 a = ((u128)a_hi << 64) | a_lo, b = ((u128)b_hi << 64) | b_lo;
    return orc_div_exact(a, b);
}

size_t orc_in_size(void) { return sizeof(orc_in); }
size_t orc_out_size(void) { return sizeof(orc_out); }

/* ------------------------------------------------------------------ */
/* EXTENSIONS (not in the reference)      */
/*                                                                     */
/* Monitoring regions: region j is a window [a_j, b_j).  Its trace is   */
/* the full trace with every record intersected with the window         */
/* (intervals.py:98-105 semantics: empty results dropped) and shifted   */
/* by -a_j; a zero-length record is kept iff a_j <= s < b_j.  The       */
/* region's metric tree is compute_report (metrics.py:125-154) of that  */
/* trace -- restated here by literally building it and calling          */
/* orc_analyze.                                                         */
/*                                                                     */
/* Offload-wait / device-busy overlap, per device g with owner rank p:  */
/*   busy_g = |A_p  ∩  B_g|, A_p = flatten(offload records of p)        */
/*   ∩ [0,E), B_g = flatten(records of g) ∩ [0,E), computed as          */
/*   |A| - |subtract(A, B)| with the intervals.py:40-105 restatements;  */
/*   fraction = sum_g busy_g / sum_g d_offload(owner(g)).               */
/* ------------------------------------------------------------------ */
typedef struct {
    const uint64_t *win_start, *win_end;
    int32_t count;
    const int32_t *dev_owner;            /* [d_ids] dense host id owning the device, -1 none */
    /* per-rank regions (TALP regions are annotated per process): NULL, or
     * [count][h_ids][2] window of each rank -- then win_start / win_end are unused, a
     * rank's records are clipped to its own window, a device's records to its owner's
     * window, and the records of a device without an owner to the empty window */
    const uint64_t *host_win;
    /* sharded use (tests, oracle.regions_sharded): 0 compute_report per region; 1 the
     * host pass only (summarize_host per region: host rows + the block's E, devices
     * skipped); 2 the device pass with the GLOBAL E of each region, elapsed_in[j]
     * (summarize_device + overlap; metric trees left to the caller) */
    int32_t pass;
    const uint64_t *elapsed_in;
} orc_regions_in;

typedef struct {
    int32_t *status;                     /* [R] ORC_OK / ORC_ANALYSIS (E == 0) / ... */
    uint64_t *elapsed;                   /* [R] */
    uint64_t *host_sum;                  /* [R][n][4] */
    uint64_t *dev_sum;                   /* [R][m][4] */
    uint64_t *busy;                      /* [R][m] */
    double *host_m; uint32_t *host_mask; /* [R][5], [R] */
    double *dev_m; uint32_t *dev_mask;   /* [R][4], [R] */
    double *busy_frac; uint32_t *busy_mask; /* [R], [R] */
} orc_regions_out;

/* clip one record set to [a, b) (or, with `win`, record i to win[2 * rank_of(r[i])],
 * rank_of = identity for host records, the owner table for device records, an
 * empty window when rank_of < 0), shifted; returns the kept count */
static int64_t clip_records(const uint64_t *s, const uint64_t *e, const int32_t *r, const uint8_t *k, int64_t n,
                            uint64_t a0, uint64_t b0, const uint64_t *win, const int32_t *owner, int32_t h_ids,
                            uint64_t *os, uint64_t *oe, int32_t *orr, uint8_t *ok)
{
    int64_t w = 0;
    for (int64_t i = 0; i < n; ++i) {
        uint64_t a = a0, b = b0;
        if (win) {
            const int32_t q = owner ? (owner[r[i]]) : r[i];
            if (q < 0 || q >= h_ids) continue;
            a = win[2 * (size_t)q]; b = win[2 * (size_t)q + 1];
        }
        uint64_t cs, ce;
        if (s[i] == e[i]) {
            if (!(s[i] >= a && s[i] < b)) continue;
            cs = ce = s[i];
        } else {
            cs = s[i] > a ? s[i] : a;
            ce = e[i] < b ? e[i] : b;
            if (!(cs < ce)) continue;
        }
        os[w] = cs - a; oe[w] = ce - a; orr[w] = r[i]; ok[w] = k[i]; ++w;
    }
    return w;
}

/* records of dense id `id` in a canonical (res-grouped) set, optionally one kind, as intervals */
static int64_t gather_ivs(const uint64_t *s, const uint64_t *e, const int32_t *r, const uint8_t *k, int64_t n,
                          int32_t id, int kind, iv_t *out)
{
    int64_t w = 0;
    for (int64_t i = 0; i < n; ++i)
        if (r[i] == id && (kind < 0 || k[i] == kind)) { out[w].s = s[i]; out[w].e = e[i]; ++w; }
    return w;
}

int orc_regions(const orc_in *in, const orc_regions_in *rg, orc_regions_out *o)
{
    const int64_t hn = in->h_count, dn = in->d_count;
    const int32_t n = in->n, m = in->m;
    uint64_t *hs = malloc(8 * (size_t)(hn + 1)), *he = malloc(8 * (size_t)(hn + 1));
    int32_t *hr = malloc(4 * (size_t)(hn + 1)); uint8_t *hk = malloc((size_t)hn + 1);
    uint64_t *ds = malloc(8 * (size_t)(dn + 1)), *de = malloc(8 * (size_t)(dn + 1));
    int32_t *dr = malloc(4 * (size_t)(dn + 1)); uint8_t *dk = malloc((size_t)dn + 1);
    iv_t *A = malloc(sizeof(iv_t) * (size_t)(hn + 1)), *B = malloc(sizeof(iv_t) * (size_t)(dn + 1));
    iv_t *D = malloc(sizeof(iv_t) * (size_t)(hn + dn + 1));
    if (!hs || !he || !hr || !hk || !ds || !de || !dr || !dk || !A || !B || !D) return ORC_NOMEM;
    for (int32_t j = 0; j < rg->count; ++j) {
        const uint64_t *win = rg->host_win ? rg->host_win + (size_t)j * (size_t)in->h_ids * 2 : NULL;
        const uint64_t a = win ? 0 : rg->win_start[j], b = win ? 0 : rg->win_end[j];
        static const int32_t no_owner = -1;
        const int64_t kh = clip_records(in->h_start, in->h_end, in->h_res, in->h_kind, hn, a, b, win, NULL, in->h_ids,
                                        hs, he, hr, hk);
        /* device ids index the owner table (all -1 without one) */
        int32_t *own = NULL;
        if (win) {
            own = malloc(4 * (size_t)(in->d_ids > 0 ? in->d_ids : 1));
            for (int32_t q = 0; q < in->d_ids; ++q) own[q] = rg->dev_owner ? rg->dev_owner[q] : no_owner;
        }
        const int64_t kd = rg->pass == 1 ? 0 : clip_records(in->d_start, in->d_end, in->d_res, in->d_kind, dn, a, b,
                                                            win, own, in->h_ids, ds, de, dr, dk);
        free(own);
        orc_in ri = *in;
        ri.h_start = hs; ri.h_end = he; ri.h_res = hr; ri.h_kind = hk; ri.h_count = kh;
        ri.d_start = ds; ri.d_end = de; ri.d_res = dr; ri.d_kind = dk; ri.d_count = kd;
        ri.mode = rg->pass == 1 ? MODE_SUMMARIZE_HOST : rg->pass == 2 ? MODE_SUMMARIZE_DEVICE : MODE_REPORT;
        ri.elapsed_arg = rg->pass == 2 ? rg->elapsed_in[j] : 0;
        ri.cap = 0; ri.host_elapsed_floor = 0;
        orc_out ro; memset(&ro, 0, sizeof(ro));
        ro.host_sum = o->host_sum + (size_t)j * (size_t)(n > 0 ? n : 1) * 4;
        ro.dev_sum = o->dev_sum + (size_t)j * (size_t)(m > 0 ? m : 1) * 4;
        o->status[j] = rg->pass == 2 && ri.elapsed_arg == 0 ? ORC_ANALYSIS : orc_analyze(&ri, &ro);
        o->elapsed[j] = rg->pass == 2 ? ri.elapsed_arg : ro.elapsed;
        for (int q = 0; q < 5; ++q) o->host_m[5 * j + q] = ro.host_m[q];
        for (int q = 0; q < 4; ++q) o->dev_m[4 * j + q] = ro.dev_m[q];
        o->host_mask[j] = ro.host_mask; o->dev_mask[j] = ro.dev_mask;
        o->busy_mask[j] = 0; o->busy_frac[j] = 0.0;
        uint64_t *busy = o->busy + (size_t)j * (size_t)(m > 0 ? m : 1);
        for (int32_t q = 0; q < m; ++q) busy[q] = 0;
        if (o->status[j] != ORC_OK || rg->pass == 1) continue;
        const uint64_t E = o->elapsed[j];
        u128 num = 0, den = 0;
        for (int32_t did = 0; did < in->d_ids; ++did) {
            const int32_t q = in->d_decl ? in->d_decl[did] : did;     /* declaration position */
            if (q < 0 || q >= m) continue;
            const int32_t hid = rg->dev_owner ? rg->dev_owner[did] : -1;
            if (hid < 0 || hid >= in->h_ids) continue;
            const int32_t p = in->h_decl ? in->h_decl[hid] : hid;
            if (p < 0 || p >= n) continue;
            int64_t ka = gather_ivs(hs, he, hr, hk, kh, hid, 1, A);
            ka = iv_flatten(A, ka); ka = iv_intersect(A, ka, 0, E);
            int64_t kb = gather_ivs(ds, de, dr, dk, kd, did, -1, B);
            kb = iv_flatten(B, kb); kb = iv_intersect(B, kb, 0, E);
            const int64_t kdiff = iv_subtract(A, ka, B, kb, D);
            const u128 ov = iv_total(A, ka) - iv_total(D, kdiff);
            busy[q] = (uint64_t)ov;
            num += ov;
            den += o->host_sum[((size_t)j * (size_t)n + (size_t)p) * 4 + 1];
        }
        if (den > 0) { o->busy_frac[j] = orc_div_exact(num, den); o->busy_mask[j] = 1; }
    }
    free(hs); free(he); free(hr); free(hk); free(ds); free(de); free(dr); free(dk); free(A); free(B); free(D);
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* exported interval algebra restatements (tests pin them to fixtures  */
/* generated from the reference's intervals.py)                        */
/* ------------------------------------------------------------------ */
int64_t orc_iv_flatten(const uint64_t *s, const uint64_t *e, int64_t n, uint64_t *os, uint64_t *oe, int64_t *bad)
{
    *bad = -1;
    for (int64_t i = 0; i < n; ++i) if (s[i] > e[i]) { *bad = i; return -1; }   /* intervals.py:49-51 */
    iv_t *v = malloc(sizeof(iv_t) * (size_t)(n + 1));
    for (int64_t i = 0; i < n; ++i) { v[i].s = s[i]; v[i].e = e[i]; }
    int64_t k = iv_flatten(v, n);
    for (int64_t i = 0; i < k; ++i) { os[i] = v[i].s; oe[i] = v[i].e; }
    free(v);
    return k;
}

int64_t orc_iv_subtract(const uint64_t *as, const uint64_t *ae, int64_t na, const uint64_t *bs, const uint64_t *be,
                        int64_t nb, uint64_t *os, uint64_t *oe)
{
    iv_t *a = malloc(sizeof(iv_t) * (size_t)(na + 1)), *b = malloc(sizeof(iv_t) * (size_t)(nb + 1));
    iv_t *o = malloc(sizeof(iv_t) * (size_t)(na + nb + 1));
    for (int64_t i = 0; i < na; ++i) { a[i].s = as[i]; a[i].e = ae[i]; }
    for (int64_t i = 0; i < nb; ++i) { b[i].s = bs[i]; b[i].e = be[i]; }
    int64_t k = iv_subtract(a, na, b, nb, o);
    for (int64_t i = 0; i < k; ++i) { os[i] = o[i].s; oe[i] = o[i].e; }
    free(a); free(b); free(o);
    return k;
}

int64_t orc_iv_intersect(const uint64_t *s, const uint64_t *e, int64_t n, uint64_t lo, uint64_t hi, uint64_t *os,
                         uint64_t *oe)
{
    iv_t *v = malloc(sizeof(iv_t) * (size_t)(n + 1));
    for (int64_t i = 0; i < n; ++i) { v[i].s = s[i]; v[i].e = e[i]; }
    int64_t k = iv_intersect(v, n, lo, hi);
    for (int64_t i = 0; i < k; ++i) { os[i] = v[i].s; oe[i] = v[i].e; }
    free(v);
    return k;
}

void orc_iv_total(const uint64_t *s, const uint64_t *e, int64_t n, uint64_t out[2])
{
    u128 t = 0;
    for (int64_t i = 0; i < n; ++i) t += e[i] - s[i];
    out[0] = (uint64_t)t; out[1] = (uint64_t)(t >> 64);
}
