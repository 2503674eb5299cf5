// ingest.cpp -- native trace documents (docs/formats.md:9-85, the reference's
// read_trace, trace_io.py:96-158) parsed straight into record columns.
//
// Two phases:
//   1. one sequential, string-aware skip scan over the document finds the
//      top-level fields and the byte range of every hosts[] / devices[] entry
//      (no values are decoded);
//   2. the entries are parsed in parallel (std::thread, dynamic claiming), each
//      by a strict recursive-descent parser of exactly the reference schema,
//      into per-entry column slices; a prefix sum places every slice.
// Records come out in FILE order with their original rank / device ids; the
// Python layer assigns dense ids and the canonical order (or hands unsorted
// columns to the K3 GPU sort).
//
// Anything the fast path does not decide exactly -- a schema error (whose
// message carries a JSON path), an integer beyond u64, a duplicate key, a
// non-integer number -- returns HETEFF_PARSE_FALLBACK with the byte offset;
// the Python layer then re-parses with its strict restatement of read_trace,
// which produces the reference's exact TraceFormatError text.
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <climits>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/heteff_b200.h"

namespace {

struct Cursor {
    const char *p, *e;
    bool ok = true;
    void ws()
    {
        while (p < e && (*p == ' ' || *p == '\n' || *p == '\r' || *p == '\t')) ++p;
    }
    bool eat(char c)
    {
        ws();
        if (p < e && *p == c) { ++p; return true; }
        return false;
    }
    bool peek(char c)
    {
        ws();
        return p < e && *p == c;
    }
};

// a JSON string without escapes (keys and enum values of the schema); escapes -> fallback
bool plain_string(Cursor &c, const char *&s, size_t &n)
{
    c.ws();
    if (c.p >= c.e || *c.p != '"') return false;
    const char *q = static_cast<const char *>(memchr(c.p + 1, '"', (size_t)(c.e - c.p - 1)));
    if (!q) return false;
    for (const char *t = c.p + 1; t < q; ++t)
        if (*t == '\\' || (unsigned char)*t < 0x20) return false;
    s = c.p + 1;
    n = (size_t)(q - s);
    c.p = q + 1;
    return true;
}

// non-negative integer that fits u64; anything else (sign, fraction, exponent, overflow) -> false
bool u64_number(Cursor &c, uint64_t &v)
{
    c.ws();
    const char *q = c.p;
    if (q >= c.e || *q < '0' || *q > '9') return false;
    if (*q == '0' && q + 1 < c.e && q[1] >= '0' && q[1] <= '9') return false;   // leading zero: invalid JSON
    uint64_t x = 0;
    const char *b = q;
    while (q < c.e && (unsigned)(*q - '0') < 10u) {
        if (q - b >= 19) {   // a 20th digit may overflow: checked multiply-add
            unsigned long long y;
            if (__builtin_mul_overflow((unsigned long long)x, 10ull, &y) ||
                __builtin_add_overflow(y, (unsigned long long)(*q - '0'), &y))
                return false;
            x = y;
        } else {
            x = x * 10 + (uint64_t)(*q - '0');
        }
        ++q;
    }
    if (q < c.e && (*q == '.' || *q == 'e' || *q == 'E')) return false;
    v = x;
    c.p = q;
    return true;
}

bool is_null(Cursor &c)
{
    c.ws();
    if (c.e - c.p >= 4 && memcmp(c.p, "null", 4) == 0) { c.p += 4; return true; }
    return false;
}

template <size_t L>
inline bool key_is(const char *s, size_t n, const char (&lit)[L])
{
    return n == L - 1 && memcmp(s, lit, L - 1) == 0;
}

// structural-character table for the phase-1 skip scan
struct Structural {
    bool t[256];
    Structural()
    {
        memset(t, 0, sizeof(t));
        t[(unsigned char)'"'] = t[(unsigned char)'{'] = t[(unsigned char)'['] = true;
        t[(unsigned char)'}'] = t[(unsigned char)']'] = true;
    }
};
const Structural kStruct;

// end of a string body starting at p (just after the opening quote): the closing quote
inline const char *string_end(const char *p, const char *e)
{
    for (;;) {
        const char *q = static_cast<const char *>(memchr(p, '"', (size_t)(e - p)));
        if (!q) return nullptr;
        // count the backslashes right before the quote: an even number means it closes
        const char *b = q;
        while (b > p && b[-1] == '\\') --b;
        if (((q - b) & 1) == 0) return q;
        p = q + 1;
    }
}

// skip any JSON value (string-aware), used only by the phase-1 scan
bool skip_value(Cursor &c)
{
    c.ws();
    if (c.p >= c.e) return false;
    const char ch = *c.p;
    if (ch == '"') {
        ++c.p;
        while (c.p < c.e && *c.p != '"') {
            if (*c.p == '\\') ++c.p;
            ++c.p;
        }
        if (c.p >= c.e) return false;
        ++c.p;
        return true;
    }
    if (ch == '{' || ch == '[') {
        int depth = 0;
        const char *p = c.p, *e = c.e;
        while (p < e) {
            while (p < e && !kStruct.t[(unsigned char)*p]) ++p;
            if (p >= e) break;
            const char x = *p;
            if (x == '"') {
                p = string_end(p + 1, e);
                if (!p) return false;
            } else if (x == '{' || x == '[') {
                ++depth;
            } else if (--depth == 0) {
                c.p = p + 1;
                return true;
            }
            ++p;
        }
        return false;
    }
    while (c.p < c.e && *c.p != ',' && *c.p != '}' && *c.p != ']' && *c.p != ' ' && *c.p != '\n' && *c.p != '\r' &&
           *c.p != '\t')
        ++c.p;
    return true;
}

struct Entry {
    const char *b, *e;   // the entry object's bytes
    bool device;
};

struct Slice {
    uint64_t id = 0;
    int64_t owner = -1;
    const char *stop = nullptr;   // one past the entry's closing brace
    std::vector<uint8_t> kind;
    std::vector<int64_t> stream;
    std::vector<uint64_t> start, end;
    const char *fail = nullptr;   // first byte the fast path could not decide
};

// { "state": s, "start": a, "end": b } / { "kind": k, ["stream": x,] "start": a, "end": b } in any key order
bool parse_record(Cursor &c, bool device, Slice &out)
{
    if (!c.eat('{')) return false;
    bool h_state = false, h_start = false, h_end = false, h_stream = false;
    uint8_t kind = 0;
    int64_t stream = -1;
    uint64_t s = 0, e = 0;
    if (!c.peek('}')) {
        do {
            const char *k;
            size_t kn;
            if (!plain_string(c, k, kn) || !c.eat(':')) return false;
            if (!device && key_is(k, kn, "state")) {
                if (h_state) return false;
                const char *v;
                size_t vn;
                if (!plain_string(c, v, vn)) return false;
                if (key_is(v, vn, "useful")) kind = 0;
                else if (key_is(v, vn, "offload")) kind = 1;
                else if (key_is(v, vn, "mpi")) kind = 2;
                else return false;
                h_state = true;
            } else if (device && key_is(k, kn, "kind")) {
                if (h_state) return false;
                const char *v;
                size_t vn;
                if (!plain_string(c, v, vn)) return false;
                if (key_is(v, vn, "kernel")) kind = 0;
                else if (key_is(v, vn, "memory")) kind = 1;
                else return false;
                h_state = true;
            } else if (device && key_is(k, kn, "stream")) {
                if (h_stream) return false;
                if (!is_null(c)) {
                    uint64_t x;
                    if (!u64_number(c, x) || x > (uint64_t)INT64_MAX) return false;
                    stream = (int64_t)x;
                }
                h_stream = true;
            } else if (key_is(k, kn, "start")) {
                if (h_start || !u64_number(c, s)) return false;
                h_start = true;
            } else if (key_is(k, kn, "end")) {
                if (h_end || !u64_number(c, e)) return false;
                h_end = true;
            } else {
                return false;   // unknown field
            }
        } while (c.eat(','));
    }
    if (!c.eat('}') || !h_state || !h_start || !h_end) return false;
    out.kind.push_back(kind);
    if (device) out.stream.push_back(stream);
    out.start.push_back(s);
    out.end.push_back(e);
    return true;
}

bool parse_entry(const Entry &en, Slice &out)
{
    Cursor c{en.b, en.e};
    const size_t guess = (size_t)(en.e - en.b) / 40 + 4;
    out.kind.reserve(guess);
    out.start.reserve(guess);
    out.end.reserve(guess);
    if (en.device) out.stream.reserve(guess);
    if (!c.eat('{')) { out.fail = c.p; return false; }
    bool h_id = false, h_owner = false, h_recs = false;
    if (!c.peek('}')) {
        do {
            const char *k;
            size_t kn;
            if (!plain_string(c, k, kn) || !c.eat(':')) { out.fail = c.p; return false; }
            if (!en.device && key_is(k, kn, "rank")) {
                if (h_id || !u64_number(c, out.id)) { out.fail = c.p; return false; }
                h_id = true;
            } else if (en.device && key_is(k, kn, "id")) {
                if (h_id || !u64_number(c, out.id)) { out.fail = c.p; return false; }
                h_id = true;
            } else if (en.device && key_is(k, kn, "owner_rank")) {
                if (h_owner) { out.fail = c.p; return false; }
                if (!is_null(c)) {
                    uint64_t x;
                    if (!u64_number(c, x) || x > (uint64_t)INT64_MAX) { out.fail = c.p; return false; }
                    out.owner = (int64_t)x;
                }
                h_owner = true;
            } else if (key_is(k, kn, "records")) {
                if (h_recs || !c.eat('[')) { out.fail = c.p; return false; }
                if (!c.peek(']')) {
                    do {
                        if (!parse_record(c, en.device, out)) { out.fail = c.p; return false; }
                    } while (c.eat(','));
                }
                if (!c.eat(']')) { out.fail = c.p; return false; }
                h_recs = true;
            } else {
                out.fail = c.p;
                return false;
            }
        } while (c.eat(','));
    }
    if (!c.eat('}') || !h_id || !h_recs) { out.fail = c.p; return false; }
    out.stop = c.p;
    return true;
}

// entry-start candidate at '{': the first key is "rank" (host) or "id" (device)
// -- what every writer emits; records start with other keys
int entry_kind_at(const char *q, const char *e)
{
    ++q;
    while (q < e && (*q == ' ' || *q == '\n' || *q == '\r' || *q == '\t')) ++q;
    if (e - q >= 6 && memcmp(q, "\"rank\"", 6) == 0) return 0;
    if (e - q >= 4 && memcmp(q, "\"id\"", 4) == 0) return 1;
    return -1;
}

// phase 0 of one chunk [a, b): speculative discovery + parse of the entries starting there
struct Spec {
    size_t off;          // entry start offset
    int dev;
    Slice slice;
};

void discover(const char *data, size_t len, size_t a, size_t b, std::vector<Spec> &found)
{
    const char *e = data + len;
    const char *q = data + a;
    while (q < data + b) {
        q = static_cast<const char *>(memchr(q, '{', (size_t)(data + b - q)));
        if (!q) break;
        const int kind = entry_kind_at(q, e);
        if (kind < 0) { ++q; continue; }
        Spec sp;
        sp.off = (size_t)(q - data);
        sp.dev = kind;
        if (parse_entry(Entry{q, e, kind == 1}, sp.slice) && sp.slice.stop) {
            q = sp.slice.stop;
            found.push_back(std::move(sp));
        } else {
            ++q;   // not an entry after all (or an error the skeleton pass will meet)
        }
    }
}

}  // namespace


// ---------------------------------------------------------------------------
// Chrome-trace-event documents + mapping rules (import_mapped, trace_io.py:263-342)
// ---------------------------------------------------------------------------
namespace {

struct Event {
    const char *b, *e;
};

// a JSON number as exact nanoseconds (value * 1000): integers, or floats whose
// value is an integer (the reference's _us_to_ns); anything else -> false
bool us_to_ns(Cursor &c, uint64_t &ns)
{
    c.ws();
    const char *q = c.p;
    if (q >= c.e) return false;
    if (*q == '-') return false;
    const char *t = q;
    bool fl = false;
    while (t < c.e && ((*t >= '0' && *t <= '9') || *t == '.' || *t == 'e' || *t == 'E' || *t == '+' || *t == '-')) {
        if (*t == '.' || *t == 'e' || *t == 'E') fl = true;
        ++t;
    }
    if (t == q) return false;
    uint64_t v = 0;
    if (!fl) {
        Cursor d{q, t};
        if (!u64_number(d, v) || d.p != t) return false;
    } else {
        char buf[64];
        if (t - q >= (long)sizeof(buf)) return false;
        memcpy(buf, q, (size_t)(t - q));
        buf[t - q] = 0;
        char *endp = nullptr;
        const double x = strtod(buf, &endp);
        if (endp != buf + (t - q) || !(x >= 0) || x != (double)(uint64_t)x || x >= 1.8e19) return false;
        v = (uint64_t)x;
    }
    if (v > UINT64_MAX / 1000) return false;
    ns = v * 1000;
    c.p = t;
    return true;
}

struct RawEvent {
    bool is_x = false;
    const char *name = nullptr, *cat = nullptr;
    size_t name_n = 0, cat_n = 0;
    bool has_cat = false, has_ts = false, has_dur = false, has_pid = false, has_tid = false;
    uint64_t ts = 0, dur = 0, pid = 0, tid = 0;
    bool pid_ok = false, tid_ok = false;
};

// 1: parsed, 0: not an "X" event (skipped), -1: undecided (fallback)
int parse_event(const Event &ev, RawEvent &r)
{
    Cursor c{ev.b, ev.e};
    c.ws();
    if (c.p >= c.e || *c.p != '{') return 0;   // not an object: ignored by the reference
    ++c.p;
    bool h_ph = false, h_name = false;
    bool ph_x = false;
    if (!c.peek('}')) {
        do {
            const char *k;
            size_t kn;
            if (!plain_string(c, k, kn) || !c.eat(':')) return -1;
            if (key_is(k, kn, "ph")) {
                if (h_ph) return -1;
                h_ph = true;
                c.ws();
                if (c.p < c.e && *c.p == '"') {
                    const char *v;
                    size_t vn;
                    if (!plain_string(c, v, vn)) return -1;
                    ph_x = vn == 1 && v[0] == 'X';
                } else if (!skip_value(c)) {
                    return -1;
                }
            } else if (key_is(k, kn, "name") || key_is(k, kn, "cat")) {
                const bool nm = k[0] == 'n';
                if (nm ? h_name : r.has_cat) return -1;
                c.ws();
                if (c.p >= c.e || *c.p != '"') {   // a non-string name / cat is an error if the event is "X"
                    if (!skip_value(c)) return -1;
                    if (nm) { h_name = true; r.name = nullptr; }
                    else { r.has_cat = true; r.cat = nullptr; }
                    continue;
                }
                const char *v;
                size_t vn;
                if (!plain_string(c, v, vn)) return -1;
                if (nm) { h_name = true; r.name = v; r.name_n = vn; }
                else { r.has_cat = true; r.cat = v; r.cat_n = vn; }
            } else if (key_is(k, kn, "ts") || key_is(k, kn, "dur")) {
                const bool ts = k[0] == 't';
                if (ts ? r.has_ts : r.has_dur) return -1;
                const char *save = c.p;
                uint64_t v;
                if (!us_to_ns(c, v)) { c.p = save; if (!skip_value(c)) return -1; v = UINT64_MAX; }
                if (ts) { r.has_ts = true; r.ts = v; } else { r.has_dur = true; r.dur = v; }
            } else if (key_is(k, kn, "pid") || key_is(k, kn, "tid")) {
                const bool pid = k[0] == 'p';
                if (pid ? r.has_pid : r.has_tid) return -1;
                const char *save = c.p;
                uint64_t v = 0;
                bool ok = u64_number(c, v);
                if (!ok) { c.p = save; if (!skip_value(c)) return -1; }
                if (pid) { r.has_pid = true; r.pid = v; r.pid_ok = ok; }
                else { r.has_tid = true; r.tid = v; r.tid_ok = ok; }
            } else {
                if (!skip_value(c)) return -1;
            }
        } while (c.eat(','));
    }
    if (!c.eat('}')) return -1;
    if (!h_ph || !ph_x) return 0;
    r.is_x = true;
    // the reference raises for these on an "X" event: leave the exact message to the fallback
    if (!h_name || !r.name) return -1;
    if (r.has_cat && !r.cat) return -1;
    if (!r.has_ts || !r.has_dur || r.ts == UINT64_MAX || r.dur == UINT64_MAX) return -1;
    if (r.ts > UINT64_MAX - r.dur) return -1;
    return 1;
}

bool contains(const char *h, size_t hn, const char *n, size_t nn)
{
    if (nn == 0) return true;
    if (nn > hn) return false;
    const void *p = memmem(h, hn, n, nn);
    return p != nullptr;
}

}  // namespace

struct heteff_imported {
    std::vector<uint8_t> is_dev, kind;
    std::vector<uint64_t> res, start, end;
    std::vector<int64_t> unmapped;            // event indices of unmapped "X" events
    std::vector<int64_t> name_off;            // byte offset of each unmapped event's name in the document
    std::vector<int64_t> name_len;
};

extern "C" {

int heteff_import_events(const char *data, size_t len, const heteff_rule *rules, int nrules, int nthreads,
                         heteff_imported **out, int64_t *fail_offset)
{
    if (!data || !out || !fail_offset || (nrules > 0 && !rules)) return HETEFF_BAD_ARG;
    *out = nullptr;
    *fail_offset = -1;
    Cursor c{data, data + len};
    auto fail = [&](const char *at) {
        *fail_offset = (int64_t)(at - data);
        return HETEFF_PARSE_FALLBACK;
    };
    if (c.e - c.p >= 3 && (unsigned char)c.p[0] == 0xEF && (unsigned char)c.p[1] == 0xBB) return fail(c.p);
    // the events array: a bare array, or the traceEvents field of an object
    std::vector<Event> events;
    auto scan_array = [&](Cursor &a) -> bool {
        if (!a.eat('[')) return false;
        if (!a.peek(']')) {
            do {
                a.ws();
                const char *b = a.p;
                if (!skip_value(a)) return false;
                events.push_back(Event{b, a.p});
            } while (a.eat(','));
        }
        return a.eat(']');
    };
    c.ws();
    if (c.peek('[')) {
        if (!scan_array(c)) return fail(c.p);
    } else if (c.eat('{')) {
        bool found = false;
        if (!c.peek('}')) {
            do {
                const char *k;
                size_t kn;
                if (!plain_string(c, k, kn) || !c.eat(':')) return fail(c.p);
                if (key_is(k, kn, "traceEvents")) {
                    if (found) return fail(c.p);
                    found = true;
                    if (!c.peek('[')) return fail(c.p);
                    if (!scan_array(c)) return fail(c.p);
                } else if (!skip_value(c)) {
                    return fail(c.p);
                }
            } while (c.eat(','));
        }
        if (!c.eat('}') || !found) return fail(c.p);
    } else {
        return fail(c.p);
    }
    c.ws();
    if (c.p != c.e) return fail(c.p);

    // events in parallel: parse + first-match-wins rules
    const size_t n = events.size();
    std::vector<int8_t> status(n, 0);   // 1 mapped, 2 unmapped, 0 skipped, -1 fallback
    std::vector<uint8_t> is_dev(n), kind(n);
    std::vector<uint64_t> res(n), st(n), en(n);
    std::vector<int64_t> noff(n), nlen(n);
    std::atomic<size_t> next{0};
    std::atomic<int64_t> first_fail{INT64_MAX};
    const size_t chunk = 4096;
    auto work = [&]() {
        for (;;) {
            const size_t c0 = next.fetch_add(chunk);
            if (c0 >= n) break;
            const size_t c1 = c0 + chunk < n ? c0 + chunk : n;
            for (size_t i = c0; i < c1; ++i) {
                RawEvent r;
                const int pr = parse_event(events[i], r);
                if (pr <= 0) { status[i] = (int8_t)pr; if (pr < 0) { int64_t cur = first_fail.load(); while ((int64_t)i < cur && !first_fail.compare_exchange_weak(cur, (int64_t)i)) {} } continue; }
                int hit = -1;
                for (int q = 0; q < nrules && hit < 0; ++q) {
                    const heteff_rule &R = rules[q];
                    const char *subj = R.field == 0 ? r.name : (r.has_cat ? r.cat : "");
                    const size_t sn = R.field == 0 ? r.name_n : (r.has_cat ? r.cat_n : 0);
                    const bool m = R.mode == 0 ? contains(subj, sn, R.pattern, (size_t)R.pattern_len)
                                               : ((size_t)R.pattern_len == sn && memcmp(subj, R.pattern, sn) == 0);
                    if (m) hit = q;
                }
                st[i] = r.ts;
                en[i] = r.ts + r.dur;
                noff[i] = (int64_t)(r.name - data);
                nlen[i] = (int64_t)r.name_n;
                if (hit < 0) { status[i] = 2; continue; }
                const heteff_rule &R = rules[hit];
                uint64_t rid = 0;
                if (R.resource >= 0) {
                    rid = (uint64_t)R.resource;
                } else {
                    const bool pid = R.resource == -1;
                    const bool has = pid ? r.has_pid : r.has_tid, ok = pid ? r.pid_ok : r.tid_ok;
                    if (!has || !ok) {   // the reference's _nonneg_int error: exact text from the fallback
                        status[i] = -1;
                        int64_t cur = first_fail.load();
                        while ((int64_t)i < cur && !first_fail.compare_exchange_weak(cur, (int64_t)i)) {}
                        continue;
                    }
                    rid = pid ? r.pid : r.tid;
                }
                status[i] = 1;
                is_dev[i] = R.target >= 3;
                kind[i] = (uint8_t)(R.target >= 3 ? R.target - 3 : R.target);
                res[i] = rid;
            }
        }
    };
    int nt = nthreads > 0 ? nthreads : (int)std::thread::hardware_concurrency();
    if (nt < 1) nt = 1;
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto &th : pool) th.join();
    if (first_fail.load() != INT64_MAX) return fail(events[(size_t)first_fail.load()].b);

    heteff_imported *I = new heteff_imported();
    for (size_t i = 0; i < n; ++i) {
        if (status[i] == 1) {
            I->is_dev.push_back(is_dev[i]);
            I->kind.push_back(kind[i]);
            I->res.push_back(res[i]);
            I->start.push_back(st[i]);
            I->end.push_back(en[i]);
        } else if (status[i] == 2) {
            I->unmapped.push_back((int64_t)i);
            I->name_off.push_back(noff[i]);
            I->name_len.push_back(nlen[i]);
        }
    }
    *out = I;
    return HETEFF_OK;
}

void heteff_imported_info(const heteff_imported *I, heteff_imported_view *v)
{
    v->n_records = (int64_t)I->start.size();
    v->n_unmapped = (int64_t)I->unmapped.size();
    v->is_dev = I->is_dev.data();
    v->kind = I->kind.data();
    v->res = I->res.data();
    v->start = I->start.data();
    v->end = I->end.data();
    v->unmapped = I->unmapped.data();
    v->name_off = I->name_off.data();
    v->name_len = I->name_len.data();
}

void heteff_imported_free(heteff_imported *I) { delete I; }

}  // extern "C"

struct heteff_parsed {
    std::vector<uint64_t> host_rank, dev_id;
    std::vector<int64_t> dev_owner;
    std::vector<int64_t> host_off, dev_off;   // [entries + 1] record offsets per entry
    std::vector<uint8_t> h_kind, d_kind;
    std::vector<int64_t> d_stream;
    std::vector<uint64_t> h_start, h_end, d_start, d_end;
};

extern "C" {

int heteff_parse_trace(const char *data, size_t len, int nthreads, heteff_parsed **out, int64_t *fail_offset)
{
    if (!data || !out || !fail_offset) return HETEFF_BAD_ARG;
    *out = nullptr;
    *fail_offset = -1;
    Cursor c{data, data + len};
    auto fail = [&](const char *at) {
        *fail_offset = (int64_t)(at - data);
        return HETEFF_PARSE_FALLBACK;
    };
    int nt = nthreads > 0 ? nthreads : (int)std::thread::hardware_concurrency();
    if (nt < 1) nt = 1;
    if (c.e - c.p >= 3 && (unsigned char)c.p[0] == 0xEF && (unsigned char)c.p[1] == 0xBB) return fail(c.p);   // BOM
    // ---- phase 0 (parallel): every chunk finds and parses the entries that start in it
    std::vector<std::vector<Spec>> spec((size_t)nt);
    {
        std::vector<std::thread> pool;
        const size_t chunk = (len + (size_t)nt - 1) / (size_t)nt;
        for (int t = 0; t < nt; ++t) {
            const size_t a = (size_t)t * chunk, b = a + chunk < len ? a + chunk : len;
            if (a >= b) continue;
            if (t == 0) continue;   // run chunk 0 on this thread below
            pool.emplace_back(discover, data, len, a, b, std::ref(spec[(size_t)t]));
        }
        if (len > 0) discover(data, len, 0, chunk < len ? chunk : len, spec[0]);
        for (auto &th : pool) th.join();
    }
    // chunks are disjoint and in order, so the candidates are sorted by offset
    std::vector<Spec *> cand;
    for (auto &v : spec)
        for (auto &x : v) cand.push_back(&x);
    auto lookup = [&](size_t off) -> Spec * {
        size_t lo = 0, hi = cand.size();
        while (lo < hi) {
            const size_t mid = (lo + hi) >> 1;
            if (cand[mid]->off < off) lo = mid + 1;
            else hi = mid;
        }
        return lo < cand.size() && cand[lo]->off == off ? cand[lo] : nullptr;
    };
    // ---- phase 1 (sequential skeleton): the top level; each entry is taken from phase 0 by
    // its offset, or skipped and queued for phase 2 when phase 0 did not decide it
    if (!c.eat('{')) return fail(c.p);
    bool h_ver = false, h_tu = false, h_hosts = false, h_devs = false;
    std::vector<Entry> entries;
    std::vector<Slice> slices;
    std::vector<size_t> todo;   // entries phase 0 did not parse
    size_t n_hosts = 0;
    std::vector<Entry> dev_entries;
    std::vector<Slice> dev_slices;
    std::vector<size_t> dev_todo;
    if (!c.peek('}')) {
        do {
            const char *k;
            size_t kn;
            if (!plain_string(c, k, kn) || !c.eat(':')) return fail(c.p);
            if (key_is(k, kn, "version")) {
                uint64_t v;
                if (h_ver || !u64_number(c, v) || v != 1) return fail(c.p);
                h_ver = true;
            } else if (key_is(k, kn, "time_unit")) {
                const char *v;
                size_t vn;
                if (h_tu || !plain_string(c, v, vn) || !key_is(v, vn, "ns")) return fail(c.p);
                h_tu = true;
            } else if (key_is(k, kn, "hosts") || key_is(k, kn, "devices")) {
                const bool dev = key_is(k, kn, "devices");
                if ((dev ? h_devs : h_hosts) || !c.eat('[')) return fail(c.p);
                std::vector<Entry> &E = dev ? dev_entries : entries;
                std::vector<Slice> &S = dev ? dev_slices : slices;
                std::vector<size_t> &T = dev ? dev_todo : todo;
                if (!c.peek(']')) {
                    do {
                        c.ws();
                        const char *b = c.p;
                        if (!c.peek('{')) return fail(b);
                        Spec *sp = lookup((size_t)(b - data));
                        if (sp && sp->dev == (dev ? 1 : 0)) {
                            c.p = sp->slice.stop;
                            E.push_back(Entry{b, c.p, dev});
                            S.push_back(std::move(sp->slice));
                        } else {
                            if (!skip_value(c)) return fail(b);
                            T.push_back(E.size());
                            E.push_back(Entry{b, c.p, dev});
                            S.emplace_back();
                        }
                    } while (c.eat(','));
                }
                if (!c.eat(']')) return fail(c.p);
                if (dev) h_devs = true;
                else { h_hosts = true; n_hosts = entries.size(); }
            } else {
                return fail(c.p);
            }
        } while (c.eat(','));
    }
    if (!c.eat('}') || !h_ver || !h_tu || !h_hosts || !h_devs) return fail(c.p);
    c.ws();
    if (c.p != c.e) return fail(c.p);
    for (size_t i : dev_todo) todo.push_back(n_hosts + i);   // hosts first, then devices
    entries.insert(entries.end(), dev_entries.begin(), dev_entries.end());
    for (auto &x : dev_slices) slices.push_back(std::move(x));

    // ---- phase 2 (parallel): entries phase 0 left (unusual key order, errors)
    std::atomic<size_t> next{0};
    auto work = [&]() {
        for (;;) {
            const size_t q = next.fetch_add(1);
            if (q >= todo.size()) break;
            const size_t i = todo[q];
            if (!parse_entry(entries[i], slices[i]) && !slices[i].fail) slices[i].fail = entries[i].b;
        }
    };
    std::vector<std::thread> pool;
    const int nt2 = (size_t)nt > todo.size() ? (todo.empty() ? 1 : (int)todo.size()) : nt;
    for (int t = 1; t < nt2; ++t) pool.emplace_back(work);
    work();
    for (auto &th : pool) th.join();
    for (const Slice &sl : slices)
        if (sl.fail) return fail(sl.fail);

    // ---- merge in file order
    heteff_parsed *P = new heteff_parsed();
    size_t nh = 0, nd = 0;
    P->host_off.push_back(0);
    P->dev_off.push_back(0);
    for (size_t i = 0; i < entries.size(); ++i) {
        if (i < n_hosts) { nh += slices[i].start.size(); P->host_off.push_back((int64_t)nh); }
        else { nd += slices[i].start.size(); P->dev_off.push_back((int64_t)nd); }
    }
    P->h_kind.resize(nh); P->h_start.resize(nh); P->h_end.resize(nh);
    P->d_kind.resize(nd); P->d_stream.resize(nd); P->d_start.resize(nd); P->d_end.resize(nd);
    std::atomic<size_t> nx{0};
    auto copy = [&]() {
        for (;;) {
            const size_t i = nx.fetch_add(1);
            if (i >= entries.size()) break;
            const Slice &s = slices[i];
            const size_t k = s.start.size();
            if (!k) continue;
            if (i < n_hosts) {
                const size_t o = (size_t)P->host_off[i];
                memcpy(&P->h_kind[o], s.kind.data(), k);
                memcpy(&P->h_start[o], s.start.data(), 8 * k);
                memcpy(&P->h_end[o], s.end.data(), 8 * k);
            } else {
                const size_t o = (size_t)P->dev_off[i - n_hosts];
                memcpy(&P->d_kind[o], s.kind.data(), k);
                memcpy(&P->d_stream[o], s.stream.data(), 8 * k);
                memcpy(&P->d_start[o], s.start.data(), 8 * k);
                memcpy(&P->d_end[o], s.end.data(), 8 * k);
            }
        }
    };
    pool.clear();
    for (int t = 1; t < nt; ++t) pool.emplace_back(copy);
    copy();
    for (auto &th : pool) th.join();
    for (size_t i = 0; i < entries.size(); ++i) {
        if (i < n_hosts) P->host_rank.push_back(slices[i].id);
        else { P->dev_id.push_back(slices[i].id); P->dev_owner.push_back(slices[i].owner); }
    }
    *out = P;
    return HETEFF_OK;
}

void heteff_parsed_info(const heteff_parsed *P, heteff_parsed_view *v)
{
    v->n_hosts = (int64_t)P->host_rank.size();
    v->n_devices = (int64_t)P->dev_id.size();
    v->n_host_records = (int64_t)P->h_start.size();
    v->n_dev_records = (int64_t)P->d_start.size();
    v->host_rank = P->host_rank.data();
    v->host_off = P->host_off.data();
    v->dev_id = P->dev_id.data();
    v->dev_owner = P->dev_owner.data();
    v->dev_off = P->dev_off.data();
    v->h_kind = P->h_kind.data();
    v->h_start = P->h_start.data();
    v->h_end = P->h_end.data();
    v->d_kind = P->d_kind.data();
    v->d_stream = P->d_stream.data();
    v->d_start = P->d_start.data();
    v->d_end = P->d_end.data();
}

void heteff_parsed_free(heteff_parsed *P) { delete P; }

}  // extern "C"
