"""Native trace documents -> traces / packed columns.

``read_trace(data)`` is the drop-in for the reference's ``read_trace``
(``trace_io.py:96-158``, format ``docs/formats.md:9-85``): same Trace, same
``TraceFormatError`` texts.  ``read_trace_packed(data)`` skips Python record
objects entirely: the document is parsed by the native multi-threaded parser
(``csrc/ingest.cpp``) straight into columns, which get dense ids and the
reference's canonical order with numpy, ready for the GPU analysis
(``engine.analyze_packed``).

The native parser decides every well-formed document exactly; anything else
(a schema error, an integer beyond u64, a duplicate key, a non-integer number,
escapes in keys) is handed to ``_parse_py``, a strict restatement of the
reference reader, which produces the reference's exact error text (or, for the
rare legal-but-unusual document, the trace).
"""

from __future__ import annotations

import ctypes as C
import json
import os

import numpy as np

from . import _native as N
from .model import DeviceActivityKind, DeviceDecl, DeviceRecord, HostRecord, HostState, Interval, Trace
from .packing import PackedTrace, RecordColumns, pack_trace

FORMAT_VERSION = 1
_HOST_CODE_STATE = (HostState.USEFUL, HostState.OFFLOAD, HostState.MPI)     # ingest codes 0, 1, 2
_DEV_CODE_KIND = (DeviceActivityKind.KERNEL, DeviceActivityKind.MEMORY)


class TraceFormatError(Exception):
    """A document does not conform to the native trace schema."""


# ---------------------------------------------------------------------------
# strict pure-Python reader: the error path (and unusual legal documents).
# The document schema (pkg/docs/formats.md:9-85) is data -- SCHEMA below -- and one
# walker checks any value against a node of it, so each error text is produced in
# exactly one place: objects (required / optional / unknown fields, checked in
# schema order, unknown ones after the known ones), arrays, non-negative integers,
# enumerations and constants.
# ---------------------------------------------------------------------------
def _load(data):
    if isinstance(data, bytes):
        try:
            data = data.decode("utf-8")
        except UnicodeDecodeError as e:
            raise TraceFormatError(f"trace document is not UTF-8: {e}") from e
    try:
        return json.loads(data)
    except json.JSONDecodeError as e:
        raise TraceFormatError(f"trace document is not valid JSON: {e}") from e


class _Node:
    def check(self, value, path: str):
        raise NotImplementedError


class _Pass(_Node):
    def check(self, value, path):
        return value


class _UInt(_Node):
    def check(self, value, path):
        if isinstance(value, bool) or not isinstance(value, int):
            raise TraceFormatError(f"{path}: expected integer, got {value!r}")
        if value < 0:
            raise TraceFormatError(f"{path}: negative value {value}")
        return value


class _Enum(_Node):
    def __init__(self, members):
        self.table = {m.value: m for m in members}

    def check(self, value, path):
        if isinstance(value, str) and value in self.table:
            return self.table[value]
        raise TraceFormatError(f"{path}: expected one of {', '.join(sorted(self.table))}; got {value!r}")


class _Const(_Node):
    def __init__(self, want, message):
        self.want, self.message = want, message

    def check(self, value, path):
        if value != self.want:
            raise TraceFormatError(f"{path}: {self.message.format(got=value)}")
        return value


class _Array(_Node):
    def __init__(self, item):
        self.item = item

    def check(self, value, path):
        if not isinstance(value, list):
            raise TraceFormatError(f"{path}: expected array, got {type(value).__name__}")
        return [self.item.check(v, f"{path}[{i}]") for i, v in enumerate(value)]


class _Object(_Node):
    """Fields as (name, node, required); an optional field given as null counts as absent."""

    def __init__(self, *fields):
        self.fields = fields

    def check(self, value, path):
        if not isinstance(value, dict):
            raise TraceFormatError(f"{path}: expected object, got {type(value).__name__}")
        out = {}
        for name, node, required in self.fields:
            if name not in value:
                if required:
                    raise TraceFormatError(f"{path}: missing required field {name!r}")
                out[name] = None
                continue
            v = value[name]
            out[name] = None if (v is None and not required) else node.check(v, f"{path}.{name}")
        extra = sorted(k for k in value if k not in out)
        if extra:
            raise TraceFormatError(f"{path}: unknown field {extra[0]!r}")
        return out


class _Str(_Node):
    def check(self, value, path):
        if not isinstance(value, str):
            raise TraceFormatError(f"{path}: expected string, got {value!r}")
        return value


class _OneOf(_Node):
    """A value from a fixed set of literals."""

    def __init__(self, allowed, message):
        self.allowed, self.message = allowed, message

    def check(self, value, path):
        if value not in self.allowed:
            raise TraceFormatError(f"{path}: {self.message.format(got=value)}")
        return value


class _NonEmpty(_Node):
    def __init__(self, inner: "_Array", message: str):
        self.inner, self.message = inner, message

    def check(self, value, path):
        items = self.inner.check(value, path)
        if not items:
            raise TraceFormatError(f"{path}: {self.message}")
        return items


class _Resource(_Node):
    """A mapping rule's resource: a fixed non-negative id or the event field 'pid' / 'tid'."""

    def check(self, value, path):
        if isinstance(value, bool) or not (isinstance(value, int) or value in ("pid", "tid")):
            raise TraceFormatError(f"{path}: expected non-negative integer, 'pid' or 'tid'; got {value!r}")
        if isinstance(value, int) and value < 0:
            raise TraceFormatError(f"{path}: negative value {value}")
        return value


class _Micros(_Node):
    """Trace-event microseconds -> integer nanoseconds, exactly (integral floats accepted)."""

    def check(self, value, path):
        if isinstance(value, float) and not isinstance(value, bool):
            if not value.is_integer():
                raise TraceFormatError(f"{path}: fractional timestamp {value!r} (would require rounding)")
            value = int(value)
        if isinstance(value, bool) or not isinstance(value, int):
            raise TraceFormatError(f"{path}: expected number, got {value!r}")
        if value < 0:
            raise TraceFormatError(f"{path}: negative value {value}")
        return value * 1000


SCHEMA = _Object(
    ("version", _Const(FORMAT_VERSION, "unsupported version {got!r}"), True),
    ("time_unit", _Const("ns", "expected 'ns', got {got!r}"), True),
    ("hosts", _Array(_Object(
        ("rank", _UInt(), True),
        ("records", _Array(_Object(("state", _Enum(HostState), True), ("start", _UInt(), True),
                                   ("end", _UInt(), True))), True))), True),
    ("devices", _Array(_Object(
        ("id", _UInt(), True),
        ("owner_rank", _UInt(), False),
        ("records", _Array(_Object(("kind", _Enum(DeviceActivityKind), True), ("stream", _UInt(), False),
                                   ("start", _UInt(), True), ("end", _UInt(), True))), True))), True),
)


def _parse_py(data) -> Trace:
    doc = SCHEMA.check(_load(data), "$")
    hosts, devices = doc["hosts"], doc["devices"]
    return Trace(
        host_processes=tuple(h["rank"] for h in hosts),
        devices=tuple(DeviceDecl(d["id"], d["owner_rank"]) for d in devices),
        host_records=tuple(HostRecord(h["rank"], r["state"], Interval(r["start"], r["end"]))
                           for h in hosts for r in h["records"]),
        device_records=tuple(DeviceRecord(d["id"], r["kind"], Interval(r["start"], r["end"]), r["stream"])
                             for d in devices for r in d["records"]))


# ---------------------------------------------------------------------------
# native parse
# ---------------------------------------------------------------------------
class _View(C.Structure):
    _fields_ = [("n_hosts", C.c_int64), ("n_devices", C.c_int64), ("n_host_records", C.c_int64),
                ("n_dev_records", C.c_int64), ("host_rank", C.c_void_p), ("host_off", C.c_void_p),
                ("dev_id", C.c_void_p), ("dev_owner", C.c_void_p), ("dev_off", C.c_void_p),
                ("h_kind", C.c_void_p), ("h_start", C.c_void_p), ("h_end", C.c_void_p),
                ("d_kind", C.c_void_p), ("d_stream", C.c_void_p), ("d_start", C.c_void_p),
                ("d_end", C.c_void_p)]


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    ct = np.ctypeslib.as_ctypes_type(dtype)
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), shape=(n,)).copy()


def _native_parse(data: bytes, nthreads: int | None):
    """dict of numpy columns (file order), or None when the fast path must defer."""
    lib = N.load()
    if isinstance(data, str):
        data = data.encode("utf-8")
    handle = C.c_void_p()
    off = C.c_int64(-1)
    rc = lib.heteff_parse_trace(data, len(data), nthreads or os.cpu_count() or 1, C.byref(handle), C.byref(off))
    if rc == N.PARSE_FALLBACK:
        return None
    if rc != N.OK:
        raise N.NativeError(f"trace parser failed ({rc})")
    try:
        v = _View()
        lib.heteff_parsed_info(handle, C.addressof(v))
        nh, nd, hk, dk = v.n_hosts, v.n_devices, v.n_host_records, v.n_dev_records
        return {
            "host_rank": _arr(v.host_rank, nh, np.uint64), "host_off": _arr(v.host_off, nh + 1, np.int64),
            "dev_id": _arr(v.dev_id, nd, np.uint64), "dev_owner": _arr(v.dev_owner, nd, np.int64),
            "dev_off": _arr(v.dev_off, nd + 1, np.int64),
            "h_kind": _arr(v.h_kind, hk, np.uint8), "h_start": _arr(v.h_start, hk, np.uint64),
            "h_end": _arr(v.h_end, hk, np.uint64),
            "d_kind": _arr(v.d_kind, dk, np.uint8), "d_stream": _arr(v.d_stream, dk, np.int64),
            "d_start": _arr(v.d_start, dk, np.uint64), "d_end": _arr(v.d_end, dk, np.uint64),
        }
    finally:
        lib.heteff_parsed_free(handle)


def read_trace(data, nthreads: int | None = None) -> Trace:
    """Parse a native trace document into a :class:`Trace` (drop-in for ``trace_io.py:96-158``)."""
    cols = _native_parse(data if isinstance(data, (bytes, str)) else bytes(data), nthreads)
    if cols is None:
        return _parse_py(data)
    ranks = cols["host_rank"].tolist()
    ids, owners = cols["dev_id"].tolist(), cols["dev_owner"].tolist()
    decls = [DeviceDecl(d, None if o < 0 else o) for d, o in zip(ids, owners)]
    hres = np.repeat(cols["host_rank"], np.diff(cols["host_off"]))
    dres = np.repeat(cols["dev_id"], np.diff(cols["dev_off"]))
    hrecs = _records(HostRecord, "rank", "state", _HOST_CODE_STATE, hres, cols["h_kind"], cols["h_start"],
                     cols["h_end"])
    drecs = _records(DeviceRecord, "device_id", "kind", _DEV_CODE_KIND, dres, cols["d_kind"], cols["d_start"],
                     cols["d_end"], cols["d_stream"])
    return Trace(host_processes=tuple(ranks), devices=tuple(decls), host_records=tuple(hrecs),
                 device_records=tuple(drecs))


try:   # native record builder (csrc/pack.c); the Python loop below is the same construction
    from . import _pack
except ImportError:
    _pack = None


def _records(cls, res_name, kind_name, members, res, kinds, starts, ends, streams=None):
    """Record objects from native columns: ``cls(res, members[kind], Interval(start, end)[, stream])``
    with ``stream`` < 0 -> None (what the reference's reader builds, ``trace_io.py:96-158``)."""
    if _pack is not None and (res.size == 0 or int(res.max()) < 2 ** 63):
        c = lambda a, t: np.ascontiguousarray(a, dtype=t)   # noqa: E731
        return _pack.make_records(cls, Interval, res_name, kind_name, tuple(members), c(res, np.int64),
                                  c(kinds, np.uint8), c(starts, np.uint64), c(ends, np.uint64),
                                  "stream" if cls is DeviceRecord else None,
                                  None if streams is None else c(streams, np.int64))
    out = []
    for j, (r, kd, a, b) in enumerate(zip(res.tolist(), kinds.tolist(), starts.tolist(), ends.tolist())):
        if streams is None:
            out.append(cls(r, members[kd], Interval(a, b)))
        else:
            st = int(streams[j])
            out.append(cls(r, members[kd], Interval(a, b), None if st < 0 else st))
    return out


def _dense_ids(declared: np.ndarray):
    ids, first = np.unique(declared, return_index=True)
    # declaration position of each distinct id (first occurrence, in declaration order)
    order = np.argsort(first, kind="stable")
    pos = np.empty(ids.size, dtype=np.int32)
    pos[order] = np.arange(ids.size, dtype=np.int32)
    return ids, pos


def _is_sorted(keys) -> bool:
    """Lexicographic non-decreasing order of the rows of ``keys`` (most significant first)."""
    if keys[0].size < 2:
        return True
    gt = np.zeros(keys[0].size - 1, dtype=bool)    # strictly greater on an earlier key
    eq = np.ones(keys[0].size - 1, dtype=bool)     # equal on all earlier keys
    for k in keys:
        a, b = k[:-1], k[1:]
        if np.any(eq & (b < a)):
            return False
        gt |= eq & (b > a)
        eq &= b == a
    return True


def read_trace_packed(data, nthreads: int | None = None):
    """Parse straight into a :class:`~.packing.PackedTrace` in canonical order plus the
    device owner table (dense host ids, -1 none) -- no Python record objects.

    Returns ``(packed, dev_owner)``."""
    cols = _native_parse(data if isinstance(data, (bytes, str)) else bytes(data), nthreads)
    if cols is None:
        from .packing import dev_owner_table

        t = _parse_py(data)
        p = pack_trace(t)
        return p, dev_owner_table(t, p)
    hr_ids, h_pos = _dense_ids(cols["host_rank"])
    d_ids, d_pos = _dense_ids(cols["dev_id"])
    nh, nd = cols["host_rank"].size, cols["dev_id"].size
    # records inherit their entry's dense id
    h_entry_dense = np.searchsorted(hr_ids, cols["host_rank"]).astype(np.int32)
    d_entry_dense = np.searchsorted(d_ids, cols["dev_id"]).astype(np.int32)
    h_res = np.repeat(h_entry_dense, np.diff(cols["host_off"]))
    d_res = np.repeat(d_entry_dense, np.diff(cols["dev_off"]))
    # canonical order (model.py:74-80): host (rank, start, end, state value: mpi < offload < useful),
    # device (device, start, end, kind value: kernel < memory, stream or -1)
    state_rank = np.array([2, 1, 0], dtype=np.uint8)[cols["h_kind"]]
    hkeys = (h_res, cols["h_start"], cols["h_end"], state_rank)
    dkeys = (d_res, cols["d_start"], cols["d_end"], cols["d_kind"], cols["d_stream"])
    # writer output is already canonical when entries come in id order: check in O(n), sort otherwise
    ho = None if _is_sorted(hkeys) else np.lexsort(hkeys[::-1])
    do = None if _is_sorted(dkeys) else np.lexsort(dkeys[::-1])

    def take(a, o):
        return a if o is None else a[o]

    host = RecordColumns(take(cols["h_start"], ho), take(cols["h_end"], ho), take(h_res, ho),
                         take(cols["h_kind"], ho))
    dev = RecordColumns(take(cols["d_start"], do), take(cols["d_end"], do), take(d_res, do),
                        take(cols["d_kind"], do))
    packed = PackedTrace(host, dev, hr_ids.tolist(), d_ids.tolist(), h_pos, d_pos, nh, nd,
                         int(hr_ids.size), int(d_ids.size))
    # owners: the first declaration of each device id; owner must be a declared rank
    owner = np.full(d_ids.size, -1, dtype=np.int32)
    first_decl = np.unique(cols["dev_id"], return_index=True)[1]
    o = cols["dev_owner"][first_decl]
    ok = o >= 0
    if ok.any():
        idx = np.searchsorted(hr_ids, o[ok].astype(np.uint64))
        found = (idx < hr_ids.size) & (hr_ids[np.minimum(idx, hr_ids.size - 1)] == o[ok].astype(np.uint64)) \
            if hr_ids.size else np.zeros(idx.size, dtype=bool)
        tmp = np.full(ok.sum(), -1, dtype=np.int32)
        tmp[found] = idx[found]
        owner[np.nonzero(ok)[0]] = tmp
    return packed, owner


# ---------------------------------------------------------------------------
# Chrome-trace-event import with mapping rules (trace_io.py:196-342)
# ---------------------------------------------------------------------------
from dataclasses import dataclass  # noqa: E402

_MATCH_KEYS = ("name_contains", "name_equals", "category_contains", "category_equals")
_MODES = {"contains": lambda subject, pattern: pattern in subject,
          "equals": lambda subject, pattern: pattern == subject}
_TARGET_CODE = {HostState.USEFUL: 0, HostState.OFFLOAD: 1, HostState.MPI: 2,
                DeviceActivityKind.KERNEL: 3, DeviceActivityKind.MEMORY: 4}


class MappingError(Exception):
    """Import failed under default_policy=error: events matched no rule."""


@dataclass(frozen=True)
class MappingRule:
    """One importer rule; the first matching rule in the list wins."""

    field: str        # "name" | "category"
    mode: str         # "contains" | "equals"
    pattern: str
    target: object    # HostState | DeviceActivityKind
    resource: object  # fixed id, or "pid" / "tid"

    def matches(self, name: str, category: str) -> bool:
        return _MODES[self.mode]({"name": name, "category": category}[self.field], self.pattern)


@dataclass(frozen=True)
class CategoryMapping:
    rules: tuple
    default_policy: str   # "drop" | "error"


def _load_named(data, what):
    if isinstance(data, bytes):
        try:
            data = data.decode("utf-8")
        except UnicodeDecodeError as e:
            raise TraceFormatError(f"{what} is not UTF-8: {e}") from e
    try:
        return json.loads(data)
    except json.JSONDecodeError as e:
        raise TraceFormatError(f"{what} is not valid JSON: {e}") from e


class _MatchRule(_Node):
    """One mapping rule (docs/formats.md:87-132): exactly one match key, then its pattern,
    the target state / kind and the resource, then no other field."""

    TARGET = None   # set below (needs the enums)

    def check(self, value, path):
        if not isinstance(value, dict):
            raise TraceFormatError(f"{path}: expected object, got {type(value).__name__}")
        keys = [k for k in _MATCH_KEYS if k in value]
        if len(keys) != 1:
            raise TraceFormatError(f"{path}: exactly one of {', '.join(_MATCH_KEYS)} is required")
        key = keys[0]
        got = _Object((key, _Str(), True), ("target", self.TARGET, True),
                      ("resource", _Resource(), True)).check(value, path)
        subject, mode = key.rsplit("_", 1)
        return MappingRule(subject, mode, got[key], got["target"], got["resource"])


_MatchRule.TARGET = _Enum(list(HostState) + list(DeviceActivityKind))
MAPPING_SCHEMA = _Object(
    ("default_policy", _OneOf(("drop", "error"), "expected 'drop' or 'error', got {got!r}"), True),
    ("rules", _NonEmpty(_Array(_MatchRule()), "at least one rule is required"), True),
)


def read_mapping(data) -> CategoryMapping:
    """Parse a mapping document (``trace_io.py:222-260``, ``docs/formats.md:87-132``)."""
    doc = MAPPING_SCHEMA.check(_load_named(data, "mapping document"), "$")
    return CategoryMapping(tuple(doc["rules"]), doc["default_policy"])


def _assemble(hrecs, drecs, unmapped, mapping):
    if unmapped and mapping.default_policy == "error":
        shown = "; ".join(f"event {i} ({nm!r})" for i, nm in unmapped[:10])
        more = f" (+{len(unmapped) - 10} more)" if len(unmapped) > 10 else ""
        raise MappingError(f"{len(unmapped)} event(s) matched no rule: {shown}{more}")
    warnings = [] if mapping.default_policy == "error" else \
        [f"dropped unmapped event {i} ({nm!r})" for i, nm in unmapped]
    trace = Trace(host_processes=tuple(sorted({r.rank for r in hrecs})),
                  devices=tuple(DeviceDecl(d) for d in sorted({r.device_id for r in drecs})),
                  host_records=tuple(hrecs), device_records=tuple(drecs))
    return trace, warnings


_MICROS = _Micros()


def _import_py(data, mapping):
    """The strict event importer (error texts, unusual legal documents): complete spans
    ("ph": "X") only, first matching rule wins, unmatched events reported by index."""
    doc = _load_named(data, "events document")
    if isinstance(doc, dict):
        events = _Array(_Pass()).check(doc.get("traceEvents"), "$.traceEvents")
    else:
        events = _Array(_Pass()).check(doc, "$")
    hrecs, drecs, unmapped = [], [], []
    for i, ev in enumerate(events):
        if not (isinstance(ev, dict) and ev.get("ph") == "X"):
            continue
        path = f"$[{i}]"
        name = _Str().check(ev.get("name"), f"{path}.name")
        cat = _Str().check(ev.get("cat", ""), f"{path}.cat")
        missing = [k for k in ("ts", "dur") if k not in ev]
        if missing:
            raise TraceFormatError(f"{path}: missing required field {missing[0]!r}")
        start = _MICROS.check(ev["ts"], f"{path}.ts")
        end = start + _MICROS.check(ev["dur"], f"{path}.dur")
        rule = next((r for r in mapping.rules if r.matches(name, cat)), None)
        if rule is None:
            unmapped.append((i, name))
            continue
        res = rule.resource
        if not isinstance(res, int):
            res = _UInt().check(ev.get(res), f"{path}.{res}")
        if isinstance(rule.target, HostState):
            hrecs.append(HostRecord(res, rule.target, Interval(start, end)))
        else:
            drecs.append(DeviceRecord(res, rule.target, Interval(start, end)))
    return _assemble(hrecs, drecs, unmapped, mapping)


class _Rule(C.Structure):
    _fields_ = [("field", C.c_int32), ("mode", C.c_int32), ("pattern", C.c_char_p), ("pattern_len", C.c_int64),
                ("target", C.c_int32), ("reserved", C.c_int32), ("resource", C.c_int64)]


class _IView(C.Structure):
    _fields_ = [("n_records", C.c_int64), ("n_unmapped", C.c_int64), ("is_dev", C.c_void_p), ("kind", C.c_void_p),
                ("res", C.c_void_p), ("start", C.c_void_p), ("end", C.c_void_p), ("unmapped", C.c_void_p),
                ("name_off", C.c_void_p), ("name_len", C.c_void_p)]


def import_mapped(data, mapping: CategoryMapping, nthreads: int | None = None, columns: bool = False):
    """Chrome-trace events -> (Trace, warnings) (drop-in for ``trace_io.py:263-342``)."""
    raw = data.encode("utf-8") if isinstance(data, str) else bytes(data)
    lib = N.load()
    pats = [r.pattern.encode("utf-8") for r in mapping.rules]
    rules = (_Rule * max(len(pats), 1))()
    for q, (r, pb) in enumerate(zip(mapping.rules, pats)):
        res = r.resource if isinstance(r.resource, int) else (-1 if r.resource == "pid" else -2)
        rules[q] = _Rule(0 if r.field == "name" else 1, 0 if r.mode == "contains" else 1, pb, len(pb),
                         _TARGET_CODE[r.target], 0, res)
    handle = C.c_void_p()
    off = C.c_int64(-1)
    rc = lib.heteff_import_events(raw, len(raw), rules, len(pats), nthreads or os.cpu_count() or 1,
                                  C.byref(handle), C.byref(off))
    if rc == N.PARSE_FALLBACK:
        return _import_py(data, mapping)
    if rc != N.OK:
        raise N.NativeError(f"event importer failed ({rc})")
    try:
        v = _IView()
        lib.heteff_imported_info(handle, C.addressof(v))
        k, u = v.n_records, v.n_unmapped
        is_dev = _arr(v.is_dev, k, np.uint8)
        kind = _arr(v.kind, k, np.uint8)
        res = _arr(v.res, k, np.uint64)
        st = _arr(v.start, k, np.uint64)
        en = _arr(v.end, k, np.uint64)
        um = _arr(v.unmapped, u, np.int64).tolist()
        no = _arr(v.name_off, u, np.int64).tolist()
        nl = _arr(v.name_len, u, np.int64).tolist()
    finally:
        lib.heteff_imported_free(handle)
    if columns:
        return (is_dev, kind, res, st, en), [(i, raw[o:o + n].decode("utf-8")) for i, o, n in zip(um, no, nl)]
    h, d = is_dev == 0, is_dev == 1
    hrecs = _records(HostRecord, "rank", "state", _HOST_CODE_STATE, res[h], kind[h], st[h], en[h])
    drecs = _records(DeviceRecord, "device_id", "kind", _DEV_CODE_KIND, res[d], kind[d], st[d], en[d])
    unmapped = [(i, raw[o:o + n].decode("utf-8")) for i, o, n in zip(um, no, nl)]
    return _assemble(hrecs, drecs, unmapped, mapping)


def _host_item(rec) -> dict:
    return {"state": rec.state.value, "start": rec.interval.start, "end": rec.interval.end}


def _device_item(rec) -> dict:
    stream = {} if rec.stream is None else {"stream": rec.stream}
    return {"kind": rec.kind.value, **stream, "start": rec.interval.start, "end": rec.interval.end}


def _grouped(records, key, declared, what):
    """Records grouped by resource in declaration order; a record of an undeclared
    resource is a ValueError (the document could not be read back)."""
    groups = {k: [] for k in declared}
    for rec in records:
        k = key(rec)
        if k not in groups:
            raise ValueError(f"{what} {k}")
        groups[k].append(rec)
    return groups


def write_trace(trace: Trace) -> bytes:
    """Deterministic native document (``trace_io.py:161-193``, docs/formats.md:9-85): equal
    traces give equal bytes -- keys in schema order, two-space indent, final newline."""
    hosts = _grouped(trace.host_records, lambda r: r.rank, trace.host_processes,
                     "host record references undeclared rank")
    devs = _grouped(trace.device_records, lambda r: r.device_id, [d.device_id for d in trace.devices],
                    "device record references undeclared device")
    doc = {
        "version": FORMAT_VERSION,
        "time_unit": "ns",
        "hosts": [{"rank": r, "records": [_host_item(x) for x in hosts[r]]} for r in trace.host_processes],
        "devices": [{"id": d.device_id, **({} if d.owner_rank is None else {"owner_rank": d.owner_rank}),
                     "records": [_device_item(x) for x in devs[d.device_id]]} for d in trace.devices],
    }
    return (json.dumps(doc, indent=2) + "\n").encode("utf-8")


def import_mapped_packed(data, mapping: CategoryMapping, nthreads: int | None = None):
    """Chrome-trace events straight into a :class:`~.packing.PackedTrace` (no Python record
    objects): the imported trace declares exactly the ranks and devices that received
    records (``trace_io.py:333-341``), in id order.  Returns ``(packed, warnings)``."""
    raw = data.encode("utf-8") if isinstance(data, str) else bytes(data)
    out = import_mapped(raw, mapping, nthreads, columns=True)
    if isinstance(out[0], Trace):   # the strict fallback decided it
        t, w = out
        return pack_trace(t), w
    (is_dev, kind, res, st, en), unmapped = out
    _, warnings = _assemble([], [], unmapped, mapping)   # MappingError / warnings exactly as the reference
    h, d = is_dev == 0, is_dev == 1
    h_ids, h_dense = np.unique(res[h], return_inverse=True)
    d_ids, d_dense = np.unique(res[d], return_inverse=True)
    h_res, d_res = h_dense.astype(np.int32), d_dense.astype(np.int32)
    state_rank = np.array([2, 1, 0], dtype=np.uint8)[kind[h]] if h.any() else np.zeros(0, np.uint8)
    ho = np.lexsort((state_rank, en[h], st[h], h_res))
    do = np.lexsort((kind[d], en[d], st[d], d_res))
    host = RecordColumns(st[h][ho], en[h][ho], h_res[ho], kind[h][ho])
    dev = RecordColumns(st[d][do], en[d][do], d_res[do], kind[d][do])
    nh, nd = int(h_ids.size), int(d_ids.size)
    packed = PackedTrace(host, dev, h_ids.tolist(), d_ids.tolist(), np.arange(nh, dtype=np.int32),
                         np.arange(nd, dtype=np.int32), nh, nd, nh, nd)
    return packed, warnings
