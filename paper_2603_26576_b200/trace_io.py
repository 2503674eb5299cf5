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
_HOST_STATES = {s.value: s for s in HostState}
_DEVICE_KINDS = {k.value: k for k in DeviceActivityKind}
_HOST_CODE_STATE = (HostState.USEFUL, HostState.OFFLOAD, HostState.MPI)     # ingest codes 0, 1, 2
_DEV_CODE_KIND = (DeviceActivityKind.KERNEL, DeviceActivityKind.MEMORY)


class TraceFormatError(Exception):
    """A document does not conform to the native trace schema."""


# ---------------------------------------------------------------------------
# strict pure-Python reader: the error path (and unusual legal documents)
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


def _expect_obj(v, path):
    if not isinstance(v, dict):
        raise TraceFormatError(f"{path}: expected object, got {type(v).__name__}")
    return dict(v)


def _expect_list(v, path):
    if not isinstance(v, list):
        raise TraceFormatError(f"{path}: expected array, got {type(v).__name__}")
    return v


def _pop(d, path, key, required=True):
    if key not in d:
        if required:
            raise TraceFormatError(f"{path}: missing required field {key!r}")
        return None
    return d.pop(key)


def _done(d, path):
    if d:
        raise TraceFormatError(f"{path}: unknown field {sorted(d)[0]!r}")


def _uint(v, path):
    if isinstance(v, bool) or not isinstance(v, int):
        raise TraceFormatError(f"{path}: expected integer, got {v!r}")
    if v < 0:
        raise TraceFormatError(f"{path}: negative value {v}")
    return v


def _choice(v, table, path):
    if not isinstance(v, str) or v not in table:
        raise TraceFormatError(f"{path}: expected one of {', '.join(sorted(table))}; got {v!r}")
    return table[v]


def _parse_py(data) -> Trace:
    doc = _expect_obj(_load(data), "$")
    version = _pop(doc, "$", "version")
    if version != FORMAT_VERSION:
        raise TraceFormatError(f"$.version: unsupported version {version!r}")
    unit = _pop(doc, "$", "time_unit")
    if unit != "ns":
        raise TraceFormatError(f"$.time_unit: expected 'ns', got {unit!r}")
    hp, hrecs = [], []
    for i, entry in enumerate(_expect_list(_pop(doc, "$", "hosts"), "$.hosts")):
        path = f"$.hosts[{i}]"
        entry = _expect_obj(entry, path)
        rank = _uint(_pop(entry, path, "rank"), f"{path}.rank")
        hp.append(rank)
        for j, rec in enumerate(_expect_list(_pop(entry, path, "records"), f"{path}.records")):
            rp = f"{path}.records[{j}]"
            rec = _expect_obj(rec, rp)
            state = _choice(_pop(rec, rp, "state"), _HOST_STATES, f"{rp}.state")
            s = _uint(_pop(rec, rp, "start"), f"{rp}.start")
            e = _uint(_pop(rec, rp, "end"), f"{rp}.end")
            _done(rec, rp)
            hrecs.append(HostRecord(rank, state, Interval(s, e)))
        _done(entry, path)
    decls, drecs = [], []
    for i, entry in enumerate(_expect_list(_pop(doc, "$", "devices"), "$.devices")):
        path = f"$.devices[{i}]"
        entry = _expect_obj(entry, path)
        did = _uint(_pop(entry, path, "id"), f"{path}.id")
        owner = _pop(entry, path, "owner_rank", required=False)
        if owner is not None:
            owner = _uint(owner, f"{path}.owner_rank")
        decls.append(DeviceDecl(did, owner))
        for j, rec in enumerate(_expect_list(_pop(entry, path, "records"), f"{path}.records")):
            rp = f"{path}.records[{j}]"
            rec = _expect_obj(rec, rp)
            kind = _choice(_pop(rec, rp, "kind"), _DEVICE_KINDS, f"{rp}.kind")
            stream = _pop(rec, rp, "stream", required=False)
            if stream is not None:
                stream = _uint(stream, f"{rp}.stream")
            s = _uint(_pop(rec, rp, "start"), f"{rp}.start")
            e = _uint(_pop(rec, rp, "end"), f"{rp}.end")
            _done(rec, rp)
            drecs.append(DeviceRecord(did, kind, Interval(s, e), stream))
        _done(entry, path)
    _done(doc, "$")
    return Trace(host_processes=tuple(hp), devices=tuple(decls), host_records=tuple(hrecs),
                 device_records=tuple(drecs))


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
    hoff = cols["host_off"].tolist()
    hk, hs, he = cols["h_kind"].tolist(), cols["h_start"].tolist(), cols["h_end"].tolist()
    hrecs = []
    for i, r in enumerate(ranks):
        for j in range(hoff[i], hoff[i + 1]):
            hrecs.append(HostRecord(r, _HOST_CODE_STATE[hk[j]], Interval(hs[j], he[j])))
    ids, owners, doff = cols["dev_id"].tolist(), cols["dev_owner"].tolist(), cols["dev_off"].tolist()
    dk, dst, ds, de = cols["d_kind"].tolist(), cols["d_stream"].tolist(), cols["d_start"].tolist(), cols["d_end"].tolist()
    decls, drecs = [], []
    for i, d in enumerate(ids):
        decls.append(DeviceDecl(d, None if owners[i] < 0 else owners[i]))
        for j in range(doff[i], doff[i + 1]):
            drecs.append(DeviceRecord(d, _DEV_CODE_KIND[dk[j]], Interval(ds[j], de[j]),
                                      None if dst[j] < 0 else dst[j]))
    return Trace(host_processes=tuple(ranks), devices=tuple(decls), host_records=tuple(hrecs),
                 device_records=tuple(drecs))


def _dense_ids(declared: np.ndarray):
    ids, first = np.unique(declared, return_index=True)
    # declaration position of each distinct id (first occurrence, in declaration order)
    order = np.argsort(first, kind="stable")
    pos = np.empty(ids.size, dtype=np.int32)
    pos[order] = np.arange(ids.size, dtype=np.int32)
    return ids, pos


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
    ho = np.lexsort((state_rank, cols["h_end"], cols["h_start"], h_res))
    do = np.lexsort((cols["d_stream"], cols["d_kind"], cols["d_end"], cols["d_start"], d_res))
    host = RecordColumns(cols["h_start"][ho], cols["h_end"][ho], h_res[ho], cols["h_kind"][ho])
    dev = RecordColumns(cols["d_start"][do], cols["d_end"][do], d_res[do], cols["d_kind"][do])
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
