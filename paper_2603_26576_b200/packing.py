"""Ingest: turn a :class:`~.model.Trace` (or raw columns) into the packed SoA.

The engine reads five columns per record set (include/heteff_b200.h):
``start u64``, ``end u64``, ``res i32`` (dense resource id), ``kind u8``.
Dense ids are assigned in ascending order of the reference's rank / device
id, so the reference's canonical order (``model.py:74-80,99-107``) is also
"sorted by (res, start)" -- the contract the scan kernels check per record.
``decl[id]`` maps a dense id to its declaration position, ``-1`` when the id
is used by records but never declared (an error the kernels report).

Records whose timestamps cannot be represented as u64 at all (non-int,
negative, > 2**64-1) cannot enter the SoA; this is the type check every
typed ingest does (the reference's ``trace_io._nonneg_int`` rejects them at
parse time too).  They are kept out of the columns, and their reference
messages (``model.py:140-157``) are produced here from the record's own
values -- see :class:`Quarantined`.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from operator import attrgetter

import numpy as np

from .model import DEVICE_KIND_CODE, HOST_STATE_CODE, U64_MAX, Trace


@dataclass
class Quarantined:
    """A record whose timestamps are outside the u64 domain."""

    index: int            # canonical position in trace.host_records / device_records
    errors: list[str]     # messages in reference order (model.py:143-156)
    warnings: list[str]


@dataclass
class RecordColumns:
    start: np.ndarray     # uint64
    end: np.ndarray       # uint64
    res: np.ndarray       # int32 dense ids, non-decreasing
    kind: np.ndarray      # uint8
    index: np.ndarray | None = None   # SoA position -> canonical position (None = identity)

    @property
    def count(self) -> int:
        return int(self.start.shape[0])


@dataclass
class PackedTrace:
    host: RecordColumns
    dev: RecordColumns
    host_ids: list            # dense id -> reference rank id
    dev_ids: list             # dense id -> reference device id
    host_decl: np.ndarray     # int32 [len(host_ids)]: first declaration position or -1
    dev_decl: np.ndarray
    n: int                    # trace.n (declarations, duplicates included)
    m: int
    n_unique: int
    m_unique: int
    host_q: list[Quarantined] = field(default_factory=list)
    dev_q: list[Quarantined] = field(default_factory=list)
    host_elapsed_floor: int = 0   # max end of quarantined host records, clipped to u64


def _interval_domain_messages(where: str, start, end) -> tuple[bool, list[str], list[str]]:
    """(representable, errors, warnings) for one interval, reference order."""
    if not isinstance(start, int) or not isinstance(end, int):
        return False, [f"{where}: timestamps must be integers"], []
    if 0 <= start <= U64_MAX and 0 <= end <= U64_MAX:
        return True, [], []
    errs: list[str] = []
    warns: list[str] = []
    if start < 0:
        errs.append(f"{where}: negative timestamp {start}")
    if end > U64_MAX:
        errs.append(f"{where}: end {end} exceeds 64-bit range")
    if start > end:
        errs.append(f"{where}: start {start} > end {end}")
    elif start == end:
        warns.append(f"{where}: zero-length interval at {start}")
    return False, errs, warns


def _dense(declared, used):
    ids = sorted(set(declared) | set(used))
    return ids, {rid: i for i, rid in enumerate(ids)}


def _decl_table(ids, declared) -> tuple[np.ndarray, int]:
    first: dict = {}
    for pos, rid in enumerate(declared):
        first.setdefault(rid, len(first))
    table = np.full(len(ids), -1, dtype=np.int32)
    for i, rid in enumerate(ids):
        if rid in first:
            table[i] = first[rid]
    return table, len(first)


try:   # one-pass native packer (csrc/pack.c), built in-tree by __graft_entry__.build()
    from . import _pack
except ImportError:   # host-side ingest only: the Python packer below is the same mapping
    _pack = None


def _members(codes: dict) -> tuple:
    out = [None] * (max(codes.values()) + 1)
    for member, code in codes.items():
        out[code] = member
    return tuple(out)


_HOST_MEMBERS = _members(HOST_STATE_CODE)
_DEV_MEMBERS = _members(DEVICE_KIND_CODE)


def _pack_side(records, res_of, code_of, dense, label, res_label, native=None):
    k = len(records)
    if _pack is not None and native is not None and k:
        cols = (np.empty(k, np.uint64), np.empty(k, np.uint64), np.empty(k, np.int32), np.empty(k, np.uint8))
        if _pack.pack_side(records, native[0], native[1], dense, native[2], *cols):
            return RecordColumns(*cols, None), [], 0
    try:  # fast path: every timestamp is a plain in-range int
        if all(type(r.interval.start) is int and type(r.interval.end) is int for r in records):
            start = np.fromiter((r.interval.start for r in records), dtype=np.uint64, count=k)
            end = np.fromiter((r.interval.end for r in records), dtype=np.uint64, count=k)
            res = np.fromiter((dense[res_of(r)] for r in records), dtype=np.int32, count=k)
            kind = np.fromiter((code_of(r) for r in records), dtype=np.uint8, count=k)
            return RecordColumns(start, end, res, kind, None), [], 0
    except OverflowError:
        pass
    start = np.empty(k, dtype=np.uint64)
    end = np.empty(k, dtype=np.uint64)
    res = np.empty(k, dtype=np.int32)
    kind = np.empty(k, dtype=np.uint8)
    quarantined: list[Quarantined] = []
    keep = []
    floor = 0
    w = 0
    for i, rec in enumerate(records):
        iv = rec.interval
        s, e = iv.start, iv.end
        if (type(s) is int and type(e) is int and 0 <= s <= U64_MAX and 0 <= e <= U64_MAX):
            start[w] = s
            end[w] = e
            res[w] = dense[res_of(rec)]
            kind[w] = code_of(rec)
            keep.append(i)
            w += 1
            continue
        where = f"{label} record {i} ({res_label} {res_of(rec)})"
        ok, errs, warns = _interval_domain_messages(where, s, e)
        if ok:  # bool subclasses of int: representable after all
            start[w] = int(s)
            end[w] = int(e)
            res[w] = dense[res_of(rec)]
            kind[w] = code_of(rec)
            keep.append(i)
            w += 1
            continue
        quarantined.append(Quarantined(i, errs, warns))
        if isinstance(e, int) and e > 0:
            floor = max(floor, min(e, U64_MAX))
    index = None
    if quarantined:
        start, end, res, kind = start[:w], end[:w], res[:w], kind[:w]
        index = np.asarray(keep, dtype=np.int64)
    return RecordColumns(start, end, res, kind, index), quarantined, floor


def pack_trace(trace: Trace) -> PackedTrace:
    """Pack a :class:`Trace` into SoA columns in canonical order."""
    hp = trace.host_processes
    dev_decl_ids = [d.device_id for d in trace.devices]
    host_ids, hdense = _dense(hp, map(attrgetter("rank"), trace.host_records))
    dev_ids, ddense = _dense(dev_decl_ids, map(attrgetter("device_id"), trace.device_records))
    host_decl, n_unique = _decl_table(host_ids, hp)
    dev_decl, m_unique = _decl_table(dev_ids, dev_decl_ids)
    host, host_q, floor = _pack_side(
        trace.host_records, lambda r: r.rank, lambda r: HOST_STATE_CODE[r.state],
        hdense, "host", "rank", ("rank", "state", _HOST_MEMBERS))
    dev, dev_q, _ = _pack_side(
        trace.device_records, lambda r: r.device_id, lambda r: DEVICE_KIND_CODE[r.kind],
        ddense, "device", "device", ("device_id", "kind", _DEV_MEMBERS))
    return PackedTrace(host, dev, host_ids, dev_ids, host_decl, dev_decl,
                       trace.n, trace.m, n_unique, m_unique, host_q, dev_q, floor)


def columns(start, end, res, kind) -> RecordColumns:
    """Wrap caller arrays (already canonical) as :class:`RecordColumns`."""
    return RecordColumns(np.ascontiguousarray(start, dtype=np.uint64),
                         np.ascontiguousarray(end, dtype=np.uint64),
                         np.ascontiguousarray(res, dtype=np.int32),
                         np.ascontiguousarray(kind, dtype=np.uint8))


def dev_owner_table(trace: Trace, packed: PackedTrace) -> np.ndarray:
    """int32 [len(dev_ids)]: dense host id of each device's ``owner_rank``, -1 when it
    has none or the owner is not a declared rank (``DeviceDecl.owner_rank``, model.py:66-71)."""
    host_dense = {rank: i for i, rank in enumerate(packed.host_ids)}
    declared = set(trace.host_processes)
    owner_of = {}
    for d in trace.devices:
        owner_of.setdefault(d.device_id, d.owner_rank)
    out = np.full(len(packed.dev_ids), -1, dtype=np.int32)
    for i, dev in enumerate(packed.dev_ids):
        o = owner_of.get(dev)
        if o is not None and o in declared and o in host_dense:
            out[i] = host_dense[o]
    return out
