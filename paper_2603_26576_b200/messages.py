"""Reference-exact validation / clamp messages from engine findings.

The kernels report *which* records are malformed, zero-length, undeclared,
overlapping or late (as SoA positions); this module only turns those index
lists into the reference's strings, in the reference's order
(``model.py:160-230``, ``summarize.py:133-137``).  Declaration-level checks
(no resources, duplicate ids, time unit, unknown owner ranks) are metadata
checks on the ``Trace`` object, ``model.py:173-189``.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .engine import Findings, overlap_covers
from .model import Trace, ValidationReport
from .packing import PackedTrace


def declaration_messages(trace: Trace) -> tuple[list[str], list[str]]:
    errors: list[str] = []
    warnings: list[str] = []
    if trace.n == 0 and trace.m == 0:
        errors.append("trace declares no host processes and no devices")
    if len(set(trace.host_processes)) != trace.n:
        errors.append("duplicate rank ids in host_processes")
    if len({d.device_id for d in trace.devices}) != trace.m:
        errors.append("duplicate device ids in devices")
    if trace.time_unit != "ns":
        errors.append(f"unsupported time unit {trace.time_unit!r}")
    ranks = set(trace.host_processes)
    for d in trace.devices:
        if d.owner_rank is not None and d.owner_rank not in ranks:
            warnings.append(f"device {d.device_id}: owner_rank {d.owner_rank} is not a declared rank")
    return errors, warnings


def _canon(pos: np.ndarray, index: np.ndarray | None) -> list[int]:
    if index is None:
        return [int(x) for x in pos]
    return [int(index[x]) for x in pos]


def _after(end, host_elapsed) -> bool:
    """``end > host_elapsed`` as the reference evaluates it (model.py:224); ends the
    reference itself cannot compare are not late."""
    try:
        return bool(end > host_elapsed)
    except TypeError:
        return False


def _record_events(records, label: str, res_label: str, res_of, declared: set, f: Findings, packed_cols,
                   quarantined, cls_malformed: int, cls_zero: int, cls_undecl: int, cls_late: int | None,
                   host_elapsed, late: list[int] | None = None):
    """(errors, warnings) as lists of (canonical index, order, text).

    ``late``: canonical indices of device records ending after ``host_elapsed``, when the
    caller had to decide them itself (quarantined host records), else None."""
    errs: list[tuple[int, int, str]] = []
    warns: list[tuple[int, int, str]] = []
    index = packed_cols.index

    def where(i):
        return f"{label} record {i} ({res_label} {res_of(records[i])})"

    for i in _canon(f.lists[cls_malformed], index):
        iv = records[i].interval
        errs.append((i, 0, f"{where(i)}: start {iv.start} > end {iv.end}"))
    for i in _canon(f.lists[cls_zero], index):
        warns.append((i, 0, f"{where(i)}: zero-length interval at {records[i].interval.start}"))
    for i in _canon(f.lists[cls_undecl], index):
        errs.append((i, 1, f"{where(i)}: {res_label if res_label == 'device' else 'rank'} not declared"))
    if cls_late is not None:
        if late is None:   # the kernel's list (in-domain records) + quarantined records
            late = _canon(f.lists[cls_late], index)
            late += [q.index for q in quarantined if _after(records[q.index].interval.end, host_elapsed)]
        for i in late:
            warns.append((i, 1, f"{where(i)}: ends at {records[i].interval.end}, after host elapsed time "
                                f"{host_elapsed}; it will be clamped"))
    for q in quarantined:
        for t in q.errors:
            errs.append((q.index, 0, t))
        for t in q.warnings:
            warns.append((q.index, 0, t))
        if res_of(records[q.index]) not in declared:
            errs.append((q.index, 1, f"{where(q.index)}: {res_label if res_label == 'device' else 'rank'} not declared"))
    # stable: per record, interval findings (order 0) before declaration findings (order 1)
    errs.sort(key=lambda x: (x[0], x[1]))
    warns.sort(key=lambda x: (x[0], x[1]))
    return errs, warns


def validation_report(trace: Trace, packed: PackedTrace, f: Findings) -> ValidationReport:
    """Rebuild ``validate(trace)`` exactly from the engine's findings."""
    errors, warnings = declaration_messages(trace)
    ranks = set(trace.host_processes)
    devs = {d.device_id for d in trace.devices}
    h_err, h_warn = _record_events(trace.host_records, "host", "rank", lambda r: r.rank, ranks, f, packed.host,
                                   packed.host_q, N.HOST_MALFORMED, N.HOST_ZERO, N.HOST_UNDECLARED, None, 0)
    errors += [t for _, _, t in h_err]
    warnings += [t for _, _, t in h_warn]
    # overlaps (model.py:203-215): grouped by rank in declaration order
    ovl = f.lists[N.HOST_OVERLAP]
    if len(ovl):
        cover = overlap_covers(packed, ovl)
        idx = packed.host.index
        by_rank: dict = {}
        for pos, cpos in zip(ovl.tolist(), cover.tolist()):
            i = int(idx[pos]) if idx is not None else pos
            c = int(idx[cpos]) if idx is not None else cpos
            by_rank.setdefault(trace.host_records[i].rank, []).append((i, c))
        for rank in trace.host_processes:
            for i, c in sorted(by_rank.get(rank, ())):
                a, b = trace.host_records[c].interval, trace.host_records[i].interval
                errors.append(f"rank {rank}: host records {c} and {i} overlap: "
                              f"[{a.start}, {a.end}) and [{b.start}, {b.end})")
    # model.py:217-228: late device records, only when ranks are declared.  The kernel compares
    # in-domain records against the max in-domain host end; a quarantined host record (its end
    # outside u64 or not an int) moves the reference's host elapsed, so then the comparison is
    # made here, on the unclipped values, for every device record.
    host_elapsed, late = f.host_elapsed, None
    if trace.n >= 1 and packed.host_q:
        host_elapsed = max((r.interval.end for r in trace.host_records), default=0)
        late = [i for i, r in enumerate(trace.device_records) if _after(r.interval.end, host_elapsed)]
    d_err, d_warn = _record_events(trace.device_records, "device", "device", lambda r: r.device_id, devs, f,
                                   packed.dev, packed.dev_q, N.DEV_MALFORMED, N.DEV_ZERO, N.DEV_UNDECLARED,
                                   N.DEV_LATE if trace.n >= 1 else None, host_elapsed, late)
    errors += [t for _, _, t in d_err]
    warnings += [t for _, _, t in d_warn]
    return ValidationReport(errors, warnings)


def clamp_warnings(trace: Trace, f: Findings, elapsed: int) -> list[str]:
    """``summarize.py:133-137``: one warning per device with clamped records."""
    out = []
    for pos, d in enumerate(_unique_devices(trace)):
        clamped = int(f.dev_sum[pos][3]) if pos < len(f.dev_sum) else 0
        if clamped:
            out.append(f"device {d}: clamped {clamped} record(s) extending beyond elapsed time {elapsed}")
    return out


def _unique_devices(trace: Trace) -> list:
    seen: dict = {}
    for d in trace.devices:
        seen.setdefault(d.device_id, None)
    return list(seen)
