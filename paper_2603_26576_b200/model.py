"""Trace data model of the drop-in API.

Mirrors the reference's public types (``heteff/model.py:24-137``) name for
name, field for field, so code written against ``heteff`` runs unchanged:

* :class:`Interval` -- half-open ``[start, end)`` integer nanoseconds
  (``model.py:39-48``).
* :class:`HostState` / :class:`DeviceActivityKind` -- the recorded states
  (``model.py:24-36``); idle is derived, never recorded.
* :class:`HostRecord`, :class:`DeviceRecord`, :class:`DeviceDecl`
  (``model.py:51-71``).
* :class:`Trace` -- immutable; records are held in the reference's canonical
  order (``model.py:74-80,99-107``) because validation messages name records
  by their canonical position.
* :class:`ValidationReport`, :class:`InvalidTraceError` (``model.py:118-137``).

:func:`validate` itself lives in :mod:`.api` -- it runs on the GPU engine.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

U64_MAX = (1 << 64) - 1


class HostState(Enum):
    """What a rank's host thread is doing (reference ``model.py:24-29``)."""

    USEFUL = "useful"
    OFFLOAD = "offload"
    MPI = "mpi"


class DeviceActivityKind(Enum):
    """Recorded device activity (reference ``model.py:32-36``)."""

    KERNEL = "kernel"
    MEMORY = "memory"


#: wire codes of the packed SoA ``kind`` column (include/heteff_b200.h)
HOST_STATE_CODE = {HostState.USEFUL: 0, HostState.OFFLOAD: 1, HostState.MPI: 2}
DEVICE_KIND_CODE = {DeviceActivityKind.KERNEL: 0, DeviceActivityKind.MEMORY: 1}


@dataclass(frozen=True, order=True)
class Interval:
    """Half-open ``[start, end)`` span in integer nanoseconds."""

    start: int
    end: int

    @property
    def duration(self) -> int:
        return self.end - self.start


@dataclass(frozen=True)
class HostRecord:
    rank: int
    state: HostState
    interval: Interval


@dataclass(frozen=True)
class DeviceRecord:
    device_id: int
    kind: DeviceActivityKind
    interval: Interval
    stream: int | None = None


@dataclass(frozen=True)
class DeviceDecl:
    """A declared device; ``owner_rank`` only drives sharding and warnings."""

    device_id: int
    owner_rank: int | None = None


_HOST_BY_VALUE = tuple(sorted(HostState, key=lambda m: m.value))
_DEV_BY_VALUE = tuple(sorted(DeviceActivityKind, key=lambda m: m.value))


def _already_canonical(records, res_attr, kind_attr, members, stream_attr) -> bool:
    if len(records) < 2:
        return True
    try:
        from . import _pack
    except ImportError:
        return False
    return _pack.is_canonical(records, res_attr, kind_attr, members, stream_attr)


def _native_sorted(records, res_attr, kind_attr, members, stream_attr, key) -> tuple:
    """``tuple(sorted(records, key=key))`` -- by a stable numpy lexsort over natively
    extracted key columns when every key fits 64-bit integers (csrc/pack.c)."""
    try:
        from . import _pack
    except ImportError:
        _pack = None
    if _pack is not None:
        import numpy as np

        n = len(records)
        cols = (np.empty(n, np.int64), np.empty(n, np.uint64), np.empty(n, np.uint64), np.empty(n, np.uint8),
                np.empty(n, np.int64))
        if _pack.sort_keys(records, res_attr, kind_attr, members, stream_attr, *cols):
            order = np.lexsort((cols[4], cols[3], cols[2], cols[1], cols[0]))   # stable, last key primary
            return tuple(map(records.__getitem__, order.tolist()))
    return tuple(sorted(records, key=key))


def _canonical_host(rec: HostRecord):
    iv = rec.interval
    return (rec.rank, iv.start, iv.end, rec.state.value)


def _canonical_device(rec: DeviceRecord):
    iv = rec.interval
    return (rec.device_id, iv.start, iv.end, rec.kind.value, -1 if rec.stream is None else rec.stream)


@dataclass(frozen=True)
class Trace:
    """Declared resources plus their records, records in canonical order.

    Canonical order is per resource by ``(start, end, state/kind[, stream])``
    exactly as the reference orders them, so two traces with the same records
    compare equal and record indices in messages agree with the reference.
    Declaration order of ``host_processes`` / ``devices`` is kept as given.
    """

    host_processes: tuple[int, ...] = ()
    devices: tuple[DeviceDecl, ...] = ()
    host_records: tuple[HostRecord, ...] = ()
    device_records: tuple[DeviceRecord, ...] = ()
    time_unit: str = "ns"

    def __post_init__(self) -> None:
        set_ = object.__setattr__
        set_(self, "host_processes", tuple(self.host_processes))
        set_(self, "devices", tuple(self.devices))
        hr, dr = tuple(self.host_records), tuple(self.device_records)
        # records that already arrive in canonical order (files, time-ordered generators)
        # skip the key-function sort: one native pass decides it (csrc/pack.c)
        if not _already_canonical(hr, "rank", "state", _HOST_BY_VALUE, None):
            hr = _native_sorted(hr, "rank", "state", _HOST_BY_VALUE, None, _canonical_host)
        if not _already_canonical(dr, "device_id", "kind", _DEV_BY_VALUE, "stream"):
            dr = _native_sorted(dr, "device_id", "kind", _DEV_BY_VALUE, "stream", _canonical_device)
        set_(self, "host_records", hr)
        set_(self, "device_records", dr)

    @property
    def n(self) -> int:
        return len(self.host_processes)

    @property
    def m(self) -> int:
        return len(self.devices)


@dataclass
class ValidationReport:
    """Validation findings; any error makes the trace unusable."""

    errors: list[str] = field(default_factory=list)
    warnings: list[str] = field(default_factory=list)

    @property
    def ok(self) -> bool:
        return not self.errors


class InvalidTraceError(Exception):
    """An operation that needs a valid trace got one with validation errors."""

    def __init__(self, report: ValidationReport):
        self.report = report
        shown = "; ".join(report.errors[:3])
        extra = len(report.errors) - 3
        tail = f" (+{extra} more)" if extra > 0 else ""
        super().__init__(f"trace failed validation: {shown}{tail}")
