"""The drop-in hot-path API: same names, arguments, results and exceptions as
the reference's ``heteff`` stage functions, computed by the B200 engine.

=====================  ==========================================
this module            reference
=====================  ==========================================
``validate``           ``model.py:160-230``
``summarize_host``     ``summarize.py:57-92``
``summarize_device``   ``summarize.py:95-138``
``host_metrics``       ``metrics.py:66-93``
``device_metrics``     ``metrics.py:96-122``
``compute_report``     ``metrics.py:125-154``
=====================  ==========================================

Every function packs the trace (host-side ingest, :mod:`.packing`) and runs
the fused analysis kernel; there is no CPU compute path.
"""

from __future__ import annotations

from collections.abc import Mapping
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .engine import Findings, analyze_packed, metrics_from_summaries
from .messages import clamp_warnings, declaration_messages, validation_report
from .model import U64_MAX, InvalidTraceError, Trace, ValidationReport
from .packing import PackedTrace, dev_owner_table, pack_trace


class AnalysisError(Exception):
    """The trace is structurally fine but cannot be analyzed (e.g. zero elapsed)."""


@dataclass(frozen=True)
class HostSummary:
    """Per-rank state totals, gaps and lead-in counted as useful."""

    rank: int
    d_useful: int
    d_offload: int
    d_mpi: int
    span_end: int


@dataclass(frozen=True)
class DeviceSummary:
    """Per-device activity totals; kernel + memory + idle == elapsed."""

    device_id: int
    d_kernel: int
    d_memory: int
    d_idle: int


@dataclass(frozen=True)
class HostMetrics:
    parallel_efficiency: float
    mpi_parallel_efficiency: float | None
    mpi_communication_efficiency: float | None
    mpi_load_balance: float | None
    device_offload_efficiency: float | None


@dataclass(frozen=True)
class DeviceMetrics:
    parallel_efficiency: float
    load_balance: float | None
    communication_efficiency: float | None
    orchestration_efficiency: float | None


@dataclass(frozen=True)
class MetricsReport:
    elapsed_ns: int
    n: int
    m: int
    host: HostMetrics | None
    device: DeviceMetrics | None
    host_summaries: tuple[HostSummary, ...]
    device_summaries: tuple[DeviceSummary, ...]
    warnings: tuple[str, ...]


def _run(trace: Trace, mode: int, elapsed: int = 0, want_lists: bool = True):
    packed = pack_trace(trace)
    f = analyze_packed(packed, mode, elapsed, want_lists=want_lists)
    if f.status == N.CONTRACT:  # packing always produces canonical order
        raise N.NativeError(f"packed trace violates the canonical-order contract at record {f.contract_index}")
    return packed, f


def _invalid(trace: Trace, packed: PackedTrace, f: Findings) -> bool:
    """Errors the reference's validate() reports (model.py:160-230): declaration errors,
    kernel findings, and records the packer quarantined (non-int / negative / beyond-u64
    timestamps never reach the kernel, model.py:140-157)."""
    decl_errors, _ = declaration_messages(trace)
    return bool(decl_errors) or bool(packed.host_q) or bool(packed.dev_q) or f.status == N.INVALID_TRACE


def _raise_invalid(trace: Trace, packed: PackedTrace, f: Findings, report: ValidationReport | None = None):
    if report is None:
        report = validation_report(trace, packed, f)
    raise InvalidTraceError(report)


def _host_summaries(trace: Trace, f: Findings) -> list[HostSummary]:
    out = []
    for pos, rank in enumerate(trace.host_processes):
        u, w, p, s = (int(x) for x in f.host_sum[pos])
        out.append(HostSummary(rank, u, w, p, s))
    return out


def _device_summaries(trace: Trace, f: Findings, elapsed: int) -> list[DeviceSummary]:
    out = []
    for pos, d in enumerate(trace.devices):
        k, mem, idle, _ = (int(x) for x in f.dev_sum[pos])
        if elapsed > U64_MAX:   # window beyond the u64 domain: idle is the exact remainder
            idle = elapsed - k - mem
        out.append(DeviceSummary(d.device_id, k, mem, idle))
    return out


def validate(trace: Trace) -> ValidationReport:
    """Every trace invariant, as data (never raises); ``model.py:160-230``."""
    packed, f = _run(trace, N.MODE_VALIDATE)
    return validation_report(trace, packed, f)


def summarize_host(trace: Trace) -> tuple[list[HostSummary], int]:
    """Per-rank totals and the elapsed time E; ``summarize.py:57-92``."""
    packed, f = _run(trace, N.MODE_SUMMARIZE_HOST, want_lists=False)
    if _invalid(trace, packed, f):
        _, f = _run(trace, N.MODE_VALIDATE)
        _raise_invalid(trace, packed, f)
    return _host_summaries(trace, f), f.elapsed


def summarize_device(trace: Trace, elapsed: int) -> tuple[list[DeviceSummary], list[str]]:
    """Per-device kernel / memory / idle inside ``[0, elapsed)``; ``summarize.py:95-138``."""
    if elapsed <= 0:
        raise ValueError(f"elapsed must be positive, got {elapsed}")
    packed, f = _run(trace, N.MODE_SUMMARIZE_DEVICE, min(elapsed, U64_MAX), want_lists=False)
    if _invalid(trace, packed, f):
        _, f = _run(trace, N.MODE_VALIDATE)
        _raise_invalid(trace, packed, f)
    return _device_summaries(trace, f, elapsed), clamp_warnings(trace, f, elapsed)


def _u64_rows(rows) -> np.ndarray:
    try:
        return np.array(rows, dtype=np.uint64).reshape(-1, 4)
    except OverflowError as e:
        raise OverflowError("summary durations must fit in 64 bits") from e


def _u64_elapsed(elapsed: int) -> None:
    """The metric kernels take E as a u64 (include/heteff_b200.h); a larger E is refused
    loudly rather than truncated by the C call."""
    if elapsed > U64_MAX:
        raise OverflowError("elapsed must fit in 64 bits")


def host_metrics(summaries: list[HostSummary], elapsed: int) -> HostMetrics:
    """Host tree from per-rank totals; ``metrics.py:66-93``."""
    if len(summaries) < 1:
        raise ValueError("host_metrics requires at least one rank")
    if elapsed <= 0:
        raise ValueError(f"elapsed must be positive, got {elapsed}")
    _u64_elapsed(elapsed)
    rows = _u64_rows([(s.d_useful, s.d_offload, s.d_mpi, s.span_end) for s in summaries])
    return HostMetrics(*metrics_from_summaries(rows, elapsed, host_side=True))


def device_metrics(summaries: list[DeviceSummary], elapsed: int) -> DeviceMetrics:
    """Device tree from per-device totals; ``metrics.py:96-122``."""
    if len(summaries) < 1:
        raise ValueError("device_metrics requires at least one device")
    if elapsed <= 0:
        raise ValueError(f"elapsed must be positive, got {elapsed}")
    _u64_elapsed(elapsed)
    rows = _u64_rows([(s.d_kernel, s.d_memory, s.d_idle, 0) for s in summaries])
    return DeviceMetrics(*metrics_from_summaries(rows, elapsed, host_side=False))


def compute_report(trace: Trace) -> MetricsReport:
    """Validate, summarize and evaluate both trees in ONE kernel launch; ``metrics.py:125-154``."""
    packed, f = _run(trace, N.MODE_REPORT)
    report = validation_report(trace, packed, f)
    if not report.ok:
        raise InvalidTraceError(report)
    if f.status == N.ANALYSIS_ERROR:
        raise AnalysisError("elapsed time is zero: trace records no activity")
    E = f.elapsed
    warnings = list(report.warnings)
    if trace.m >= 1:
        warnings += clamp_warnings(trace, f, E)
    host = HostMetrics(*f.host_metrics) if trace.n >= 1 else None
    device = DeviceMetrics(*f.device_metrics) if trace.m >= 1 else None
    return MetricsReport(
        elapsed_ns=E, n=trace.n, m=trace.m, host=host, device=device,
        host_summaries=tuple(_host_summaries(trace, f)),
        device_summaries=tuple(_device_summaries(trace, f, E)) if trace.m >= 1 else (),
        warnings=tuple(warnings))


# ---------------------------------------------------------------------------
# EXTENSIONS beyond the reference: monitoring regions and
# the offload-wait / device-busy overlap.  Not part of the reference API.
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class RegionReport:
    """One monitoring region: ``report`` is the reference's compute_report of the
    window-clipped trace (``None`` when the region records no activity, where the
    reference raises AnalysisError); ``offload_busy[g]`` is the owner's offload
    time during which device g was busy, inside the region."""

    window: object               # (start, end) or {rank: (start, end)}, as given
    report: MetricsReport | None
    offload_busy: tuple[int, ...]
    offload_busy_fraction: float | None


def region_reports(trace: Trace, windows) -> list[RegionReport]:
    """Region metric trees (K5 + K6 kernels).  ``windows`` lists the regions; each is
    ``(start, end)`` -- one window for every rank and device -- or a mapping
    ``{rank: (start, end)}`` -- a per-rank region (TALP annotates regions per process,
    PAPER.md:113): each rank's records are clipped to its own window and shifted by its
    own start, devices follow their ``owner_rank``; ranks missing from the mapping and
    devices without a declared owner record nothing in that region.  With any mapping
    present every region is evaluated per rank (a plain window applies to all ranks).

    Raises InvalidTraceError for an invalid trace (validation runs first).
    Region reports carry summaries and metrics; their ``warnings`` are empty.
    ``RegionReport.window`` is the region as given."""
    import torch

    from .engine import DeviceTrace, analyze_regions

    packed = pack_trace(trace)
    windows = list(windows)
    per_rank = any(isinstance(w, Mapping) for w in windows)
    if per_rank:   # [R][host_ids][2] over the dense host ids
        dense = {rank: i for i, rank in enumerate(packed.host_ids)}
        table = np.zeros((len(windows), len(packed.host_ids), 2), dtype=np.uint64)
        for j, w in enumerate(windows):
            if isinstance(w, Mapping):
                for rank, (a, b) in w.items():
                    if rank in dense:
                        table[j, dense[rank]] = (int(a), int(b))
            else:
                table[j, :] = (int(w[0]), int(w[1]))
        given, windows = windows, table
    else:
        windows = [(int(a), int(b)) for a, b in windows]
        given = windows
    dev = torch.device("cuda", int(__import__("os").environ.get("HETEFF_DEVICE", "0")))

    def up(a):
        a = np.ascontiguousarray(a)
        if a.dtype == np.uint64:
            a = a.view(np.int64)
        return torch.from_numpy(a).to(dev)

    H, D = packed.host, packed.dev
    dt = DeviceTrace(up(H.start), up(H.end), up(H.res), up(H.kind), up(D.start), up(D.end), up(D.res),
                     up(D.kind), packed.n_unique, packed.m_unique, packed.host_elapsed_floor)
    owner = dev_owner_table(trace, packed)
    run = analyze_regions(dt, windows, owner, host_decl=up(packed.host_decl), dev_decl=up(packed.dev_decl),
                          host_ids=len(packed.host_ids), dev_ids=len(packed.dev_ids))
    if run.status not in (N.OK, N.ANALYSIS_ERROR) or packed.host_q or packed.dev_q:
        _, f = _run(trace, N.MODE_VALIDATE)
        _raise_invalid(trace, packed, f)
    out = []
    for w, r in zip(given, run.regions):
        if r.status != N.OK:
            out.append(RegionReport(w, None, tuple(int(x) for x in r.offload_busy), None))
            continue
        hs = tuple(HostSummary(rank, *(int(x) for x in r.host_sum[pos]))
                   for pos, rank in enumerate(trace.host_processes))
        ds = tuple(DeviceSummary(d.device_id, *(int(x) for x in r.dev_sum[pos][:3]))
                   for pos, d in enumerate(trace.devices)) if trace.m >= 1 else ()
        rep = MetricsReport(
            elapsed_ns=r.elapsed, n=trace.n, m=trace.m,
            host=HostMetrics(*r.host_metrics) if trace.n >= 1 else None,
            device=DeviceMetrics(*r.device_metrics) if trace.m >= 1 else None,
            host_summaries=hs, device_summaries=ds, warnings=())
        out.append(RegionReport(w, rep, tuple(int(x) for x in r.offload_busy), r.offload_busy_fraction))
    return out
