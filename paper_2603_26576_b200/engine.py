"""Calls into the B200 engine: packed trace in, :class:`Findings` out.

Two entry shapes:

* :func:`analyze_packed` -- a :class:`~.packing.PackedTrace` in host memory
  (the drop-in API path); the C ABI stages the columns to HBM.
* :func:`analyze_device` -- columns already resident in HBM (torch CUDA
  tensors or raw device pointers); the bench / large-trace path.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .packing import PackedTrace, RecordColumns


@dataclass
class Findings:
    status: int
    contract_flags: int
    contract_index: int
    host_elapsed: int
    elapsed: int
    dev_max_end: int
    host_metrics: tuple          # 5 floats or None
    device_metrics: tuple        # 4 floats or None
    counts: tuple                # 8 ints (heteff list classes)
    host_sum: np.ndarray         # uint64 [n][4] useful, offload, mpi, span_end (declaration order)
    dev_sum: np.ndarray          # uint64 [m][4] kernel, memory, idle, clamped
    lists: list = field(default_factory=list)   # 8 arrays of SoA positions (sorted), or empty
    kernel_ms: float = 0.0


def _ptr(a: np.ndarray | None) -> int | None:
    return None if a is None or a.size == 0 else a.ctypes.data


def _records(cols: RecordColumns) -> N.Records:
    return N.Records(_ptr(cols.start), _ptr(cols.end), _ptr(cols.res), _ptr(cols.kind), cols.count)


def _metrics(vals, mask, k):
    return tuple(float(vals[i]) if (mask >> i) & 1 else None for i in range(k))


def _findings(res: N.Result, host_sum, dev_sum, lists) -> Findings:
    return Findings(
        status=res.status, contract_flags=res.contract_flags, contract_index=res.contract_index,
        host_elapsed=int(res.host_elapsed), elapsed=int(res.elapsed), dev_max_end=int(res.dev_max_end),
        host_metrics=_metrics(res.host_metrics, res.host_mask, 5),
        device_metrics=_metrics(res.device_metrics, res.device_mask, 4),
        counts=tuple(int(c) for c in res.counts), host_sum=host_sum, dev_sum=dev_sum, lists=lists,
        kernel_ms=float(res.kernel_ms))


def _check(ctx, rc):
    if rc in (N.CUDA_ERROR, N.NOMEM, N.BAD_ARG):
        raise N.NativeError(f"engine error {rc}: {N.last_error(ctx)}")


def analyze_packed(packed: PackedTrace, mode: int, elapsed: int = 0, want_lists: bool = True,
                   capacity: int = 1 << 14, device: int | None = None, sort_if_needed: bool = False) -> Findings:
    """Run the engine on a host-resident packed trace (copies inside the call)."""
    ctx = N.context(device)
    lib = N.load()
    t = N.TraceABI(_records(packed.host), _records(packed.dev),
                   len(packed.host_ids), len(packed.dev_ids),
                   _ptr(packed.host_decl), _ptr(packed.dev_decl),
                   packed.n_unique, packed.m_unique, packed.host_elapsed_floor)
    total = packed.host.count + packed.dev.count
    cap = min(capacity, max(total, 1)) if want_lists else 0
    while True:
        host_sum = np.zeros((max(packed.n_unique, 1), 4), dtype=np.uint64)
        dev_sum = np.zeros((max(packed.m_unique, 1), 4), dtype=np.uint64)
        lists = [np.empty(cap, dtype=np.int64) for _ in range(N.NUM_LISTS)] if cap else []
        out = N.Outputs(_ptr(host_sum), _ptr(dev_sum),
                        (C.c_void_p * N.NUM_LISTS)(*[_ptr(x) for x in lists]) if cap
                        else (C.c_void_p * N.NUM_LISTS)())
        opt = N.Options(mode, N.FLAG_SORT_IF_NEEDED if sort_if_needed else 0, elapsed, cap)
        res = N.Result()
        rc = lib.heteff_analyze_host(ctx, C.byref(t), C.byref(opt), C.byref(res), C.byref(out), None)
        _check(ctx, rc)
        need = max(res.counts) if want_lists else 0
        if need <= cap:
            break
        cap = int(need)
    if cap:
        lists = [np.sort(lists[i][: res.counts[i]]) for i in range(N.NUM_LISTS)]
    return _findings(res, host_sum[: packed.n_unique], dev_sum[: packed.m_unique], lists)


def overlap_covers(packed: PackedTrace, error_pos: np.ndarray, device: int | None = None) -> np.ndarray:
    """Cover record (model.py:208-215) of each overlap error, by SoA position."""
    ctx = N.context(device)
    lib = N.load()
    err = np.ascontiguousarray(error_pos, dtype=np.int64)
    cover = np.empty_like(err)
    t = N.TraceABI(_records(packed.host), _records(packed.dev), len(packed.host_ids), len(packed.dev_ids),
                   None, None, packed.n_unique, packed.m_unique, 0)
    rc = lib.heteff_overlap_covers(ctx, C.byref(t), 1, _ptr(err), err.size, _ptr(cover), None)
    _check(ctx, rc)
    return cover


def metrics_from_summaries(rows: np.ndarray, elapsed: int, host_side: bool, device: int | None = None):
    """host_metrics / device_metrics stage functions on the GPU."""
    ctx = N.context(device)
    lib = N.load()
    rows = np.ascontiguousarray(rows, dtype=np.uint64)
    k = 5 if host_side else 4
    vals = (C.c_double * k)()
    mask = C.c_uint32(0)
    fn = lib.heteff_host_metrics if host_side else lib.heteff_device_metrics
    rc = fn(ctx, _ptr(rows), rows.shape[0], elapsed, C.cast(vals, C.c_void_p), C.byref(mask), None)
    if rc == N.VALUE_ERROR:
        raise ValueError(N.last_error(ctx))
    _check(ctx, rc)
    return _metrics(vals, mask.value, k)


# ---------------------------------------------------------------------------
# device-resident columns (bench / columnar fast path)
# ---------------------------------------------------------------------------
@dataclass
class DeviceTrace:
    """Packed SoA resident in HBM: torch CUDA tensors (or anything with data_ptr)."""

    h_start: object
    h_end: object
    h_res: object
    h_kind: object
    d_start: object
    d_end: object
    d_res: object
    d_kind: object
    n: int                 # declared ranks (dense ids 0..n-1)
    m: int                 # declared devices
    host_elapsed_floor: int = 0
    # CSR offsets (int64 [n + 1] / [m + 1], same memory as the columns): when present the
    # analysis reads them instead of the res columns -- 17 instead of 21 B per interval
    h_seg: object = None
    d_seg: object = None

    def columns_only(self) -> "DeviceTrace":
        """The same trace addressed through its res columns (no CSR offsets)."""
        return DeviceTrace(self.h_start, self.h_end, self.h_res, self.h_kind, self.d_start, self.d_end, self.d_res,
                           self.d_kind, self.n, self.m, self.host_elapsed_floor)

    def with_csr(self) -> "DeviceTrace":
        """Attach CSR offsets computed from the res columns (ids 0..n-1 / 0..m-1, grouped)."""
        import torch

        def seg(res, k):
            out = torch.zeros(k + 1, dtype=torch.int64, device=res.device)
            if res.numel():
                torch.cumsum(torch.bincount(res.long(), minlength=k)[:k], 0, out=out[1:])
            return out

        return DeviceTrace(self.h_start, self.h_end, self.h_res, self.h_kind, self.d_start, self.d_end, self.d_res,
                           self.d_kind, self.n, self.m, self.host_elapsed_floor, seg(self.h_res, self.n),
                           seg(self.d_res, self.m))

    @property
    def host_count(self) -> int:
        return int(self.h_start.numel())

    @property
    def dev_count(self) -> int:
        return int(self.d_start.numel())


def _dptr(t) -> int | None:
    return t.data_ptr() if t is not None and t.numel() > 0 else None


def _segptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def device_trace_abi(dt: DeviceTrace) -> N.TraceABI:
    hs, ds = _segptr(dt.h_seg), _segptr(dt.d_seg)
    return N.TraceABI(
        N.Records(_dptr(dt.h_start), _dptr(dt.h_end), None if hs else _dptr(dt.h_res), _dptr(dt.h_kind),
                  dt.host_count),
        N.Records(_dptr(dt.d_start), _dptr(dt.d_end), None if ds else _dptr(dt.d_res), _dptr(dt.d_kind),
                  dt.dev_count),
        dt.n, dt.m, None, None, dt.n, dt.m, dt.host_elapsed_floor, hs, ds)


def analyze_device(dt: DeviceTrace, mode: int = N.MODE_REPORT, elapsed: int = 0, stream: int | None = None,
                   device: int | None = None, host_sum: np.ndarray | None = None,
                   dev_sum: np.ndarray | None = None, sort_if_needed: bool = False) -> Findings:
    """Analyze HBM-resident columns (counts only, no per-record lists).

    ``sort_if_needed``: columns that are not in canonical order are sorted on the
    GPU (K3, :func:`sort_records`) and analyzed again instead of failing with
    ``CONTRACT``."""
    ctx = N.context(device)
    lib = N.load()
    t = device_trace_abi(dt)
    if host_sum is None:
        host_sum = np.zeros((max(dt.n, 1), 4), dtype=np.uint64)
    if dev_sum is None:
        dev_sum = np.zeros((max(dt.m, 1), 4), dtype=np.uint64)
    out = N.Outputs(_ptr(host_sum), _ptr(dev_sum), (C.c_void_p * N.NUM_LISTS)())
    opt = N.Options(mode, N.FLAG_SORT_IF_NEEDED if sort_if_needed else 0, elapsed, 0)
    res = N.Result()
    rc = lib.heteff_analyze(ctx, C.byref(t), C.byref(opt), C.byref(res), C.byref(out), stream)
    _check(ctx, rc)
    return _findings(res, host_sum[: dt.n], dev_sum[: dt.m], [])


class AnalysisPlan:
    """Repeated analysis of the same HBM-resident columns (online monitoring, benches):
    the ABI structs and the host output arrays are built once, so a call is one C
    entry (launch + one D2H of the result block + sync) with no per-call Python
    allocation.  ``run()`` returns the shared :class:`Findings` (overwritten by the
    next call)."""

    def __init__(self, dt: DeviceTrace, mode: int = N.MODE_REPORT, elapsed: int = 0, stream: int | None = None,
                 device: int | None = None, sort_if_needed: bool = False):
        self.ctx = N.context(device)
        self.lib = N.load()
        self.dt = dt   # keeps the columns alive
        self.t = device_trace_abi(dt)
        self.host_sum = np.zeros((max(dt.n, 1), 4), dtype=np.uint64)
        self.dev_sum = np.zeros((max(dt.m, 1), 4), dtype=np.uint64)
        self.out = N.Outputs(_ptr(self.host_sum), _ptr(self.dev_sum), (C.c_void_p * N.NUM_LISTS)())
        self.opt = N.Options(mode, N.FLAG_SORT_IF_NEEDED if sort_if_needed else 0, elapsed, 0)
        self.res = N.Result()
        self.stream = C.c_void_p(stream) if stream else None
        self._args = (self.ctx, C.byref(self.t), C.byref(self.opt), C.byref(self.res), C.byref(self.out),
                      self.stream)

    def run(self) -> Findings:
        rc = self.lib.heteff_analyze(*self._args)
        _check(self.ctx, rc)
        return _findings(self.res, self.host_sum[: self.dt.n], self.dev_sum[: self.dt.m], [])

    def run_status(self) -> int:
        """The analysis only; results stay in ``self.res`` / ``self.host_sum`` / ``self.dev_sum``."""
        rc = self.lib.heteff_analyze(*self._args)
        _check(self.ctx, rc)
        return rc


def analyze_host_columns(dt: DeviceTrace, mode: int = N.MODE_REPORT, stream: int | None = None,
                         device: int | None = None, sort_if_needed: bool = False, csr=None) -> Findings:
    """Same as :func:`analyze_device` but the columns are HOST tensors (pinned); H2D inside.

    ``csr=(host_seg, dev_seg)`` (int64 host arrays / tensors of ``ids + 1`` offsets) sends
    the resource ids as CSR offsets instead of the res columns (``heteff_analyze_host_csr``:
    17 instead of 21 bytes per interval over PCIe; ``dt``'s res columns are not read)."""
    ctx = N.context(device)
    lib = N.load()
    t = device_trace_abi(dt)
    host_sum = np.zeros((max(dt.n, 1), 4), dtype=np.uint64)
    dev_sum = np.zeros((max(dt.m, 1), 4), dtype=np.uint64)
    out = N.Outputs(_ptr(host_sum), _ptr(dev_sum), (C.c_void_p * N.NUM_LISTS)())
    opt = N.Options(mode, N.FLAG_SORT_IF_NEEDED if sort_if_needed else 0, 0, 0)
    res = N.Result()
    if csr is not None:
        hseg, dseg = (np.ascontiguousarray(x.numpy() if hasattr(x, "numpy") else x, dtype=np.int64) for x in csr)
        rc = lib.heteff_analyze_host_csr(ctx, C.byref(t), _ptr(hseg), _ptr(dseg), C.byref(opt), C.byref(res),
                                         C.byref(out), stream)
    else:
        rc = lib.heteff_analyze_host(ctx, C.byref(t), C.byref(opt), C.byref(res), C.byref(out), stream)
    _check(ctx, rc)
    return _findings(res, host_sum[: dt.n], dev_sum[: dt.m], [])


@dataclass
class SortResult:
    start: object
    end: object
    res: object
    kind: object
    perm: object           # int64: input position of each output record
    key_bits: int
    passes: int
    wide: bool
    start_sorted: bool     # input was start-ordered: sorted by res alone
    ms: float


def sort_records(start, end, res, kind, stream: int | None = None, device: int | None = None) -> SortResult:
    """K3: stable GPU sort of one record set (CUDA tensors) by (res, start).

    The canonical order of ``Trace.__post_init__`` (``model.py:74-80,99-107``)
    for columns that arrive unsorted; ties keep their input order."""
    import torch

    ctx = N.context(device)
    lib = N.load()
    n = int(start.numel())
    dev = start.device
    os_ = torch.empty(n, dtype=torch.int64, device=dev)   # u64 bits
    oe = torch.empty(n, dtype=torch.int64, device=dev)
    orr = torch.empty(n, dtype=torch.int32, device=dev)
    ok = torch.empty(n, dtype=torch.uint8, device=dev)
    perm = torch.empty(n, dtype=torch.int64, device=dev)
    rec = N.Records(_dptr(start), _dptr(end), _dptr(res), _dptr(kind), n)
    cols = N.Columns(_dptr(os_), _dptr(oe), _dptr(orr), _dptr(ok))
    info = N.SortInfo()
    rc = lib.heteff_sort_records(ctx, C.byref(rec), C.byref(cols), _dptr(perm), C.byref(info), stream)
    _check(ctx, rc)
    if rc != N.OK:
        raise N.NativeError(f"sort failed ({rc}): {N.last_error(ctx)}")
    return SortResult(os_, oe, orr, ok, perm, info.key_bits, info.passes, bool(info.wide),
                      bool(info.start_sorted), info.ms)


# ---------------------------------------------------------------------------
# EXTENSIONS: monitoring regions (K5) + offload-wait / device-busy overlap (K6)
# ---------------------------------------------------------------------------
@dataclass
class RegionFindings:
    status: int                 # OK, or ANALYSIS_ERROR when the region records no activity
    elapsed: int
    host_metrics: tuple         # 5 floats or None
    device_metrics: tuple       # 4 floats or None
    offload_busy_fraction: float | None
    host_sum: np.ndarray        # uint64 [n][4] useful, offload, mpi, span_end
    dev_sum: np.ndarray         # uint64 [m][4] kernel, memory, idle, clamped
    offload_busy: np.ndarray    # uint64 [m]


@dataclass
class RegionsRun:
    status: int                 # status of the whole-trace analysis that precedes the regions
    regions: list
    kernel_ms: float


def analyze_regions(dt: DeviceTrace, windows, dev_owner=None, stream: int | None = None,
                    device: int | None = None, host_decl=None, dev_decl=None, host_ids: int | None = None,
                    dev_ids: int | None = None) -> RegionsRun:
    """Region reports for ``windows`` of HBM-resident columns.

    ``windows``: ``[R][2]`` -- one window per region for every rank and device -- or
    ``[R][host_ids][2]`` -- per-rank regions: each rank's own window (dense host ids),
    devices follow their owner, unowned devices record nothing in the region.
    ``dev_owner``: int32 [dev_ids] dense host id owning each device (-1 none)."""
    ctx = N.context(device)
    lib = N.load()
    t = device_trace_abi(dt)
    if host_ids is not None:
        t.host_ids, t.dev_ids = host_ids, dev_ids
        t.host_decl, t.dev_decl = _dptr(host_decl), _dptr(dev_decl)
    warr = np.asarray(windows, dtype=np.uint64)
    per_rank = warr.ndim == 3
    if per_rank:
        if warr.shape[1:] != (t.host_ids, 2):
            raise ValueError(f"per-rank windows must be [R][{t.host_ids}][2], got {list(warr.shape)}")
        ws, we = np.ascontiguousarray(warr[:, :, 0]), np.ascontiguousarray(warr[:, :, 1])
    else:
        w = np.ascontiguousarray(warr.reshape(-1, 2))
        ws, we = np.ascontiguousarray(w[:, 0]), np.ascontiguousarray(w[:, 1])
    R = warr.shape[0]
    owner = None if dev_owner is None else np.ascontiguousarray(dev_owner, dtype=np.int32)
    n, m = t.n, t.m
    results = (N.RegionResult * max(R, 1))()
    hs = np.zeros((max(R, 1), max(n, 1), 4), dtype=np.uint64)
    ds = np.zeros((max(R, 1), max(m, 1), 4), dtype=np.uint64)
    busy = np.zeros((max(R, 1), max(m, 1)), dtype=np.uint64)
    rg = N.RegionsABI(_ptr(ws), _ptr(we), R, N.REGIONS_PER_RANK if per_rank else 0, _ptr(owner))
    out = N.RegionOutputs(C.cast(results, C.c_void_p), hs.ctypes.data, ds.ctypes.data, busy.ctypes.data, 0.0)
    rc = lib.heteff_analyze_regions(ctx, C.byref(t), C.byref(rg), C.byref(out), stream)
    _check(ctx, rc)
    regs = []
    if rc in (N.OK, N.ANALYSIS_ERROR):
        for j in range(R):
            x = results[j]
            regs.append(RegionFindings(
                int(x.status), int(x.elapsed), _metrics(x.host_metrics, x.host_mask, 5),
                _metrics(x.device_metrics, x.device_mask, 4),
                float(x.offload_busy_fraction) if x.offload_busy_defined else None,
                hs[j, :n], ds[j, :m], busy[j, :m]))
    return RegionsRun(rc, regs, float(out.kernel_ms))
