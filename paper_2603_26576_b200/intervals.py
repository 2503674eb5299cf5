"""The reference's interval algebra (``intervals.py:20-105``) on the GPU.

Same names, arguments, results and exceptions as ``heteff.intervals``:
``FlatSet``, ``EMPTY``, ``flatten``, ``subtract``, ``complement``,
``total_duration``, ``intersect``.  Each call ships the interval arrays to
HBM and runs the kernels of ``csrc/intervals.cu`` (flatten uses the K3 radix
sort); torch is used only for device memory.  Timestamps must fit in u64
(the trace model's own domain, ``model.py:21,149``).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Iterable

import numpy as np

from . import _native as N
from .model import Interval

U64_MAX = 2**64 - 1


@dataclass(frozen=True)
class FlatSet:
    """Disjoint union of intervals, canonically normalized (sorted, disjoint,
    non-adjacent, no zero-length members)."""

    intervals: tuple[Interval, ...] = ()

    def __iter__(self):
        return iter(self.intervals)

    def __len__(self) -> int:
        return len(self.intervals)


EMPTY = FlatSet()


def _dev():
    import torch

    return torch.device("cuda", int(__import__("os").environ.get("HETEFF_DEVICE", "0")))


def _to_gpu(starts, ends):
    import torch

    try:
        s = np.asarray(starts, dtype=np.uint64)
        e = np.asarray(ends, dtype=np.uint64)
    except OverflowError as exc:
        raise OverflowError("interval timestamps must be integers in [0, 2**64 - 1]") from exc
    d = _dev()
    return (torch.from_numpy(s.view(np.int64).copy()).to(d), torch.from_numpy(e.view(np.int64).copy()).to(d))


def _ptr(t):
    return t.data_ptr() if t.numel() > 0 else None


def _from_gpu(s, e, k: int) -> FlatSet:
    if k == 0:
        return EMPTY
    ss = s[:k].cpu().numpy().view(np.uint64).tolist()
    ee = e[:k].cpu().numpy().view(np.uint64).tolist()
    return FlatSet(tuple(Interval(a, b) for a, b in zip(ss, ee)))


def _check(ctx, rc):
    if rc != N.OK:
        raise N.NativeError(f"interval kernel failed ({rc}): {N.last_error(ctx)}")


def flatten(raw: Iterable[Interval]) -> FlatSet:
    """Merge an arbitrary interval list into its disjoint union (``intervals.py:40-61``).

    Raises ValueError naming the first interval with ``start > end``."""
    import torch

    items = list(raw)
    if not items:
        return EMPTY
    ctx, lib = N.context(), N.load()
    for iv in items:   # values outside u64 cannot enter HBM; malformed ones are reported by the kernel
        if not (0 <= iv.start <= U64_MAX and 0 <= iv.end <= U64_MAX):
            bad = next(i for i, x in enumerate(items) if x.start > x.end) if any(
                x.start > x.end for x in items) else None
            if bad is not None:
                raise ValueError(f"malformed interval at index {bad}: [{items[bad].start}, {items[bad].end})")
            raise OverflowError("interval timestamps must be integers in [0, 2**64 - 1]")
    s, e = _to_gpu([iv.start for iv in items], [iv.end for iv in items])
    n = len(items)
    os_ = torch.empty(n, dtype=torch.int64, device=s.device)
    oe = torch.empty(n, dtype=torch.int64, device=s.device)
    k, bad = C.c_int64(0), C.c_int64(-1)
    rc = lib.heteff_flatten(ctx, _ptr(s), _ptr(e), n, _ptr(os_), _ptr(oe), C.byref(k), C.byref(bad), None)
    if rc == N.VALUE_ERROR and bad.value >= 0:
        iv = items[bad.value]
        raise ValueError(f"malformed interval at index {bad.value}: [{iv.start}, {iv.end})")
    _check(ctx, rc)
    return _from_gpu(os_, oe, k.value)


def subtract(a: FlatSet, b: FlatSet) -> FlatSet:
    """Points in ``a`` and not in ``b`` (``intervals.py:64-81``)."""
    import torch

    if len(a) == 0:
        return EMPTY
    ctx, lib = N.context(), N.load()
    as_, ae = _to_gpu([iv.start for iv in a], [iv.end for iv in a])
    bs, be = _to_gpu([iv.start for iv in b], [iv.end for iv in b])
    cap = len(a) + len(b)
    os_ = torch.empty(cap, dtype=torch.int64, device=as_.device)
    oe = torch.empty(cap, dtype=torch.int64, device=as_.device)
    k = C.c_int64(0)
    rc = lib.heteff_subtract(ctx, _ptr(as_), _ptr(ae), len(a), _ptr(bs), _ptr(be), len(b), _ptr(os_), _ptr(oe),
                             C.byref(k), None)
    _check(ctx, rc)
    return _from_gpu(os_, oe, k.value)


def complement(a: FlatSet, bounds: Interval) -> FlatSet:
    """Points in ``bounds`` not covered by ``a`` (``intervals.py:84-90``)."""
    if bounds.start > bounds.end:
        raise ValueError(f"malformed bounds: [{bounds.start}, {bounds.end})")
    if bounds.duration == 0:
        return EMPTY
    return subtract(FlatSet((bounds,)), a)


def total_duration(a: FlatSet) -> int:
    """Sum of interval durations, exact (``intervals.py:93-95``)."""
    if len(a) == 0:
        return 0
    ctx, lib = N.context(), N.load()
    s, e = _to_gpu([iv.start for iv in a], [iv.end for iv in a])
    out = (C.c_uint64 * 2)()
    rc = lib.heteff_total_duration(ctx, _ptr(s), _ptr(e), len(a), C.cast(out, C.c_void_p), None)
    _check(ctx, rc)
    return int(out[0]) + (int(out[1]) << 64)


def intersect(a: FlatSet, bounds: Interval) -> FlatSet:
    """Restrict ``a`` to ``bounds`` (``intervals.py:98-105``)."""
    import torch

    if len(a) == 0:
        return EMPTY
    lo, hi = max(bounds.start, 0), min(bounds.end, U64_MAX)
    if hi <= lo:
        return EMPTY
    ctx, lib = N.context(), N.load()
    s, e = _to_gpu([iv.start for iv in a], [iv.end for iv in a])
    n = len(a)
    os_ = torch.empty(n, dtype=torch.int64, device=s.device)
    oe = torch.empty(n, dtype=torch.int64, device=s.device)
    k = C.c_int64(0)
    rc = lib.heteff_intersect(ctx, _ptr(s), _ptr(e), n, lo, hi, _ptr(os_), _ptr(oe), C.byref(k), None)
    _check(ctx, rc)
    return _from_gpu(os_, oe, k.value)
