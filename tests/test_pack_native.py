"""The native Trace -> SoA packer and canonical-order check (csrc/pack.c) against the
pure-Python packer and the key-function sort they short-cut (host-side ingest)."""

from __future__ import annotations

import random

import numpy as np
import pytest

import paper_2603_26576_b200 as hb
from paper_2603_26576_b200 import packing

pytest.importorskip("paper_2603_26576_b200._pack")

HS, DK = list(hb.HostState), list(hb.DeviceActivityKind)


def _trace(seed, n=5, m=6, k=400, shuffle=True, streams=True):
    rng = random.Random(seed)
    host = [hb.HostRecord(rng.randrange(n), rng.choice(HS), hb.Interval(s, s + rng.randrange(0, 50)))
            for s in (rng.randrange(0, 10 ** 6) for _ in range(k))]
    dev = [hb.DeviceRecord(rng.randrange(m), rng.choice(DK), hb.Interval(s, s + rng.randrange(0, 50)),
                           rng.choice([None, 0, 3, -2]) if streams else None)
           for s in (rng.randrange(0, 10 ** 6) for _ in range(k))]
    # ties on (res, start, end) exercise the state / kind / stream tie-break
    host += [hb.HostRecord(1, st, hb.Interval(77, 99)) for st in HS]
    dev += [hb.DeviceRecord(2, kd, hb.Interval(77, 99), sid) for kd in DK for sid in (None, 1, 0)]
    if shuffle:
        rng.shuffle(host)
        rng.shuffle(dev)
    return hb.Trace(host_processes=tuple(range(n)), devices=tuple(hb.DeviceDecl(d, d % n) for d in range(m)),
                    host_records=tuple(host), device_records=tuple(dev))


@pytest.mark.parametrize("seed", range(6))
def test_canonical_order_matches_the_key_sort(seed):
    t = _trace(seed)
    assert list(t.host_records) == sorted(t.host_records, key=packing_key_host)
    assert list(t.device_records) == sorted(t.device_records, key=packing_key_dev)
    # already-canonical input is kept as is (the native check says so) and stays equal
    again = hb.Trace(t.host_processes, t.devices, t.host_records, t.device_records)
    assert again == t


def packing_key_host(r):
    return (r.rank, r.interval.start, r.interval.end, r.state.value)


def packing_key_dev(r):
    return (r.device_id, r.interval.start, r.interval.end, r.kind.value, -1 if r.stream is None else r.stream)


def _packed_both(t, monkeypatch):
    native = packing.pack_trace(t)
    with monkeypatch.context() as mp:
        mp.setattr(packing, "_pack", None)
        python = packing.pack_trace(t)
    return native, python


def _same(a, b):
    for side in ("host", "dev"):
        x, y = getattr(a, side), getattr(b, side)
        for col in ("start", "end", "res", "kind"):
            assert np.array_equal(getattr(x, col), getattr(y, col)), (side, col)
        assert (x.index is None) == (y.index is None)
        if x.index is not None:
            assert np.array_equal(x.index, y.index)
    assert a.host_q == b.host_q and a.dev_q == b.dev_q and a.host_elapsed_floor == b.host_elapsed_floor


@pytest.mark.parametrize("seed", range(4))
def test_native_packer_equals_python_packer(seed, monkeypatch):
    t = _trace(seed)
    _same(*_packed_both(t, monkeypatch))


@pytest.mark.parametrize("bad", [True, -5, 2 ** 64, 3.0])
def test_native_packer_defers_unusual_timestamps_to_the_exact_path(bad, monkeypatch):
    t = _trace(9, shuffle=False)
    host = list(t.host_records)
    host[3] = hb.HostRecord(host[3].rank, host[3].state, hb.Interval(bad, 2 ** 64 + 7 if bad == 2 ** 64 else 10))
    t2 = hb.Trace(t.host_processes, t.devices, tuple(host), t.device_records) if not isinstance(bad, float) else None
    if t2 is None:   # float timestamps do not even order against ints in every position: pack directly
        t2 = t
        object.__setattr__(t2, "host_records", tuple(host))
    _same(*_packed_both(t2, monkeypatch))


def test_native_records_equal_the_dataclass_constructors():
    from paper_2603_26576_b200 import trace_io

    res = np.array([0, 5, 2 ** 62], np.uint64)
    kinds = np.array([0, 1, 0], np.uint8)
    st = np.array([0, 7, 2 ** 64 - 3], np.uint64)
    en = np.array([0, 9, 2 ** 64 - 1], np.uint64)
    streams = np.array([-1, 3, 0], np.int64)
    got = trace_io._records(hb.DeviceRecord, "device_id", "kind", trace_io._DEV_CODE_KIND, res, kinds, st, en, streams)
    ref = [hb.DeviceRecord(0, DK[0], hb.Interval(0, 0), None), hb.DeviceRecord(5, DK[1], hb.Interval(7, 9), 3),
           hb.DeviceRecord(2 ** 62, DK[0], hb.Interval(2 ** 64 - 3, 2 ** 64 - 1), 0)]
    assert got == ref and [hash(x) for x in got] == [hash(x) for x in ref] and repr(got) == repr(ref)
    host = trace_io._records(hb.HostRecord, "rank", "state", trace_io._HOST_CODE_STATE, res[:2], np.array([2, 1], np.uint8),
                             st[:2], en[:2])
    assert host == [hb.HostRecord(0, trace_io._HOST_CODE_STATE[2], hb.Interval(0, 0)),
                    hb.HostRecord(5, trace_io._HOST_CODE_STATE[1], hb.Interval(7, 9))]
    # ids beyond int64: the Python construction path
    big = trace_io._records(hb.HostRecord, "rank", "state", trace_io._HOST_CODE_STATE,
                            np.array([2 ** 64 - 1], np.uint64), np.array([0], np.uint8), st[:1], en[:1])
    assert big == [hb.HostRecord(2 ** 64 - 1, trace_io._HOST_CODE_STATE[0], hb.Interval(0, 0))]
