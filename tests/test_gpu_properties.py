"""Property tests on the GPU engine, mirroring the reference's own strategy
(per-nanosecond sweep oracle, exact partition, product
identities, stream obliviousness; pkg/tests/sweep_oracle.py,
test_intervals.py:88-140, test_summarize.py:133-174, test_metrics.py:231-287).

The sweep oracle marks every covered nanosecond in a numpy bool array, so it
is independent of both the reference's sort-and-merge and the engine's
running-max identity."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

from hypothesis import given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

import paper_2603_26576_b200 as hb  # noqa: E402

IV = hb.Interval
SPAN = 300


def sweep(intervals, lo=0, hi=SPAN + 80):
    m = np.zeros(hi - lo, dtype=bool)
    for iv in intervals:
        a, b = max(iv.start, lo), min(iv.end, hi)
        if a < b:
            m[a - lo:b - lo] = True
    return m


def runs(mask, lo=0):
    out, i, n = [], 0, mask.size
    while i < n:
        if mask[i]:
            j = i
            while j < n and mask[j]:
                j += 1
            out.append(IV(lo + i, lo + j))
            i = j
        else:
            i += 1
    return out


ivs = st.lists(st.tuples(st.integers(0, SPAN), st.integers(0, 60)).map(lambda t: IV(t[0], t[0] + t[1])),
               max_size=25)


@settings(max_examples=150, deadline=None)
@given(a=ivs, b=ivs, lo=st.integers(0, SPAN), w=st.integers(0, SPAN))
def test_interval_algebra_against_sweep(a, b, lo, w):
    fa, fb = hb.flatten(a), hb.flatten(b)
    assert list(fa) == runs(sweep(a))
    assert list(hb.subtract(fa, fb)) == runs(sweep(a) & ~sweep(b))
    bounds = IV(lo, lo + w)
    comp = hb.complement(fa, bounds)
    assert list(comp) == runs(~sweep(a, lo, lo + w), lo) if w else list(comp) == []
    assert list(hb.intersect(fa, bounds)) == runs(sweep(a, lo, lo + w), lo) if w else True
    assert hb.total_duration(fa) == int(sweep(a).sum())


@st.composite
def traces(draw):
    n = draw(st.integers(0, 3))
    m = draw(st.integers(1 if n == 0 else 0, 3))
    host = []
    for r in range(n):
        t = 0
        for _ in range(draw(st.integers(1 if r == 0 else 0, 8))):
            t += draw(st.integers(0, 20))
            d = draw(st.integers(1, 40))
            host.append(hb.HostRecord(r, draw(st.sampled_from(list(hb.HostState))), IV(t, t + d)))
            t += d
    span = max([h.interval.end for h in host] + [60])
    dev = []
    for d in range(m):
        for _ in range(draw(st.integers(1 if (n == 0 and d == 0) else 0, 10))):
            s = draw(st.integers(0, span))
            dev.append(hb.DeviceRecord(d, draw(st.sampled_from(list(hb.DeviceActivityKind))),
                                       IV(s, s + draw(st.integers(1, 50))), draw(st.sampled_from([None, 0, 1, 2]))))
    return hb.Trace(host_processes=tuple(range(n)), devices=tuple(hb.DeviceDecl(d, d if d < n else None)
                                                                  for d in range(m)),
                    host_records=tuple(host), device_records=tuple(dev))


@settings(max_examples=120, deadline=None)
@given(t=traces())
def test_summaries_against_sweep_and_identities(t):
    r = hb.compute_report(t)
    E = r.elapsed_ns
    for s in r.host_summaries:
        mine = [x for x in t.host_records if x.rank == s.rank]
        off = sum(x.interval.duration for x in mine if x.state == hb.HostState.OFFLOAD)
        mpi = sum(x.interval.duration for x in mine if x.state == hb.HostState.MPI)
        assert (s.d_offload, s.d_mpi) == (off, mpi)
        assert s.d_useful + s.d_offload + s.d_mpi == s.span_end
    for s in r.device_summaries:
        recs = [x for x in t.device_records if x.device_id == s.device_id]
        k = sweep([x.interval for x in recs if x.kind == hb.DeviceActivityKind.KERNEL], 0, E)
        km = sweep([x.interval for x in recs], 0, E)
        assert s.d_kernel == int(k.sum())
        assert s.d_memory == int((km & ~k).sum())
        assert s.d_kernel + s.d_memory + s.d_idle == E
    if r.host is not None and r.host.mpi_parallel_efficiency is not None:
        h = r.host
        assert abs(h.parallel_efficiency - h.mpi_parallel_efficiency * h.device_offload_efficiency) <= \
            1e-12 * max(h.parallel_efficiency, 1e-300)
        assert abs(h.mpi_parallel_efficiency - h.mpi_communication_efficiency * h.mpi_load_balance) <= \
            1e-12 * h.mpi_parallel_efficiency
    if r.device is not None and r.device.load_balance is not None:
        d = r.device
        prod = d.load_balance * d.communication_efficiency * d.orchestration_efficiency
        assert abs(d.parallel_efficiency - prod) <= 1e-12 * max(d.parallel_efficiency, 1e-300)
    # stream obliviousness (acceptance criterion 6)
    t2 = hb.Trace(host_processes=t.host_processes, devices=t.devices, host_records=t.host_records,
                  device_records=tuple(hb.DeviceRecord(x.device_id, x.kind, x.interval,
                                                       None if x.stream else 5) for x in t.device_records))
    r2 = hb.compute_report(t2)
    assert (r2.elapsed_ns, r2.host, r2.device, r2.device_summaries) == (r.elapsed_ns, r.host, r.device,
                                                                         r.device_summaries)
