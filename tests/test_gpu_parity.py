"""Parity of the B200 engine (through the drop-in API and the C ABI) with the
reference's own outputs (golden fixtures) and with the C oracle."""

from __future__ import annotations

import re

import numpy as np
import pytest

from conftest import gpu_available
from golden_io import load, to_trace, unhex

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

import paper_2603_26576_b200 as hb  # noqa: E402
from paper_2603_26576_b200 import _native as N  # noqa: E402
from paper_2603_26576_b200.engine import analyze_packed  # noqa: E402
from paper_2603_26576_b200.packing import PackedTrace, RecordColumns  # noqa: E402

HOST_FIELDS = ("parallel_efficiency", "mpi_parallel_efficiency", "mpi_communication_efficiency",
               "mpi_load_balance", "device_offload_efficiency")
DEV_FIELDS = ("parallel_efficiency", "load_balance", "communication_efficiency", "orchestration_efficiency")

CASES = load("presets") + load("acceptance") + load("invalid")


def _check_report(r, rep):
    assert r.elapsed_ns == rep["E"]
    assert (r.n, r.m) == (rep["n"], rep["m"])
    assert [[s.rank, s.d_useful, s.d_offload, s.d_mpi, s.span_end] for s in r.host_summaries] == rep["hs"]
    assert [[s.device_id, s.d_kernel, s.d_memory, s.d_idle] for s in r.device_summaries] == rep["ds"]
    if rep["host"] is None:
        assert r.host is None
    else:
        assert [getattr(r.host, f) for f in HOST_FIELDS] == [unhex(v) for v in rep["host"]]
    if rep["device"] is None:
        assert r.device is None
    else:
        assert [getattr(r.device, f) for f in DEV_FIELDS] == [unhex(v) for v in rep["device"]]
    assert list(r.warnings) == rep["warnings"]


@pytest.mark.parametrize("case", CASES, ids=[c["tag"] for c in CASES])
def test_compute_report_and_validate_match_reference(case):
    t = to_trace(case["trace"])
    rep = case["report"]
    if rep.get("raise") == "InvalidTraceError":
        with pytest.raises(hb.InvalidTraceError) as ei:
            hb.compute_report(t)
        assert str(ei.value) == rep["msg"]
    elif rep.get("raise") == "AnalysisError":
        with pytest.raises(hb.AnalysisError) as ei:
            hb.compute_report(t)
        assert str(ei.value) == rep["msg"]
    else:
        _check_report(hb.compute_report(t), rep)
    v = hb.validate(t)
    assert v.errors == case["validate"]["errors"]
    assert v.warnings == case["validate"]["warnings"]


SD = load("summarize_device")


@pytest.mark.parametrize("case", SD[::3], ids=[c["tag"] for c in SD[::3]])
def test_summarize_device_window(case):
    t = to_trace(case["trace"])
    s, w = hb.summarize_device(t, case["elapsed"])
    assert [[x.device_id, x.d_kernel, x.d_memory, x.d_idle] for x in s] == case["ds"]
    assert w == case["warnings"]


def test_metrics_stage_functions():
    for c in load("metrics"):
        hs = [hb.HostSummary(*x) for x in c["hs"]]
        got = hb.host_metrics(hs, c["E"])
        assert [getattr(got, f) for f in HOST_FIELDS] == [unhex(v) for v in c["host"]]
        ds = [hb.DeviceSummary(*x) for x in c["ds"]]
        got = hb.device_metrics(ds, c["Ed"])
        assert [getattr(got, f) for f in DEV_FIELDS] == [unhex(v) for v in c["device"]]


def test_stage_function_errors():
    with pytest.raises(ValueError):
        hb.host_metrics([], 10)
    with pytest.raises(ValueError):
        hb.device_metrics([hb.DeviceSummary(0, 1, 0, 0)], 0)
    t = hb.Trace(host_processes=(0,), devices=(hb.DeviceDecl(0),),
                 host_records=(hb.HostRecord(0, hb.HostState.USEFUL, hb.Interval(0, 10)),))
    with pytest.raises(ValueError):
        hb.summarize_device(t, 0)
    bad = hb.Trace(host_processes=(0,), host_records=(hb.HostRecord(0, hb.HostState.USEFUL, hb.Interval(0, 10)),
                                                      hb.HostRecord(0, hb.HostState.MPI, hb.Interval(5, 15))))
    with pytest.raises(hb.InvalidTraceError, match="overlap"):
        hb.summarize_host(bad)


# ---------------------------------------------------------------------------
# engine vs oracle on adversarial SoA shapes (tile boundaries, long carries)
# ---------------------------------------------------------------------------
def _canonical(start, end, res, kind, host):
    kr = np.array([2, 1, 0], dtype=np.uint8)[kind] if host else kind
    order = np.lexsort((kr, end, start, res))
    return start[order], end[order], res[order], kind[order]


def _random_side(rng, n_res, counts, host, long_frac=0.0, zero_frac=0.0, bad_frac=0.0, span=10 ** 6):
    res = np.repeat(np.arange(n_res, dtype=np.int32), counts)
    k = res.size
    start = rng.integers(0, span, size=k, dtype=np.uint64)
    dur = rng.integers(1, max(2, span // max(1, k // max(n_res, 1)) * 3), size=k, dtype=np.uint64)
    if long_frac:
        longm = rng.random(k) < long_frac
        dur[longm] = rng.integers(span // 4, span, size=int(longm.sum()), dtype=np.uint64)
    if zero_frac:
        dur[rng.random(k) < zero_frac] = 0
    end = start + dur
    if bad_frac:
        badm = rng.random(k) < bad_frac
        end[badm] = start[badm] - np.minimum(start[badm], np.uint64(3))
    kind = rng.integers(0, 3 if host else 2, size=k, dtype=np.uint8)
    return _canonical(start, end, res, kind, host)


def _host_chain(rng, n_res, counts, gap=20, dur=200):
    res = np.repeat(np.arange(n_res, dtype=np.int32), counts)
    g = rng.integers(0, gap + 1, size=res.size).astype(np.uint64)
    d = rng.integers(1, dur + 1, size=res.size).astype(np.uint64)
    inc = g + d
    cs = np.cumsum(inc)
    offs = np.concatenate([[0], np.cumsum(counts)])
    base = np.zeros(n_res, dtype=np.uint64)
    nz = offs[:-1] > 0
    base[nz] = cs[offs[:-1][nz] - 1]
    start = cs - np.repeat(base, counts) - d
    kind = rng.integers(0, 3, size=res.size, dtype=np.uint8)
    return _canonical(start.astype(np.uint64), (start + d).astype(np.uint64), res, kind, True)


def _engine_vs_oracle(h, d, n, m, mode=N.MODE_REPORT, elapsed=0):
    from oracle import oracle as O
    packed = PackedTrace(RecordColumns(*h), RecordColumns(*d), list(range(n)), list(range(m)),
                         np.arange(n, dtype=np.int32), np.arange(m, dtype=np.int32), n, m, n, m)
    got = analyze_packed(packed, mode, elapsed, want_lists=True, capacity=1 << 20)
    ref = O.analyze(h, d, n, m, mode=mode, elapsed=elapsed, cap=1 << 20)
    assert got.status == ref.status
    # summarize_device never reports validate()'s late warnings (summarize.py:95-138)
    lists = (0, 1, 2, 4, 5, 6, 7) if mode != N.MODE_SUMMARIZE_DEVICE else (0, 1, 2, 4, 5, 6)
    assert [got.counts[c] for c in lists + (3,)] == [ref.counts[c] for c in lists + (3,)]
    for c in lists:
        assert np.array_equal(got.lists[c], np.sort(ref.lists[c])), c
    assert np.array_equal(got.lists[3], np.sort(ref.lists[3][:, 1]))
    if ref.status == 0:
        assert got.elapsed == ref.elapsed
        assert np.array_equal(got.host_sum, ref.host_sum)
        assert np.array_equal(got.dev_sum, ref.dev_sum)
        assert got.host_metrics == ref.host_metrics
        assert got.device_metrics == ref.device_metrics
    return got, ref


SHAPES = [
    # (name, n, host counts, m, dev counts, long_frac)
    ("tiny_segments", 300, "small", 700, "small", 0.0),
    ("one_giant_device", 1, "big", 1, "huge", 0.001),
    ("giant_long_carry", 2, "big", 3, "huge", 0.0002),
    ("ragged", 37, "mixed", 91, "mixed", 0.01),
    ("empty_resources", 50, "sparse", 50, "sparse", 0.0),
]


def _counts(rng, kind, k):
    if kind == "small":
        return rng.integers(0, 6, size=k)
    if kind == "big":
        return rng.integers(20_000, 60_000, size=k)
    if kind == "huge":
        return rng.integers(150_000, 400_000, size=k)
    if kind == "sparse":
        c = rng.integers(0, 3000, size=k)
        c[rng.random(k) < 0.5] = 0
        return c
    return rng.integers(0, 9000, size=k)


@pytest.mark.parametrize("shape", SHAPES, ids=[s[0] for s in SHAPES])
@pytest.mark.parametrize("seed", [1, 2])
def test_engine_matches_oracle_on_shapes(shape, seed):
    name, n, hc, m, dc, long_frac = shape
    rng = np.random.default_rng(seed * 1000 + len(name))
    h = _host_chain(rng, n, _counts(rng, hc, n))
    d = _random_side(rng, m, _counts(rng, dc, m), host=False, long_frac=long_frac,
                     span=int(h[1].max()) if h[1].size else 10 ** 6)
    _engine_vs_oracle(h, d, n, m)
    for el in (1, int(h[1].max() // 2) + 1 if h[1].size else 7):
        _engine_vs_oracle(h, d, n, m, N.MODE_SUMMARIZE_DEVICE, el)


@pytest.mark.parametrize("seed", [3, 4, 5])
def test_engine_matches_oracle_on_invalid_traces(seed):
    rng = np.random.default_rng(seed)
    n, m = 40, 60
    h = _random_side(rng, n, rng.integers(0, 12000, size=n), host=True, zero_frac=0.01, bad_frac=0.001,
                     span=10 ** 7)
    d = _random_side(rng, m, rng.integers(0, 12000, size=m), host=False, zero_frac=0.01, bad_frac=0.001,
                     long_frac=0.001, span=10 ** 7)
    got, ref = _engine_vs_oracle(h, d, n, m, N.MODE_VALIDATE)
    assert got.counts[3] > 0   # overlaps, many of them across tile boundaries


def test_device_only_trace_matches_oracle():
    rng = np.random.default_rng(11)
    m = 5
    d = _random_side(rng, m, rng.integers(5000, 30000, size=m), host=False, long_frac=0.001)
    empty = (np.zeros(0, np.uint64), np.zeros(0, np.uint64), np.zeros(0, np.int32), np.zeros(0, np.uint8))
    _engine_vs_oracle(empty, d, 0, m)


def test_contract_violation_is_reported():
    rng = np.random.default_rng(5)
    n = 3
    h = list(_host_chain(rng, n, np.array([5000, 5000, 5000])))
    h[0] = h[0].copy()
    h[0][7000] = 0   # start goes backwards inside rank 1
    packed = PackedTrace(RecordColumns(*h), RecordColumns(np.zeros(0, np.uint64), np.zeros(0, np.uint64),
                                                          np.zeros(0, np.int32), np.zeros(0, np.uint8)),
                         list(range(n)), [], np.arange(n, dtype=np.int32), np.zeros(0, np.int32), n, 0, n, 0)
    f = analyze_packed(packed, N.MODE_REPORT, want_lists=False)
    assert f.status == N.CONTRACT
    assert f.contract_flags & 1
    assert f.contract_index == 7000


def test_repeated_calls_are_deterministic_and_self_cleaning():
    rng = np.random.default_rng(9)
    h = _host_chain(rng, 8, rng.integers(1000, 40000, size=8))
    d = _random_side(rng, 8, rng.integers(1000, 40000, size=8), host=False, long_frac=0.001,
                     span=int(h[1].max()))
    first, _ = _engine_vs_oracle(h, d, 8, 8)
    for _ in range(5):
        again, _ = _engine_vs_oracle(h, d, 8, 8)
        assert np.array_equal(first.dev_sum, again.dev_sum)


@pytest.mark.parametrize("k", [20_000, 5_281, 3])
def test_device_start_outside_the_tile_window(k):
    """A malformed last record (start > end) whose START lies 2^32 ns past its
    predecessor's while its end stays inside the tile's 2^32 window: tile-relative
    32-bit values would show a well-ordered, positive-length record."""
    rng = np.random.default_rng(21)
    n, m = 1, 1
    h = _host_chain(rng, n, np.array([3000]))
    base = np.uint64(10 ** 12)
    s = base + np.sort(rng.integers(0, 2 ** 31, size=k, dtype=np.uint64))
    e = s + rng.integers(1, 5000, size=k, dtype=np.uint64)
    s[-1] = s[-2] + np.uint64(2 ** 32 + 1)
    e[-1] = s[-2] + np.uint64(1000)
    d = (s, e, np.zeros(k, np.int32), rng.integers(0, 2, size=k, dtype=np.uint8))
    he = h[1] + base
    he[-1] += np.uint64(2 ** 34)                 # E after every device end
    got, ref = _engine_vs_oracle((h[0] + base, he, h[2], h[3]), d, n, m, N.MODE_VALIDATE)
    assert ref.counts[4] == 1 and got.counts[4] == 1 and ref.counts[3] == 0


@pytest.mark.parametrize("depth", [2, 8, 64])
def test_device_carry_correction_on_overlapping_streams(depth):
    """Overlapping device streams (arrival process): most threads' first records start
    before the running max carried in from earlier threads of the tile."""
    rng = np.random.default_rng(depth)
    n, m = 4, 4
    h = _host_chain(rng, n, np.array([20_000] * n))
    counts = np.array([60_000] * m)
    res = np.repeat(np.arange(m, dtype=np.int32), counts)
    gaps = rng.integers(0, 40, size=res.size).astype(np.uint64)
    start = np.concatenate([np.cumsum(gaps[o:o + c]) for o, c in zip(np.r_[0, np.cumsum(counts)[:-1]], counts)])
    dur = rng.integers(1, 40 * depth, size=res.size).astype(np.uint64)
    d = _canonical(start.astype(np.uint64), start.astype(np.uint64) + dur, res,
                   rng.integers(0, 2, size=res.size, dtype=np.uint8), False)
    _engine_vs_oracle(h, d, n, m)
    for el in (int(h[1].max() // 3) + 1, int(d[1].max()) + 10):
        _engine_vs_oracle(h, d, n, m, N.MODE_SUMMARIZE_DEVICE, el)


@pytest.mark.parametrize("offset", [2 ** 64 - 10 ** 9, 2 ** 64 - 2 ** 33 - 12345, 2 ** 32 - 5000])
def test_timestamps_at_the_top_of_u64_and_across_a_32_bit_boundary(offset):
    """Records near U64_MAX (the tile-relative 32-bit windows and E sit at the top of
    the range) and records straddling a 2^32 boundary, through the engine vs the oracle."""
    rng = np.random.default_rng(offset % 997)
    n, m = 3, 4
    h = _host_chain(rng, n, np.array([6000, 9000, 7000]))
    d = _random_side(rng, m, np.array([8000, 12000, 0, 9000]), host=False, long_frac=0.001,
                     span=int(h[1].max()))
    top = np.uint64(offset)
    hs = (h[0] + top, h[1] + top, h[2], h[3])
    ds = (d[0] + top, d[1] + top, d[2], d[3])
    assert int(max(hs[1].max(), ds[1].max())) <= 2 ** 64 - 1
    got, _ = _engine_vs_oracle(hs, ds, n, m)        # report mode compares the finding lists too
    assert got.elapsed == int(hs[1].max())
    _engine_vs_oracle(hs, ds, n, m, N.MODE_SUMMARIZE_DEVICE, int(hs[1].max()) - 1000)


QUARANTINE = load("quarantine")


def _expect(fn, want):
    if "raise" in want:
        exc = {"InvalidTraceError": hb.InvalidTraceError, "ValueError": ValueError,
               "AnalysisError": hb.AnalysisError}[want["raise"]]
        with pytest.raises(exc) as ei:
            fn()
        assert str(ei.value) == want["msg"]
    else:
        assert fn() == want["ok"]


@pytest.mark.parametrize("case", QUARANTINE, ids=[c["tag"] for c in QUARANTINE])
def test_out_of_domain_timestamps_match_reference(case):
    """Records outside the u64 domain never reach the kernels (packing.py quarantine); the
    reference still reports them -- validate() (incl. their late-device warnings,
    model.py:217-228), compute_report, and the stage functions summarize_host /
    summarize_device must raise exactly as the reference does (summarize.py:57-138)."""
    test_compute_report_and_validate_match_reference(case)
    t = to_trace(case["trace"])

    def sh():
        s, E = hb.summarize_host(t)
        return [[x.rank, x.d_useful, x.d_offload, x.d_mpi, x.span_end] for x in s] + [E]

    _expect(sh, case["summarize_host"])
    for E, want in case["summarize_device"].items():
        def sd(E=int(E)):
            s, w = hb.summarize_device(t, E)
            return [[[x.device_id, x.d_kernel, x.d_memory, x.d_idle] for x in s], w]
        _expect(sd, want)
