"""The analysis kernel reading CSR offsets directly (17 B per interval: the producer
warp locates each tile's resources in the offset table and writes their ids into
shared memory) must equal the res-column path AND the C oracle bit for bit -- on
tiny segments (many resources per tile: several offset windows), empty resources,
>16384 ids (a third search level), one-resource traces, invalid traces (the error
path expands the offsets), every mode, and broken offset tables (CONTRACT, never
an out-of-range access).  Also: the persistent kernel makes progress without
co-residency (grids of 1 CTA and of many waves give the same results)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

import torch  # noqa: E402

from paper_2603_26576_b200 import _native as N  # noqa: E402
from paper_2603_26576_b200.engine import DeviceTrace, analyze_device  # noqa: E402
from test_gpu_parity import _host_chain, _random_side  # noqa: E402

EMPTY = (np.zeros(0, np.uint64), np.zeros(0, np.uint64), np.zeros(0, np.int32), np.zeros(0, np.uint8))


def _cuda(x):
    x = np.ascontiguousarray(x)
    return torch.from_numpy(x.view(np.int64) if x.dtype == np.uint64 else x).cuda()


def _seg(res, k):
    return np.concatenate([[0], np.cumsum(np.bincount(res, minlength=k)[:k])]).astype(np.int64)


def _dt(h, d, n, m, csr=True, hseg=None, dseg=None):
    dt = DeviceTrace(*(_cuda(x) for x in (*h, *d)), n, m)
    if not csr:
        return dt
    hs = _seg(h[2], n) if hseg is None else hseg
    ds = _seg(d[2], m) if dseg is None else dseg
    return DeviceTrace(dt.h_start, dt.h_end, dt.h_res, dt.h_kind, dt.d_start, dt.d_end, dt.d_res, dt.d_kind, n, m,
                       0, _cuda(hs), _cuda(ds))


def _same(a, b):
    assert (a.status, a.contract_flags, a.contract_index) == (b.status, b.contract_flags, b.contract_index)
    assert (a.elapsed, a.host_elapsed, a.dev_max_end, a.counts) == (b.elapsed, b.host_elapsed, b.dev_max_end, b.counts)
    if a.status != N.OK:
        # an invalid trace's partial sums are never observable (the reference raises;
        # api.py raises) and may differ between the two kernel compilations
        return
    assert a.host_metrics == b.host_metrics and a.device_metrics == b.device_metrics
    assert np.array_equal(a.host_sum, b.host_sum) and np.array_equal(a.dev_sum, b.dev_sum)


def _vs_oracle(f, h, d, n, m, mode, elapsed):
    from oracle import oracle as O
    ref = O.analyze(h, d, n, m, mode=mode, elapsed=elapsed)
    assert f.status == ref.status
    # summarize_device never reports validate()'s late warnings (summarize.py:95-138)
    lists = {N.MODE_SUMMARIZE_DEVICE: range(7), N.MODE_SUMMARIZE_HOST: range(4)}.get(mode, range(8))
    assert [f.counts[c] for c in lists] == [ref.counts[c] for c in lists]
    if ref.status == 0 and mode in (N.MODE_REPORT, N.MODE_SUMMARIZE_HOST):
        assert f.elapsed == ref.elapsed and np.array_equal(f.host_sum, ref.host_sum)
    if ref.status == 0 and mode in (N.MODE_REPORT, N.MODE_SUMMARIZE_DEVICE):
        assert np.array_equal(f.dev_sum, ref.dev_sum)
    if ref.status == 0 and mode == N.MODE_REPORT:
        assert f.host_metrics == ref.host_metrics and f.device_metrics == ref.device_metrics


SHAPES = {
    # name: (n, host counts, m, device counts, long_frac)
    "tiny_segments": (3000, "tiny", 7000, "tiny", 0.0),        # ~0-3 records per resource: many windows per tile
    "beyond_16k_ids": (20000, "tiny", 40000, "tiny", 0.0),      # three search levels
    "empty_resources": (80, "sparse", 80, "sparse", 0.001),
    "ragged": (37, "mixed", 91, "mixed", 0.01),
    "one_resource": (1, "huge", 1, "huge", 0.001),
    "device_only": (0, None, 9, "mixed", 0.001),
    "host_only": (9, "mixed", 0, None, 0.0),
}


def _counts(rng, kind, k):
    if kind == "tiny":
        return rng.integers(0, 4, size=k)
    if kind == "sparse":
        c = rng.integers(0, 9000, size=k)
        c[rng.random(k) < 0.5] = 0
        c[0] = c[-1] = 0
        return c
    if kind == "huge":
        return rng.integers(150_000, 300_000, size=k)
    return rng.integers(0, 9000, size=k)


def _make(name, seed):
    n, hk, m, dk, lf = SHAPES[name]
    rng = np.random.default_rng(seed * 77 + len(name))
    h = _host_chain(rng, n, _counts(rng, hk, n)) if n else EMPTY
    span = int(h[1].max()) if h[1].size else 10 ** 6
    d = _random_side(rng, m, _counts(rng, dk, m), host=False, long_frac=lf, span=span) if m else EMPTY
    return h, d, n, m


@pytest.mark.parametrize("name", list(SHAPES))
@pytest.mark.parametrize("mode", [N.MODE_REPORT, N.MODE_VALIDATE, N.MODE_SUMMARIZE_HOST, N.MODE_SUMMARIZE_DEVICE])
def test_csr_equals_columns_and_oracle(name, mode):
    h, d, n, m = _make(name, 1)
    el = (int(h[1].max()) // 2 + 1 if h[1].size else 12345) if mode == N.MODE_SUMMARIZE_DEVICE else 0
    got = analyze_device(_dt(h, d, n, m, csr=True), mode, elapsed=el)
    ref = analyze_device(_dt(h, d, n, m, csr=False), mode, elapsed=el)
    _same(got, ref)
    _vs_oracle(got, h, d, n, m, mode, el)


@pytest.mark.parametrize("seed", [3, 4])
def test_csr_invalid_traces_take_the_error_path(seed):
    """Overlapping host records (the error-path kernels walk an expanded res column),
    zero-length and malformed records, late device records."""
    rng = np.random.default_rng(seed)
    n, m = 40, 60
    h = _random_side(rng, n, rng.integers(0, 12000, size=n), host=True, zero_frac=0.01, bad_frac=0.001,
                     span=10 ** 7)
    d = _random_side(rng, m, rng.integers(0, 12000, size=m), host=False, zero_frac=0.01, bad_frac=0.001,
                     long_frac=0.001, span=10 ** 7)
    got = analyze_device(_dt(h, d, n, m, csr=True), N.MODE_VALIDATE)
    ref = analyze_device(_dt(h, d, n, m, csr=False), N.MODE_VALIDATE)
    _same(got, ref)
    assert got.counts[3] > 0
    _vs_oracle(got, h, d, n, m, N.MODE_VALIDATE, 0)


def test_csr_start_order_violation_is_a_contract_error():
    rng = np.random.default_rng(5)
    n = 3
    h = list(_host_chain(rng, n, np.array([5000, 5000, 5000])))
    h[0] = h[0].copy()
    h[0][7000] = 0
    got = analyze_device(_dt(tuple(h), EMPTY, n, 0, csr=True))
    ref = analyze_device(_dt(tuple(h), EMPTY, n, 0, csr=False))
    assert got.status == N.CONTRACT and got.contract_index == 7000
    _same(got, ref)


@pytest.mark.parametrize("bad", ["decreasing", "not_from_zero", "short_total", "long_total"])
def test_broken_offset_tables_are_contract_errors(bad):
    rng = np.random.default_rng(8)
    n = 6
    counts = np.array([3000, 9000, 100, 7000, 4000, 2500])
    h = _host_chain(rng, n, counts)
    seg = _seg(h[2], n)
    if bad == "decreasing":
        seg[3], seg[4] = seg[4], seg[3]
    elif bad == "not_from_zero":
        seg[0] = 5
    elif bad == "short_total":
        seg[-1] -= 17
    else:
        seg[-1] += 17
    f = analyze_device(_dt(h, EMPTY, n, 0, csr=True, hseg=seg))
    assert f.status == N.CONTRACT and f.contract_flags & N.CONTRACT_HOST_ORDER


@pytest.mark.parametrize("grid", [1, 7, 148 * 6, 5000])
def test_progress_without_co_residency(grid):
    """The device tiles wait for E only on a count of finished HOST tiles (claimed in
    order by running CTAs), never on the whole grid being resident: a grid of many waves
    (CTAs that cannot all be resident at once) completes and matches the default grid."""
    h, d, n, m = _make("ragged", 2)
    ctx = N.context()
    lib = N.load()
    base = analyze_device(_dt(h, d, n, m))
    try:
        assert lib.heteff_set_grid(ctx, grid) == N.OK
        for csr in (True, False):
            _same(analyze_device(_dt(h, d, n, m, csr=csr)), base)
    finally:
        lib.heteff_set_grid(ctx, 0)


def test_many_wave_grid_on_a_config_shard():
    """C3-shaped shard (overlapping streams: look-back + carry fix-ups) on 20 waves of CTAs."""
    from paper_2603_26576_b200.configs import CONFIGS
    from paper_2603_26576_b200.synth import generate
    dt = generate(CONFIGS["c3"], 0, 8)
    base = analyze_device(dt)
    ctx, lib = N.context(), N.load()
    try:
        lib.heteff_set_grid(ctx, 148 * 20)
        _same(analyze_device(dt), base)
        _same(analyze_device(dt.columns_only()), base)
    finally:
        lib.heteff_set_grid(ctx, 0)
