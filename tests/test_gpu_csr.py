"""heteff_analyze_host_csr: the res columns as CSR offsets must give
exactly what the res-column path gives -- empty resources, one-sided traces, ragged
groups, contract violations inside a group."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

from paper_2603_26576_b200 import _native as N  # noqa: E402
from paper_2603_26576_b200.engine import DeviceTrace, analyze_host_columns  # noqa: E402
from test_gpu_parity import _host_chain, _random_side  # noqa: E402


def _seg(res, k):
    return np.concatenate([[0], np.cumsum(np.bincount(res, minlength=k))]).astype(np.int64)


def _pinned(h, d, n, m):
    cols = [torch.from_numpy(np.ascontiguousarray(x).view(np.int64) if x.dtype == np.uint64 else
                             np.ascontiguousarray(x)).pin_memory() for x in (*h, *d)]
    return DeviceTrace(*cols, n, m)


def _same(a, b):
    assert (a.status, a.contract_flags, a.contract_index) == (b.status, b.contract_flags, b.contract_index)
    assert (a.elapsed, a.host_elapsed, a.dev_max_end, a.counts) == (b.elapsed, b.host_elapsed, b.dev_max_end, b.counts)
    if a.status != N.OK:
        # an invalid trace's partial sums are never observable (the reference raises;
        # api.py raises) and may differ between the two kernel compilations
        return
    assert a.host_metrics == b.host_metrics and a.device_metrics == b.device_metrics
    assert np.array_equal(a.host_sum, b.host_sum) and np.array_equal(a.dev_sum, b.dev_sum)


EMPTY = (np.zeros(0, np.uint64), np.zeros(0, np.uint64), np.zeros(0, np.int32), np.zeros(0, np.uint8))


@pytest.mark.parametrize("shape", ["mixed", "empty_groups", "device_only", "host_only", "one_giant_group"])
@pytest.mark.parametrize("mode", [N.MODE_REPORT, N.MODE_VALIDATE, N.MODE_SUMMARIZE_HOST])
def test_csr_matches_res_columns(shape, mode):
    rng = np.random.default_rng(hash(shape) % 1000)
    n, m = {"mixed": (37, 91), "empty_groups": (60, 60), "device_only": (0, 7), "host_only": (9, 0),
            "one_giant_group": (1, 1)}[shape]
    hc = rng.integers(0, 9000, size=n)
    dc = rng.integers(0, 9000, size=m)
    if shape == "empty_groups":
        hc[rng.random(n) < 0.5] = 0
        dc[rng.random(m) < 0.5] = 0
        hc[0] = hc[-1] = dc[0] = dc[-1] = 0       # empty first / last groups
    if shape == "one_giant_group":
        hc, dc = np.array([300_000]), np.array([700_000])
    h = _host_chain(rng, n, hc) if n else EMPTY
    d = _random_side(rng, m, dc, host=False, long_frac=0.001) if m else EMPTY
    dt = _pinned(h, d, n, m)
    ref = analyze_host_columns(dt, mode)
    got = analyze_host_columns(dt, mode, csr=(_seg(h[2], n), _seg(d[2], m)))
    _same(got, ref)


def test_csr_order_violation_inside_a_group_is_a_contract_error():
    rng = np.random.default_rng(3)
    n, m = 3, 2
    h = list(_host_chain(rng, n, np.array([5000, 5000, 5000])))
    h[0] = h[0].copy()
    h[0][7000] = 0
    d = _random_side(rng, m, np.array([4000, 4000]), host=False)
    dt = _pinned(tuple(h), d, n, m)
    got = analyze_host_columns(dt, csr=(_seg(h[2], n), _seg(d[2], m)))
    ref = analyze_host_columns(dt)
    assert got.status == N.CONTRACT and got.contract_index == 7000
    _same(got, ref)
