"""The block-compressed host -> HBM column transfer of the host-buffer entry points
(csrc/transfer.cu): whatever the widths a block needs -- 1-, 2-, 4-byte offsets and
durations, raw 8-byte starts (spans beyond 32 bits, timestamps near 2^64), raw ends
(durations beyond 32 bits, ends before their starts) -- and at every block / chunk
boundary, the analysis of the transferred columns must be bit-identical to the raw copy
and to the device-resident analysis of the same columns."""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

from paper_2603_26576_b200 import _native as N  # noqa: E402
from paper_2603_26576_b200.configs import CONFIGS, scaled  # noqa: E402
from paper_2603_26576_b200.engine import DeviceTrace, analyze_device, analyze_host_columns  # noqa: E402
from paper_2603_26576_b200.synth import generate  # noqa: E402
from test_gpu_csr import _same, _seg  # noqa: E402


def _identical(a, b):
    """Codec vs raw copy: the same kernel on what must be the same columns -- every output,
    partial sums of invalid traces included."""
    assert (a.status, a.contract_flags, a.contract_index) == (b.status, b.contract_flags, b.contract_index)
    assert (a.elapsed, a.host_elapsed, a.dev_max_end, a.counts) == (b.elapsed, b.host_elapsed, b.dev_max_end, b.counts)
    assert a.host_metrics == b.host_metrics and a.device_metrics == b.device_metrics
    assert np.array_equal(a.host_sum, b.host_sum) and np.array_equal(a.dev_sum, b.dev_sum)


def _host_trace(h, d, n, m):
    cols = [torch.from_numpy(np.ascontiguousarray(x).view(np.int64) if x.dtype == np.uint64 else
                             np.ascontiguousarray(x)).pin_memory() for x in (*h, *d)]
    return DeviceTrace(*cols, n, m)


def _dev_trace(h, d, n, m):
    cols = [torch.from_numpy(np.ascontiguousarray(x).view(np.int64) if x.dtype == np.uint64 else
                             np.ascontiguousarray(x)).cuda() for x in (*h, *d)]
    return DeviceTrace(*cols, n, m)


def _run_host(h, d, n, m, mode, codec: bool):
    old = {k: os.environ.get(k) for k in ("HETEFF_CODEC_MIN", "HETEFF_RAW_TRANSFER")}
    os.environ["HETEFF_CODEC_MIN"] = "1" if codec else str(1 << 62)
    os.environ["HETEFF_RAW_TRANSFER"] = "0" if codec else "1"
    try:
        return analyze_host_columns(_host_trace(h, d, n, m), mode, csr=(_seg(h[2], n), _seg(d[2], m)))
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _side(rng, k, n_res, start0, span_bits, dur_bits, sort=True):
    res = np.sort(rng.integers(0, n_res, size=k)).astype(np.int32)
    s = (np.uint64(start0) + rng.integers(0, 1 << span_bits, size=k, dtype=np.uint64)).astype(np.uint64)
    dur = rng.integers(0, 1 << dur_bits, size=k, dtype=np.uint64)
    e = s + dur
    kind = rng.integers(0, 3, size=k, dtype=np.uint8)
    if sort:
        o = np.lexsort((e, s, res))
        s, e, res, kind = s[o], e[o], res[o], kind[o]
    return s, e, res, kind


CASES = {
    # name: (host records, device records, span bits, duration bits, start0)
    "narrow": (70_000, 90_000, 20, 7, 10 ** 9),
    "two_byte": (5000, 4097, 12, 15, 7),
    "four_byte": (4096, 8193, 31, 31, 2 ** 40),
    "raw_spans": (12_000, 9000, 40, 10, 5),
    "raw_durations": (9000, 12_000, 24, 36, 3),
    "top_of_u64": (4097, 4095, 30, 20, 2 ** 64 - 2 ** 31),
    "chunk_edges": ((1 << 20) + 1, (1 << 20) - 1, 22, 9, 123),
    "one_record": (1, 1, 4, 4, 9),
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("mode", [N.MODE_REPORT, N.MODE_VALIDATE])
def test_codec_equals_raw_transfer_and_device(name, mode):
    hk, dk, span, durb, s0 = CASES[name]
    rng = np.random.default_rng(len(name) * 7 + mode)
    n, m = 5, 6
    h = _side(rng, hk, n, s0, span, durb)
    d = _side(rng, dk, m, s0, span, durb)
    h = (h[0], h[1], h[2], (h[3] % 3).astype(np.uint8))
    d = (d[0], d[1], d[2], (d[3] % 2).astype(np.uint8))
    a = _run_host(h, d, n, m, mode, codec=True)
    b = _run_host(h, d, n, m, mode, codec=False)
    _identical(a, b)
    dt = _dev_trace(h, d, n, m)
    c = analyze_device(DeviceTrace(dt.h_start, dt.h_end, dt.h_res, dt.h_kind, dt.d_start, dt.d_end, dt.d_res,
                                   dt.d_kind, n, m), mode)
    _same(a, c)


def test_codec_with_malformed_unsorted_and_zero_length_records():
    """Ends before starts (raw ends), unsorted blocks (the min start as base), zero-length
    records: the transferred columns must reproduce the findings and the contract index."""
    rng = np.random.default_rng(5)
    n, m = 3, 4
    h = _side(rng, 20_000, n, 10 ** 6, 18, 8)
    d = _side(rng, 30_000, m, 10 ** 6, 18, 8)
    hs, he = h[0].copy(), h[1].copy()
    he[::997] = hs[::997]                      # zero-length
    he[5::1999] = hs[5::1999] - np.uint64(3)   # malformed
    ds = d[0].copy()
    ds[100:110] = ds[100:110][::-1]            # out of order inside a block
    h = (hs, he, h[2], (h[3] % 3).astype(np.uint8))
    d = (ds, d[1], d[2], (d[3] % 2).astype(np.uint8))
    for mode in (N.MODE_REPORT, N.MODE_VALIDATE):
        _identical(_run_host(h, d, n, m, mode, True), _run_host(h, d, n, m, mode, False))


def test_codec_on_a_c5_rank_shard():
    """A 1.2e7-interval C5 shard (4-GPU ranks, overlapping streams) through the host-buffer
    CSR entry point, codec on: identical to the device-resident analysis."""
    cfg = CONFIGS["c5"]
    dt = generate(cfg, 0, 24)
    f = analyze_device(dt)
    host = DeviceTrace(*[None if x is None else x.cpu().pin_memory() for x in
                         (dt.h_start, dt.h_end, None, dt.h_kind, dt.d_start, dt.d_end, None, dt.d_kind)], dt.n, dt.m)
    g = analyze_host_columns(host, csr=(dt.h_seg.cpu().numpy(), dt.d_seg.cpu().numpy()))
    assert f.status == N.OK
    _same(f, g)


@pytest.mark.parametrize("k", [4095, 4097, 70_000, (1 << 20) + 3])
def test_codec_on_valid_traces_equals_device_resident(k):
    """Valid traces (disjoint host chains, overlapping device streams): status OK, so every
    summary and float is compared with the device-resident analysis (the other kernel
    compilation) as well as with the raw copy."""
    from test_gpu_parity import _host_chain
    rng = np.random.default_rng(k)
    n, m = 4, 4
    h = _host_chain(rng, n, np.array([k] * n))
    res = np.repeat(np.arange(m, dtype=np.int32), k)
    start = np.concatenate([np.cumsum(rng.integers(0, 300, size=k)) for _ in range(m)]).astype(np.uint64)
    dur = rng.integers(1, 3000, size=m * k).astype(np.uint64)
    kind = rng.integers(0, 2, size=m * k, dtype=np.uint8)
    d = (start, start + dur, res, kind)
    a = _run_host(h, d, n, m, N.MODE_REPORT, codec=True)
    assert a.status == N.OK
    _identical(a, _run_host(h, d, n, m, N.MODE_REPORT, codec=False))
    _same(a, analyze_device(_dev_trace(h, d, n, m)))
