"""K3 (csrc/sort.cu): the GPU radix sort into canonical order, and the
analysis of unsorted columns through it (``HETEFF_FLAG_SORT_IF_NEEDED``).

Oracles: numpy's stable lexsort for the permutation (bit-exact, ties in input
order) and the C oracle, which sorts its input canonically the way
``Trace.__post_init__`` does (model.py:74-80,99-107), for the analysis."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

import torch  # noqa: E402

from oracle import gen as ogen  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2603_26576_b200 import _native as N  # noqa: E402
from paper_2603_26576_b200.configs import CONFIGS  # noqa: E402
from paper_2603_26576_b200.engine import (DeviceTrace, analyze_device, analyze_host_columns,  # noqa: E402
                                          analyze_packed, sort_records)
from paper_2603_26576_b200.packing import PackedTrace, RecordColumns  # noqa: E402

TILE = 512 * 11


def _cuda(a: np.ndarray) -> torch.Tensor:
    if a.dtype == np.uint64:
        a = a.view(np.int64)
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _u64(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


def _check_sort(s, e, r, k):
    got = sort_records(_cuda(s), _cuda(e), _cuda(r), _cuda(k))
    perm = np.lexsort((s, r.astype(np.int64)))          # stable: ties keep input order
    assert np.array_equal(got.perm.cpu().numpy(), perm)
    assert np.array_equal(_u64(got.start), s[perm])
    assert np.array_equal(_u64(got.end), e[perm])
    assert np.array_equal(got.res.cpu().numpy(), r[perm])
    assert np.array_equal(got.kind.cpu().numpy(), k[perm])
    return got


def _random(rng, n, ids, span, lo=0):
    s = rng.integers(lo, lo + span, n, dtype=np.uint64) if span > 0 else np.full(n, lo, dtype=np.uint64)
    e = s + rng.integers(0, 100, n, dtype=np.uint64)
    r = rng.integers(0, ids, n, dtype=np.int32)
    k = rng.integers(0, 3, n, dtype=np.uint8)
    return s, e, r, k


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, TILE - 1, TILE, TILE + 1, 3 * TILE + 17, 250_000])
def test_sort_matches_stable_lexsort(n):
    rng = np.random.default_rng(n)
    _check_sort(*_random(rng, n, 97, 1 << 20))


def test_sort_many_ties_and_single_key():
    rng = np.random.default_rng(5)
    _check_sort(*_random(rng, 100_000, 3, 7))                # heavy ties: stability
    got = _check_sort(*_random(rng, 50_000, 1, 0, lo=123))   # zero key bits: identity
    assert got.passes == 0


def test_sort_extreme_timestamps_and_negative_ids():
    rng = np.random.default_rng(6)
    n = 40_000
    s = rng.integers(0, 1 << 63, n, dtype=np.uint64) * np.uint64(2) + rng.integers(0, 2, n, dtype=np.uint64)
    s[:3] = [0, (1 << 64) - 1, (1 << 63)]
    e = s.copy()
    r = rng.integers(-5, 1 << 20, n, dtype=np.int32)
    k = rng.integers(0, 2, n, dtype=np.uint8)
    got = _check_sort(s, e, r, k)
    assert got.wide          # 64 start bits + 21 id bits: two stable stages


def test_sort_time_ordered_log_sorts_by_resource_only():
    """A globally time-ordered event log (all devices interleaved) needs only the id passes."""
    rng = np.random.default_rng(8)
    n = 200_000
    s = np.sort(rng.integers(0, 1 << 40, n, dtype=np.uint64))
    r = rng.integers(0, 3000, n, dtype=np.int32)
    got = _check_sort(s, s + np.uint64(5), r, rng.integers(0, 2, n, dtype=np.uint8))
    assert got.start_sorted and got.key_bits == 12 and got.passes == 2


@pytest.mark.parametrize("ids,passes", [(200, 1), (70_000, 3), (1, 0)])
def test_sort_time_ordered_payload_pass_counts(ids, passes):
    """Start-ordered input carries start/end/kind through 0, 1 (odd) or 3 passes."""
    rng = np.random.default_rng(ids)
    n = 150_000
    s = np.sort(rng.integers(0, 1 << 50, n, dtype=np.uint64))
    r = rng.integers(0, ids, n, dtype=np.int32)
    got = _check_sort(s, s + rng.integers(0, 9, n, dtype=np.uint64), r, rng.integers(0, 2, n, dtype=np.uint8))
    assert got.start_sorted and got.passes == passes


@pytest.mark.parametrize("bits", [8, 17, 33, 47, 64])
def test_sort_key_widths(bits):
    rng = np.random.default_rng(bits)
    n = 60_000
    hi = (1 << bits) - 1
    s = (rng.integers(0, 1 << 62, n, dtype=np.uint64) & np.uint64(hi)) if bits < 64 else \
        rng.integers(0, 1 << 63, n, dtype=np.uint64) * np.uint64(2)
    r = rng.integers(0, 50, n, dtype=np.int32)
    got = _check_sort(s, s + np.uint64(0), r, np.zeros(n, dtype=np.uint8))
    assert got.passes >= 1


def test_sort_repeated_calls_and_shrinking_sizes():
    rng = np.random.default_rng(9)
    for n in (300_000, 1000, 300_000, 5, 120_000):
        _check_sort(*_random(rng, n, 1000, 1 << 30))


# ---------------------------------------------------------------------------
# analysis of unsorted columns
# ---------------------------------------------------------------------------
def _shuffled_config(name, seed, local=True):
    cfg = CONFIGS[name]
    (hs, he, hr, hk), (ds, de, dr, dk) = ogen.generate(cfg)
    rng = np.random.default_rng(seed)
    ph = rng.permutation(hs.size) if local else np.arange(hs.size)
    pd = rng.permutation(ds.size)
    return cfg, (hs, he, hr, hk), (ds, de, dr, dk), ph, pd


def _dt(h, d, n, m):
    return DeviceTrace(*(_cuda(x) for x in (*h, *d)), n, m)


def test_analyze_unsorted_columns_matches_oracle():
    cfg, h, d, ph, pd = _shuffled_config("c1", 3)
    n, m = cfg.n_ranks, cfg.n_devices
    hsh = tuple(x[ph] for x in h)
    dsh = tuple(x[pd] for x in d)
    plain = analyze_device(_dt(hsh, dsh, n, m))
    assert plain.status == N.CONTRACT
    assert plain.contract_flags & (N.CONTRACT_HOST_ORDER | N.CONTRACT_DEV_ORDER)
    got = analyze_device(_dt(hsh, dsh, n, m), sort_if_needed=True)
    ref = O.analyze(hsh, dsh, n, m)   # the oracle sorts canonically itself
    assert got.status == ref.status == N.OK
    assert got.elapsed == ref.elapsed
    assert np.array_equal(got.host_sum, ref.host_sum)
    assert np.array_equal(got.dev_sum, ref.dev_sum)
    assert got.host_metrics == ref.host_metrics and got.device_metrics == ref.device_metrics
    # same through the host-buffer entry point
    pinned = DeviceTrace(*(torch.from_numpy(np.ascontiguousarray(x.view(np.int64) if x.dtype == np.uint64 else x))
                           for x in (*hsh, *dsh)), n, m)
    got2 = analyze_host_columns(pinned, sort_if_needed=True)
    assert np.array_equal(got2.dev_sum, ref.dev_sum) and got2.device_metrics == ref.device_metrics


def test_unsorted_device_side_only_keeps_host_unsorted_path():
    cfg, h, d, _, pd = _shuffled_config("c1", 4, local=False)
    n, m = cfg.n_ranks, cfg.n_devices
    dsh = tuple(x[pd] for x in d)
    got = analyze_device(_dt(h, dsh, n, m), sort_if_needed=True)
    ref = O.analyze(h, d, n, m)
    assert got.status == N.OK
    assert np.array_equal(got.dev_sum, ref.dev_sum) and np.array_equal(got.host_sum, ref.host_sum)


def test_unsorted_findings_map_back_to_input_positions():
    """Findings lists of a sorted re-run name the caller's record positions."""
    rng = np.random.default_rng(11)
    n, m = 6, 5
    hs, he, hr, hk = _random(rng, 3000, n, 1 << 16)
    ds, de, dr, dk = _random(rng, 4000, m + 2, 1 << 16)   # undeclared devices m, m+1
    dk = (dk % 2).astype(np.uint8)
    de[::97] = ds[::97]                                  # zero-length records
    ds[5::101] = de[5::101] + np.uint64(3)               # malformed records
    pk = lambda s, e, r, k: RecordColumns(s, e, r, k)  # noqa: E731
    packed = PackedTrace(pk(hs, he, hr, hk), pk(ds, de, dr, dk), list(range(n)), list(range(m + 2)),
                         np.arange(n, dtype=np.int32), np.array(list(range(m)) + [-1, -1], dtype=np.int32),
                         n, m, n, m)
    got = analyze_packed(packed, N.MODE_VALIDATE, sort_if_needed=True)
    ph = np.lexsort((hs, hr))
    pd = np.lexsort((ds, dr))
    canon = PackedTrace(pk(hs[ph], he[ph], hr[ph], hk[ph]), pk(ds[pd], de[pd], dr[pd], dk[pd]), packed.host_ids,
                        packed.dev_ids, packed.host_decl, packed.dev_decl, n, m, n, m)
    ref = analyze_packed(canon, N.MODE_VALIDATE)
    assert got.counts == ref.counts
    for i in range(8):
        perm = ph if i < 4 else pd
        assert np.array_equal(np.sort(got.lists[i]), np.sort(perm[ref.lists[i]])), i


def test_c2_shuffled_full_size_bit_identical():
    """1e8 intervals: a shuffled device side analyzes bit-identically (size-independent)."""
    from paper_2603_26576_b200.synth import generate

    dt = generate(CONFIGS["c2"])
    ref = analyze_device(dt)
    g = torch.Generator(device="cuda").manual_seed(7)
    p = torch.randperm(dt.dev_count, device="cuda", generator=g)
    sh = DeviceTrace(dt.h_start, dt.h_end, dt.h_res, dt.h_kind, dt.d_start[p], dt.d_end[p], dt.d_res[p],
                     dt.d_kind[p], dt.n, dt.m)
    del p
    got = analyze_device(sh, sort_if_needed=True)
    assert got.status == N.OK and ref.status == N.OK
    assert got.elapsed == ref.elapsed
    assert np.array_equal(got.dev_sum, ref.dev_sum) and np.array_equal(got.host_sum, ref.host_sum)
    assert got.device_metrics == ref.device_metrics and got.host_metrics == ref.host_metrics


def test_analysis_plan_repeated_runs_match():
    """engine.AnalysisPlan (prebuilt ABI structs, one D2H per call) == analyze_device."""
    from paper_2603_26576_b200.engine import AnalysisPlan

    cfg, h, d, _, _ = _shuffled_config("c1", 1, local=False)
    dt = _dt(h, d, cfg.n_ranks, cfg.n_devices)
    ref = analyze_device(dt)
    plan = AnalysisPlan(dt)
    for _ in range(3):
        got = plan.run()
        assert got.status == N.OK and got.elapsed == ref.elapsed
        assert np.array_equal(got.host_sum, ref.host_sum) and np.array_equal(got.dev_sum, ref.dev_sum)
        assert got.host_metrics == ref.host_metrics and got.device_metrics == ref.device_metrics


@pytest.mark.parametrize("kmax", [4, 256])
def test_sort_keeps_kind_codes_that_do_not_fit_the_index(kmax):
    """Kinds ride in the index's top two bits; codes > 3 (contract violations the
    analysis reports) must still come out unchanged -- the finish gathers them."""
    rng = np.random.default_rng(kmax)
    s, e, r, _ = _random(rng, 3 * TILE + 5, 7, 10 ** 6)
    k = rng.integers(0, kmax, s.size, dtype=np.uint16).astype(np.uint8)
    _check_sort(s, e, r, k)


@pytest.mark.parametrize("case", ["malformed", "huge_duration", "max_duration_that_fits"])
def test_sort_end_column_with_and_without_the_duration_stash(case):
    """Durations ride in the key bits above the digit passes when every one fits; a
    malformed record (end < start) or a too-long duration falls back to the gather."""
    rng = np.random.default_rng(len(case))
    s, e, r, k = _random(rng, 2 * TILE + 3, 300, 10 ** 9)
    if case == "malformed":
        e[17] = s[17] - np.uint64(1)
    elif case == "huge_duration":
        e[5] = s[5] + np.uint64(2 ** 40)
    else:
        e[5] = s[5] + np.uint64(2 ** 20)    # 30 + 9 key bits -> 5 passes x 8 = 40 covered, 24 left
    _check_sort(s, e, r, k)
