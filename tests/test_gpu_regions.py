"""K5/K6 (csrc/regions.cu, EXTENSIONS): monitoring regions and the
offload-wait / device-busy overlap on the GPU.

Parity: (1) the fixtures made by running the REFERENCE on window-clipped
traces (tests/golden/make_golden.py ``regions_corpus``) through the drop-in
``region_reports``; (2) the C oracle's composition restatement
(``orc_regions``, itself pinned to those fixtures by
tests/test_oracle_regions.py) on larger config-shaped traces; (3) at full C4
size, size-independent identities: the window [0, 2^64-1) reproduces the
whole-trace analysis bit for bit, every region satisfies the partition
identities, and nested windows are monotone."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import gpu_available
from golden_io import load, to_trace, unhex

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

import torch  # noqa: E402

import paper_2603_26576_b200 as hb  # noqa: E402
from oracle import gen as ogen  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2603_26576_b200 import _native as N  # noqa: E402
from paper_2603_26576_b200.configs import CONFIGS, scaled  # noqa: E402
from paper_2603_26576_b200.engine import DeviceTrace, analyze_device, analyze_regions  # noqa: E402

HOST_FIELDS = ("parallel_efficiency", "mpi_parallel_efficiency", "mpi_communication_efficiency",
               "mpi_load_balance", "device_offload_efficiency")
DEV_FIELDS = ("parallel_efficiency", "load_balance", "communication_efficiency", "orchestration_efficiency")
REG = load("regions")
CASES = [c for c in REG if "trace" in c]
CONFIG_CASES = [c for c in REG if "config" in c]
U64_MAX = (1 << 64) - 1


@pytest.mark.parametrize("case", CASES, ids=[c["tag"] for c in CASES])
def test_region_reports_match_reference(case):
    t = to_trace(case["trace"])
    got = hb.region_reports(t, case["windows"])
    assert len(got) == len(case["regions"])
    for g, reg in zip(got, case["regions"]):
        rep = reg["report"]
        if rep.get("raise") == "AnalysisError":
            assert g.report is None
            continue
        r = g.report
        assert r.elapsed_ns == rep["E"]
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
        assert list(g.offload_busy) == reg["busy"]
        assert g.offload_busy_fraction == unhex(reg["frac"])


def _cuda(a):
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a.view(np.int64) if a.dtype == np.uint64 else a).cuda()


def _dt(h, d, n, m):
    return DeviceTrace(*(_cuda(x) for x in (*h, *d)), n, m)


def _compare(run, ref, R):
    assert run.status == N.OK
    for j in range(R):
        g = run.regions[j]
        assert g.status == int(ref.status[j]), j
        if g.status != N.OK:
            continue
        assert g.elapsed == int(ref.elapsed[j]), j
        assert np.array_equal(g.host_sum, ref.host_sum[j]), j
        assert np.array_equal(g.dev_sum, ref.dev_sum[j]), j
        assert np.array_equal(g.offload_busy, ref.busy[j]), j
        assert g.host_metrics == ref.host_metrics[j], j
        assert g.device_metrics == ref.device_metrics[j], j
        assert g.offload_busy_fraction == ref.busy_frac[j], j


@pytest.mark.parametrize("case", CONFIG_CASES, ids=[c["tag"] for c in CONFIG_CASES])
def test_region_config_shards_match_reference(case):
    cfg = CONFIGS[case["config"]]
    r0, r1 = case["r0"], case["r1"]
    h, d = ogen.generate(cfg, r0, r1)
    n, m = r1 - r0, (r1 - r0) * cfg.gpus_per_rank
    owner = np.arange(m, dtype=np.int32) // cfg.gpus_per_rank
    run = analyze_regions(_dt(h, d, n, m), case["windows"], owner)
    for j, reg in enumerate(case["regions"]):
        g, rep = run.regions[j], reg["report"]
        assert g.elapsed == rep["E"]
        assert [[int(x) for x in row] for row in g.host_sum] == [r[1:] for r in rep["hs"]]
        assert [[int(x) for x in row[:3]] for row in g.dev_sum] == [r[1:] for r in rep["ds"]]
        assert [int(x) for x in g.offload_busy] == reg["busy"]
        assert list(g.host_metrics) == [unhex(v) for v in rep["host"]]
        assert list(g.device_metrics) == [unhex(v) for v in rep["device"]]
        assert g.offload_busy_fraction == unhex(reg["frac"])


def _windows(span, k, rng):
    w = [(0, U64_MAX), (span // 3, span // 3), (span + 10, span + 100)]
    w += [(i * span // (2 * k + 2), span - i * span // (2 * k + 2)) for i in range(k)]
    w += [(int(a), int(a) + int(rng.integers(1, span))) for a in rng.integers(0, span, 4)]
    return w


@pytest.mark.parametrize("name,ranks,k", [("c4", 6, 16), ("c3", 3, 13), ("c1", 4, 20), ("c2", 5, 2)])
def test_regions_match_oracle_on_config_shards(name, ranks, k):
    cfg = scaled(CONFIGS[name], ranks) if CONFIGS[name].n_ranks > ranks else CONFIGS[name]
    h, d = ogen.generate(cfg)
    n, m = cfg.n_ranks, cfg.n_devices
    owner = np.arange(m, dtype=np.int32) // cfg.gpus_per_rank
    span = int(max(h[1].max(), d[1].max()))
    win = _windows(span, k, np.random.default_rng(ranks))
    run = analyze_regions(_dt(h, d, n, m), win, owner)
    ref = O.regions(h, d, n, m, win, owner)
    _compare(run, ref, len(win))


def test_regions_device_only_and_unowned_devices():
    cfg = scaled(CONFIGS["c3"], 2)
    h, d = ogen.generate(cfg)
    m = cfg.n_devices
    empty = (np.zeros(0, np.uint64), np.zeros(0, np.uint64), np.zeros(0, np.int32), np.zeros(0, np.uint8))
    span = int(d[1].max())
    win = _windows(span, 5, np.random.default_rng(1))
    run = analyze_regions(_dt(empty, d, 0, m), win, None)
    ref = O.regions(empty, d, 0, m, win, None)
    _compare(run, ref, len(win))
    # half the devices unowned
    n = cfg.n_ranks
    owner = np.where(np.arange(m) % 2 == 0, np.arange(m) // cfg.gpus_per_rank, -1).astype(np.int32)
    run = analyze_regions(_dt(h, d, n, m), win, owner)
    ref = O.regions(h, d, n, m, win, owner)
    _compare(run, ref, len(win))


def test_c4_full_size_region_identities():
    """1e9 intervals: the [0, 2^64-1) region is the whole-trace analysis bit for
    bit; every region partitions exactly; nested windows are monotone."""
    from paper_2603_26576_b200.synth import generate

    cfg = CONFIGS["c4"]
    dt = generate(cfg)
    whole = analyze_device(dt)
    assert whole.status == N.OK
    E = whole.elapsed
    win = [(0, U64_MAX)] + [(i * E // 40, E - i * E // 40) for i in range(15)]
    owner = np.arange(cfg.n_devices, dtype=np.int32)
    run = analyze_regions(dt, win, owner)
    assert run.status == N.OK
    r0 = run.regions[0]
    assert r0.elapsed == E
    assert np.array_equal(r0.host_sum, whole.host_sum)
    assert np.array_equal(r0.dev_sum, whole.dev_sum)
    assert r0.host_metrics == whole.host_metrics and r0.device_metrics == whole.device_metrics
    prev_busy = None
    for j, g in enumerate(run.regions):
        assert g.status == N.OK
        hs, ds = g.host_sum.astype(object), g.dev_sum.astype(object)
        assert all(hs[:, 0] + hs[:, 1] + hs[:, 2] == hs[:, 3])
        assert all(ds[:, 0] + ds[:, 1] + ds[:, 2] == g.elapsed)
        assert all(g.offload_busy.astype(object) <= hs[owner, 1])
        tot = int(g.offload_busy.astype(object).sum())
        if prev_busy is not None and j >= 2:
            assert tot <= prev_busy                       # nested windows shrink
        prev_busy = tot
        hm = g.host_metrics
        assert abs(hm[0] - hm[1] * hm[4]) <= 1e-12 * max(abs(hm[0]), 1e-300)
        dm = g.device_metrics
        assert abs(dm[0] - dm[1] * dm[2] * dm[3]) <= 1e-12 * max(abs(dm[0]), 1e-300)
    # region 1 (the outer nested window) spot-checked against the oracle on a rank shard
    print(f"c4 regions: {run.kernel_ms:.2f} ms for 16 windows over {cfg.intervals} intervals")


# ---------------------------------------------------------------------------
# per-rank regions (TALP regions are annotated per process)
# ---------------------------------------------------------------------------
PR = load("regions_per_rank")
PR_CASES = [c for c in PR if "trace" in c]
PR_CONFIG = [c for c in PR if "config" in c]


def _check_reg(g, reg):
    rep = reg["report"]
    if rep.get("raise") == "AnalysisError":
        assert g.report is None
        return
    r = g.report
    assert r.elapsed_ns == rep["E"]
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
    assert list(g.offload_busy) == reg["busy"]
    assert g.offload_busy_fraction == unhex(reg["frac"])


@pytest.mark.parametrize("case", PR_CASES, ids=[c["tag"] for c in PR_CASES])
def test_per_rank_region_reports_match_reference(case):
    """The drop-in ``region_reports`` with ``{rank: (start, end)}`` regions against the
    reference's compute_report of the per-rank-clipped traces (make_golden.py)."""
    t = to_trace(case["trace"])
    regions = [{rank: (a, b) for rank, a, b in w} for w in case["windows"]]
    got = hb.region_reports(t, regions)
    assert len(got) == len(case["regions"])
    for g, reg in zip(got, case["regions"]):
        _check_reg(g, reg)


def _table(windows, r0, n):
    t = np.zeros((len(windows), n, 2), dtype=np.uint64)
    for j, w in enumerate(windows):
        for rank, a, b in w:
            t[j, rank - r0] = (a, b)
    return t


@pytest.mark.parametrize("case", PR_CONFIG, ids=[c["tag"] for c in PR_CONFIG])
def test_per_rank_region_config_shards_match_reference(case):
    cfg = CONFIGS[case["config"]]
    r0, r1 = case["r0"], case["r1"]
    h, d = ogen.generate(cfg, r0, r1)
    n, m = r1 - r0, (r1 - r0) * cfg.gpus_per_rank
    owner = np.arange(m, dtype=np.int32) // cfg.gpus_per_rank
    run = analyze_regions(_dt(h, d, n, m), _table(case["windows"], r0, n), owner)
    assert run.status == N.OK
    for j, reg in enumerate(case["regions"]):
        g, rep = run.regions[j], reg["report"]
        assert g.elapsed == rep["E"]
        assert [[int(x) for x in row] for row in g.host_sum] == [r[1:] for r in rep["hs"]]
        assert [[int(x) for x in row[:3]] for row in g.dev_sum] == [r[1:] for r in rep["ds"]]
        assert [int(x) for x in g.offload_busy] == reg["busy"]
        assert list(g.host_metrics) == [unhex(v) for v in rep["host"]]
        assert list(g.device_metrics) == [unhex(v) for v in rep["device"]]
        assert g.offload_busy_fraction == unhex(reg["frac"])


def per_rank_windows(spans, k, rng):
    """[R][n][2]: nested per-rank windows over each rank's own span, shifted per rank, plus
    arbitrary, empty, whole-range and past-the-end ones."""
    n = len(spans)
    out = [np.stack([np.zeros(n, np.uint64), np.full(n, U64_MAX, np.uint64)], 1)]
    for i in range(k):
        lo = np.array([i * s // (2 * k + 2) + int(rng.integers(0, 50)) for s in spans], dtype=np.uint64)
        hi = np.array([s - i * s // (2 * k + 2) for s in spans], dtype=np.uint64)
        out.append(np.stack([lo, np.maximum(lo, hi)], 1))
    a = np.array([int(rng.integers(0, max(1, s))) for s in spans], dtype=np.uint64)
    out.append(np.stack([a, a + np.array([int(rng.integers(0, max(2, s // 2))) for s in spans], np.uint64)], 1))
    out.append(np.stack([np.array(spans, np.uint64) + 5, np.array(spans, np.uint64) + 50], 1))
    e = np.stack([a, a], 1)
    e[::2] = out[1][::2]                     # some ranks empty, others not
    out.append(e)
    return np.stack(out)


@pytest.mark.parametrize("name,ranks,k", [("c4", 6, 13), ("c3", 3, 10), ("c1", 4, 16), ("c5", 5, 6)])
def test_per_rank_regions_match_oracle_on_config_shards(name, ranks, k):
    cfg = scaled(CONFIGS[name], ranks) if CONFIGS[name].n_ranks > ranks else CONFIGS[name]
    h, d = ogen.generate(cfg)
    n, m = cfg.n_ranks, cfg.n_devices
    owner = np.arange(m, dtype=np.int32) // cfg.gpus_per_rank
    spans = [int(h[1][h[2] == p].max()) for p in range(n)]
    win = per_rank_windows(spans, k, np.random.default_rng(ranks))
    run = analyze_regions(_dt(h, d, n, m), win, owner)
    ref = O.regions(h, d, n, m, win, owner)
    _compare(run, ref, win.shape[0])
    # half the devices unowned: they record nothing in any per-rank region
    owner2 = np.where(np.arange(m) % 2 == 0, owner, -1).astype(np.int32)
    run = analyze_regions(_dt(h, d, n, m), win, owner2)
    ref = O.regions(h, d, n, m, win, owner2)
    _compare(run, ref, win.shape[0])


def test_per_rank_region_with_one_window_everywhere_is_the_global_region():
    """A per-rank table whose ranks all share one window equals the global-window call."""
    cfg = scaled(CONFIGS["c3"], 3)
    h, d = ogen.generate(cfg)
    n, m = cfg.n_ranks, cfg.n_devices
    owner = np.arange(m, dtype=np.int32) // cfg.gpus_per_rank
    span = int(max(h[1].max(), d[1].max()))
    win = _windows(span, 6, np.random.default_rng(3))
    table = np.repeat(np.asarray(win, dtype=np.uint64)[:, None, :], n, axis=1)
    a = analyze_regions(_dt(h, d, n, m), win, owner)
    b = analyze_regions(_dt(h, d, n, m), table, owner)
    for x, y in zip(a.regions, b.regions):
        assert x.status == y.status and x.elapsed == y.elapsed
        if x.status == N.OK:
            assert np.array_equal(x.host_sum, y.host_sum) and np.array_equal(x.dev_sum, y.dev_sum)
            assert np.array_equal(x.offload_busy, y.offload_busy)
            assert x.host_metrics == y.host_metrics and x.device_metrics == y.device_metrics


def nested_rank_windows(spans, k: int) -> np.ndarray:
    """C4's 16 nested monitoring regions PER RANK (bench.py uses the same shape): region i of
    rank p is [i * S_p / 40 + (p % 13), S_p - i * S_p / 40) over the rank's own span S_p."""
    S = np.asarray(spans, dtype=np.uint64)
    p = np.arange(S.size, dtype=np.uint64)
    out = np.zeros((k, S.size, 2), dtype=np.uint64)
    for i in range(k):
        lo = np.uint64(i) * S // np.uint64(40) + p % np.uint64(13)
        hi = S - np.uint64(i) * S // np.uint64(40)
        out[i, :, 0], out[i, :, 1] = lo, np.maximum(lo, hi)
    return out


def test_c4_full_size_per_rank_regions_match_sharded_oracle():
    """C4 in full (1e9 intervals, 1024 ranks) with 16 nested regions PER RANK: every region's
    E, per-rank and per-device summaries, clamp counts, offload/busy overlap, metric floats
    and overlap fraction bit-exact against the oracle's region composition run rank-sharded
    (host pass per block, global E_j, device pass; oracle.regions_sharded)."""
    from paper_2603_26576_b200.synth import generate

    cfg = CONFIGS["c4"]
    dt = generate(cfg)
    whole = analyze_device(dt)
    assert whole.status == N.OK
    table = nested_rank_windows([int(x) for x in whole.host_sum[:, 3]], 16)
    owner = np.arange(cfg.n_devices, dtype=np.int32) // cfg.gpus_per_rank
    run = analyze_regions(dt, table, owner)
    assert run.status == N.OK
    g = cfg.gpus_per_rank
    hseg, dseg = dt.h_seg.cpu().numpy(), dt.d_seg.cpu().numpy()

    def fetch(r0, r1):
        a, b, c, d = int(hseg[r0]), int(hseg[r1]), int(dseg[r0 * g]), int(dseg[r1 * g])

        def col(x, lo, hi, off=None):
            v = x[lo:hi].cpu().numpy()
            return v.view(np.uint64) if v.dtype == np.int64 else (v - np.int32(off) if off is not None else v)
        return ((col(dt.h_start, a, b), col(dt.h_end, a, b), col(dt.h_res, a, b, r0), col(dt.h_kind, a, b)),
                (col(dt.d_start, c, d), col(dt.d_end, c, d), col(dt.d_res, c, d, r0 * g), col(dt.d_kind, c, d)))

    ref = O.regions_sharded(fetch, cfg.n_ranks, g, table, 8)
    _compare(run, ref, table.shape[0])
    assert int(ref.busy.astype(object).sum()) > 0
    print(f"c4 per-rank regions: {run.kernel_ms:.2f} ms for 16 regions x 1024 ranks over {cfg.intervals} intervals")
