"""Config-shaped traces generated in HBM: generator bit-exactness vs the numpy
twin, parity with the reference on rank shards, and full-scale parity with
the C oracle: C2 (1e8) whole, C3 / C4 / C5 (5e8 / 1e9 / 2e9) through the
oracle run rank-sharded with the global E, plus size-independent properties."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import gpu_available
from golden_io import load, unhex

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

from paper_2603_26576_b200 import _native as N  # noqa: E402
from paper_2603_26576_b200.configs import CONFIGS  # noqa: E402
from paper_2603_26576_b200.engine import analyze_device  # noqa: E402
from paper_2603_26576_b200.synth import generate  # noqa: E402


def _host(t):
    return t.cpu().numpy()


def _u64(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c5"])
def test_gpu_generator_matches_numpy_twin(name):
    from oracle import gen as ogen
    cfg = CONFIGS[name]
    dt = generate(cfg, 0, 2 if name != "c1" else 4)
    (hs, he, hr, hk), (ds, de, dr, dk) = ogen.generate(cfg, 0, 2 if name != "c1" else 4)
    assert np.array_equal(_u64(dt.h_start), hs) and np.array_equal(_u64(dt.h_end), he)
    assert np.array_equal(_host(dt.h_res), hr) and np.array_equal(_host(dt.h_kind), hk)
    assert np.array_equal(_u64(dt.d_start), ds) and np.array_equal(_u64(dt.d_end), de)
    assert np.array_equal(_host(dt.d_res), dr) and np.array_equal(_host(dt.d_kind), dk)


SHARDS = load("config_shards")


@pytest.mark.parametrize("shard", SHARDS, ids=[f"{s['config']}[{s['r0']}:{s['r1']}]" for s in SHARDS])
def test_config_shard_matches_reference(shard):
    cfg = CONFIGS[shard["config"]]
    dt = generate(cfg, shard["r0"], shard["r1"])
    f = analyze_device(dt)
    rep = shard["report"]
    assert f.status == N.OK
    assert f.elapsed == rep["E"]
    assert [list(map(int, r)) for r in f.host_sum] == [x[1:] for x in rep["hs"]]
    assert [list(map(int, r[:3])) for r in f.dev_sum] == [x[1:] for x in rep["ds"]]
    assert list(f.host_metrics) == [unhex(v) for v in rep["host"]]
    assert list(f.device_metrics) == [unhex(v) for v in rep["device"]]


def test_c2_full_scale_matches_oracle():
    """C2 in full (1e8 intervals): every summary bit-exact vs the C oracle."""
    from oracle import oracle as O
    cfg = CONFIGS["c2"]
    dt = generate(cfg)
    f = analyze_device(dt)
    assert f.status == N.OK
    h = (_u64(dt.h_start), _u64(dt.h_end), _host(dt.h_res), _host(dt.h_kind))
    d = (_u64(dt.d_start), _u64(dt.d_end), _host(dt.d_res), _host(dt.d_kind))
    ref = O.analyze(h, d, cfg.n_ranks, cfg.n_devices)
    assert ref.status == 0
    assert f.elapsed == ref.elapsed
    assert np.array_equal(f.host_sum, ref.host_sum)
    assert np.array_equal(f.dev_sum, ref.dev_sum)
    assert f.host_metrics == ref.host_metrics and f.device_metrics == ref.device_metrics


def _fetch(dt, g):
    """Rank block [r0, r1) of an HBM-resident generated trace as host numpy columns
    (resource ids local to the block) -- one block at a time, for the sharded oracle."""
    hseg = dt.h_seg.cpu().numpy()
    dseg = dt.d_seg.cpu().numpy()

    def fetch(r0, r1):
        a, b = int(hseg[r0]), int(hseg[r1])
        c, d = int(dseg[r0 * g]), int(dseg[r1 * g])
        h = (_u64(dt.h_start[a:b]), _u64(dt.h_end[a:b]), _host(dt.h_res[a:b]) - np.int32(r0), _host(dt.h_kind[a:b]))
        v = (_u64(dt.d_start[c:d]), _u64(dt.d_end[c:d]), _host(dt.d_res[c:d]) - np.int32(r0 * g),
             _host(dt.d_kind[c:d]))
        return h, v
    return fetch


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_full_scale_matches_sharded_oracle(name):
    """C3 (5e8), C4 (1e9) and C5 (2e9 -- the north star's trace) IN FULL on one GPU,
    bit-exact against the C oracle run rank-sharded in the reference's exact sharded form
    (summarize_host per block, E = max, summarize_device(block, E_global), the metric
    stage functions on the gathered summaries -- summarize.py:57-138, metrics.py:66-122):
    E, every per-rank and per-device summary, every device's clamp count and all nine
    metric floats ``==``.  Both input layouts (CSR offsets, res columns) are checked."""
    from oracle import oracle as O
    cfg = CONFIGS[name]
    dt = generate(cfg)
    f = analyze_device(dt)                   # resource ids as CSR offsets (17 B / interval)
    g = analyze_device(dt.columns_only())    # res columns (21 B / interval)
    assert f.status == N.OK and g.status == N.OK
    per_rank = cfg.intervals / cfg.n_ranks
    block = max(1, int(1.2e8 // per_rank))
    ref = O.analyze_sharded(_fetch(dt, cfg.gpus_per_rank), cfg.n_ranks, cfg.gpus_per_rank, block)
    for got in (f, g):
        assert got.elapsed == ref.elapsed
        assert np.array_equal(got.host_sum, ref.host_sum)
        assert np.array_equal(got.dev_sum, ref.dev_sum)          # k, mem, idle, clamp count
        assert tuple(got.host_metrics) == ref.host_metrics
        assert tuple(got.device_metrics) == ref.device_metrics
    # the workload really exercises the cross-rank coupling: devices clamp at the GLOBAL E
    if name == "c5":
        assert int(ref.dev_sum[:, 3].sum()) > 0
    assert ref.blocks > 1


@pytest.mark.parametrize("name", ["c3", "c5"])
def test_full_scale_properties(name):
    """Size-independent properties at full config size (single GPU)."""
    cfg = CONFIGS[name]
    dt = generate(cfg)
    f = analyze_device(dt)
    assert f.status == N.OK
    E = f.elapsed
    hs = f.host_sum.astype(object)
    ds = f.dev_sum.astype(object)
    # host: useful + offload + mpi == span_end, E == max span_end
    assert all(r[0] + r[1] + r[2] == r[3] for r in hs)
    assert E == max(r[3] for r in hs)
    # device partition identity (summarize.py docstring: kernel + memory + idle == elapsed)
    assert all(r[0] + r[1] + r[2] == E for r in ds)
    # a second run gives identical bits (integer sums are order independent)
    g = analyze_device(dt)
    assert np.array_equal(f.host_sum, g.host_sum) and np.array_equal(f.dev_sum, g.dev_sum)
    # metric identities (metrics.py docstring)
    pe, mpe, ce, lb, oe = f.host_metrics
    assert abs(pe - mpe * oe) <= 1e-12 * pe and abs(mpe - ce * lb) <= 1e-12 * mpe
    dpe, dlb, dce, doe = f.device_metrics
    assert abs(dpe - dlb * dce * doe) <= 1e-12 * dpe


@pytest.mark.parametrize("name,ranks", [("c3", 3), ("c5", 6), ("c2", 20)])
def test_every_kernel_compilation_matches_the_oracle(name, ranks):
    """The analysis kernel is compiled per tile geometry (15 x 11 for CSR inputs; 11 x 15 or
    8 x 19 for res columns, chosen by device run length -- capi.cu pick_compilation): every
    compilation, forced through HETEFF_COMPILATION, bit-exact against the oracle."""
    import os
    from oracle import oracle as O
    cfg = CONFIGS[name]
    dt = generate(cfg, 0, ranks)
    h = (_u64(dt.h_start), _u64(dt.h_end), _host(dt.h_res), _host(dt.h_kind))
    d = (_u64(dt.d_start), _u64(dt.d_end), _host(dt.d_res), _host(dt.d_kind))
    ref = O.analyze(h, d, dt.n, dt.m)
    runs = [analyze_device(dt)]                     # CSR offsets: the 15 x 11 compilation
    old = os.environ.get("HETEFF_COMPILATION")
    try:
        for c in ("1", "2"):
            os.environ["HETEFF_COMPILATION"] = c
            runs.append(analyze_device(dt.columns_only()))
    finally:
        if old is None:
            os.environ.pop("HETEFF_COMPILATION", None)
        else:
            os.environ["HETEFF_COMPILATION"] = old
    for f in runs:
        assert f.status == N.OK and f.elapsed == ref.elapsed
        assert np.array_equal(f.host_sum, ref.host_sum) and np.array_equal(f.dev_sum, ref.dev_sum)
        assert f.host_metrics == ref.host_metrics and f.device_metrics == ref.device_metrics


def test_split_analysis_equals_the_single_launch():
    """Large REPORT calls whose host and device sides prefer different kernel compilations
    run as two launches + the merge kernel (capi.cu run_split); forced here on a C5 shard
    (HETEFF_SPLIT_MIN) and compared with the single launch (HETEFF_NO_SPLIT): E, every
    summary (clamp counts included), the finding counts and the nine floats identical."""
    import os
    from paper_2603_26576_b200 import _native as Nn
    cfg = CONFIGS["c5"]
    dt = generate(cfg, 0, 40).columns_only()
    keys = ("HETEFF_SPLIT_MIN", "HETEFF_NO_SPLIT")
    old = {k: os.environ.get(k) for k in keys}
    try:
        os.environ["HETEFF_SPLIT_MIN"] = "1"
        os.environ.pop("HETEFF_NO_SPLIT", None)
        a = analyze_device(dt)
        name = Nn.load().heteff_kernel_name(Nn.context(0)).decode()
        os.environ["HETEFF_NO_SPLIT"] = "1"
        b = analyze_device(dt)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert name.startswith("split"), name
    assert a.status == b.status == N.OK
    assert (a.elapsed, a.host_elapsed, a.dev_max_end, a.counts) == (b.elapsed, b.host_elapsed, b.dev_max_end, b.counts)
    assert a.counts[7] > 0                       # late device records: the clamp-count hand-over is exercised
    assert np.array_equal(a.host_sum, b.host_sum) and np.array_equal(a.dev_sum, b.dev_sum)
    assert a.host_metrics == b.host_metrics and a.device_metrics == b.device_metrics


@pytest.mark.gpu
def test_block_mode_overlap_leaves_the_context_clean():
    """A block-mode launch (the split analysis, heteff_analyze_into) on a trace whose host
    records overlap defers (status -1) without the error-path kernels; the kernel must still
    reset the context's accumulators and globals, so the fallback answer and the NEXT call on
    the same context equal the oracle's (found by tools/stress.py under HETEFF_FORCE_SPLIT)."""
    import os

    import torch

    from oracle import oracle as O
    from paper_2603_26576_b200.engine import DeviceTrace

    def cols(s, e, r, k):
        return (np.array(s, np.uint64), np.array(e, np.uint64), np.array(r, np.int32), np.array(k, np.uint8))

    def cu(x):
        return torch.from_numpy(x.view(np.int64) if x.dtype == np.uint64 else x).cuda()

    bad_h = cols([0, 5, 0], [10, 15, 30], [0, 0, 1], [0, 0, 1])            # rank 0 overlaps itself
    good_h = cols([0, 12, 0], [10, 20, 30], [0, 0, 1], [0, 1, 0])
    d = cols([1, 4, 2], [3, 25, 9], [0, 0, 1], [0, 1, 0])
    old = os.environ.get("HETEFF_FORCE_SPLIT")
    os.environ["HETEFF_FORCE_SPLIT"] = "1"
    try:
        for h in (bad_h, good_h, bad_h, good_h):
            dt = DeviceTrace(*(cu(x) for x in (*h, *d)), 2, 2)
            got = analyze_device(dt)
            ref = O.analyze(h, d, 2, 2, mode=N.MODE_REPORT, cap=0)
            assert got.status == ref.status
            if ref.status == N.OK:
                assert got.elapsed == ref.elapsed
                assert np.array_equal(got.host_sum, ref.host_sum) and np.array_equal(got.dev_sum, ref.dev_sum)
                assert got.host_metrics == ref.host_metrics and got.device_metrics == ref.device_metrics
    finally:
        if old is None:
            os.environ.pop("HETEFF_FORCE_SPLIT", None)
        else:
            os.environ["HETEFF_FORCE_SPLIT"] = old
