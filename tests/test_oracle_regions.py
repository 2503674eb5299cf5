"""Pin the oracle's EXTENSION restatement (regions + offload/busy overlap,
talp_oracle.c ``orc_regions``) against fixtures made by running the
reference: ``compute_report`` of each window-clipped trace and the
reference's interval algebra for the overlap (tests/golden/make_golden.py,
``regions_corpus``).  CPU only."""

from __future__ import annotations

import numpy as np
import pytest

from golden_io import load, to_trace, unhex
from oracle import gen as ogen
from oracle import oracle as O
from paper_2603_26576_b200.configs import CONFIGS
from paper_2603_26576_b200.packing import dev_owner_table, pack_trace

CASES = [c for c in load("regions") if "trace" in c]
CONFIG_CASES = [c for c in load("regions") if "config" in c]


def check_region(res, j, reg, n, m):
    rep = reg["report"]
    if rep.get("raise") == "AnalysisError":
        assert res.status[j] == 2
        return
    assert res.status[j] == 0
    assert int(res.elapsed[j]) == rep["E"]
    assert [[int(x) for x in row] for row in res.host_sum[j][:, :4]] == [r[1:] for r in rep["hs"]]
    assert [[int(x) for x in row[:3]] for row in res.dev_sum[j]] == [r[1:] for r in rep["ds"]]
    if rep["host"] is None:
        assert n == 0
    else:
        assert list(res.host_metrics[j]) == [unhex(v) for v in rep["host"]]
    if rep["device"] is None:
        assert m == 0
    else:
        assert list(res.device_metrics[j]) == [unhex(v) for v in rep["device"]]
    assert [int(x) for x in res.busy[j]] == reg["busy"]
    assert res.busy_frac[j] == unhex(reg["frac"])


@pytest.mark.parametrize("case", CASES[::2], ids=[c["tag"] for c in CASES[::2]])
def test_oracle_regions_match_reference(case):
    t = to_trace(case["trace"])
    packed = pack_trace(t)
    owner = dev_owner_table(t, packed)
    res = O.regions_packed(packed, case["windows"], owner)
    for j, reg in enumerate(case["regions"]):
        check_region(res, j, reg, t.n, t.m)


@pytest.mark.parametrize("case", CONFIG_CASES, ids=[c["tag"] for c in CONFIG_CASES])
def test_oracle_regions_config_shard(case):
    cfg = CONFIGS[case["config"]]
    r0, r1 = case["r0"], case["r1"]
    h, d = ogen.generate(cfg, r0, r1)
    n, m = r1 - r0, (r1 - r0) * cfg.gpus_per_rank
    owner = np.arange(m, dtype=np.int32) // cfg.gpus_per_rank
    res = O.regions(h, d, n, m, case["windows"], owner)
    for j, reg in enumerate(case["regions"]):
        check_region(res, j, reg, n, m)


# ---------------------------------------------------------------------------
# per-rank regions (each rank its own window, devices follow their owner)
# ---------------------------------------------------------------------------
PR = load("regions_per_rank")
PR_CASES = [c for c in PR if "trace" in c]
PR_CONFIG = [c for c in PR if "config" in c]


def per_rank_table(windows, host_ids: list) -> np.ndarray:
    """Fixture regions ([[rank, a, b], ...] per region) -> [R][host_ids][2] over dense ids."""
    dense = {rank: i for i, rank in enumerate(host_ids)}
    t = np.zeros((len(windows), len(host_ids), 2), dtype=np.uint64)
    for j, w in enumerate(windows):
        for rank, a, b in w:
            if rank in dense:
                t[j, dense[rank]] = (a, b)
    return t


@pytest.mark.parametrize("case", PR_CASES[::2], ids=[c["tag"] for c in PR_CASES[::2]])
def test_oracle_per_rank_regions_match_reference(case):
    t = to_trace(case["trace"])
    packed = pack_trace(t)
    owner = dev_owner_table(t, packed)
    res = O.regions_packed(packed, per_rank_table(case["windows"], packed.host_ids), owner)
    for j, reg in enumerate(case["regions"]):
        check_region(res, j, reg, t.n, t.m)


@pytest.mark.parametrize("case", PR_CONFIG, ids=[c["tag"] for c in PR_CONFIG])
def test_oracle_per_rank_regions_config_shard(case):
    cfg = CONFIGS[case["config"]]
    r0, r1 = case["r0"], case["r1"]
    h, d = ogen.generate(cfg, r0, r1)
    n, m = r1 - r0, (r1 - r0) * cfg.gpus_per_rank
    owner = np.arange(m, dtype=np.int32) // cfg.gpus_per_rank
    res = O.regions(h, d, n, m, per_rank_table(case["windows"], list(range(r0, r1))), owner)
    for j, reg in enumerate(case["regions"]):
        check_region(res, j, reg, n, m)


@pytest.mark.parametrize("name,ranks,block", [("c5", 12, 5), ("c4", 7, 2), ("c3", 4, 3)])
def test_sharded_region_oracle_equals_whole(name, ranks, block):
    """oracle.regions_sharded (host pass per block, global E_j, device pass) reproduces the
    whole-trace region composition bit for bit -- the checker of the full-size C4 test."""
    from paper_2603_26576_b200.configs import scaled
    cfg = scaled(CONFIGS[name], ranks)
    h, d = ogen.generate(cfg)
    n, m, g = cfg.n_ranks, cfg.n_devices, cfg.gpus_per_rank
    spans = [int(h[1][h[2] == p].max()) for p in range(n)]
    rng = np.random.default_rng(ranks)
    t = np.zeros((6, n, 2), np.uint64)
    for j in range(6):
        for p in range(n):
            a = int(rng.integers(0, spans[p] // 3))
            t[j, p] = (a, a + int(rng.integers(1, spans[p])))
    t[5, ::2] = (7, 7)   # some ranks outside the last region
    whole = O.regions(h, d, n, m, t, np.arange(m, dtype=np.int32) // g)
    sh = O.regions_sharded(lambda a, b: ogen.generate(cfg, a, b), n, g, t, block, workers=3)
    for j in range(t.shape[0]):
        assert sh.status[j] == whole.status[j] and sh.elapsed[j] == whole.elapsed[j]
        assert np.array_equal(sh.host_sum[j], whole.host_sum[j])
        assert np.array_equal(sh.dev_sum[j], whole.dev_sum[j])
        assert np.array_equal(sh.busy[j], whole.busy[j])
        assert sh.host_metrics[j] == whole.host_metrics[j] and sh.device_metrics[j] == whole.device_metrics[j]
        assert sh.busy_frac[j] == whole.busy_frac[j]
