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
