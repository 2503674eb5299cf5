"""Pin the C oracle (oracle/talp_oracle.c) against the reference's own outputs.

Fixtures come from running /root/reference/pkg (tests/golden/make_golden.py).
CPU only: the oracle is plain C.
"""

from __future__ import annotations

import random
import re
from fractions import Fraction

import numpy as np
import pytest

from golden_io import load, to_trace, unhex
from oracle import gen as ogen
from oracle import oracle as O
from paper_2603_26576_b200.configs import CONFIGS
from paper_2603_26576_b200.messages import declaration_messages
from paper_2603_26576_b200.packing import pack_trace

HOST_METRICS = 5
CASES = load("presets") + load("acceptance") + load("invalid")


def _expect_lists(case, packed):
    """Record indices per finding class, parsed from the reference messages."""
    v = case["validate"]
    q_host = {q.index for q in packed.host_q}
    q_dev = {q.index for q in packed.dev_q}
    out = {k: set() for k in ("hmal", "hzero", "hund", "ovl", "dmal", "dzero", "dund", "late")}
    for msg in v["errors"] + v["warnings"]:
        m = re.match(r"host record (\d+) \(", msg)
        if m:
            i = int(m.group(1))
            if i in q_host:
                continue
            if " > end " in msg:
                out["hmal"].add(i)
            elif "zero-length" in msg:
                out["hzero"].add(i)
            elif "rank not declared" in msg:
                out["hund"].add(i)
            continue
        m = re.match(r"device record (\d+) \(", msg)
        if m:
            i = int(m.group(1))
            if i in q_dev:
                continue
            if " > end " in msg:
                out["dmal"].add(i)
            elif "zero-length" in msg:
                out["dzero"].add(i)
            elif "device not declared" in msg:
                out["dund"].add(i)
            elif "after host elapsed" in msg:
                out["late"].add(i)
            continue
        m = re.match(r"rank .*: host records (\d+) and (\d+) overlap", msg)
        if m:
            out["ovl"].add((int(m.group(1)), int(m.group(2))))
    return out


def _canon(pos, index):
    return {int(index[p]) if index is not None else int(p) for p in pos}


@pytest.mark.parametrize("case", CASES, ids=[c["tag"] for c in CASES])
def test_oracle_matches_reference(case):
    trace = to_trace(case["trace"])
    packed = pack_trace(trace)
    res = O.analyze_packed(packed, O.MODE_REPORT, cap=1 << 12)
    rep = case["report"]
    decl_errors, _ = declaration_messages(trace)
    # validation findings, record by record
    exp = _expect_lists(case, packed)
    hi, di = packed.host.index, packed.dev.index
    got = {
        "hmal": _canon(res.lists[0], hi), "hzero": _canon(res.lists[1], hi), "hund": _canon(res.lists[2], hi),
        "ovl": {(int(hi[c]) if hi is not None else int(c), int(hi[i]) if hi is not None else int(i))
                for c, i in res.lists[3]},
        "dmal": _canon(res.lists[4], di), "dzero": _canon(res.lists[5], di), "dund": _canon(res.lists[6], di),
        "late": _canon(res.lists[7], di),
    }
    if decl_errors and any("duplicate rank" in e for e in decl_errors):
        got.pop("ovl"); exp.pop("ovl")   # duplicated declarations repeat overlap groups; covered in API tests
    assert got == exp
    if rep.get("raise") == "InvalidTraceError":
        assert decl_errors or res.status == 1 or packed.host_q or packed.dev_q
        return
    if rep.get("raise") == "AnalysisError":
        assert res.status == 2
        return
    assert res.status == 0
    assert res.elapsed == rep["E"]
    assert [list(map(int, r)) for r in res.host_sum] == [x[1:] for x in rep["hs"]]
    assert [list(map(int, r[:3])) for r in res.dev_sum] == [x[1:] for x in rep["ds"]]
    if rep["host"] is not None:
        assert list(res.host_metrics) == [unhex(v) for v in rep["host"]]
    if rep["device"] is not None:
        assert list(res.device_metrics) == [unhex(v) for v in rep["device"]]
    # clamp warnings carry the per-device clamp count
    clamps = {}
    for w in rep["warnings"]:
        m = re.match(r"device (-?\d+): clamped (\d+) record", w)
        if m:
            clamps[int(m.group(1))] = int(m.group(2))
    got_clamps = {d.device_id: int(res.dev_sum[p][3]) for p, d in enumerate(trace.devices) if res.dev_sum[p][3]}
    assert got_clamps == clamps


SD = load("summarize_device")


@pytest.mark.parametrize("case", SD[::7], ids=[c["tag"] for c in SD[::7]])
def test_oracle_summarize_device_window(case):
    trace = to_trace(case["trace"])
    packed = pack_trace(trace)
    res = O.analyze_packed(packed, O.MODE_SUMMARIZE_DEVICE, elapsed=case["elapsed"])
    assert res.status == 0
    assert [list(map(int, r[:3])) for r in res.dev_sum] == [x[1:] for x in case["ds"]]


def test_exact_division_matches_python():
    rng = random.Random(7)
    for _ in range(20000):
        a = rng.randint(0, 1 << rng.choice((10, 53, 64, 90, 96)))
        b = rng.randint(1, 1 << rng.choice((10, 53, 64, 90, 96)))
        assert O.div_exact(a, b) == a / b
    # ties and near-ties
    for a, b in [(1, 3), (2 ** 53 + 1, 1), (2 ** 54 + 2, 2), ((2 ** 53 + 1) * 2 ** 40, 2 ** 40), (3 * 2 ** 60 + 1, 3)]:
        assert O.div_exact(a, b) == a / b


SHARDS = load("config_shards")


@pytest.mark.parametrize("shard", SHARDS, ids=[f"{s['config']}[{s['r0']}:{s['r1']}]" for s in SHARDS])
def test_oracle_config_shards(shard):
    cfg = CONFIGS[shard["config"]]
    (hs, he, hr, hk), (ds, de, dr, dk) = ogen.generate(cfg, shard["r0"], shard["r1"])
    n = shard["r1"] - shard["r0"]
    m = n * cfg.gpus_per_rank
    res = O.analyze((hs, he, hr, hk), (ds, de, dr, dk), n, m)
    rep = shard["report"]
    assert res.status == 0
    assert res.elapsed == rep["E"]
    assert [list(map(int, r)) for r in res.host_sum] == [x[1:] for x in rep["hs"]]
    assert [list(map(int, r[:3])) for r in res.dev_sum] == [x[1:] for x in rep["ds"]]
    assert list(res.host_metrics) == [unhex(v) for v in rep["host"]]
    assert list(res.device_metrics) == [unhex(v) for v in rep["device"]]


def test_generator_shapes_are_canonical():
    for name in ("c1", "c2", "c5"):
        cfg = CONFIGS[name]
        (hs, he, hr, hk), (ds, de, dr, dk) = ogen.generate(cfg, 0, 2)
        for s, e, r in ((hs, he, hr), (ds, de, dr)):
            assert (e >= s).all()
            key_ok = (np.diff(r) > 0) | ((np.diff(r) == 0) & (np.diff(s.astype(np.int64)) >= 0))
            assert key_ok.all()
        # host chains are non-overlapping per rank (valid traces)
        same = np.diff(hr) == 0
        assert (hs[1:][same] >= he[:-1][same]).all()


def test_generator_shards_compose():
    """A rank shard regenerates exactly the slice of the full-trace arrays (counter-based RNG)."""
    cfg = CONFIGS["c1"]
    full = ogen.generate(cfg, 0, 4)
    part = ogen.generate(cfg, 2, 4)
    hcut = int((full[0][2] < 2).sum())
    dcut = int((full[1][2] < 2 * cfg.gpus_per_rank).sum())
    for a, b in zip(full[0][:2], part[0][:2]):
        assert np.array_equal(a[hcut:], b)
    for a, b in zip(full[1][:2], part[1][:2]):
        assert np.array_equal(a[dcut:], b)


def test_fraction_semantics_of_fixture_metrics():
    """Fixture floats are Python int/int results -- the exact-division contract."""
    for c in load("metrics")[:50]:
        hs = c["hs"]
        E = c["E"]
        su = sum(x[1] for x in hs)
        suw = sum(x[1] + x[2] for x in hs)
        if suw:
            assert unhex(c["host"][4]) == float(Fraction(su, suw))
