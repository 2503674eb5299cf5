"""The interval algebra on the GPU (csrc/intervals.cu) through the drop-in
functions ``flatten / subtract / complement / intersect / total_duration``:
against fixtures from the reference's intervals.py and, at sizes the reference
cannot reach, against the pinned C oracle."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import gpu_available
from golden_io import load

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

import paper_2603_26576_b200 as hb  # noqa: E402
from oracle import oracle as O  # noqa: E402

CASES = load("intervals")
IV = hb.Interval


def _enc(f):
    return [[iv.start, iv.end] for iv in f]


@pytest.mark.parametrize("case", CASES, ids=[f"iv{i}" for i in range(len(CASES))])
def test_interval_algebra_matches_reference(case):
    raw_a = [IV(s, e) for s, e in case["a"]]
    if "error" in case:
        with pytest.raises(ValueError) as ei:
            hb.flatten(raw_a)
        assert str(ei.value) == case["error"]
        return
    fa = hb.flatten(raw_a)
    fb = hb.flatten(IV(s, e) for s, e in case["b"])
    assert _enc(fa) == case["flat_a"] and _enc(fb) == case["flat_b"]
    assert _enc(hb.subtract(fa, fb)) == case["sub"]
    bounds = IV(*case["bounds"])
    assert _enc(hb.complement(fa, bounds)) == case["comp"]
    assert _enc(hb.intersect(fa, bounds)) == case["inter"]
    assert hb.total_duration(fa) == case["total"]


def test_interval_edge_cases():
    assert hb.flatten([]) == hb.EMPTY
    assert hb.flatten([IV(5, 5), IV(7, 7)]) == hb.EMPTY                      # zero-length vanish
    assert _enc(hb.flatten([IV(0, 5), IV(5, 9)])) == [[0, 9]]                # adjacency merges
    assert _enc(hb.flatten([IV(3, 4), IV(0, 10), IV(2, 3)])) == [[0, 10]]
    with pytest.raises(ValueError, match=r"malformed interval at index 1: \[9, 2\)"):
        hb.flatten([IV(0, 1), IV(9, 2), IV(8, 3)])
    with pytest.raises(ValueError, match="malformed bounds"):
        hb.complement(hb.EMPTY, IV(5, 1))
    assert hb.complement(hb.flatten([IV(0, 5)]), IV(3, 3)) == hb.EMPTY
    assert _enc(hb.complement(hb.EMPTY, IV(2, 8))) == [[2, 8]]
    big = (1 << 64) - 1
    f = hb.flatten([IV(big - 10, big), IV(0, 1 << 63), IV(1 << 63, big - 10)])
    assert _enc(f) == [[0, big]] and hb.total_duration(f) == big
    many = hb.flatten([IV(2 * i, 2 * i + 1) for i in range(5000)])
    assert hb.total_duration(many) == 5000


@pytest.mark.parametrize("n,span", [(1_000, 100), (300_000, 1 << 24), (2_000_000, 1 << 40)])
def test_interval_algebra_vs_oracle_large(n, span):
    rng = np.random.default_rng(n)
    s = rng.integers(0, span, n, dtype=np.uint64)
    e = s + rng.integers(0, max(2, span // 5000), n, dtype=np.uint64)
    fa = hb.flatten(IV(int(a), int(b)) for a, b in zip(s, e))
    os_, oe = O.iv_flatten(s, e)
    assert _enc(fa) == [[int(a), int(b)] for a, b in zip(os_, oe)]
    s2 = rng.integers(0, span, n // 2, dtype=np.uint64)
    e2 = s2 + rng.integers(1, max(2, span // 2000), n // 2, dtype=np.uint64)
    fb = hb.flatten(IV(int(a), int(b)) for a, b in zip(s2, e2))
    gs, ge = O.iv_flatten(s2, e2)
    ds, de = O.iv_subtract(os_, oe, gs, ge)
    assert _enc(hb.subtract(fa, fb)) == [[int(a), int(b)] for a, b in zip(ds, de)]
    assert _enc(hb.subtract(fb, fa)) == [[int(a), int(b)] for a, b in zip(*O.iv_subtract(gs, ge, os_, oe))]
    lo, hi = span // 3, 2 * span // 3
    assert _enc(hb.intersect(fa, IV(lo, hi))) == [[int(a), int(b)] for a, b in zip(*O.iv_intersect(os_, oe, lo, hi))]
    assert hb.total_duration(fa) == O.iv_total(os_, oe)
