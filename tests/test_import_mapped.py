"""Chrome-trace import (csrc/ingest.cpp heteff_import_events + trace_io.import_mapped /
read_mapping) against the reference's import_mapped (trace_io.py:196-342): fixtures
from running the reference on random event documents and edge / error cases
(tests/golden/make_golden.py ``import_corpus``).  CPU only."""

from __future__ import annotations

import json

import pytest

from golden_io import load
from paper_2603_26576_b200 import trace_io

CASES = load("imports")


def _enc(t):
    return {
        "hp": list(t.host_processes),
        "dev": [[d.device_id, d.owner_rank] for d in t.devices],
        "h": [[r.rank, r.state.value, r.interval.start, r.interval.end] for r in t.host_records],
        "d": [[r.device_id, r.kind.value, r.interval.start, r.interval.end, r.stream] for r in t.device_records],
        "tu": t.time_unit,
    }


@pytest.mark.parametrize("case", CASES, ids=[c["tag"] for c in CASES])
def test_import_matches_reference(case):
    if "doc" not in case:   # mapping documents only
        if case.get("map_ok"):
            trace_io.read_mapping(case["map"])
        else:
            with pytest.raises(trace_io.TraceFormatError) as ei:
                trace_io.read_mapping(case["map"])
            assert str(ei.value) == case["msg"]
        return
    mapping = trace_io.read_mapping(case["map"])
    if "error" in case:
        exc = trace_io.MappingError if case["error"] == "MappingError" else trace_io.TraceFormatError
        with pytest.raises(exc) as ei:
            trace_io.import_mapped(case["doc"], mapping)
        assert str(ei.value) == case["msg"]
        return
    t, w = trace_io.import_mapped(case["doc"], mapping)
    assert _enc(t) == case["trace"]
    assert w == case["warnings"]


def test_import_native_fast_path_decides_plain_documents():
    mapping = trace_io.read_mapping(json.dumps({"default_policy": "drop", "rules": [
        {"name_contains": "k", "target": "kernel", "resource": "pid"}]}))
    evs = [{"name": f"k{i}", "ph": "X", "ts": i, "dur": 2, "pid": i % 3, "args": {"a": [1, "]"]}}
           for i in range(20000)]
    t, w = trace_io.import_mapped(json.dumps({"traceEvents": evs}), mapping, nthreads=4)
    assert len(t.device_records) == 20000 and not w
    assert min(r.interval.start for r in t.device_records) == 0
    assert max(r.interval.end for r in t.device_records) == 19999 * 1000 + 2000
    assert t.devices == tuple(trace_io.DeviceDecl(d) for d in (0, 1, 2))


@pytest.mark.parametrize("case", [c for c in CASES if "trace" in c], ids=[c["tag"] for c in CASES if "trace" in c])
def test_import_mapped_packed_equals_pack_of_reference_trace(case):
    from golden_io import to_trace
    from paper_2603_26576_b200.packing import pack_trace

    import numpy as np

    ref = pack_trace(to_trace(case["trace"]))
    got, w = trace_io.import_mapped_packed(case["doc"], trace_io.read_mapping(case["map"]))
    assert w == case["warnings"]
    for side in ("host", "dev"):
        a, b = getattr(got, side), getattr(ref, side)
        for col in ("start", "end", "res", "kind"):
            assert np.array_equal(getattr(a, col), getattr(b, col)), (side, col)
    assert list(got.host_ids) == list(ref.host_ids) and list(got.dev_ids) == list(ref.dev_ids)
    assert (got.n, got.m) == (ref.n, ref.m)
