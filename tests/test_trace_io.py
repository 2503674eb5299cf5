"""Native trace documents (csrc/ingest.cpp + trace_io.py) against the reference's
``read_trace`` (trace_io.py:96-158): fixtures made by running the reference on
its own writer's output and on hand-made edge / error documents
(tests/golden/make_golden.py ``trace_docs_corpus``).  CPU only: the parser is
host code in the engine library."""

from __future__ import annotations

import json

import numpy as np
import pytest

from golden_io import load, to_trace
from paper_2603_26576_b200 import trace_io
from paper_2603_26576_b200.packing import dev_owner_table, pack_trace

DOCS = load("trace_docs")


def _enc(t):
    return {
        "hp": list(t.host_processes),
        "dev": [[d.device_id, d.owner_rank] for d in t.devices],
        "h": [[r.rank, r.state.value, r.interval.start, r.interval.end] for r in t.host_records],
        "d": [[r.device_id, r.kind.value, r.interval.start, r.interval.end, r.stream] for r in t.device_records],
        "tu": t.time_unit,
    }


@pytest.mark.parametrize("case", DOCS, ids=[c["tag"] for c in DOCS])
def test_read_trace_matches_reference(case):
    if "error" in case:
        with pytest.raises(trace_io.TraceFormatError) as ei:
            trace_io.read_trace(case["doc"])
        assert str(ei.value) == case["error"]
        return
    t = trace_io.read_trace(case["doc"])
    assert _enc(t) == case["trace"]
    t2 = trace_io.read_trace(case["doc"].encode())
    assert _enc(t2) == case["trace"]


@pytest.mark.parametrize("case", [c for c in DOCS if "trace" in c], ids=[c["tag"] for c in DOCS if "trace" in c])
def test_read_trace_packed_equals_pack_of_reference_trace(case):
    ref_trace = to_trace(case["trace"])
    ref = pack_trace(ref_trace)
    got, owner = trace_io.read_trace_packed(case["doc"])
    for side in ("host", "dev"):
        a, b = getattr(got, side), getattr(ref, side)
        for col in ("start", "end", "res", "kind"):
            assert np.array_equal(getattr(a, col), getattr(b, col)), (side, col)
    assert list(got.host_ids) == list(ref.host_ids) and list(got.dev_ids) == list(ref.dev_ids)
    assert np.array_equal(got.host_decl, ref.host_decl) and np.array_equal(got.dev_decl, ref.dev_decl)
    assert (got.n, got.m, got.n_unique, got.m_unique) == (ref.n, ref.m, ref.n_unique, ref.m_unique)
    assert np.array_equal(owner, dev_owner_table(ref_trace, ref))


def test_native_parser_decides_wellformed_documents():
    """Writer output is parsed by the native fast path (no Python fallback)."""
    doc = next(c["doc"] for c in DOCS if c["tag"] == "usecase3").encode()
    assert trace_io._native_parse(doc, 4) is not None
    assert trace_io._native_parse(b'{"version": 1, "version": 1, "time_unit": "ns", "hosts": [], "devices": []}',
                                  1) is None


def test_parallel_parse_large_document_is_thread_count_independent():
    rng = np.random.default_rng(3)
    hosts = []
    for r in range(64):
        t = np.cumsum(rng.integers(1, 50, 400))
        hosts.append({"rank": int(r), "records": [{"state": ["useful", "offload", "mpi"][int(k)], "start": int(a),
                                                   "end": int(a) + 1} for a, k in zip(t, rng.integers(0, 3, 400))]})
    devs = [{"id": int(d), "owner_rank": int(d), "records": [{"kind": "kernel", "start": int(a), "end": int(a) + 9}
                                                             for a in rng.integers(0, 20000, 300)]} for d in range(64)]
    doc = json.dumps({"version": 1, "time_unit": "ns", "hosts": hosts, "devices": devs}).encode()
    a = trace_io._native_parse(doc, 1)
    b = trace_io._native_parse(doc, 8)
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    assert a["h_start"].size == 64 * 400 and a["d_start"].size == 64 * 300
