"""Rendering + CLI (report.py, cli.py) against the reference's render_text /
render_json on the reference's own reports (tests/golden ``renders``), and the
writer against the reference's write_trace bytes.  The renderer and writer run
on CPU; the CLI analyze path needs the GPU engine."""

from __future__ import annotations

import json

import pytest

from conftest import gpu_available
from golden_io import load, to_trace, unhex
from paper_2603_26576_b200 import trace_io
from paper_2603_26576_b200.report import RenderOptions, render_json, render_text

RENDERS = load("renders")


class _M:   # a report-shaped object built from the reference's JSON rendering (full precision)
    def __init__(self, **kw):
        self.__dict__.update(kw)


def _report_from(case):
    doc = json.loads(case["renders"]["json-raw"])
    host = None if doc["host"] is None else _M(**doc["host"])
    dev = None if doc["device"] is None else _M(**doc["device"])
    hs = [_M(rank=h["rank"], d_useful=h["useful_ns"], d_offload=h["offload_ns"], d_mpi=h["mpi_ns"],
             span_end=h["span_end_ns"]) for h in doc["raw"]["hosts"]]
    ds = [_M(device_id=d["id"], d_kernel=d["kernel_ns"], d_memory=d["memory_ns"], d_idle=d["idle_ns"])
          for d in doc["raw"]["devices"]]
    return _M(elapsed_ns=doc["elapsed_ns"], n=doc["n"], m=doc["m"], host=host, device=dev, host_summaries=hs,
              device_summaries=ds, warnings=doc["warnings"])


@pytest.mark.parametrize("case", RENDERS, ids=[c["tag"] for c in RENDERS])
def test_render_matches_reference_bytes(case):
    r = _report_from(case)
    for key, want in case["renders"].items():
        if key.startswith("text-"):
            _, prec, raw, asc = key.split("-")
            assert render_text(r, RenderOptions("text", int(prec), raw == "1", asc == "1")) == want, key
        elif key == "json-raw":
            assert render_json(r, RenderOptions("json", 2, True, False)).decode() == want
        else:
            assert render_json(r, RenderOptions("json", int(key.split("-")[1]))).decode() == want


@pytest.mark.parametrize("case", RENDERS, ids=[c["tag"] for c in RENDERS])
def test_write_trace_matches_reference_bytes(case):
    assert trace_io.write_trace(trace_io.read_trace(case["doc"])).decode() == case["doc"]


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
@pytest.mark.parametrize("case", RENDERS, ids=[c["tag"] for c in RENDERS])
def test_cli_analyze_on_the_engine_matches_reference(case, tmp_path, capsysbinary):
    from paper_2603_26576_b200.cli import main

    path = tmp_path / "t.json"
    path.write_text(case["doc"])
    for key, want in case["renders"].items():
        if key.startswith("text-"):
            _, prec, raw, asc = key.split("-")
            argv = ["analyze", str(path), "--precision", prec] + (["--show-raw"] if raw == "1" else []) + \
                   (["--ascii"] if asc == "1" else [])
        elif key == "json-raw":
            argv = ["analyze", str(path), "--format", "json", "--show-raw"]
        else:
            argv = ["analyze", str(path), "--format", "json", "--precision", key.split("-")[1]]
        assert main(argv) == 0
        assert capsysbinary.readouterr().out.decode() == want, key


def test_cli_usage_and_io_exit_codes(tmp_path, capsys):
    from paper_2603_26576_b200.cli import main

    with pytest.raises(SystemExit) as ei:
        main(["analyze"])
    assert ei.value.code == 3
    assert main(["analyze", str(tmp_path / "missing.json")]) == 2
    bad = tmp_path / "bad.json"
    bad.write_text('{"version": 2, "time_unit": "ns", "hosts": [], "devices": []}')
    assert main(["analyze", str(bad)]) == 2
    assert "$.version: unsupported version 2" in capsys.readouterr().err
