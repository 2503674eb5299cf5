"""CPU-only checks of the host side: the C ABI library exports, the packer, the
message formatter on oracle findings, configs and the generator twin."""

from __future__ import annotations

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from golden_io import load, to_trace

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_declared_symbol():
    from paper_2603_26576_b200 import _native as N
    lib = N.load()   # loading needs no GPU
    header = (ROOT / "include" / "heteff_b200.h").read_text()
    declared = set(re.findall(r"\b(heteff_[a-z_]+)\s*\(", header))
    assert declared == set(N.EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.heteff_abi_version() == 2


def test_library_is_built_for_sm100a():
    import subprocess
    lib = ROOT / "paper_2603_26576_b200" / "libheteff_b200.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts_match_the_header():
    from paper_2603_26576_b200 import _native as N
    # offsets fixed by include/heteff_b200.h (x86-64, natural alignment)
    assert C.sizeof(N.Records) == 40
    assert N.TraceABI.n.offset == 104 and N.TraceABI.host_elapsed_floor.offset == 112
    assert N.TraceABI.host_seg.offset == 120 and C.sizeof(N.TraceABI) == 136
    assert C.sizeof(N.Options) == 24
    assert N.Result.counts.offset == 128 and C.sizeof(N.Result) == 200
    assert C.sizeof(N.GenSide) == 64


def test_packer_canonical_order_and_dense_ids():
    from paper_2603_26576_b200 import DeviceActivityKind as K, DeviceDecl, DeviceRecord, HostRecord
    from paper_2603_26576_b200 import HostState as S, Interval, Trace
    from paper_2603_26576_b200.packing import pack_trace
    t = Trace(host_processes=(5, 2), devices=(DeviceDecl(9), DeviceDecl(3)),
              host_records=(HostRecord(5, S.MPI, Interval(4, 9)), HostRecord(2, S.USEFUL, Interval(0, 3)),
                            HostRecord(7, S.OFFLOAD, Interval(1, 2))),
              device_records=(DeviceRecord(9, K.KERNEL, Interval(1, 5)), DeviceRecord(3, K.MEMORY, Interval(2, 4))))
    p = pack_trace(t)
    assert p.host_ids == [2, 5, 7]                      # reference-id order
    assert p.host_decl.tolist() == [1, 0, -1]           # declaration positions, 7 undeclared
    assert p.host.res.tolist() == [0, 1, 2]
    assert p.dev_ids == [3, 9] and p.dev_decl.tolist() == [1, 0]
    assert p.n_unique == 2 and p.m_unique == 2


def test_packer_quarantines_out_of_domain_timestamps():
    from paper_2603_26576_b200 import HostRecord, HostState as S, Interval, Trace
    from paper_2603_26576_b200.packing import pack_trace
    t = Trace(host_processes=(0,), host_records=(
        HostRecord(0, S.USEFUL, Interval(-5, 10)), HostRecord(0, S.MPI, Interval(3, 2 ** 64 + 1)),
        HostRecord(0, S.USEFUL, Interval(20, 30))))
    p = pack_trace(t)
    assert p.host.count == 1 and p.host.index.tolist() == [2]
    assert [q.index for q in p.host_q] == [0, 1]
    assert p.host_q[0].errors == ["host record 0 (rank 0): negative timestamp -5"]
    assert p.host_q[1].errors == ["host record 1 (rank 0): end 18446744073709551617 exceeds 64-bit range"]
    assert p.host_elapsed_floor == 2 ** 64 - 1


class _Findings:
    """Oracle output in the engine's Findings shape (SoA positions)."""

    def __init__(self, r, overlap_pos):
        self.lists = [r.lists[i] if i != 3 else overlap_pos for i in range(8)]
        self.host_elapsed = r.host_elapsed


@pytest.mark.parametrize("case", load("invalid")[:120], ids=[c["tag"] for c in load("invalid")[:120]])
def test_message_formatter_reproduces_reference_text(case, monkeypatch):
    """messages.validation_report on oracle findings == reference validate() strings."""
    from oracle import oracle as O
    from paper_2603_26576_b200 import messages
    from paper_2603_26576_b200.packing import pack_trace
    trace = to_trace(case["trace"])
    packed = pack_trace(trace)
    r = O.analyze_packed(packed, O.MODE_VALIDATE, cap=1 << 12)
    pairs = r.lists[3]
    monkeypatch.setattr(messages, "overlap_covers",
                        lambda pk, pos: np.array([int(c) for c, i in pairs], dtype=np.int64))
    v = messages.validation_report(trace, packed, _Findings(r, np.array([int(i) for c, i in pairs], np.int64)))
    assert v.errors == case["validate"]["errors"]
    assert v.warnings == case["validate"]["warnings"]


def test_config_sides_count_every_record():
    from paper_2603_26576_b200.configs import CONFIGS
    for cfg in CONFIGS.values():
        h, d = cfg.host_side(), cfg.dev_side()
        assert h.count == cfg.host_records and d.count == cfg.dev_records
        blocks = [cfg.host_side(a, a + cfg.n_ranks // 4) for a in range(0, cfg.n_ranks, cfg.n_ranks // 4)]
        assert sum(b.count for b in blocks) == cfg.host_records


def test_engine_raises_without_gpu():
    """The product path never falls back to the CPU."""
    from conftest import gpu_available
    if gpu_available():
        pytest.skip("GPU present")
    import paper_2603_26576_b200 as hb
    t = hb.Trace(host_processes=(0,), host_records=(hb.HostRecord(0, hb.HostState.USEFUL, hb.Interval(0, 5)),))
    with pytest.raises(Exception):
        hb.compute_report(t)


@pytest.mark.parametrize("seg", [[1, 5, 10], [0, 5, 9], [0, 6, 5, 10]])
def test_csr_offsets_are_checked_before_any_device_work(seg):
    """heteff_analyze_host_csr rejects malformed CSR offsets with BAD_ARG (no GPU needed)."""
    from paper_2603_26576_b200 import _native as N

    lib = N.load()
    ids = len(seg) - 1
    t = N.TraceABI(N.Records(None, None, None, None, 10), N.Records(None, None, None, None, 0),
                   ids, 0, None, None, ids, 0, 0)
    hseg = np.array(seg, dtype=np.int64)
    dseg = np.zeros(1, dtype=np.int64)
    rc = lib.heteff_analyze_host_csr(None, C.byref(t), hseg.ctypes.data, dseg.ctypes.data, None, None, None, None)
    assert rc == N.BAD_ARG


def test_metric_stage_functions_refuse_elapsed_beyond_u64():
    """The metric kernels take E as u64; a larger E raises instead of being truncated
    by the C call (no GPU needed: the check precedes the native call)."""
    import paper_2603_26576_b200 as hb
    big = 2 ** 64 + 5
    with pytest.raises(OverflowError):
        hb.host_metrics([hb.HostSummary(0, 1, 2, 3, 6)], big)
    with pytest.raises(OverflowError):
        hb.device_metrics([hb.DeviceSummary(0, 1, 2, 3)], big)
    with pytest.raises(ValueError):   # the reference's own checks still come first
        hb.host_metrics([], big)
