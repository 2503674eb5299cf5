"""The device-resident multi-GPU protocol (sharded.DeviceMerge) on ONE GPU: each
simulated rank summarizes its host records into its block, the local E values are
max-reduced (what NCCL's all-reduce does), each rank summarizes its device records
with that global E read from device memory, and the merge kernel over the gathered
blocks must reproduce the whole-trace analysis bit for bit."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

import torch  # noqa: E402

from paper_2603_26576_b200 import _native as N  # noqa: E402
from paper_2603_26576_b200.configs import CONFIGS, scaled  # noqa: E402
from paper_2603_26576_b200.engine import _dptr, _findings, analyze_device  # noqa: E402
from paper_2603_26576_b200.sharded import rank_blocks  # noqa: E402
from paper_2603_26576_b200.synth import generate  # noqa: E402


def _simulate(cfg, world):
    lib, ctx = N.load(), N.context()
    blocks = rank_blocks(cfg.n_ranks, world)
    g = cfg.gpus_per_rank
    n_of = [b - a for a, b in blocks]
    m_of = [x * g for x in n_of]
    nmax, mmax = max(n_of), max(m_of)
    B = 512 + 32 * (nmax + mmax)
    gathered = torch.zeros(world * B // 8, dtype=torch.int64, device="cuda")
    e = torch.zeros(1, dtype=torch.int64, device="cuda")
    none = N.Records(None, None, None, None, 0)
    shards = [generate(cfg, a, b) for a, b in blocks]
    for r, dt in enumerate(shards):   # step 1 on every rank
        hrec = N.Records(_dptr(dt.h_start), _dptr(dt.h_end), _dptr(dt.h_res), _dptr(dt.h_kind), dt.host_count)
        t = N.TraceABI(hrec, none, dt.n, 0, None, None, dt.n, 0, 0)
        assert lib.heteff_analyze_into(ctx, C.byref(t), C.byref(N.Options(N.MODE_SUMMARIZE_HOST, 0, 0, 0)),
                                       gathered.data_ptr() + r * B, B, nmax, mmax, None) == N.OK
    view = gathered.view(world, B // 8)
    e.copy_(view[:, 2].max().reshape(1))   # step 2: all-reduce MAX of the local E
    for r, dt in enumerate(shards):   # step 3
        drec = N.Records(_dptr(dt.d_start), _dptr(dt.d_end), _dptr(dt.d_res), _dptr(dt.d_kind), dt.dev_count)
        t = N.TraceABI(none, drec, 0, dt.m, None, None, 0, dt.m, 0)
        opt = N.Options(N.MODE_SUMMARIZE_DEVICE, N.FLAG_ELAPSED_DEVICE_PTR, e.data_ptr(), 0)
        assert lib.heteff_analyze_into(ctx, C.byref(t), C.byref(opt), gathered.data_ptr() + r * B, B, nmax, mmax,
                                       None) == N.OK
    res = N.Result()
    hs = np.zeros((sum(n_of), 4), dtype=np.uint64)
    ds = np.zeros((sum(m_of), 4), dtype=np.uint64)
    out = N.Outputs(hs.ctypes.data, ds.ctypes.data, (C.c_void_p * N.NUM_LISTS)())
    rc = lib.heteff_merge_shards(ctx, gathered.data_ptr(), world, B, nmax, mmax, (C.c_int32 * world)(*n_of),
                                 (C.c_int32 * world)(*m_of), e.data_ptr(), C.byref(res), C.byref(out), None)
    return rc, _findings(res, hs, ds, [])


@pytest.mark.parametrize("name,ranks,world", [("c2", 64, 8), ("c3", 16, 4), ("c1", 4, 2), ("c1", 4, 4),
                                              ("c5", 40, 8), ("c4", 24, 3)])
def test_device_protocol_equals_whole_trace(name, ranks, world):
    cfg = scaled(CONFIGS[name], ranks) if CONFIGS[name].n_ranks > ranks else CONFIGS[name]
    whole = analyze_device(generate(cfg))
    rc, got = _simulate(cfg, world)
    assert rc == N.OK and got.status == N.OK
    assert got.elapsed == whole.elapsed
    assert np.array_equal(got.host_sum, whole.host_sum)
    assert np.array_equal(got.dev_sum, whole.dev_sum)         # incl. clamp counts at the global E
    assert got.host_metrics == whole.host_metrics and got.device_metrics == whole.device_metrics
