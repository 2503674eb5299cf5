"""K0: config-shaped synthetic traces generated directly in HBM.

Uses torch only for device memory; the arrays are written by the engine's
own generator kernel (``heteff_generate``, csrc/gen.cu).
"""

from __future__ import annotations

import ctypes as C

from . import _native as N
from .configs import Config, GenSideParams
from .engine import DeviceTrace


def _side(lib, ctx, p: GenSideParams, device, stream):
    import torch

    dev = torch.device("cuda", device)
    start = torch.empty(p.count, dtype=torch.int64, device=dev)   # u64 bits
    end = torch.empty(p.count, dtype=torch.int64, device=dev)
    res = torch.empty(p.count, dtype=torch.int32, device=dev)
    kind = torch.empty(p.count, dtype=torch.uint8, device=dev)
    g = N.GenSide(p.seed & ((1 << 64) - 1), p.n_res, p.res_base, p.per_res, p.extra_below, p.serialized,
                  p.count, p.gap_max, p.dur_max, p.dur_scale0, p.kernel_pct, p.is_host, 0)
    if p.count:
        rc = lib.heteff_generate(ctx, C.byref(g), start.data_ptr(), end.data_ptr(), res.data_ptr(),
                                 kind.data_ptr(), stream)
        if rc != N.OK:
            raise N.NativeError(f"heteff_generate failed ({rc}): {N.last_error(ctx)}")
    return start, end, res, kind


def generate(cfg: Config, r0: int = 0, r1: int | None = None, device: int = 0) -> DeviceTrace:
    """Ranks [r0, r1) of ``cfg`` (and the devices they own) as an HBM-resident trace."""
    import torch

    r1 = cfg.n_ranks if r1 is None else r1
    g = cfg.gpus_per_rank
    lib = N.load()
    ctx = N.context(device)
    stream = torch.cuda.current_stream(device).cuda_stream
    hp, dp = cfg.host_side(r0, r1), cfg.dev_side(r0 * g, r1 * g)
    hs, he, hr, hk = _side(lib, ctx, hp, device, stream)
    ds, de, dr, dk = _side(lib, ctx, dp, device, stream)
    torch.cuda.synchronize(device)
    return DeviceTrace(hs, he, hr, hk, ds, de, dr, dk, r1 - r0, (r1 - r0) * g, 0, _seg(hp, device), _seg(dp, device))


def _seg(p: GenSideParams, device):
    """CSR offsets of one generated side: resource i holds per_res records (+1 below extra_below)."""
    import torch

    gids = torch.arange(p.res_base, p.res_base + p.n_res, dtype=torch.int64)
    counts = p.per_res + (gids < p.extra_below).to(torch.int64)
    seg = torch.zeros(p.n_res + 1, dtype=torch.int64)
    torch.cumsum(counts, 0, out=seg[1:])
    assert int(seg[-1]) == p.count
    return seg.to(torch.device("cuda", device))
