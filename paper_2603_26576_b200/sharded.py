"""Multi-GPU: the trace sharded by rank blocks, one process per GPU.

Per-rank host summaries and per-device summaries are independent
(summarize.py:74-86, :119-132); the only global coupling is the elapsed time
E = max span_end over ALL ranks (summarize.py:88-89).  Each GPU therefore
runs the single-launch analysis on its shard with its LOCAL E (speculative),
then ONE all-gather of a fixed-size buffer exchanges ``(E_local, max device
end, status, sizes)`` plus the summaries (buffer sizes follow from the rank
blocks, so no size exchange is needed):

* devices whose records all end by E_local are unclamped, so their union
  lengths are final; only ``idle = E - kernel - memory`` is re-based on the
  global E;
* a shard with a device record ending past its local E (possible only if
  E_global > E_local) re-runs its device pass with the explicit global
  window (MODE_SUMMARIZE_DEVICE) -- exact, and rare by construction;
* the global metric trees are evaluated from the gathered summaries with the
  same exactly-rounded metric kernel (heteff_host_metrics /
  heteff_device_metrics).

Integer sums are order independent, so the result is bit-identical for any
GPU count.  ``combine`` is written against plain callables so the exchange
and merge logic is tested on CPU with the gloo backend
(tests/test_sharded_gloo.py).
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np


def rank_blocks(n_ranks: int, world: int) -> list[tuple[int, int]]:
    """Contiguous rank blocks, the first ``n_ranks % world`` one rank longer."""
    base, extra = divmod(n_ranks, world)
    out, r = [], 0
    for g in range(world):
        k = base + (1 if g < extra else 0)
        out.append((r, r + k))
        r += k
    return out


def combine(f, dist, tensor_device, recompute_device, metrics_fn, n_max: int | None = None,
            m_max: int | None = None):
    """Merge this shard's findings with every other shard's.

    f                 -- this shard's Findings (engine or oracle; needs host_elapsed, dev_max_end,
                         status, host_sum, dev_sum)
    dist              -- torch.distributed (initialised; nccl or gloo)
    tensor_device     -- "cuda:<i>" for nccl, "cpu" for gloo
    recompute_device  -- callable(E_global) -> dev_sum (uint64 [m][4]) for the explicit window
    metrics_fn        -- callable(rows uint64 [k][4], E, host_side) -> tuple of metrics
    n_max, m_max      -- the largest shard's rank / device counts (known from the rank blocks);
                         when given, the whole exchange is ONE all-gather of a fixed-size
                         buffer [meta | host rows | device rows] per rank (a second one only
                         if some shard clamped device records at its local E)
    Returns a Findings-like object with global E, global summaries and metrics (status of the job).
    """
    import torch

    world = dist.get_world_size()
    rank = dist.get_rank()
    n_loc, m_loc = f.host_sum.shape[0], f.dev_sum.shape[0]
    if n_max is None or m_max is None:   # sizes unknown: one tiny all-gather first
        sz = torch.tensor([n_loc, m_loc], dtype=torch.int64, device=tensor_device)
        szs = [torch.zeros_like(sz) for _ in range(world)]
        dist.all_gather(szs, sz)
        n_max = int(max(int(x[0]) for x in szs))
        m_max = int(max(int(x[1]) for x in szs))
    H, D = 5, 5 + 4 * n_max
    buf = np.zeros(5 + 4 * (n_max + m_max), dtype=np.uint64)
    buf[:5] = [int(f.host_elapsed), int(f.dev_max_end), int(f.status), n_loc, m_loc]
    buf[H:H + 4 * n_loc] = f.host_sum.reshape(-1)
    buf[D:D + 4 * m_loc] = f.dev_sum.reshape(-1)

    def gather(arr):
        t = torch.from_numpy(arr.view(np.int64)).to(tensor_device)
        parts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return [p.cpu().numpy().view(np.uint64) for p in parts]

    parts = gather(buf)
    E = int(max(int(p[0]) for p in parts))
    status = max(int(p[2]) for p in parts)
    n_of = [int(p[3]) for p in parts]
    m_of = [int(p[4]) for p in parts]
    host_rows = [p[H:H + 4 * n_of[r]].reshape(-1, 4) for r, p in enumerate(parts)]
    dev_rows = [p[D:D + 4 * m_of[r]].reshape(-1, 4).copy() for r, p in enumerate(parts)]
    # shards whose device records ran past their local E were clamped there: re-run them
    # with the global window (rare); everyone else only re-bases idle on the global E
    redo = [r for r, p in enumerate(parts) if int(p[1]) > int(p[0]) and E > int(p[0])]
    if redo:
        mine = np.zeros(4 * m_max, dtype=np.uint64)
        if rank in redo:
            rows = recompute_device(E)
            mine[: rows.size] = rows.reshape(-1)
        again = gather(mine)
        for r in redo:
            dev_rows[r] = again[r][: 4 * m_of[r]].reshape(-1, 4).copy()
    for r in range(world):
        if r not in redo and dev_rows[r].size:
            dev_rows[r][:, 2] = np.uint64(E) - dev_rows[r][:, 0] - dev_rows[r][:, 1]
    host_all = np.concatenate(host_rows) if host_rows else np.zeros((0, 4), np.uint64)
    dev_all = np.concatenate(dev_rows) if dev_rows else np.zeros((0, 4), np.uint64)
    hm = metrics_fn(host_all, E, True) if host_all.shape[0] and status == 0 else f.host_metrics
    dm = metrics_fn(dev_all, E, False) if dev_all.shape[0] and status == 0 else f.device_metrics
    return replace(f, status=status, elapsed=E, host_elapsed=E, host_sum=host_all, dev_sum=dev_all,
                   host_metrics=tuple(hm), device_metrics=tuple(dm))


def combine_shards(f, dt, dist, device: int, stream, n_max: int | None = None, m_max: int | None = None):
    """Engine flavour of :func:`combine` (NCCL, GPU re-run and GPU metric kernel)."""
    from . import _native as N
    from .engine import analyze_device, metrics_from_summaries

    def recompute(E):
        g = analyze_device(dt, N.MODE_SUMMARIZE_DEVICE, elapsed=E, stream=stream, device=device)
        return g.dev_sum

    def metrics(rows, E, host_side):
        return metrics_from_summaries(rows, E, host_side, device=device)

    return combine(f, dist, f"cuda:{device}", recompute, metrics, n_max, m_max)
