"""Multi-GPU: the trace sharded by rank blocks, one process per GPU.

Per-rank host summaries and per-device summaries are independent
(summarize.py:74-86, :119-132); the only global coupling is the elapsed time
E = max span_end over ALL ranks (summarize.py:88-89).  Each GPU therefore
runs the single-launch analysis on its shard with its LOCAL E (speculative),
then one small all-gather exchanges ``(E_local, max device end)`` plus the
summaries:

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


def combine(f, dist, tensor_device, recompute_device, metrics_fn):
    """Merge this shard's findings with every other shard's.

    f                 -- this shard's Findings (engine or oracle; needs host_elapsed, dev_max_end,
                         status, host_sum, dev_sum)
    dist              -- torch.distributed (initialised; nccl or gloo)
    tensor_device     -- "cuda:<i>" for nccl, "cpu" for gloo
    recompute_device  -- callable(E_global) -> dev_sum (uint64 [m][4]) for the explicit window
    metrics_fn        -- callable(rows uint64 [k][4], E, host_side) -> tuple of metrics
    Returns a Findings-like object with global E, global summaries and metrics (status of the job).
    """
    import torch

    world = dist.get_world_size()
    meta = torch.tensor([int(f.host_elapsed), int(f.dev_max_end), int(f.status), f.host_sum.shape[0],
                         f.dev_sum.shape[0]], dtype=torch.int64, device=tensor_device)
    metas = [torch.zeros_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta)
    metas = [m.cpu().numpy().astype(np.uint64) for m in metas]
    E = int(max(int(m[0]) for m in metas))
    status = max(int(m[2]) for m in metas)
    dev_sum = f.dev_sum
    if int(f.dev_max_end) > int(f.host_elapsed) and E > int(f.host_elapsed):
        dev_sum = recompute_device(E)            # some record was clamped at the local window
    else:
        dev_sum = dev_sum.copy()
        dev_sum[:, 2] = np.uint64(E) - dev_sum[:, 0] - dev_sum[:, 1]
    n_max = int(max(int(m[3]) for m in metas))
    m_max = int(max(int(m[4]) for m in metas))

    def gather_rows(rows, kmax):
        pad = np.zeros((kmax, 4), dtype=np.uint64)
        pad[: rows.shape[0]] = rows
        t = torch.from_numpy(pad.view(np.int64)).to(tensor_device)
        parts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return [p.cpu().numpy().view(np.uint64) for p in parts]

    hs = gather_rows(f.host_sum, n_max)
    ds = gather_rows(dev_sum, m_max)
    host_rows = np.concatenate([h[: int(m[3])] for h, m in zip(hs, metas)])
    dev_rows = np.concatenate([d[: int(m[4])] for d, m in zip(ds, metas)])
    hm = metrics_fn(host_rows, E, True) if host_rows.shape[0] and status == 0 else f.host_metrics
    dm = metrics_fn(dev_rows, E, False) if dev_rows.shape[0] and status == 0 else f.device_metrics
    return replace(f, status=status, elapsed=E, host_elapsed=E, host_sum=host_rows, dev_sum=dev_rows,
                   host_metrics=tuple(hm), device_metrics=tuple(dm))


def combine_shards(f, dt, dist, device: int, stream):
    """Engine flavour of :func:`combine` (NCCL, GPU re-run and GPU metric kernel)."""
    from . import _native as N
    from .engine import analyze_device, metrics_from_summaries

    def recompute(E):
        g = analyze_device(dt, N.MODE_SUMMARIZE_DEVICE, elapsed=E, stream=stream, device=device)
        return g.dev_sum

    def metrics(rows, E, host_side):
        return metrics_from_summaries(rows, E, host_side, device=device)

    return combine(f, dist, f"cuda:{device}", recompute, metrics)
