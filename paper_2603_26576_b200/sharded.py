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

    f                 -- this shard's Findings (engine or oracle; needs host_elapsed, status,
                         host_sum, dev_sum with the clamp counts in column 3)
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
    # did any device record end past the local E (clamp counts, column 3)?  Only then a
    # larger global E changes this shard's device summaries
    clamped = int(f.dev_sum[:, 3].astype(object).sum()) if f.dev_sum.shape[1] > 3 and m_loc else 0
    buf[:5] = [int(f.host_elapsed), 1 if clamped else 0, int(f.status), n_loc, m_loc]
    buf[H:H + 4 * n_loc] = f.host_sum.reshape(-1)
    buf[D:D + 4 * m_loc] = f.dev_sum.reshape(-1)

    def gather(arr):
        t = torch.from_numpy(arr.view(np.int64)).to(tensor_device)
        parts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        return [p.cpu().numpy().view(np.uint64) for p in parts]

    parts = gather(buf)
    E = int(max(int(p[0]) for p in parts))
    # a shard whose ranks recorded nothing has local E = 0 and reports ANALYSIS_ERROR on its
    # own; for the job only the GLOBAL E decides that (metrics.py:136-137), like merge_kernel
    status = max((int(p[2]) for p in parts if int(p[2]) != 2), default=0)
    if status == 0 and E == 0:
        status = 2
    n_of = [int(p[3]) for p in parts]
    m_of = [int(p[4]) for p in parts]
    host_rows = [p[H:H + 4 * n_of[r]].reshape(-1, 4) for r, p in enumerate(parts)]
    dev_rows = [p[D:D + 4 * m_of[r]].reshape(-1, 4).copy() for r, p in enumerate(parts)]
    # shards whose device records ran past their local E were clamped there: re-run them
    # with the global window (rare); everyone else only re-bases idle on the global E
    redo = [r for r, p in enumerate(parts) if int(p[1]) and E > int(p[0])]
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


class DeviceMerge:
    """The device-resident multi-GPU step (include/heteff_b200.h, "multi-GPU"): this
    rank's host records are summarized into a device result block, the local E is
    all-reduced (MAX, 8 bytes over NVLink), the device records are summarized with the
    GLOBAL E read from device memory (so no shard ever clamps at a local E and nothing
    is re-run), ONE all-gather of the fixed-size blocks follows, and one merge kernel
    evaluates the summaries and both metric trees; a single small D2H brings the report
    to the host.  Every record is read once per step, as on one GPU.  A non-OK shard
    (invalid trace, ...) defers to the synchronous host path for the exact error."""

    def __init__(self, dt, dist, device: int, stream, n_of: list[int], m_of: list[int]):
        import ctypes as C

        import torch

        from . import _native as N
        from .engine import device_trace_abi

        self.N, self.C, self.dist, self.dt, self.device, self.stream = N, C, dist, dt, device, stream
        self.lib, self.ctx = N.load(), N.context(device)
        self.world = len(n_of)
        self.n_max, self.m_max = max(n_of), max(m_of)
        self.n_of = (C.c_int32 * self.world)(*n_of)
        self.m_of = (C.c_int32 * self.world)(*m_of)
        self.bytes = 512 + 32 * (self.n_max + self.m_max)
        dev = torch.device("cuda", device)
        self.block = torch.zeros(self.bytes // 8, dtype=torch.int64, device=dev)
        self.gathered = torch.zeros(self.world * self.bytes // 8, dtype=torch.int64, device=dev)
        self.e = torch.zeros(1, dtype=torch.int64, device=dev)
        full = device_trace_abi(dt)   # res columns or CSR offsets, as the trace carries them
        none = N.Records(None, None, None, None, 0)
        self.t_host = N.TraceABI(full.host, none, dt.n, 0, None, None, dt.n, 0, dt.host_elapsed_floor,
                                 full.host_seg, None)
        self.t_dev = N.TraceABI(none, full.dev, 0, dt.m, None, None, 0, dt.m, 0, None, full.dev_seg)
        self.o_host = N.Options(N.MODE_SUMMARIZE_HOST, 0, 0, 0)
        self.o_dev = N.Options(N.MODE_SUMMARIZE_DEVICE, N.FLAG_ELAPSED_DEVICE_PTR, self.e.data_ptr(), 0)
        self.res = N.Result()
        ntot, mtot = sum(n_of), sum(m_of)
        self.host_sum = np.zeros((max(ntot, 1), 4), dtype=np.uint64)
        self.dev_sum = np.zeros((max(mtot, 1), 4), dtype=np.uint64)
        self.out = N.Outputs(self.host_sum.ctypes.data, self.dev_sum.ctypes.data, (C.c_void_p * N.NUM_LISTS)())
        self.ntot, self.mtot = ntot, mtot

    def _into(self, t, opt):
        rc = self.lib.heteff_analyze_into(self.ctx, self.C.byref(t), self.C.byref(opt), self.block.data_ptr(),
                                          self.bytes, self.n_max, self.m_max, self.stream)
        if rc != self.N.OK:
            raise self.N.NativeError(f"heteff_analyze_into failed ({rc}): {self.N.last_error(self.ctx)}")

    def step(self):
        from .engine import _findings, analyze_device

        N, C = self.N, self.C
        self._into(self.t_host, self.o_host)                       # host records -> local E (header byte 16)
        self.e.copy_(self.block[2:3])
        self.dist.all_reduce(self.e, op=self.dist.ReduceOp.MAX)    # global E, never on the host
        self._into(self.t_dev, self.o_dev)                         # device records clamped at the global E
        self.dist.all_gather_into_tensor(self.gathered, self.block)
        rc = self.lib.heteff_merge_shards(self.ctx, self.gathered.data_ptr(), self.world, self.bytes, self.n_max,
                                          self.m_max, self.n_of, self.m_of, self.e.data_ptr(), C.byref(self.res),
                                          C.byref(self.out), self.stream)
        if rc == N.PARSE_FALLBACK:   # some shard is not OK: the synchronous path reports it exactly
            f = analyze_device(self.dt, N.MODE_REPORT, stream=self.stream, device=self.device)
            return combine_shards(f, self.dt, self.dist, self.device, self.stream, self.n_max, self.m_max)
        if rc != N.OK:
            raise N.NativeError(f"heteff_merge_shards failed ({rc}): {N.last_error(self.ctx)}")
        return _findings(self.res, self.host_sum[: self.ntot], self.dev_sum[: self.mtot], [])


class HostCollectives:
    """TEST PLUMBING: the collectives this module issues, run by a gloo process group on
    host copies of the (CUDA) tensors -- lets several ranks share the one GPU of a test
    box, where NCCL refuses two ranks on one device (``tools/dist_check.py``,
    ``HETEFF_DIST_BACKEND=gloo`` in ``bench.py``).  Production runs use NCCL directly."""

    def __init__(self, dist):
        self._d = dist
        self.ReduceOp = dist.ReduceOp

    def all_reduce(self, t, op):
        h = t.cpu()
        self._d.all_reduce(h, op=op)
        t.copy_(h)

    def all_gather_into_tensor(self, out, inp):
        import torch

        h = torch.empty(out.numel(), dtype=out.dtype)
        self._d.all_gather_into_tensor(h, inp.cpu())
        out.copy_(h)

    def all_gather(self, outs, inp):
        hs = [o.cpu() for o in outs]
        self._d.all_gather(hs, inp.cpu())
        for o, h in zip(outs, hs):
            o.copy_(h)

    def __getattr__(self, name):
        return getattr(self._d, name)
