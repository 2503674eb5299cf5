"""Times the UNMODIFIED reference package on the box's host cores -- BASELINE ONLY.

``baseline/_ref`` holds the reference ``heteff`` package installed from
``/root/reference/pkg`` (``python -m pip install --no-index --no-build-isolation
--find-links /opt/wheelhouse --target baseline/_ref <copy of /root/reference/pkg>``;
git-ignored, it travels to the GPU box with the snapshot).  Nothing of this repo's
engine is on this path: the columns come from ``oracle/gen.py`` (numpy), the records
are the reference's own dataclasses, and the timed calls are the reference's stage
functions -- BASELINE.md's CPU plan, items 1-2:

* 1 core: ``summarize_host`` (summarize.py:57-92), ``summarize_device(trace, E)``
  (summarize.py:95-138), ``host_metrics`` / ``device_metrics`` (metrics.py:66-122)
  on one rank shard (the first k ranks of the config);
* all cores: the same shard split by rank over processes -- every worker runs
  ``summarize_host`` on its ranks, the parent takes E = max, every worker runs
  ``summarize_device(part, E)`` (the exact sharded form), the parent
  evaluates both metric trees on the gathered summaries.

Trace construction (Python record objects, the canonical sort) is ingest and stays
outside the timed region, as in BASELINE.md's measurements.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"


def available() -> str | None:
    """None if the reference package imports from baseline/_ref, else why not."""
    if not (REF / "heteff" / "__init__.py").exists():
        return "baseline/_ref/heteff is not installed"
    try:
        _heteff()
    except Exception as e:   # pragma: no cover - reported, not raised
        return f"import failed: {e!r}"
    return None


def _heteff():
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import heteff

    assert Path(heteff.__file__).resolve().is_relative_to(REF.resolve()), heteff.__file__
    return heteff


def _trace(hx, cfg, r0: int, r1: int):
    """The reference Trace of ranks [r0, r1) of cfg (devices follow their owner rank)."""
    sys.path.insert(0, str(ROOT))
    from oracle import gen as ogen

    (hs, he, hr, hk), (ds, de, dr, dk) = ogen.generate(cfg, r0, r1)
    g = cfg.gpus_per_rank
    states = (hx.HostState.USEFUL, hx.HostState.OFFLOAD, hx.HostState.MPI)
    kinds = (hx.DeviceActivityKind.KERNEL, hx.DeviceActivityKind.MEMORY)
    HR, DR, IV = hx.HostRecord, hx.DeviceRecord, hx.Interval
    host = [HR(r0 + int(r), states[k], IV(int(s), int(e)))
            for s, e, r, k in zip(hs.tolist(), he.tolist(), hr.tolist(), hk.tolist())]
    dev = [DR(r0 * g + int(r), kinds[k], IV(int(s), int(e)))
           for s, e, r, k in zip(ds.tolist(), de.tolist(), dr.tolist(), dk.tolist())]
    return hx.Trace(host_processes=tuple(range(r0, r1)),
                    devices=tuple(hx.DeviceDecl(d, d // g) for d in range(r0 * g, r1 * g)),
                    host_records=host, device_records=dev), len(host) + len(dev)


def _ranks_for(cfg, intervals: float) -> int:
    per_rank = cfg.intervals / cfg.n_ranks
    return max(1, min(cfg.n_ranks, int(round(intervals / per_rank))))


def time_single(cfg, intervals: float) -> dict:
    """Reference stage functions on the first k ranks, one process (the package is single-threaded)."""
    hx = _heteff()
    k = _ranks_for(cfg, intervals)
    tr, count = _trace(hx, cfg, 0, k)
    t0 = time.perf_counter()
    hsum, E = hx.summarize_host(tr)
    dsum, _ = hx.summarize_device(tr, E)
    hm = hx.host_metrics(hsum, E)
    dm = hx.device_metrics(dsum, E)
    sec = time.perf_counter() - t0
    return {"value": count / sec, "unit": "intervals/s", "cores": 1, "seconds": sec, "intervals": count,
            "ranks": k, "elapsed": E, "host_metrics": _floats(hm), "device_metrics": _floats(dm)}


def _floats(m) -> list:
    return [getattr(m, f) for f in m.__dataclass_fields__]


def _worker(cfg, r0: int, r1: int, conn, barrier) -> None:
    hx = _heteff()
    tr, count = _trace(hx, cfg, r0, r1)
    barrier.wait()
    hsum, E = hx.summarize_host(tr)
    conn.send((E, count))
    Eg = conn.recv()
    dsum, _ = hx.summarize_device(tr, Eg)
    conn.send((hsum, dsum))
    conn.close()


def time_parallel(cfg, intervals: float, procs: int | None = None) -> dict:
    """The same shard split by rank over ``procs`` processes (default: every host core)."""
    hx = _heteff()
    procs = procs or os.cpu_count() or 1
    k = _ranks_for(cfg, intervals)
    procs = max(1, min(procs, k))
    bounds = [k * i // procs for i in range(procs + 1)]
    ctx = mp.get_context("fork")
    barrier = ctx.Barrier(procs + 1)
    pipes, workers = [], []
    for i in range(procs):
        a, b = ctx.Pipe()
        w = ctx.Process(target=_worker, args=(cfg, bounds[i], bounds[i + 1], b, barrier))
        w.start()
        pipes.append(a)
        workers.append(w)
    barrier.wait()                      # every worker holds its Trace
    t0 = time.perf_counter()
    got = [p.recv() for p in pipes]
    E = max(e for e, _ in got)
    count = sum(c for _, c in got)
    for p in pipes:
        p.send(E)
    parts = [p.recv() for p in pipes]
    hsum = [h for hs, _ in parts for h in hs]
    dsum = [d for _, ds in parts for d in ds]
    hm = hx.host_metrics(hsum, E)
    dm = hx.device_metrics(dsum, E)
    sec = time.perf_counter() - t0
    for w in workers:
        w.join()
    return {"value": count / sec, "unit": "intervals/s", "cores": procs, "seconds": sec, "intervals": count,
            "ranks": k, "elapsed": E, "host_metrics": _floats(hm), "device_metrics": _floats(dm)}
