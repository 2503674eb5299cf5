"""Multi-process (world size 2, gloo, CPU) test of the rank-sharded merge.

Each process analyses its rank block with the C oracle (stand-in for the
per-GPU engine launch), then ``sharded.combine`` exchanges E and the
summaries exactly as the NCCL path does on B200s.  The merged result must be
bit-identical to analysing the whole trace at once (summarize.py:88-89 makes
E the only global coupling).
"""

from __future__ import annotations

import os
import socket
import sys
from dataclasses import dataclass
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


@dataclass
class ShardFindings:
    status: int
    elapsed: int
    host_elapsed: int
    dev_max_end: int
    host_sum: np.ndarray
    dev_sum: np.ndarray
    host_metrics: tuple
    device_metrics: tuple


def _exact_metrics(rows, E, host_side):
    """metrics.py:66-122 with Python's exact int/int (test-side reference)."""
    rows = [[int(x) for x in r] for r in rows]
    k = len(rows)
    if host_side:
        su = sum(r[0] for r in rows)
        uw = [r[0] + r[1] for r in rows]
        suw, muw = sum(uw), max(uw)
        if suw == 0:
            return (0.0, None, None, None, None)
        return (su / (E * k), suw / (E * k), muw / E, suw / (k * muw), su / suw)
    sk = sum(r[0] for r in rows)
    mk = max(r[0] for r in rows)
    mkm = max(r[0] + r[1] for r in rows)
    pe = sk / (E * k)
    if mk == 0:
        return (pe, None, None, mkm / E if mkm > 0 else 0.0)
    return (pe, sk / (k * mk), mk / mkm, mkm / E)


def _trace():
    """Two ranks x 2 devices; rank 1's host ends early, its devices run past it."""
    rng = np.random.default_rng(7)

    def chain(n, step_max):
        d = rng.integers(1, step_max, size=n).astype(np.uint64)
        g = rng.integers(0, 5, size=n).astype(np.uint64)
        e = np.cumsum(g + d)
        return (e - d).astype(np.uint64), e.astype(np.uint64)

    hs0, he0 = chain(4000, 60)
    hs1, he1 = chain(1500, 60)
    hs = np.concatenate([hs0, hs1])
    he = np.concatenate([he0, he1])
    hr = np.concatenate([np.zeros(4000, np.int32), np.ones(1500, np.int32)])
    hk = rng.integers(0, 3, size=hs.size).astype(np.uint8)
    dev = []
    for d, span in ((0, int(he0[-1])), (1, int(he0[-1]) // 2), (2, int(he1[-1]) * 3), (3, int(he1[-1]))):
        s = np.sort(rng.integers(0, span, size=3000)).astype(np.uint64)
        e = s + rng.integers(1, 300, size=3000).astype(np.uint64)
        dev.append((s, e, np.full(3000, d, np.int32), rng.integers(0, 2, size=3000).astype(np.uint8)))
    ds, de, dr, dk = (np.concatenate([x[i] for x in dev]) for i in range(4))
    return (hs, he, hr, hk), (ds, de, dr, dk)


def _shard(h, d, r0, r1, g):
    hm = (h[2] >= r0) & (h[2] < r1)
    dm = (d[2] >= r0 * g) & (d[2] < r1 * g)
    hh = tuple(x[hm] for x in h)
    dd = tuple(x[dm] for x in d)
    hh = (hh[0], hh[1], (hh[2] - r0).astype(np.int32), hh[3])
    dd = (dd[0], dd[1], (dd[2] - r0 * g).astype(np.int32), dd[3])
    return hh, dd


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    from oracle import oracle as O
    from paper_2603_26576_b200.sharded import combine, rank_blocks

    dist.init_process_group("gloo", rank=rank, world_size=world)
    h, d = _trace()
    g = 2
    r0, r1 = rank_blocks(2, world)[rank]
    hh, dd = _shard(h, d, r0, r1, g)
    n, m = r1 - r0, (r1 - r0) * g
    res = O.analyze(hh, dd, n, m)
    f = ShardFindings(res.status, res.elapsed, res.host_elapsed, int(dd[1].max()) if dd[1].size else 0,
                      res.host_sum, res.dev_sum, res.host_metrics, res.device_metrics)

    def recompute(E):
        return O.analyze(hh, dd, n, m, mode=O.MODE_SUMMARIZE_DEVICE, elapsed=E).dev_sum

    sizes = [b - a for a, b in rank_blocks(2, world)]
    out = combine(f, dist, "cpu", recompute, _exact_metrics, max(sizes), max(sizes) * g)
    out2 = combine(f, dist, "cpu", recompute, _exact_metrics)   # sizes exchanged first
    assert out2.elapsed == out.elapsed and np.array_equal(out2.dev_sum, out.dev_sum)
    if rank == 0:
        q.put((out.elapsed, out.host_sum.tolist(), out.dev_sum[:, :3].tolist(), out.host_metrics,
               out.device_metrics))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_rank_blocks():
    from paper_2603_26576_b200.sharded import rank_blocks
    assert rank_blocks(10, 4) == [(0, 3), (3, 6), (6, 8), (8, 10)]
    assert rank_blocks(1024, 8)[-1] == (896, 1024)


@pytest.mark.timeout(240)
def test_two_process_merge_matches_whole_trace():
    import torch.multiprocessing as mp

    from oracle import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=200)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    h, d = _trace()
    full = O.analyze(h, d, 2, 4)
    E, hs, ds, hm, dm = got
    assert E == full.elapsed
    assert hs == full.host_sum.tolist()
    assert ds == full.dev_sum[:, :3].tolist()
    assert tuple(hm) == full.host_metrics
    assert tuple(dm) == full.device_metrics
    # the shard of rank 1 really exercised the re-run with the global window
    hh, dd = _shard(h, d, 1, 2, 2)
    assert int(dd[1].max()) > int(hh[1].max())
