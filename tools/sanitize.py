"""Workloads for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool racecheck python tools/sanitize.py [small|shard|all]

Drives every kernel family of the engine at sanitizer-friendly sizes:
``analyze_kernel`` (CSR and res-column instantiations, all four modes, a grid of
four waves forced through heteff_set_grid so CTAs are NOT co-resident), the
error-path kernels (overlap detection + covers on an invalid trace), K3
(``heteff_sort_records`` on shuffled records), K5/K6 (regions + overlap), the
interval-algebra kernels and the shard merge kernel.  ``shard`` adds 2e6-record
rank shards of C3 (overlapping streams) and C5.  Each workload's results are
compared with a second, unsanitized-equivalent run (the grid-forced and default
launches must agree bit for bit); correctness against the oracle is the tests'
job (tests/test_gpu_*.py)."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import paper_2603_26576_b200 as hb  # noqa: E402
from paper_2603_26576_b200 import _native as N  # noqa: E402
from paper_2603_26576_b200.configs import CONFIGS, scaled  # noqa: E402
from paper_2603_26576_b200.engine import analyze_device, analyze_regions, sort_records  # noqa: E402
from paper_2603_26576_b200.synth import generate  # noqa: E402


def same(a, b):
    return (a.status == b.status and a.elapsed == b.elapsed and np.array_equal(a.host_sum, b.host_sum)
            and np.array_equal(a.dev_sum, b.dev_sum) and a.host_metrics == b.host_metrics
            and a.device_metrics == b.device_metrics)


def analysis(dt, label):
    lib, ctx = N.load(), N.context(0)
    base = analyze_device(dt)
    assert base.status == N.OK, (label, base.status)
    for mode in (N.MODE_VALIDATE, N.MODE_SUMMARIZE_HOST):
        assert analyze_device(dt, mode).status == N.OK
    sd = analyze_device(dt, N.MODE_SUMMARIZE_DEVICE, elapsed=max(1, base.elapsed // 2))
    assert sd.status == N.OK
    for variant in (dt, dt.columns_only()):
        assert lib.heteff_set_grid(ctx, 148 * 4) == N.OK      # 4 waves: CTAs not co-resident
        try:
            g = analyze_device(variant)
        finally:
            lib.heteff_set_grid(ctx, 0)
        assert same(base, g), label
    print(f"analysis {label}: E={base.elapsed} ok", flush=True)


def invalid_trace():
    from paper_2603_26576_b200.model import Interval
    H, D = hb.HostState, hb.DeviceActivityKind
    recs = []
    for i in range(3000):   # overlaps across tile boundaries -> detection + covers kernels
        recs.append(hb.HostRecord(i % 3, H.USEFUL, Interval(10 * i, 10 * i + 25)))
    t = hb.Trace(host_processes=(0, 1, 2), devices=(hb.DeviceDecl(0, 0),),
                 host_records=tuple(recs),
                 device_records=(hb.DeviceRecord(0, D.KERNEL, Interval(5, 10 ** 6)),
                                 hb.DeviceRecord(0, D.MEMORY, Interval(7, 3))))
    v = hb.validate(t)
    assert v.errors
    print(f"validate invalid: {len(v.errors)} errors ok", flush=True)


def sort(n=200_000):
    g = torch.Generator(device="cuda").manual_seed(3)
    res = torch.randint(0, 97, (n,), device="cuda", dtype=torch.int32, generator=g)
    start = torch.randint(0, 1 << 40, (n,), device="cuda", dtype=torch.int64, generator=g)
    end = start + torch.randint(0, 1000, (n,), device="cuda", dtype=torch.int64, generator=g)
    kind = torch.randint(0, 2, (n,), device="cuda", dtype=torch.uint8, generator=g)
    r = sort_records(start, end, res, kind)
    key = r.res.to(torch.int64) * (1 << 41) + r.start
    assert bool((key[1:] >= key[:-1]).all())
    # start-ordered input (the res-only path)
    o = torch.argsort(start)
    r2 = sort_records(start[o], end[o], res[o], kind[o])
    assert r2.start_sorted
    print(f"sort {n}: {r.passes} passes ok", flush=True)


def regions():
    cfg = CONFIGS["c1"]
    dt = generate(cfg)
    E = analyze_device(dt).elapsed
    windows = [(i * E // 40, E - i * E // 40) for i in range(16)]
    owner = np.arange(dt.m, dtype=np.int32) // cfg.gpus_per_rank
    for v in (dt, dt.columns_only()):
        run = analyze_regions(v, windows, owner)
        assert run.status == N.OK
    print("regions c1 x16 ok", flush=True)


def intervals():
    from paper_2603_26576_b200.model import Interval
    rng = np.random.default_rng(5)
    s = rng.integers(0, 10 ** 6, 20_000)
    a = hb.flatten([Interval(int(x), int(x) + int(d)) for x, d in zip(s, rng.integers(0, 500, s.size))])
    s2 = rng.integers(0, 10 ** 6, 20_000)
    b = hb.flatten([Interval(int(x), int(x) + int(d)) for x, d in zip(s2, rng.integers(0, 500, s2.size))])
    c = hb.subtract(a, b)
    hb.intersect(c, Interval(1000, 900_000))
    hb.total_duration(c)
    hb.complement(a, Interval(0, 10 ** 6 + 600))
    print("intervals ok", flush=True)


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "small"
    torch.cuda.set_device(0)
    analysis(generate(CONFIGS["c1"]), "c1")
    for name in ("c2", "c3", "c5"):
        analysis(generate(scaled(CONFIGS[name], 4 if name != "c3" else 2)), f"{name} small shard")
    invalid_trace()
    sort(20_000 if what == "small" else 200_000)
    regions()
    intervals()
    if what in ("shard", "all"):
        for name, ranks in (("c3", 2), ("c5", 4)):
            cfg = CONFIGS[name]
            k = max(1, int(2e6 // (cfg.intervals / cfg.n_ranks)))
            analysis(generate(cfg, 0, k), f"{name}[0:{k}] ({cfg.block_intervals(0, k)} records)")
    torch.cuda.synchronize()
    print("sanitize workloads done", flush=True)


if __name__ == "__main__":
    main()
