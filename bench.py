"""Benchmark: trace intervals/s -> full host + device TALP metric tree.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--scaling strong|weak]
                    [--impl engine|reference]

One step = one pass of the hot path (validate + summarize_host +
summarize_device + both metric trees, i.e. ``compute_report``,
/root/reference/pkg/src/heteff/metrics.py:125-154) over the config-shaped
synthetic trace.  The default workload is C5 -- 4096 ranks x 4 GPUs, 2e9
intervals, the north star's target trace -- STRONG-scaled: at N GPUs every
rank analyses a contiguous block of 4096/N ranks (and the devices they own)
of the one 2e9-interval trace and the shards are combined with one all-reduce
(E) and one all-gather (summary blocks) over NCCL.  Other configs default to
weak scaling (every rank owns a C-sized block of an N-times larger trace).

``value`` is whole-job intervals/s with the SoA already resident in HBM,
generated there by the engine's generator: ``--layout columns`` (default;
start u64, end u64, res i32, kind u8: 21 B per interval) or ``--layout csr``
(resource ids as CSR offsets: 17 B per interval -- fewer bytes, but at C5 the
analysis kernel is bound by per-tile work and the column layout is the faster
one); ``e2e`` is the same metric through the C ABI from
pinned HOST buffers, H2D copies and the result D2H inside the timed region, on
the CSR layout by default (``heteff_analyze_host_csr``: PCIe-bound, so the 17 B
layout).

``--impl reference`` times the reference's CPU path on the host cores on the
SAME config dict: the C oracle port of the reference algorithm
(``cpu_baseline.kind = "port"``, all host threads, a bounded rank-shard
sample), plus the unmodified reference package itself from baseline/_ref on
a rank shard, on 1 core and over every core (``reference_pkg``).  Rank 0
only; the arm never imports the engine package.

Without torchrun, ``--gpus N`` (N > 1) re-launches this script under
``torch.distributed.run`` with N processes on 127.0.0.1.
"""

from __future__ import annotations

import argparse
import importlib.util
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BYTES_CSR = 17               # start u64 + end u64 + kind u8 (resource ids as CSR offsets)
BYTES_COLUMNS = 21           # + res i32 when the ids travel as a column
L2_BYTES = 126 * 2 ** 20     # B200 L2
METRIC = "trace intervals/sec -> full TALP metric tree (1/2/4/8 B200, % HBM roofline)"
UNIT = "intervals/s"


def _configs():
    """paper_2603_26576_b200/configs.py loaded by path: the reference arm must not import
    the engine package (its import maps the native libraries)."""
    name = "_heteff_bench_configs"
    if name not in sys.modules:
        spec = importlib.util.spec_from_file_location(name, ROOT / "paper_2603_26576_b200" / "configs.py")
        mod = importlib.util.module_from_spec(spec)
        sys.modules[name] = mod
        spec.loader.exec_module(mod)
    return sys.modules[name]


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def _traffic():
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            return None
    return None


class Clocks:
    """nvidia-smi sampling of SM clocks / throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        try:
            rows = [ln.split(",") for ln in Path(self.path).read_text().splitlines() if ln.strip()]
        except Exception:
            rows = []
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if len(r) > 5 + i and "Active" in r[5 + i]
                          and "Not" not in r[5 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# the workload both arms name (identical config dicts)
# ---------------------------------------------------------------------------
def _scaling(args) -> str:
    return args.scaling or ("strong" if args.config == "c5" else "weak")


def _global_config(args, world: int):
    """The trace the whole job analyses: the config itself (strong) or N blocks of it (weak)."""
    M = _configs()
    c = M.CONFIGS[args.config]
    if world == 1 or _scaling(args) == "strong":
        return c
    return M.Config(f"{c.name}x{world}", c.description, c.n_ranks * world, c.gpus_per_rank,
                    c.host_records * world, c.dev_records * world, c.overlap, c.serialized_dev, c.dur_scale0,
                    c.seed, c.kernel_pct)


def _rank_block(cfg, world: int, rank: int) -> tuple[int, int]:
    return cfg.n_ranks * rank // world, cfg.n_ranks * (rank + 1) // world


def _value_csr(args) -> bool:
    """The device-resident layout `value` is measured on: resource ids as CSR offsets
    (17 B / interval) or as a res column (21 B; the default: at C5 the kernel is bound by
    per-tile work, not bytes, and the column layout is the faster of the two)."""
    return args.layout == "csr" and not args.shuffle


def _e2e_csr(args) -> bool:
    """The host-buffer layout of `e2e` (PCIe-bound: the 17 B CSR layout by default)."""
    return args.e2e_layout == "csr" and not args.shuffle


def _flush_l2(cfg, world: int, bpi: int) -> bool:
    """Inputs of one GPU that fit in L2 are flushed between timed steps."""
    return cfg.intervals // world * bpi < 2 * L2_BYTES


def _config_dict(args, cfg, world: int) -> dict:
    scaling = _scaling(args)
    bpi = BYTES_CSR if _value_csr(args) else BYTES_COLUMNS
    d = {"workload": args.config, "trace": cfg.name, "intervals": cfg.intervals, "ranks": cfg.n_ranks,
         "devices": cfg.n_devices, "parallelism": f"dp{world} (rank-sharded, {scaling} scaling)",
         "input": ("start u64 + end u64 + kind u8 + CSR offsets per rank / device (17 B/interval)" if bpi == BYTES_CSR
                   else "start u64 + end u64 + res i32 + kind u8 (21 B/interval)"),
         "l2": ("L2 flushed between timed steps (512 MB write outside the step's events): inputs fit in the 126 MB L2"
                if _flush_l2(cfg, world, bpi) else f"inputs larger than L2 ({bpi} B x intervals per GPU >> 126 MB)")}
    if args.shuffle:
        d["device_order"] = "random permutation (K3 sort inside every step)"
    if args.config == "c4" or args.regions:
        d["regions"] = (f"{args.regions if args.regions is not None else 16} nested monitoring regions per rank "
                        "(each rank its own windows over its own span; devices follow their owner)")
    return d


# ---------------------------------------------------------------------------
# reference arm: the reference's CPU path on the host cores
# ---------------------------------------------------------------------------
def _cpu_sample(cfg, target_intervals: float):
    from oracle import gen as ogen
    per_rank = cfg.intervals / cfg.n_ranks
    ranks = max(1, min(cfg.n_ranks, int(target_intervals // per_rank)))
    (h, d) = ogen.generate(cfg, 0, ranks)
    return h, d, ranks, ranks * cfg.gpus_per_rank, h[0].size + d[0].size


def _reference_pkg(cfg, args) -> dict:
    """The unmodified reference package (baseline/_ref) on a rank shard: 1 core, all cores."""
    sys.path.insert(0, str(ROOT / "baseline"))
    import ref_pkg
    why = ref_pkg.available()
    if why:
        return {"unavailable": why}
    out = {"source": "baseline/_ref/heteff (pip-installed from /root/reference/pkg, unmodified)",
           "timed": "summarize_host + summarize_device(shard, E) + host_metrics + device_metrics "
                    "(summarize.py:57-138, metrics.py:66-122); Trace construction outside the timed region",
           "extrapolated": True}
    try:
        one = ref_pkg.time_single(cfg, args.ref_pkg_intervals)
        out["one_core"] = one
        allc = ref_pkg.time_parallel(cfg, args.ref_pkg_intervals)
        out["all_cores"] = allc
        # the same shard through the C oracle port: identical E and metric floats
        from oracle import gen as ogen
        from oracle import oracle as O
        h, d = ogen.generate(cfg, 0, one["ranks"])
        r = O.analyze(h, d, one["ranks"], one["ranks"] * cfg.gpus_per_rank)
        out["port_identical"] = bool(r.elapsed == one["elapsed"] == allc["elapsed"]
                                     and list(r.host_metrics) == one["host_metrics"] == allc["host_metrics"]
                                     and list(r.device_metrics) == one["device_metrics"] == allc["device_metrics"])
    except Exception as e:   # reported, never fatal for the arm's line
        out["error"] = repr(e)
    return out


def run_reference(args, world, rank):
    if rank != 0:
        return
    from oracle import oracle as O
    cfg = _global_config(args, world)
    h, d, n, m, k = _cpu_sample(cfg, args.cpu_sample)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        O.analyze(h, d, n, m, nthreads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        r = O.analyze(h, d, n, m, nthreads=threads)
        times.append(time.perf_counter() - t0)
        assert r.status == 0
    sec = sum(times) / len(times)
    value = k / sec
    sample = (f"C oracle port (oracle/talp_oracle.c, restates summarize.py / metrics.py) on the first {n} of "
              f"{cfg.n_ranks} ranks of {cfg.name} ({k} intervals, numpy-generated by oracle/gen.py), "
              f"{threads} threads; rate extrapolated to the whole trace")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": _scaling(args),
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (the engine arm's trace, regenerated on the host)",
        "config": _config_dict(args, cfg, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if args.ref_pkg_intervals > 0:
        line["reference_pkg"] = _reference_pkg(cfg, args)
    _emit(line)


# ---------------------------------------------------------------------------
# engine arm
# ---------------------------------------------------------------------------
def run_engine(args, world, rank, local):
    import numpy as np
    import torch

    from paper_2603_26576_b200 import _native as N
    from paper_2603_26576_b200.engine import AnalysisPlan, DeviceTrace, analyze_device, analyze_host_columns
    from paper_2603_26576_b200.synth import generate

    # test plumbing: HETEFF_DIST_BACKEND=gloo puts every rank on cuda:0 and runs the
    # collectives through gloo on host copies (several ranks on the one GPU of a test box)
    gloo = os.environ.get("HETEFF_DIST_BACKEND") == "gloo"
    if gloo:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    # HETEFF_FORCE_DIST=1 runs the multi-GPU protocol even at world size 1 (exercises the
    # NCCL all-reduce / all-gather and the merge kernel on a single GPU)
    if world > 1 or os.environ.get("HETEFF_FORCE_DIST") == "1":
        import torch.distributed as tdist
        if gloo:
            from paper_2603_26576_b200.sharded import HostCollectives
            tdist.init_process_group("gloo")
            dist = HostCollectives(tdist)
        else:
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist = tdist
    cfg = _global_config(args, world)
    blocks = [_rank_block(cfg, world, r) for r in range(world)]
    r0, r1 = blocks[rank]
    dt_gen = generate(cfg, r0, r1, device=local)   # res columns + CSR offsets
    csr = _value_csr(args)
    e2e_csr = _e2e_csr(args)
    dt = dt_gen if csr else dt_gen.columns_only()
    bpi = BYTES_CSR if csr else BYTES_COLUMNS
    intervals_local = dt.host_count + dt.dev_count
    intervals_total = cfg.intervals
    stream = torch.cuda.current_stream(local)

    def sync():
        torch.cuda.synchronize(local)
        if dist:
            dist.barrier()

    from paper_2603_26576_b200.sharded import combine_shards

    n_regions = args.regions if args.regions is not None else (16 if args.config == "c4" else 0)
    windows, owner = None, None
    if n_regions:
        from paper_2603_26576_b200.engine import analyze_regions
        # per-rank regions (TALP annotates regions per process): region i of rank p is
        # [i * S_p / 40 + (p % 13), S_p - i * S_p / 40) over the rank's own span S_p --
        # nested per rank, different on every rank (tests/test_gpu_regions.py, same shape)
        f0 = analyze_device(dt, N.MODE_REPORT, stream=stream.cuda_stream, device=local)
        S = f0.host_sum[:, 3].astype(np.uint64)
        pr = np.arange(S.size, dtype=np.uint64)
        windows = np.zeros((n_regions, S.size, 2), dtype=np.uint64)
        for i in range(n_regions):
            lo = np.uint64(i) * S // np.uint64(40) + pr % np.uint64(13)
            windows[i, :, 0], windows[i, :, 1] = lo, np.maximum(lo, S - np.uint64(i) * S // np.uint64(40))
        owner = np.arange(dt.m, dtype=np.int32) // cfg.gpus_per_rank
    if args.shuffle:   # device records in random order: the step includes the K3 sort
        g = torch.Generator(device=f"cuda:{local}").manual_seed(1)
        perm = torch.randperm(dt.dev_count, device=f"cuda:{local}", generator=g)
        dt = DeviceTrace(dt.h_start, dt.h_end, dt.h_res, dt.h_kind, dt.d_start[perm], dt.d_end[perm],
                         dt.d_res[perm], dt.d_kind[perm], dt.n, dt.m)
        del perm
    region_ms = []
    # our kernels per step (regions.cu / sort.cu launch sequences)
    launches_per_step = 1 if dist is None else 3   # host pass + device pass + merge (+ NCCL all-reduce / all-gather)
    if windows is not None:
        passes = (len(windows) + 15) // 16
        launches_per_step = 1 + (2 if csr else 0) + 14 + passes * (4 + (1 if dt.n == 0 else 0))
    elif args.shuffle:
        from paper_2603_26576_b200.engine import sort_records
        probe = sort_records(dt.d_start, dt.d_end, dt.d_res, dt.d_kind, device=local)
        # failed first pass + the narrow-key sort (range_init, range, build_keys with the first
        # pass's counts; per pass three scans + downsweep, an upsweep from the second pass on;
        # the last pass writes the columns) + the re-run counted above
        launches_per_step += 1 + 2 + 5 * probe.passes
        del probe

    plan = AnalysisPlan(dt, N.MODE_REPORT, stream=stream.cuda_stream, device=local, sort_if_needed=args.shuffle)
    merge = None
    if dist:   # device-resident protocol: host pass, all-reduce E, device pass, all-gather, merge kernel
        from paper_2603_26576_b200.sharded import DeviceMerge
        n_of = [b - a for a, b in blocks]
        merge = DeviceMerge(dt, dist, local, stream.cuda_stream, n_of, [x * cfg.gpus_per_rank for x in n_of])

    def step():
        if windows is not None:   # compute_report of the trace + every region tree + overlap, one call
            run = analyze_regions(dt, windows, owner, stream=stream.cuda_stream, device=local)
            assert run.status == N.OK, run.status
            region_ms.append(run.kernel_ms)
            return None
        if merge is not None:
            return merge.step()
        return plan.run()

    for _ in range(max(args.warmup, 3)):
        f = step()
    assert f is None or f.status == N.OK, f.status
    kernel_ms = []
    region_ms.clear()
    sync()
    # inputs that fit in L2 (126 MB): flush it between timed steps (a 512 MB write, outside
    # the per-step event pairs); larger inputs stream from HBM anyway
    flush = _flush_l2(cfg, world, bpi)
    scratch = torch.empty(4 * L2_BYTES, dtype=torch.uint8, device=f"cuda:{local}") if flush else None
    with Clocks(local) as clk:
        if not flush:
            ev0 = torch.cuda.Event(enable_timing=True)
            ev1 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            for _ in range(args.steps):
                f = step()
                if f is not None and merge is None:
                    kernel_ms.append(f.kernel_ms)
            ev1.record(stream)
            sync()
            ms = ev0.elapsed_time(ev1) / args.steps
        else:
            pairs = []
            for _ in range(args.steps):
                with torch.cuda.stream(stream):
                    scratch.fill_(1)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                f = step()
                b.record(stream)
                pairs.append((a, b))
                if f is not None and merge is None:
                    kernel_ms.append(f.kernel_ms)
            sync()
            ms = sum(a.elapsed_time(b) for a, b in pairs) / args.steps
    if dist:
        t = torch.tensor([ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = intervals_total / (ms / 1e3)
    # the analysis kernel compilation the timed steps ran (before the e2e calls below); a
    # split analysis is three launches (host pass, device pass, merge)
    kernel_name = (N.load().heteff_kernel_name(N.context(local)) or b"?").decode()
    if kernel_name.startswith("split") and merge is None and windows is None and not args.shuffle:
        launches_per_step = 3

    # e2e: the same call from pinned host buffers (H2D + result D2H inside the timed region)
    def pinned(x):
        return None if x is None else torch.empty(x.shape, dtype=x.dtype, pin_memory=True).copy_(x)

    host_cols = [pinned(x) for x in (dt.h_start, dt.h_end)] + [None if e2e_csr else pinned(dt.h_res), pinned(dt.h_kind)] \
        + [pinned(x) for x in (dt.d_start, dt.d_end)] + [None if e2e_csr else pinned(dt.d_res), pinned(dt.d_kind)]
    host_dt = DeviceTrace(*host_cols, dt.n, dt.m)
    seg = (dt_gen.h_seg.cpu().numpy(), dt_gen.d_seg.cpu().numpy()) if e2e_csr else None
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    f = analyze_host_columns(host_dt, stream=stream.cuda_stream, device=local, sort_if_needed=args.shuffle, csr=seg)
    if not kernel_ms:   # region / multi-GPU steps: the one-launch analysis kernel's time on this shard
        kernel_ms.append(analyze_device(dt, N.MODE_REPORT, stream=stream.cuda_stream, device=local).kernel_ms)
    sync()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        fe = analyze_host_columns(host_dt, stream=stream.cuda_stream, device=local, sort_if_needed=args.shuffle,
                                  csr=seg)
        if dist:
            fe = combine_shards(fe, dt, dist, local, stream.cuda_stream, max(b - a for a, b in blocks),
                                max(b - a for a, b in blocks) * cfg.gpus_per_rank)
    sync()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    if dist:
        t = torch.tensor([e2e_ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    # the merged (global) E of the device-resident protocol and of the host-buffer path agree
    assert fe.status == N.OK and fe.elapsed == (merge.step().elapsed if merge is not None else f.elapsed)
    h2d = sum(int(x.numel()) * x.element_size() for x in host_cols if x is not None)
    if seg is not None:
        h2d += sum(s.nbytes for s in seg)
    d2h = 256 + (dt.n + dt.m) * 32

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    peak, peak_kind = _peaks()
    kms = statistics.mean(kernel_ms)
    algo = intervals_local * bpi + (8 * (dt.n + dt.m + 2) if csr else 0)
    achieved = algo / (kms / 1e3) / 1e9
    traffic = _traffic()
    tkey = f"{args.config}/{'csr' if csr else 'columns'}/{world}"
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": _scaling(args),
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (generated in HBM by the engine's K0 generator)",
        "config": _config_dict(args, cfg, world),
        "e2e": {"value": intervals_total / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "input": ("pinned host SoA, resource ids as CSR offsets (heteff_analyze_host_csr, 17 B/interval "
                          "in host memory; the library moves them block-compressed, ~4 B/interval over PCIe)")
                if e2e_csr else "pinned host SoA with res columns (heteff_analyze_host, 21 B/interval)"},
        "gpu_launches": args.steps * launches_per_step,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "peak_source": peak_kind,
                     "traffic": (traffic or {}).get(tkey, {}).get("bytes_per_launch") if traffic else None,
                     "kernel": "analyze_kernel, %s (tiles: compute warps x records per thread)" % kernel_name,
                     "kernel_ms": kms,
                     "algorithmic_bytes_per_launch": algo,
                     "bytes_per_interval": bpi,
                     "per_gpu_intervals": intervals_local},
        "clocks": clk.summary(),
    }
    if windows is not None:
        line["regions"] = {"windows": len(windows), "per_rank": True, "nested": True, "overlap_metric": True,
                           "ms_per_call": statistics.mean(region_ms),
                           "note": "value = compute_report + every region tree + offload/busy overlap per call; "
                                   "e2e covers the compute_report path"}
    if world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        h, d, n, m, k = _cpu_sample(cfg, args.cpu_sample)
        threads = os.cpu_count() or 1
        O.analyze(h, d, n, m, nthreads=threads)
        t0 = time.perf_counter()
        reps = 0
        while True:
            O.analyze(h, d, n, m, nthreads=threads)
            reps += 1
            if time.perf_counter() - t0 > args.cpu_seconds:
                break
        sec = (time.perf_counter() - t0) / reps
        line["cpu_baseline"] = {"value": k / sec, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": f"C oracle on the first {n} of {cfg.n_ranks} ranks of {cfg.name} "
                                          f"({k} intervals), {reps} reps, {threads} threads"}
    _emit(line)
    if dist:
        dist.destroy_process_group()


_JSON_OUT = None


def _emit(line: dict) -> None:
    """The one JSON line, on the ORIGINAL stdout (see main)."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(args_list: list[str], gpus: int) -> int:
    """--gpus N without torchrun: N processes under torch.distributed.run on 127.0.0.1."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()), *args_list]
    p = subprocess.run(cmd, stdout=subprocess.PIPE, text=True)
    for ln in p.stdout.splitlines():
        if ln.startswith("{"):
            _emit(json.loads(ln))
    return p.returncode


def main():
    global _JSON_OUT
    # stdout carries exactly one JSON line: keep a duplicate of it for that line and point
    # fd 1 at stderr, so banners native libraries print (NCCL's version line, ...) never mix in
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c5", choices=sorted(_configs().CONFIGS))
    ap.add_argument("--scaling", choices=["strong", "weak"], default=None,
                    help="strong: N GPUs split the one trace (default for c5); weak: N x the trace")
    ap.add_argument("--impl", default="engine", choices=["engine", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-sample", type=float, default=2e7)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-pkg-intervals", type=float, default=1e7,
                    help="reference arm: rank shard for the reference package itself (0: skip)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--layout", choices=["columns", "csr"], default="columns",
                    help="device-resident input of `value`: res column (21 B/interval) or CSR offsets (17 B)")
    ap.add_argument("--e2e-layout", choices=["csr", "columns"], default="csr",
                    help="host-buffer input of `e2e` (PCIe-bound): CSR offsets (17 B/interval) or res columns (21 B)")
    ap.add_argument("--regions", type=int, default=None, help="monitoring regions per step (default: 16 for c4)")
    ap.add_argument("--shuffle", action="store_true", help="device records in random order (step includes K3)")
    args = ap.parse_args()
    world, rank, local = _dist()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_spawn(sys.argv[1:], args.gpus))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_engine(args, world, rank, local)


if __name__ == "__main__":
    main()
