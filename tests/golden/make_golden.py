"""Generate the golden fixtures by running the REFERENCE package.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``heteff`` from /root/reference/pkg/src (read-only) and the
reference's own corpus generator ``random_valid_trace``
(pkg/tests/strategies.py:39-78), runs the reference's hot path on

  * every preset at scales 1, 7, 1000 (pkg/tests/test_scenario.py:226-248,
    test_acceptance.py:270-280),
  * the acceptance corpora, seeds 0x5EED01 / 0x5EED05 / 0x5EED06
    (test_acceptance.py:69-267), the last one with its stream reassignment,
  * a corpus of deliberately INVALID traces (overlaps, malformed, zero-length,
    undeclared, duplicate declarations, late device records, out-of-domain
    timestamps) for exact validation-message parity (model.py:160-230),
  * summarize_device with explicit elapsed windows (summarize.py:95-138),
  * host_metrics / device_metrics on random and extreme summaries
    (metrics.py:66-122, exact int/int division),
  * config-shaped traces from oracle/gen.py: C1 in full and rank shards of
    C2, C3, C5,
  * EXTENSIONS (not in the reference): monitoring-region
    reports = the reference's compute_report on the window-clipped trace, and
    offload-wait / device-busy overlap = the reference's flatten / intersect /
    subtract / total_duration (intervals.py:40-105) on the owner's offload
    records and the device's records,

and writes the inputs plus the reference's outputs (floats as float.hex) to
tests/golden/*.json.gz.  Nothing on the GPU box reads /root/reference.
"""

from __future__ import annotations

import gzip
import json
import random
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
sys.path.insert(0, str(ROOT))

import heteff  # noqa: E402  (the reference)
from heteff import (  # noqa: E402
    AnalysisError, DeviceActivityKind, DeviceDecl, DeviceRecord, DeviceSummary, HostRecord, HostState,
    HostSummary, Interval, InvalidTraceError, Trace, compute_report, device_metrics, host_metrics,
    summarize_device, validate,
)
from strategies import random_valid_trace  # noqa: E402  (reference corpus generator)

from oracle import gen as ogen  # noqa: E402
from paper_2603_26576_b200.configs import CONFIGS  # noqa: E402

KINDS = {"kernel": DeviceActivityKind.KERNEL, "memory": DeviceActivityKind.MEMORY}
STATES = {"useful": HostState.USEFUL, "offload": HostState.OFFLOAD, "mpi": HostState.MPI}


def fx(v):
    return None if v is None else float(v).hex()


def enc_trace(t: Trace) -> dict:
    return {
        "hp": list(t.host_processes),
        "dev": [[d.device_id, d.owner_rank] for d in t.devices],
        "h": [[r.rank, r.state.value, r.interval.start, r.interval.end] for r in t.host_records],
        "d": [[r.device_id, r.kind.value, r.interval.start, r.interval.end, r.stream] for r in t.device_records],
        "tu": t.time_unit,
    }


def dec_trace(x: dict) -> Trace:
    return Trace(
        host_processes=tuple(x["hp"]),
        devices=tuple(DeviceDecl(i, o) for i, o in x["dev"]),
        host_records=tuple(HostRecord(r, STATES[s], Interval(a, b)) for r, s, a, b in x["h"]),
        device_records=tuple(DeviceRecord(d, KINDS[k], Interval(a, b), st) for d, k, a, b, st in x["d"]),
        time_unit=x["tu"],
    )


def enc_report(t: Trace) -> dict:
    try:
        r = compute_report(t)
    except InvalidTraceError as e:
        return {"raise": "InvalidTraceError", "msg": str(e)}
    except AnalysisError as e:
        return {"raise": "AnalysisError", "msg": str(e)}
    host = None if r.host is None else [fx(getattr(r.host, f)) for f in (
        "parallel_efficiency", "mpi_parallel_efficiency", "mpi_communication_efficiency", "mpi_load_balance",
        "device_offload_efficiency")]
    dev = None if r.device is None else [fx(getattr(r.device, f)) for f in (
        "parallel_efficiency", "load_balance", "communication_efficiency", "orchestration_efficiency")]
    return {
        "E": r.elapsed_ns, "n": r.n, "m": r.m, "host": host, "device": dev,
        "hs": [[s.rank, s.d_useful, s.d_offload, s.d_mpi, s.span_end] for s in r.host_summaries],
        "ds": [[s.device_id, s.d_kernel, s.d_memory, s.d_idle] for s in r.device_summaries],
        "warnings": list(r.warnings),
    }


def enc_validate(t: Trace) -> dict:
    v = validate(t)
    return {"errors": v.errors, "warnings": v.warnings}


def case(t: Trace, tag: str) -> dict:
    return {"tag": tag, "trace": enc_trace(t), "report": enc_report(t), "validate": enc_validate(t)}


def write(name: str, obj) -> None:
    path = HERE / f"{name}.json.gz"
    with gzip.open(path, "wt", encoding="utf-8") as f:
        json.dump(obj, f, separators=(",", ":"))
    print(f"wrote {path.relative_to(ROOT)} ({path.stat().st_size} bytes)")


# ---------------------------------------------------------------------------
def presets() -> list:
    out = []
    for name in heteff.PRESET_NAMES:
        for k in (1, 7, 1000):
            out.append(case(heteff.build(heteff.preset(name, k)), f"{name}@{k}"))
    return out


def acceptance_corpora() -> list:
    out = []
    rng = random.Random(0x5EED01)
    for i in range(1000):
        out.append(case(random_valid_trace(rng), f"5EED01/{i}"))
    rng = random.Random(0x5EED05)
    for i in range(200):
        out.append(case(random_valid_trace(rng, require_devices=True), f"5EED05/{i}"))
    rng = random.Random(0x5EED06)
    for i in range(100):
        t = random_valid_trace(rng, require_devices=True)
        shuffled = Trace(
            host_processes=t.host_processes, devices=t.devices, host_records=t.host_records,
            device_records=tuple(DeviceRecord(r.device_id, r.kind, r.interval, rng.choice([None, 0, 3, 7]))
                                 for r in t.device_records))
        out.append(case(t, f"5EED06/{i}"))
        out.append(case(shuffled, f"5EED06/{i}/shuffled"))
    return out


def invalid_corpus() -> list:
    """Traces that exercise every validation message (model.py:160-230)."""
    rng = random.Random(0xBAD5EED)
    out = []
    for i in range(400):
        base = random_valid_trace(rng, max_ranks=4, max_devices=3, max_segments=8)
        hp = list(base.host_processes)
        devs = list(base.devices)
        hrec = list(base.host_records)
        drec = list(base.device_records)
        span = max((r.interval.end for r in hrec), default=100)
        for _ in range(rng.randint(1, 4)):
            what = rng.randrange(12)
            if what == 0 and hp:        # overlapping host record
                r = rng.choice(hp)
                a = rng.randint(0, span)
                hrec.append(HostRecord(r, rng.choice(list(HostState)), Interval(a, a + rng.randint(1, 50))))
            elif what == 1 and hp:      # malformed host
                r = rng.choice(hp)
                a = rng.randint(1, span + 1)
                hrec.append(HostRecord(r, rng.choice(list(HostState)), Interval(a, a - rng.randint(1, a))))
            elif what == 2 and hp:      # zero-length host
                r = rng.choice(hp)
                a = rng.randint(0, span + 20)
                hrec.append(HostRecord(r, rng.choice(list(HostState)), Interval(a, a)))
            elif what == 3:             # undeclared rank
                a = rng.randint(0, span)
                hrec.append(HostRecord(rng.choice([7, 9, -3]), HostState.MPI, Interval(a, a + 5)))
            elif what == 4:             # undeclared device
                a = rng.randint(0, span)
                drec.append(DeviceRecord(rng.choice([5, 11]), DeviceActivityKind.KERNEL, Interval(a, a + 3)))
            elif what == 5 and devs:    # malformed / zero-length device
                dd = rng.choice(devs).device_id
                a = rng.randint(1, span)
                b = a - rng.randint(0, a)
                drec.append(DeviceRecord(dd, rng.choice(list(DeviceActivityKind)), Interval(a, b)))
            elif what == 6 and devs:    # late device record (clamped)
                dd = rng.choice(devs).device_id
                a = rng.randint(span - 10 if span > 10 else 0, span + 50)
                drec.append(DeviceRecord(dd, rng.choice(list(DeviceActivityKind)), Interval(a, a + rng.randint(0, 80))))
            elif what == 7 and hp:      # duplicate rank declaration
                hp.append(rng.choice(hp))
            elif what == 8 and devs:    # duplicate device declaration / unknown owner
                d = rng.choice(devs)
                devs.append(DeviceDecl(d.device_id, d.owner_rank) if rng.random() < 0.5
                            else DeviceDecl(d.device_id + 50, 99))
            elif what == 9 and hp:      # out-of-domain timestamps (quarantined by the packer)
                r = rng.choice(hp)
                kind = rng.randrange(4)
                iv = [Interval(-5, 10), Interval(3, 2 ** 64 + 1), Interval(-5, -9), Interval(2 ** 64 + 5, 2 ** 64 + 1)][kind]
                hrec.append(HostRecord(r, HostState.USEFUL, iv))
            elif what == 10 and devs:   # out-of-domain device timestamps
                dd = rng.choice(devs).device_id
                drec.append(DeviceRecord(dd, DeviceActivityKind.MEMORY, Interval(-1, 4)))
            elif what == 11 and hp:     # exact-duplicate and touching host records
                r = rng.choice(hp)
                recs = [x for x in hrec if x.rank == r]
                if recs:
                    x = rng.choice(recs)
                    hrec.append(x)
        t = Trace(host_processes=tuple(hp), devices=tuple(devs), host_records=tuple(hrec),
                  device_records=tuple(drec))
        out.append(case(t, f"invalid/{i}"))
    # declaration-level specials
    out.append(case(Trace(), "empty"))
    out.append(case(Trace(host_processes=(0,), time_unit="us",
                          host_records=(HostRecord(0, HostState.USEFUL, Interval(0, 1)),)), "time_unit"))
    out.append(case(Trace(host_processes=(0,)), "zero_elapsed"))
    out.append(case(Trace(devices=(DeviceDecl(0),)), "zero_elapsed_dev"))
    return out


def _stage(fn):
    try:
        return {"ok": fn()}
    except InvalidTraceError as e:
        return {"raise": "InvalidTraceError", "msg": str(e)}
    except (ValueError, AnalysisError) as e:
        return {"raise": type(e).__name__, "msg": str(e)}


def quarantine_corpus() -> list:
    """Out-of-u64-domain timestamps (negative, beyond 2**64-1, non-int) on either side,
    through compute_report / validate AND the stage functions summarize_host /
    summarize_device (model.py:140-157, :217-228; summarize.py:57-138)."""
    rng = random.Random(0x0A7A)
    H, D = HostState, DeviceActivityKind
    bad = [Interval(-5, 10), Interval(3, 2 ** 64 + 5), Interval(-1, 20), Interval(2 ** 64 + 5, 2 ** 64 + 1),
           Interval(-5, -9), Interval(4, 20.5), Interval(2.5, 3), Interval(-7, 2 ** 64 + 9), Interval(30, 2 ** 70)]
    traces = []
    for iv in bad:
        for side in ("host", "device"):
            base_h = [HostRecord(0, H.USEFUL, Interval(0, 10)), HostRecord(1, H.MPI, Interval(2, 8))]
            base_d = [DeviceRecord(0, D.KERNEL, Interval(1, 6)), DeviceRecord(1, D.MEMORY, Interval(3, 9))]
            if side == "host":
                base_h.append(HostRecord(rng.choice((0, 1)), H.OFFLOAD, iv))
            else:
                base_d.append(DeviceRecord(rng.choice((0, 1)), D.KERNEL, iv))
            traces.append(Trace(host_processes=(0, 1), devices=(DeviceDecl(0, 0), DeviceDecl(1, 1)),
                                host_records=tuple(base_h), device_records=tuple(base_d)))
            # device-only twin: no late warnings (n == 0), E from the device side
            if side == "device":
                traces.append(Trace(devices=(DeviceDecl(0), DeviceDecl(1)), device_records=tuple(base_d)))
    for i in range(120):
        base = random_valid_trace(rng, max_ranks=3, max_devices=3, max_segments=6)
        hrec, drec = list(base.host_records), list(base.device_records)
        for _ in range(rng.randint(1, 3)):
            iv = rng.choice(bad + [Interval(rng.randint(0, 300), rng.randint(300, 400))])
            if base.host_processes and rng.random() < 0.5:
                hrec.append(HostRecord(rng.choice(base.host_processes), rng.choice(list(H)), iv))
            elif base.devices:
                drec.append(DeviceRecord(rng.choice(base.devices).device_id, rng.choice(list(D)), iv))
        traces.append(Trace(host_processes=base.host_processes, devices=base.devices, host_records=tuple(hrec),
                            device_records=tuple(drec)))
    out = []
    for i, t in enumerate(traces):
        c = case(t, f"quarantine/{i}")
        c["summarize_host"] = _stage(lambda: [[s.rank, s.d_useful, s.d_offload, s.d_mpi, s.span_end]
                                              for s in heteff.summarize_host(t)[0]] + [heteff.summarize_host(t)[1]])
        c["summarize_device"] = {str(E): _stage(lambda E=E: [[[s.device_id, s.d_kernel, s.d_memory, s.d_idle]
                                                                for s in heteff.summarize_device(t, E)[0]],
                                                               heteff.summarize_device(t, E)[1]])
                                 for E in (7, 50, 2 ** 64 + 3)}
        out.append(c)
    return out


def summarize_device_corpus() -> list:
    rng = random.Random(0x5D5D)
    out = []
    for i in range(300):
        t = random_valid_trace(rng, require_devices=True)
        _, E = heteff.summarize_host(t)
        for el in {max(1, E // 2), max(1, E), E + rng.randint(1, 100), rng.randint(1, 40)}:
            s, w = summarize_device(t, el)
            out.append({"tag": f"sd/{i}/{el}", "trace": enc_trace(t), "elapsed": el,
                        "ds": [[x.device_id, x.d_kernel, x.d_memory, x.d_idle] for x in s], "warnings": w})
    return out


def metrics_corpus() -> list:
    rng = random.Random(0x3E7)
    out = []
    for i in range(600):
        k = rng.randint(1, 9)
        big = i % 3 == 0
        hi = (1 << 62) if big else 10 ** 6
        hs = []
        for r in range(k):
            u = rng.randint(0, hi)
            w = rng.randint(0, hi) if rng.random() < 0.8 else 0
            p = rng.randint(0, hi) if rng.random() < 0.5 else 0
            if rng.random() < 0.1:
                u = w = 0
            hs.append(HostSummary(r, u, w, p, u + w + p))
        E = max(s.span_end for s in hs) or 1
        if rng.random() < 0.3:
            E += rng.randint(1, hi)
        E = min(E, (1 << 64) - 1) if all(s.span_end < (1 << 64) for s in hs) else E
        hm = host_metrics(hs, E)
        ds = []
        for d in range(rng.randint(1, 9)):
            kk = rng.randint(0, hi) if rng.random() < 0.85 else 0
            mm = rng.randint(0, hi) if rng.random() < 0.6 else 0
            ds.append(DeviceSummary(d, kk, mm, 0))
        Ed = max(s.d_kernel + s.d_memory for s in ds) + rng.randint(1, hi)
        dm = device_metrics(ds, Ed)
        out.append({
            "hs": [[s.rank, s.d_useful, s.d_offload, s.d_mpi, s.span_end] for s in hs], "E": E,
            "host": [fx(getattr(hm, f)) for f in ("parallel_efficiency", "mpi_parallel_efficiency",
                                                   "mpi_communication_efficiency", "mpi_load_balance",
                                                   "device_offload_efficiency")],
            "ds": [[s.device_id, s.d_kernel, s.d_memory, s.d_idle] for s in ds], "Ed": Ed,
            "device": [fx(getattr(dm, f)) for f in ("parallel_efficiency", "load_balance",
                                                     "communication_efficiency", "orchestration_efficiency")],
        })
    return out


def config_trace(cfg, r0, r1) -> Trace:
    (hs, he, hr, hk), (ds, de, dr, dk) = ogen.generate(cfg, r0, r1)
    g = cfg.gpus_per_rank
    states = [HostState.USEFUL, HostState.OFFLOAD, HostState.MPI]
    kinds = [DeviceActivityKind.KERNEL, DeviceActivityKind.MEMORY]
    hrec = [HostRecord(int(r) + r0, states[k], Interval(int(a), int(b)))
            for a, b, r, k in zip(hs.tolist(), he.tolist(), hr.tolist(), hk.tolist())]
    drec = [DeviceRecord(int(r) + r0 * g, kinds[k], Interval(int(a), int(b)))
            for a, b, r, k in zip(ds.tolist(), de.tolist(), dr.tolist(), dk.tolist())]
    return Trace(host_processes=tuple(range(r0, r1)),
                 devices=tuple(DeviceDecl(d, d // g) for d in range(r0 * g, r1 * g)),
                 host_records=tuple(hrec), device_records=tuple(drec))


def config_shards() -> list:
    out = []
    for name, r0, r1 in (("c1", 0, 4), ("c2", 0, 2), ("c2", 127, 129), ("c3", 0, 1), ("c5", 0, 2)):
        cfg = CONFIGS[name]
        t = config_trace(cfg, r0, r1)
        rep = enc_report(t)
        out.append({"config": name, "r0": r0, "r1": r1, "records": len(t.host_records) + len(t.device_records),
                    "report": rep})
        print(f"  {name}[{r0}:{r1}] {len(t.host_records) + len(t.device_records)} records, E={rep.get('E')}")
    return out


# ---------------------------------------------------------------------------
# extensions: regions (window-clipped traces) and offload / busy overlap
# ---------------------------------------------------------------------------
from heteff.intervals import flatten, intersect, subtract, total_duration  # noqa: E402


def clip_interval(iv: Interval, a: int, b: int):
    """The region clip: intersect with [a, b), shift by -a;
    zero-length records survive iff a <= start < b."""
    if iv.start == iv.end:
        return Interval(iv.start - a, iv.start - a) if a <= iv.start < b else None
    s, e = max(iv.start, a), min(iv.end, b)
    return Interval(s - a, e - a) if s < e else None


def region_trace(t: Trace, a: int, b: int) -> Trace:
    hr = [HostRecord(r.rank, r.state, c) for r in t.host_records if (c := clip_interval(r.interval, a, b))]
    dr = [DeviceRecord(r.device_id, r.kind, c, r.stream) for r in t.device_records
          if (c := clip_interval(r.interval, a, b))]
    return Trace(host_processes=t.host_processes, devices=t.devices, host_records=tuple(hr),
                 device_records=tuple(dr), time_unit=t.time_unit)


def region_overlap(rt: Trace, E: int):
    """Per declared device: |flatten(owner offload) ∩ flatten(device) ∩ [0,E)|, plus the fraction."""
    bounds = Interval(0, E)
    busy, num, den = [], 0, 0
    offload_by_rank = {}
    for s in compute_report(rt).host_summaries if rt.n else ():
        offload_by_rank[s.rank] = s.d_offload
    for d in rt.devices:
        o = d.owner_rank
        if o is None or o not in rt.host_processes:
            busy.append(0)
            continue
        A = intersect(flatten(r.interval for r in rt.host_records
                              if r.rank == o and r.state == HostState.OFFLOAD), bounds)
        B = intersect(flatten(r.interval for r in rt.device_records if r.device_id == d.device_id), bounds)
        ov = total_duration(A) - total_duration(subtract(A, B))
        busy.append(ov)
        num += ov
        den += offload_by_rank[o]
    return busy, (fx(num / den) if den else None)


def region_case(t: Trace, windows, tag: str) -> dict:
    regs = []
    for a, b in windows:
        rt = region_trace(t, a, b)
        rep = enc_report(rt)
        ov = region_overlap(rt, rep["E"]) if "E" in rep else None
        regs.append({"report": rep, "busy": ov[0] if ov else None, "frac": ov[1] if ov else None})
    return {"tag": tag, "trace": enc_trace(t), "windows": [list(w) for w in windows], "regions": regs}


def random_windows(rng: random.Random, span: int, k: int):
    out = [(0, span + 1000), (0, 1), (span + 5, span + 50)]          # whole trace, tiny, past the end
    lo, hi = 0, span + rng.randint(0, 30)
    for _ in range(k):                                                # nested
        out.append((lo, hi))
        w = hi - lo
        lo += rng.randint(0, max(1, w // 6))
        hi -= rng.randint(0, max(1, w // 6))
        if hi <= lo:
            break
    for _ in range(3):                                                # arbitrary
        a = rng.randint(0, span + 10)
        out.append((a, a + rng.randint(0, span // 2 + 1)))
    return out


def regions_corpus() -> list:
    out = []
    rng = random.Random(0x5EED40)
    for i in range(300):
        t = random_valid_trace(rng, max_ranks=4, max_devices=4, max_segments=12)
        span = max([r.interval.end for r in t.host_records] + [r.interval.end for r in t.device_records] + [1])
        out.append(region_case(t, random_windows(rng, span, 6), f"rand{i}"))
    # config-shaped shards (owners = rank of each device)
    for name, r0, r1 in (("c1", 0, 4), ("c4", 0, 1), ("c3", 0, 1)):
        cfg = CONFIGS[name]
        (hs, he, hr, hk), (ds, de, dr, dk) = ogen.generate(cfg, r0, r1)
        t = config_trace(cfg, r0, r1)
        span = int(max(he.max(), de.max()))
        nw = 4 if name == "c3" else 16
        win = [(k * span // 40, span - k * span // 40) for k in range(nw)]
        c = region_case(t, win, f"{name}[{r0}:{r1}]")
        del c["trace"]                       # regenerated by the tests from oracle/gen.py
        c.update({"config": name, "r0": r0, "r1": r1})
        out.append(c)
        print(f"  regions {name}[{r0}:{r1}] {len(t.host_records) + len(t.device_records)} records")
    return out


def region_trace_per_rank(t: Trace, wins: dict) -> Trace:
    """Per-rank region: every rank's records clipped to ITS window, every
    device's records to its owner's window; ranks without a window and devices without
    a declared owner record nothing in the region."""
    owner = {d.device_id: d.owner_rank for d in t.devices}
    hr = [HostRecord(r.rank, r.state, c) for r in t.host_records
          if r.rank in wins and (c := clip_interval(r.interval, *wins[r.rank]))]
    dr = [DeviceRecord(r.device_id, r.kind, c, r.stream) for r in t.device_records
          if owner.get(r.device_id) in wins and owner[r.device_id] in t.host_processes
          and (c := clip_interval(r.interval, *wins[owner[r.device_id]]))]
    return Trace(host_processes=t.host_processes, devices=t.devices, host_records=tuple(hr),
                 device_records=tuple(dr), time_unit=t.time_unit)


def region_case_per_rank(t: Trace, regions, tag: str) -> dict:
    regs = []
    for wins in regions:
        rt = region_trace_per_rank(t, wins)
        rep = enc_report(rt)
        ov = region_overlap(rt, rep["E"]) if "E" in rep else None
        regs.append({"report": rep, "busy": ov[0] if ov else None, "frac": ov[1] if ov else None})
    return {"tag": tag, "trace": enc_trace(t), "windows": [[[r, a, b] for r, (a, b) in w.items()] for w in regions],
            "regions": regs}


def regions_per_rank_corpus() -> list:
    """Per-rank monitoring regions: each region a window per rank (nested per rank, shifted
    between ranks, some ranks absent, empty and past-the-end windows)."""
    out = []
    rng = random.Random(0x5EED41)
    for i in range(250):
        t = random_valid_trace(rng, max_ranks=4, max_devices=4, max_segments=12)
        if rng.random() < 0.3 and t.devices:   # some devices without an owner
            t = Trace(host_processes=t.host_processes,
                      devices=tuple(DeviceDecl(d.device_id, None if rng.random() < 0.5 else d.owner_rank)
                                    for d in t.devices),
                      host_records=t.host_records, device_records=t.device_records)
        span = {}
        for r in t.host_records:
            span[r.rank] = max(span.get(r.rank, 0), r.interval.end)
        regions = []
        k = rng.randint(1, 6)
        for j in range(k):                  # nested per rank, each rank its own span
            w = {}
            for p in t.host_processes:
                sp = span.get(p, 0) + rng.randint(0, 20)
                if rng.random() < 0.1:
                    continue                # rank without this region
                lo = j * sp // (2 * k + 1) + rng.randint(0, 3)
                w[p] = (lo, max(lo, sp - j * sp // (2 * k + 1)))
            regions.append(w)
        for _ in range(2):                  # arbitrary per-rank windows
            w = {}
            for p in t.host_processes:
                a = rng.randint(0, span.get(p, 0) + 10)
                w[p] = (a, a + rng.randint(0, span.get(p, 0) // 2 + 2))
            regions.append(w)
        regions.append({p: (span.get(p, 0) + 5, span.get(p, 0) + 50) for p in t.host_processes})   # past the end
        out.append(region_case_per_rank(t, regions, f"prank{i}"))
    for name, r0, r1 in (("c1", 0, 4), ("c4", 0, 2), ("c3", 0, 1)):
        cfg = CONFIGS[name]
        (hs, he, hr, hk), (ds, de, dr, dk) = ogen.generate(cfg, r0, r1)
        t = config_trace(cfg, r0, r1)
        spans = {r0 + p: int(he[hr == p].max()) for p in range(r1 - r0)}
        nw = 4 if name == "c3" else 16
        regions = [{p: (k * sp // 40 + 7 * (p - r0), sp - k * sp // 40) for p, sp in spans.items()} for k in range(nw)]
        c = region_case_per_rank(t, regions, f"{name}[{r0}:{r1}]")
        del c["trace"]
        c.update({"config": name, "r0": r0, "r1": r1})
        out.append(c)
        print(f"  per-rank regions {name}[{r0}:{r1}] {len(t.host_records) + len(t.device_records)} records")
    return out


# ---------------------------------------------------------------------------
# interval algebra (intervals.py:40-105), acceptance criterion 2 shapes
# ---------------------------------------------------------------------------
def _enc_flat(f):
    return [[iv.start, iv.end] for iv in f]


def intervals_corpus() -> list:
    from heteff.intervals import complement

    rng = random.Random(0x5EED02)
    out = []
    for i in range(400):
        k = rng.randint(0, 40)
        hi = rng.choice([30, 200, 10_000])
        raw_a = []
        for _ in range(k):
            s = rng.randint(0, hi)
            raw_a.append((s, s + rng.choice([0, 0, 1, 2, rng.randint(0, hi // 3 + 1)])))
        raw_b = []
        for _ in range(rng.randint(0, 40)):
            s = rng.randint(0, hi)
            raw_b.append((s, s + rng.randint(0, hi // 4 + 1)))
        case = {"a": raw_a, "b": raw_b}
        if i % 25 == 7 and raw_a:                       # malformed input
            j = rng.randrange(len(raw_a))
            raw_a[j] = (raw_a[j][0] + 5, raw_a[j][0])
            case["a"] = raw_a
            try:
                flatten(Interval(s, e) for s, e in raw_a)
                case["flat_a"] = None
            except ValueError as exc:
                case["error"] = str(exc)
            out.append(case)
            continue
        fa = flatten(Interval(s, e) for s, e in raw_a)
        fb = flatten(Interval(s, e) for s, e in raw_b)
        b0 = rng.randint(0, hi)
        bounds = (b0, b0 + rng.randint(0, hi))
        case.update({
            "flat_a": _enc_flat(fa), "flat_b": _enc_flat(fb), "sub": _enc_flat(subtract(fa, fb)),
            "bounds": list(bounds), "comp": _enc_flat(complement(fa, Interval(*bounds))),
            "inter": _enc_flat(intersect(fa, Interval(*bounds))), "total": total_duration(fa),
        })
        out.append(case)
    return out


# ---------------------------------------------------------------------------
# native trace documents (trace_io.py:96-193, docs/formats.md:9-85)
# ---------------------------------------------------------------------------
def trace_docs_corpus() -> list:
    from heteff import TraceFormatError, read_trace, write_trace

    out = []
    rng = random.Random(0x5EED08)
    for i in range(150):                                   # acceptance criterion 8 shapes
        t = random_valid_trace(rng, max_ranks=4, max_devices=3, max_segments=8)
        doc = write_trace(t).decode()
        out.append({"tag": f"rt{i}", "doc": doc, "trace": enc_trace(read_trace(doc))})
    for name in ("usecase1", "usecase3", "usecase7b"):
        doc = write_trace(heteff.build(heteff.preset(name, 7))).decode()
        out.append({"tag": name, "doc": doc, "trace": enc_trace(read_trace(doc))})
    base = {"version": 1, "time_unit": "ns",
            "hosts": [{"rank": 3, "records": [{"state": "mpi", "start": 0, "end": 5},
                                              {"state": "useful", "start": 5, "end": 9}]},
                      {"rank": 1, "records": []}],
            "devices": [{"id": 7, "owner_rank": 3, "records": [{"kind": "kernel", "stream": 2, "start": 1, "end": 4},
                                                               {"kind": "memory", "start": 0, "end": 2}]},
                        {"id": 2, "owner_rank": None, "records": []}]}
    variants = {
        "compact": json.dumps(base, separators=(",", ":")),
        "reordered_keys": json.dumps({"devices": base["devices"], "hosts": base["hosts"], "time_unit": "ns",
                                      "version": 1}),
        "spaces": json.dumps(base, indent=5).replace(":", " : "),
        "big_u64": json.dumps({**base, "hosts": [{"rank": 0, "records": [
            {"state": "offload", "start": 2**64 - 5, "end": 2**64 - 1}]}]}),
        "beyond_u64": json.dumps({**base, "hosts": [{"rank": 0, "records": [
            {"state": "offload", "start": 1, "end": 2**64 + 7}]}]}),
        "dup_key": '{"version": 1, "version": 1, "time_unit": "ns", "hosts": [], "devices": []}',
        "escaped_key": '{"version": 1, "time_\u0075nit": "ns", "hosts": [], "devices": []}',
        "float_version": '{"version": 1.0, "time_unit": "ns", "hosts": [], "devices": []}',
        "bool_version": '{"version": true, "time_unit": "ns", "hosts": [], "devices": []}',
        "not_json": '{"version": 1,, }',
        "not_object": '[1, 2]',
        "bad_version": json.dumps({**base, "version": 2}),
        "bad_unit": json.dumps({**base, "time_unit": "us"}),
        "missing_hosts": json.dumps({k: v for k, v in base.items() if k != "hosts"}),
        "extra_top": json.dumps({**base, "zeta": 1}),
        "hosts_not_list": json.dumps({**base, "hosts": {}}),
        "neg_start": json.dumps({**base, "hosts": [{"rank": 0, "records": [{"state": "mpi", "start": -1, "end": 3}]}]}),
        "float_end": json.dumps({**base, "hosts": [{"rank": 0, "records": [{"state": "mpi", "start": 1, "end": 3.5}]}]}),
        "bool_rank": json.dumps({**base, "hosts": [{"rank": True, "records": []}]}),
        "bad_state": json.dumps({**base, "hosts": [{"rank": 0, "records": [{"state": "MPI", "start": 1, "end": 3}]}]}),
        "bad_kind": json.dumps({**base, "devices": [{"id": 0, "records": [{"kind": "idle", "start": 1, "end": 3}]}]}),
        "extra_rec": json.dumps({**base, "hosts": [{"rank": 0, "records": [
            {"state": "mpi", "start": 1, "end": 3, "x": 0}]}]}),
        "missing_end": json.dumps({**base, "devices": [{"id": 0, "records": [{"kind": "kernel", "start": 1}]}]}),
        "neg_stream": json.dumps({**base, "devices": [{"id": 0, "records": [
            {"kind": "kernel", "stream": -2, "start": 1, "end": 3}]}]}),
        "neg_owner": json.dumps({**base, "devices": [{"id": 0, "owner_rank": -1, "records": []}]}),
        "rec_not_obj": json.dumps({**base, "hosts": [{"rank": 0, "records": [5]}]}),
        "entry_not_obj": json.dumps({**base, "devices": [7]}),
        "trailing": json.dumps(base) + " x",
        "empty": "",
        "nan": '{"version": 1, "time_unit": "ns", "hosts": [{"rank": NaN, "records": []}], "devices": []}',
        "string_brace": json.dumps({**base, "hosts": [{"rank": 0, "records": [{"state": "mp}i", "start": 1, "end": 3}]}]}),
        "null_stream": json.dumps({**base, "devices": [{"id": 0, "records": [
            {"kind": "kernel", "stream": None, "start": 1, "end": 3}]}]}),
    }
    for tag, doc in variants.items():
        try:
            t = read_trace(doc)
            out.append({"tag": tag, "doc": doc, "trace": enc_trace(t)})
        except TraceFormatError as e:
            out.append({"tag": tag, "doc": doc, "error": str(e)})
    return out


# ---------------------------------------------------------------------------
# Chrome-trace import with mapping rules (trace_io.py:196-342)
# ---------------------------------------------------------------------------
def import_corpus() -> list:
    from heteff import MappingError, TraceFormatError, import_mapped, read_mapping

    rng = random.Random(0x5EED09)
    names = ["cudaLaunchKernel", "my_kernel<128>", "Memcpy HtoD", "MPI_Allreduce", "compute", "cudaMemset",
             "MPI_Wait", "kernel_b", "idle", "cudaDeviceSynchronize", "Ω-kernel"]
    cats = ["cuda", "mpi", "cpu", "", "gpu"]
    maps = [
        {"default_policy": "drop", "rules": [
            {"name_contains": "Memcpy", "target": "memory", "resource": "pid"},
            {"name_contains": "kernel", "target": "kernel", "resource": "pid"},
            {"name_contains": "cudaLaunch", "target": "offload", "resource": "tid"},
            {"name_equals": "compute", "target": "useful", "resource": 0},
            {"category_equals": "mpi", "target": "mpi", "resource": "pid"}]},
        {"default_policy": "error", "rules": [
            {"category_contains": "", "target": "useful", "resource": "tid"}]},
        {"default_policy": "error", "rules": [
            {"name_contains": "MPI", "target": "mpi", "resource": 3}]},
    ]
    out = []
    for i in range(120):
        evs = []
        for _ in range(rng.randint(0, 40)):
            ev = {"name": rng.choice(names), "ph": rng.choice(["X", "X", "X", "B", "M"]),
                  "ts": rng.choice([rng.randint(0, 10**6), float(rng.randint(0, 10**5))]),
                  "dur": rng.randint(0, 5000), "pid": rng.randint(0, 3), "tid": rng.randint(0, 5)}
            if rng.random() < 0.7:
                ev["cat"] = rng.choice(cats)
            if rng.random() < 0.3:
                ev["args"] = {"x": [1, {"y": "}]"}], "s": "a\"b"}
            evs.append(ev)
        doc = json.dumps({"traceEvents": evs, "displayTimeUnit": "ms"} if i % 2 else evs)
        mp = json.dumps(maps[i % len(maps)])
        case = {"tag": f"imp{i}", "doc": doc, "map": mp}
        try:
            t, w = import_mapped(doc, read_mapping(mp))
            case.update({"trace": enc_trace(t), "warnings": w})
        except (TraceFormatError, MappingError) as e:
            case.update({"error": type(e).__name__, "msg": str(e)})
        out.append(case)
    m0 = json.dumps(maps[0])
    odd = {
        "frac_ts": [{"name": "compute", "ph": "X", "ts": 1.5, "dur": 1}],
        "neg_dur": [{"name": "compute", "ph": "X", "ts": 1, "dur": -1}],
        "no_dur": [{"name": "compute", "ph": "X", "ts": 1}],
        "bool_ts": [{"name": "compute", "ph": "X", "ts": True, "dur": 1}],
        "str_ts": [{"name": "compute", "ph": "X", "ts": "1", "dur": 1}],
        "name_int": [{"name": 5, "ph": "X", "ts": 1, "dur": 1}],
        "cat_int": [{"name": "compute", "cat": 3, "ph": "X", "ts": 1, "dur": 1}],
        "pid_missing": [{"name": "my_kernel", "ph": "X", "ts": 1, "dur": 1}],
        "pid_neg": [{"name": "my_kernel", "ph": "X", "ts": 1, "dur": 1, "pid": -4}],
        "pid_float": [{"name": "my_kernel", "ph": "X", "ts": 1, "dur": 1, "pid": 2.0}],
        "not_x_bad": [{"name": 5, "ph": "B", "ts": "q"}, {"name": "compute", "ph": "X", "ts": 2, "dur": 3}],
        "events_not_list": {"traceEvents": 7},
        "escaped_name": [{"name": "my\u005fkernel", "ph": "X", "ts": 1, "dur": 1, "pid": 1}],
        "big_ts": [{"name": "compute", "ph": "X", "ts": 2**62, "dur": 1}],
        "exp_ts": [{"name": "compute", "ph": "X", "ts": 1.5e3, "dur": 2e0}],
        "dup_name": '[{"name": "x", "name": "compute", "ph": "X", "ts": 1, "dur": 1}]',
    }
    for tag, evs in odd.items():
        doc = evs if isinstance(evs, str) else json.dumps(evs)
        if tag == "escaped_name":
            doc = doc.replace("\\\\u005f", "\\u005f")
        case = {"tag": tag, "doc": doc, "map": m0}
        try:
            t, w = import_mapped(doc, read_mapping(m0))
            case.update({"trace": enc_trace(t), "warnings": w})
        except (TraceFormatError, MappingError) as e:
            case.update({"error": type(e).__name__, "msg": str(e)})
        out.append(case)
    for tag, mp in {"no_rules": {"default_policy": "drop", "rules": []},
                    "two_keys": {"default_policy": "drop", "rules": [
                        {"name_contains": "a", "name_equals": "b", "target": "mpi", "resource": 0}]},
                    "bad_policy": {"default_policy": "warn", "rules": []},
                    "bad_resource": {"default_policy": "drop", "rules": [
                        {"name_contains": "a", "target": "mpi", "resource": "rank"}]},
                    "neg_resource": {"default_policy": "drop", "rules": [
                        {"name_contains": "a", "target": "mpi", "resource": -1}]},
                    "bad_target": {"default_policy": "drop", "rules": [
                        {"name_contains": "a", "target": "idle", "resource": 0}]}}.items():
        try:
            read_mapping(json.dumps(mp))
            out.append({"tag": tag, "map": json.dumps(mp), "map_ok": True})
        except TraceFormatError as e:
            out.append({"tag": tag, "map": json.dumps(mp), "error": "TraceFormatError", "msg": str(e)})
    return out


# ---------------------------------------------------------------------------
# rendering + CLI (report.py:35-138, cli.py:80-100)
# ---------------------------------------------------------------------------
def render_corpus() -> list:
    from heteff import RenderOptions, render_json, render_text, write_trace

    out = []
    traces = [(f"{n}x{k}", heteff.build(heteff.preset(n, k))) for n in ("usecase1", "usecase3", "usecase7b")
              for k in (1, 1000)]
    rng = random.Random(0x5EED0A)
    traces += [(f"rand{i}", random_valid_trace(rng)) for i in range(12)]
    traces.append(("late", Trace(host_processes=(0,), devices=(DeviceDecl(0, 0),),
                                 host_records=(HostRecord(0, HostState.OFFLOAD, Interval(0, 100)),),
                                 device_records=(DeviceRecord(0, DeviceActivityKind.KERNEL, Interval(90, 120)),
                                                 DeviceRecord(0, DeviceActivityKind.MEMORY, Interval(95, 95))))))
    for tag, t in traces:
        r = compute_report(t)
        renders = {}
        for prec in (0, 2, 6):
            for raw in (False, True):
                for asc in (False, True):
                    o = RenderOptions("text", prec, raw, asc)
                    renders[f"text-{prec}-{int(raw)}-{int(asc)}"] = render_text(r, o)
            renders[f"json-{prec}"] = render_json(r, RenderOptions("json", prec, False, False)).decode()
        renders["json-raw"] = render_json(r, RenderOptions("json", 2, True, False)).decode()
        out.append({"tag": tag, "doc": write_trace(t).decode(), "renders": renders})
    return out


def main() -> None:
    only = sys.argv[sys.argv.index("--only") + 1].split(",") if "--only" in sys.argv else None
    jobs = {"presets": presets, "acceptance": acceptance_corpora, "invalid": invalid_corpus, "quarantine": quarantine_corpus,
            "summarize_device": summarize_device_corpus, "metrics": metrics_corpus,
            "config_shards": config_shards, "regions": regions_corpus, "regions_per_rank": regions_per_rank_corpus, "intervals": intervals_corpus,
            "trace_docs": trace_docs_corpus, "imports": import_corpus, "renders": render_corpus}
    for name, fn in jobs.items():
        if only is None or name in only:
            write(name, fn())


if __name__ == "__main__":
    main()
