"""Throughput of the interval-algebra C ABI (device arrays) and of Chrome-trace import,
next to CPU restatements of the reference algorithms (test infrastructure: the C oracle's
intervals.py restatement, the strict Python importer)."""
import ctypes as C
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import oracle as O  # noqa: E402
from paper_2603_26576_b200 import _native as N  # noqa: E402
from paper_2603_26576_b200 import trace_io  # noqa: E402

lib, ctx = N.load(), N.context()
rng = np.random.default_rng(1)
for n in (10**6, 10**7, 10**8):
    s = rng.integers(0, 10**12, n, dtype=np.uint64)
    e = s + rng.integers(0, 10**5, n, dtype=np.uint64)
    S = torch.from_numpy(s.view(np.int64)).cuda()
    Ee = torch.from_numpy(e.view(np.int64)).cuda()
    os_ = torch.empty_like(S)
    oe = torch.empty_like(S)
    k, bad = C.c_int64(0), C.c_int64(-1)
    for _ in range(2):
        lib.heteff_flatten(ctx, S.data_ptr(), Ee.data_ptr(), n, os_.data_ptr(), oe.data_ptr(), C.byref(k),
                           C.byref(bad), None)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        lib.heteff_flatten(ctx, S.data_ptr(), Ee.data_ptr(), n, os_.data_ptr(), oe.data_ptr(), C.byref(k),
                           C.byref(bad), None)
    torch.cuda.synchronize()
    gpu = (time.perf_counter() - t0) / 5
    line = f"flatten n={n:>10}: GPU (device arrays) {gpu * 1e3:8.2f} ms = {n / gpu / 1e9:6.2f} G intervals/s, {k.value} runs"
    if n <= 10**7:
        t0 = time.perf_counter()
        O.iv_flatten(s, e)
        cpu = time.perf_counter() - t0
        line += f" | C restatement (qsort, 1 core) {cpu * 1e3:8.1f} ms = {n / cpu / 1e6:.1f} M/s"
    print(line, flush=True)
    # subtract of two flat sets
    fa_s, fa_e = os_[: k.value].clone(), oe[: k.value].clone()
    na = k.value
    s2 = rng.integers(0, 10**12, n // 2, dtype=np.uint64)
    S2 = torch.from_numpy(s2.view(np.int64)).cuda()
    E2 = torch.from_numpy((s2 + np.uint64(5000)).view(np.int64)).cuda()
    lib.heteff_flatten(ctx, S2.data_ptr(), E2.data_ptr(), n // 2, os_.data_ptr(), oe.data_ptr(), C.byref(k),
                       C.byref(bad), None)
    fb_s, fb_e, nb = os_[: k.value].clone(), oe[: k.value].clone(), k.value
    out_s = torch.empty(na + nb, dtype=torch.int64, device="cuda")
    out_e = torch.empty_like(out_s)
    lib.heteff_subtract(ctx, fa_s.data_ptr(), fa_e.data_ptr(), na, fb_s.data_ptr(), fb_e.data_ptr(), nb,
                        out_s.data_ptr(), out_e.data_ptr(), C.byref(k), None)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        lib.heteff_subtract(ctx, fa_s.data_ptr(), fa_e.data_ptr(), na, fb_s.data_ptr(), fb_e.data_ptr(), nb,
                            out_s.data_ptr(), out_e.data_ptr(), C.byref(k), None)
    torch.cuda.synchronize()
    sub = (time.perf_counter() - t0) / 5
    print(f"subtract |a|={na} |b|={nb}: GPU {sub * 1e3:.2f} ms = {(na + nb) / sub / 1e9:.2f} G intervals/s", flush=True)

# Chrome-trace import
evs = [{"name": ("kernel_%d" % (i % 7)) if i % 3 else "cudaLaunchKernel", "cat": "cuda", "ph": "X", "ts": i,
        "dur": 3, "pid": i % 8, "tid": i % 4, "args": {"grid": [i % 5, 1, 1]}} for i in range(2_000_000)]
doc = json.dumps({"traceEvents": evs}).encode()
mapping = trace_io.read_mapping(json.dumps({"default_policy": "drop", "rules": [
    {"name_contains": "kernel", "target": "kernel", "resource": "pid"},
    {"name_contains": "cudaLaunch", "target": "offload", "resource": "pid"}]}))
t0 = time.perf_counter()
t, w = trace_io.import_mapped(doc, mapping)
t1 = time.perf_counter()
del t
import gc  # noqa: E402

gc.collect()   # the baseline below runs without the 2e6 imported records alive
small = json.dumps({"traceEvents": evs[:200_000]}).encode()
t2 = time.perf_counter()
trace_io._import_py(small, mapping)
t3 = time.perf_counter()
print(f"import_mapped: {len(evs)} events ({len(doc) / 1e6:.0f} MB) in {t1 - t0:.2f} s incl. Trace objects "
      f"= {len(evs) / (t1 - t0) / 1e6:.2f} M events/s; strict Python importer (reference algorithm) "
      f"{200_000 / (t3 - t2) / 1e6:.3f} M events/s; {os.cpu_count()} cores")
t4 = time.perf_counter()
pk, w2 = trace_io.import_mapped_packed(doc, mapping)
t5 = time.perf_counter()
from paper_2603_26576_b200 import engine as EN  # noqa: E402
EN.analyze_packed(pk, N.MODE_REPORT)
t6 = time.perf_counter()
EN.analyze_packed(pk, N.MODE_REPORT)
t7 = time.perf_counter()
print(f"import_mapped_packed: {len(evs)} events in {t5 - t4:.2f} s = {len(evs) / (t5 - t4) / 1e6:.2f} M events/s "
      f"(columns, no record objects); analyze_packed of it {(t7 - t6) * 1e3:.1f} ms (warm)")

# the drop-in API: compute_report(Trace) on a pre-built 2e6-record Trace (packing + H2D + kernel + result objects)
import paper_2603_26576_b200 as hb  # noqa: E402

host = [hb.HostRecord(j // 125000, hb.HostState.OFFLOAD if j % 3 == 1 else hb.HostState.USEFUL,
                      hb.Interval(j * 10, j * 10 + 5)) for j in range(1_000_000)]
dev = [hb.DeviceRecord(h.rank, hb.DeviceActivityKind.KERNEL if j % 5 else hb.DeviceActivityKind.MEMORY,
                       hb.Interval(h.interval.start + 2, h.interval.end + 4), None) for j, h in enumerate(host)]
t0 = time.perf_counter()
tr = hb.Trace(host_processes=tuple(range(8)), devices=tuple(hb.DeviceDecl(d, d) for d in range(8)),
              host_records=tuple(host), device_records=tuple(dev))
t1 = time.perf_counter()
hb.compute_report(tr)
t2 = time.perf_counter()
rep = hb.compute_report(tr)
t3 = time.perf_counter()
print(f"compute_report(Trace) of 2e6 records: {(t3 - t2) * 1e3:.0f} ms = {2e6 / (t3 - t2) / 1e6:.2f} M intervals/s "
      f"(Trace construction {t1 - t0:.2f} s, by the caller); E={rep.elapsed_ns}")
