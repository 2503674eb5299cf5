"""Throughput of native trace-document ingest (csrc/ingest.cpp) vs the strict
Python reader (the reference's algorithm: json.loads + per-record objects)."""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import gen as ogen  # noqa: E402
from paper_2603_26576_b200 import trace_io  # noqa: E402
from paper_2603_26576_b200.configs import CONFIGS, scaled  # noqa: E402

STATE = ("useful", "offload", "mpi")
KIND = ("kernel", "memory")


def document(cfg):
    (hs, he, hr, hk), (ds, de, dr, dk) = ogen.generate(cfg)
    parts = ['{\n  "version": 1,\n  "time_unit": "ns",\n  "hosts": [']
    hoff = np.searchsorted(hr, np.arange(cfg.n_ranks + 1))
    for r in range(cfg.n_ranks):
        a, b = hoff[r], hoff[r + 1]
        recs = ",".join(f'{{"state": "{STATE[k]}", "start": {s}, "end": {e}}}'
                        for s, e, k in zip(hs[a:b].tolist(), he[a:b].tolist(), hk[a:b].tolist()))
        parts.append(("," if r else "") + f'{{"rank": {r}, "records": [{recs}]}}')
    parts.append('],\n  "devices": [')
    doff = np.searchsorted(dr, np.arange(cfg.n_devices + 1))
    for d in range(cfg.n_devices):
        a, b = doff[d], doff[d + 1]
        recs = ",".join(f'{{"kind": "{KIND[k]}", "stream": {i % 8}, "start": {s}, "end": {e}}}'
                        for i, (s, e, k) in enumerate(zip(ds[a:b].tolist(), de[a:b].tolist(), dk[a:b].tolist())))
        parts.append(("," if d else "") + f'{{"id": {d}, "owner_rank": {d // cfg.gpus_per_rank}, "records": [{recs}]}}')
    parts.append("]\n}\n")
    return "".join(parts).encode()


def main():
    cfg = scaled(CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
    doc = document(cfg)
    n = cfg.intervals
    threads = os.cpu_count() or 1
    trace_io._native_parse(doc, threads)
    t0 = time.perf_counter(); trace_io._native_parse(doc, 1); t1 = time.perf_counter()
    trace_io._native_parse(doc, threads); t2 = time.perf_counter()
    packed, owner = trace_io.read_trace_packed(doc); t3 = time.perf_counter()
    print(f"{cfg.name}: {n} intervals, {len(doc) / 1e6:.1f} MB")
    print(f"  native parse, 1 thread : {t1 - t0:.3f} s  {n / (t1 - t0) / 1e6:8.2f} M intervals/s  "
          f"{len(doc) / (t1 - t0) / 1e9:.2f} GB/s")
    print(f"  native parse, {threads} threads: {t2 - t1:.3f} s  {n / (t2 - t1) / 1e6:8.2f} M intervals/s  "
          f"{len(doc) / (t2 - t1) / 1e9:.2f} GB/s")
    print(f"  read_trace_packed (parse + dense ids + canonical order): {t3 - t2:.3f} s  "
          f"{n / (t3 - t2) / 1e6:.2f} M intervals/s")
    k = min(n, 200_000)
    small = document(scaled(CONFIGS[cfg.name.split('[')[0]], max(1, cfg.n_ranks * k // n)))
    m = sum(1 for _ in range(small.count(b'"start"')))
    t4 = time.perf_counter(); trace_io._parse_py(small); t5 = time.perf_counter()
    print(f"  strict Python reader (reference algorithm) on {m} intervals: {t5 - t4:.3f} s  "
          f"{m / (t5 - t4) / 1e6:.3f} M intervals/s")
    try:
        import torch
        if torch.cuda.is_available():
            from paper_2603_26576_b200 import _native as N
            from paper_2603_26576_b200.engine import analyze_packed
            f = analyze_packed(packed, N.MODE_REPORT, want_lists=False)
            t6 = time.perf_counter()
            p2, _ = trace_io.read_trace_packed(doc)
            f = analyze_packed(p2, N.MODE_REPORT, want_lists=False)
            t7 = time.perf_counter()
            print(f"  file bytes -> metric tree on the GPU: {t7 - t6:.3f} s  {n / (t7 - t6) / 1e6:.2f} M intervals/s "
                  f"(status {f.status}, E={f.elapsed})")
    except Exception as e:  # noqa: BLE001
        print("  (GPU leg skipped:", e, ")")


if __name__ == "__main__":
    main()
