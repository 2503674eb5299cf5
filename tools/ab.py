"""A/B of engine library builds on the same box: kernel time of the analysis launch.

    python tools/ab.py c5 lib_a.so[:csr|:col] lib_b.so[:csr|:col] ... [--reps 10]

Every library gets its own context; the trace is generated once (current build)
and the builds run interleaved, so box-to-box variance cancels.  ``:csr`` passes
the CSR offsets (17 B / interval), ``:col`` the res columns (21 B)."""
from __future__ import annotations

import argparse
import ctypes as C
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_26576_b200 import _native as N  # noqa: E402
from paper_2603_26576_b200.configs import CONFIGS  # noqa: E402
from paper_2603_26576_b200.engine import device_trace_abi  # noqa: E402
from paper_2603_26576_b200.synth import generate  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import numpy as np
    dt = generate(CONFIGS[a.config])
    arms = []
    for spec in a.libs:
        path, _, mode = spec.partition(":")
        lib = C.CDLL(str(Path(path).resolve()))
        lib.heteff_create.restype = C.c_void_p
        lib.heteff_create.argtypes = [C.c_int]
        lib.heteff_analyze.restype = C.c_int
        lib.heteff_analyze.argtypes = [C.c_void_p, C.POINTER(N.TraceABI), C.POINTER(N.Options), C.POINTER(N.Result),
                                       C.POINTER(N.Outputs), C.c_void_p]
        ctx = lib.heteff_create(0)
        t = device_trace_abi(dt if mode != "col" else dt.columns_only())
        hs = np.zeros((dt.n, 4), np.uint64)
        ds = np.zeros((dt.m, 4), np.uint64)
        out = N.Outputs(hs.ctypes.data, ds.ctypes.data, (C.c_void_p * N.NUM_LISTS)())
        arms.append((spec, lib, ctx, t, out, [], hs, ds))
    opt = N.Options(N.MODE_REPORT, 0, 0, 0)
    for rep in range(a.reps + 2):
        for spec, lib, ctx, t, out, ms, hs, ds in arms:
            res = N.Result()
            rc = lib.heteff_analyze(ctx, C.byref(t), C.byref(opt), C.byref(res), C.byref(out), None)
            assert rc == 0, (spec, rc)
            if rep >= 2:
                ms.append(res.kernel_ms)
    ref = arms[0]
    for spec, lib, ctx, t, out, ms, hs, ds in arms:
        same = np.array_equal(hs, ref[6]) and np.array_equal(ds, ref[7])
        print(f"{spec:60s} kernel median {statistics.median(ms):.4f} ms  min {min(ms):.4f}  identical={same}")


if __name__ == "__main__":
    main()
