"""Randomized engine-vs-oracle stress run (test infrastructure): random trace shapes --
counts around tile boundaries, time ranges crossing 2^32 or near U64_MAX, overlapping
streams, zero-length / malformed records, empty resources -- through the engine's
columnar path in REPORT / VALIDATE / SUMMARIZE_DEVICE mode against the C oracle -- both
compilations of the analysis kernel (res columns, and CSR offsets when the ids allow).
Usage: python tools/stress.py SECONDS [SEED]"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from oracle import oracle as O  # noqa: E402
from paper_2603_26576_b200 import _native as N  # noqa: E402
from paper_2603_26576_b200.engine import analyze_packed  # noqa: E402
from paper_2603_26576_b200.packing import PackedTrace, RecordColumns  # noqa: E402

TILE = 15 * 32 * 11


def canonical(s, e, r, k, host):
    kr = np.array([2, 1, 0], dtype=np.uint8)[k] if host else k
    o = np.lexsort((kr, e, s, r))
    return s[o], e[o], r[o], k[o]


def side(rng, n_res, host):
    if n_res == 0:
        return np.zeros(0, np.uint64), np.zeros(0, np.uint64), np.zeros(0, np.int32), np.zeros(0, np.uint8)
    pick = rng.integers(0, 4)
    if pick == 0:
        counts = rng.integers(0, 6, n_res)
    elif pick == 1:
        counts = rng.choice([TILE - 1, TILE, TILE + 1, 2 * TILE - 3, 1, 0, 31, 32, 33], n_res)
    else:
        counts = rng.integers(0, 3 * TILE, n_res)
    r = np.repeat(np.arange(n_res, dtype=np.int32), counts)
    k = r.size
    scale = rng.choice([10 ** 3, 10 ** 6, 2 ** 33, 2 ** 40])
    base = rng.choice([0, 2 ** 32 - 10 ** 6, 2 ** 63, 2 ** 64 - 2 ** 41])
    if host:   # a serialized chain per rank (valid), with a few anomalies
        g = rng.integers(0, 20, k).astype(np.uint64)
        d = rng.integers(1, 200, k).astype(np.uint64)
        cs = np.cumsum(g + d)
        offs = np.concatenate([[0], np.cumsum(counts)])
        b0 = np.zeros(n_res, np.uint64)
        nz = offs[:-1] > 0
        b0[nz] = cs[offs[:-1][nz] - 1]
        s = cs - np.repeat(b0, counts) - d
        e = s + d
    else:
        s = rng.integers(0, max(2, int(scale)), k, dtype=np.uint64)
        e = s + rng.integers(1, max(2, int(scale) // max(1, k // max(n_res, 1)) * int(rng.choice([1, 4, 16]))), k,
                             dtype=np.uint64)
    s = s + np.uint64(base)
    e = np.minimum(e + np.uint64(base), np.uint64(2 ** 64 - 1))
    if rng.random() < 0.3 and k:
        z = rng.random(k) < 0.01
        e[z] = s[z]
    if rng.random() < 0.1 and k:
        bad = rng.random(k) < 0.001
        e[bad] = s[bad] - np.minimum(s[bad], np.uint64(3))
    kind = rng.integers(0, 3 if host else 2, k, dtype=np.uint8)
    return canonical(s, e, r, kind, host)


def one(rng):
    n, m = int(rng.integers(0, 6)), int(rng.integers(0, 6))
    if n == 0 and m == 0:
        m = 1
    h, d = side(rng, n, True), side(rng, m, False)
    packed = PackedTrace(RecordColumns(*h), RecordColumns(*d), list(range(n)), list(range(m)),
                         np.arange(n, dtype=np.int32), np.arange(m, dtype=np.int32), n, m, n, m)
    modes = [(N.MODE_REPORT, 0), (N.MODE_VALIDATE, 0)]
    if m:
        top = int(max([int(d[1].max()) if d[1].size else 1, int(h[1].max()) if h[1].size else 1]))
        modes.append((N.MODE_SUMMARIZE_DEVICE, max(1, int(rng.random() * top))))
    for mode, el in modes:
        got = analyze_packed(packed, mode, el, want_lists=True, capacity=1 << 18)
        ref = O.analyze(h, d, n, m, mode=mode, elapsed=el, cap=1 << 18)
        assert got.status == ref.status, (mode, got.status, ref.status)
        lists = (0, 1, 2, 4, 5, 6, 7) if mode != N.MODE_SUMMARIZE_DEVICE else (0, 1, 2, 4, 5, 6)
        assert [got.counts[c] for c in lists + (3,)] == [ref.counts[c] for c in lists + (3,)], mode
        if ref.status == 0 and mode != N.MODE_VALIDATE:   # the oracle's validate mode computes no E
            assert got.elapsed == ref.elapsed, (mode, got.elapsed, ref.elapsed)
            assert np.array_equal(got.host_sum, ref.host_sum) and np.array_equal(got.dev_sum, ref.dev_sum), mode
            assert got.host_metrics == ref.host_metrics and got.device_metrics == ref.device_metrics, mode
    # the CSR compilation of the analysis kernel on the same columns (res ids as offsets),
    # when every id is a declared dense id (offsets cannot express the others)
    if (h[2].size == 0 or int(h[2].max()) < n) and (d[2].size == 0 or int(d[2].max()) < m):
        import torch

        from paper_2603_26576_b200.engine import DeviceTrace, analyze_device

        def cu(x):
            x = np.ascontiguousarray(x)
            return torch.from_numpy(x.view(np.int64) if x.dtype == np.uint64 else x).cuda()
        dt = DeviceTrace(*(cu(x) for x in (*h, *d)), n, m).with_csr()
        for mode, el in modes:
            got = analyze_device(dt, mode, el)
            ref = O.analyze(h, d, n, m, mode=mode, elapsed=el, cap=1 << 18)
            assert got.status == ref.status, ("csr", mode, got.status, ref.status)
            lists = (0, 1, 2, 4, 5, 6, 7) if mode != N.MODE_SUMMARIZE_DEVICE else (0, 1, 2, 4, 5, 6)
            assert [got.counts[c] for c in lists + (3,)] == [ref.counts[c] for c in lists + (3,)], ("csr", mode)
            if ref.status == 0 and mode != N.MODE_VALIDATE:
                assert got.elapsed == ref.elapsed, ("csr", mode)
                assert np.array_equal(got.host_sum, ref.host_sum) and np.array_equal(got.dev_sum, ref.dev_sum)
                assert got.host_metrics == ref.host_metrics and got.device_metrics == ref.device_metrics
    return h[0].size + d[0].size


def one_regions(rng):
    """K5/K6: random windows (whole range, empty, beyond the span, random) and random
    owners (some devices unowned) against the oracle's composition restatement."""
    import torch

    from paper_2603_26576_b200.engine import DeviceTrace, analyze_regions

    n, m = int(rng.integers(0, 5)), int(rng.integers(1, 5))
    h, d = side(rng, n, True), side(rng, m, False)
    owner = np.array([int(rng.integers(-1, n)) if n else -1 for _ in range(m)], np.int32)
    top = int(max([int(x[1].max()) for x in (h, d) if x[1].size] + [1]))
    lo = int(min([int(x[0].min()) for x in (h, d) if x[0].size] + [0]))
    win = [(0, 2 ** 64 - 1), (lo, lo), (top + 5, top + 50)]
    for _ in range(int(rng.integers(1, 20))):
        a = lo + int(rng.random() * max(1, top - lo))
        win.append((a, min(2 ** 64 - 1, a + 1 + int(rng.random() * max(1, top - a)))))
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64) if a.dtype == np.uint64  # noqa: E731
                                    else np.ascontiguousarray(a)).cuda()
    dt = DeviceTrace(*(cu(x) for x in (*h, *d)), n, m)
    run = analyze_regions(dt, win, owner)
    whole = O.analyze(h, d, n, m, mode=N.MODE_REPORT, cap=0)
    if whole.status == N.INVALID_TRACE:   # invalid traces fail the call as a whole
        assert run.status == N.INVALID_TRACE, run.status
        return h[0].size + d[0].size
    assert run.status == N.OK, run.status   # per-region analysis errors are the regions' own
    ref = O.regions(h, d, n, m, win, owner)
    for j in range(len(win)):
        g = run.regions[j]
        assert g.status == int(ref.status[j]), ("status", j)
        if g.status != N.OK:
            continue
        assert g.elapsed == int(ref.elapsed[j]), ("E", j)
        assert np.array_equal(g.host_sum, ref.host_sum[j]) and np.array_equal(g.dev_sum, ref.dev_sum[j]), ("sums", j)
        assert np.array_equal(g.offload_busy, ref.busy[j]), ("busy", j)
        assert g.host_metrics == ref.host_metrics[j] and g.device_metrics == ref.device_metrics[j], ("metrics", j)
        assert g.offload_busy_fraction == ref.busy_frac[j], ("frac", j)
    return h[0].size + d[0].size


def _iv_cols(rng, n):
    scale = int(rng.choice([10, 10 ** 3, 10 ** 6, 2 ** 40]))
    base = np.uint64(int(rng.choice([0, 2 ** 32 - 500, 2 ** 63, 2 ** 64 - 2 ** 41])))
    st = base + rng.integers(0, scale, n, dtype=np.uint64)
    d = rng.integers(0, max(2, scale // max(1, n) * int(rng.choice([1, 3, 30]))), n, dtype=np.uint64)
    return st, st + np.minimum(d, np.uint64(2 ** 64 - 1) - st)   # ends never wrap past u64


def one_intervals(rng):
    """flatten / subtract / intersect / total_duration through the C ABI on device arrays
    against the oracle's restatement of intervals.py:40-105."""
    import ctypes as C

    import torch

    lib, ctx = N.load(), N.context()
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()   # noqa: E731
    u64 = lambda t: t.cpu().numpy().view(np.uint64)   # noqa: E731
    n = int(rng.choice([0, 1, 2, 31, 33, 1000, 3 * TILE + 7, int(rng.integers(1, 300_000))]))
    s, e = _iv_cols(rng, n)
    if n and rng.random() < 0.1:
        j = int(rng.integers(0, n))
        s[j], e[j] = e[j] + np.uint64(1), s[j]   # malformed
    S, E = cu(s), cu(e)
    os_, oe = torch.empty(max(n, 1), dtype=torch.int64, device="cuda"), torch.empty(max(n, 1), dtype=torch.int64,
                                                                                    device="cuda")
    k, bad = C.c_int64(0), C.c_int64(-1)
    rc = lib.heteff_flatten(ctx, S.data_ptr() if n else None, E.data_ptr() if n else None, n, os_.data_ptr(),
                            oe.data_ptr(), C.byref(k), C.byref(bad), None)
    try:
        rs, re_ = O.iv_flatten(s, e)
    except ValueError as x:
        assert rc == N.VALUE_ERROR and bad.value == int(x.args[0]), (rc, bad.value, x.args)
        return n
    assert rc == N.OK and np.array_equal(u64(os_[:k.value]), rs) and np.array_equal(u64(oe[:k.value]), re_), "flatten"
    a_s, a_e = rs, re_
    t, u = _iv_cols(rng, int(rng.integers(0, max(2, n))))
    b_s, b_e = O.iv_flatten(t, u)
    out_s = torch.empty(len(a_s) + len(b_s) + 1, dtype=torch.int64, device="cuda")
    out_e = torch.empty_like(out_s)
    A_s, A_e, B_s, B_e = cu(a_s), cu(a_e), cu(b_s), cu(b_e)
    p_ = lambda x, m: x.data_ptr() if m else None   # noqa: E731
    rc = lib.heteff_subtract(ctx, p_(A_s, len(a_s)), p_(A_e, len(a_s)), len(a_s), p_(B_s, len(b_s)), p_(B_e, len(b_s)),
                             len(b_s), out_s.data_ptr(), out_e.data_ptr(), C.byref(k), None)
    ws, we = O.iv_subtract(a_s, a_e, b_s, b_e)
    assert rc == N.OK and np.array_equal(u64(out_s[:k.value]), ws) and np.array_equal(u64(out_e[:k.value]), we), "sub"
    if len(a_s):
        lo = int(a_s[0]) + int(rng.random() * max(1, int(a_e[-1]) - int(a_s[0])))
        hi = min(2 ** 64 - 1, lo + int(rng.random() * max(1, int(a_e[-1]) - lo + 10)))
        rc = lib.heteff_intersect(ctx, A_s.data_ptr(), A_e.data_ptr(), len(a_s), lo, hi, out_s.data_ptr(),
                                  out_e.data_ptr(), C.byref(k), None)
        xs, xe = O.iv_intersect(a_s, a_e, lo, hi)
        assert rc == N.OK and np.array_equal(u64(out_s[:k.value]), xs) and np.array_equal(u64(out_e[:k.value]), xe), \
            "intersect"
        tot = (C.c_uint64 * 2)()
        rc = lib.heteff_total_duration(ctx, A_s.data_ptr(), A_e.data_ptr(), len(a_s), C.cast(tot, C.c_void_p), None)
        assert rc == N.OK and int(tot[0]) + (int(tot[1]) << 64) == O.iv_total(a_s, a_e), "total"
    return n


def one_sort(rng):
    """K3 on random columns (resource counts, start ranges, durations that do / do not fit
    the key's spare bits, malformed records, kinds > 3) against a stable lexsort."""
    import torch

    from paper_2603_26576_b200.engine import sort_records

    n = int(rng.choice([1, 2, 31, 33, 5631, 5632, 5633, int(rng.integers(1, 400_000))]))
    ids = int(rng.choice([1, 2, 7, 1000, 70_000]))
    span = int(rng.choice([1, 100, 10 ** 6, 2 ** 40, 2 ** 62]))
    s = rng.integers(0, span, n, dtype=np.uint64) if span > 1 else np.zeros(n, np.uint64)
    if rng.random() < 0.3:
        s = np.sort(s)   # start-ordered input: the res-only path
    d = rng.integers(0, int(rng.choice([2, 1000, 2 ** 30, 2 ** 50])), n, dtype=np.uint64)
    e = s + d
    if rng.random() < 0.1:
        e[int(rng.integers(0, n))] = s[0] - np.minimum(s[0], np.uint64(1))   # a malformed record
    r = rng.integers(0, ids, n, dtype=np.int32) - (int(rng.integers(0, 3)) if rng.random() < 0.2 else 0)
    k = rng.integers(0, 256 if rng.random() < 0.05 else 2, n, dtype=np.int32).astype(np.uint8)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64) if a.dtype == np.uint64  # noqa: E731
                                    else np.ascontiguousarray(a)).cuda()
    got = sort_records(cu(s), cu(e), cu(r), cu(k))
    perm = np.lexsort((s, r.astype(np.int64)))
    assert np.array_equal(got.perm.cpu().numpy(), perm), "perm"
    assert np.array_equal(got.start.cpu().numpy().view(np.uint64), s[perm]), "start"
    assert np.array_equal(got.end.cpu().numpy().view(np.uint64), e[perm]), "end"
    assert np.array_equal(got.res.cpu().numpy(), r[perm]) and np.array_equal(got.kind.cpu().numpy(), k[perm]), "res/kind"
    return n


def main():
    seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 60.0
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    global one
    mode = sys.argv[3] if len(sys.argv) > 3 else "analysis"
    one = {"analysis": one, "regions": one_regions, "intervals": one_intervals, "sort": one_sort}[mode]
    rng = np.random.default_rng(seed)
    t0, cases, recs = time.time(), 0, 0
    while time.time() - t0 < seconds:
        case_seed = int(rng.integers(0, 2 ** 31))
        try:
            recs += one(np.random.default_rng(case_seed))
        except AssertionError as e:
            print(f"MISMATCH seed={case_seed}: {e}", flush=True)
            raise
        cases += 1
    what = {"analysis": "traces, 2-3 modes each", "regions": "region sets", "intervals": "interval-algebra cases",
            "sort": "sort cases"}[mode]
    print(f"stress ok: {cases} random {what} ({recs} records), engine == oracle", flush=True)


if __name__ == "__main__":
    main()
