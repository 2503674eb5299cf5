"""Differential stress of the front ends against the REFERENCE package (test
infrastructure; runs only where /root/reference exists, i.e. the build container):
random native trace documents -- valid and deliberately broken -- through this package's
read_trace and the reference's, comparing records, declarations, error texts and
write_trace bytes.  Usage: python tools/frontend_stress.py SECONDS [SEED]"""
import json
import random
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, "/root/reference/pkg/src")
import heteff as R  # noqa: E402  (the reference)

import paper_2603_26576_b200 as H  # noqa: E402


def doc(rng):
    hosts, devs = [], []
    for i in range(rng.randrange(0, 5)):
        recs = []
        t = rng.randrange(0, 1000)
        for _ in range(rng.randrange(0, 40)):
            d = rng.choice([0, 1, 5, 100, 2 ** 33])
            a = rng.choice([t, rng.randrange(0, t + 2)])   # some out of order
            recs.append({"state": rng.choice(["useful", "offload", "mpi"]), "start": a, "end": a + d})
            t = a + d + rng.randrange(0, 10)
        hosts.append({"rank": rng.choice([i, i * 7, 2 ** 40 + i]), "records": recs})
    for i in range(rng.randrange(0, 5)):
        recs = []
        for _ in range(rng.randrange(0, 40)):
            a = rng.randrange(0, 10 ** 6)
            r = {"kind": rng.choice(["kernel", "memory"]), "start": a, "end": a + rng.choice([0, 1, 50, 10 ** 5])}
            if rng.random() < 0.5:
                r["stream"] = rng.randrange(0, 4)
            recs.append(r)
        e = {"id": rng.choice([i, 100 + i]), "records": recs}
        if rng.random() < 0.5:
            e["owner_rank"] = rng.randrange(0, 5)
        devs.append(e)
    d = {"version": 1, "time_unit": "ns", "hosts": hosts, "devices": devs}
    if rng.random() < 0.15:   # break it somewhere
        how = rng.randrange(6)
        if how == 0:
            d["version"] = 2
        elif how == 1 and hosts and hosts[0]["records"]:
            hosts[0]["records"][0]["start"] = -1
        elif how == 2 and devs and devs[0]["records"]:
            devs[0]["records"][0]["kind"] = "idle"
        elif how == 3:
            d["extra"] = 1
        elif how == 4 and hosts:
            del hosts[0]["rank"]
        elif how == 5 and devs and devs[0]["records"]:
            devs[0]["records"][0]["end"] = 2 ** 64
    return json.dumps(d)


NAMES = ["kernel_a", "cudaLaunchKernel", "MPI_Wait", "Memcpy HtoD", "other", "k", "MPI_Allreduce"]


def events(rng):
    evs = []
    for _ in range(rng.randrange(0, 60)):
        e = {"name": rng.choice(NAMES), "cat": rng.choice(["cuda", "mpi", "cpu"]), "ph": rng.choice(["X", "X", "X", "B"]),
             "ts": rng.choice([rng.randrange(0, 10 ** 6), rng.randrange(0, 10 ** 6) + 0.5, rng.randrange(0, 10 ** 4) / 4]),
             "dur": rng.choice([0, 1, 3, 2.25, 100]), "pid": rng.randrange(0, 4), "tid": rng.randrange(0, 3)}
        if rng.random() < 0.05:
            del e[rng.choice(["ts", "dur", "pid", "name"])]
        evs.append(e)
    return json.dumps({"traceEvents": evs} if rng.random() < 0.8 else evs)


def mapping(rng):
    rules = []
    for _ in range(rng.randrange(1, 5)):
        key = rng.choice(["name_contains", "name_equals", "category_contains", "category_equals"])
        val = rng.choice(NAMES + ["cuda", "mpi", "MPI_", "Memcpy"])
        rules.append({key: val, "target": rng.choice(["useful", "offload", "mpi", "kernel", "memory"]),
                      "resource": rng.choice(["pid", "tid", 0, 3])})
    return json.dumps({"default_policy": rng.choice(["drop", "error"]), "rules": rules})


def outcome(mod, ev, mp):
    try:
        t, w = mod.import_mapped(ev, mod.read_mapping(mp))
        return ("ok", repr(t), list(w), mod.write_trace(t))
    except Exception as x:   # noqa: BLE001
        return (type(x).__name__, str(x))


def same(a, b):
    if type(a).__name__ != type(b).__name__:
        return False
    return repr(a) == repr(b)


def main():
    seconds = float(sys.argv[1]) if len(sys.argv) > 1 else 30
    rng = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    t0, n = time.time(), 0
    while time.time() - t0 < seconds:
        text = doc(rng)
        try:
            ref = R.read_trace(text)
            ref_err = None
        except Exception as x:   # noqa: BLE001
            ref, ref_err = None, (type(x).__name__, str(x))
        try:
            got = H.read_trace(text)
            got_err = None
        except Exception as x:   # noqa: BLE001
            got, got_err = None, (type(x).__name__, str(x))
        assert ref_err == got_err, (text, ref_err, got_err)
        if ref is not None:
            assert same(ref, got), text
            assert R.write_trace(ref) == H.write_trace(got), text
        ev, mp = events(rng), mapping(rng)
        ro, go = outcome(R, ev, mp), outcome(H, ev, mp)
        assert ro == go, (ev, mp, ro[:2], go[:2])
        n += 1
    print(f"frontend stress ok: {n} random trace documents and {n} random (event timeline, mapping) pairs: "
          "read_trace / write_trace / import_mapped identical to the reference (records, warnings, error texts, bytes)")


if __name__ == "__main__":
    main()
