"""Load the reference-generated fixtures (tests/golden/*.json.gz)."""

from __future__ import annotations

import gzip
import json
from functools import lru_cache
from pathlib import Path

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def load(name: str):
    with gzip.open(GOLDEN / f"{name}.json.gz", "rt", encoding="utf-8") as f:
        return json.load(f)


def unhex(v):
    return None if v is None else float.fromhex(v)


def to_trace(x: dict):
    """Fixture trace -> this package's Trace (same field names as the reference)."""
    from paper_2603_26576_b200.model import (DeviceActivityKind, DeviceDecl, DeviceRecord, HostRecord, HostState,
                                             Interval, Trace)
    states = {s.value: s for s in HostState}
    kinds = {k.value: k for k in DeviceActivityKind}
    return Trace(
        host_processes=tuple(x["hp"]),
        devices=tuple(DeviceDecl(i, o) for i, o in x["dev"]),
        host_records=tuple(HostRecord(r, states[s], Interval(a, b)) for r, s, a, b in x["h"]),
        device_records=tuple(DeviceRecord(d, kinds[k], Interval(a, b), st) for d, k, a, b, st in x["d"]),
        time_unit=x["tu"],
    )
