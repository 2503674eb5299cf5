"""numpy twin of the GPU trace generator (csrc/gen.cu) -- ORACLE / TEST
INFRASTRUCTURE ONLY.

Regenerates the exact arrays ``heteff_generate`` writes in HBM, so tests can
check the generator bit for bit and the ``--impl reference`` bench arm can
build its CPU sample without touching the engine.  Same counter-based RNG:
u1 = splitmix64(seed ^ (gid << 40) ^ j), u2 = splitmix64(u1 ^ C).
"""

from __future__ import annotations

import numpy as np

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_G = np.uint64(0x9E3779B97F4A7C15)
_C = np.uint64(0xD1B54A32D192ED03)
_LO = np.uint64(0xFFFFFFFF)


def mix64(z: np.ndarray) -> np.ndarray:
    z = z + _G
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def generate_side(p) -> tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
    """(start u64, end u64, res i32 local ids, kind u8) for a GenSideParams."""
    gids = np.arange(p.res_base, p.res_base + p.n_res, dtype=np.int64)
    counts = p.per_res + (gids < p.extra_below).astype(np.int64)
    total = int(counts.sum())
    assert total == p.count, (total, p.count)
    res = np.repeat(np.arange(p.n_res, dtype=np.int32), counts)
    offsets = np.zeros(p.n_res + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    j = (np.arange(total, dtype=np.int64) - np.repeat(offsets[:-1], counts)).astype(np.uint64)
    gid = np.repeat(gids, counts).astype(np.uint64)
    with np.errstate(over="ignore"):
        u1 = mix64(np.uint64(p.seed) ^ (gid << np.uint64(40)) ^ j)
        u2 = mix64(u1 ^ _C)
        gap = ((u1 & _LO) * np.uint64(p.gap_max + 1)) >> np.uint64(32)
        dur = np.uint64(1) + (((u1 >> np.uint64(32)) * np.uint64(p.dur_max)) >> np.uint64(32))
        if p.dur_scale0 > 1:
            dur = np.where(gid == 0, dur * np.uint64(p.dur_scale0), dur)
        inc = gap + dur if p.serialized else gap
        cs = np.cumsum(inc, dtype=np.uint64)
        base = np.zeros(p.n_res, dtype=np.uint64)
        nz = offsets[:-1] > 0
        base[nz] = cs[offsets[:-1][nz] - 1]
        incl = cs - np.repeat(base, counts)
        start = incl - dur if p.serialized else incl
        end = start + dur
        lo32 = u2 & _LO
        if p.is_host:
            kind = ((lo32 * np.uint64(3)) >> np.uint64(32)).astype(np.uint8)
        else:
            kind = np.where(((lo32 * np.uint64(100)) >> np.uint64(32)) < np.uint64(p.kernel_pct), 0, 1).astype(np.uint8)
    return start.astype(np.uint64), end.astype(np.uint64), res, kind


def generate(cfg, r0: int = 0, r1: int | None = None):
    """Host and device columns of ranks [r0, r1) of ``cfg`` (devices follow their owner rank)."""
    r1 = cfg.n_ranks if r1 is None else r1
    g = cfg.gpus_per_rank
    host = generate_side(cfg.host_side(r0, r1))
    dev = generate_side(cfg.dev_side(r0 * g, r1 * g))
    return host, dev
