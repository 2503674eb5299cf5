"""The BASELINE.json workload configs as synthetic-trace shapes.

``BASELINE.json`` names five configs (C1..C5); it does not fix their
host/device split or timing distributions, so the shapes below follow
SURVEY.md section 8(d): host chains per rank with gap ~ U[0,20] ns and
duration ~ U[1,200] ns (the reference corpus shape, tests/strategies.py:52-59)
and device records from an arrival process sized so a device's span matches
its owner rank's host span, with mean overlap depth S.

Generation runs on the GPU (``heteff_generate``, csrc/gen.cu); the numpy twin
in ``oracle/gen.py`` reproduces every array bit for bit.
"""

from __future__ import annotations

from dataclasses import dataclass

HOST_GAP_MAX = 20
HOST_DUR_MAX = 200
HOST_MEAN_STEP = (HOST_GAP_MAX / 2) + (1 + HOST_DUR_MAX) / 2   # 110.5 ns


@dataclass(frozen=True)
class GenSideParams:
    """Mirror of ``heteff_gen_side`` (include/heteff_b200.h)."""

    seed: int
    n_res: int
    res_base: int
    per_res: int
    extra_below: int
    serialized: int
    count: int
    gap_max: int
    dur_max: int
    dur_scale0: int
    kernel_pct: int
    is_host: int


@dataclass(frozen=True)
class Config:
    name: str
    description: str
    n_ranks: int
    gpus_per_rank: int
    host_records: int
    dev_records: int
    overlap: int             # mean device overlap depth S (1 = none)
    serialized_dev: bool     # device records form a serialized chain (one stream)
    dur_scale0: int          # duration multiplier of device 0 (imbalance)
    seed: int
    kernel_pct: int = 80

    @property
    def n_devices(self) -> int:
        return self.n_ranks * self.gpus_per_rank

    @property
    def intervals(self) -> int:
        return self.host_records + self.dev_records

    def _split(self, total: int, k: int) -> tuple[int, int]:
        return total // k, total % k

    def _count(self, per: int, extra: int, lo: int, hi: int) -> int:
        return per * (hi - lo) + max(0, min(hi, extra) - min(lo, extra))

    def block_intervals(self, r0: int, r1: int) -> int:
        """Records of ranks [r0, r1) and the devices they own (one shard of a rank-sharded run)."""
        g = self.gpus_per_rank
        return self.host_side(r0, r1).count + self.dev_side(r0 * g, r1 * g).count

    def host_side(self, r0: int = 0, r1: int | None = None) -> GenSideParams:
        r1 = self.n_ranks if r1 is None else r1
        per, extra = self._split(self.host_records, self.n_ranks)
        return GenSideParams(self.seed, r1 - r0, r0, per, extra, 1, self._count(per, extra, r0, r1),
                             HOST_GAP_MAX, HOST_DUR_MAX, 1, 0, 1)

    def dev_side(self, d0: int = 0, d1: int | None = None) -> GenSideParams:
        d1 = self.n_devices if d1 is None else d1
        per, extra = self._split(self.dev_records, self.n_devices)
        span = (self.host_records / self.n_ranks) * HOST_MEAN_STEP      # expected host span per rank
        step = span / max(per, 1)                                        # mean record spacing per device
        if self.serialized_dev:
            gap_max = max(1, int(round(2 * 0.2 * step)))
            dur_max = max(1, int(round(2 * 0.8 * step)))
        else:
            gap_max = max(1, int(round(2 * step)))
            dur_max = max(1, int(round(2 * self.overlap * step)))
        return GenSideParams(self.seed ^ 0xDE71CE5EED000000, d1 - d0, d0, per, extra, int(self.serialized_dev),
                             self._count(per, extra, d0, d1), gap_max, dur_max, self.dur_scale0,
                             self.kernel_pct, 0)


CONFIGS = {
    "c1": Config("c1", "paper synthetic benchmark trace: 4 MPI ranks x 1 GPU, 1e5 intervals, imbalanced kernels",
                 4, 1, 50_000, 50_000, 1, False, 10, 0x5EED10),
    "c2": Config("c2", "1024 ranks x 1 GPU, 1e8 intervals, serialized stream",
                 1024, 1, 50_000_000, 50_000_000, 1, True, 1, 0x5EED20),
    "c3": Config("c3", "256 ranks x 4 GPUs x 8 concurrent streams, 5e8 heavily overlapping intervals",
                 256, 4, 50_000_000, 450_000_000, 8, False, 1, 0x5EED30),
    "c4": Config("c4", "1024 ranks x 1 GPU, 1e9 intervals (regions / overlap metrics: see DESIGN.md)",
                 1024, 1, 500_000_000, 500_000_000, 4, False, 1, 0x5EED40),
    "c5": Config("c5", "4096 ranks x 4 GPUs, 2e9 intervals, rank-sharded",
                 4096, 4, 1_000_000_000, 1_000_000_000, 4, False, 1, 0x5EED50),
}


def scaled(cfg: Config, ranks: int) -> Config:
    """The first ``ranks`` ranks of ``cfg`` with the same per-rank shape (a rank shard)."""
    per_h = cfg.host_records // cfg.n_ranks
    per_d = cfg.dev_records // cfg.n_devices
    return Config(f"{cfg.name}[:{ranks}]", cfg.description, ranks, cfg.gpus_per_rank, per_h * ranks,
                  per_d * ranks * cfg.gpus_per_rank, cfg.overlap, cfg.serialized_dev, cfg.dur_scale0, cfg.seed,
                  cfg.kernel_pct)
