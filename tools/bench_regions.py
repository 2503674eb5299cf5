"""Time the region passes (K5/K6) on a config trace with nested PER-RANK windows (the
shape bench.py's C4 line uses): python tools/bench_regions.py [c4] [regions] [reps]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_26576_b200.configs import CONFIGS  # noqa: E402
from paper_2603_26576_b200.engine import analyze_device, analyze_regions  # noqa: E402
from paper_2603_26576_b200.synth import generate  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
R = int(sys.argv[2]) if len(sys.argv) > 2 else 16
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
dt = generate(cfg)
S = analyze_device(dt).host_sum[:, 3].astype(np.uint64)
p = np.arange(S.size, dtype=np.uint64)
win = np.zeros((R, S.size, 2), dtype=np.uint64)
for i in range(R):
    lo = np.uint64(i) * S // np.uint64(40) + p % np.uint64(13)
    win[i, :, 0], win[i, :, 1] = lo, np.maximum(lo, S - np.uint64(i) * S // np.uint64(40))
owner = np.arange(cfg.n_devices, dtype=np.int32) // cfg.gpus_per_rank
for _ in range(reps):
    run = analyze_regions(dt, win, owner)
    print(f"{cfg.name}: {R} per-rank regions over {cfg.intervals} intervals: {run.kernel_ms:.3f} ms "
          f"({cfg.intervals / run.kernel_ms / 1e6:.3f} G intervals/s)")
