"""Per-phase clock64 breakdown of the analysis kernel (needs a -DHB_PROF build via HETEFF_LIB)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_26576_b200 import _native as N  # noqa: E402
from paper_2603_26576_b200.configs import CONFIGS  # noqa: E402
from paper_2603_26576_b200.engine import analyze_device  # noqa: E402
from paper_2603_26576_b200.synth import generate  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
dt = generate(cfg)
if len(sys.argv) > 2 and sys.argv[2] == "col":   # res columns instead of CSR offsets
    dt = dt.columns_only()
for _ in range(3):
    f = analyze_device(dt)
buf = np.zeros(1024 * 32, dtype=np.uint64)
k = N.load().heteff_prof_read(buf.ctypes.data, buf.size)
grid = N.load()  # noqa
P = buf[: k].reshape(-1, 32)
P = P[P[:, 2] > 0]
names = {0: ("c.wait_full", 2), 1: ("c.compute", 2), 16: ("host.loop+devpub", 18), 17: ("host.emit+max", 18),
         3: ("dev.phaseA", 19), 20: ("dev.barrier", 19), 4: ("dev.E+view", 19), 5: ("dev.phaseB", 19), 6: ("dev.emit", 19),
         8: ("tma.wait_empty", 12), 9: ("tma.produce", 12), 13: ("tma.claim_done", 12), 14: ("tma.claim_start", 12), 10: ("epi.work", 19), 11: ("epi.wait_info", 19)}
print(f"{cfg.name}: kernel {f.kernel_ms:.3f} ms, CTAs {P.shape[0]}, tiles/CTA {P[:, 2].mean():.1f}")
print(f"  host tiles/CTA {P[:, 18].mean():.1f}, device tiles/CTA {P[:, 19].mean():.1f}")
print(f"  single-segment device tiles run in one pass (warp 0): {P[:, 21].mean():.1f}/CTA, needing a carry fix: {P[:, 22].mean():.1f}/CTA")
for i, (nm, den) in names.items():
    per = P[:, i].astype(float) / np.maximum(P[:, den], 1)
    print(f"  {nm:14s} mean {per.mean():9.0f} cyc/tile   p10 {np.percentile(per, 10):9.0f}  p90 {np.percentile(per, 90):9.0f}")
