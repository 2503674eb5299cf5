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
for _ in range(3):
    f = analyze_device(dt)
buf = np.zeros(1024 * 16, dtype=np.uint64)
k = N.load().heteff_prof_read(buf.ctypes.data, buf.size)
grid = N.load()  # noqa
P = buf[: k].reshape(-1, 16)
P = P[P[:, 2] > 0]
names = {0: "c.wait_full", 1: "c.compute", 3: "c.phaseA", 4: "c.bar+view", 5: "c.phaseB", 6: "c.emit",
         8: "p.wait_empty", 9: "p.produce", 10: "p.epilogue"}
print(f"{cfg.name}: kernel {f.kernel_ms:.3f} ms, CTAs {P.shape[0]}, tiles/CTA {P[:, 2].mean():.1f}")
for i, nm in names.items():
    per = P[:, i].astype(float) / np.maximum(P[:, 2 if i < 8 else 12], 1)
    print(f"  {nm:14s} mean {per.mean():9.0f} cyc/tile   p10 {np.percentile(per, 10):9.0f}  p90 {np.percentile(per, 90):9.0f}")
