"""Where the per-step time goes beyond the analysis kernel (C2)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_26576_b200.configs import CONFIGS  # noqa: E402
from paper_2603_26576_b200.engine import AnalysisPlan  # noqa: E402
from paper_2603_26576_b200.synth import generate  # noqa: E402

dt = generate(CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
s = torch.cuda.current_stream().cuda_stream
plan = AnalysisPlan(dt, stream=s)
for _ in range(10):
    plan.run()
K = 200
t0 = time.perf_counter()
for _ in range(K):
    plan.run_status()
t1 = time.perf_counter()
for _ in range(K):
    plan.run()
t2 = time.perf_counter()
print(f"C call (launch + D2H + sync): {(t1 - t0) / K * 1e3:.4f} ms/step; with Findings: {(t2 - t1) / K * 1e3:.4f} ms;"
      f" kernel {plan.res.kernel_ms:.4f} ms")
