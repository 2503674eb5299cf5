"""Time K3 (GPU radix sort into canonical order) on a shuffled config side."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_26576_b200.configs import CONFIGS  # noqa: E402
from paper_2603_26576_b200.engine import DeviceTrace, analyze_device, sort_records  # noqa: E402
from paper_2603_26576_b200.synth import generate  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
dt = generate(cfg)
g = torch.Generator(device="cuda").manual_seed(1)
p = torch.randperm(dt.dev_count, device="cuda", generator=g)
cols = [x[p] for x in (dt.d_start, dt.d_end, dt.d_res, dt.d_kind)]
del p
for _ in range(2):
    r = sort_records(*cols)
ms = []
for _ in range(5):
    r = sort_records(*cols)
    ms.append(r.ms)
n = dt.dev_count
best = min(ms)
print(f"{cfg.name}: sort {n} device records: {best:.3f} ms  ({n / best / 1e6:.3f} G rec/s), start_sorted={r.start_sorted} "
      f"key_bits={r.key_bits} passes={r.passes} wide={r.wide}")
# sorted-in-place input: the analysis of the sorted columns == the generated canonical trace
sh = DeviceTrace(dt.h_start, dt.h_end, dt.h_res, dt.h_kind, r.start, r.end, r.res, r.kind, dt.n, dt.m)
a, b = analyze_device(dt), analyze_device(sh)
print("analysis identical:", (a.dev_sum == b.dev_sum).all() and a.device_metrics == b.device_metrics)
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
sh2 = DeviceTrace(dt.h_start, dt.h_end, dt.h_res, dt.h_kind, *cols, dt.n, dt.m)
analyze_device(sh2, sort_if_needed=True)
t0.record()
for _ in range(3):
    f = analyze_device(sh2, sort_if_needed=True)
t1.record(); torch.cuda.synchronize()
print(f"analyze(unsorted, sort_if_needed): {t0.elapsed_time(t1) / 3:.3f} ms per call, status {f.status}")
# a globally time-ordered event log: all devices interleaved by start
o = torch.argsort(dt.d_start, stable=True)
cols = [x[o] for x in (dt.d_start, dt.d_end, dt.d_res, dt.d_kind)]
del o
for _ in range(2):
    r = sort_records(*cols)
ms = [sort_records(*cols).ms for _ in range(5)]
print(f"{cfg.name}: sort time-ordered log: {min(ms):.3f} ms ({n / min(ms) / 1e6:.3f} G rec/s), "
      f"start_sorted={r.start_sorted} passes={r.passes}")
