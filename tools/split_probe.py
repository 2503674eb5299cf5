"""Single launch vs the two-pass protocol at world size 1 (host pass -> E -> device pass ->
merge kernel, sharded.DeviceMerge with identity collectives): time per analysis on a config,
and bit-identity of the two.   python tools/split_probe.py [c5] [columns|csr]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_26576_b200 import _native as N  # noqa: E402
from paper_2603_26576_b200.configs import CONFIGS  # noqa: E402
from paper_2603_26576_b200.engine import AnalysisPlan  # noqa: E402
from paper_2603_26576_b200.sharded import DeviceMerge  # noqa: E402
from paper_2603_26576_b200.synth import generate  # noqa: E402


class Local:
    """World size 1: the collectives are identities."""
    class ReduceOp:
        MAX = None

    def all_reduce(self, t, op=None):
        return t

    def all_gather_into_tensor(self, out, inp):
        out.copy_(inp)


cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"]
dt = generate(cfg)
if (sys.argv[2] if len(sys.argv) > 2 else "columns") == "columns":
    dt = dt.columns_only()
s = torch.cuda.current_stream()
plan = AnalysisPlan(dt, N.MODE_REPORT, stream=s.cuda_stream)
merge = DeviceMerge(dt, Local(), 0, s.cuda_stream, [dt.n], [dt.m])
a = plan.run()
b = merge.step()
same = (a.elapsed == b.elapsed and np.array_equal(a.host_sum, b.host_sum) and np.array_equal(a.dev_sum[:, :3], b.dev_sum[:, :3])
        and a.host_metrics == b.host_metrics and a.device_metrics == b.device_metrics)
for name, fn in (("single launch", plan.run), ("two passes + merge", merge.step)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    print(f"{cfg.name}: {name}: {e0.elapsed_time(e1) / 10:.3f} ms per analysis")
print("identical:", same)
