"""A few analysis launches of one config (for ncu captures): python tools/one_launch.py c2 [csr|col] [launches]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_26576_b200.configs import CONFIGS  # noqa: E402
from paper_2603_26576_b200.engine import analyze_device  # noqa: E402
from paper_2603_26576_b200.synth import generate  # noqa: E402

dt = generate(CONFIGS[sys.argv[1]])
if len(sys.argv) > 2 and sys.argv[2] == "col":
    dt = dt.columns_only()
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 3):
    f = analyze_device(dt)
print(sys.argv[1:], f.status, f.kernel_ms)
