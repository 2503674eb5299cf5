import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent)); sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from test_gpu_parity import _random_side, _engine_vs_oracle
from paper_2603_26576_b200 import _native as N
from paper_2603_26576_b200.engine import analyze_packed
from paper_2603_26576_b200.packing import PackedTrace, RecordColumns
from oracle import oracle as O
for seed in (3, 4, 5):
    rng = np.random.default_rng(seed)
    n, m = 40, 60
    h = _random_side(rng, n, rng.integers(0, 12000, size=n), host=True, zero_frac=0.01, bad_frac=0.001, span=10 ** 7)
    d = _random_side(rng, m, rng.integers(0, 12000, size=m), host=False, zero_frac=0.01, bad_frac=0.001, long_frac=0.001, span=10 ** 7)
    packed = PackedTrace(RecordColumns(*h), RecordColumns(*d), list(range(n)), list(range(m)),
                         np.arange(n, dtype=np.int32), np.arange(m, dtype=np.int32), n, m, n, m)
    for rep in range(3):
        got = analyze_packed(packed, N.MODE_VALIDATE, 0, want_lists=True, capacity=1 << 20)
        ref = O.analyze(h, d, n, m, mode=2, cap=1 << 20)
        a, b = set(got.lists[7].tolist()), set(ref.lists[7].tolist())
        print(seed, rep, "E", got.host_elapsed, ref.host_elapsed, "true max", int(h[1].max()), "late", len(a), len(b), "extra", sorted(a - b)[:5], "missing", sorted(b - a)[:5])
        for i in sorted(a - b)[:3]:
            print("   rec", i, "dev", int(d[2][i]), "s", int(d[0][i]), "e", int(d[1][i]))
