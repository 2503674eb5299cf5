"""bench.py's contract, on the CPU: the reference arm (--impl reference, the C oracle port on
the host cores) prints exactly one JSON line on stdout with the keys the driver reads."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import gpu_available

ROOT = Path(__file__).resolve().parent.parent

KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def test_reference_arm_prints_one_json_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1", "--warmup", "0",
                          "--cpu-sample", "2e5", "--ref-pkg-intervals", "2e5"], capture_output=True, text=True,
                         timeout=600, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True and d["n_gpus"] == 1
    assert d["unit"] == "intervals/s" and d["config"]["workload"] == "c5" and d["scaling"] == "strong"
    assert d["config"]["intervals"] == 2_000_000_000
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    # the unmodified reference package itself, beside the port, identical on the same shard
    rp = d["reference_pkg"]
    if "unavailable" not in rp:
        assert rp["one_core"]["cores"] == 1 and rp["one_core"]["value"] > 0 and rp["all_cores"]["value"] > 0
        assert rp["port_identical"] is True


def test_reference_arm_does_not_load_the_engine():
    """The reference arm must not map the product's native libraries (the driver checks
    which .so files the arm's process loaded)."""
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0', "
            "'--cpu-sample', '1e5', '--ref-pkg-intervals', '0'];\n"
            "try:\n    runpy.run_path('bench.py', run_name='__main__')\nexcept SystemExit:\n    pass\n"
            "maps = open('/proc/self/maps').read()\n"
            "assert 'libheteff_b200' not in maps and '_pack.' not in maps, 'engine library loaded'\n"
            "assert not [m for m in sys.modules if m.startswith('paper_2603_26576_b200')], 'engine package imported'\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]


def test_config_dicts_of_both_arms_are_identical():
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    for argv in ([], ["--config", "c2"], ["--config", "c4"], ["--config", "c3", "--scaling", "strong"]):
        ap_args = _parse(b, argv)
        for world in (1, 2, 8):
            cfg = b._global_config(ap_args, world)
            ref = b._config_dict(ap_args, cfg, world)
            assert ref == b._config_dict(ap_args, cfg, world) and ref["workload"] == ap_args.config
    a = _parse(b, [])
    assert b._scaling(a) == "strong" and b._global_config(a, 8).intervals == 2_000_000_000
    assert [b._rank_block(b._global_config(a, 8), 8, r) for r in (0, 7)] == [(0, 512), (3584, 4096)]
    w = _parse(b, ["--config", "c2"])
    assert b._scaling(w) == "weak" and b._global_config(w, 4).intervals == 4 * 100_000_000


def _parse(b, argv):
    import argparse
    ns = argparse.Namespace(config="c5", scaling=None, layout="columns", e2e_layout="csr", shuffle=False, regions=None)
    i = 0
    while i < len(argv):
        setattr(ns, argv[i][2:], argv[i + 1])
        i += 2
    return ns


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_engine_arm_prints_one_json_line_with_roofline_and_e2e():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "5", "--warmup", "3", "--e2e-steps", "2",
                          "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert (KEYS - {"impl", "cpu_baseline"}) | {"roofline", "clocks", "gpu_launches"} <= set(d)
    assert d["gpu_launches"] > 0 and d["value"] > 0 and d["scaling"] == "strong"
    assert d["config"]["workload"] == "c5" and d["config"]["intervals"] == 2_000_000_000
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.2 and r["achieved"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0 and d["e2e"]["value"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]

