"""The multi-GPU merge protocol with real processes (torch.distributed.run, W ranks)
on the one GPU available: every rank's shard goes through the real kernels and the
merged report must equal the single-process analysis bit for bit (tools/dist_check.py)."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.parametrize("world,cfg,ranks,port", [(2, "c2", 64, 29611), (3, "c3", 16, 29612), (4, "c5", 10, 29613)])
def test_merge_protocol_across_processes(world, cfg, ranks, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "tools" / "dist_check.py"), cfg, str(ranks)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["world"] == world and line["status"] == 0
    assert line["identical_to_single_process"], line


@pytest.mark.parametrize("cfg,world,port,scaling", [("c2", 2, 29621, "weak"), ("c1", 2, 29622, "weak"),
                                                    ("c2", 8, 29623, "weak"), ("c2", 2, 29624, "strong"),
                                                    ("c1", 3, 29625, "strong")])
def test_bench_under_torchrun(cfg, world, port, scaling):
    """bench.py exactly as the driver's scaling run launches it (torchrun, W ranks), with
    the collectives on gloo so the ranks can share the one GPU: it must finish and print
    one JSON line for the whole job."""
    import os

    env = dict(os.environ, HETEFF_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py"), "--gpus", str(world),
           "--config", cfg, "--scaling", scaling, "--steps", "5", "--warmup", "3", "--e2e-steps", "2",
           "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=str(ROOT), env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == world and d["value"] > 0 and d["e2e"]["value"] > 0 and d["scaling"] == scaling
    from paper_2603_26576_b200.configs import CONFIGS
    c = CONFIGS[cfg]
    if scaling == "weak":   # every rank a C-sized block of a world-times larger trace
        import types
        sys.path.insert(0, str(ROOT))
        import bench
        g = bench._global_config(types.SimpleNamespace(config=cfg, scaling=scaling), world)
        assert d["config"]["intervals"] == world * c.intervals == g.intervals
        # rank 0's block: its ranks hold the remainder records of the larger trace
        assert d["roofline"]["per_gpu_intervals"] == g.block_intervals(0, g.n_ranks // world)
    else:                   # the one trace split by rank blocks (rank 0's block: the first n // world ranks)
        assert d["config"]["intervals"] == c.intervals
        assert d["roofline"]["per_gpu_intervals"] == c.block_intervals(0, c.n_ranks // world)


def test_bench_gpus_without_torchrun_spawns_the_ranks():
    """--gpus N without torchrun re-launches itself under torch.distributed.run (N ranks)."""
    import os

    env = dict(os.environ, HETEFF_DIST_BACKEND="gloo")
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--config", "c1", "--steps", "3", "--warmup", "3",
           "--e2e-steps", "1", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=str(ROOT), env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    assert json.loads(lines[0])["n_gpus"] == 2
