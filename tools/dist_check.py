"""Multi-rank check of the device-resident merge protocol on ONE GPU (test infrastructure).

Launched as ``python -m torch.distributed.run --nproc-per-node W tools/dist_check.py CFG RANKS``:
every rank binds cuda:0 (NCCL refuses two ranks on one device, so the protocol's two
collectives go through gloo on host copies -- the only difference from the NCCL run),
generates its rank shard, runs ``sharded.DeviceMerge.step`` (host pass, all-reduce MAX
of E, device pass with the global E read from device memory, all-gather of the result
blocks, merge kernel).  Rank 0 compares the merged report with one single-process
analysis of the whole trace and prints one JSON line."""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_26576_b200 import _native as N  # noqa: E402
from paper_2603_26576_b200.configs import CONFIGS, scaled  # noqa: E402
from paper_2603_26576_b200.engine import analyze_device  # noqa: E402
from paper_2603_26576_b200.sharded import DeviceMerge, HostCollectives  # noqa: E402
from paper_2603_26576_b200.synth import generate  # noqa: E402


def main():
    cfg_name, ranks = sys.argv[1], int(sys.argv[2])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    cfg = scaled(CONFIGS[cfg_name], ranks)
    per = ranks // world
    n_of = [per + (1 if r < ranks % world else 0) for r in range(world)]   # uneven shards allowed
    r0 = sum(n_of[:rank])
    dt = generate(cfg, r0, r0 + n_of[rank], device=0)
    stream = torch.cuda.current_stream(0).cuda_stream
    merge = DeviceMerge(dt, HostCollectives(dist), 0, stream, n_of, [k * cfg.gpus_per_rank for k in n_of])
    f = merge.step()
    f = merge.step()                       # a second step: the workspace resets correctly
    if rank == 0:
        ref = analyze_device(generate(cfg, device=0), N.MODE_REPORT, stream=stream, device=0)
        same = (f.status == ref.status and f.elapsed == ref.elapsed and
                np.array_equal(f.host_sum, ref.host_sum) and np.array_equal(f.dev_sum, ref.dev_sum) and
                f.host_metrics == ref.host_metrics and f.device_metrics == ref.device_metrics)
        print(json.dumps({"world": world, "config": cfg.name, "shards": n_of, "status": f.status,
                          "elapsed": f.elapsed, "identical_to_single_process": bool(same)}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
