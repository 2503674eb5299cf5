#!/bin/bash
# Round evidence on a B200 (run under gpurun): every bench line, the C2 launch list, one
# ncu --set full capture of the analysis kernel, and the component benches.  Outputs land
# in gpurun_out/r/; the files judged are copied into profiles/ by hand.
set -x
mkdir -p gpurun_out/r
timeout 600 python bench.py > gpurun_out/r/bench_c2.json 2> gpurun_out/r/bench_c2.err
for c in c1 c3 c5; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r/bench_$c.json 2>/dev/null; done
timeout 600 python bench.py --config c4 --steps 20 --no-cpu-baseline > gpurun_out/r/bench_c4_regions.json 2>/dev/null
timeout 600 python bench.py --shuffle --steps 50 --no-cpu-baseline > gpurun_out/r/bench_c2_shuffled.json 2>/dev/null
HETEFF_FORCE_DIST=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --no-cpu-baseline > gpurun_out/r/bench_c2_dist.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r/bench_reference_c2.json 2>/dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r/launches_c2.csv \
    timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:analyze_kernel -s 3 -c 1 -f -o gpurun_out/r/prof_analyze_c2 \
    timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r/ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r/prof_analyze_c2.ncu-rep "ncu --set full --clock-control none, hb::analyze_kernel, c2, one launch" \
    > gpurun_out/r/ncu_summary.txt 2>&1
timeout 300 python tools/bench_sort.py c2 > gpurun_out/r/sort_c2.txt 2>&1
timeout 300 python tools/bench_regions.py c4 16 3 > gpurun_out/r/regions_c4.txt 2>&1
timeout 600 python tools/bench_api.py > gpurun_out/r/api.txt 2>&1
ls -la gpurun_out/r
