#!/bin/bash
# Round evidence on a B200 (run under gpurun): every bench line (both input layouts), the
# default line's launch list, one ncu --set full capture of the analysis kernel, the
# component benches and the sanitizers.  Outputs land in gpurun_out/r/; the files judged
# are copied into profiles/ by hand.
set -x
mkdir -p gpurun_out/r
timeout 900 python bench.py > gpurun_out/r/bench_c5_columns.json 2> gpurun_out/r/bench_c5.err
timeout 900 python bench.py --layout csr --no-cpu-baseline > gpurun_out/r/bench_c5_csr.json 2>/dev/null
for c in c1 c2 c3 c4; do
  for l in columns csr; do
    timeout 600 python bench.py --config $c --layout $l --no-cpu-baseline > gpurun_out/r/bench_${c}_$l.json 2>/dev/null
  done
done
timeout 600 python bench.py --config c2 --shuffle --steps 50 --no-cpu-baseline > gpurun_out/r/bench_c2_shuffled.json 2>/dev/null
HETEFF_RAW_TRANSFER=1 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r/bench_c5_e2e_raw_transfer.json 2>/dev/null
HETEFF_FORCE_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port 29533 bench.py --no-cpu-baseline > gpurun_out/r/bench_c5_dist_world1.json 2>/dev/null
timeout 900 python bench.py --impl reference > gpurun_out/r/bench_reference_c5.json 2>/dev/null
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
    --log-file gpurun_out/r/launches_c5.csv timeout 600 python bench.py --steps 2 --warmup 3 --e2e-steps 1 --no-cpu-baseline > /dev/null 2>&1
# one analysis call of the default line = the split: host pass, device pass, merge (3 launches)
ncu --set full --clock-control none --import-source on -k regex:"analyze_kernel|merge_kernel" -c 3 -f -o gpurun_out/r/prof_analyze_c5 \
    timeout 900 python tools/one_launch.py c5 col 1 > gpurun_out/r/ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/r/prof_analyze_c5.ncu-rep "ncu --set full --clock-control none, c5 columns, one analysis call (split: host pass, device pass, merge)" \
    > gpurun_out/r/ncu_summary.txt 2>&1
ncu -i gpurun_out/r/prof_analyze_c5.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r/src_c5.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/r/src_c5.csv 40 > gpurun_out/r/ncu_lines_c5.txt 2>&1
timeout 300 python tools/bench_sort.py c2 > gpurun_out/r/sort_c2.txt 2>&1
timeout 300 python tools/bench_regions.py c4 16 3 > gpurun_out/r/regions_c4.txt 2>&1
timeout 600 python tools/bench_api.py > gpurun_out/r/api.txt 2>&1
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 30 python tools/sanitize.py shard > gpurun_out/r/san_$tool.log 2>&1
done
ls -la gpurun_out/r
